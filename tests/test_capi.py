"""CPU: the C-ABI library loads, exports every function include/rgo/capi.h
declares, validates like the reference, and refuses to compute without a GPU
(no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

from conftest import ROOT


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "rgo", "capi.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rgo_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported(rgo):
    lib = rgo._lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
        assert s in rgo._lib.SIGNATURES, f"{s} missing from the Python binding"


def test_keep_threshold_via_capi(rgo):
    lib = rgo._lib.lib()
    t, f = C.c_uint64(), C.c_float()
    assert lib.rgo_keep_threshold(0.9, C.byref(t), C.byref(f)) == 0
    assert t.value == 3865470464 and abs(f.value - 0.9) < 1e-7
    assert lib.rgo_keep_threshold(1.0, C.byref(t), None) == 0 and t.value == 1 << 32
    assert lib.rgo_keep_threshold(1.5, C.byref(t), None) == rgo._lib.RGO_EINVAL
    assert b"keep_prob" in lib.rgo_last_error()


def test_threshold_python_mirror_matches_oracle(rgo, golden):
    for p, thr in golden["thresholds"].items():
        assert rgo.KeepThreshold(float(p)).threshold() == thr


def test_validation_errors(rgo):
    lib = rgo._lib.lib()
    d = rgo._lib.mask_desc(0, 1, 1, 7, 0, 0, 1 << 31)
    assert lib.rgo_mask_generate(d, None, 0, None) == rgo._lib.RGO_EINVAL
    assert b"zero elements" in lib.rgo_last_error()
    d = rgo._lib.mask_desc(1, 1, 4, 17, 0, 0, 1 << 31)
    assert lib.rgo_mask_generate(d, None, 0, None) == rgo._lib.RGO_EINVAL
    assert b"rounds" in lib.rgo_last_error()
    # capacity guard (mask.hpp:148-155): message carries "bytes" and "guard"
    with pytest.raises(ValueError) as e:
        rgo.generate_mask(rgo.MaskLayout(1, 96, 1 << 17), rgo.KeepThreshold(0.5), 7)
    assert "bytes" in str(e.value) and "guard" in str(e.value)
    with pytest.raises(ValueError):
        rgo.generate_mask(rgo.MaskLayout(1, 1, 4), rgo.KeepThreshold(0.5), 0)
    with pytest.raises(ValueError):
        rgo.MaskLayout(1, 2, 4).linear_index(0, 2, 0, 0)


def test_no_cpu_fallback(rgo):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(rgo._lib.RgoError) as e:
        rgo.generate_mask(rgo.MaskLayout(1, 1, 16, 3), rgo.KeepThreshold(0.9), 10)
    assert e.value.code == rgo._lib.RGO_ENODEV


def test_mask_file_roundtrip_and_errors(rgo, tmp_path, mask_blobs, golden):
    # test_mask.cpp:172-219 with reference bits from the golden fixture
    m = next(x for x in golden["masks"] if x["seed"] == 31337)
    mask = rgo.DropoutMask(rgo.MaskLayout(m["batch"], m["heads"], m["seq"], m["seed"], m["base_offset"]),
                           rgo.KeepThreshold(m["p"]).keep_prob, m["rounds"], mask_blobs[m["blob"]])
    p = tmp_path / "m.bin"
    rgo.save_mask(mask, p)
    assert p.stat().st_size == 40 + (mask.layout.elem_count() + 7) // 8
    r = rgo.load_mask(p)
    assert r.layout == mask.layout and r.keep_prob == mask.keep_prob and r.rounds == mask.rounds
    assert (r.bits == mask.bits).all()
    raw = bytearray(p.read_bytes())
    raw[0] = ord("X")
    (tmp_path / "bad.bin").write_bytes(bytes(raw))
    with pytest.raises(rgo._lib.RgoIOError):
        rgo.load_mask(tmp_path / "bad.bin")
    (tmp_path / "short.bin").write_bytes(p.read_bytes()[:-1])
    with pytest.raises(rgo._lib.RgoIOError):
        rgo.load_mask(tmp_path / "short.bin")


def test_element_source_carry(rgo):
    # test_mask.cpp:23-61
    lay = rgo.MaskLayout(1, 2, 4)
    assert rgo.element_source(lay, 0) == (rgo.PhiloxCounter(0, 0, 0, 0), 0)
    assert rgo.element_source(lay, 7) == (rgo.PhiloxCounter(1, 0, 0, 0), 3)
    with pytest.raises(ValueError):
        rgo.element_source(lay, 32)
    lay = rgo.MaskLayout(1, 4, 65536, 0, 0xFFFFFFFF)
    c, lane = rgo.element_source(lay, 1 << 33)
    assert lane == 0 and c.c1 == 1 and c.c0 == ((0xFFFFFFFF + (1 << 31)) & 0xFFFFFFFF)


def _block_desc(rgo, keep_prob=0.9, rng_block=0):
    d = rgo._lib.block_desc()
    d.batch, d.seq, d.heads, d.head_dim, d.ffn, d.gated = 1, 256, 2, 128, 256, 1
    d.keep_prob, d.rounds = keep_prob, 10
    d.rng_launch = rgo._lib.launch(0, rng_block, 0, 0)
    return d


def test_block_create_validation(rgo):
    """rgo_block_create rejects, before touching any buffer or device: a keep
    probability whose float threshold is 2^32 or 0 (the in-GEMM queue's 32-bit
    compare cannot express it), and an unsupported in-GEMM RNG-warp count."""
    lib = rgo._lib.lib()
    h = C.c_void_p()
    bufs = rgo._lib.block_buffers()
    for kp in (0.99999999, 1e-12):
        assert lib.rgo_block_create(_block_desc(rgo, kp), bufs, 2, C.byref(h)) == rgo._lib.RGO_EINVAL
        assert b"threshold" in lib.rgo_last_error()
    for rw in (10, 256, 5):
        assert lib.rgo_block_create(_block_desc(rgo, 0.9, rw), bufs, 2, C.byref(h)) == rgo._lib.RGO_EINVAL
        assert b"RNG warps" in lib.rgo_last_error()
    # the same launch shape is a mechanism-A (STREAMS) mask-kernel block size: not rejected there
    assert lib.rgo_block_create(_block_desc(rgo, 0.9, 256), bufs, 1, C.byref(h)) == rgo._lib.RGO_EINVAL
    assert b"missing buffer" in lib.rgo_last_error()


def test_fnv1a64_via_capi(rgo, golden, mask_blobs):
    """The C-ABI checksum equals the golden fixtures' FNV-1a-64."""
    import numpy as np
    for m in [x for x in golden["masks"] if x.get("blob")][:8]:
        assert f"{rgo.mask.fnv1a64(mask_blobs[m['blob']]):016x}" == m["fnv"]
    assert rgo.mask.fnv1a64(np.zeros(0, np.uint8)) == 0xcbf29ce484222325


def test_block_create_tp_validation(rgo):
    """rgo_block_create_tp (tensor-parallel block) rejects bad plans before touching any buffer or
    device: tp size/rank, tp_degree not dividing nH (capacity.hpp:22-23), per-rank widths that
    break the GEMM tiling, missing peer buffers, and peer[rank] not being the rank's own y1/x."""
    lib = rgo._lib.lib()
    E = rgo._lib.RGO_EINVAL
    h = C.c_void_p()
    bufs = rgo._lib.block_buffers()
    d = _block_desc(rgo)
    d.heads, d.seq, d.ffn = 4, 512, 512
    tp = rgo._lib.block_tp()
    for size, rank in ((1, 0), (9, 0), (2, 2)):
        tp.size, tp.rank = size, rank
        assert lib.rgo_block_create_tp(d, bufs, C.byref(tp), 2, C.byref(h)) == E
        assert b"size" in lib.rgo_last_error()
    tp.size, tp.rank = 3, 0
    assert lib.rgo_block_create_tp(d, bufs, C.byref(tp), 2, C.byref(h)) == E
    assert b"tp_degree must divide nH" in lib.rgo_last_error()
    tp.size = 4  # one head (128 columns) per rank
    d.ffn = 256  # ffn/size = 64: not a multiple of 128
    assert lib.rgo_block_create_tp(d, bufs, C.byref(tp), 2, C.byref(h)) == E
    assert b"(ffn/size)" in lib.rgo_last_error()
    d.ffn = 512
    assert lib.rgo_block_create_tp(d, bufs, C.byref(tp), 2, C.byref(h)) == E
    assert b"missing peer buffer" in lib.rgo_last_error()
    for t in range(4):
        tp.peer_part[t] = tp.peer_y1[t] = tp.peer_x[t] = 0x1000 * (t + 1)
    assert lib.rgo_block_create_tp(d, bufs, C.byref(tp), 2, C.byref(h)) == E
    assert b"this rank's y1/x" in lib.rgo_last_error()


def test_ipc_and_large_head_dim_validation(rgo):
    lib = rgo._lib.lib()
    E = rgo._lib.RGO_EINVAL
    off = C.c_uint64()
    assert lib.rgo_ipc_handle(None, None, C.byref(off)) == E
    assert lib.rgo_ipc_open(None, None) == E
    assert lib.rgo_ipc_close(None) == E
    # the drop-in attention accepts any head_dim up to 1024 (K5g above 128); beyond: invalid
    ad = rgo._lib.attn_host_desc(1, 8, 1025, 0, 1.0, 0, 0, 7, 0)
    x = (C.c_float * 16)()
    assert lib.rgo_attention_host(C.byref(ad), x, x, x, None, 0, x) == E
    assert b"1024" in lib.rgo_last_error()
