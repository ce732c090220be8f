"""ctypes wrapper of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Loads oracle/liboracle.so (C restatement of the reference, rgo_oracle.c) and,
when present, oracle/_ref/librgo_ref.so (the reference itself compiled from
/root/reference/proj/include).  Imported only by tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs, as the checker or the
CPU baseline -- never by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "librgo_ref.so")

_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C")


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


_o = None
_r = None


def lib():
    global _o
    if _o is None:
        if not os.path.exists(ORACLE_SO):
            build()
        d = C.CDLL(ORACLE_SO)
        d.oracle_philox_block.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.c_int, _u32p]
        d.oracle_keep_threshold.argtypes = [C.c_double, C.POINTER(C.c_uint64), C.POINTER(C.c_float)]
        d.oracle_keep_bit_direct.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_uint64]
        d.oracle_generate_mask.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                           C.c_uint, _u8p, C.c_uint64]
        d.oracle_fill_uniform.argtypes = [C.c_uint64, C.c_uint32, _f32p, C.c_uint64]
        d.oracle_fill_uniform.restype = None
        d.oracle_attention.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, _f32p, _f32p, _f32p, C.c_int,
                                       C.c_uint64, C.c_uint64, C.c_uint64, C.c_float, C.c_int,
                                       C.c_void_p, C.c_uint32, C.c_uint32, _f32p]
        d.oracle_fnv1a64.argtypes = [_u8p, C.c_uint64]
        d.oracle_fnv1a64.restype = C.c_uint64
        _o = d
    return _o


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference compiled in place (oracle/_ref); None if unavailable."""
    global _r
    if _r is None:
        if not os.path.exists(REF_SO):
            if os.path.isdir("/root/reference/proj/include/rgo"):
                build()
            if not os.path.exists(REF_SO):
                return None
        d = C.CDLL(REF_SO)
        d.ref_philox_block.argtypes = [C.c_uint32, C.c_uint32, _u32p, C.c_int, _u32p]
        d.ref_keep_threshold.argtypes = [C.c_double, C.POINTER(C.c_uint64), C.POINTER(C.c_float)]
        d.ref_generate_mask.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64,
                                        C.c_double, C.c_int, C.c_uint, _u8p, C.c_uint64]
        d.ref_random_attention_input.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint64,
                                                 _f32p, _f32p, _f32p]
        d.ref_random_attention_input.restype = None
        d.ref_attention.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, _f32p, _f32p, _f32p, C.c_int,
                                    C.c_uint64, C.c_uint64, C.c_double, C.c_int, _f32p]
        d.ref_attention_decoupled.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, _f32p, _f32p, _f32p, _u8p,
                                              C.c_uint64, C.c_double, C.c_int, _f32p]
        d.ref_gemm_shapes.argtypes = [C.c_uint32] * 5 + [np.ctypeslib.ndpointer(np.uint64, flags="C")]
        d.ref_philox_test_vectors.argtypes = [C.c_uint64, C.c_int, C.c_int, _u32p, _u32p, _i32p, _u32p]
        d.ref_philox_test_vectors.restype = None
        _r = d
    return _r


# ------------------------------------------------------------------ helpers
def philox_block(key, ctr, rounds):
    out = np.zeros(4, np.uint32)
    rc = lib().oracle_philox_block(int(key[0]), int(key[1]), np.asarray(ctr, np.uint32), rounds, out)
    if rc != 0:
        raise ValueError("philox_block: rounds must be in [1,16]")
    return tuple(int(x) for x in out)


def keep_threshold(p):
    t = C.c_uint64()
    f = C.c_float()
    if lib().oracle_keep_threshold(p, C.byref(t), C.byref(f)) != 0:
        raise ValueError("keep_prob must be in [0,1]")
    return t.value, f.value


def generate_mask(batch, heads, seq, seed, base_offset, p, rounds, workers=0):
    n = batch * heads * seq * seq
    thr, _ = keep_threshold(p)
    out = np.zeros((n + 7) // 8, np.uint8)
    if workers == 0:
        workers = os.cpu_count() or 1
    rc = lib().oracle_generate_mask(n, seed, base_offset, thr, rounds, workers, out, out.size)
    if rc != 0:
        raise ValueError(f"oracle_generate_mask rc={rc}")
    return out


def uniform(seed, stream, n):
    out = np.empty(n, np.float32)
    lib().oracle_fill_uniform(seed, stream, out, n)
    return out


def random_attention_input(slices, seq, head_dim, seed):
    n = slices * seq * head_dim
    return uniform(seed, 1, n), uniform(seed, 2, n), uniform(seed, 3, n)


def attention(q, k, v, slices, seq, head_dim, mode=0, seed=0, base_offset=0, p=1.0, rounds=7,
              mask_bits=None, s_begin=0, s_end=None):
    """mode 0 plain, 1 fused (Philox inline), 2 decoupled (mask_bits)."""
    thr, pf = keep_threshold(p)
    if mode != 0 and not (0.0 < p <= 1.0):
        raise ValueError("attention_dropout: p must be in (0,1]")
    o = np.zeros(slices * seq * head_dim, np.float32)
    mb = None
    if mode == 2:
        mask_bits = np.ascontiguousarray(mask_bits, np.uint8)
        mb = mask_bits.ctypes.data
    rc = lib().oracle_attention(slices, seq, head_dim, np.ascontiguousarray(q, np.float32),
                                np.ascontiguousarray(k, np.float32), np.ascontiguousarray(v, np.float32),
                                mode, seed, base_offset, thr, pf, rounds, mb, s_begin,
                                slices if s_end is None else s_end, o)
    if rc != 0:
        raise ValueError("oracle_attention: bad arguments")
    return o


def fnv1a64(data: np.ndarray) -> int:
    data = np.ascontiguousarray(data, np.uint8)
    return int(lib().oracle_fnv1a64(data, data.size))


# ---------------------------------------------------------------- backward
def unpack_keep(bits, slices, seq):
    """Packed LSB-first mask (mask.hpp:183-186, 291-295) -> bool [slices, seq, seq]."""
    n = slices * seq * seq
    return np.unpackbits(np.ascontiguousarray(bits, np.uint8), bitorder="little")[:n].astype(bool).reshape(
        slices, seq, seq)


def attention_backward(q, k, v, do, slices, seq, head_dim, keep=None, p=1.0):
    """Analytic gradient of the reference forward (ref_attention.hpp:56-92) in
    float64.  The reference has no backward: this restates the
    derivative of forward_impl's semantics -- softmax over ALL keys before
    dropout (:78-82), kept weights scaled by 1/float(p) (:84-85, :125) -- and
    is cross-checked against torch float64 autograd in tests/test_oracle.py.
    q, k, v, do: arrays of slices*seq*head_dim; keep: bool [slices, seq, seq]
    or None (no dropout).  Returns (o, dq, dk, dv), each [slices, seq, head_dim]."""
    sh = (slices, seq, head_dim)
    q, k, v, do = (np.asarray(x, np.float64).reshape(sh) for x in (q, k, v, do))
    scale = float(np.float32(1.0) / np.sqrt(np.float32(head_dim)))
    pf = float(np.float32(p))
    s = scale * (q @ k.transpose(0, 2, 1))
    s -= s.max(axis=-1, keepdims=True)
    e = np.exp(s)
    P = e / e.sum(axis=-1, keepdims=True)
    km = np.ones_like(P) if keep is None else keep.astype(np.float64)
    W = km * P / pf
    o = W @ v
    dv = W.transpose(0, 2, 1) @ do
    dP = km * (do @ v.transpose(0, 2, 1)) / pf
    D = (P * dP).sum(axis=-1, keepdims=True)
    dS = P * (dP - D)
    dq = scale * (dS @ k)
    dk = scale * (dS.transpose(0, 2, 1) @ q)
    return o, dq, dk, dv
