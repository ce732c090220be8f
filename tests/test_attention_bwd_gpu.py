"""GPU parity for K7, the tcgen05 flash-attention backward with dropout
(csrc/attn_bwd_sm100.cu), against the float64 backward oracle
(oracle.attention_backward: the analytic derivative of ref_attention.hpp:56-92)
on bf16-rounded inputs.  Tolerance (north_star, BF16): relative Frobenius
error <= 5e-3 for O and <= TOL_GRAD for dQ/dK/dV (P and dS pass through bf16
on the tensor cores).  The decoupled (mask bits) and fused (Philox inline)
backwards use identical keep decisions: dK, dV bitwise equal; dQ is reduced
with fp32 reductions across key tiles (order-dependent rounding) and must agree
to fp32-accumulation accuracy."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
TOL_O = 5e-3
TOL_GRAD = 5e-3


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def make_inputs(B, H, S, D, seed, qscale=1.0):
    import torch
    g = torch.Generator(device="cpu").manual_seed(seed)
    q, k, v, do = ((torch.rand(B, H, S, D, generator=g) * 2 - 1) for _ in range(4))
    q = q * qscale
    return [t.bfloat16().cuda() for t in (q, k, v, do)]


def run(rgo, q, k, v, do, mode, p=0.9, seed=42, base=0, rounds=10, bits=None, deterministic=False):
    import torch
    B, H, S, D = q.shape
    lse = torch.empty(B * H * S, dtype=torch.float32, device=q.device)
    o = rgo.attn_fwd(q, k, v, mask_source=mode, keep_prob=p, bits=bits, seed=seed, base_offset=base, rounds=rounds,
                     lse=lse)
    dq, dk, dv = rgo.attn_bwd(q, k, v, o, do, lse, mask_source=mode, keep_prob=p, bits=bits, seed=seed,
                              base_offset=base, rounds=rounds, deterministic=deterministic)
    torch.cuda.synchronize()
    return o, dq, dk, dv


def np64(t):
    return t.float().cpu().numpy().astype(np.float64)


def check_vs_oracle(q, k, v, do, o, dq, dk, dv, keep, p):
    B, H, S, D = q.shape
    N = B * H
    want = oracle.attention_backward(np64(q), np64(k), np64(v), np64(do), N, S, D, keep, p)
    got = [np64(x).reshape(N, S, D) for x in (o, dq, dk, dv)]
    errs = [rel(g, w) for g, w in zip(got, want)]
    assert errs[0] < TOL_O, errs
    assert max(errs[1:]) < TOL_GRAD, errs
    return errs


@pytest.mark.parametrize("B,H,S,D", [(1, 2, 256, 64), (2, 1, 384, 128), (1, 2, 200, 64), (1, 1, 520, 128)])
def test_bwd_no_dropout(rgo, cuda, B, H, S, D):
    q, k, v, do = make_inputs(B, H, S, D, 1)
    o, dq, dk, dv = run(rgo, q, k, v, do, rgo.ref_attention.MASK_NONE, p=1.0)
    check_vs_oracle(q, k, v, do, o, dq, dk, dv, None, 1.0)


@pytest.mark.parametrize("B,H,S,D", [(1, 2, 256, 64), (2, 2, 256, 128), (1, 1, 200, 128)])
@pytest.mark.parametrize("rounds", [10, 7])
def test_bwd_bits_and_philox(rgo, cuda, B, H, S, D, rounds):
    import torch
    q, k, v, do = make_inputs(B, H, S, D, 2, qscale=3.0)
    p, seed, base = 0.9, 1234, 777
    lay = rgo.MaskLayout(B, H, S, seed, base)
    bits = rgo.generate_mask_device(lay, rgo.KeepThreshold(p), rounds)
    ob, dqb, dkb, dvb = run(rgo, q, k, v, do, rgo.ref_attention.MASK_BITS, p, seed, base, rounds, bits)
    of, dqf, dkf, dvf = run(rgo, q, k, v, do, rgo.ref_attention.MASK_PHILOX, p, seed, base, rounds)
    assert torch.equal(ob, of)
    assert torch.equal(dkb, dkf) and torch.equal(dvb, dvf)
    assert rel(np64(dqb), np64(dqf)) < 1e-3
    nb = B * H * S * S
    keep = oracle.unpack_keep(bits[: (nb + 7) // 8].cpu().numpy(), B * H, S)
    check_vs_oracle(q, k, v, do, ob, dqb, dkb, dvb, keep, p)


def test_bwd_cpu_config_keep_fraction(rgo, cuda):
    """CPU-oracle config O (B1 nH8 SQ512 dH64, keep 0.9, Philox-10)."""
    q, k, v, do = make_inputs(1, 8, 512, 64, 3)
    bits = rgo.generate_mask_device(rgo.MaskLayout(1, 8, 512, 42, 0), rgo.KeepThreshold(0.9), 10)
    o, dq, dk, dv = run(rgo, q, k, v, do, rgo.ref_attention.MASK_BITS, 0.9, 42, 0, 10, bits)
    keep = oracle.unpack_keep(bits[: 8 * 512 * 512 // 8].cpu().numpy(), 8, 512)
    check_vs_oracle(q, k, v, do, o, dq, dk, dv, keep, 0.9)


def test_bwd_token_major_views(rgo, cuda):
    """Q/K/V as column blocks of the QKV GEMM output [B*S, 3*H*D] (the block's layout)."""
    import torch
    B, H, S, D = 2, 2, 256, 128
    qkv = (torch.rand(B, S, 3, H, D, device="cuda") * 2 - 1).bfloat16()
    q, k, v = (qkv[:, :, i].permute(0, 2, 1, 3) for i in range(3))
    do = (torch.rand(B, H, S, D, device="cuda") * 2 - 1).bfloat16()
    o1, dq1, dk1, dv1 = run(rgo, q, k, v, do, rgo.ref_attention.MASK_PHILOX, 0.8, 5, 0, 10)
    o2, dq2, dk2, dv2 = run(rgo, q.contiguous(), k.contiguous(), v.contiguous(), do,
                            rgo.ref_attention.MASK_PHILOX, 0.8, 5, 0, 10)
    assert torch.equal(o1, o2) and torch.equal(dk1, dk2) and torch.equal(dv1, dv2)
    assert rel(np64(dq1), np64(dq2)) < 1e-3


def test_autograd_function(rgo, cuda):
    import torch
    q, k, v, do = make_inputs(1, 2, 256, 64, 4)
    q.requires_grad_(True)
    k.requires_grad_(True)
    v.requires_grad_(True)
    o = rgo.DropoutAttention.apply(q, k, v, rgo.ref_attention.MASK_PHILOX, 0.9, None, 9, 0, 10)
    o.backward(do)
    _, dq, dk, dv = run(rgo, q.detach(), k.detach(), v.detach(), do, rgo.ref_attention.MASK_PHILOX, 0.9, 9, 0, 10)
    assert torch.equal(k.grad, dk) and torch.equal(v.grad, dv)
    assert rel(np64(q.grad), np64(dq)) < 1e-3


def test_bwd_validation(rgo, cuda):
    q, k, v, do = make_inputs(1, 1, 128, 64, 5)
    import torch
    lse = torch.empty(128, dtype=torch.float32, device="cuda")
    o = rgo.attn_fwd(q, k, v, lse=lse)
    with pytest.raises(ValueError, match="p must be in"):
        rgo.attn_bwd(q, k, v, o, do, lse, mask_source=rgo.ref_attention.MASK_PHILOX, keep_prob=0.0)
    with pytest.raises(ValueError, match="mask needs"):
        rgo.attn_bwd(q, k, v, o, do, lse, mask_source=rgo.ref_attention.MASK_BITS, keep_prob=0.9,
                     bits=torch.zeros(16, dtype=torch.uint8, device="cuda"))


def test_random_shapes_fwd_bwd_vs_oracle(rgo, cuda):
    """Seeded random sweep: ragged SQ (multiples of 128 and not), both head dims,
    keep probabilities, round counts, seeds and counter offsets; mask bits from
    K1 vs inline Philox agree (O, dK, dV bitwise) and match the float64 oracle."""
    import torch
    rng = np.random.default_rng(2410)
    for case in range(12):
        B, H = int(rng.integers(1, 3)), int(rng.integers(1, 4))
        S = int(rng.choice([int(rng.integers(1, 700)), 128 * int(rng.integers(1, 5))]))
        D = int(rng.choice([64, 128]))
        p = float(rng.choice([0.5, 0.75, 0.9, 0.99]))
        rounds = int(rng.choice([10, 7, 5]))
        seed, base = int(rng.integers(0, 2**63)), int(rng.integers(0, 2**40))
        q, k, v, do = make_inputs(B, H, S, D, 100 + case, qscale=2.0)
        bits = rgo.generate_mask_device(rgo.MaskLayout(B, H, S, seed, base), rgo.KeepThreshold(p), rounds)
        ob, dqb, dkb, dvb = run(rgo, q, k, v, do, rgo.ref_attention.MASK_BITS, p, seed, base, rounds, bits)
        of, dqf, dkf, dvf = run(rgo, q, k, v, do, rgo.ref_attention.MASK_PHILOX, p, seed, base, rounds)
        ctx = dict(B=B, H=H, S=S, D=D, p=p, rounds=rounds)
        assert torch.equal(ob, of), ctx
        assert torch.equal(dkb, dkf) and torch.equal(dvb, dvf), ctx
        nb = B * H * S * S
        keep = oracle.unpack_keep(bits[: (nb + 7) // 8].cpu().numpy(), B * H, S)
        check_vs_oracle(q, k, v, do, ob, dqb, dkb, dvb, keep, p)


@pytest.mark.parametrize("S", [640, 200, 4096])
def test_split_bwd_dq_deterministic(rgo, cuda, S):
    """RGO_ATTN_BWD_DETERMINISTIC (head dim 128): the split backward (dK/dV kernel
    + dQ kernel with dQ accumulated in TMEM) has no fp32 reductions across CTAs,
    so dQ too is bitwise equal between mask bits and inline Philox and between
    repeated runs; all of it within 5e-3 of the float64 oracle."""
    import torch
    B, H, D = 1, 2, 128
    q, k, v, do = make_inputs(B, H, S, D, 7, qscale=2.0)
    bits = rgo.generate_mask_device(rgo.MaskLayout(B, H, S, 3, 99), rgo.KeepThreshold(0.8), 10)
    ob, dqb, dkb, dvb = run(rgo, q, k, v, do, rgo.ref_attention.MASK_BITS, 0.8, 3, 99, 10, bits, deterministic=True)
    of, dqf, dkf, dvf = run(rgo, q, k, v, do, rgo.ref_attention.MASK_PHILOX, 0.8, 3, 99, 10, deterministic=True)
    _, dq2, _, _ = run(rgo, q, k, v, do, rgo.ref_attention.MASK_BITS, 0.8, 3, 99, 10, bits, deterministic=True)
    assert torch.equal(dqb, dqf) and torch.equal(dqb, dq2)
    assert torch.equal(dkb, dkf) and torch.equal(dvb, dvf)
    keep = oracle.unpack_keep(bits[: (B * H * S * S + 7) // 8].cpu().numpy(), B * H, S)
    check_vs_oracle(q, k, v, do, ob, dqb, dkb, dvb, keep, 0.8)


def test_bwd_implementations_agree(rgo, cuda):
    """The three head-dim-128 backward implementations (RGO_BWD_IMPL 1/2/3, read
    once per process -> subprocesses) agree: dK/dV bitwise between 1 and 3 (same
    kernel, same MMA order), dQ within fp32-accumulation differences."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import paper_2410_07531_b200 as rgo
from test_attention_bwd_gpu import make_inputs, run
q, k, v, do = make_inputs(2, 2, 384, 128, 11, qscale=2.0)
bits = rgo.generate_mask_device(rgo.MaskLayout(2, 2, 384, 8, 0), rgo.KeepThreshold(0.9), 10)
o, dq, dk, dv = run(rgo, q, k, v, do, rgo.ref_attention.MASK_BITS, 0.9, 8, 0, 10, bits)
np.save(sys.argv[2], np.stack([t.float().cpu().numpy() for t in (o, dq, dk, dv)]))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for impl in ("1", "2", "3"):
        path = f"/tmp/rgo_bwd_impl{impl}_{os.getpid()}.npy"
        r = subprocess.run([sys.executable, "-c", code, root, path], env=dict(os.environ, RGO_BWD_IMPL=impl),
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        out[impl] = np.load(path)
        os.remove(path)
    np.testing.assert_array_equal(out["1"][2:], out["3"][2:])  # dK, dV
    for impl in ("1", "2"):
        np.testing.assert_array_equal(out[impl][0], out["3"][0])  # O (same forward)
        assert rel(out[impl][1], out["3"][1]) < 1e-3             # dQ
        assert rel(out[impl][2:], out["3"][2:]) < 1e-3
