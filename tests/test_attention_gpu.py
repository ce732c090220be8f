"""GPU parity for the tcgen05 flash-attention forward (K5 mask / K6 inline
Philox) against the CPU oracle (restated ref_attention.hpp) on bf16-rounded
inputs.  Tolerance (north_star, BF16): ||o - ref||_2 / ||ref||_2 <= 5e-3.
Fused and decoupled GPU outputs must be bitwise equal (acceptance C2)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu
TOL = 5e-3


def bf16_round(x):
    import torch
    return torch.from_numpy(np.ascontiguousarray(x, np.float32)).bfloat16().float().numpy()


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def rounded_input(rgo, inp):
    return rgo.AttentionInput(inp.slices, inp.seq, inp.head_dim, bf16_round(inp.q), bf16_round(inp.k),
                              bf16_round(inp.v))


def test_random_input_matches_reference_generator(rgo, cuda):
    inp = rgo.random_attention_input(2, 64, 32, 1000 ^ 0xA77E)
    q, k, v = oracle.random_attention_input(2, 64, 32, 1000 ^ 0xA77E)
    for a, b in ((inp.q, q), (inp.k, k), (inp.v, v)):
        np.testing.assert_array_equal(a.view(np.uint32), b.view(np.uint32))


def test_plain_forward_vs_oracle_cpu_config(rgo, cuda):
    # CPU-oracle config O: B1 nH8 SQ512 dH64
    inp = rounded_input(rgo, rgo.random_attention_input(8, 512, 64, 42 ^ 0xA77E))
    got = rgo.attention_forward(inp)
    want = oracle.attention(inp.q, inp.k, inp.v, 8, 512, 64, 0)
    assert rel(got.o, want) < TOL


@pytest.mark.parametrize("rounds", [10, 7])
def test_fused_and_decoupled_cpu_config(rgo, cuda, rounds):
    inp = rounded_input(rgo, rgo.random_attention_input(8, 512, 64, 42 ^ 0xA77E))
    fused = rgo.attention_dropout_fused(inp, 42, 0.9, rounds)
    mask = rgo.generate_mask(rgo.MaskLayout(1, 8, 512, 42), rgo.KeepThreshold(0.9), rounds)
    dec = rgo.attention_dropout_decoupled(inp, mask, 0.9)
    assert fused == dec
    want = oracle.attention(inp.q, inp.k, inp.v, 8, 512, 64, 1, 42, 0, 0.9, rounds)
    assert rel(fused.o, want) < TOL


def test_equivalence_grid(rgo, cuda):
    """ref_attention.hpp:164-227: 16 cases, fused == decoupled bitwise, and
    both within tolerance of the oracle."""
    results = rgo.run_equiv_suite(rgo.default_equiv_grid())
    assert len(results) == 16 and all(r.bitwise_equal for r in results)
    for c in rgo.default_equiv_grid():
        inp = rounded_input(rgo, rgo.random_attention_input(c.slices, c.seq, c.head_dim, c.seed ^ 0xA77E))
        got = rgo.attention_dropout_fused(inp, c.seed, c.p, 7)
        want = oracle.attention(inp.q, inp.k, inp.v, c.slices, c.seq, c.head_dim, 1, c.seed, 0, c.p, 7)
        assert rel(got.o, want) < TOL, c


def test_p1_is_identity(rgo, cuda):
    # test_attention.cpp:72-84
    inp = rgo.random_attention_input(4, 32, 16, 77)
    plain = rgo.attention_forward(inp)
    assert rgo.attention_dropout_fused(inp, 123, 1.0, 7) == plain
    ones = rgo.generate_mask(rgo.MaskLayout(1, 4, 32, 123), rgo.KeepThreshold(1.0), 7)
    assert rgo.attention_dropout_decoupled(inp, ones, 1.0) == plain


def test_validation(rgo, cuda):
    inp = rgo.random_attention_input(2, 16, 8, 3)
    with pytest.raises(ValueError):
        rgo.attention_dropout_fused(inp, 1, 0.0, 7)
    m = rgo.generate_mask(rgo.MaskLayout(1, 2, 8), rgo.KeepThreshold(0.9), 7)
    with pytest.raises(ValueError):
        rgo.attention_dropout_decoupled(inp, m, 0.9)
    m2 = rgo.generate_mask(rgo.MaskLayout(1, 2, 16), rgo.KeepThreshold(0.9), 7)
    with pytest.raises(ValueError):
        rgo.attention_dropout_decoupled(inp, m2, 0.8)


def test_seed_determinism(rgo, cuda):
    inp = rgo.random_attention_input(2, 16, 8, 3)
    a = rgo.attention_dropout_fused(inp, 42, 0.9, 7)
    assert a == rgo.attention_dropout_fused(inp, 42, 0.9, 7)
    assert not (a == rgo.attention_dropout_fused(inp, 43, 0.9, 7))


def test_one_bit_flip_changes_one_row(rgo, cuda):
    # test_attention.cpp:158-183
    inp = rgo.random_attention_input(3, 12, 6, 55)
    m = rgo.generate_mask(rgo.MaskLayout(1, 3, 12, 4), rgo.KeepThreshold(0.9), 7)
    base = rgo.attention_dropout_decoupled(inp, m, 0.9)
    s, i, j = 1, 5, 7
    idx = m.layout.linear_index(0, s, i, j)
    m.bits[idx >> 3] ^= np.uint8(1 << (idx & 7))
    t = rgo.attention_dropout_decoupled(inp, m, 0.9)
    d = (base.o.reshape(3, 12, 6) != t.o.reshape(3, 12, 6)).any(-1)
    assert d[s, i] and d.sum() == 1


def test_llama_head_shape_slice_vs_oracle(rgo, cuda):
    """dH=128, SQ=2048, 2 slices, Philox-10, keep 0.9: fused == decoupled
    bitwise; slice 1 (base_offset arithmetic) within tolerance of the oracle."""
    import torch
    S, D, N = 2048, 128, 2
    inp = rounded_input(rgo, rgo.random_attention_input(N, S, D, 7))
    fused = rgo.attention_dropout_fused(inp, 42, 0.9, 10)
    mask = rgo.generate_mask(rgo.MaskLayout(1, N, S, 42), rgo.KeepThreshold(0.9), 10)
    assert fused == rgo.attention_dropout_decoupled(inp, mask, 0.9)
    want = oracle.attention(inp.q, inp.k, inp.v, N, S, D, 1, 42, 0, 0.9, 10, s_begin=1, s_end=2)
    assert rel(fused.o[S * D:], want[S * D:]) < TOL


def test_token_major_layout_and_lse(rgo, cuda):
    """Q/K/V as column slices of a [B*S, 3*H*D] QKV-GEMM output give the same
    bits as the head-major layout; LSE matches a torch fp32 reference."""
    import torch
    B, H, S, D = 2, 3, 384, 128
    g = torch.Generator(device="cuda").manual_seed(0)
    qkv = (torch.rand(B * S, 3 * H * D, generator=g, device="cuda") * 2 - 1).bfloat16()
    v4 = qkv.view(B, S, 3, H, D)
    q, k, v = (v4[:, :, i].permute(0, 2, 1, 3) for i in range(3))  # [B, H, S, D] strided views
    o_tok = torch.empty(B, S, H, D, dtype=torch.bfloat16, device="cuda")
    lse = torch.empty(B * H * S, dtype=torch.float32, device="cuda")
    rgo.attn_fwd(q, k, v, o_tok.permute(0, 2, 1, 3), mask_source=2, keep_prob=0.9, seed=5, rounds=10, lse=lse)
    qc, kc, vc = (x.contiguous() for x in (q, k, v))
    o_hm = rgo.attn_fwd(qc, kc, vc, mask_source=2, keep_prob=0.9, seed=5, rounds=10)
    assert torch.equal(o_tok.permute(0, 2, 1, 3), o_hm)
    sc = (qc.float() @ kc.float().transpose(-1, -2)) / np.sqrt(D)
    ref_lse = torch.logsumexp(sc, -1).reshape(-1)
    torch.testing.assert_close(lse, ref_lse, rtol=1e-3, atol=1e-3)


@pytest.mark.parametrize("base", [(1 << 32) - 5000, (1 << 64) - 3000])
def test_counter_carry_and_wrap_fwd_bwd(rgo, cuda, base):
    """The Philox counter crosses a 2^32 boundary (carry into c1) or wraps 2^64
    (element_source, mask.hpp:72-85) inside a slice: the inline-Philox forward
    and backward (K6, K7) must still make K1's keep decisions bit for bit."""
    import torch
    B, H, S, D = 1, 2, 512, 128
    g = torch.Generator(device="cpu").manual_seed(11)
    q, k, v, do = ((torch.rand(B, H, S, D, generator=g) * 2 - 1).bfloat16().cuda() for _ in range(4))
    bits = rgo.generate_mask_device(rgo.MaskLayout(B, H, S, 99, base), rgo.KeepThreshold(0.9), 10)
    lse_b = torch.empty(B * H * S, device="cuda")
    lse_f = torch.empty(B * H * S, device="cuda")
    ob = rgo.attn_fwd(q, k, v, mask_source=1, keep_prob=0.9, bits=bits, lse=lse_b)
    of = rgo.attn_fwd(q, k, v, mask_source=2, keep_prob=0.9, seed=99, base_offset=base, rounds=10, lse=lse_f)
    assert torch.equal(ob, of)
    gb = rgo.attn_bwd(q, k, v, ob, do, lse_b, mask_source=1, keep_prob=0.9, bits=bits)
    gf = rgo.attn_bwd(q, k, v, of, do, lse_f, mask_source=2, keep_prob=0.9, seed=99, base_offset=base, rounds=10)
    assert torch.equal(gb[1], gf[1]) and torch.equal(gb[2], gf[2])
    # and the mask itself is the oracle's
    want = oracle.generate_mask(B, H, S, 99, base, 0.9, 10)
    assert np.array_equal(bits[: want.size].cpu().numpy(), want)


@pytest.mark.parametrize("hd", [160, 256, 520])
def test_large_head_dim_generic_kernel(rgo, cuda, hd):
    """head_dim > 128 (the reference accepts any head_dim): the drop-in's host entry point
    (rgo_attention_host) runs the fp32 CUDA-core kernel K5g (csrc/attn_generic.cu) on the fp32
    arrays -- no bf16 rounding, so within 1e-5 of the oracle; fused == decoupled bitwise (with a
    base_offset); p = 1 is the plain forward bitwise."""
    N, S = 3, 200
    inp = rgo.random_attention_input(N, S, hd, 11)
    fused = rgo.attention_dropout_fused(inp, 42, 0.9, 10, base_offset=5)
    mask = rgo.generate_mask(rgo.MaskLayout(1, N, S, 42, 5), rgo.KeepThreshold(0.9), 10)
    assert fused == rgo.attention_dropout_decoupled(inp, mask, 0.9)
    want = oracle.attention(inp.q, inp.k, inp.v, N, S, hd, 1, 42, 5, 0.9, 10)
    assert rel(fused.o, want) < 1e-5
    plain = rgo.attention_forward(inp)
    assert rel(plain.o, oracle.attention(inp.q, inp.k, inp.v, N, S, hd, 0)) < 1e-5
    assert rgo.attention_dropout_fused(inp, 42, 1.0, 10) == plain


def test_head_dim_limit(rgo, cuda):
    inp = rgo.random_attention_input(1, 8, 1025, 3)
    with pytest.raises(ValueError):
        rgo.attention_forward(inp)
