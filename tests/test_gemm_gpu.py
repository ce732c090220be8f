"""GPU numerics of the tcgen05 GEMMs (K2/K3/K4) against a plain PyTorch fp32
reference of the same op (dequantised inputs).  Tolerances (north_star):
BF16 <= 5e-3, FP8 <= 2e-2 relative (Frobenius norm of the error over the norm
of the reference), plus an elementwise bound scaled by the output rounding."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm())


def make(shape, dtype, seed, scale=1.0):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = (torch.rand(shape, generator=g, device="cuda") * 2 - 1) * scale
    return x.to(dtype)


@pytest.mark.parametrize("m,n,k", [(128, 256, 64), (256, 512, 256), (200, 352, 320), (1024, 768, 1024)])
def test_bf16_gemm(rgo, cuda, m, n, k):
    import torch
    a, b = make((m, k), torch.bfloat16, 1), make((n, k), torch.bfloat16, 2)
    c = rgo.gemm(a, b, alpha=0.5)
    ref = (a.float() @ b.float().T) * 0.5
    assert rel(c, ref) < 5e-3
    torch.testing.assert_close(c.float(), ref, rtol=1e-2, atol=1e-2 * float(ref.abs().max()))


@pytest.mark.parametrize("m,n,k", [(128, 256, 128), (384, 512, 512), (200, 288, 384), (2048, 1024, 4096)])
def test_fp8_gemm(rgo, cuda, m, n, k):
    import torch
    a = make((m, k), torch.float32, 3, 4.0).to(torch.float8_e4m3fn)
    b = make((n, k), torch.float32, 4, 4.0).to(torch.float8_e4m3fn)
    c = rgo.gemm(a, b, alpha=1.0 / 64)
    ref = (a.float() @ b.float().T) / 64
    assert rel(c, ref) < 5e-3  # exact products, fp32 accumulate, bf16 output
    c8 = rgo.gemm(a, b, alpha=1.0 / 64, out_scale=0.5, out_dtype=torch.float8_e4m3fn)
    # e4m3 output rounding (3 mantissa bits) dominates: compare with the
    # fp8-rounded reference, then bound the total error by the format's RMS
    assert rel(c8.float(), (ref * 0.5).to(torch.float8_e4m3fn).float()) < 2e-2
    assert rel(c8.float(), ref * 0.5) < 4e-2


def test_swiglu_epilogue(rgo, cuda):
    import torch
    m, f, k = 256, 384, 256   # 3 tiles of [128 gate | 128 up]
    a = make((m, k), torch.bfloat16, 5)
    gate, up = make((f, k), torch.bfloat16, 6), make((f, k), torch.bfloat16, 7)
    w = torch.cat([gate.view(-1, 128, k), up.view(-1, 128, k)], dim=1).reshape(2 * f, k)
    c = rgo.gemm(a, w, epilogue="swiglu", alpha=0.25)
    g, u = (a.float() @ gate.float().T) * 0.25, (a.float() @ up.float().T) * 0.25
    ref = torch.nn.functional.silu(g) * u
    assert c.shape == (m, f) and rel(c, ref) < 5e-3


def test_gelu_epilogue_fp8_out(rgo, cuda):
    import torch
    a = make((256, 512), torch.float32, 8, 2.0).to(torch.float8_e4m3fn)
    b = make((512, 512), torch.float32, 9, 2.0).to(torch.float8_e4m3fn)
    c = rgo.gemm(a, b, epilogue="gelu", alpha=1 / 32, out_scale=4.0, out_dtype=torch.float8_e4m3fn)
    ref = torch.nn.functional.gelu((a.float() @ b.float().T) / 32, approximate="tanh") * 4.0
    assert rel(c.float(), ref.to(torch.float8_e4m3fn).float()) < 2e-2


def test_gelu_epilogue_fp8_in_bf16_out(rgo, cuda):
    """FP8 inputs + GELU + BF16 output (the GPT-3 block's ungated FFN1 with a bf16 result)."""
    import torch
    a = make((256, 512), torch.float32, 12, 2.0).to(torch.float8_e4m3fn)
    b = make((512, 512), torch.float32, 13, 2.0).to(torch.float8_e4m3fn)
    c = rgo.gemm(a, b, epilogue="gelu", alpha=1 / 32)
    assert c.dtype == torch.bfloat16
    ref = torch.nn.functional.gelu((a.float() @ b.float().T) / 32, approximate="tanh")
    assert rel(c.float(), ref) < 5e-3


@pytest.mark.parametrize("warps", [0, 4, 12, 16])
def test_gemm_with_rng_mask_and_output(rgo, cuda, warps):
    """K4: co-resident RNG warps leave the GEMM result unchanged and, with the
    tail drain, produce the K1 mask bit-exactly."""
    import torch
    a, b = make((2048, 1024), torch.bfloat16, 10), make((1024, 1024), torch.bfloat16, 11)
    lay = rgo.MaskLayout(1, 4, 1024, 77, 1234)
    thr = rgo.KeepThreshold(0.9)
    d = rgo.mask.desc(lay, thr, 10)
    bits = torch.zeros(lay.elem_count() // 8, dtype=torch.uint8, device="cuda")
    counter = torch.zeros(1, dtype=torch.int64, device="cuda")
    c0 = rgo.gemm(a, b)
    c1 = torch.empty_like(c0)
    rgo.gemm_with_rng(a, b, c1, d, bits, counter, rng_warps=warps)
    torch.testing.assert_close(c1, c0, rtol=0, atol=0)
    rgo.mask_queue_drain(d, bits, counter)
    want = rgo.generate_mask_device(lay, thr, 10)
    assert torch.equal(bits, want[: bits.numel()])


def test_queue_drain_alone_matches_k1(rgo, cuda):
    import torch
    for rounds in (7, 10, 5, 1, 6, 16):
        lay = rgo.MaskLayout(2, 3, 512, 5, 0xFFFFFFFF - 300)
        thr = rgo.KeepThreshold(0.8)
        bits = torch.zeros(lay.elem_count() // 8, dtype=torch.uint8, device="cuda")
        counter = torch.zeros(1, dtype=torch.int64, device="cuda")
        rgo.mask_queue_drain(rgo.mask.desc(lay, thr, rounds), bits, counter, grid=7)
        want = rgo.generate_mask_device(lay, thr, rounds)
        assert torch.equal(bits, want[: bits.numel()])


@pytest.mark.parametrize("rounds", [6, 1, 16])
def test_gemm_with_rng_runtime_rounds(rgo, cuda, rounds):
    """Round counts without a compiled drain: the in-GEMM warps use the
    runtime-rounds Philox and still produce K1's bits (no silent tail-only)."""
    import torch
    a, b = make((2048, 1024), torch.bfloat16, 14), make((1024, 1024), torch.bfloat16, 15)
    lay = rgo.MaskLayout(1, 2, 512, 91, 77)
    thr = rgo.KeepThreshold(0.85)
    d = rgo.mask.desc(lay, thr, rounds)
    bits = torch.zeros(lay.elem_count() // 8, dtype=torch.uint8, device="cuda")
    counter = torch.zeros(1, dtype=torch.int64, device="cuda")
    c = torch.empty(2048, 1024, dtype=torch.bfloat16, device="cuda")
    rgo.gemm_with_rng(a, b, c, d, bits, counter, rng_warps=8)
    torch.cuda.synchronize()
    assert int(counter.item()) > 0  # the GEMM's RNG warps claimed work
    rgo.mask_queue_drain(d, bits, counter)
    assert torch.equal(bits, rgo.generate_mask_device(lay, thr, rounds)[: bits.numel()])


def test_gemm_validation(rgo, cuda):
    import torch
    a = torch.zeros(128, 100, dtype=torch.bfloat16, device="cuda")
    b = torch.zeros(256, 100, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        rgo.gemm(a, b)  # k*2 not a multiple of 128 bytes
    a = torch.zeros(128, 128, dtype=torch.bfloat16, device="cuda")
    b = torch.zeros(256, 128, dtype=torch.bfloat16, device="cuda")
    c = rgo.gemm(a, b)
    lay = rgo.MaskLayout(1, 1, 128, 1)
    bits = torch.zeros(lay.elem_count() // 8, dtype=torch.uint8, device="cuda")
    counter = torch.zeros(1, dtype=torch.int64, device="cuda")
    with pytest.raises(ValueError):
        rgo.gemm_with_rng(a, b, c, rgo.mask.desc(lay, rgo.KeepThreshold(0.9), 10), bits, counter, rng_warps=5)


def test_random_shapes_vs_torch(rgo, cuda):
    """Seeded random sweep of ragged M, N (multiple of 32) and K (multiple of 128
    bytes), FP8 and BF16, against the fp32 product of the same (dequantised) inputs."""
    import torch
    rng = np.random.default_rng(7531)
    for case in range(16):
        fp8 = bool(case % 2)
        m = int(rng.integers(1, 1500))
        n = 32 * int(rng.integers(1, 40))
        k = (128 if fp8 else 64) * int(rng.integers(1, 12))
        dt = torch.float8_e4m3fn if fp8 else torch.bfloat16
        a = make((m, k), torch.float32, 1000 + case, 2.0).to(dt)
        b = make((n, k), torch.float32, 2000 + case, 2.0).to(dt)
        alpha = 1.0 / k
        c = rgo.gemm(a, b, alpha=alpha)
        ref = (a.float() @ b.float().T) * alpha
        assert rel(c, ref) < 5e-3, (m, n, k, fp8)
