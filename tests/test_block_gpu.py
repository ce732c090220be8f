"""GPU: one transformer-block step (csrc/block.cu) in each overlap mode.
All three modes must produce bitwise-identical results (the fused and
decoupled attention agree bitwise, GEMMs are deterministic), the mask must
equal K1's, and every stage must match a PyTorch fp32 reference computed from
that stage's actual inputs (FP8 <= 2e-2, BF16 <= 5e-3 relative)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm())


def small_cfg(rgo):
    return rgo.WorkloadConfig(batch=2, seq=512, heads=4, head_dim=128, ffn_dim=384, gated=True, keep_prob=0.9,
                              philox_rounds=10)


def snapshot(b):
    return {k: getattr(b, k).clone() for k in ("x", "qkv", "attn_o", "attn_o8", "y1", "h")}


def test_modes_bitwise_identical(rgo, cuda):
    import torch
    cfg = small_cfg(rgo)
    outs = {}
    for mode in ("serial_fused", "streams", "in_gemm"):
        b = rgo.Block(cfg, mode, seed=42, use_graph=(mode != "in_gemm"))
        b.step()
        torch.cuda.synchronize()
        outs[mode] = (snapshot(b), b.mask.clone())
        b.close()
    base = outs["serial_fused"][0]
    for mode in ("streams", "in_gemm"):
        for k, v in outs[mode][0].items():
            assert torch.equal(v.view(torch.uint8), base[k].view(torch.uint8)), (mode, k)
    lay = rgo.MaskLayout(cfg.batch, cfg.heads, cfg.seq, 42)
    want = rgo.generate_mask_device(lay, rgo.KeepThreshold(0.9), 10)
    for mode in ("streams", "in_gemm"):
        assert torch.equal(outs[mode][1], want[: outs[mode][1].numel()]), mode


@pytest.mark.parametrize("warps", [4, 6, 8, 12, 16])
def test_in_gemm_rng_warp_counts(rgo, cuda, warps):
    """Mechanism B with each co-resident RNG-warp count: K1's mask, the
    serial-fused block's outputs."""
    import torch
    cfg = small_cfg(rgo)
    ref = rgo.Block(cfg, "serial_fused", seed=42)
    ref.step()
    b = rgo.Block(cfg, "in_gemm", seed=42, rng_launch=(0, warps, 0))
    b.step()
    torch.cuda.synchronize()
    for k, v in snapshot(b).items():
        assert torch.equal(v.view(torch.uint8), getattr(ref, k).view(torch.uint8)), k
    want = rgo.generate_mask_device(rgo.MaskLayout(cfg.batch, cfg.heads, cfg.seq, 42), rgo.KeepThreshold(0.9), 10)
    assert torch.equal(b.mask, want[: b.mask.numel()])
    ref.close()
    b.close()


def test_block_stages_vs_torch(rgo, cuda):
    import torch
    import torch.nn.functional as F
    cfg = small_cfg(rgo)
    b = rgo.Block(cfg, "streams", seed=7)
    attn_in = b.attn_in.clone()
    b.step()
    torch.cuda.synchronize()
    d, Fd = b.d, b.F
    w = b.weights
    dq = b.desc
    f8 = torch.float8_e4m3fn
    assert rel(b.attn_o8.float(), (attn_in.float() * dq.s_attn).to(f8).float()) < 2e-2
    y1 = (b.attn_o8.float() @ w["wo"].float().T) * dq.a_proj * dq.s_proj
    assert rel(b.y1.float(), y1.to(f8).float()) < 2e-2
    hh = (b.y1.float() @ w["w1"].float().T) * dq.a_ffn1
    hh = hh.view(b.M, -1, 2, 128)
    hact = F.silu(hh[:, :, 0]) * hh[:, :, 1] * dq.s_ffn1
    assert rel(b.h.float(), hact.reshape(b.M, Fd).to(f8).float()) < 2e-2
    x = (b.h.float() @ w["w2"].float().T) * dq.a_ffn2 * dq.s_ffn2
    assert rel(b.x.float(), x.to(f8).float()) < 2e-2
    qkv = (b.x.float() @ w["wqkv"].float().T) * dq.a_qkv
    assert rel(b.qkv.float(), qkv) < 5e-3
    # attention from the actual QKV with the stored mask
    B, S, H, D = cfg.batch, cfg.seq, cfg.heads, cfg.head_dim
    q, k, v = b.qkv.float().view(B, S, 3, H, D).permute(2, 0, 3, 1, 4)
    sc = (q @ k.transpose(-1, -2)) / np.sqrt(D)
    pr = torch.softmax(sc, -1)
    bits = np.unpackbits(b.mask.cpu().numpy(), bitorder="little")[: B * H * S * S]
    keep = torch.from_numpy(bits.reshape(B, H, S, S).astype(np.float32)).cuda()
    o = ((pr * keep / np.float32(0.9)) @ v).permute(0, 2, 1, 3).reshape(B * S, d)
    assert rel(b.attn_o.float(), o) < 5e-3
    b.close()


def test_graph_replay_is_deterministic(rgo, cuda):
    import torch
    cfg = small_cfg(rgo)
    b1 = rgo.Block(cfg, "streams", seed=3, use_graph=True, chained=True)
    b2 = rgo.Block(cfg, "streams", seed=3, use_graph=False, chained=True)
    for _ in range(3):
        b1.step()
        b2.step()
    torch.cuda.synchronize()
    for k in ("x", "qkv", "attn_o"):
        assert torch.equal(getattr(b1, k).view(torch.uint8), getattr(b2, k).view(torch.uint8)), k
    b1.close()
    b2.close()


def moe_cfg(rgo):
    return rgo.WorkloadConfig(batch=2, seq=256, heads=4, head_dim=128, ffn_dim=256, gated=True, keep_prob=0.9,
                              philox_rounds=10, experts=4, top_k=2)


def test_moe_modes_bitwise_identical(rgo, cuda):
    import torch
    cfg = moe_cfg(rgo)
    outs = {}
    for mode in ("serial_fused", "streams", "in_gemm"):
        b = rgo.Block(cfg, mode, seed=11)
        b.step()
        torch.cuda.synchronize()
        outs[mode] = {k: getattr(b, k).clone() for k in ("x", "qkv", "attn_o", "xd", "ye", "h")}
        b.close()
    for mode in ("streams", "in_gemm"):
        for k, v in outs[mode].items():
            assert torch.equal(v.view(torch.uint8), outs["serial_fused"][k].view(torch.uint8)), (mode, k)


def test_moe_stages_vs_torch(rgo, cuda):
    """Dispatch (balanced routing: pair p = t*k + j -> expert p % E, row p / E),
    per-expert FFN1 (SwiGLU) / FFN2, combine (mean of the top-k outputs)."""
    import torch
    import torch.nn.functional as F
    cfg = moe_cfg(rgo)
    b = rgo.Block(cfg, "streams", seed=5)
    b.step()
    torch.cuda.synchronize()
    E, k, M, d, Fd = cfg.experts, cfg.top_k, b.M, b.d, b.F
    me = M * k // E
    n1 = 2 * Fd
    f8 = torch.float8_e4m3fn
    dq, w = b.desc, b.weights
    p = torch.arange(M * k, device="cuda")
    slot = (p % E) * me + p // E
    assert torch.equal(b.xd.view(torch.uint8)[slot], b.y1.view(torch.uint8)[p // k])
    for e in range(E):
        xe = b.xd[e * me:(e + 1) * me].float()
        hh = (xe @ w["w1"][e * n1:(e + 1) * n1].float().T) * dq.a_ffn1
        hh = hh.view(me, -1, 2, 128)
        hact = (F.silu(hh[:, :, 0]) * hh[:, :, 1] * dq.s_ffn1).reshape(me, Fd)
        assert rel(b.h[e * me:(e + 1) * me].float(), hact.to(f8).float()) < 2e-2
        ye = (b.h[e * me:(e + 1) * me].float() @ w["w2"][e * d:(e + 1) * d].float().T) * dq.a_ffn2 * dq.s_ffn2
        assert rel(b.ye[e * me:(e + 1) * me].float(), ye) < 5e-3
    comb = b.ye.float()[slot].view(M, k, d).sum(1) / k
    assert rel(b.x.float(), comb.to(f8).float()) < 2e-2
    b.close()


def chunked_vs_unchunked(rgo, cfg, mode, chunks, seed=21):
    """SQ-chunk pipeline (schedule.hpp:205-239) against the unchunked block.
    The chunked step computes attention(qkv) -> attn_o, then Proj/FFN/QKV(attn_o)
    -> qkv_out, window by window; the unchunked step computes QKV(chain(attn_in))
    -> qkv, attention(qkv) -> attn_o.  So with the chunked input qkv = the
    unchunked step's qkv, its attn_o must equal the unchunked attn_o bitwise, and
    its qkv_out must equal the qkv of an unchunked step whose input is that attn_o."""
    import torch
    u = rgo.Block(cfg, mode, seed=seed)
    u.step()
    torch.cuda.synchronize()
    p = rgo.Block(cfg, mode, seed=seed, weights=u.weights, chunks=chunks)
    p.qkv.copy_(u.qkv)
    p.step()
    torch.cuda.synchronize()
    assert torch.equal(p.attn_o.view(torch.uint8), u.attn_o.view(torch.uint8))
    u2 = rgo.Block(cfg, mode, seed=seed, weights=u.weights)
    u2.attn_in.copy_(p.attn_o)
    u2.step()
    torch.cuda.synchronize()
    assert torch.equal(p.qkv_out.view(torch.uint8), u2.qkv.view(torch.uint8))
    # live mask: a 2-slot ring of window masks = 2/C of the full mask
    B, H, S = cfg.batch, cfg.heads, cfg.seq
    assert p.mask.numel() == 2 * (B * H * S * S // 8) // chunks
    if mode in ("streams", "in_gemm"):
        # after a step, slot 0 holds window 0 (generated for the next step by the last
        # stage) and slot 1 window C-1 (C even) -- rows of the full layout's mask
        full = rgo.generate_mask_device(rgo.MaskLayout(B, H, S, seed), rgo.KeepThreshold(cfg.keep_prob),
                                        cfg.philox_rounds)[: B * H * S * S // 8].view(B * H, S, S // 8)
        Sc = S // chunks
        w0 = full[:, :Sc].reshape(-1)
        wl = full[:, (chunks - 1) * Sc:].reshape(-1)
        half = p.mask.numel() // 2
        assert torch.equal(p.mask[:half], w0)
        if chunks % 2 == 0:
            assert torch.equal(p.mask[half:], wl)
    for b in (u, p, u2):
        b.close()


@pytest.mark.parametrize("mode", ["serial_fused", "streams", "in_gemm"])
def test_seq_chunked_pipeline_matches_unchunked(rgo, cuda, mode):
    # (NO_RNG is a measurement floor: its ring holds windows 0 and 1 for good, so
    # windows >= 2 attend with a stale -- but real -- keep pattern)
    cfg = rgo.WorkloadConfig(batch=2, seq=1024, heads=4, head_dim=128, ffn_dim=384, gated=True, keep_prob=0.9,
                             philox_rounds=10)
    chunked_vs_unchunked(rgo, cfg, mode, 4)


@pytest.mark.parametrize("chunks", [2, 3, 8])
def test_seq_chunked_pipeline_chunk_counts(rgo, cuda, chunks):
    """Odd chunk counts (slot parity of the next step's window 0) and 128-row windows."""
    cfg = rgo.WorkloadConfig(batch=1, seq=1024 if chunks != 3 else 768, heads=2, head_dim=128, ffn_dim=256,
                             gated=False, keep_prob=0.85, philox_rounds=7)
    chunked_vs_unchunked(rgo, cfg, "in_gemm", chunks)
    chunked_vs_unchunked(rgo, cfg, "streams", chunks)


def test_seq_chunked_graph_replay_steady(rgo, cuda):
    """Replayed chunked steps recompute the same outputs (stationary input qkv)."""
    import torch
    cfg = rgo.WorkloadConfig(batch=1, seq=1024, heads=4, head_dim=128, ffn_dim=384, gated=True, keep_prob=0.9,
                             philox_rounds=10)
    for mode in ("streams", "in_gemm"):
        p = rgo.Block(cfg, mode, seed=5, chunks=4)
        p.step()
        torch.cuda.synchronize()
        a, q = p.attn_o.clone(), p.qkv_out.clone()
        for _ in range(3):
            p.step()
        torch.cuda.synchronize()
        assert torch.equal(p.attn_o, a) and torch.equal(p.qkv_out, q)
        p.close()


def test_pdl_chain_does_not_change_results(rgo, cuda):
    """The programmatic-dependent-launch chain (default) against plain stream
    order (RGO_BLOCK_PDL=0, read once per process: run in a subprocess)."""
    import hashlib
    import os
    import subprocess
    import sys
    code = r'''
import hashlib, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2410_07531_b200 as rgo
cfg = rgo.WorkloadConfig(batch=2, seq=512, heads=4, head_dim=128, ffn_dim=384, gated=True, keep_prob=0.9,
                         philox_rounds=10)
h = hashlib.sha256()
for mode in ("in_gemm", "no_rng", "serial_fused"):
    b = rgo.Block(cfg, mode, seed=42)
    b.step(); b.step()
    torch.cuda.synchronize()
    for k in ("x", "qkv", "attn_o", "y1", "h"):
        h.update(getattr(b, k).view(torch.uint8).cpu().numpy().tobytes())
    h.update(b.mask.cpu().numpy().tobytes())
    b.close()
print(h.hexdigest())
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for pdl in ("1", "0"):
        env = dict(os.environ, RGO_BLOCK_PDL=pdl)
        r = subprocess.run([sys.executable, "-c", code, root], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        out[pdl] = r.stdout.strip().splitlines()[-1]
    assert out["1"] == out["0"]


def test_random_configs_modes_identical(rgo, cuda):
    """Seeded random block configs: every overlap mode produces the serial-fused
    block's outputs bitwise, and mechanism A/B masks equal K1's."""
    import torch
    rng = np.random.default_rng(11)
    for case in range(5):
        cfg = rgo.WorkloadConfig(batch=int(rng.integers(1, 3)), seq=int(rng.choice([256, 384, 512, 640])),
                                 heads=int(rng.integers(2, 5)), head_dim=128,
                                 ffn_dim=int(rng.choice([256, 384, 512])), gated=bool(rng.integers(0, 2)),
                                 keep_prob=float(rng.choice([0.8, 0.9])), philox_rounds=int(rng.choice([7, 10])))
        seed = int(rng.integers(0, 2**40))
        outs = {}
        for mode in ("serial_fused", "streams", "in_gemm"):
            b = rgo.Block(cfg, mode, seed=seed)
            b.step()
            torch.cuda.synchronize()
            outs[mode] = (snapshot(b), b.mask.clone())
            b.close()
        for mode in ("streams", "in_gemm"):
            for k, v in outs[mode][0].items():
                assert torch.equal(v.view(torch.uint8), outs["serial_fused"][0][k].view(torch.uint8)), (cfg, mode, k)
        want = rgo.generate_mask_device(rgo.MaskLayout(cfg.batch, cfg.heads, cfg.seq, seed),
                                        rgo.KeepThreshold(cfg.keep_prob), cfg.philox_rounds)
        for mode in ("streams", "in_gemm"):
            assert torch.equal(outs[mode][1], want[: outs[mode][1].numel()]), (cfg, mode)


@pytest.mark.parametrize("rounds", [5, 3, 6, 12])
def test_reduced_round_in_gemm_block(rgo, cuda, rounds):
    """Philox-5/-3 (compiled drains) and 6/12 (runtime-rounds drain): the
    in-GEMM drains (and the matching inline-Philox baseline) keep the modes
    bitwise equal and the mask equal to K1's."""
    import torch
    cfg = rgo.WorkloadConfig(batch=2, seq=512, heads=4, head_dim=128, ffn_dim=384, gated=True, keep_prob=0.9,
                             philox_rounds=rounds)
    outs = {}
    for mode in ("serial_fused", "in_gemm"):
        b = rgo.Block(cfg, mode, seed=9)
        b.step()
        torch.cuda.synchronize()
        outs[mode] = (snapshot(b), b.mask.clone())
        b.close()
    for k, v in outs["in_gemm"][0].items():
        assert torch.equal(v.view(torch.uint8), outs["serial_fused"][0][k].view(torch.uint8)), k
    want = rgo.generate_mask_device(rgo.MaskLayout(2, 4, 512, 9), rgo.KeepThreshold(0.9), rounds)
    assert torch.equal(outs["in_gemm"][1], want[: outs["in_gemm"][1].numel()])


def test_block_rejects_threshold_edge_keep_prob(rgo, cuda):
    """keep_prob 0.99999999 is < 1 as a double but 1.0f as the float the
    reference stores (mask.hpp:59): threshold 2^32 cannot run through the
    in-GEMM queue's 32-bit compare, so creation fails instead of the modes
    silently disagreeing."""
    cfg = small_cfg(rgo)
    cfg.keep_prob = 0.99999999
    for mode in ("serial_fused", "streams", "in_gemm"):
        with pytest.raises(ValueError, match="threshold"):
            rgo.Block(cfg, mode, seed=1)


def test_block_rejects_bad_rng_warps(rgo, cuda):
    cfg = small_cfg(rgo)
    with pytest.raises(ValueError, match="RNG warps"):
        rgo.Block(cfg, "in_gemm", seed=1, rng_launch=(0, 10, 0))
