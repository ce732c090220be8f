"""Small invocation of every kernel, for compute-sanitizer (scripts/sanitize.sh):
K1, K2 (bf16 + FP8 with each epilogue), K4 (12 RNG warps) + queue tail, K5/K6
(mask bits by TMA), K7 (head dim 64 and 128, bits and Philox), K5g (head_dim 160),
an in-GEMM and a streams block step, an SQ-chunked step, and one rank of a
tensor-parallel step (emulated pair: the two-shot all-reduce kernels, the head-window
mask)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_07531_b200 as rgo

torch.manual_seed(0)
dev = "cuda"
lay = rgo.MaskLayout(1, 2, 384, 42)
thr = rgo.KeepThreshold(0.9)
bits = rgo.generate_mask_device(lay, thr, 10)                          # K1
f8 = torch.float8_e4m3fn
a = (torch.rand(256, 256, device=dev) - 0.5).bfloat16()
w = (torch.rand(512, 256, device=dev) - 0.5).bfloat16()
rgo.gemm(a, w)                                                         # K3
rgo.gemm(a.to(f8), w.to(f8), epilogue="swiglu", out_dtype=f8)          # K2
rgo.gemm(a.to(f8), w.to(f8), epilogue="gelu", out_dtype=f8)
d = rgo.mask.desc(lay, thr, 10)
qbits = torch.zeros_like(bits)
counter = torch.zeros(1, dtype=torch.int64, device=dev)
c = torch.empty(256, 512, dtype=torch.bfloat16, device=dev)
rgo.gemm_with_rng(a, w, c, d, qbits, counter, rng_warps=12)           # K4
rgo.mask_queue_drain(d, qbits, counter)
for D in (64, 128):
    B, H, S = 1, 2, 384
    q, k, v, do = ((torch.rand(B, H, S, D, device=dev) * 2 - 1).bfloat16() for _ in range(4))
    o = torch.empty_like(q)
    lse = torch.empty(B * H * S, device=dev)
    for kw in (dict(mask_source=1, keep_prob=0.9, bits=bits), dict(mask_source=2, keep_prob=0.9, seed=42, rounds=10)):
        rgo.attn_fwd(q, k, v, o, lse=lse, **kw)                        # K5 / K6
        rgo.attn_bwd(q, k, v, o, do, lse, **kw)                        # K7
cfg = rgo.WorkloadConfig(batch=1, seq=256, heads=2, head_dim=128, ffn_dim=256, gated=True, keep_prob=0.9,
                         philox_rounds=10)
for mode in ("in_gemm", "streams"):
    blk = rgo.Block(cfg, mode, seed=42, use_graph=False)
    blk.step()
    torch.cuda.synchronize()
    blk.close()
blk = rgo.Block(rgo.WorkloadConfig(batch=1, seq=512, heads=2, head_dim=128, ffn_dim=256, gated=True, keep_prob=0.9,
                                   philox_rounds=10), "in_gemm", seed=42, use_graph=False, chunks=2)
blk.step()
torch.cuda.synchronize()
blk.close()
tcfg = rgo.WorkloadConfig(batch=1, seq=256, heads=4, head_dim=128, ffn_dim=512, gated=True, keep_prob=0.9,
                          philox_rounds=10)
for mode in ("in_gemm", "serial_fused"):
    tb = rgo.TPBlock(tcfg, mode, seed=42, emulate=(2, 1))
    tb.step()
    torch.cuda.synchronize()
    tb.close()
inp = rgo.random_attention_input(2, 64, 160, 5)                        # K5g
rgo.attention_dropout_fused(inp, 42, 0.9, 10)
print("sanitize cases done")
