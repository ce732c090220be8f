"""Is the attention (or the tail drain) slower right after the GEMM window?  Time
each piece of an in-GEMM block step with events, eagerly: 4 GEMMs with RNG
warps -> tail drain -> attention, vs the same attention after plain GEMMs."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_07531_b200 as rgo

M, d, F, B, H, S, D = 16384, 4096, 11008, 4, 32, 4096, 128
f8 = torch.float8_e4m3fn
mk = lambda r, c: (torch.rand(r, c, device="cuda") - 0.5).to(f8)
gem = [(mk(M, d), mk(d, d), "none", d), (mk(M, d), mk(2 * F, d), "swiglu", F), (mk(M, F), mk(d, F), "none", d),
       (mk(M, d), mk(3 * d, d), "none", 3 * d)]
outs = [torch.empty(M, n, dtype=f8, device="cuda") for *_, n in gem]
lay = rgo.MaskLayout(B, H, S, 42)
desc = rgo.mask.desc(lay, rgo.KeepThreshold(0.9), 10)
bits = torch.empty(lay.elem_count() // 8, dtype=torch.uint8, device="cuda")
counter = torch.zeros(1, dtype=torch.int64, device="cuda")
qkv = (torch.rand(B * S, 3 * H * D, device="cuda") * 2 - 1).bfloat16()
v4 = qkv.view(B, S, 3, H, D)
q, k, v = (v4[:, :, i].permute(0, 2, 1, 3) for i in range(3))
o = torch.empty(B, S, H, D, dtype=torch.bfloat16, device="cuda").permute(0, 2, 1, 3)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for rep in range(4):
    rng = rep % 2 == 0
    counter.zero_()
    ev[0].record()
    for (a, b, epi, n), c in zip(gem, outs):
        if rng:
            rgo.gemm_with_rng(a, b, c, desc, bits, counter, epilogue=epi, alpha=0.01)
        else:
            rgo.gemm(a, b, c, epilogue=epi, alpha=0.01)
    ev[1].record()
    if rng:
        rgo.mask_queue_drain(desc, bits, counter)
    ev[2].record()
    rgo.attn_fwd(q, k, v, o, mask_source=1, keep_prob=0.9, bits=bits)
    ev[3].record()
    torch.cuda.synchronize()
    print(json.dumps({"rng": rng, "gemms": round(ev[0].elapsed_time(ev[1]), 4), "tail": round(ev[1].elapsed_time(ev[2]), 4),
                      "attn": round(ev[2].elapsed_time(ev[3]), 4)}))
