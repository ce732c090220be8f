"""Long-context backward sanity: S = 16K/32K, bits vs inline Philox agree (dK, dV bitwise)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_07531_b200 as rgo
for S in (16384, 32768):
    B, H, D = 1, 2, 128
    q, k, v, do = ((torch.rand(B, H, S, D, device="cuda") * 2 - 1).bfloat16() for _ in range(4))
    bits = rgo.generate_mask_device(rgo.MaskLayout(B, H, S, 5), rgo.KeepThreshold(0.9), 10)
    lse = torch.empty(B * H * S, device="cuda")
    o = rgo.attn_fwd(q, k, v, mask_source=1, keep_prob=0.9, bits=bits, lse=lse)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gb = rgo.attn_bwd(q, k, v, o, do, lse, mask_source=1, keep_prob=0.9, bits=bits)
    e1.record()
    gf = rgo.attn_bwd(q, k, v, o, do, lse, mask_source=2, keep_prob=0.9, seed=5, rounds=10)
    torch.cuda.synchronize()
    print(json.dumps({"S": S, "bwd_bits_ms": round(e0.elapsed_time(e1), 3),
                      "dk_equal": bool(torch.equal(gb[1], gf[1])), "dv_equal": bool(torch.equal(gb[2], gf[2])),
                      "dq_rel": float((gb[0].float() - gf[0].float()).norm() / gf[0].float().norm()),
                      "finite": bool(torch.isfinite(gb[0].float()).all())}))
