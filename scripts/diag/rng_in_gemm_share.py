"""How much of the Llama2-7B mask the in-GEMM RNG warps produce during each of
the block's four FP8 GEMMs (mechanism B), run back to back like the block step."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_07531_b200 as rgo

M, d, F = 16384, 4096, 11008
f8 = torch.float8_e4m3fn
mk = lambda r, c: (torch.rand(r, c, device="cuda") - 0.5).to(f8)
shapes = [("Proj", mk(M, d), mk(d, d), "none", d), ("FFN1", mk(M, d), mk(2 * F, d), "swiglu", F),
          ("FFN2", mk(M, F), mk(d, F), "none", d), ("QKV", mk(M, d), mk(3 * d, d), "none", 3 * d)]
lay = rgo.MaskLayout(4, 32, 4096, 42)
desc = rgo.mask.desc(lay, rgo.KeepThreshold(0.9), 10)
bits = torch.empty(lay.elem_count() // 8, dtype=torch.uint8, device="cuda")
counter = torch.zeros(1, dtype=torch.int64, device="cuda")
total = lay.elem_count() // 128
for rep in range(3):
    counter.zero_()
    out = []
    for name, a, b, epi, n_out in shapes:
        c = torch.empty(M, n_out, dtype=f8, device="cuda")
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        before = int(counter.item())
        e0.record()
        rgo.gemm_with_rng(a, b, c, desc, bits, counter, epilogue=epi, alpha=0.01)
        e1.record()
        torch.cuda.synchronize()
        out.append({"gemm": name, "ms": round(e0.elapsed_time(e1), 4),
                    "share": round((min(int(counter.item()), total) - before) / total, 4)})
    print(json.dumps({"rep": rep, "gemms": out, "total_share": round(min(int(counter.item()), total) / total, 4)}))
