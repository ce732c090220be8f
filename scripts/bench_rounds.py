"""Stand-alone K1 mask runtime per Philox round count (Llama2-7B mask)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_07531_b200 as rgo

lay = rgo.MaskLayout(4, 32, 4096, 42)
out = torch.empty(lay.elem_count() // 8, dtype=torch.uint8, device="cuda")
res = {}
for rep in range(2):
    for R in ((3, 4, 5, 6, 7, 10) if rep == 0 else (10, 7, 6, 5, 4, 3)):
        for _ in range(3):
            rgo.generate_mask_device(lay, rgo.KeepThreshold(0.9), R, out=out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            rgo.generate_mask_device(lay, rgo.KeepThreshold(0.9), R, out=out)
        e1.record()
        torch.cuda.synchronize()
        res.setdefault(R, []).append(e0.elapsed_time(e1) / 10)
print(json.dumps({f"R{R}": round(sum(v) / len(v), 4) for R, v in sorted(res.items())}))
