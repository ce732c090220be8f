"""Time the attention forward at the Llama2-7B shape (B4 H32 S4096 D128),
token-major QKV layout, for each mask source."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_07531_b200 as rgo

B, H, S, D = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (4, 32, 4096, 128))]
qkv = (torch.rand(B * S, 3 * H * D, device="cuda") * 2 - 1).bfloat16()
v4 = qkv.view(B, S, 3, H, D)
q, k, v = (v4[:, :, i].permute(0, 2, 1, 3) for i in range(3))
o = torch.empty(B, S, H, D, dtype=torch.bfloat16, device="cuda").permute(0, 2, 1, 3)
lay = rgo.MaskLayout(B, H, S, 42)
bits = rgo.generate_mask_device(lay, rgo.KeepThreshold(0.9), 10)
flops = 4 * B * H * S * S * D
for name, kw in (("none", dict(mask_source=0)), ("bits", dict(mask_source=1, keep_prob=0.9, bits=bits)),
                 ("philox10", dict(mask_source=2, keep_prob=0.9, seed=42, rounds=10)),
                 ("philox7", dict(mask_source=2, keep_prob=0.9, seed=42, rounds=7))):
    for _ in range(3):
        rgo.attn_fwd(q, k, v, o, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n):
        rgo.attn_fwd(q, k, v, o, **kw)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(json.dumps({"attn": name, "B": B, "H": H, "S": S, "D": D, "ms": round(ms, 4),
                      "tflops": round(flops / ms / 1e9, 1)}), flush=True)
