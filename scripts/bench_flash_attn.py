"""The installed flash-attn package (FA2, fused Philox dropout) at the Llama2-7B
attention shape: the library form of the conventional fused-dropout baseline."""
import json, os, sys
import torch

B, H, S, D = 4, 32, 4096, 128
try:
    from flash_attn import flash_attn_func
except Exception as e:  # noqa: BLE001
    print(json.dumps({"flash_attn": f"unavailable: {e}"[:200]}))
    sys.exit(0)
q, k, v = ((torch.rand(B, S, H, D, device="cuda") * 2 - 1).bfloat16().requires_grad_(True) for _ in range(3))
do = (torch.rand(B, S, H, D, device="cuda") * 2 - 1).bfloat16()
res = {}
for p in (0.0, 0.1):
    for _ in range(2):
        o = flash_attn_func(q, k, v, dropout_p=p)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    n = 5
    fwd = bwd = 0.0
    for _ in range(n):
        e0.record()
        o = flash_attn_func(q, k, v, dropout_p=p)
        e1.record()
        o.backward(do)
        e2.record()
        torch.cuda.synchronize()
        fwd += e0.elapsed_time(e1) / n
        bwd += e1.elapsed_time(e2) / n
    res[f"dropout_{p}"] = {"fwd_ms": round(fwd, 4), "bwd_ms": round(bwd, 4)}
import flash_attn
print(json.dumps({"flash_attn": flash_attn.__version__, "shape": "B4 S4096 H32 D128 bf16", **res}))
