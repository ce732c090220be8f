"""Why is the block's attention phase slower than the stand-alone kernel?
Run NO_RNG steps, then time the same attention call on the block's own QKV /
mask buffers stand-alone, then on random inputs."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_07531_b200 as rgo

wl = rgo.workload_preset("llama2_7b")
b = rgo.Block(wl, "no_rng", seed=42)
B, H, S, D = 4, 32, 4096, 128
for _ in range(5):
    b.step()
torch.cuda.synchronize()
ph = b.last_timings3()
v4 = b.qkv.view(B, S, 3, H, D)
q, k, v = (v4[:, :, i].permute(0, 2, 1, 3) for i in range(3))
o = torch.empty(B, S, H, D, dtype=torch.bfloat16, device="cuda").permute(0, 2, 1, 3)

def t(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / n, 4)

own = t(lambda: rgo.attn_fwd(q, k, v, o, mask_source=1, keep_prob=0.9, bits=b.mask))
qf = q.float()
stats = {"q_std": float(qf.std()), "q_absmax": float(qf.abs().max()), "k_std": float(k.float().std()),
         "v_std": float(v.float().std()), "mask_ones": float(torch.unpackbits(b.mask[:1 << 20].cpu()).float().mean()) if hasattr(torch, "unpackbits") else None}
rq = (torch.rand_like(qf) * 2 - 1).bfloat16()
rk = (torch.rand_like(qf) * 2 - 1).bfloat16()
rv = (torch.rand_like(qf) * 2 - 1).bfloat16()
rnd = t(lambda: rgo.attn_fwd(rq, rk, rv, o, mask_source=1, keep_prob=0.9, bits=b.mask))
print(json.dumps({"in_step_phases": [round(x, 4) for x in ph], "standalone_on_block_qkv": own,
                  "standalone_random_qkv": rnd, **stats}))
