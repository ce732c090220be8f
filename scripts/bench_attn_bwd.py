"""Time the attention backward (K7) at the Llama2-7B shape (B4 H32 S4096 D128),
token-major QKV layout, per mask source; also the three kernels' split and
the parity of a smaller case against the float64 oracle."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import numpy as np
import torch
import paper_2410_07531_b200 as rgo

B, H, S, D = [int(x) for x in (sys.argv[1:5] if len(sys.argv) > 4 else (4, 32, 4096, 128))]
qkv = (torch.rand(B * S, 3 * H * D, device="cuda") * 2 - 1).bfloat16()
v4 = qkv.view(B, S, 3, H, D)
q, k, v = (v4[:, :, i].permute(0, 2, 1, 3) for i in range(3))
o = torch.empty(B, S, H, D, dtype=torch.bfloat16, device="cuda").permute(0, 2, 1, 3)
do = (torch.rand(B, S, H, D, device="cuda") * 2 - 1).bfloat16().permute(0, 2, 1, 3)
grads = [torch.empty(B, S, H, D, dtype=torch.bfloat16, device="cuda").permute(0, 2, 1, 3) for _ in range(3)]
lse = torch.empty(B * H * S, dtype=torch.float32, device="cuda")
lay = rgo.MaskLayout(B, H, S, 42)
bits = rgo.generate_mask_device(lay, rgo.KeepThreshold(0.9), 10)
need = rgo._lib.C.c_uint64()
work = None
flops_fwd = 4 * B * H * S * S * D
flops_bwd = 2.5 * flops_fwd
for name, kw in (("none", dict(mask_source=0)), ("bits", dict(mask_source=1, keep_prob=0.9, bits=bits)),
                 ("philox10", dict(mask_source=2, keep_prob=0.9, seed=42, rounds=10)),
                 ("philox7", dict(mask_source=2, keep_prob=0.9, seed=42, rounds=7))):
    rgo.attn_fwd(q, k, v, o, lse=lse, **kw)
    if work is None:
        _, _, _ = rgo.attn_bwd(q, k, v, o, do, lse, dq=grads[0], dk=grads[1], dv=grads[2], **kw)
        a = rgo._lib.attn_desc(B, H, S, D, 0.0, 0, 1.0, 0, 0, 10, 0)
        rgo._lib.check(rgo._lib.lib().rgo_attn_bwd_workspace(a, rgo._lib.C.byref(need)))
        work = torch.empty(need.value, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        rgo.attn_bwd(q, k, v, o, do, lse, dq=grads[0], dk=grads[1], dv=grads[2], work=work, **kw)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 10
    e0.record()
    for _ in range(n):
        rgo.attn_bwd(q, k, v, o, do, lse, dq=grads[0], dk=grads[1], dv=grads[2], work=work, **kw)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(json.dumps({"attn_bwd": name, "B": B, "H": H, "S": S, "D": D, "ms": round(ms, 4),
                      "tflops_2.5x": round(flops_bwd / ms / 1e9, 1)}), flush=True)

# parity record (smaller case)
import oracle
Bs, Hs, Ss, Ds = 1, 4, 1024, 128
g = torch.Generator().manual_seed(0)
t = [((torch.rand(Bs, Hs, Ss, Ds, generator=g) * 2 - 1)).bfloat16().cuda() for _ in range(4)]
t[0] = (t[0].float() * 3).bfloat16()
bits2 = rgo.generate_mask_device(rgo.MaskLayout(Bs, Hs, Ss, 7), rgo.KeepThreshold(0.9), 10)
l2 = torch.empty(Bs * Hs * Ss, device="cuda")
o2 = rgo.attn_fwd(t[0], t[1], t[2], mask_source=1, keep_prob=0.9, bits=bits2, lse=l2)
dq, dk, dv = rgo.attn_bwd(t[0], t[1], t[2], o2, t[3], l2, mask_source=1, keep_prob=0.9, bits=bits2)
keep = oracle.unpack_keep(bits2[: Bs * Hs * Ss * Ss // 8].cpu().numpy(), Bs * Hs, Ss)
f = lambda x: x.float().cpu().numpy().astype(np.float64)
want = oracle.attention_backward(*(f(x) for x in t), Bs * Hs, Ss, Ds, keep, 0.9)
got = [f(x).reshape(Bs * Hs, Ss, Ds) for x in (o2, dq, dk, dv)]
print(json.dumps({"parity": "B1 H4 S1024 D128 keep0.9 bits, rel Frobenius vs float64 oracle",
                  **{n: float(np.linalg.norm(a - b) / np.linalg.norm(b)) for n, a, b in
                     zip(("o", "dq", "dk", "dv"), got, want)}}))
