"""Per-CTA phase timestamps of the attention forward (diagnostic build with
-DRGO_FWD_TIMING, selected through RGO_LIB_PATH): prologue, pipeline fill,
KV loop, last PV, epilogue, teardown, and the gap before the next CTA on the
same SM.  usage: RGO_LIB_PATH=.../timing.so python scripts/diag/fwd_timing.py [B H S]"""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
import paper_2410_07531_b200 as rgo

B, H, S = [int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (4, 32, 4096))]
D = 128
qkv = (torch.rand(B * S, 3 * H * D, device="cuda") * 2 - 1).bfloat16()
v4 = qkv.view(B, S, 3, H, D)
q, k, v = (v4[:, :, i].permute(0, 2, 1, 3) for i in range(3))
o = torch.empty(B, S, H, D, dtype=torch.bfloat16, device="cuda").permute(0, 2, 1, 3)
bits = rgo.generate_mask_device(rgo.MaskLayout(B, H, S, 42), rgo.KeepThreshold(0.9), 10)
n_cta = B * H * ((S + 255) // 256)
dbg = torch.zeros(n_cta * 8, dtype=torch.int64, device="cuda")
lib = rgo._lib.lib()
lib.rgo_debug_fwd_timing.argtypes = [C.c_void_p]
for name, kw in (("none", dict(mask_source=0)), ("bits", dict(mask_source=1, keep_prob=0.9, bits=bits))):
    for _ in range(3):
        rgo.attn_fwd(q, k, v, o, **kw)
    torch.cuda.synchronize()
    assert lib.rgo_debug_fwd_timing(C.c_void_p(dbg.data_ptr())) == 0
    rgo.attn_fwd(q, k, v, o, **kw)
    torch.cuda.synchronize()
    assert lib.rgo_debug_fwd_timing(C.c_void_p(0)) == 0
    t = dbg.view(n_cta, 8).cpu().numpy().astype(np.int64)
    t0 = t[:, 0].min()
    ph = {"prologue": t[:, 1] - t[:, 0], "fill(first S)": t[:, 2] - t[:, 1], "kv loop": t[:, 3] - t[:, 2],
          "last PV": t[:, 4] - t[:, 3], "epilogue": t[:, 5] - t[:, 4], "teardown": t[:, 6] - t[:, 5],
          "cta total": t[:, 6] - t[:, 0]}
    gaps = []
    for sm in np.unique(t[:, 7]):
        idx = np.where(t[:, 7] == sm)[0]
        idx = idx[np.argsort(t[idx, 0])]
        gaps += list(t[idx[1:], 0] - t[idx[:-1], 6])
    out = {k: round(float(np.mean(v)) / 1e3, 3) for k, v in ph.items()}
    out["gap to next CTA on SM"] = round(float(np.mean(gaps)) / 1e3, 3) if gaps else None
    out["kernel span"] = round(float(t[:, 6].max() - t0) / 1e3, 3)
    out["ctas"] = int(n_cta)
    print(json.dumps({"attn": name, "B": B, "H": H, "S": S, "us": out}), flush=True)
