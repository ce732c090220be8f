"""Rasterisation-group sweep of the block's FP8 GEMMs (the
B operand is re-streamed once per GROUP_M group).  For each group size (passed
to the library through RGO_GEMM_GROUP_M, read once per process, so one
subprocess per value) time the four Llama2-7B GEMMs back to back on
unit-variance e4m3 data.  Under ncu (--metrics dram__bytes_read.sum) the same
script gives the DRAM reads per launch.

    python scripts/diag/gemm_group_sweep.py [groups...]      # sweep, JSON lines
    python scripts/diag/gemm_group_sweep.py --one            # one pass at $RGO_GEMM_GROUP_M
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)


def one(reps=20):
    import torch
    import paper_2410_07531_b200 as rgo
    cfg = rgo.workload_preset("llama2_7b")
    f8 = torch.float8_e4m3fn
    out = {"group_m": int(os.environ.get("RGO_GEMM_GROUP_M", "0"))}
    for sh in rgo.gemm_shapes(cfg):
        g = torch.Generator(device="cuda").manual_seed(sh.m + sh.n + sh.k)
        a = ((torch.rand(sh.m, sh.k, device="cuda", generator=g) * 2 - 1) * 1.7).to(f8)
        b = ((torch.rand(sh.n, sh.k, device="cuda", generator=g) * 2 - 1) * 1.7).to(f8)
        epi = "swiglu" if sh.name.startswith("FFN1") else "none"
        out_dt = torch.bfloat16 if sh.name == "QKV" else f8
        c = torch.empty(sh.m, sh.n // 2 if epi == "swiglu" else sh.n, dtype=out_dt, device="cuda")
        for _ in range(3):
            rgo.gemm(a, b, c, epilogue=epi, alpha=1.0 / sh.k)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            rgo.gemm(a, b, c, epilogue=epi, alpha=1.0 / sh.k)
        e1.record()
        torch.cuda.synchronize()
        out[sh.name] = round(e0.elapsed_time(e1) / reps, 4)
        del a, b, c
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    if "--one" in sys.argv:
        one()
    else:
        groups = [int(x) for x in sys.argv[1:]] or [8, 16, 24, 32, 48, 64]
        for rep in range(2):
            for gm in groups:
                env = dict(os.environ, RGO_GEMM_GROUP_M=str(gm))
                subprocess.run([sys.executable, __file__, "--one"], env=env, check=True)
