"""Mechanism B: how many of the step's GEMMs should carry co-resident RNG
warps?  For each preset and RGO_RNG_GEMMS = k (first k GEMMs; 0 = all), time
the in-GEMM step against the no-RNG floor (graph replays, CUDA events,
interleaved; one child process per k since the variable is read once).

    python scripts/diag/rng_attach_sweep.py [presets...]
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r'''
import json, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_2410_07531_b200 as rgo
cfg = rgo.workload_preset(sys.argv[2]); cfg.philox_rounds = 10
w = rgo.block.make_weights(cfg, 42, torch.device("cuda"))
bl = {m: rgo.Block(cfg, m, seed=42, weights=w) for m in ("in_gemm", "no_rng", "streams")}
res = {m: [] for m in bl}
for rep in range(4):
    for m in (list(bl) if rep % 2 == 0 else list(bl)[::-1]):
        b = bl[m]
        for _ in range(5): b.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): b.step()
        e1.record(); torch.cuda.synchronize()
        res[m].append(e0.elapsed_time(e1) / 20)
print(json.dumps({m: round(sum(v) / len(v), 4) for m, v in res.items()}))
'''

if __name__ == "__main__":
    presets = sys.argv[1:] or ["gpt3", "llama2_7b", "moe"]
    for pr in presets:
        ks = (0, 1, 2, 3) if pr != "moe" else (0, 1, 2, 4, 8)
        for k in ks:
            env = dict(os.environ, RGO_RNG_GEMMS=str(k))
            r = subprocess.run([sys.executable, "-c", CHILD, ROOT, pr], env=env, capture_output=True, text=True,
                               timeout=600)
            out = r.stdout.strip().splitlines()[-1] if r.returncode == 0 else r.stderr[-300:]
            print(json.dumps({"preset": pr, "rng_gemms": k, "ms": json.loads(out) if r.returncode == 0 else out}),
                  flush=True)
