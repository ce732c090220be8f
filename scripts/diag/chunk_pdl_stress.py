"""Stress the SQ-chunk pipeline with programmatic dependent launch on
(RGO_CHUNK_PDL=1) against the plain-stream-order chain: every mode at the
Llama2-7B shape (C = 4) runs `steps` graph replays and `steps` eager steps in a
child process under a timeout; a hang is reported as such (the child is killed),
and the outputs must hash the same with and without PDL.

    python scripts/diag/chunk_pdl_stress.py [steps]
"""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CHILD = r'''
import hashlib, sys, time, torch
sys.path.insert(0, sys.argv[1])
import paper_2410_07531_b200 as rgo
mode, steps, graph, C = sys.argv[2], int(sys.argv[3]), sys.argv[4] == "1", int(sys.argv[5])
cfg = rgo.workload_preset("llama2_7b")
b = rgo.Block(cfg, mode, seed=42, chunks=C, use_graph=graph)
t0 = time.time()
for i in range(steps):
    b.step()
    if i % 50 == 0:
        torch.cuda.synchronize()
torch.cuda.synchronize()
h = hashlib.sha256()
for t in (b.attn_o, b.qkv_out, b.mask):
    h.update(t.view(torch.uint8).cpu().numpy().tobytes())
print(h.hexdigest(), round(time.time() - t0, 2))
'''


def run(mode, steps, graph, pdl, C=4, timeout=180):
    env = dict(os.environ, RGO_CHUNK_PDL="1" if pdl else "0")
    try:
        r = subprocess.run([sys.executable, "-c", CHILD, ROOT, mode, str(steps), "1" if graph else "0", str(C)],
                           env=env, capture_output=True, text=True, timeout=timeout)
    except subprocess.TimeoutExpired:
        return {"status": "HANG", "timeout_s": timeout}
    if r.returncode != 0:
        return {"status": "ERROR", "stderr": r.stderr[-500:]}
    digest, secs = r.stdout.split()[-2:]
    return {"status": "ok", "hash": digest[:16], "s": float(secs)}


if __name__ == "__main__":
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    for mode in ("streams", "in_gemm", "serial_fused", "no_rng"):
        for graph in (True, False):
            off = run(mode, 5, graph, False)
            on = run(mode, steps, graph, True)
            same = off.get("hash") == on.get("hash")
            print(json.dumps({"mode": mode, "graph": graph, "pdl_off": off, "pdl_on": on, "same_output": same}),
                  flush=True)
