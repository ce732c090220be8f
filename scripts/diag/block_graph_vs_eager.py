"""Block step time per mode, CUDA graph vs eager launches."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_07531_b200 as rgo

wl = rgo.workload_preset("llama2_7b")
w = rgo.block.make_weights(wl, 42, torch.device("cuda"))

def t(b, n=10):
    for _ in range(3):
        b.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        b.step()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / n, 4), [round(x, 4) for x in b.last_timings()]

for rep in range(2):
    for mode in ("no_rng", "in_gemm", "streams"):
        for graph in (True, False):
            b = rgo.Block(wl, mode, seed=42, weights=w, use_graph=graph,
                          rng_launch=(0, 8, 0) if mode == "in_gemm" else (0, 0, 0))
            ms, ph = t(b); ph = [round(x, 4) for x in b.last_timings3()]
            print(json.dumps({"mode": mode, "graph": graph, "ms": ms, "phases": ph}), flush=True)
            b.close()
