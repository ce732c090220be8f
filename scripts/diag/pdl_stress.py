"""Stress the PDL chain: many back-to-back block steps per mode (eager and graph),
Llama2-7B shape; prints per-mode completion."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_07531_b200 as rgo
wl = rgo.workload_preset(os.environ.get("PRESET", "llama2_7b"))
w = rgo.block.make_weights(wl, 42, torch.device("cuda"))
n = int(os.environ.get("STEPS", "200"))
modes = os.environ.get("MODES", "streams,in_gemm,no_rng,serial_fused").split(",")
graphs = [g == "graph" for g in os.environ.get("GRAPHS", "graph,eager").split(",")]
for mode in modes:
    for graph in graphs:
        b = rgo.Block(wl, mode, seed=42, weights=w, use_graph=graph)
        t = time.time()
        for i in range(n):
            b.step()
            if os.environ.get("SYNC_EVERY"):
                torch.cuda.synchronize()
                if i % 50 == 0:
                    print(mode, "graph" if graph else "eager", "step", i, flush=True)
        torch.cuda.synchronize()
        b.close()
        print(mode, "graph" if graph else "eager", n, "steps ok", round(time.time() - t, 2), "s", flush=True)
