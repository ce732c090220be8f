"""Why can the pipelined e2e loop be faster than the plain step loop?  Time
the plain loop, the e2e loop and the plain loop again, and a two-replica
plain loop (no copies)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_07531_b200 as rgo

wl = rgo.workload_preset("llama2_7b")
w = rgo.block.make_weights(wl, 42, torch.device("cuda"))
a = rgo.Block(wl, "in_gemm", seed=42, weights=w, rng_launch=(0, 8, 0))
b = rgo.Block(wl, "in_gemm", seed=42, weights=w, rng_launch=(0, 8, 0))
s = torch.cuda.current_stream()

def timeit(fn, n=20):
    for _ in range(3):
        fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(n):
        fn(k)
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / n, 4)

print(json.dumps({
    "single": timeit(lambda k: a.step()),
    "alternate_two": timeit(lambda k: (a if k % 2 == 0 else b).step()),
    "single_again": timeit(lambda k: a.step()),
    "alternate_again": timeit(lambda k: (a if k % 2 == 0 else b).step()),
}))
