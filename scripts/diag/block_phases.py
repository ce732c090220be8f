"""Per-phase timings (GEMM window / RNG tail or join / attention) of the
Llama2-7B block step per overlap mode and in-GEMM RNG warp count, modes
interleaved (forward then reverse order) so power state is shared."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_07531_b200 as rgo

wl = rgo.workload_preset(os.environ.get("PRESET", "llama2_7b"))
w = rgo.block.make_weights(wl, 42, torch.device("cuda"))
cfgs = [(m, (0, 0, 0)) for m in os.environ.get("MODES", "no_rng,streams,serial_fused").split(",") if m]
cfgs += [("in_gemm", (0, int(r), 0)) for r in os.environ.get("RW", "4,6,8").split(",")]
blocks = {c: rgo.Block(wl, c[0], seed=42, weights=w, rng_launch=c[1]) for c in cfgs}
acc = {c: [] for c in cfgs}
for order in [cfgs, cfgs[::-1]] * int(os.environ.get("REPS", "2")):
    for c in order:
        b = blocks[c]
        for _ in range(3):
            b.step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            b.step()
        e1.record()
        torch.cuda.synchronize()
        t3 = b.last_timings3()
        acc[c].append((e0.elapsed_time(e1) / 10, *t3))
for c in cfgs:
    v = acc[c]
    mean = [sum(x[i] for x in v) / len(v) for i in range(4)]
    print(json.dumps({"mode": c[0], "rng_warps": c[1][1], "ms": round(mean[0], 4), "gemm_window": round(mean[1], 4),
                      "tail": round(mean[2], 4), "attention": round(mean[3], 4),
                      "ms_samples": [round(x[0], 3) for x in v]}), flush=True)
