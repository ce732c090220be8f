"""Diagnose GEMM/RNG co-run: per-kernel times alone vs concurrent, with
nvidia-smi clocks/power sampled at 20 ms."""
import json, os, subprocess, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_07531_b200 as rgo


class Sampler:
    def __init__(self):
        self.s, self.stop = [], threading.Event()
        self.p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap,"
                                   "clocks_event_reasons.hw_slowdown", "--format=csv,noheader,nounits", "-lms", "20"],
                                  stdout=subprocess.PIPE, text=True)

    def close(self):
        self.p.terminate()
        out = self.p.communicate()[0]
        rows = [r.split(", ") for r in out.strip().splitlines() if r.strip()]
        return rows


def summarize(rows):
    if not rows:
        return {}
    clk = sorted(float(r[0]) for r in rows)
    pw = sorted(float(r[1]) for r in rows)
    cap = sum(1 for r in rows if r[2].strip() == "Active")
    return {"n": len(rows), "sm_mhz_med": clk[len(clk) // 2], "sm_mhz_min": clk[0], "power_med": pw[len(pw) // 2],
            "power_max": pw[-1], "power_cap_frac": round(cap / len(rows), 2)}


M, N, K = 16384, 22016, 4096
a = (torch.rand(M, K, device="cuda") - 0.5).to(torch.float8_e4m3fn)
b = (torch.rand(N, K, device="cuda") - 0.5).to(torch.float8_e4m3fn)
c = torch.empty(M, N // 2, dtype=torch.float8_e4m3fn, device="cuda")
lay = rgo.MaskLayout(4, 32, 4096, 42)
thr = rgo.KeepThreshold(0.9)
bits = torch.empty(lay.elem_count() // 8, dtype=torch.uint8, device="cuda")
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
s_g = torch.cuda.Stream(priority=-1)
s_r = torch.cuda.Stream(priority=0)
shape = tuple(int(x) for x in os.environ.get("RNG_SHAPE", "148,256").split(","))


def gemm():
    rgo.gemm(a, b, c, epilogue="swiglu", alpha=0.05, stream=s_g)


def rng():
    rgo.generate_mask_device(lay, thr, 10, out=bits, stream=s_r, grid=shape[0], block=shape[1])


def timed_loop(fns, seconds=1.5):
    # each fn: (callable, stream); run round-robin until time elapses; return per-fn avg ms via events
    torch.cuda.synchronize()
    evs = {i: [] for i in range(len(fns))}
    t_end = time.time() + seconds
    while time.time() < t_end:
        for i, (fn, st) in enumerate(fns):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            evs[i].append((e0, e1))
        torch.cuda.synchronize()
    return [sum(x.elapsed_time(y) for x, y in v[2:]) / max(1, len(v) - 2) for v in evs.values()]


for _ in range(3):
    gemm(); rng()
torch.cuda.synchronize()
for name, fns in (("gemm_alone", [(gemm, s_g)]), ("rng_alone", [(rng, s_r)]),
                  ("both", [(gemm, s_g), (rng, s_r)]), ("gemm_alone2", [(gemm, s_g)])):
    smp = Sampler()
    time.sleep(0.1)
    ms = timed_loop(fns)
    rows = smp.close()
    print(json.dumps({"case": name, "ms": [round(x, 4) for x in ms], "rng_shape": shape, **summarize(rows)}), flush=True)
