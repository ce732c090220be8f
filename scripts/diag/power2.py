"""Long back-to-back loops: GEMM alone, mask alone, both concurrently (two
streams), with clocks/power sampled every 10 ms (diagnostic)."""
import json, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_07531_b200 as rgo

M, N, K = 16384, 22016, 4096
a = (torch.rand(M, K, device="cuda") - 0.5).to(torch.float8_e4m3fn)
b = (torch.rand(N, K, device="cuda") - 0.5).to(torch.float8_e4m3fn)
c = torch.empty(M, N // 2, dtype=torch.float8_e4m3fn, device="cuda")
lay = rgo.MaskLayout(4, 32, 4096, 42)
bits = torch.empty(lay.elem_count() // 8, dtype=torch.uint8, device="cuda")
s_g, s_r = torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=0)
shape = tuple(int(x) for x in os.environ.get("RNG_SHAPE", "148,256").split(","))
ROUNDS = int(os.environ.get("ROUNDS", "10"))


def run(ng, nr):
    smp = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "10"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(s_g); r0.record(s_r)
    for i in range(max(ng, nr)):
        if i < ng:
            rgo.gemm(a, b, c, epilogue="swiglu", alpha=0.05, stream=s_g)
        if i < nr:
            rgo.generate_mask_device(lay, rgo.KeepThreshold(0.9), ROUNDS, out=bits, stream=s_r, grid=shape[0],
                                     block=shape[1])
    g1.record(s_g); r1.record(s_r)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) * 1e3
    smp.terminate()
    rows = [r.split(", ") for r in smp.communicate()[0].strip().splitlines() if r.strip()]
    clk = sorted(float(r[0]) for r in rows)
    pw = sorted(float(r[1]) for r in rows)
    return {"gemms": ng, "masks": nr, "wall_ms": round(wall, 2), "gemm_stream_ms": round(g0.elapsed_time(g1), 2),
            "rng_stream_ms": round(r0.elapsed_time(r1), 2), "sm_mhz_med": clk[len(clk) // 2] if clk else None,
            "power_med": pw[len(pw) // 2] if pw else None, "samples": len(rows), "rng_shape": shape}


for _ in range(3):
    rgo.gemm(a, b, c, epilogue="swiglu", alpha=0.05, stream=s_g)
torch.cuda.synchronize()
for ng, nr in ((40, 0), (0, 40), (40, 40), (40, 20)):
    print(json.dumps(run(ng, nr)), flush=True)
