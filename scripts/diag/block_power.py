"""Per block mode: run ~1.5 s of steps, sample nvidia-smi clocks/power at 20 ms (diagnostic)."""
import json, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2410_07531_b200 as rgo

wl = rgo.WorkloadConfig(batch=4, seq=4096, heads=32, head_dim=128, ffn_dim=11008, gated=True, keep_prob=0.9,
                        philox_rounds=10)
weights = rgo.block.make_weights(wl, 42, torch.device("cuda"))
for mode in ("no_rng", "serial_fused", "in_gemm", "streams"):
    b = rgo.Block(wl, mode, seed=42, weights=weights, rng_launch=(148, 128, 0) if mode == "streams" else (0, 0, 0))
    for _ in range(5):
        b.step()
    torch.cuda.synchronize()
    smp = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                            "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    n = 300
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        b.step()
    e1.record()
    torch.cuda.synchronize()
    time.sleep(0.05)
    smp.terminate()
    rows = [r.split(", ") for r in smp.communicate()[0].strip().splitlines() if r.strip()]
    rows = rows[15:-3] if len(rows) > 25 else rows
    clk = sorted(float(r[0]) for r in rows)
    pw = sorted(float(r[1]) for r in rows)
    cap = sum(r[2].strip() == "Active" for r in rows) / max(1, len(rows))
    ph = b.last_timings()
    print(json.dumps({"mode": mode, "ms": round(e0.elapsed_time(e1) / n, 4), "gemm_window": round(ph[0], 4),
                      "attention": round(ph[1], 4), "sm_mhz_med": clk[len(clk) // 2], "sm_mhz_p10": clk[len(clk) // 10],
                      "power_med": pw[len(pw) // 2], "power_cap_frac": round(cap, 2), "samples": len(rows)}), flush=True)
    b.close()
