"""bench.py -- Llama2-7B dropout-RNG pipeline on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload mask]

One JSON line on rank 0.  Under torchrun each rank runs its own replica with a
disjoint Philox counter range (weak scaling, no collective on the data path).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Llama2-7B block (BASELINE.json configs[1]).
L_CFG = dict(batch=4, seq=4096, heads=32, head_dim=128, d_model=4096, ffn=11008, keep_prob=0.9, rounds=10)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.samples, self._stop = index, [], threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i] == "Active"})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# --------------------------------------------------------------- CPU side
def cpu_mask_baseline(cfg, kind="port", target_s=10.0):
    """generate_mask on the host cores on a bounded sample (whole (b,h)
    slices of the Llama2 mask), all hardware threads.  kind "reference" runs
    the reference compiled in place (oracle/_ref), "port" the C oracle."""
    import numpy as np
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    cores = os.cpu_count() or 1
    S = cfg["seq"]
    per_slice = S * S
    thr, _ = oracle.keep_threshold(cfg["keep_prob"])
    buf = np.zeros(per_slice * 64 // 8, np.uint8)

    def run(slices):
        if kind == "reference" and oracle.ref_available():
            r = oracle.ref()
            t0 = time.perf_counter()
            rc = r.ref_generate_mask(1, slices, S, 42, 0, cfg["keep_prob"], cfg["rounds"], cores, buf, buf.size)
            assert rc == 0
        else:
            t0 = time.perf_counter()
            oracle.lib().oracle_generate_mask(slices * per_slice, 42, 0, thr, cfg["rounds"], cores, buf, buf.size)
        return time.perf_counter() - t0

    t1 = run(1)
    slices = int(max(1, min(64, target_s / max(t1, 1e-6))))
    dt = run(slices)
    elems = slices * per_slice
    return {"value": elems / dt / 1e9, "unit": "Gbit/s", "cores": cores,
            "kind": "reference" if (kind == "reference" and oracle.ref_available()) else "port",
            "sample": f"generate_mask over {slices} of {cfg['batch'] * cfg['heads']} (b,h) slices "
                      f"(SQ {S}, R{cfg['rounds']}, keep {cfg['keep_prob']}), {dt:.2f} s",
            "seconds": dt, "elements": elems}


# --------------------------------------------------------------- GPU side
def bench_mask(args, rank, world):
    """K1 alone at the Llama2-7B shape: mask Gbit/s."""
    import torch
    import paper_2410_07531_b200 as rgo
    cfg = dict(L_CFG)
    cfg["rounds"] = args.rounds
    B, H, S = cfg["batch"], cfg["heads"], cfg["seq"]
    elems = B * H * S * S
    # disjoint counter range per rank: rank r is batch replica r
    lay = rgo.MaskLayout(B, H, S, 42, rank * elems // 4)
    thr = rgo.KeepThreshold(cfg["keep_prob"])
    out = torch.empty(elems // 8, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    for _ in range(args.warmup):
        rgo.generate_mask_device(lay, thr, args.rounds, out=out)
    torch.cuda.synchronize()
    barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        torch.cuda.synchronize()
        barrier(world)
        ev0.record(s)
        for _ in range(args.steps):
            rgo.generate_mask_device(lay, thr, args.rounds, out=out)  # 256 MiB output > L2
        ev1.record(s)
        torch.cuda.synchronize()
        barrier(world)
    ms = ev0.elapsed_time(ev1) / args.steps
    ms = max_over_ranks(ms, world)
    gbit = elems * world / (ms * 1e-3) / 1e9
    peaks, src = load_peaks()
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    int_peak = 148 * 128 * sm_mhz * 1e6  # INT32 lanes x clock (op/s)
    ops = elems * (args.rounds + 2)
    achieved = ops / (ms * 1e-3)
    # e2e: through the drop-in host API (D2H of the bits inside the timing)
    t0 = time.perf_counter()
    mk = rgo.generate_mask(lay, thr, args.rounds)
    e2e_s = time.perf_counter() - t0
    line = {
        "metric": "mask_gbit_s", "value": round(gbit, 2), "unit": "Gbit/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": f"Llama2-7B dropout mask B{B} nH{H} SQ{S} keep{cfg['keep_prob']} R{args.rounds}",
                   "l2": "output 256 MiB > L2 (no flush needed)"},
        "roofline": {"bound": "int", "achieved": achieved / 1e12, "peak": int_peak / 1e12, "unit": "Tint-op/s",
                     "frac": achieved / int_peak, "traffic": None,
                     "note": f"(R+2) int ops/element; peak = 148 SMs x 128 INT32 lanes x {sm_mhz} MHz ({src} clock)"},
        "hbm_write_gbs": elems / 8 / (ms * 1e-3) / 1e9,
        "e2e": {"value": round(elems / e2e_s / 1e9, 2), "unit": "Gbit/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": int(mk.bits.size)},
        "clocks": clk.summary(), "gpu_launches": args.steps,
    }
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="mask", choices=["mask"])
    ap.add_argument("--rounds", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        if rank != 0:
            return
        cfg = dict(L_CFG, rounds=args.rounds)
        vals = [cpu_mask_baseline(cfg, "reference", target_s=5.0) for _ in range(max(1, args.steps // 10))]
        v = sum(x["value"] for x in vals) / len(vals)
        b = vals[-1]
        print(json.dumps({"metric": "mask_gbit_s", "value": round(v, 4), "unit": "Gbit/s", "n_gpus": 0,
                          "impl": "reference", "steps": len(vals), "warmup": 0, "higher_is_better": True,
                          "config": {"workload": f"Llama2-7B dropout mask R{args.rounds} (sampled slices)"},
                          "cpu_baseline": {"value": round(v, 4), "unit": "Gbit/s", "cores": b["cores"],
                                           "kind": b["kind"], "sample": b["sample"]},
                          "e2e": {"value": round(v, 4), "unit": "Gbit/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return

    rank, world, _ = dist_setup()
    line = bench_mask(args, rank, world)
    if rank == 0:
        if not args.no_cpu_baseline:
            cb = cpu_mask_baseline(dict(L_CFG, rounds=args.rounds), "reference")
            line["cpu_baseline"] = {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
