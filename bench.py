"""bench.py -- Llama2-7B transformer block with attention dropout on B200.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload block|mask]

Headline (BASELINE.json metric "Llama2 block ms & speedup (RNG hidden vs fused
dropout); mask Gbit/s"): ms per steady-state block step (Proj+FFN1+FFN2 of
block L-1, QKV of block L, attention of block L; FP8 GEMMs, bf16 attention,
keep 0.9, Philox-10) with the dropout RNG hidden under the GEMMs, the same step
with Philox fused into attention (the baseline), their ratio, and the
stand-alone mask kernel's Gbit/s.  One JSON line on rank 0.  Under torchrun
each rank runs its own block replica with a disjoint Philox counter range
(weak scaling; no collective on the data path; timing = max over ranks).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Llama2-7B block (BASELINE.json configs[1]): batch 4, seq 4096, 32 heads, d 4096, FFN 11008 (SwiGLU).
L = dict(batch=4, seq=4096, heads=32, head_dim=128, ffn=11008, keep_prob=0.9, rounds=10)


# The headline line once the main measurement is complete (extras are added to the same
# dict as they finish) and the section running now: the watchdog prints the line it has
# rather than losing the headline to a wedged extra.
_PARTIAL = {"line": None, "section": None, "since": time.time()}


def log(msg):
    """Progress on stderr (the JSON line is the only stdout output)."""
    _PARTIAL["section"] = msg
    _PARTIAL["since"] = time.time()
    if int(os.environ.get("RANK", "0")) == 0:
        print(f"[bench {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

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
                fields = [x.strip() for x in out.split(",")] if out else []
                if len(fields) == 7:  # skip error text (e.g. an index with no device)
                    self.samples.append(fields)
            except Exception:
                pass
            self._stop.wait(0.02)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = sorted(v for v in (num(s[0]) for s in self.samples) if v is not None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if len(s) > 3 + i and s[3 + i] == "Active"})
        pw = [v for v in (num(s[2]) for s in self.samples) if v is not None]
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": num(self.samples[0][1]),
                "reasons": reasons, "power_w_max": max(pw) if pw else None, "samples": len(self.samples)}


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        # one process per GPU; BENCH_DIST_BACKEND=gloo with more ranks than GPUs
        # lets the multi-rank code paths be exercised on a single device
        dev = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(dev)
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            # communicator set-up visible in the log (ranks, NVLS/P2P transport); NCCL
            # carries only the max-over-ranks timing scalars -- no data-path collective
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
        t = torch.ones(1, device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t)  # create the communicator now, outside any timed region
        assert int(t.item()) == world
    else:
        torch.cuda.set_device(0)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    from paper_2410_07531_b200.sharding import max_over_ranks as mor
    return x if world == 1 else mor(x)


# --------------------------------------------------------------------- CPU side
def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    return oracle


def cpu_reference_block(cfg, target_s=10.0, kind="reference"):
    """The reference's CPU path for this workload, on this host's cores:
    generate_mask (mask.hpp:142-179, all threads) over a sample of (b,h)
    slices, and attention_dropout_fused (ref_attention.hpp:114-126), one slice
    per core in parallel (base_offset = s*SQ^2/4, bitwise identical to that
    slice of the full run).  Extrapolated to the full B*nH slices.  The
    reference has no GEMM arithmetic (workload.hpp:44-52 are shapes only), so
    the GEMM part of the block is absent from this number."""
    import numpy as np
    oracle = _oracle()
    use_ref = kind == "reference" and oracle.ref_available()
    cores = os.cpu_count() or 1
    S, D, slices = cfg["seq"], cfg["head_dim"], cfg["batch"] * cfg["heads"]
    thr, _ = oracle.keep_threshold(cfg["keep_prob"])
    # mask: time a sample of whole slices with all threads
    per_slice = S * S
    ms_slices = max(1, min(slices, int(2 ** 31 // per_slice // 8) or 1))
    buf = np.zeros(ms_slices * per_slice // 8, np.uint8)
    t0 = time.perf_counter()
    if use_ref:
        assert oracle.ref().ref_generate_mask(1, ms_slices, S, 42, 0, cfg["keep_prob"], cfg["rounds"], cores, buf,
                                              buf.size) == 0
    else:
        oracle.lib().oracle_generate_mask(ms_slices * per_slice, 42, 0, thr, cfg["rounds"], cores, buf, buf.size)
    t_mask = (time.perf_counter() - t0) * slices / ms_slices
    # fused attention: one slice per core (bounded sample)
    q, k, v = oracle.random_attention_input(1, S, D, 42 ^ 0xA77E)
    n_att = min(cores, slices)

    def one(s):
        o = np.zeros_like(q)
        if use_ref:
            rc = oracle.ref().ref_attention(1, S, D, q, k, v, 1, 42, s * per_slice // 4, cfg["keep_prob"],
                                            cfg["rounds"], o)
        else:
            rc = oracle.lib().oracle_attention(1, S, D, q, k, v, 1, 42, s * per_slice // 4, thr,
                                               np.float32(cfg["keep_prob"]), cfg["rounds"], None, 0, 1, o)
        assert rc == 0
        return o

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(n_att) as ex:
        list(ex.map(one, range(n_att)))
    t_att_wall = time.perf_counter() - t0
    t_att = t_att_wall * slices / n_att
    ms = (t_mask + t_att) * 1e3
    return {"value": ms, "unit": "ms", "cores": cores, "kind": "reference" if use_ref else "port",
            "sample": f"generate_mask {ms_slices}/{slices} slices + attention_dropout_fused {n_att}/{slices} slices "
                      f"(SQ {S}, dH {D}, keep {cfg['keep_prob']}, Philox-{cfg['rounds']}) in parallel on {cores} threads, "
                      f"extrapolated to B{cfg['batch']}xnH{cfg['heads']}; the reference has no GEMM arithmetic",
            "mask_s": t_mask, "attention_s": t_att, "sample_wall_s": t_att_wall}


def host_cpu_info():
    """lscpu model name + the thread count the CPU arms use (= std::thread::
    hardware_concurrency(), mask.hpp:163)."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:  # noqa: BLE001
        pass
    if model is None:
        try:
            with open("/proc/cpuinfo") as f:
                model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), None)
        except OSError:
            pass
    return {"model": model, "hardware_concurrency": os.cpu_count() or 1}


def cpu_baseline_suite(rounds=10, kind="reference"):
    """BASELINE.md section 4 on this host's cores: the reference's generate_mask
    (mask.hpp:142-179, workers = hardware_concurrency) at the O, L, G and S
    shapes (S: a bounded per-slice sample of B1 nH32 at each SQ, extrapolated
    to 32 slices, as the 2^36-bit guard forces for the larger layouts), and
    attention_forward / _decoupled / _fused (ref_attention.hpp:108-146) at the
    O config both single-threaded (as the reference runs it) and one slice per
    core (base_offset = s*SQ^2/4, bitwise that slice of the full run)."""
    import numpy as np
    oracle = _oracle()
    use_ref = kind == "reference" and oracle.ref_available()
    R = oracle.ref() if use_ref else None
    O = oracle.lib()
    info = host_cpu_info()
    cores = info["hardware_concurrency"]
    out = {"kind": "reference" if use_ref else "port", "host": info, "rounds": rounds}

    def mask_s(B, H, S, workers, base=0):
        n = B * H * S * S
        buf = np.zeros((n + 7) // 8, np.uint8)
        t0 = time.perf_counter()
        if use_ref:
            assert R.ref_generate_mask(B, H, S, 42, base, 0.9, rounds, workers, buf, buf.size) == 0
        else:
            thr, _ = oracle.keep_threshold(0.9)
            O.oracle_generate_mask(n, 42, base, thr, rounds, workers, buf, buf.size)
        return time.perf_counter() - t0, buf

    masks = {}
    for name, (B, H, S) in {"O": (1, 8, 512), "L": (4, 32, 4096), "G": (1, 96, 2048)}.items():
        t, buf = mask_s(B, H, S, cores)
        n = B * H * S * S
        masks[name] = {"layout": f"B{B} nH{H} SQ{S}", "s": round(t, 4), "gbit_s": round(n / t / 1e9, 3),
                       "threads": cores}
        if name == "O":
            t1, _ = mask_s(B, H, S, 1)
            masks["O"]["s_1thread"] = round(t1, 4)
    sweep = []
    for S in (1024, 2048, 4096, 8192, 16384, 32768):
        n_sl = max(1, min(32, (1 << 31) // (S * S)))
        t, _ = mask_s(1, n_sl, S, cores)
        sweep.append({"seq": S, "slices_timed": n_sl, "s_32_slices": round(t * 32 / n_sl, 3),
                      "gbit_s": round(n_sl * S * S / t / 1e9, 3)})
    masks["S_sweep_B1_nH32"] = sweep
    out["masks"] = masks
    # attention at config O (B1 nH8 SQ512 dH64, keep 0.9)
    sl, S, D = 8, 512, 64
    q, k, v = oracle.random_attention_input(sl, S, D, 42 ^ 0xA77E)
    _, bits = mask_s(1, sl, S, cores)

    def attn(mode, s0, s1):
        """mode 0 plain, 1 fused, 2 decoupled over slices [s0, s1)."""
        n = (s1 - s0) * S * D
        qs, ks, vs = (x[s0 * S * D: s1 * S * D].copy() for x in (q, k, v))
        o = np.zeros(n, np.float32)
        base = s0 * S * S // 4
        if use_ref:
            if mode == 2:
                mb = bits[s0 * S * S // 8: s1 * S * S // 8].copy()
                rc = R.ref_attention_decoupled(s1 - s0, S, D, qs, ks, vs, mb, mb.size, 0.9, rounds, o)
            else:
                rc = R.ref_attention(s1 - s0, S, D, qs, ks, vs, mode, 42, base, 0.9, rounds, o)
        else:
            thr, pf = oracle.keep_threshold(0.9)
            mb = bits[s0 * S * S // 8:].copy() if mode == 2 else None
            rc = O.oracle_attention(s1 - s0, S, D, qs, ks, vs, mode, 42, base, thr, pf, rounds,
                                    None if mb is None else mb.ctypes.data, 0, s1 - s0, o)
        assert rc == 0
        return o

    att = {"config": "O: B1 nH8 SQ512 dH64 keep 0.9"}
    for mode, name in ((0, "plain"), (2, "decoupled"), (1, "fused")):
        t0 = time.perf_counter()
        attn(mode, 0, sl)
        att[f"{name}_s_1thread"] = round(time.perf_counter() - t0, 4)
        t0 = time.perf_counter()
        with cf.ThreadPoolExecutor(min(cores, sl)) as ex:
            list(ex.map(lambda s: attn(mode, s, s + 1), range(sl)))
        att[f"{name}_s_slice_per_core"] = round(time.perf_counter() - t0, 4)
    att["threads_slice_per_core"] = min(cores, sl)
    out["attention_O"] = att
    return out


# --------------------------------------------------------------------- GPU side
def time_steps(fn, steps, world, stream):
    import torch
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    barrier(world)
    ev0.record(stream)
    launches = 0
    for _ in range(steps):
        launches += fn()
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    return ev0.elapsed_time(ev1) / steps, launches


def bench_mask_kernel(rgo, cfg, rank, steps, warmup):
    import torch
    B, H, S = cfg["batch"], cfg["heads"], cfg["seq"]
    elems = B * H * S * S
    from paper_2410_07531_b200.sharding import replica_base_offset
    lay = rgo.MaskLayout(B, H, S, 42, replica_base_offset(B, H, S, rank))
    thr = rgo.KeepThreshold(cfg["keep_prob"])
    out = torch.empty(elems // 8, dtype=torch.uint8, device="cuda")
    for _ in range(warmup):
        rgo.generate_mask_device(lay, thr, cfg["rounds"], out=out)
    s = torch.cuda.current_stream()
    ms, _ = time_steps(lambda: (rgo.generate_mask_device(lay, thr, cfg["rounds"], out=out), 1)[1], steps, 1, s)
    return ms, elems


def run_block_modes(rgo, wl, rank, world, args, modes, chunks=1, passes=1):
    """Each mode: W warm-up steps, then exactly K timed steps bracketed by
    barrier + synchronize (CUDA events, max over ranks).  The modes are
    measured 2 x passes times, in alternating orders, and averaged, so the GPU's
    power / clock state (the FP8 GEMMs run at the 1 kW cap) biases none of them."""
    import torch
    from paper_2410_07531_b200.sharding import replica_base_offset
    base = replica_base_offset(wl.batch, wl.heads, wl.seq, rank)  # disjoint Philox counters per rank
    weights = rgo.block.make_weights(wl, 42, torch.device("cuda"))
    launch = {"streams": tuple(args.rng_launch), "in_gemm": (0, args.rng_warps, 0)}
    blocks = {m: rgo.Block(wl, m, seed=42, base_offset=base, weights=weights, rng_launch=launch.get(m, (0, 0, 0)),
                           chunks=chunks) for m in modes}
    stream = torch.cuda.current_stream()
    samples = {m: [] for m in modes}
    phases, launches = {}, {}
    for order in [modes, modes[::-1]] * passes:
        for m in order:
            b = blocks[m]
            for _ in range(args.warmup):
                b.step()
            ms, n = time_steps(b.step, args.steps, world, stream)
            samples[m].append(max_over_ranks(ms, world))
            phases[m] = b.last_timings()
            launches[m] = n
    res = {m: sum(v) / len(v) for m, v in samples.items()}
    return blocks, res, samples, phases, launches


class Energy:
    """NVML total-energy counter (mJ) of the device this rank runs on."""

    def __init__(self):
        import torch
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            idx = torch.cuda.current_device()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                idx = int(vis.split(",")[idx])
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(idx)
            self.limit_w = pynvml.nvmlDeviceGetEnforcedPowerLimit(self.h) / 1e3
            self.read()
        except Exception:  # noqa: BLE001
            self.h = None

    def read(self):
        return self.nv.nvmlDeviceGetTotalEnergyConsumption(self.h) / 1e3  # J

    def sm_mhz(self):
        return self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)


def bench_energy(blocks, modes, mask_fn, seconds=1.5):
    """Energy per step of each mode (and of the stand-alone mask kernel), from
    the NVML energy counter around ~`seconds` of back-to-back steps, with the
    device time of the same run.  On a power-capped part time = energy / P, so
    the RNG's exposed time should equal its extra energy over the cap:
    (t_mode - t_no_rng) ~ (E_mode - E_no_rng) / P_cap."""
    import torch
    en = Energy()
    if en.h is None:
        return {"unavailable": "NVML energy counter not readable"}
    out = {"power_limit_w": round(en.limit_w, 1)}
    stream = torch.cuda.current_stream()

    def run(fn, name):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        n = max(20, int(seconds * 1e3 / e0.elapsed_time(e1)))
        clocks = []
        j0 = en.read()
        e0.record(stream)
        for i in range(n):
            fn()
            if i % max(1, n // 8) == 0:
                clocks.append(en.sm_mhz())
        e1.record(stream)
        torch.cuda.synchronize()
        j1 = en.read()
        ms = e0.elapsed_time(e1) / n
        joules = (j1 - j0) / n
        out[name] = {"ms": round(ms, 4), "j_per_step": round(joules, 4), "avg_w": round(joules / ms * 1e3, 1),
                     "sm_mhz_median": sorted(clocks)[len(clocks) // 2], "steps": n}

    for m in modes:
        run(blocks[m].step, m)
    run(mask_fn, "mask_kernel")
    if "no_rng" in out:
        for m in modes:
            if m == "no_rng":
                continue
            dt = out[m]["ms"] - out["no_rng"]["ms"]
            de = out[m]["j_per_step"] - out["no_rng"]["j_per_step"]
            out[m]["extra_ms_vs_no_rng"] = round(dt, 4)
            out[m]["extra_j_vs_no_rng"] = round(de, 4)
            out[m]["extra_j_over_cap_ms"] = round(de / en.limit_w * 1e3, 4)
    return out


def golden_mask_fnv(name, rounds):
    """The reference's FNV-1a-64 of the full mask (tests/golden/golden.json, recorded
    from the reference compiled in place, oracle/make_golden.py), or None."""
    try:
        with open(os.path.join(ROOT, "tests", "golden", "golden.json")) as f:
            big = json.load(f)["big_masks"]
    except (OSError, ValueError, KeyError):
        return None
    for m in big:
        if m["name"] == name and m["rounds"] == rounds and m["base_offset"] == 0 and m["seed"] == 42:
            return m["fnv"]
    return None


def block_parity(rgo, blocks, golden_name, rounds, rank):
    """Self-check of the timed run, after the timed region: the in-GEMM (and
    streams) mask left by the last timed step is copied back and hashed
    (FNV-1a-64 through the C ABI) against the reference's hash of the same
    layout; every mode's attention output must equal the serial-fused
    (Philox-inline) baseline's bitwise.  Rank r > 0 checks its own replica's
    disjoint counter range against rank 0's hash only when r == 0."""
    import torch
    torch.cuda.synchronize()
    out = {"golden": golden_name, "rounds": rounds}
    ok = True
    want = golden_mask_fnv(golden_name, rounds) if rank == 0 else None
    for m in ("in_gemm", "streams"):
        if m not in blocks:
            continue
        h = f"{rgo.mask.fnv1a64(blocks[m].mask.cpu()):016x}"
        out[f"mask_fnv_{m}"] = h
        if want is not None:
            ok &= h == want
    out["golden_fnv"] = want
    base = blocks["serial_fused"].attn_o.view(torch.uint8)
    eq = {m: bool(torch.equal(b.attn_o.view(torch.uint8), base)) for m, b in blocks.items() if m != "serial_fused"}
    out["attn_o_bitwise_equal_to_fused"] = eq
    ok &= all(eq.values())
    out["ok"] = bool(ok)
    return out


def measure_fp8_peak(seconds=4.0):
    """Dense FP8 (e4m3 x e4m3 -> bf16) tensor peak of THIS GPU, measured like
    MEASURED_PEAKS.json's bf16 figure: cuBLASLt through torch._scaled_mm at
    8192^3 (2*N^3 flop), best of 10 (burst) and back to back for `seconds`
    (sustained, i.e. at the power-capped clock a long step runs at)."""
    import torch
    N = 8192
    a = torch.randn(N, N, device="cuda").to(torch.float8_e4m3fn)
    b = torch.randn(N, N, device="cuda").to(torch.float8_e4m3fn).t()  # column-major operand
    one = torch.ones((), device="cuda")

    def mm():
        return torch._scaled_mm(a, b, scale_a=one, scale_b=one, out_dtype=torch.bfloat16)
    for _ in range(3):
        mm()
    best = float("inf")
    for _ in range(10):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        mm()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = max(10, int(seconds * 1e3 / best))
    e0.record()
    for _ in range(iters):
        mm()
    e1.record()
    torch.cuda.synchronize()
    flop = 2.0 * N ** 3
    del a, b
    return {"fp8_tflops": round(flop / best / 1e9, 1),
            "fp8_tflops_sustained": round(flop / (e0.elapsed_time(e1) / iters) / 1e9, 1),
            "how": f"torch._scaled_mm e4m3 {N}^3 -> bf16: best of 10 (burst), {iters} back to back (sustained)"}


def block_summary(rgo, wl, res, phases, mask_ms, peaks):
    gemm_flops = sum(g.flops() for g in rgo.gemm_shapes(wl))
    attn_flops = rgo.attention_work(wl)[0]
    fp8_peak = peaks["fp8_tflops"]
    roof_ms = gemm_flops / fp8_peak / 1e9 + attn_flops / peaks["bf16_tflops"] / 1e9
    # the step is a long run at the power-capped clock: its roofline at the sustained peaks too
    roof_sus_ms = None
    if peaks.get("fp8_tflops_sustained") and peaks.get("bf16_tflops_sustained"):
        roof_sus_ms = (gemm_flops / peaks["fp8_tflops_sustained"] / 1e9
                       + attn_flops / peaks["bf16_tflops_sustained"] / 1e9)
    best = min((m for m in ("streams", "in_gemm") if m in res), key=lambda m: res[m])
    value = res[best]
    hidden = 1.0 - (value - res["no_rng"]) / mask_ms if res.get("no_rng") else None
    return best, value, {
        "speedup_vs_fused": round(res["serial_fused"] / value, 4),
        "modes_ms": {m: round(v, 4) for m, v in res.items()},
        "phases_ms": {m: {"gemm_window": round(p[0], 4), "attention": round(p[1], 4)} for m, p in phases.items()},
        "rng_hidden_fraction": None if hidden is None else round(hidden, 4),
        "mask_ms": round(mask_ms, 4),
        "block_roofline": {"ms": round(roof_ms, 4), "frac": round(roof_ms / value, 4),
                           "ms_sustained": None if roof_sus_ms is None else round(roof_sus_ms, 4),
                           "frac_sustained": None if roof_sus_ms is None else round(roof_sus_ms / value, 4)},
    }


def bench_e2e(rgo, wl, b, mode, args, world):
    import torch
    stream = torch.cuda.current_stream()
    b2 = rgo.Block(wl, mode, seed=42, base_offset=b.desc.base_offset, weights=b.weights,
                   rng_launch=(tuple(args.rng_launch) if mode == "streams" else (0, args.rng_warps, 0)))
    pair = (b, b2)
    host_in = [t.cpu().pin_memory() for t in (b.attn_in, (b.attn_in.float() * -1.0).bfloat16())]
    host_out = [torch.empty_like(b.attn_o, device="cpu").pin_memory() for _ in range(2)]
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_step = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]   # replica's previous result is in host memory
    # (ev_step: the replica's last step -- and with it the read of its attn_in -- is done)
    state = {"k": 0}

    def stage_input(slot, k):
        # the replica's previous step must have read its input; its previous result's D2H
        # only has to finish before the replica's next step (which overwrites attn_o), so
        # the H2D of step k+1 overlaps both step k and the D2H of step k-1
        with torch.cuda.stream(h2d):
            h2d.wait_event(ev_step[slot])
            pair[slot].attn_in.copy_(host_in[k % 2], non_blocking=True)
            ev_in[slot].record(h2d)

    for slot in range(2):
        ev_done[slot].record(stream)
        ev_step[slot].record(stream)
    stage_input(0, 0)

    def e2e_step():
        k = state["k"]
        cur, nxt = k % 2, (k + 1) % 2
        stage_input(nxt, k + 1)                 # H2D of step k+1's input, overlapped
        stream.wait_event(ev_in[cur])
        stream.wait_event(ev_done[cur])         # this replica's previous result is in host memory
        n = pair[cur].step()
        ev_step[cur].record(stream)
        with torch.cuda.stream(d2h):            # D2H of the whole result, overlapped
            d2h.wait_event(ev_step[cur])
            host_out[cur].copy_(pair[cur].attn_o, non_blocking=True)
            ev_done[cur].record(d2h)
        state["k"] = k + 1
        return n

    for _ in range(max(10, args.warmup)):  # back to the steady power state the modes ran in
        e2e_step()
    torch.cuda.synchronize()
    barrier(world)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    for slot in range(2):                   # the timed region ends with the last D2H
        stream.wait_event(ev_done[slot])
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps, world)
    # the last result really is the step's output
    last = (state["k"] - 1) % 2
    assert torch.equal(host_out[last].view(torch.uint8), pair[last].attn_o.cpu().view(torch.uint8))
    b2.close()
    h2d_bytes = int(host_in[0].numel() * host_in[0].element_size())
    d2h_bytes = int(host_out[0].numel() * host_out[0].element_size())
    return ms, h2d_bytes, d2h_bytes


def bench_dropin_O(rgo, reps=20):
    """The drop-in surface end to end at config O (B1 nH8 SQ512 dH64, keep 0.9,
    Philox-10): generate_mask (mask.hpp:142-179) then attention_dropout_decoupled
    (ref_attention.hpp:129-146) on HOST float arrays through the C ABI the
    include/rgo/*.hpp drop-in calls (rgo_generate_mask_host + rgo_attention_host:
    H2D, K1 / K5, D2H inside each call).  Wall clock per pair of calls, median."""
    import ctypes as C
    import numpy as np
    L_ = rgo._lib
    lib = L_.lib()
    sl, S, D = 8, 512, 64
    n = sl * S * D
    q, k, v = (np.empty(n, np.float32) for _ in range(3))
    L_.check(lib.rgo_random_attention_input_host(sl, S, D, 42 ^ 0xA77E, q.ctypes.data, k.ctypes.data, v.ctypes.data))
    thr = C.c_uint64()
    L_.check(lib.rgo_keep_threshold(0.9, C.byref(thr), None))
    md = L_.mask_desc(1, sl, S, 10, 42, 0, thr.value)
    bits = np.empty(sl * S * S // 8, np.uint8)
    o = np.empty(n, np.float32)
    ad = L_.attn_host_desc(sl, S, D, 1, 0.9, 0, 0, 10, 0)  # RGO_MASK_BITS

    def once():
        L_.check(lib.rgo_generate_mask_host(md, bits.ctypes.data, bits.size, 1))
        L_.check(lib.rgo_attention_host(C.byref(ad), q.ctypes.data, k.ctypes.data, v.ctypes.data, bits.ctypes.data,
                                        bits.size, o.ctypes.data))
    for _ in range(3):
        once()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        once()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return {"value_ms": round(ts[len(ts) // 2] * 1e3, 3), "unit": "ms per generate_mask + attention_dropout_decoupled",
            "h2d_bytes": int(3 * n * 4 + bits.size), "d2h_bytes": int(bits.size + n * 4),
            "config": "O: B1 nH8 SQ512 dH64 keep 0.9 Philox-10, host float arrays through the C ABI "
                      "(rgo_generate_mask_host + rgo_attention_host), median of %d" % reps,
            "mask_fnv": f"{rgo.mask.fnv1a64(bits):016x}"}


def bench_chunked(rgo, wl, rank, world, args, peaks, mask_ms_l):
    import torch
    out = {}
    cmodes = ["serial_fused", "streams", "in_gemm", "no_rng"]
    s32 = rgo.WorkloadConfig(batch=1, seq=32768, heads=32, head_dim=128, ffn_dim=11008, gated=True,
                             keep_prob=0.9, philox_rounds=args.rounds)
    for name, cfg, C in (("llama2_7b_C4", wl, 4), ("seq32k_C8", s32, 8)):
        elems = cfg.batch * cfg.heads * cfg.seq ** 2
        row = {"chunks": C, "full_mask_mib": elems // 8 // 2 ** 20, "live_mask_mib": 2 * elems // 8 // C // 2 ** 20,
               "config": f"B{cfg.batch} nH{cfg.heads} SQ{cfg.seq} dH128 d4096 FFN11008 SwiGLU, keep 0.9, "
                         f"Philox-{args.rounds}, {C} query-row windows"}
        for label, chunks in (("chunked", C), ("unchunked", 1)):
            blocks, res, _, ph, _ = run_block_modes(rgo, cfg, rank, world, args, cmodes, chunks=chunks)
            for blk in blocks.values():
                blk.close()
            del blocks
            torch.cuda.empty_cache()
            row[f"{label}_modes_ms"] = {m: round(v, 4) for m, v in res.items()}
            best = min(("streams", "in_gemm"), key=lambda m: res[m])
            row[f"{label}_best"] = best
            row[f"{label}_speedup_vs_fused"] = round(res["serial_fused"] / res[best], 4)
        out[name] = row
    return out


def bench_tp_emulated(rgo, wl, world, steps=10):
    """One rank's share of a tensor-parallel (tp = 2) Llama2-7B step (rgo_block_create_tp) on this
    GPU: half the heads (and their compact mask), half the FFN, the two two-shot all-reduce
    kernels at full size and the four host barriers of a step -- with the peer's buffers emulated
    by local scratch (the all-reduce reads HBM instead of NVLink; no second GPU here)."""
    import torch
    out = {"config": "Llama2-7B block, tp=2, rank 0 of an emulated pair (peer buffers local, barriers no-op): "
                     "heads 16, FFN 5504, mask 128 MiB per rank",
           "modes_ms": {}}
    for mode in ("serial_fused", "in_gemm", "no_rng"):
        blk = rgo.TPBlock(wl, mode, seed=42, emulate=(2, 0))
        out["modes_ms"][mode] = round(event_ms(blk.step, steps, world, warm=3), 4)
        blk.close()
        del blk
        torch.cuda.empty_cache()
    m = out["modes_ms"]
    out["speedup_vs_fused"] = round(m["serial_fused"] / m["in_gemm"], 4)
    return out


def bench_gemms(rgo, wl, world, peaks):
    import torch
    f8 = torch.float8_e4m3fn
    out, tot_flop, tot_ms = {}, 0.0, 0.0
    for sh in rgo.gemm_shapes(wl):
        g = torch.Generator(device="cuda").manual_seed(sh.m + sh.n + sh.k)
        a = ((torch.rand(sh.m, sh.k, device="cuda", generator=g) * 2 - 1) * 1.7).to(f8)
        b = ((torch.rand(sh.n, sh.k, device="cuda", generator=g) * 2 - 1) * 1.7).to(f8)
        epi = "swiglu" if sh.name.startswith("FFN1") and wl.gated else ("gelu" if sh.name.startswith("FFN1") else "none")
        out_dt = torch.bfloat16 if sh.name == "QKV" else f8
        c = torch.empty(sh.m, sh.n // 2 if epi == "swiglu" else sh.n, dtype=out_dt, device="cuda")
        ms = event_ms(lambda: rgo.gemm(a, b, c, epilogue=epi, alpha=1.0 / sh.k), 10, world, warm=3)
        out[sh.name] = {"ms": round(ms, 4), "tflops": round(sh.flops() / ms / 1e9, 1)}
        tot_flop += sh.flops()
        tot_ms += ms
        del a, b, c
    peak = peaks["fp8_tflops"]
    ach = tot_flop / tot_ms / 1e9
    return {"bound": "tensor", "achieved": round(ach, 1), "peak": round(peak, 1), "unit": "TFLOP/s",
            "frac": round(ach / peak, 4), "per_gemm": out,
            "note": "FP8 peak measured in this run (cuBLASLt e4m3 8192^3 burst, fp8_peak); stand-alone GEMMs"}


def event_ms(fn, reps, world, warm=1):
    import torch
    for _ in range(warm):
        fn()
    ms, _ = time_steps(lambda: (fn(), 1)[1], reps, world, torch.cuda.current_stream())
    return max_over_ranks(ms, world)


def bench_attention_bwd(rgo, rank, world, peaks):
    """North star (4): attention forward + backward reading the precomputed
    bitmask vs the same kernels with Philox-10 fused in, at the Llama2-7B
    attention shape (B4 nH32 SQ4096 dH128, token-major QKV), per rank."""
    import torch
    from paper_2410_07531_b200.sharding import replica_base_offset
    B, H, S, D = L["batch"], L["heads"], L["seq"], L["head_dim"]
    base = replica_base_offset(B, H, S, rank)
    qkv = (torch.rand(B * S, 3 * H * D, device="cuda") * 2 - 1).bfloat16()
    v4 = qkv.view(B, S, 3, H, D)
    q, k, v = (v4[:, :, i].permute(0, 2, 1, 3) for i in range(3))
    o = torch.empty(B, S, H, D, dtype=torch.bfloat16, device="cuda").permute(0, 2, 1, 3)
    do = (torch.rand(B, S, H, D, device="cuda") * 2 - 1).bfloat16().permute(0, 2, 1, 3)
    g = [torch.empty(B, S, H, D, dtype=torch.bfloat16, device="cuda").permute(0, 2, 1, 3) for _ in range(3)]
    lse = torch.empty(B * H * S, dtype=torch.float32, device="cuda")
    bits = rgo.generate_mask_device(rgo.MaskLayout(B, H, S, 42, base), rgo.KeepThreshold(L["keep_prob"]), 10)
    a = rgo._lib.attn_desc(B, H, S, D, 0.0, 0, 1.0, 0, 0, 10, 0)
    need = rgo._lib.C.c_uint64()
    rgo._lib.check(rgo._lib.lib().rgo_attn_bwd_workspace(a, rgo._lib.C.byref(need)))
    work = torch.empty(need.value, dtype=torch.uint8, device="cuda")
    flops_f = 4 * B * H * S * S * D
    out = {}
    for name, kw in (("bits", dict(mask_source=1, keep_prob=L["keep_prob"], bits=bits)),
                     ("philox_fused", dict(mask_source=2, keep_prob=L["keep_prob"], seed=42, base_offset=base,
                                           rounds=10)),
                     ("no_dropout", dict(mask_source=0))):
        fwd = event_ms(lambda: rgo.attn_fwd(q, k, v, o, lse=lse, **kw), 5, world)
        bwd = event_ms(lambda: rgo.attn_bwd(q, k, v, o, do, lse, dq=g[0], dk=g[1], dv=g[2], work=work, **kw),
                       5, world)
        out[name] = {"fwd_ms": round(fwd, 4), "bwd_ms": round(bwd, 4),
                     "fwd_tflops": round(flops_f / fwd / 1e9, 1), "bwd_tflops": round(2.5 * flops_f / bwd / 1e9, 1)}
    mask_ms = event_ms(lambda: rgo.generate_mask_device(rgo.MaskLayout(B, H, S, 42, base),
                                                        rgo.KeepThreshold(L["keep_prob"]), 10, out=bits), 5, world)
    det = event_ms(lambda: rgo.attn_bwd(q, k, v, o, do, lse, dq=g[0], dk=g[1], dv=g[2], work=work, mask_source=1,
                                        keep_prob=L["keep_prob"], bits=bits, deterministic=True), 5, world)
    out["bits_deterministic_bwd"] = {
        "bwd_ms": round(det, 4), "bwd_tflops": round(2.5 * flops_f / det / 1e9, 1),
        "what": "RGO_ATTN_BWD_DETERMINISTIC: split dK/dV + dQ kernels, dQ accumulated in TMEM (no cross-CTA "
                "reductions, 7 instead of 5 MMAs per 128x128 block)"}
    out["mask_ms"] = round(mask_ms, 4)
    out["bwd_speedup_bits_vs_fused"] = round(out["philox_fused"]["bwd_ms"] / out["bits"]["bwd_ms"], 4)
    out["fwd_bwd_speedup_bits_vs_fused"] = round(
        (out["philox_fused"]["fwd_ms"] + out["philox_fused"]["bwd_ms"]) / (out["bits"]["fwd_ms"] + out["bits"]["bwd_ms"]),
        4)
    out["bwd_roofline"] = {"bound": "tensor", "achieved": out["bits"]["bwd_tflops"], "peak": peaks["bf16_tflops"],
                           "unit": "TFLOP/s", "frac": round(out["bits"]["bwd_tflops"] / peaks["bf16_tflops"], 4),
                           "algorithmic": "2.5 x 4*B*nH*SQ^2*dH (5 GEMMs of the backward)"}
    out["config"] = "B4 nH32 SQ4096 dH128 keep 0.9, Philox-10; the same mask serves forward and backward"
    del qkv, o, do, g, work, bits
    return out


def bench_flash_attn(world):
    """The installed flash-attn (FA2, Philox fused in the kernel) with dropout 0.1
    at the Llama2-7B attention shape: the library form of the conventional
    fused-dropout baseline (PAPER's comparison), timed beside ours."""
    import torch
    try:
        import flash_attn
        from flash_attn import flash_attn_func
    except Exception as e:  # noqa: BLE001
        return {"unavailable": str(e)[:120]}
    B, H, S, D = L["batch"], L["heads"], L["seq"], L["head_dim"]
    q, k, v = ((torch.rand(B, S, H, D, device="cuda") * 2 - 1).bfloat16().requires_grad_(True) for _ in range(3))
    do = (torch.rand(B, S, H, D, device="cuda") * 2 - 1).bfloat16()
    fwd = event_ms(lambda: flash_attn_func(q, k, v, dropout_p=1.0 - L["keep_prob"]), 5, world, warm=2)
    o = flash_attn_func(q, k, v, dropout_p=1.0 - L["keep_prob"])
    bwd = event_ms(lambda: torch.autograd.grad(o, (q, k, v), do, retain_graph=True), 5, world, warm=2)
    return {"version": flash_attn.__version__, "fwd_ms": round(fwd, 4), "bwd_ms": round(bwd, 4),
            "config": "flash_attn_func(dropout_p=0.1), B4 S4096 H32 D128 bf16 (sm_100 runs its sm80 kernels)"}


def graph_ms(fn, reps, world, replays=3):
    """Device ms per call of `fn` with `reps` calls captured in one CUDA graph and replayed
    (short kernels: the per-call host work -- ctypes, tensor-map encoding -- would otherwise
    leave the GPU idle between launches and be timed as kernel time)."""
    import torch
    fn()
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    torch.cuda.synchronize()
    ms, _ = time_steps(lambda: (g.replay(), 1)[1], replays, world, torch.cuda.current_stream())
    return max_over_ranks(ms, world) / reps


def bench_seq_sweep(rgo, rank, world, lens):
    """BASELINE configs[4]: SQ sweep at the Llama2 head config (B1 nH32 dH128),
    batch x head sharded over the ranks (rank r owns heads [r*32/n, (r+1)*32/n)
    and that shard's Philox counter range; no collective).  Per SQ: mask
    kernel, attention forward reading it, and the fused-Philox forward."""
    import torch
    from paper_2410_07531_b200.sharding import shard_slices
    H_all, D = 32, 128
    rows = []
    for S in lens:
        s0, s1, base = shard_slices(1, H_all, S, world, rank)
        H = s1 - s0
        q, k, v = ((torch.rand(1, H, S, D, device="cuda") * 2 - 1).bfloat16() for _ in range(3))
        o = torch.empty_like(q)
        lay = rgo.MaskLayout(1, H, S, 42, base)
        bits = torch.empty(H * S * S // 8, dtype=torch.uint8, device="cuda")
        thr = rgo.KeepThreshold(L["keep_prob"])
        reps = 3 if S >= 16384 else 10
        # short sequences: replayed CUDA graphs, so host launch work is not timed as kernel time
        timer = graph_ms if S <= 4096 else event_ms
        m_ms = timer(lambda: rgo.generate_mask_device(lay, thr, 10, out=bits), reps, world)
        a_ms = timer(lambda: rgo.attn_fwd(q, k, v, o, mask_source=1, keep_prob=L["keep_prob"], bits=bits),
                     reps, world)
        f_ms = timer(lambda: rgo.attn_fwd(q, k, v, o, mask_source=2, keep_prob=L["keep_prob"], seed=42,
                                          base_offset=base, rounds=10), reps, world)
        rows.append({"seq": S, "mask_ms": round(m_ms, 4), "attn_bits_ms": round(a_ms, 4),
                     "attn_fused_ms": round(f_ms, 4),
                     "mask_gbit_s": round(H_all * S * S / (m_ms * 1e-3) / 1e9, 1),
                     "attn_bits_tflops": round(4 * H_all * S * S * D / (a_ms * 1e-3) / 1e12, 1)})
        del q, k, v, o, bits
        torch.cuda.empty_cache()
    return {"config": f"B1 nH32 dH128 keep 0.9 Philox-10, heads sharded over {world} rank(s)", "rows": rows}


def bench_block(args, rank, world):
    import torch
    import paper_2410_07531_b200 as rgo
    cfg = dict(L, rounds=args.rounds)
    wl = rgo.WorkloadConfig(batch=cfg["batch"], seq=cfg["seq"], heads=cfg["heads"], head_dim=cfg["head_dim"],
                            ffn_dim=cfg["ffn"], gated=True, keep_prob=cfg["keep_prob"], philox_rounds=cfg["rounds"])
    elems = cfg["batch"] * cfg["heads"] * cfg["seq"] ** 2
    modes = ["serial_fused", "streams", "in_gemm", "no_rng"]
    peaks, src = load_peaks()
    log("FP8 peak (cuBLASLt e4m3 8192^3)")
    fp8 = measure_fp8_peak()
    peaks.update(fp8_tflops=fp8["fp8_tflops"], fp8_tflops_sustained=fp8["fp8_tflops_sustained"])
    log("Llama2-7B block modes")
    with ClockSampler(torch.cuda.current_device()) as clk:
        blocks, res, samples, phases, launches = run_block_modes(rgo, wl, rank, world, args, modes, passes=3)
    log("mask kernel")
    att_ms = phases["no_rng"][1]  # the mask-reading attention kernel alone, in situ
    clocks = clk.summary()
    mask_ms, _ = bench_mask_kernel(rgo, cfg, rank, max(5, args.steps // 2), 3)
    mask_ms = max_over_ranks(mask_ms, world)
    best, value, summ = block_summary(rgo, wl, res, phases, mask_ms, peaks)
    parity = block_parity(rgo, blocks, "L", cfg["rounds"], rank)
    log("energy per mode (NVML)")
    lay_l = rgo.MaskLayout(cfg["batch"], cfg["heads"], cfg["seq"], 42, blocks["in_gemm"].desc.base_offset)
    mask_buf = torch.empty(elems // 8, dtype=torch.uint8, device="cuda")
    energy = bench_energy(blocks, modes, lambda: rgo.generate_mask_device(lay_l, rgo.KeepThreshold(cfg["keep_prob"]),
                                                                          cfg["rounds"], out=mask_buf))
    del mask_buf
    # ----- e2e through the public API with host buffers.  A step's input is the
    # previous block's attention output (`attn_in`, bf16 [M, d], 128 MiB, read by the
    # step's first kernel) and its result is this block's attention output (`attn_o`,
    # bf16 [M, d], 128 MiB).  Every timed step copies a fresh input from pinned host
    # memory (H2D copy stream) and copies its WHOLE result back into pinned host memory
    # (D2H copy stream).  Two block replicas alternate so step k+1's H2D and step k's
    # D2H overlap the compute of the neighbouring steps, as a serving loop would; the
    # timed region ends when the last step's result has landed in host memory.
    log("e2e")
    e2e_ms, h2d_bytes, d2h_bytes = bench_e2e(rgo, wl, blocks[best], best, args, world)
    for blk in blocks.values():
        blk.close()
    del blocks
    torch.cuda.empty_cache()

    attn_flops = rgo.attention_work(wl)[0]
    bf16_peak = peaks["bf16_tflops"]
    bf16_sus = peaks.get("bf16_tflops_sustained") or bf16_peak
    line = {
        "metric": "llama2_block_ms", "value": round(value, 4), "unit": "ms", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(value, 4), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "e4m3 GEMMs + bf16 attention (fp32 accumulate)",
        "data": "synthetic (Philox-uniform activations, random-init e4m3 weights)",
        "config": {"workload": "Llama2-7B transformer block FP8: batch 4, seq 4096, 32 heads x 128, d_model 4096, "
                               "FFN 11008 SwiGLU, attn dropout 0.1 (keep 0.9), Philox-10; step = Proj+FFN1+FFN2 "
                               "of block L-1 + QKV and attention of block L",
                   "global_batch": cfg["batch"] * world, "seq_len": cfg["seq"], "parallelism": f"replicas x{world}",
                   "overlap_mechanism": best,
                   "l2": "no flush: every step streams > 1 GB (mask 256 MiB, QKV 384 MiB) through a 126 MB L2"},
        "speedup_vs_fused": summ["speedup_vs_fused"],
        # the paper's block speedups (GH100, FP8); ours are measured on B200
        "paper_speedup_gh100": {"llama2": 1.14, "moe": 1.13, "gpt3": 1.06, "source": "PAPER.md:57,197"},
        "modes_ms": summ["modes_ms"],
        "modes_ms_samples": {m: [round(x, 4) for x in v] for m, v in samples.items()},
        "phases_ms": summ["phases_ms"],
        "rng_hidden_fraction": summ["rng_hidden_fraction"],
        "mask_gbit_s": round(elems * world / (mask_ms * 1e-3) / 1e9, 2),
        "mask_ms": round(mask_ms, 4),
        # K1's limiter is the fma-heavy pipe: (2R-1)/4 IMAD.WIDE.U32 per element (round 1's
        # multiply of the shared high counter word is hoisted), ~32 per clock per SM
        # (scripts/diag/mulwide.cu); the 1-bit output is ~0.2 TB/s of HBM.
        "rng_roofline": {"bound": "fma-heavy pipe (IMAD.WIDE.U32)",
                         "achieved": round(elems * (2 * cfg["rounds"] - 1) / 4 / (mask_ms * 1e-3) / 1e12, 3),
                         "peak": round(32 * 148 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12, 3),
                         "unit": "T IMAD.WIDE/s",
                         "frac": round(elems * (2 * cfg["rounds"] - 1) / 4 / (mask_ms * 1e-3)
                                       / (32 * 148 * peaks.get("sm_max_mhz", 1965.0) * 1e6), 4),
                         "hbm_write_gbs": round(elems / 8 / (mask_ms * 1e-3) / 1e9, 1)},
        "blocks_per_s": round(world * 1e3 / value, 3),
        "block_roofline": dict(summ["block_roofline"],
                               **{"def": f"sum(GEMM flop)/FP8 peak + attention flop/BF16 peak; FP8 peak "
                                         f"{peaks['fp8_tflops']} TF/s measured in this run (fp8_peak), bf16 "
                                         f"{bf16_peak} TF/s ({src})"}),
        "fp8_peak": fp8,
        # timed inside the step (a long run at the power-capped clock): against the SUSTAINED
        # bf16 peak, as the measurement contract asks; the burst fraction alongside
        "roofline": {"bound": "tensor", "kernel": "attention fwd (mask bits), in situ (no-RNG step phase)",
                     "achieved": round(attn_flops / (att_ms * 1e-3) / 1e12, 2), "peak": bf16_sus,
                     "peak_kind": "sustained bf16 (MEASURED_PEAKS.json bf16_tflops_sustained)",
                     "unit": "TFLOP/s", "frac": round(attn_flops / (att_ms * 1e-3) / 1e12 / bf16_sus, 4),
                     "frac_vs_burst": round(attn_flops / (att_ms * 1e-3) / 1e12 / bf16_peak, 4),
                     "traffic": profiled_traffic("attn_fwd_bits"),
                     "algorithmic": f"4*B*nH*SQ^2*dH = {attn_flops:.4e} flop per launch (workload.hpp:59-64)"},
        "e2e": {"value": round(e2e_ms, 4), "unit": "ms", "h2d_bytes_per_step": h2d_bytes,
                "d2h_bytes_per_step": d2h_bytes,
                "how": "public API (Block.step), step input (previous attention output, bf16 [M, d]) copied "
                       "from pinned host memory every step on an H2D stream, the step's whole result "
                       "(attention output, bf16 [M, d]) copied back to pinned host memory every step on a "
                       "D2H stream; two replicas alternate so copies overlap neighbouring steps (the H2D of "
                       "step k+1 waits only for step k-1 to have read its replica's input, the replica's next "
                       "step for its previous D2H); the timed region ends when the last result is in host "
                       "memory. With the copies fully overlapped e2e is within the power-state noise of "
                       "`value` (which is the mean of six samples interleaved with the other modes)"},
        "parity": parity,
        "energy": energy,
        "clocks": clocks, "gpu_launches": launches[best],
    }
    _PARTIAL["line"] = line
    if not args.no_extras:
        # K2 stand-alone: the block's four FP8 GEMMs (their epilogues as in the block),
        # each timed alone on unit-variance e4m3 data, against the FP8 peak
        log("GEMMs stand-alone")
        line["gemm_roofline"] = bench_gemms(rgo, wl, world, peaks)
        # BASELINE configs[2]: GPT-3 175B block (B1 SQ2048 nH96 d12288, GELU FFN 49152)
        log("GPT-3 block")
        g = rgo.workload_preset("gpt3")
        g.philox_rounds = args.rounds
        gblocks, gres, _, gph, _ = run_block_modes(rgo, g, rank, world, args, modes, passes=2)
        gparity = block_parity(rgo, gblocks, "G", args.rounds, rank)
        for blk in gblocks.values():
            blk.close()
        del gblocks
        torch.cuda.empty_cache()
        gm = dict(L, batch=1, heads=96, seq=2048, rounds=args.rounds)
        gmask, _ = bench_mask_kernel(rgo, gm, rank, 10, 3)
        _, gval, gsum = block_summary(rgo, g, gres, gph, max_over_ranks(gmask, world), peaks)
        line["gpt3_block"] = dict({"value_ms": round(gval, 4),
                                   "config": "GPT-3 175B block FP8: B1 SQ2048 nH96 dH128 d12288, GELU FFN 49152, "
                                             "keep 0.9, Philox-10", "parity": gparity}, **gsum)
        line["parity"]["ok"] = bool(line["parity"]["ok"] and gparity["ok"])
        # BASELINE configs[3]: MoE block (Mixtral-8x7B-like): 8 experts top-2 SwiGLU FFN 14336
        log("MoE block")
        mo = rgo.workload_preset("moe")
        mo.philox_rounds = args.rounds
        mblocks, mres, _, mph, _ = run_block_modes(rgo, mo, rank, world, args, modes, passes=2)
        for blk in mblocks.values():
            blk.close()
        del mblocks
        torch.cuda.empty_cache()
        _, mval, msum = block_summary(rgo, mo, mres, mph, mask_ms, peaks)
        line["moe_block"] = dict({"value_ms": round(mval, 4),
                                  "config": "MoE block FP8: B4 SQ4096 nH32 dH128 d4096, 8 experts top-2 SwiGLU FFN "
                                            "14336 (balanced synthetic routing: 4096 tokens per expert), keep 0.9, "
                                            "Philox-10; RNG hidden under 2 + 16 expert GEMMs"}, **msum)
        # batch-chunk pipelining of RNG -> GEMMs -> attention (schedule.hpp:206-239):
        # 4 chunks of one batch item each, live mask = 2 x 64 MiB instead of 256 MiB
        # SQ-chunk pipelining (pipeline_schedule, schedule.hpp:205-239): query-row
        # windows, stage c = attention(c) -> GEMMs of window c with window c+1's RNG hidden under
        # them; live mask = 2 windows.  Llama2-7B (C = 4) and the long-context config S
        # (B1 nH32 SQ32K, C = 8: 1 GiB live instead of 4 GiB), against the unchunked step.
        log("SQ-chunk pipeline")
        line["chunked_pipeline"] = bench_chunked(rgo, wl, rank, world, args, peaks, mask_ms)
        if world == 1 and wl.ffn() % 256 == 0:
            log("tensor-parallel rank (emulated pair)")
            try:
                line["tp2_rank_emulated"] = bench_tp_emulated(rgo, wl, world)
            except Exception as e:  # an extra: never lose the main line over it
                line["tp2_rank_emulated"] = {"error": str(e)[:200]}
        log("attention fwd+bwd")
        line["attention_fwd_bwd"] = bench_attention_bwd(rgo, rank, world, peaks)
        log("flash-attn library baseline")
        line["flash_attn_dropout_baseline"] = bench_flash_attn(world)
        fa = line["flash_attn_dropout_baseline"]
        if "fwd_ms" in fa:
            # the block step with the library's fused-dropout attention in place of
            # ours: this run's GEMM window + flash-attn's forward (composed, not one graph)
            comp = summ["phases_ms"]["serial_fused"]["gemm_window"] + fa["fwd_ms"]
            line["speedup_vs_flash_attn_block"] = {"composed_ms": round(comp, 4),
                                                   "speedup": round(comp / value, 4)}
        log("SQ sweep")
        line["seq_sweep"] = bench_seq_sweep(rgo, rank, world, (1024, 2048, 4096, 8192, 16384, 32768))
        # reduced-round Philox, stand-alone mask runtime ratios
        # vs the paper's silicon (R5/R7 ~ 0.81, R3/R7 ~ 0.67; PAPER.md 5.2).
        log("Philox rounds")
        rr = {}
        for R in (3, 5, 7, 10):
            rr[R], _ = bench_mask_kernel(rgo, dict(cfg, rounds=R), rank, 10, 3)
            rr[R] = max_over_ranks(rr[R], world)
        line["philox_rounds"] = {"mask_ms": {f"R{R}": round(v, 4) for R, v in rr.items()},
                                 "ratio_R5_R7": round(rr[5] / rr[7], 4), "ratio_R3_R7": round(rr[3] / rr[7], 4),
                                 "paper_ratio_R5_R7": 0.81, "paper_ratio_R3_R7": 0.67,
                                 "config": "K1 stand-alone, Llama2-7B mask (2^31 elements), keep 0.9"}
        # the Llama2-7B block with reduced-round Philox: fused baseline vs
        # mechanism B at the same round count
        log("block at reduced rounds")
        br = {}
        for R in (3, 5, 7):
            wr = rgo.workload_preset("llama2_7b")
            wr.philox_rounds = R
            rblocks, rres, _, _, _ = run_block_modes(rgo, wr, rank, world, args, ["serial_fused", "in_gemm", "no_rng"])
            for blk in rblocks.values():
                blk.close()
            del rblocks
            torch.cuda.empty_cache()
            br[f"R{R}"] = {"modes_ms": {m: round(v, 4) for m, v in rres.items()},
                           "speedup_vs_fused": round(rres["serial_fused"] / rres["in_gemm"], 4)}
        br["R10"] = {"modes_ms": {m: line["modes_ms"][m] for m in ("serial_fused", "in_gemm", "no_rng")},
                     "speedup_vs_fused": round(line["modes_ms"]["serial_fused"] / line["modes_ms"]["in_gemm"], 4)}
        line["block_rounds"] = br
    return line


def profiled_traffic(kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed ncu --set full capture (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f).get(kernel)
    except (OSError, ValueError):
        return None


def bench_mask_only(args, rank, world):
    import paper_2410_07531_b200 as rgo
    cfg = dict(L, rounds=args.rounds)
    import torch
    with ClockSampler(torch.cuda.current_device()) as clk:
        ms, elems = bench_mask_kernel(rgo, cfg, rank, args.steps, args.warmup)
    ms = max_over_ranks(ms, world)
    peaks, src = load_peaks()
    sm_mhz = peaks.get("sm_max_mhz", 1965.0)
    int_peak = 148 * 128 * sm_mhz * 1e6
    achieved = elems * (args.rounds + 2) / (ms * 1e-3)
    return {"metric": "mask_gbit_s", "value": round(elems * world / (ms * 1e-3) / 1e9, 2), "unit": "Gbit/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": f"Llama2-7B dropout mask B4 nH32 SQ4096 keep0.9 R{args.rounds}"},
            "roofline": {"bound": "int", "achieved": achieved / 1e12, "peak": int_peak / 1e12, "unit": "Tint-op/s",
                         "frac": achieved / int_peak, "traffic": None},
            "clocks": clk.summary(), "gpu_launches": args.steps}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="block", choices=["block", "mask"])
    ap.add_argument("--rounds", type=int, default=10)
    ap.add_argument("--rng-launch", type=int, nargs=3, default=[0, 0, 0], metavar=("GRID", "BLOCK", "SMEM"),
                    help="mechanism A mask-kernel launch shape (0 = one 256-thread CTA per SM)")
    ap.add_argument("--rng-warps", type=int, default=0, choices=[0, 4, 6, 8, 12, 16],
                    help="mechanism B: RNG warps co-resident in each GEMM CTA (0 = the block's per-workload choice)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the secondary configs (GPT-3 block, attention fwd+bwd, SQ sweep)")
    ap.add_argument("--stall-s", type=float, default=240.0,
                    help="watchdog: exit (printing what was measured) if one section makes no progress this long")
    ap.add_argument("--watchdog-s", type=float, default=600.0,
                    help="exit with an error line if the GPU part has not finished after this many seconds (0 = off)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "reference":
        if rank != 0:
            return
        cfg = dict(L, rounds=args.rounds)
        steps = max(1, min(args.steps, 3))  # each step is a ~10 s CPU sample
        warm = min(max(args.warmup, 0), 1)   # one untimed sample warms caches / thread pool
        for _ in range(warm):
            cpu_reference_block(cfg)
        vals = [cpu_reference_block(cfg) for _ in range(steps)]
        v = sum(x["value"] for x in vals) / len(vals)
        b = vals[-1]
        suite = cpu_baseline_suite(args.rounds)
        print(json.dumps({
            "metric": "llama2_block_ms", "value": round(v, 1), "unit": "ms", "n_gpus": 0, "impl": "reference",
            "steps": steps, "warmup": warm, "higher_is_better": False, "scaling": "weak",
            "config": {"workload": "Llama2-7B block (reference CPU path: generate_mask + attention_dropout_fused; "
                                   "no GEMMs in the reference)", "global_batch": cfg["batch"], "seq_len": cfg["seq"]},
            "cpu_baseline": {"value": round(v, 1), "unit": "ms", "cores": b["cores"], "kind": b["kind"],
                             "sample": b["sample"], "host": suite["host"], "suite": suite},
            "e2e": {"value": round(v, 1), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))
        return

    rank, world, _ = dist_setup()
    # Watchdog: a wedged kernel would otherwise hold the GPU until an outside
    # timeout; exiting the process tears the context down and frees the GPU.
    import threading

    def _watchdog():
        section = _PARTIAL["section"]
        log(f"watchdog: no progress (limit {args.watchdog_s} s, or {args.stall_s} s in one section) "
            f"in: {section}; exiting")
        if rank == 0 and _PARTIAL["line"] is not None:
            # the headline was measured: report it with the extras that completed
            out = dict(_PARTIAL["line"])
            out["watchdog"] = f"extras incomplete: wedged in '{section}' (no progress for {args.stall_s} s)"
            print(json.dumps(out), flush=True)
            os._exit(0)
        if rank == 0:
            print(json.dumps({"metric": "llama2_block_ms",
                              "error": f"watchdog: wedged in '{section}' (limits: {args.watchdog_s} s total, "
                                       f"{args.stall_s} s per section)"}), flush=True)
        os._exit(3)

    wd_stop = threading.Event()
    t_start = time.time()

    def _watch():  # total limit, and a per-section stall limit (every section takes < 1 min)
        while not wd_stop.wait(2.0):
            now = time.time()
            if now - t_start > args.watchdog_s or now - _PARTIAL["since"] > args.stall_s:
                _watchdog()

    wd = threading.Thread(target=_watch, daemon=True)
    _PARTIAL["since"] = time.time()
    if args.watchdog_s > 0:
        wd.start()
    line = bench_block(args, rank, world) if args.workload == "block" else bench_mask_only(args, rank, world)
    if rank == 0 and args.workload == "block":
        import paper_2410_07531_b200 as rgo
        log("drop-in e2e at config O (host arrays through the C ABI)")
        line["e2e_dropin_O"] = bench_dropin_O(rgo)
    wd_stop.set()
    if rank == 0:
        if not args.no_cpu_baseline and world == 1:  # the CPU baseline is an N=1 measurement
            log("CPU baseline (reference, host cores)")
            cb = cpu_reference_block(dict(L, rounds=args.rounds))
            line["cpu_baseline"] = {k: (round(cb[k], 1) if k == "value" else cb[k])
                                    for k in ("value", "unit", "cores", "kind", "sample")}
            log("CPU baseline suite (BASELINE.md section 4)")
            suite = cpu_baseline_suite(args.rounds)
            line["cpu_baseline"]["host"] = suite["host"]
            line["cpu_baseline"]["suite"] = suite
            if "e2e_dropin_O" in line:
                ref_ms = (suite["masks"]["O"]["s"] + suite["attention_O"]["decoupled_s_1thread"]) * 1e3
                line["e2e_dropin_O"]["reference_cpu_ms"] = round(ref_ms, 3)
                line["e2e_dropin_O"]["reference_cpu_how"] = (
                    "the reference's generate_mask (all threads) + attention_dropout_decoupled (single thread, as "
                    "the reference runs it) at config O, same host")
                line["e2e_dropin_O"]["speedup_vs_reference_cpu"] = round(ref_ms / line["e2e_dropin_O"]["value_ms"], 2)
        print(json.dumps(line))
        if "parity" in line and not line["parity"]["ok"]:
            log(f"PARITY FAILURE: {line['parity']}")
            sys.exit(1)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
