"""Turn the profile_round.sh CSVs (gpurun_out/) into profiles/rNN_*.md."""
import csv, gzip, io, json, os, sys
from collections import defaultdict

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_summary import KEYS

SRC = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
RND = sys.argv[2] if len(sys.argv) > 2 else "r01"
NAME = sys.argv[3] if len(sys.argv) > 3 else "kernels"   # profiles/{RND}_{NAME}.md
DST = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
os.makedirs(DST, exist_ok=True)
EXTRA = ["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
         "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
         "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
         "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
         "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active"]

lines = [f"# {RND}: ncu --set full, one launch per hot kernel (B200, Llama2-7B shapes)", "",
         "Captured by `scripts/profile_round.sh` (`ncu --set full --clock-control none --import-source on`,",
         "one GPU), reduced by `scripts/make_profiles.py`. Per-launch times under ncu are cold-cache and",
         "serialised: compare shares, not absolutes.", ""]
for k, title in (("mask", "K1 rng_mask_kernel<10> (2^31 elements)"), ("gemm", "K2 FP8 GEMM FFN1 SwiGLU 16384x22016x4096"),
                 ("gemm_rng", "K4 FP8 GEMM FFN1 + co-resident RNG warps (12 per CTA, the Llama2-7B block's count)"),
                 ("gemm_rng16", "K4 FP8 GEMM FFN1 + 16 co-resident RNG warps per CTA"),
                 ("attn_bits", "K5 attention fwd, mask bits (B4 H32 S4096 D128)"),
                 ("attn_philox", "K6 attention fwd, inline Philox-10"),
                 ("bwd_bits", "K7 attention bwd, mask bits (B4 H32 S4096 D128)"),
                 ("bwd_philox", "K7 attention bwd, inline Philox-10 (fused baseline)"),
                 ("bwd_none", "K7 attention bwd, no dropout")):
    p = os.path.join(SRC, f"raw_{k}.csv")
    if not os.path.exists(p):
        continue
    rows = list(csv.reader(open(p)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    lines.append(f"## {title}")
    lines.append(f"`{vals[hdr.index('Kernel Name')][:110]}`")
    lines.append("")
    lines.append("| metric | value |")
    lines.append("|---|---|")
    for key in KEYS + EXTRA:
        if key in hdr:
            i = hdr.index(key)
            lines.append(f"| {key} | {vals[i]} {units[i]} |")
    # dram traffic per launch
    try:
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
        tot = float(vals[ir]) * scale[units[ir]] + float(vals[iw]) * scale[units[iw]]
        lines.append(f"| traffic (read+write) | {tot / 1e6:.1f} Mbyte |")
    except (ValueError, KeyError):
        pass
    # top stall lines from the source page
    sp = os.path.join(SRC, f"source_{k}.csv.gz")
    if os.path.exists(sp):
        srows = list(csv.reader(io.TextIOWrapper(gzip.open(sp), encoding="utf-8")))
        sh = srows[1]
        isrc, iall = sh.index("Source"), sh.index("Warp Stall Sampling (All Samples)")
        tot = sum(float(r[iall] or 0) for r in srows[2:])
        top = sorted(srows[2:], key=lambda r: -float(r[iall] or 0))[:8]
        lines.append("")
        lines.append(f"Top stall-sampled SASS ({int(tot)} samples):")
        lines.append("")
        for r in top:
            lines.append(f"- {float(r[iall]) / tot * 100:5.1f}%  `{r[isrc].strip()[:90]}`")
    lines.append("")
open(os.path.join(DST, f"{RND}_{NAME}.md"), "w").write("\n".join(lines) + "\n")

# launch list: kernel time shares over the bench's timed steps
p = os.path.join(SRC, "launches_block.csv")
if os.path.exists(p):
    txt = open(p).read()
    body = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
    rows = list(csv.DictReader(io.StringIO(body)))
    tot = defaultdict(float); cnt = defaultdict(int)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")[:70]
        v = float(r["Metric Value"]) * (1e-3 if r["Metric Unit"] == "ns" else (1.0 if r["Metric Unit"] == "us" else 1e3))
        tot[name] += v; cnt[name] += 1
    s = sum(tot.values())
    out = [f"# {RND}: launch list of `bench.py --steps 2 --warmup 3 --no-cpu-baseline` under ncu "
           "(gpu__time_duration.sum)", "",
           "All kernels of the run: the Llama2-7B, GPT-3 and MoE blocks (4 modes x alternating passes x (warm-up + timed) steps), the chunked pipeline, the",
           "stand-alone mask runs, attention fwd+bwd (bits / fused Philox / none) and the SQ sweep.",
           "Serialised, cold-cache times: use the shares.", "", "| kernel | launches | total us | share |",
           "|---|---|---|---|"]
    for name, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"| `{name}` | {cnt[name]} | {v:.0f} | {v / s * 100:.1f}% |")
    open(os.path.join(DST, f"{RND}_launches.md"), "w").write("\n".join(out) + "\n")
print("wrote", DST)
