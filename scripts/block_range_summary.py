"""profiles/rNN_block_range.md from profile_round.sh's app-range CSVs."""
import csv, io, os, sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/rng_range"
rnd = sys.argv[2] if len(sys.argv) > 2 else "r01"
modes = ["no_rng", "streams", "in_gemm", "serial_fused"]
data = {}
for m in modes:
    txt = open(os.path.join(src, f"{m}.csv")).read()
    body = txt[txt.index('"ID"'):]
    data[m] = {r["Metric Name"]: float(r["Metric Value"].replace(",", "")) for r in csv.DictReader(io.StringIO(body))}
lines = [f"# {rnd}: whole block steps under `ncu --replay-mode app-range` (concurrency preserved)", "",
         "`scripts/prof_block_range.py MODE` runs one Llama2-7B block step (graph replay) between",
         "cudaProfilerStart/Stop; app-range replay profiles the range as a whole, so mechanism A's",
         "mask kernel is measured *while* it runs beside the GEMMs (kernel replay would serialise",
         "them). Command: `ncu --replay-mode app-range --clock-control none --metrics ...`", "",
         "| mode | step ms | SM clock GHz | tensor pipe active % | tensor-active cycles (M) | fma-heavy active % "
         "| ALU % | issue active % | DRAM write MB |", "|---|---|---|---|---|---|---|---|---|"]
for m in modes:
    d = data[m]
    ms = d["gpu__time_duration.sum"] / 1e6
    ghz = d["sm__cycles_elapsed.avg.per_second"] / 1e9
    ten = d["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]
    cyc = ten / 100 * ms * 1e-3 * ghz * 1e9 / 1e6
    lines.append(f"| {m} | {ms:.3f} | {ghz:.3f} | {ten:.1f} | {cyc:.2f} | "
                 f"{d['sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed']:.1f} | "
                 f"{d['sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_elapsed']:.1f} | "
                 f"{d['smsp__issue_active.avg.pct_of_peak_sustained_elapsed']:.1f} | {d['dram__bytes_write.sum'] / 1e6:.0f} |")
cyc = {m: data[m]["gpu__time_duration.sum"] * data[m]["sm__cycles_elapsed.avg.per_second"] / 1e9 / 1e6 for m in modes}
lines += ["", "SM cycles per step (M): " + ", ".join(f"{m} {cyc[m]:.2f}" for m in modes), "",
          "Reading: the tensor-active cycle count is the same in every mode -- the GEMM and attention",
          "MMA work does not change -- and with realistic (unit-variance) data every mode runs against",
          "the 1 kW power cap, the no-RNG floor included (SM clock 1.47-1.64 GHz of 1.965). The RNG",
          "therefore costs (a) SM clock where its IMAD.WIDE work (fma-heavy pipe) runs beside the",
          "tensor cores and (b) extra SM cycles for the part of the mask that does not fit in the GEMM",
          "window (mechanism B's tail drain, mechanism A's join before attention; the fused baseline's",
          "whole Philox inside attention). Mechanism B with the per-workload RNG-warp count keeps the",
          "clock of the no-RNG floor and adds the fewest cycles: it is the mechanism the bench reports."]
out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", f"{rnd}_block_range.md")
open(out, "w").write("\n".join(lines) + "\n")
print("\n".join(lines[7:13]))
