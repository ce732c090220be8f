"""profiles/rNN_block_sweep.md tables from scripts/sweep_block.py's JSON.
usage: sweep_table.py sweep.json"""
import json, sys

rows = json.load(open(sys.argv[1]))
seqs, heads = sorted({r["seq"] for r in rows}), sorted({r["heads"] for r in rows})
R = {(r["seq"], r["heads"]): r for r in rows}


def table(title, cell):
    out = [title, "", "| SQ \\ nH | " + " | ".join(map(str, heads)) + " |", "|---" * (len(heads) + 1) + "|"]
    out += [f"| {s} | " + " | ".join(cell(R[s, h]) for h in heads) + " |" for s in seqs]
    return out + [""]


def best(r):
    return min(r["in_gemm"], r["streams"])


lines = table("Speedup = fused-dropout baseline / best overlap mechanism (B = in-GEMM RNG warps, A = streams)",
              lambda r: f"{r['speedup']:.2f}× ({'B' if r['mechanism'] == 'in_gemm' else 'A'})")
lines += table("Step times (ms): no RNG / fused baseline / best overlap",
               lambda r: f"{r['no_rng']:.2f} / {r['serial_fused']:.2f} / {best(r):.2f}")
lines += table("Hidden fraction of the fused baseline's dropout cost: (fused - overlap) / (fused - no RNG)",
               lambda r: f"{(r['serial_fused'] - best(r)) / max(r['serial_fused'] - r['no_rng'], 1e-9):.2f}")
print("\n".join(lines))
