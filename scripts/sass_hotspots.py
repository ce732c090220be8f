"""Top stall-sampled SASS instructions of an ncu source-page CSV (gz ok)."""
import csv, gzip, io, sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
opener = gzip.open if path.endswith(".gz") else open
rows = list(csv.reader(io.TextIOWrapper(opener(path, "rb"), encoding="utf-8")))
hdr = rows[1]
ia, isrc, iall, inot = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), \
    hdr.index("Warp Stall Sampling (Not-issued Samples)")
body = rows[2:]
tot = sum(int(r[iall] or 0) for r in body)
print("total samples", tot, "instructions", len(body))
idx = sorted(range(len(body)), key=lambda i: -int(body[i][iall] or 0))[:n]
for i in sorted(idx):
    r = body[i]
    print(f"{i:5d} {int(r[iall]):7d} {int(r[inot]):7d}  {r[isrc].strip()[:90]}")
