"""Per-kernel census of the Blackwell-native SASS in librgo_b200.so:
tcgen05 MMAs (UTCQMMA = kind::f8f6f4, UTCHMMA = kind::f16), TMEM loads/stores
(LDTM/STTM), TMA tensor loads (UTMALDG), bulk reduce-adds (UBLKRED), the
Philox multiplies (IMAD.WIDE.U32) and MUFU.EX2, from `cuobjdump -sass`.

    python scripts/sass_census.py [lib.so] > profiles/r02_sass_census.md
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ["UTCQMMA", "UTCHMMA", "LDTM", "STTM", "UTMALDG", "UBLKRED", "UBLKCP", "IMAD.WIDE.U32", "MUFU.EX2",
       "FFMA2", "ELECT", "SYNCS"]


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2410_07531_b200", "librgo_b200.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for ln in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", ln)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_.]+)", ln)
        if not m:
            continue
        op = m.group(1)
        for o in OPS:
            if op == o or op.startswith(o + "."):
                kernels[cur][o] += 1
    demangled = {}
    try:
        out = subprocess.run(["c++filt"], input="\n".join(kernels), capture_output=True, text=True).stdout.splitlines()
        demangled = dict(zip(kernels, out))
    except OSError:
        pass
    tot = collections.Counter()
    print("# SASS census of librgo_b200.so (sm_100a)\n")
    print("`python scripts/sass_census.py` over `cuobjdump -sass`; static instruction counts per kernel "
          "(unrolled loops count once per unrolled copy).  Kernels with none of the listed ops are omitted.\n")
    print("| kernel | " + " | ".join(OPS) + " |")
    print("|---|" + "---|" * len(OPS))
    for k, c in kernels.items():
        tot.update(c)
        if not any(c[o] for o in OPS[:6]) and not c["IMAD.WIDE.U32"]:
            continue
        name = demangled.get(k, k)
        name = re.sub(r"\(.*", "", name)[:90]
        print(f"| `{name}` | " + " | ".join(str(c[o]) for o in OPS) + " |")
    print("| **total (all kernels)** | " + " | ".join(f"**{tot[o]}**" for o in OPS) + " |")
    print(f"\n{len(kernels)} kernels in the library.")


if __name__ == "__main__":
    main()
