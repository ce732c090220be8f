#!/bin/bash
# A/B a benchmark script across alternative library builds, interleaved:
#   scripts/diag/ab_libs.sh "python scripts/bench_attn.py" [rounds]  (builds in ablibs/*.so)
# Each build is selected through RGO_LIB_PATH (paper_2410_07531_b200/_lib.py).
CMD=${1:-"python scripts/bench_attn.py"}
ROUNDS=${2:-3}
for r in $(seq $ROUNDS); do
  for f in ablibs/*.so; do
    echo "== $(basename $f) round $r"; RGO_LIB_PATH=$PWD/$f timeout 300 $CMD 2>&1 | tail -${TAIL:-4}
  done
done
