#!/bin/bash
# A/B a benchmark script across alternative library builds, interleaved:
#   scripts/diag/ab_libs.sh "python scripts/bench_attn.py" [rounds]  (builds in scripts/diag/libs/*.so)
CMD=${1:-"python scripts/bench_attn.py"}
ROUNDS=${2:-3}
cp paper_2410_07531_b200/librgo_b200.so /tmp/orig.so
for r in $(seq $ROUNDS); do
  for f in scripts/diag/libs/*.so; do
    cp $f paper_2410_07531_b200/librgo_b200.so
    echo "== $(basename $f) round $r"; timeout 300 $CMD 2>&1 | tail -${TAIL:-4}
  done
done
cp /tmp/orig.so paper_2410_07531_b200/librgo_b200.so
