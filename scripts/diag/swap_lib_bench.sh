#!/bin/bash
# Run bench_attn.py against alternative builds of the library (diagnostics).
for f in scripts/diag/libs/*.so; do
  cp paper_2410_07531_b200/librgo_b200.so /tmp/orig.so
  cp $f paper_2410_07531_b200/librgo_b200.so
  echo "== $f"; timeout 200 python scripts/bench_attn.py > /tmp/ba.txt 2>&1; head -3 /tmp/ba.txt
  cp /tmp/orig.so paper_2410_07531_b200/librgo_b200.so
done
