#!/bin/bash
# compute-sanitizer over scripts/sanitize_cases.py (run under gpurun, one GPU).
OUT=${1:-gpurun_out/sanitize}
mkdir -p $OUT
for tool in memcheck synccheck racecheck initcheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > $OUT/$tool.log 2>&1
    echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' $OUT/$tool.log | tail -1)"
done
