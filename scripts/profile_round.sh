#!/bin/bash
# Capture the round's ncu evidence on ONE GPU (run under gpurun).  Reports are
# reduced to CSV on the box (raw metrics + per-instruction source page) so the
# returned gpurun_out/ stays small:
#   launch list of a short bench run (per-launch device times, serialised)
#   --set full of each hot kernel: mask (K1), GEMM FP8 (K2), GEMM + RNG warps (K4),
#   attention fwd with mask bits (K5) / inline Philox (K6), attention bwd (K7)
#   with mask bits / inline Philox / no dropout
set -u
OUT=${1:-gpurun_out}
KEEP=${KEEP_REPORTS:-""}
KERNELS=${KERNELS:-"mask gemm gemm_rng attn_bits attn_philox bwd_bits bwd_philox bwd_none"}
mkdir -p $OUT
if [ -z "${SKIP_LAUNCHES:-}" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_block.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $OUT/bench_under_ncu.log 2>&1
fi
for k in $KERNELS; do
    case $k in
        bwd_*) RX="bwd_main"; SKIP=1 ;;
        *) RX="gemm_kernel|attn_fwd|rng_mask_kernel"; SKIP=1 ;;
    esac
    timeout 400 ncu -f --set full --clock-control none --import-source on -k regex:"$RX" \
        -s $SKIP -c 1 -o /tmp/prof_$k python scripts/prof_kernels.py $k > $OUT/ncu_$k.log 2>&1
    ncu -i /tmp/prof_$k.ncu-rep --page raw --csv > $OUT/raw_$k.csv 2>/dev/null
    ncu -i /tmp/prof_$k.ncu-rep --page source --csv --print-source sass > $OUT/source_$k.csv 2>/dev/null
    gzip -f $OUT/source_$k.csv
    if [ -n "$KEEP" ]; then cp /tmp/prof_$k.ncu-rep $OUT/; fi
    tail -1 $OUT/ncu_$k.log
done
# whole block steps per overlap mode, concurrency preserved (app-range replay)
if [ -z "${SKIP_RANGE:-}" ]; then
mkdir -p $OUT/rng_range
for m in no_rng streams in_gemm serial_fused; do
    timeout 300 ncu --replay-mode app-range --clock-control none --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second,dram__bytes_write.sum,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_elapsed \
        --csv python scripts/prof_block_range.py $m > $OUT/rng_range/$m.csv 2>&1
done
fi
du -sh $OUT
