#!/bin/bash
# Build an alternative librgo_b200.so with extra nvcc flags into ablibs/NAME.so (repo root; remove it after the A/B run)
# (for scripts/diag/ab_libs.sh):  scripts/diag/build_variant.sh NAME "-DRGO_POLY_EVERY=0" [files...]
# With files listed (e.g. attn_fwd_sm100.cu), the objects of the in-tree build are reused and
# only those units are recompiled with the extra flags.
set -e
NAME=$1; FLAGS=$2; shift 2 || true
ROOT=$(cd "$(dirname "$0")/../.." && pwd)
T=/tmp/rgo_variant_$NAME
rm -rf $T && mkdir -p $T/pkg && cp -a $ROOT/paper_2410_07531_b200/csrc $T/pkg/ && cp -r $ROOT/include $T/
if [ $# -gt 0 ]; then
  sleep 1; for f in "$@"; do touch $T/pkg/csrc/$f; done
else
  rm -rf $T/pkg/csrc/build
fi
mkdir -p $ROOT/ablibs
make -s -j16 -C $T/pkg/csrc NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$T/include -I. --expt-relaxed-constexpr $FLAGS" OUT=$ROOT/ablibs/$NAME.so
