#!/bin/bash
# Interleaved per-shape A/B of GEMM kernel variants (memo_gemm_args.variant via
# GEMM_VARIANT): REPS rounds of every variant in VARIANTS on the shapes in
# GEMM_ONLY (indices into tools/bench_gemm.py's list).  Usage:
#   GEMM_ONLY=0,1 VARIANTS="0 2 4" REPS=4 tools/gemm_ab.sh [outfile] [S]
OUT=${1:-gpurun_out/gemm_ab.jsonl}; S=${2:-131072}
mkdir -p $(dirname $OUT)
for rep in $(seq ${REPS:-4}); do
  for v in ${VARIANTS:-0 2 4}; do
    GEMM_VARIANT=$v GEMM_RASTER=${RASTER:-0} timeout 300 python tools/bench_gemm.py $S | sed "s/^{/{\"variant\": $v, \"raster\": ${RASTER:-0}, \"rep\": $rep, /" >> $OUT
  done
done
