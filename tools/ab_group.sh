#!/bin/bash
# Raster-band A/B of the clustered single-CTA GEMM (MEMO_GEMM_GROUP_M, in M-tiles)
# on the whole cfg2 step, alternating arms.
OUT=${1:-gpurun_out/ab_group}
mkdir -p $OUT
for rep in 1 2; do
  for g in ${ARMS:-8 16 32}; do
    MEMO_GEMM_GROUP_M=$g timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/b_${g}_$rep.json 2>> $OUT/err.txt
  done
done
