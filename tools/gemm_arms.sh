#!/bin/bash
# Per-shape GEMM A/B: the default kernel choice against the forced single-CTA (2) and
# CTA-pair (4) kernels (memo_gemm_args.variant via GEMM_VARIANT), at the
# 7B and 13B layer shapes, alternating arms.  Usage: tools/gemm_arms.sh [outdir] [S]
OUT=${1:-gpurun_out/gemm_arms}; S=${2:-131072}
mkdir -p $OUT
for rep in 1 2; do
  for model in 7b 13b; do
    for arm in 0 2 4; do
      GEMM_VARIANT=$arm GEMM_MODEL=$model timeout 300 python tools/bench_gemm.py $S > $OUT/${model}_${arm}_$rep.jsonl 2>> $OUT/err.txt
    done
  done
done
