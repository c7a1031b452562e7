#!/bin/bash
# Per-shape GEMM A/B: the default kernel choice against MEMO_GEMM_PAIR=0/1, at the
# 7B and 13B layer shapes, alternating arms.  Usage: tools/gemm_arms.sh [outdir] [S]
OUT=${1:-gpurun_out/gemm_arms}; S=${2:-131072}
mkdir -p $OUT
for rep in 1 2; do
  for model in 7b 13b; do
    for arm in auto 0 1; do
      if [ $arm = auto ]; then env_arm=""; else env_arm="MEMO_GEMM_PAIR=$arm"; fi
      env $env_arm GEMM_MODEL=$model timeout 300 python tools/bench_gemm.py $S > $OUT/${model}_${arm}_$rep.jsonl 2>> $OUT/err.txt
    done
  done
done
