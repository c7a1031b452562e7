#!/bin/bash
# B-multicast cluster GEMM (MEMO_GEMM_MC=1): bitwise check vs the single-CTA
# kernel, per-shape micro-benchmarks, then alternating cfg2 bench runs.
OUT=${1:-gpurun_out/ab_mc}
mkdir -p $OUT
timeout -s KILL 300 python -m pytest tests/test_gemm_gpu.py -x -q > $OUT/tests.log 2>&1 || { tail -30 $OUT/tests.log; exit 1; }
tail -1 $OUT/tests.log
for rep in 1 2; do
  for arm in ${ARMS:-1 0}; do
    MEMO_GEMM_MC=$arm timeout -s KILL 300 python tools/bench_gemm.py 131072 > $OUT/g_${arm}_$rep.jsonl 2>> $OUT/err.txt
  done
done
for rep in 1 2 3; do
  for arm in ${ARMS:-1 0}; do
    MEMO_GEMM_MC=$arm timeout -s KILL 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/b_${arm}_$rep.json 2>> $OUT/err.txt
  done
done
