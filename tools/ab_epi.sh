#!/bin/bash
# A/B of the staged GEMM epilogue: GEMM parity tests, then alternating cfg2 bench
# runs and per-shape GEMM micro-benchmarks with MEMO_GEMM_EPI_STAGE=1 (default) / 0.
OUT=${1:-gpurun_out/ab_epi}
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_step_gpu.py -x -q > $OUT/tests.log 2>&1 || { tail -30 $OUT/tests.log; exit 1; }
tail -1 $OUT/tests.log
for rep in 1 2 3; do
  for arm in ${ARMS:-1 0}; do
    MEMO_GEMM_EPI_STAGE=$arm timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > $OUT/b_${arm}_$rep.json 2>> $OUT/err.txt
  done
done
for rep in 1 2; do
  for arm in ${ARMS:-1 0}; do
    MEMO_GEMM_EPI_STAGE=$arm timeout 300 python tools/bench_gemm.py 131072 > $OUT/g_${arm}_$rep.jsonl 2>> $OUT/err.txt
  done
done
