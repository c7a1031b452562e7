#!/bin/bash
# ncu evidence for profiles/: launch list of bench.py and one `--set full` capture of each top kernel
# at the bench shapes (S=131072, H=32, D=128; GEMMs of the 7B layer).  Usage: tools/profile.sh [outdir]
OUT=${1:-gpurun_out/prof}
mkdir -p $OUT
set -x
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-swap-delta > $OUT/bench_under_ncu.json 2> $OUT/launch_err.txt
for k in attn_bwd_dkdv_tm attn_bwd_dq attn_fwd_pp; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o $OUT/prof_$k python tools/bench_attn.py 131072 > /dev/null 2>> $OUT/prof_err.txt
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -c 1 \
    -o $OUT/prof_gemm_tc python tools/bench_gemm.py 131072 > /dev/null 2>> $OUT/prof_err.txt
ls -la $OUT
