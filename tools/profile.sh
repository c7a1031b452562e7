#!/bin/bash
# ncu evidence for profiles/: launch list of bench.py and full captures of the top kernels.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.json 2> gpurun_out/launch_err.txt
for k in attn_bwd_dkdv attn_bwd_dq attn_fwd_kernel; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/prof_$k python tools/bench_attn.py 131072 > /dev/null 2>> gpurun_out/prof_err.txt
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -c 1 \
    -o gpurun_out/prof_gemm python tools/bench_gemm.py 131072 > /dev/null 2>> gpurun_out/prof_err.txt
ls -la gpurun_out
