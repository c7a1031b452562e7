#!/bin/bash
# full ncu captures of the attention kernels at S=131072 (one launch each); tag = $1
tag=${1:-cur}
mkdir -p gpurun_out
for k in attn_bwd_dkdv attn_bwd_dq attn_fwd; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -c 1 \
      -o gpurun_out/prof_${tag}_$k python tools/bench_attn.py 131072 > /dev/null 2>> gpurun_out/prof_err.txt
done
ls -la gpurun_out
