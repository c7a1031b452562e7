#!/bin/bash
# Interleaved A/B of the attention kernels between two builds of libmemo.so
# (default: the HEAD build in paper_2407_12117_b200/_lib_base vs the working
# tree's _lib), plus a bitwise comparison of their outputs.
#   tools/ab_attn.sh [S] [reps]     (run under gpurun)
S=${1:-131072}; REPS=${2:-2}
A=${LIB_A:-paper_2407_12117_b200/_lib_base/libmemo.so}
B=${LIB_B:-paper_2407_12117_b200/_lib/libmemo.so}
out=gpurun_out/ab_attn; mkdir -p $out
MEMO_LIB_PATH=$A python tools/attn_golden_probe.py save 8192 4 128 $out/golden_a.pt
MEMO_LIB_PATH=$B python tools/attn_golden_probe.py check 8192 4 128 $out/golden_a.pt 2>&1 | tail -2
for r in $(seq $REPS); do
  for lib in A B; do
    eval path=\$$lib
    echo -n "$lib " ; MEMO_NO_FA2=1 MEMO_LIB_PATH=$path python tools/bench_attn.py $S
  done
done
# forward FMA-share sweep on the ablation library (FWD_SWEEP="8 11 14 10 9")
for v in ${FWD_SWEEP:-}; do
  echo -n "fwd_variant=$v "; MEMO_NO_FA2=1 MEMO_ATTN_FWD_VARIANT=$v MEMO_LIB_PATH=paper_2407_12117_b200/_lib_ablations/libmemo.so \
    python tools/bench_attn.py $S | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['S'], round(d['fwd_ms'],2), round(d['fwd_tflops'],1))"
done
