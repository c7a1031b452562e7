#!/bin/bash
# compute-sanitizer passes on small configs (race detection / sanitizers).
#   memcheck  : out-of-bounds / misaligned global & shared accesses, leaks of device allocations
#   racecheck : shared-memory data races (TMA/mbarrier traffic is asynchronous-proxy and not tracked)
#   synccheck : illegal barrier / warp-sync usage
OUT=${1:-gpurun_out/sanitize}
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
      python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$tool.txt 2>&1
  echo "smoke $tool rc=$?" | tee -a $OUT/summary.txt
  timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
      python tools/stress_attn.py 512 2 128 2 > $OUT/attn128_$tool.txt 2>&1
  echo "attn D=128 $tool rc=$?" | tee -a $OUT/summary.txt
  timeout 900 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
      python tools/stress_attn.py 512 2 64 2 > $OUT/attn64_$tool.txt 2>&1
  echo "attn D=64 $tool rc=$?" | tee -a $OUT/summary.txt
done
