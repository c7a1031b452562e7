# fused attention backward: parity tests, timing (dbg 0 = product, 3 = no dQ reduce/ordering), ncu capture
set -x
timeout 200 python -m pytest tests/test_attention_gpu.py -x -q 2>&1 | tail -2
for d in ${DBGS:-0 3}; do MEMO_ATTN_DEBUG=$d timeout 200 python tools/bench_attn.py 32768 131072 2>&1 | tail -2 | cut -c1-420; done
MEMO_ATTN_DEBUG=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_fused -c 1 -o gpurun_out/prof_fused_${TAG:-x} python tools/bench_attn.py 32768 > /dev/null 2>&1
ls gpurun_out
