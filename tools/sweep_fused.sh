timeout 200 python -m pytest tests/test_attention_gpu.py -x -q 2>&1 | tail -1
timeout 100 python tools/bench_attn.py 32768 131072 2>&1 | tail -2 | cut -c1-470
MEMO_ATTN_BWD=fused timeout 100 python tools/bench_attn.py 32768 131072 2>&1 | grep -o '"S": [0-9]*\|"dkdv_ms": [0-9.]*' | paste -sd' '
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_dq -c 1 -o gpurun_out/prof_e_dq python tools/bench_attn.py 32768 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:attn_bwd_dkdv -c 1 -o gpurun_out/prof_e_dkdv python tools/bench_attn.py 32768 > /dev/null 2>&1
