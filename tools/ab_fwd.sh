# forward-variant A/B: standalone kernel TF/s, then whole-step throughput (power-capped)
for v in ${VARIANTS:-8 9 10}; do echo "v=$v $(MEMO_ATTN_FWD_VARIANT=$v timeout 100 python tools/bench_attn.py 32768 131072 2>&1 | grep -o '"S": [0-9]*\|"fwd_tflops": [0-9.]*' | paste -sd' ')"; done
for v in ${STEP_VARIANTS:-8 5}; do
  MEMO_ATTN_FWD_VARIANT=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json')); print('step v=$v', round(d['value']), round(d['mfu'],4), d['clocks']['sm_mhz'], {k:(round(x['ms_per_step'],1)) for k,x in d['kernels'].items()})"
done
