for v in 5 6 1 5; do
  MEMO_ATTN_FWD_VARIANT=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/ab_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json')); print('v=$v', round(d['value']), round(d['mfu'],4), d['clocks']['sm_mhz'], {k:(round(x['ms_per_step'],1)) for k,x in d['kernels'].items()})"
done
