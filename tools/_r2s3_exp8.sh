# cross-gate AG row groups (FICCO_AG_GROUP_GATES) on EP and C3': op vs plain-kernel ratio in the same run
set -x
for rep in 1 2; do
for v in 1 0; do
  FICCO_AG_GROUP_GATES=$v timeout 900 python bench.py --workload ep --steps 10 --warmup 3 --headline-only --no-cpu > gpurun_out/agg_ep_${v}_$rep.json 2>/dev/null
  FICCO_AG_GROUP_GATES=$v timeout 900 python bench.py --workload c3p --steps 20 --warmup 5 --headline-only --no-cpu > gpurun_out/agg_c3p_${v}_$rep.json 2>/dev/null
done
done
for f in gpurun_out/agg_*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', d['value'], r['kernel_alone_us'], round(d['value']/r['kernel_alone_us'],4), d.get('own_serial_us'), d['clocks']['sm_mhz'])"; done
