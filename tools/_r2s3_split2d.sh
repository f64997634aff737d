set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "slab_split or 2d or ring_split" > gpurun_out/split2d_tests.log 2>&1
tail -2 gpurun_out/split2d_tests.log
timeout 900 python tools/fine_ab.py c2 uniform_fused_2d:full:0:FICCO_2D_SPLIT=1 uniform_fused_2d:full:0:FICCO_2D_SPLIT=2 shard_overlap_p2p:full:0 > gpurun_out/split2d_c2.log 2>&1
tail -5 gpurun_out/split2d_c2.log
for rep in 1 2; do for sp in 1 2 3; do
  FICCO_2D_SPLIT=$sp timeout 600 python bench.py --workload c1 --steps 20 --warmup 5 --headline-only --no-cpu > gpurun_out/split2d_c1_${sp}_$rep.json 2>/dev/null
done; done
for f in gpurun_out/split2d_c1_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', d['value'], r['kernel_alone_us'], round(d['value']/r['kernel_alone_us'],4), d['own_serial_us'], d['copy_program_GBps'])"; done
