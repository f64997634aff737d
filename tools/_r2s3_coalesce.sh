set -x
FICCO_COALESCE=1 timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "virtual_matches_oracle or cp_qk or a2a or input_slot or kv_slot or ragged or core_agent or full_size or c1" > gpurun_out/coalesce_tests.log 2>&1
tail -2 gpurun_out/coalesce_tests.log
K="hetero_unfused_1d hetero_fused_1d uniform_fused_1d uniform_fused_2d"
specs=""; for k in $K; do specs="$specs $k:full:0:FICCO_COALESCE=0 $k:full:0:FICCO_COALESCE=1"; done
timeout 1200 python tools/fine_ab.py c2 $specs shard_overlap_p2p:full:0 > gpurun_out/coalesce_c2.log 2>&1
tail -11 gpurun_out/coalesce_c2.log
specs=""; for k in hetero_unfused_1d hetero_fused_1d uniform_fused_1d; do specs="$specs $k:full:0:FICCO_COALESCE=0 $k:full:0:FICCO_COALESCE=1"; done
timeout 1200 python tools/fine_ab.py c4 $specs shard_overlap_p2p:full:0 > gpurun_out/coalesce_c4.log 2>&1
tail -9 gpurun_out/coalesce_c4.log
for rep in 1 2; do for v in 0 1; do
  FICCO_COALESCE=$v timeout 600 python bench.py --workload c1 --steps 20 --warmup 5 --headline-only --no-cpu > gpurun_out/coalesce_c1_${v}_$rep.json 2>/dev/null
done; done
for f in gpurun_out/coalesce_c1_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
print('$f', d['value'], r['kernel_alone_us'], round(d['value']/r['kernel_alone_us'],4), d['own_serial_us'], d['copy_program_GBps'])" 2>&1 | tail -1; done
