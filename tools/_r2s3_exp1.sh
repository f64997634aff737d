# session-3 experiments: host enqueue gap, C3 traffic vs L2 policy / raster, RS kinds table
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python tools/host_gap.py hetero_unfused_1d shard_overlap_p2p hetero_fused_1d > gpurun_out/host_gap.log 2>&1
tail -8 gpurun_out/host_gap.log
timeout 1200 bash tools/c3_traffic_ab.sh > gpurun_out/c3_traffic_ab.log 2>&1
tail -70 gpurun_out/c3_traffic_ab.txt
timeout 900 python bench.py --workload c3 --steps 20 --warmup 5 > gpurun_out/r2s3_bench_c3.json 2> gpurun_out/r2s3_bench_c3.err
tail -c 1500 gpurun_out/r2s3_bench_c3.json
