# RS grouping at 128-row-block granularity (G = 2/4/8), CP zero-copy K slot: parity, A/B, traffic, C4 bench
set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_multiproc_fullsize.py -m gpu -q -x -p no:cacheprovider -k "rs or c3 or reduce or RS or scatter or cp or c4" > gpurun_out/r2s3_rs_cp_parity.log 2>&1
tail -3 gpurun_out/r2s3_rs_cp_parity.log
for G in 2 4; do
timeout 900 python tools/rs_ab.py $G hetero_unfused_1d:core hetero_unfused_1d:core:FICCO_RS_GROUP=0 hetero_fused_1d:core hetero_fused_1d:core:FICCO_RS_GROUP=0 > gpurun_out/rs_group_ab2_g$G.log 2>&1
tail -6 gpurun_out/rs_group_ab2_g$G.log
done
out=gpurun_out/rs_group_traffic2.txt; : > $out
for G in 2 4 8; do for grp in 1 0; do
  FICCO_RS_GROUP=$grp timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control base -k regex:tile_gemm -s 2 -c 1 --csv python tools/op_once.py c3 hetero_unfused_1d core 3 $G 2>/dev/null | grep -E '"(gpu__time|dram__bytes)' | awk -F'","' -v v="g${G}_rs_group=$grp" '{print v, $(NF-2), $NF}' >> $out
done; done
cat $out
timeout 900 python bench.py --workload c4 --steps 20 --warmup 5 > gpurun_out/r2s3_bench_c4_slot.json 2> gpurun_out/r2s3_bench_c4_slot.err
tail -c 1200 gpurun_out/r2s3_bench_c4_slot.json
