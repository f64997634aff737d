# RS grouped raster: parity, interleaved A/B vs piece-by-piece, op DRAM traffic
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_multiproc_fullsize.py -m gpu -q -x -p no:cacheprovider -k "rs or c3 or reduce or RS or scatter or tile_gemm" > gpurun_out/r2s3_rs_parity.log 2>&1
tail -3 gpurun_out/r2s3_rs_parity.log
timeout 900 python tools/rs_ab.py 8 hetero_unfused_1d:core hetero_unfused_1d:core:FICCO_RS_GROUP=0 hetero_fused_1d:core hetero_fused_1d:core:FICCO_RS_GROUP=0 shard_overlap_p2p:core shard_overlap_p2p:core:FICCO_RS_GROUP=0 hetero_unfused_1d:dma hetero_unfused_1d:dma:FICCO_RS_GROUP=0 > gpurun_out/rs_group_ab_g8.log 2>&1
tail -12 gpurun_out/rs_group_ab_g8.log
timeout 900 python tools/rs_ab.py 4 hetero_unfused_1d:core hetero_unfused_1d:core:FICCO_RS_GROUP=0 uniform_fused_1d:core uniform_fused_1d:core:FICCO_RS_GROUP=0 > gpurun_out/rs_group_ab_g4.log 2>&1
tail -8 gpurun_out/rs_group_ab_g4.log
out=gpurun_out/rs_group_traffic.txt; : > $out
for grp in 1 0; do
  FICCO_RS_GROUP=$grp timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:tile_gemm -s 2 -c 1 --csv python tools/op_once.py c3 hetero_unfused_1d core 3 8 2>/dev/null | grep -E '"(gpu__time|dram__bytes)' | awk -F'","' -v v="rs_group=$grp" '{print v, $(NF-2), $NF}' >> $out
done
cat $out
