# C3 / C2 plain-GEMM raster + A-pinning A/B at real clocks (interleaved), plus DRAM bytes of the wider groups
set -x
for rep in 1 2; do
timeout 600 python tools/ab_env.py 25 16384 8192 3584 1.0 default= alast=FICCO_A_EVICT_LAST:1 g8a=FICCO_GEMM_GROUP_M:8,FICCO_A_EVICT_LAST:1 g16a=FICCO_GEMM_GROUP_M:16,FICCO_A_EVICT_LAST:1 g32a=FICCO_GEMM_GROUP_M:32,FICCO_A_EVICT_LAST:1 > gpurun_out/ab_c3_raster_$rep.log 2>&1
done
timeout 600 python tools/ab_env.py 25 8192 3584 4096 1.0 default= alast=FICCO_A_EVICT_LAST:1 g8a=FICCO_GEMM_GROUP_M:8,FICCO_A_EVICT_LAST:1 g16a=FICCO_GEMM_GROUP_M:16,FICCO_A_EVICT_LAST:1 > gpurun_out/ab_c2_raster.log 2>&1
tail -8 gpurun_out/ab_c3_raster_*.log gpurun_out/ab_c2_raster.log
out=gpurun_out/c3_traffic_ab2.txt; : > $out
for g in 24 32; do
  FICCO_GEMM_GROUP_M=$g FICCO_A_EVICT_LAST=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control base -k regex:tile_gemm -s 1 -c 1 --csv python tools/kernel_once.py 16384 8192 3584 2>/dev/null | grep -E '"(gpu__time|dram__bytes)' | awk -F'","' -v v="g${g}a" '{print v, $(NF-2), $NF}' >> $out
done
FICCO_GEMM_GROUP_M=16 FICCO_A_EVICT_LAST=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control base -k regex:tile_gemm -s 1 -c 1 --csv python tools/kernel_once.py 8192 3584 4096 2>/dev/null | grep -E '"(gpu__time|dram__bytes)' | awk -F'","' '{print "c2_g16a", $(NF-2), $NF}' >> $out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control base -k regex:tile_gemm -s 1 -c 1 --csv python tools/kernel_once.py 8192 3584 4096 2>/dev/null | grep -E '"(gpu__time|dram__bytes)' | awk -F'","' '{print "c2_default", $(NF-2), $NF}' >> $out
cat $out
