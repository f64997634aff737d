# W beyond L2: group size x W policy at real clocks (interleaved), and EP's W policy
set -x
timeout 900 python tools/ab_env.py 12 16384 8192 14336 1.0 first=FICCO_B_HINT:first last=FICCO_B_HINT:last last_g8=FICCO_B_HINT:last,FICCO_GEMM_GROUP_M:8,FICCO_A_EVICT_LAST:1 last_g16=FICCO_B_HINT:last,FICCO_GEMM_GROUP_M:16,FICCO_A_EVICT_LAST:1 > gpurun_out/ab_grp_g2.log 2>&1
timeout 900 python tools/ab_env.py 15 16384 8192 7168 1.0 first=FICCO_B_HINT:first last=FICCO_B_HINT:last last_g16=FICCO_B_HINT:last,FICCO_GEMM_GROUP_M:16,FICCO_A_EVICT_LAST:1 > gpurun_out/ab_grp_g4.log 2>&1
timeout 900 python tools/ab_env.py 15 16384 7168 8192 1.0 first=FICCO_B_HINT:first last=FICCO_B_HINT:last last_g16=FICCO_B_HINT:last,FICCO_GEMM_GROUP_M:16,FICCO_A_EVICT_LAST:1 > gpurun_out/ab_grp_c3p.log 2>&1
timeout 1200 python tools/ab_env.py 5 147456 28672 4096 1.0 first=FICCO_B_HINT:first last=FICCO_B_HINT:last normal=FICCO_B_HINT:normal > gpurun_out/ab_grp_ep.log 2>&1
grep -h median gpurun_out/ab_grp_*.log
out=gpurun_out/ep_traffic.txt; : > $out
for v in first last; do
  FICCO_B_HINT=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control base -k regex:tile_gemm -s 1 -c 1 --csv python tools/kernel_once.py 147456 28672 4096 2>/dev/null | grep -E '"(gpu__time|dram__bytes)' | awk -F'","' -v v="ep_$v" '{print v, $(NF-2), $NF}' >> $out
done
cat $out
