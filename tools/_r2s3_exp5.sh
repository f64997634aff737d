# W beyond L2: B (weight) L2 policy and group size, plain GEMM (ncu bytes at base clocks + interleaved real clocks)
set -x
out=gpurun_out/bhint_traffic.txt; : > $out
for shape in "16384 8192 14336" "16384 8192 7168" "16384 7168 8192"; do
  set -- $shape
  for v in first last normal; do
    FICCO_B_HINT=$v ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control base -k regex:tile_gemm -s 1 -c 1 --csv python tools/kernel_once.py $1 $2 $3 2>/dev/null | grep -E '"(gpu__time|dram__bytes)' | awk -F'","' -v v="$1x$2x$3_$v" '{print v, $(NF-2), $NF}' >> $out
  done
  for gm in 8 16; do
    FICCO_B_HINT=last FICCO_GEMM_GROUP_M=$gm FICCO_A_EVICT_LAST=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control base -k regex:tile_gemm -s 1 -c 1 --csv python tools/kernel_once.py $1 $2 $3 2>/dev/null | grep -E '"(gpu__time|dram__bytes)' | awk -F'","' -v v="$1x$2x$3_last_g$gm" '{print v, $(NF-2), $NF}' >> $out
  done
done
cat $out
timeout 900 python tools/ab_env.py 15 16384 8192 14336 1.0 first=FICCO_B_HINT:first last=FICCO_B_HINT:last normal=FICCO_B_HINT:normal > gpurun_out/ab_bhint_g2.log 2>&1
timeout 900 python tools/ab_env.py 20 16384 8192 7168 1.0 first=FICCO_B_HINT:first last=FICCO_B_HINT:last normal=FICCO_B_HINT:normal > gpurun_out/ab_bhint_g4.log 2>&1
timeout 900 python tools/ab_env.py 15 16384 7168 8192 1.0 first=FICCO_B_HINT:first last=FICCO_B_HINT:last normal=FICCO_B_HINT:normal > gpurun_out/ab_bhint_c3p.log 2>&1
grep median gpurun_out/ab_bhint_*.log
