# does an L2 persisting set-aside make evict_last pinning hold? (EP and C3 G2 plain GEMM DRAM bytes)
set -x
out=gpurun_out/persist_traffic.txt; : > $out
for shape in "147456 28672 4096" "16384 8192 14336"; do
  set -- $shape
  for mb in none 32 64 96; do
    if [ $mb = none ]; then e=""; else e="FICCO_L2_PERSIST_MB=$mb"; fi
    env $e ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control base -k regex:tile_gemm -s 1 -c 1 --csv python tools/kernel_once.py $1 $2 $3 2>/dev/null | grep -E '"(gpu__time|dram__bytes)' | awk -F'","' -v v="$1x$2x$3_persist$mb" '{print v, $(NF-2), $NF}' >> $out
  done
done
cat $out
