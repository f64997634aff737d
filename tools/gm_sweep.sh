for shape in "16384 8192 3584" "16384 131072 128" "8192 3584 4096"; do
for gm in 1 4 16 64; do
  FICCO_GEMM_GROUP_M=$gm ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control base -k regex:tile_gemm -s 1 -c 2 --csv python tools/kernel_once.py $shape 2>/dev/null | grep -E '"(gpu__time|dram__bytes_read)' | awk -F'","' -v v="$shape gm$gm" '{print v, $(NF-2), $NF}'
done; done
