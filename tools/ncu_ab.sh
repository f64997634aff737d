# usage: ncu_ab.sh M N K variant...   (run on the GPU box from the repo root)
M=$1; N=$2; K=$3; shift 3
for v in "$@"; do
  ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.max,dram__bytes_read.sum,dram__bytes_write.sum --clock-control base -k regex:tile_gemm -s 1 -c 3 --csv \
    env FICCO_LIB_PATH=build_variants/$v.so python tools/kernel_once.py $M $N $K 2>/dev/null | grep -E '"(gpu__time|gpc__cycles|dram__bytes)' | awk -F'","' -v v=$v '{print v, $(NF-2), $NF}'
done
