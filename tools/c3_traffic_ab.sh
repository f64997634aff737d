# C3 plain-GEMM DRAM traffic vs L2 policy / raster (run on the GPU box from the repo root).
# usage: bash tools/c3_traffic_ab.sh [M N K]   -> gpurun_out/c3_traffic_ab.txt
M=${1:-16384}; N=${2:-8192}; K=${3:-3584}
out=gpurun_out/c3_traffic_ab.txt
: > $out
run() {
  label=$1; shift
  env "$@" ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control base -k regex:tile_gemm -s 1 -c 2 --csv python tools/kernel_once.py $M $N $K 2>/dev/null \
    | grep -E '"(gpu__time|dram__bytes|lts__t_sector)' | awk -F'","' -v v="$label" '{print v, $(NF-2), $NF}' >> $out
}
run default X=1
run a_last FICCO_A_EVICT_LAST=1
run a_first FICCO_A_EVICT_LAST=0
run out_plain FICCO_OUT_HINT=none
run a_last_out_plain FICCO_A_EVICT_LAST=1 FICCO_OUT_HINT=none
for g in 2 4 8 16; do run group$g FICCO_GEMM_GROUP_M=$g; run group${g}_alast FICCO_GEMM_GROUP_M=$g FICCO_A_EVICT_LAST=1; done
cat $out
