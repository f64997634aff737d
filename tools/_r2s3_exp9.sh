# EP plain GEMM: DRAM reads vs row-group size and A policy (which operand is re-read?)
set -x
out=gpurun_out/ep_groups.txt; : > $out
M=147456; N=28672; K=4096
for v in "g8a FICCO_GEMM_GROUP_M=8 FICCO_A_EVICT_LAST=1" "g16a FICCO_GEMM_GROUP_M=16 FICCO_A_EVICT_LAST=1" "g32a FICCO_GEMM_GROUP_M=32 FICCO_A_EVICT_LAST=1" "g16f FICCO_GEMM_GROUP_M=16 FICCO_A_EVICT_LAST=0" "g16a_bn FICCO_GEMM_GROUP_M=16 FICCO_A_EVICT_LAST=1 FICCO_B_HINT=normal" "g16a_bf FICCO_GEMM_GROUP_M=16 FICCO_A_EVICT_LAST=1 FICCO_B_HINT=first"; do
  set -- $v; name=$1; shift
  env "$@" ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum --clock-control base -k regex:tile_gemm -s 1 -c 1 --csv python tools/kernel_once.py $M $N $K 2>/dev/null | grep -E '"(gpu__time|dram__bytes|lts__t)' | awk -F'","' -v v="$name" '{print v, $(NF-2), $NF}' >> $out
done
cat $out
