# final-code ncu evidence for the default headline (C2) and the C4 score-write kernel; launch list of the default command
set -x
mkdir -p gpurun_out/final7
for spec in "c2 hetero_unfused_1d dma 8" "c4 hetero_unfused_1d dma 8"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_gemm -s 2 -c 1 -f -o gpurun_out/r2_ncu_op_$1_g$4_$2_$3 python tools/op_once.py $1 $2 $3 3 $4 > gpurun_out/final7/ncu_op_$1.log 2>&1
done
python tools/traffic_files.py gpurun_out > gpurun_out/final7/traffic_files.log 2>&1
cp profiles/r02_ncu_traffic_c2_*.json profiles/r02_ncu_op_c2_*.json profiles/r02_ncu_traffic_c4_*.json profiles/r02_ncu_op_c4_*.json gpurun_out/final7/
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final7/launches_c2.csv python bench.py --steps 3 --warmup 3 --headline-only --no-cpu > gpurun_out/final7/launches_c2.log 2>&1
cat gpurun_out/final7/traffic_files.log
