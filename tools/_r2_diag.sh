# fine-grain vs ring diagnosis + ncu launch list + op-kernel captures (one B200)
set -x
timeout 300 python tools/fine_vs_ring.py c2 dma > gpurun_out/r2_fvr_c2_dma.json 2>&1
timeout 300 python tools/fine_vs_ring.py c2 core > gpurun_out/r2_fvr_c2_core.json 2>&1
timeout 300 python tools/fine_vs_ring.py c4 dma > gpurun_out/r2_fvr_c4_dma.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_c2.csv python bench.py --steps 2 --warmup 3 --headline-only --no-cpu > gpurun_out/r2_launches_c2.log 2>&1
for spec in "c2 hetero_unfused_1d dma" "c3 hetero_unfused_1d core" "c4 hetero_unfused_1d dma"; do
  set -- $spec
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile_gemm -s 2 -c 1 -f -o gpurun_out/r2_ncu_op_$1_$2_$3 python tools/op_once.py $1 $2 $3 3 > gpurun_out/r2_ncu_op_$1.log 2>&1
done
ls -la gpurun_out
