set -x
mkdir -p gpurun_out/final
timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/final/gputest2.log 2>&1
tail -3 gpurun_out/final/gputest2.log
for spec in "c1 uniform_fused_2d dma 4" "c3p hetero_unfused_1d dma 8"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_gemm -s 2 -c 1 -f -o gpurun_out/r2_ncu_op_$1_g$4_$2_$3 python tools/op_once.py $1 $2 $3 3 $4 > gpurun_out/final/ncu_op_$1_g$4.log 2>&1
done
python tools/traffic_files.py gpurun_out > gpurun_out/final/traffic_files2.log 2>&1
cp profiles/r02_ncu_traffic_c1_*.json profiles/r02_ncu_op_c1_*.json profiles/r02_ncu_traffic_c3p_*.json profiles/r02_ncu_op_c3p_*.json gpurun_out/final/
for w in c1 c3p; do timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/final/bench_$w.json 2> gpurun_out/final/bench_$w.err; done
for w in c1 c3p; do tail -c 300 gpurun_out/final/bench_$w.json; done
