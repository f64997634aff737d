set -x
mkdir -p gpurun_out/final
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_gemm -s 2 -c 1 -f -o gpurun_out/r2_ncu_op_c1_g4_uniform_fused_2d_dma python tools/op_once.py c1 uniform_fused_2d dma 3 4 > gpurun_out/final/ncu_op_c1_g4.log 2>&1
python tools/traffic_files.py gpurun_out > gpurun_out/final/traffic_files_c1.log 2>&1
cp profiles/r02_ncu_traffic_c1_*.json profiles/r02_ncu_op_c1_*.json gpurun_out/final/
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k c1 > gpurun_out/final/c1_test.log 2>&1
tail -2 gpurun_out/final/c1_test.log
timeout 900 python bench.py --workload c1 --steps 20 --warmup 5 > gpurun_out/final/bench_c1.json 2> gpurun_out/final/bench_c1.err
timeout 600 python bench.py --impl reference --workload c1 --steps 5 --warmup 2 > gpurun_out/final/bench_reference_arm_c1.json 2> gpurun_out/final/bench_reference_arm_c1.err
tail -c 1500 gpurun_out/final/bench_c1.json
