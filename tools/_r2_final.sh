# round-2 evidence on one B200 (final code): smoke, op-kernel ncu captures -> per-shape traffic files,
# every bench workload (N=1, virtual ranks) + the reference arm, the launch list of the default command
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
mkdir -p gpurun_out/final
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1
for spec in "c1 uniform_fused_2d dma 4" "c2 hetero_unfused_1d dma 8" "c3 hetero_unfused_1d core 8" "c3 hetero_unfused_1d core 4" "c3 hetero_unfused_1d core 2" "c4 hetero_unfused_1d dma 8" "c3p hetero_unfused_1d dma 8" "ep hetero_unfused_1d dma 8"; do
  set -- $spec
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tile_gemm -s 2 -c 1 -f -o gpurun_out/r2_ncu_op_$1_g$4_$2_$3 python tools/op_once.py $1 $2 $3 3 $4 > gpurun_out/final/ncu_op_$1_g$4.log 2>&1
done
python tools/traffic_files.py gpurun_out > gpurun_out/final/traffic_files.log 2>&1
cp profiles/r02_ncu_traffic_*.json profiles/r02_ncu_op_*.json gpurun_out/final/
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final/bench_reference_arm.json 2> gpurun_out/final/bench_reference_arm.err
timeout 600 python bench.py > gpurun_out/final/bench_default.json 2> gpurun_out/final/bench_default.err
for w in c1 c2 c4 c3 c3p ep; do timeout 900 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/final/bench_$w.json 2> gpurun_out/final/bench_$w.err; done
for g in 4 2; do timeout 900 python bench.py --workload c3 --virtual-ranks $g --steps 20 --warmup 5 > gpurun_out/final/bench_c3_g$g.json 2> gpurun_out/final/bench_c3_g$g.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final/launches_c2.csv python bench.py --steps 3 --warmup 3 --headline-only --no-cpu > gpurun_out/final/launches_c2.log 2>&1
rm -f gpurun_out/r2_ncu_op_*.ncu-rep.bak
ls -la gpurun_out/final
tail -c 600 gpurun_out/final/bench_default.json
