# round-2 final bench lines (code after the launch-order / host-cost changes): smoke, every workload,
# reference arms, launch list, then the GPU suite. Op-kernel ncu captures are kept from tools/_r2_final.sh
# (the tile programs did not change since).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
mkdir -p gpurun_out/final2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final2/bench_reference_arm.json 2> gpurun_out/final2/bench_reference_arm.err
timeout 600 python bench.py > gpurun_out/final2/bench_default.json 2> gpurun_out/final2/bench_default.err
for w in c1 c4 c3 c3p ep; do timeout 1200 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/final2/bench_$w.json 2> gpurun_out/final2/bench_$w.err; done
for g in 4 2; do timeout 900 python bench.py --workload c3 --virtual-ranks $g --steps 20 --warmup 5 > gpurun_out/final2/bench_c3_g$g.json 2> gpurun_out/final2/bench_c3_g$g.err; done
timeout 600 python bench.py --impl reference --workload c1 --steps 5 --warmup 2 > gpurun_out/final2/bench_c1_reference_arm.json 2> gpurun_out/final2/bench_c1_reference_arm.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final2/launches_c2.csv python bench.py --steps 3 --warmup 3 --headline-only --no-cpu > gpurun_out/final2/launches_c2.log 2>&1
timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/final2/gputest.log 2>&1
tail -2 gpurun_out/final2/gputest.log
ls -la gpurun_out/final2
