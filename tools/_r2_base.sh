set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
for w in c2 c4 c3; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r2_base_$w.json 2> gpurun_out/r2_base_$w.err; done
tail -c 3000 gpurun_out/r2_base_c2.json
