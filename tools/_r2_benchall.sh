# every bench workload, N=1 (virtual ranks), plus the reference arm; lines into gpurun_out/r2_bench_<w>.json
set -x
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2_bench_reference_arm.json 2> gpurun_out/r2_bench_reference_arm.err
for w in c2 c4 c3 c3p ep; do timeout 600 python bench.py --workload $w --steps 20 --warmup 5 > gpurun_out/r2_bench_$w.json 2> gpurun_out/r2_bench_$w.err; done
timeout 600 python bench.py --workload c3 --virtual-ranks 4 --steps 20 --warmup 5 > gpurun_out/r2_bench_c3_g4.json 2> gpurun_out/r2_bench_c3_g4.err
timeout 600 python bench.py --workload c3 --virtual-ranks 2 --steps 20 --warmup 5 > gpurun_out/r2_bench_c3_g2.json 2> gpurun_out/r2_bench_c3_g2.err
