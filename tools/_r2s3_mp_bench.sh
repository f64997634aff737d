# N>1 bench plumbing on one GPU (gloo, every rank on cuda:0): not a measurement, a does-it-run check
set -x
for w in c2 c3 c4 ep; do
  FICCO_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload $w --steps 3 --warmup 3 --no-cpu > gpurun_out/mp_bench_$w.json 2> gpurun_out/mp_bench_$w.err
  echo "exit $w $?"; tail -c 400 gpurun_out/mp_bench_$w.json; tail -3 gpurun_out/mp_bench_$w.err
done
FICCO_BENCH_SHARED_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/mp_bench_ref.json 2> gpurun_out/mp_bench_ref.err
echo "exit ref $?"; tail -c 300 gpurun_out/mp_bench_ref.json
