set -x
mkdir -p gpurun_out/final3
timeout 2400 python tools/stress_parity.py 2000 gpurun_out/final3/stress_parity_2000.json > gpurun_out/final3/stress_parity.log 2>&1
tail -2 gpurun_out/final3/stress_parity.log
timeout 900 compute-sanitizer --tool racecheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final3/racecheck_smoke.log 2>&1
tail -4 gpurun_out/final3/racecheck_smoke.log
timeout 1800 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_executor.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "trace or c1" > gpurun_out/final3/memcheck_exec.log 2>&1
tail -3 gpurun_out/final3/memcheck_exec.log
