# final-code quality evidence: full-size back-to-back stress with a bit-exact check of every call; sanitizers
set -x
mkdir -p gpurun_out/final
timeout 1800 python tools/stress_parity.py 500 gpurun_out/final/stress_parity.json > gpurun_out/final/stress_parity.log 2>&1
tail -3 gpurun_out/final/stress_parity.log
timeout 900 compute-sanitizer --tool memcheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/memcheck_smoke.log 2>&1
tail -3 gpurun_out/final/memcheck_smoke.log
timeout 1800 compute-sanitizer --tool memcheck python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "ragged or core_agent or cp_qk or a2a or rs_virtual or kv_slot or input_slot or mixed" > gpurun_out/final/memcheck_tests.log 2>&1
tail -3 gpurun_out/final/memcheck_tests.log
timeout 900 compute-sanitizer --tool synccheck python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/synccheck_smoke.log 2>&1
tail -3 gpurun_out/final/synccheck_smoke.log
