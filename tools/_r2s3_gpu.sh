set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s3_smoke.log 2>&1
timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=30 > gpurun_out/r2s3_gputest.log 2>&1
tail -45 gpurun_out/r2s3_gputest.log
