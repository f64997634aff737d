set -x
timeout 2700 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > gpurun_out/final/gputest.log 2>&1
tail -20 gpurun_out/final/gputest.log
bash tools/_r2_final.sh
