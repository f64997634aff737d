# tile width vs shape (plain tile GEMM, interleaved, real clocks): calibrate lowering.choose_tile_n's cost model
set -x
for shape in "4096 4096 4096" "2048 2048 2048" "8192 3584 4096" "16384 7168 8192" "8192 8192 8192" "4096 14336 4096" "16384 8192 3584"; do
  set -- $shape
  timeout 600 python tools/ab_env.py 20 $1 $2 $3 1.0 auto= w128=TILE_N:128 w160=TILE_N:160 w192=TILE_N:192 w224=TILE_N:224 w256=TILE_N:256 > gpurun_out/tn_$1x$2x$3.log 2>&1
  grep median gpurun_out/tn_$1x$2x$3.log
done
