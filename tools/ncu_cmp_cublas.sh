# Tile kernel vs cuBLAS on plain GEMM shapes at base clocks (ncu), one CSV per (impl, shape).
# usage (GPU box, repo root): bash tools/ncu_cmp_cublas.sh "M N K" ...
MET=gpu__time_duration.sum,gpc__cycles_elapsed.max,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active,lts__t_bytes.sum,dram__bytes_read.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed
for shape in "$@"; do
  tag=$(echo $shape | tr ' ' x)
  ncu --metrics $MET --clock-control base -k regex:tile_gemm -s 1 -c 2 --csv python tools/kernel_once.py $shape > gpurun_out/ncu_ours_$tag.csv 2>/dev/null
  ncu --metrics $MET --clock-control base -k 'regex:nvjet|gemm|sm100|cutlass' -s 1 -c 2 --csv python tools/cublas_once.py $shape > gpurun_out/ncu_cublas_$tag.csv 2>/dev/null
done
