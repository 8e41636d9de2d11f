# Dynamic-schedule overhead: queue hand-off with the static order (LINA_GEMM_DYN=3) vs static (0) vs dynamic everywhere (2), C5 / C2 per-GEMM cycles
set -x
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum"
for c in C2 C5; do
for dy in 3 2 0; do
  LINA_GEMM_DYN=$dy timeout 600 ncu --metrics $M --clock-control none -k regex:tc_gemm_kernel --launch-skip 12 -c 12 --csv --log-file gpurun_out/r02c11_${c}_d$dy.csv python bench.py --config $c --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu $c d=$dy rc=$?"
done
done
