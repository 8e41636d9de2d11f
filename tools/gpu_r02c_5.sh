# elect-issuer gate / dX / dWg kernels: parity; C5 GEMM DRAM traffic with and without half tails (tile drift check)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r02c5_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/r02c5_pytest.log
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum"
for h in 0 1; do
  LINA_HALF128=$h timeout 600 ncu --metrics $M --clock-control none -k regex:tc_gemm_kernel --launch-skip 12 -c 12 --csv --log-file gpurun_out/r02c5_C5_h$h.csv python bench.py --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu h=$h rc=$?"
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gate|dx_|dwg|permute|combine|route|split" --launch-skip 20 -c 40 --csv --log-file gpurun_out/r02c5_C5_small.csv python bench.py --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu small rc=$?"
