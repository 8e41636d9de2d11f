# Dynamic GEMM tile schedule (LINA_GEMM_DYN, default on): parity, A/B benches, per-GEMM cycles and DRAM bytes
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shared.py tests/test_gpu_infer.py -q -x > gpurun_out/r02c6_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/r02c6_pytest.log
for i in 1 2; do
  for dy in 1 0; do
    LINA_GEMM_DYN=$dy timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02c6_bench_c5_d$dy.$i.json 2>/dev/null; echo "c5 d=$dy rc=$?"
  done
done
for dy in 1 0; do LINA_GEMM_DYN=$dy timeout 300 python bench.py --config C2 --no-cpu-baseline --no-e2e > gpurun_out/r02c6_bench_c2_d$dy.json 2>/dev/null; echo "c2 d=$dy rc=$?"; done
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum"
for dy in 1 0; do
  LINA_GEMM_DYN=$dy timeout 600 ncu --metrics $M --clock-control none -k regex:tc_gemm_kernel --launch-skip 12 -c 12 --csv --log-file gpurun_out/r02c6_C5_d$dy.csv python bench.py --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu d=$dy rc=$?"
done
