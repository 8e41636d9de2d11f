# Tile-queue hand-off by st.async + relaxed remote arrives (no MEMBAR.ALL.GPU per tile): parity with the dynamic schedule on every GEMM; A/B per-GEMM cycles
set -x
LINA_GEMM_DYN=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shared.py -q -x > gpurun_out/r02c12_pytest_dyn2.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/r02c12_pytest_dyn2.log
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum"
for c in C2 C5; do
for dy in 2 0 1; do
  LINA_GEMM_DYN=$dy timeout 600 ncu --metrics $M --clock-control none -k regex:tc_gemm_kernel --launch-skip 12 -c 12 --csv --log-file gpurun_out/r02c12_${c}_d$dy.csv python bench.py --config $c --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu $c d=$dy rc=$?"
done
done
for dy in 2 1; do LINA_GEMM_DYN=$dy timeout 300 python bench.py --config C2 --no-cpu-baseline --no-e2e > gpurun_out/r02c12_bench_c2_d$dy.json 2>/dev/null; echo "c2 d=$dy rc=$?"; done
for dy in 2 1; do LINA_GEMM_DYN=$dy timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02c12_bench_c5_d$dy.json 2>/dev/null; echo "c5 d=$dy rc=$?"; done
