# Half tails (M = 128 cta_group::2 last tiles) + per-GEMM epilogue width: parity, A/B benches, ncu --set full of the C5 GEMMs
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rs > gpurun_out/r02c2_pytest_parity.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/r02c2_pytest_parity.log
for i in 1 2; do
  for h in 1 0; do
    LINA_HALF128=$h timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02c2_bench_c5_h$h.$i.json 2>/dev/null; echo "c5 h=$h rc=$?"
    LINA_HALF128=$h timeout 300 python bench.py --config C2 --no-cpu-baseline --no-e2e > gpurun_out/r02c2_bench_c2_h$h.$i.json 2>/dev/null; echo "c2 h=$h rc=$?"
  done
done
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum"
for h in 1 0; do
  LINA_HALF128=$h timeout 600 ncu --metrics $M --clock-control none -k regex:tc_gemm_kernel --launch-skip 12 -c 12 --csv --log-file gpurun_out/r02c2_C5_h$h.csv python bench.py --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu C5 h=$h rc=$?"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_gemm_kernel --launch-skip 12 -c 6 -o gpurun_out/r02c2_gemm_c5_full python bench.py --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02c2_ncu_full.log 2>&1; echo "ncu full rc=$?"
ls -la gpurun_out/
