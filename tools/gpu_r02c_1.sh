# Round-2 re-entry check (1 GPU): GPU suite, smoke, default bench, GEMM epilogue geometry A/B at C5 / C2
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1200 python -m pytest tests -m gpu -q -rs > gpurun_out/r02c1_pytest_gpu_n1.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/r02c1_pytest_gpu_n1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c1_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02c1_bench_c5_n1.json 2> gpurun_out/r02c1_bench_c5_n1.err; echo "bench rc=$?"
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum"
for cfg in C5 C2; do
  for v in "1 0" "2 0" "0 0" "1 2"; do
    set -- $v
    LINA_GEMM_WIDE=$1 LINA_WGRAD_WIDE=$2 timeout 600 ncu --metrics $M --clock-control none -k regex:tc_gemm_kernel --launch-skip 12 -c 12 --csv --log-file gpurun_out/r02c1_${cfg}_w$1_g$2.csv python bench.py --config $cfg --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "$cfg $v rc=$?"
  done
done
