# GEMM epilogue geometry A/B (1 GPU): per-launch time, SM clock and tensor-pipe activity of the
# 6 expert GEMMs of one eager step, C5 and C2; plus parity of the variants
set -x
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
for cfg in C5 C2; do
  for v in "1 0" "2 0" "1 2" "2 2"; do
    set -- $v
    LINA_GEMM_WIDE=$1 LINA_WGRAD_WIDE=$2 timeout 600 ncu --metrics $M --clock-control none -k regex:tc_gemm_kernel --launch-skip 12 -c 12 --csv --log-file gpurun_out/r02b7_${cfg}_w$1_g$2.csv python bench.py --config $cfg --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "$cfg $v rc=$?"
  done
done
LINA_GEMM_WIDE=2 LINA_WGRAD_WIDE=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c5_shapes or c2_full or c2_reduced or chunk_invariance_bf16 or dropless_c5" > gpurun_out/r02b7_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/r02b7_pytest.log
for v in "1 0" "2 2"; do
  set -- $v
  LINA_GEMM_WIDE=$1 LINA_WGRAD_WIDE=$2 timeout 300 python bench.py --config C2 --no-cpu-baseline --no-e2e > gpurun_out/r02b7_bench_c2_w$1_g$2.json 2>/dev/null; echo "bench c2 $v rc=$?"
  LINA_GEMM_WIDE=$1 LINA_WGRAD_WIDE=$2 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02b7_bench_c5_w$1_g$2.json 2>/dev/null; echo "bench c5 $v rc=$?"
done
