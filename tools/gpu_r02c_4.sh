# Warp-converged MMA issuer / TMA producer (elect.sync, uniform descriptors): parity, benches, per-GEMM cycles
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shared.py -q -x > gpurun_out/r02c4_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/r02c4_pytest.log
for i in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02c4_bench_c5.$i.json 2>/dev/null; echo "c5 rc=$?"
  timeout 300 python bench.py --config C2 --no-cpu-baseline --no-e2e > gpurun_out/r02c4_bench_c2.$i.json 2>/dev/null; echo "c2 rc=$?"
done
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum"
for c in C5 C2; do
  timeout 600 ncu --metrics $M --clock-control none -k regex:tc_gemm_kernel --launch-skip 12 -c 12 --csv --log-file gpurun_out/r02c4_$c.csv python bench.py --config $c --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu $c rc=$?"
done
