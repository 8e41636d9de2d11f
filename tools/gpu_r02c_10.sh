# Round-2 default build at 1 GPU: GPU suite, smoke, default bench (C5) + C2, per-GEMM cycles, launch list, ncu --set full of the C5 GEMMs
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1200 python -m pytest tests -m gpu -q -rs > gpurun_out/r02c10_pytest_gpu_n1.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/r02c10_pytest_gpu_n1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c10_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02c10_bench_c5_n1.json 2> gpurun_out/r02c10_bench_c5_n1.err; echo "bench rc=$?"
timeout 300 python bench.py --config C2 > gpurun_out/r02c10_bench_c2_n1.json 2> gpurun_out/r02c10_bench_c2_n1.err; echo "bench c2 rc=$?"
M="gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 600 ncu --metrics $M --clock-control none -k regex:tc_gemm_kernel --launch-skip 12 -c 12 --csv --log-file gpurun_out/r02c10_C5_gemm.csv python bench.py --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu gemm rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c10_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_gemm_kernel --launch-skip 12 -c 6 -o gpurun_out/r02c10_gemm_c5_full python bench.py --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu full rc=$?"
