# Final 1-GPU check of the round-2 build: GPU suite, smoke, default bench (C5) and C2, ncu --set full of the C5 gate launch
set -x
timeout 1200 python -m pytest tests -m gpu -q -rs > gpurun_out/r02c16_pytest_gpu_n1.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/r02c16_pytest_gpu_n1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c16_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/r02c16_bench_c5_n1.json 2> gpurun_out/r02c16_bench_c5_n1.err; echo "bench rc=$?"
timeout 300 python bench.py --config C2 > gpurun_out/r02c16_bench_c2_n1.json 2> gpurun_out/r02c16_bench_c2_n1.err; echo "bench c2 rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gate_tc --launch-skip 2 -c 1 -o gpurun_out/r02c16_gate_c5_full python bench.py --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu gate rc=$?"
