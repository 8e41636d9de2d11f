# Final build: ncu launch list of the C5 step and ncu --set full of its 6 expert GEMMs (traffic for bench.py's roofline)
set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02c25_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_gemm_kernel --launch-skip 12 -c 6 -o gpurun_out/r02c25_gemm_c5_full python bench.py --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu full rc=$?"
