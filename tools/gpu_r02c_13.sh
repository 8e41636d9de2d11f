# Gate with two token blocks per CTA at large T (gate_tc.cu TB = 2): parity (incl. full-token C5 routing), small-kernel ncu, C5 bench
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r02c13_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/r02c13_pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gate|dx_|dwg|permute|combine|route|split" --launch-skip 20 -c 40 --csv --log-file gpurun_out/r02c13_C5_small.csv python bench.py --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu small rc=$?"
for i in 1 2; do timeout 900 python bench.py > gpurun_out/r02c13_bench_c5.$i.json 2>/dev/null; echo "c5 rc=$?"; done
