# dX by bulk-copy row gather (dx_gather_kernel): parity of the gate backward / full layer; small-kernel DRAM rates at C5 and C2
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_shared.py -q -x > gpurun_out/r02c8_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/r02c8_pytest.log
for c in C5 C2; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gate|dx_|dwg|permute|combine|route|split" --launch-skip 20 -c 40 --csv --log-file gpurun_out/r02c8_${c}_small.csv python bench.py --config $c --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu small $c rc=$?"
done
for i in 1 2; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02c8_bench_c5.$i.json 2>/dev/null; echo "c5 rc=$?"
done
