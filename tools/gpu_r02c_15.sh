# Gate: L2 prefetch of 512-byte row segments; TB = 2 vs 1 (LINA_GATE_TB=1); parity of the gate paths
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gate or c5 or c4 or dropless" > gpurun_out/r02c15_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/r02c15_pytest.log
for tb in 2 1; do
LINA_GATE_TB=$tb timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gate_tc" --launch-skip 2 -c 3 --csv --log-file gpurun_out/r02c15_gate_tb$tb.csv python bench.py --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo "ncu tb=$tb rc=$?"
done
