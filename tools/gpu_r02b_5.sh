# dX pipelining parity + C5 N=1 launch list; scheduler window A/B (2 GPUs)
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rA -x -k "gate_backward or c5 or c2_full" > gpurun_out/r02b5_pytest.log 2>&1; echo "pytest rc=$?"
tail -n 3 gpurun_out/r02b5_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02b5_c5_n1.json 2> gpurun_out/r02b5_c5_n1.err; echo "c5 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b5_launches_c5_n1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02b5_ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
TRN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
for w in full dispatch; do
  LINA_SCHED_WINDOW=$w timeout 600 $TRN --master-port 29531 tools/bench_sched_layers.py --layers 4 --grads 2 --reps 8 > gpurun_out/r02b5_sched_layers_n2_$w.json 2>/dev/null; echo "sched_layers $w rc=$?"
  LINA_SCHED_WINDOW=$w timeout 600 $TRN --master-port 29532 tools/bench_c3.py --chunks 1 --partitions 4,30 --reps 8 > gpurun_out/r02b5_c3_n2_$w.jsonl 2>/dev/null; echo "c3 $w rc=$?"
done
