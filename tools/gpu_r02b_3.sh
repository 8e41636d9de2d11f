# persistent dX / one-wave dWg / 2-stage gate: parity, C5 + C2 benches and launch lists;
# tail split and split dispatch A/B at C2/C3 (2 GPUs)
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_infer.py -q -rA -x > gpurun_out/r02b3_pytest.log 2>&1; echo "pytest rc=$?"
tail -n 3 gpurun_out/r02b3_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02b3_c5_n1.json 2> gpurun_out/r02b3_c5_n1.err; echo "c5 rc=$?"
for t in 1 0; do
  LINA_TAIL128=$t timeout 300 python bench.py --config C2 --no-cpu-baseline --no-e2e > gpurun_out/r02b3_c2_n1_tail$t.json 2>/dev/null; echo "c2 tail=$t rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b3_launches_c5_n1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02b3_ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02b3_launches_c2_n1.csv python bench.py --config C2 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02b3_ncu_c2.log 2>&1; echo "ncu c2 rc=$?"
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --no-cpu-baseline --no-e2e"
for cfg in C2 C3; do
  for sp in 1 0; do
    for t in 1 0; do
      LINA_TAIL128=$t LINA_SPLIT_DISPATCH=$sp timeout 400 $TR --config $cfg > gpurun_out/r02b3_${cfg}_n2_sp${sp}_t${t}.json 2>/dev/null; echo "$cfg split=$sp tail=$t rc=$?"
    done
  done
done
