# split dispatch: multi-rank parity + C5/C2 benches with the split on / off (2 GPUs)
set -x
timeout 900 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_shared.py -q -rA -x > gpurun_out/r02b_split_pytest.log 2>&1; echo "pytest rc=$?"
tail -n 4 gpurun_out/r02b_split_pytest.log
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --no-cpu-baseline --no-e2e"
for cfg in C5 C2; do
  for sp in 1 0; do
    LINA_SPLIT_DISPATCH=$sp timeout 600 $TR --config $cfg > gpurun_out/r02b_split_${cfg}_${sp}.json 2> gpurun_out/r02b_split_${cfg}_${sp}.err; echo "$cfg split=$sp rc=$?"
  done
done
for n in 74 296; do
  LINA_DISPATCH_CTAS=$n timeout 600 $TR --config C5 > gpurun_out/r02b_split_C5_ctas$n.json 2> gpurun_out/r02b_split_C5_ctas$n.err; echo "ctas=$n rc=$?"
done
