for nc in 1 2 4; do
  for tr in fused nccl; do
    LINA_TRANSPORT=$tr python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2952$nc bench.py --gpus 2 --steps 20 --warmup 5 --n-chunks $nc > gpurun_out/sweep_n2_${tr}_c${nc}.log 2>&1
    echo "$tr c=$nc $(tail -1 gpurun_out/sweep_n2_${tr}_c${nc}.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,2), round(d["ms_per_step"],4), d["a2a"]["exposed_ms_per_step"] if d.get("a2a") else None)')"
  done
done
