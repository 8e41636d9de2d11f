# C3 at 4 GPUs: micro-op count n x allreduce partition sweep under BASELINE / LINA / NAIVE / DEFER
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 1200 $TR --nproc-per-node 4 --master-port 29741 tools/bench_c3.py --chunks 1,2,4,8,16 --partitions 1,4,16,30 --reps 6 > gpurun_out/r02c20_c3_sweep_n4.jsonl 2> gpurun_out/r02c20_c3_sweep_n4.err; echo "c3 sweep n4 rc=$?"
