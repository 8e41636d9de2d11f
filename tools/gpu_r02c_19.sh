# S10 at 4 GPUs with skews that replicate (Zipf 1.5 / 2.0 / 3.0 over E = 32): static vs Eq. (1) + FFD placement
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29731 tools/bench_c4.py --zipf 0,1.2,1.5,2.0,3.0 --iters 50 > gpurun_out/r02c19_c4_infer_n4.jsonl 2> gpurun_out/r02c19_c4_infer_n4.err; echo "c4 n4 rc=$?"
