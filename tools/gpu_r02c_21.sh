# n = 8 micro-ops at N = 4 (C5 and C2): completes the n in {1, 2, 4, 8} sweep of SURVEY §8(d)
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29751 bench.py --gpus 4 --sweep-chunks 8 --no-cpu-baseline --no-e2e > gpurun_out/r02c21_bench_c5_n4_n8.json 2> gpurun_out/r02c21_bench_c5_n4_n8.err; echo "c5 rc=$?"
timeout 600 $TR --nproc-per-node 4 --master-port 29752 bench.py --gpus 4 --config C2 --sweep-chunks 8 --no-cpu-baseline --no-e2e > gpurun_out/r02c21_bench_c2_n4_n8.json 2> gpurun_out/r02c21_bench_c2_n4_n8.err; echo "c2 rc=$?"
