set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1500 python -m pytest tests -m gpu -q -rA -x > gpurun_out/r02b_pytest_n2.log 2>&1; echo "pytest rc=$?"
tail -n 5 gpurun_out/r02b_pytest_n2.log
timeout 600 python bench.py > gpurun_out/r02b_bench_n1.json 2> gpurun_out/r02b_bench_n1.err; echo "bench1 rc=$?"
cat gpurun_out/r02b_bench_n1.json | head -c 600
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/r02b_bench_n2.json 2> gpurun_out/r02b_bench_n2.err; echo "bench2 rc=$?"
cat gpurun_out/r02b_bench_n2.json | head -c 600
