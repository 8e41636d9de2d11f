# 4 GPUs, final build: benches at N = 4 and 2 (clock sampler started before the timed region), C5 and C2; the multi-rank GPU tests
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29711 bench.py --gpus 4 > gpurun_out/r02c14_bench_c5_n4.json 2> gpurun_out/r02c14_bench_c5_n4.err; echo "c5 n4 rc=$?"
timeout 600 $TR --nproc-per-node 4 --master-port 29712 bench.py --gpus 4 --config C2 > gpurun_out/r02c14_bench_c2_n4.json 2> gpurun_out/r02c14_bench_c2_n4.err; echo "c2 n4 rc=$?"
timeout 900 $TR --nproc-per-node 2 --master-port 29713 bench.py --gpus 2 > gpurun_out/r02c14_bench_c5_n2.json 2> gpurun_out/r02c14_bench_c5_n2.err; echo "c5 n2 rc=$?"
timeout 600 $TR --nproc-per-node 2 --master-port 29714 bench.py --gpus 2 --config C2 > gpurun_out/r02c14_bench_c2_n2.json 2> gpurun_out/r02c14_bench_c2_n2.err; echo "c2 n2 rc=$?"
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -rs > gpurun_out/r02c14_pytest_multirank_n4.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/r02c14_pytest_multirank_n4.log
