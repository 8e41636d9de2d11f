# 4 GPUs, round-2 default build: multi-rank GPU suite (+ the 2-rank cases with the dynamic schedule on every GEMM),
# C5 / C2 benches at N = 4 with the micro-op sweep (H(n), pipelining efficiency), C5 at N = 2 and 4
set -x
nvidia-smi --query-gpu=index,name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests/test_gpu_multirank.py -q -rs > gpurun_out/r02c3_pytest_multirank_n4.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/r02c3_pytest_multirank_n4.log
LINA_GEMM_DYN=2 timeout 900 python -m pytest tests/test_gpu_multirank.py -q -k "two_ranks" > gpurun_out/r02c3_pytest_multirank_dyn2.log 2>&1; echo "pytest dyn2 rc=$?"; tail -n 2 gpurun_out/r02c3_pytest_multirank_dyn2.log
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29701 bench.py --gpus 4 --sweep-chunks 1,2,4 --no-cpu-baseline > gpurun_out/r02c3_bench_c5_n4_sweep.json 2> gpurun_out/r02c3_bench_c5_n4_sweep.err; echo "c5 n4 sweep rc=$?"
timeout 600 $TR --nproc-per-node 4 --master-port 29702 bench.py --gpus 4 --config C2 --sweep-chunks 1,2,4 --no-cpu-baseline > gpurun_out/r02c3_bench_c2_n4_sweep.json 2> gpurun_out/r02c3_bench_c2_n4_sweep.err; echo "c2 n4 sweep rc=$?"
timeout 900 $TR --nproc-per-node 2 --master-port 29704 bench.py --gpus 2 > gpurun_out/r02c3_bench_c5_n2.json 2> gpurun_out/r02c3_bench_c5_n2.err; echo "c5 n2 rc=$?"
