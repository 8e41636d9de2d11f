# full GPU suite at 2 GPUs; S9 multi-layer ablation; C3 n x partition sweep; C4 replication skews; chunk sweeps
set -x
timeout 1500 python -m pytest tests -m gpu -q -rA -x > gpurun_out/r02b4_pytest.log 2>&1; echo "pytest rc=$?"
tail -n 3 gpurun_out/r02b4_pytest.log
TRN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $TRN --master-port 29521 tools/bench_sched_layers.py --layers 4 --grads 2 --reps 8 > gpurun_out/r02b4_sched_layers_n2.json 2> gpurun_out/r02b4_sched_layers_n2.err; echo "sched_layers rc=$?"
timeout 900 $TRN --master-port 29522 tools/bench_c3.py --chunks 1,2,4,8,16 --partitions 1,4,16,30 --reps 6 > gpurun_out/r02b4_c3_sweep_n2.jsonl 2> gpurun_out/r02b4_c3_sweep_n2.err; echo "c3 sweep rc=$?"
timeout 600 $TRN --master-port 29523 tools/bench_c4.py --zipf 0,1.2,2.0,3.0 --iters 30 > gpurun_out/r02b4_c4_n2.jsonl 2> gpurun_out/r02b4_c4_n2.err; echo "c4 rc=$?"
timeout 900 $TRN --master-port 29524 bench.py --gpus 2 --config C2 --no-cpu-baseline --no-e2e --sweep-chunks 1,2,4,8 > gpurun_out/r02b4_c2_n2_sweep.json 2> gpurun_out/r02b4_c2_n2_sweep.err; echo "c2 sweep rc=$?"
timeout 1200 $TRN --master-port 29525 bench.py --gpus 2 --no-cpu-baseline --no-e2e --sweep-chunks 1,2,4 > gpurun_out/r02b4_c5_n2_sweep.json 2> gpurun_out/r02b4_c5_n2_sweep.err; echo "c5 sweep rc=$?"
