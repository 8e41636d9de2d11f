# device-timeline scheduler: parity + S9 ablations (2 GPUs); C5 GEMM ncu --set full capture (GPU 0)
set -x
timeout 900 python -m pytest tests/test_gpu_multirank.py -q -rA -x -k "sched" > gpurun_out/r02b6_pytest.log 2>&1; echo "pytest rc=$?"
tail -n 3 gpurun_out/r02b6_pytest.log
TRN="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $TRN --master-port 29541 tools/bench_sched_layers.py --layers 4 --grads 2 --reps 8 > gpurun_out/r02b6_sched_layers_n2.json 2>/dev/null; echo "sched_layers rc=$?"
timeout 600 $TRN --master-port 29542 tools/bench_sched_layers.py --layers 4 --grads 2 --reps 8 --partition-mb 4 > gpurun_out/r02b6_sched_layers_n2_p4.json 2>/dev/null; echo "sched_layers p4 rc=$?"
timeout 600 $TRN --master-port 29543 tools/bench_c3.py --chunks 1,4 --partitions 4,16,30 --reps 8 > gpurun_out/r02b6_c3_n2.jsonl 2>/dev/null; echo "c3 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm_kernel --launch-skip 12 -c 6 -o gpurun_out/r02_ncu_gemm_c5 python bench.py --eager --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02b6_ncu_full.log 2>&1; echo "ncu full rc=$?"
