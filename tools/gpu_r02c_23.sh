# e2e at N = 4 (C5): host <-> device copies split over 2 copy streams per direction (bench.py --copy-streams)
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29761 bench.py --gpus 4 --copy-streams 2 --no-cpu-baseline > gpurun_out/r02c23_bench_c5_n4_cs2.json 2> gpurun_out/r02c23_bench_c5_n4_cs2.err; echo "cs2 rc=$?"
