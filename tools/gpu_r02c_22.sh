# The driver's round-end commands at N = 1: the reference arm first, then the GPU arm (K = 20, W = 5)
set -x
t0=$(date +%s); timeout 1700 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02c22_ref.json 2> gpurun_out/r02c22_ref.err; echo "ref rc=$? wall=$(( $(date +%s) - t0 ))s"
t0=$(date +%s); timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r02c22_bench.json 2> gpurun_out/r02c22_bench.err; echo "bench rc=$? wall=$(( $(date +%s) - t0 ))s"
