# e2e at N = 1 (C5) with 2 copy streams per direction vs 1
set -x
for cs in 2 1; do timeout 600 python bench.py --copy-streams $cs --no-cpu-baseline > gpurun_out/r02c24_bench_c5_n1_cs$cs.json 2>/dev/null; echo "cs$cs rc=$?"; done
