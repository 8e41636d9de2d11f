# Reference arm (oracle) at C5 on the box: per-step time (wall clock around the whole run)
set -x
free -g | head -2; nproc
t0=$(date +%s); timeout 1500 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r02c17_ref.json 2> gpurun_out/r02c17_ref.err; echo "ref rc=$? wall=$(( $(date +%s) - t0 ))s"
