# S9 at 4 GPUs: the multi-layer backward under NONE / BASELINE / LINA / NAIVE / DEFER (tools/bench_sched_layers.py, C3 shape, 4 layers)
set -x
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $TR --nproc-per-node 4 --master-port 29721 tools/bench_sched_layers.py > gpurun_out/r02c18_sched_layers_n4.json 2> gpurun_out/r02c18_sched_layers_n4.err; echo "sched n4 rc=$?"
timeout 900 $TR --nproc-per-node 4 --master-port 29722 tools/bench_sched_layers.py --partition-mb 4 > gpurun_out/r02c18_sched_layers_n4_p4.json 2> gpurun_out/r02c18_sched_layers_n4_p4.err; echo "sched n4 p4 rc=$?"
