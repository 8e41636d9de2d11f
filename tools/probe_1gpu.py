"""Probe: can two processes share one GPU as two lina ranks (NCCL bootstrap)?
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/probe_1gpu.py
"""
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    import paper_2210_17223_b200 as lina
    uid = [lina.lina_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    try:
        comm = lina.Comm(world, rank, 0, uid[0], 8)
        print(f"rank {rank}: lina comm on shared GPU OK", flush=True)
        comm.close() if hasattr(comm, "close") else None
    except Exception as e:  # noqa: BLE001
        print(f"rank {rank}: lina comm on shared GPU FAILED: {e}", flush=True)
    dist.barrier()


if __name__ == "__main__":
    main()
