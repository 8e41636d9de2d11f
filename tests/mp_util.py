"""Process setup shared by the multi-rank scripts (tests/mp_*.py): one rank per GPU over
NCCL (lina_comm_init), or --shared-gpu: every rank on GPU 0 with a host-bootstrap
communicator (lina_comm_init_host) whose exchanges go over a torch gloo group — NCCL
refuses two ranks on one GPU, the fused transport does not need it."""
import os

import torch
import torch.distributed as dist


def setup(shared_gpu: bool, nccl_max_ctas: int = 0):
    """Returns (world, rank, device, comm, flag_device)."""
    world, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    import paper_2210_17223_b200 as lina
    if shared_gpu:
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        dist.init_process_group("gloo")

        def allgather(data: bytes):
            out = [None] * world
            dist.all_gather_object(out, data)
            return out

        return world, rank, dev, lina.lina.Comm.host(world, rank, 0, allgather), "cpu"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    uid = [lina.lina_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    return world, rank, dev, lina.Comm(world, rank, local, uid[0], nccl_max_ctas), dev
