"""Multi-rank data path on ONE GPU: two processes share GPU 0 through a host-bootstrap
communicator (lina_comm_init_host: bootstrap over a gloo group, no NCCL — NCCL refuses two
ranks on one device).  The fused all-to-alls (NVLink peer stores + in-kernel flags; here
the peer is the same GPU, reached through CUDA IPC), the dropless count exchange and the
inference replica routing with r_e >= 2 then run against the oracle on a single-GPU box.
The ranks' kernels time-slice, so these are correctness runs, not timings."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _run(script, token, *args, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", script),
           "--shared-gpu", *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and token in out, out[-4000:]
    return out


@pytest.mark.skipif(_ngpu() < 1, reason="needs a GPU")
@pytest.mark.parametrize("extra", [["--n-chunks", "2", "--check-chunks", "1", "--poison"],
                                   ["--n-chunks", "1", "--dropless", "--poison"],
                                   ["--n-chunks", "1", "--interleave", "--shared-ws"],
                                   ["--n-chunks", "2", "--ragged-ranks", "37"]])
def test_two_ranks_one_gpu_training(extra):
    """S3-S8 with the fused dispatch / combine all-to-alls (and the dropless layout) at world 2."""
    _run("mp_parity.py", "MP_PARITY OK", "--config", "C2", "--tokens", "256", *extra, port=29681)


@pytest.mark.skipif(_ngpu() < 1, reason="needs a GPU")
def test_two_ranks_one_gpu_replicated_inference():
    """S10 with r_0 = 2 (E = 8, Zipf 3): replica token split, unequal peer-store all-to-all,
    received rows = the oracle's route counts, output bitwise equal to the static placement."""
    _run("mp_infer.py", "MP_INFER OK", "--tokens", "512", "--zipf", "3.0", "--experts", "8", "--min-replicas", "2",
         port=29682)
