"""Multi-GPU parity (needs >= 2 GPUs on one box; skipped otherwise): the NCCL
all-to-all micro-op pipeline against the oracle simulating all ranks."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _run(nproc, *args, port=29611):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", "mp_parity.py"), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "MP_PARITY OK" in out, out[-4000:]
    return out


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("cfg,tokens,n,extra", [
    ("C1", 256, 2, ["--experts", "4"]),
    ("C2", 512, 2, ["--check-chunks", "1", "--poison", "--graph"]),
    ("C3", 256, 3, []),
])
def test_two_ranks(cfg, tokens, n, extra):
    _run(2, "--config", cfg, "--tokens", str(tokens), "--n-chunks", str(n), *extra)


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
def test_two_ranks_interleaved_layers_shared_workspace():
    """fwd A, fwd B, bwd B, bwd A on one comm, B using A's workspace: the backward FREE is
    posted after each backward's last read of dO / dXs, so A's gradients stay exact."""
    _run(2, "--config", "C2", "--tokens", "512", "--n-chunks", "2", "--interleave", "--shared-ws", port=29613)


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
def test_two_ranks_unequal_token_counts():
    """Ranks with different num_tokens (512 and 475) and one capacity: every peer-visible
    buffer region sits at a T-independent offset, so the peer stores land right."""
    _run(2, "--config", "C2", "--tokens", "512", "--n-chunks", "2", "--ragged-ranks", "37", "--poison", port=29618)


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("cfg,tokens,extra", [
    ("C2", 512, ["--poison", "--graph"]),
    ("C3", 256, ["--interleave", "--shared-ws"]),
])
def test_two_ranks_dropless(cfg, tokens, extra):
    """§8(f) row 4: capacity 0 — count exchange, unequal-split dispatch / return by peer stores,
    expert GEMMs over virtual segments — against the oracle with C = T."""
    _run(2, "--config", cfg, "--tokens", str(tokens), "--n-chunks", "1", "--dropless", *extra, port=29614)


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("extra", [["--dropless", "--pack-exchange"], ["--poison", "--graph"]])
def test_two_ranks_packed(extra):
    """Expert packing m = 2 at 2 ranks: both ranks host all experts, each takes the rows
    of the sources with its residue (its own rows stay local), dW summed over the group; the
    packed weights built by lina_pack_weights; with and without a capacity bound."""
    _run(2, "--config", "C2", "--tokens", "512", "--n-chunks", "1", "--pack", "2", *extra, port=29616)


@pytest.mark.skipif(_ngpu() < 4, reason="needs 4 GPUs")
@pytest.mark.parametrize("pack", [2, 4])
def test_four_ranks_packed(pack):
    _run(4, "--config", "C3", "--tokens", "256", "--n-chunks", "1", "--pack", str(pack), "--dropless",
         "--pack-exchange", port=29617)


@pytest.mark.skipif(_ngpu() < 4, reason="needs 4 GPUs")
def test_four_ranks_dropless():
    _run(4, "--config", "C2", "--tokens", "384", "--n-chunks", "1", "--dropless", "--poison", "--graph", port=29615)


@pytest.mark.skipif(_ngpu() < 4, reason="needs 4 GPUs")
def test_four_ranks():
    _run(4, "--config", "C2", "--tokens", "384", "--n-chunks", "4", "--check-chunks", "1", "--poison", "--graph", port=29612)


def _run_infer(nproc, *args, port=29621):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", "mp_infer.py"), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "MP_INFER OK" in out, out[-4000:]
    return out


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
@pytest.mark.parametrize("zipf,experts", [(1.0, 8), (1.2, 32), (0.5, 32)])
def test_infer_replication_two_ranks(zipf, experts):
    _run_infer(2, "--tokens", "512", "--zipf", str(zipf), "--experts", str(experts))


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
def test_scheduler_allreduce_two_ranks():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port=29631", os.path.join(ROOT, "tests", "mp_sched.py"),
           "--config", "C3", "--tokens", "1024", "--reps", "2"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "MP_SCHED OK" in out, out[-4000:]


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
def test_infer_replicas_two_ranks():
    """Eq. (1) gives r_0 = 2 (E=8, Zipf 3: n_0 ~ 1.67): the replica token split runs."""
    _run_infer(2, "--tokens", "512", "--zipf", "3.0", "--experts", "8", "--min-replicas", "2", port=29623)


@pytest.mark.skipif(_ngpu() < 4, reason="needs 4 GPUs")
@pytest.mark.parametrize("zipf,experts,min_r", [(1.5, 32, 2), (2.0, 8, 3)])
def test_infer_replicas_four_ranks(zipf, experts, min_r):
    """r_e >= 2 at 4 ranks (E=32 Zipf 1.5: n_0 ~ 1.8; E=8 Zipf 2: n_0 ~ 2.6)."""
    _run_infer(4, "--tokens", "512", "--zipf", str(zipf), "--experts", str(experts), "--min-replicas", str(min_r),
               port=29624)


def _run_full(nproc, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tests", "mp_fullsize.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "MP_FULLSIZE OK" in out, out[-4000:]


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
def test_full_size_two_ranks_graph():
    """configs[1] at full size per rank, fused transport, CUDA-graph replays (the bench launch)."""
    _run_full(2, 29651)


@pytest.mark.skipif(_ngpu() < 4, reason="needs 4 GPUs")
def test_full_size_four_ranks_graph():
    _run_full(4, 29652)


@pytest.mark.skipif(_ngpu() < 4, reason="needs 4 GPUs")
@pytest.mark.parametrize("zipf", [1.0, 1.2])
def test_infer_replication_four_ranks(zipf):
    """S10 at 4 ranks: plan = oracle, replicated = static bitwise, fused peer-store all-to-all."""
    _run_infer(4, "--tokens", "512", "--zipf", str(zipf), "--experts", "32", port=29622)
