"""Multi-GPU parity on real B200s (NCCL): runs when the box has >= 2 GPUs."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _ngpus():
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:  # noqa: BLE001
        return 0


@pytest.mark.parametrize("world,p2p", [(2, "1"), (2, "0"), (4, "1")])
def test_golden_plans_on_n_gpus(world, p2p):
    """p2p=1: kernel reductions gathered through the NVLink peer boards; 0: NCCL all-gather."""
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29511", os.path.join(HERE, "mgpu_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=dict(os.environ, DK_P2P=p2p))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "MGPU" in r.stdout and "bad=[]" in r.stdout
    if p2p == "1":
        assert "p2p_folds=0 " not in r.stdout, r.stdout[-2000:]


@pytest.mark.parametrize("world", [2, 4])
def test_peer_protocols_under_rank_skew(world):
    """Random host delays per rank while CG cycles through the epoch-tagged peer boards and the
    copy-engine halo mailboxes; results bit-identical to the same stream on one GPU."""
    if _ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29521", os.path.join(HERE, "mgpu_stress.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "STRESS" in r.stdout and "bad=[]" in r.stdout, r.stdout[-2000:]
