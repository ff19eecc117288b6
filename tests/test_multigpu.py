"""NCCL over NVLink parity (needs >= 2 GPUs; run via `gpurun --gpus 2|4`):
launches tests/dist_worker.py under torchrun."""
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
HERE = os.path.dirname(os.path.abspath(__file__))


def _nproc():
    import torch

    return min(torch.cuda.device_count(), int(os.environ.get("DEAR_TEST_NPROC", "4")))


@pytest.mark.parametrize("case", ["runtime", "peer", "push", "push_mismatch", "distoptim", "nvls",
                                  "distoptim_nvls"])
def test_nccl_parity(case):
    n = _nproc()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + (os.getpid() % 1000)),
           os.path.join(HERE, "dist_worker.py"), case]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    print(out.stdout[-4000:])
    assert out.returncode == 0, out.stdout[-4000:] + out.stderr[-4000:]


def test_peer_timeout_traps():
    """A rank that never reports its gradients: the other rank's peer kernel
    traps after DEAR_PEER_TIMEOUT_S instead of hanging (dist_worker "timeout")."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(31500 + (os.getpid() % 1000)),
           os.path.join(HERE, "dist_worker.py"), "timeout"]
    env = dict(os.environ, DEAR_PEER_TIMEOUT_S="3")
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env)
    print(out.stdout[-4000:])
    assert "trapped after" in out.stdout, out.stdout[-4000:] + out.stderr[-4000:]
