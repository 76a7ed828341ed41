"""Launch tests/mgpu_check.py with torchrun on 2 (and 4, 8) GPUs of this box."""

import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 4, 8])
def test_multi_gpu_engine_parity(world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs, have {torch.cuda.device_count()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "tests", "mgpu_check.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-4000:]
    assert f"MGPU OK world={world}" in res.stdout


def test_multi_gpu_push_staging_parity():
    """The optional push staging of the exact correction (CDSGD_STAGE_PUSH=1: K2 stores each
    element into its owner's receive row, the reduce reads locally) at N=2."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "tests", "mgpu_check.py"), "p2p-exact"]
    env = dict(os.environ, CDSGD_STAGE_PUSH="1")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-4000:]
    assert "MGPU OK world=2" in res.stdout


@pytest.mark.parametrize("world", [2, 4])
def test_multi_gpu_copy_engine_correction_parity(world):
    """The p2p exchange with the copy-engine share of the correction all-reduce forced on
    (by default it starts at 8M elements, above these test layouts)."""
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "tests", "mgpu_check.py"), "p2p"]
    env = dict(os.environ, CDSGD_CE_FRAC="0.5")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-4000:]
    assert f"MGPU OK world={world}" in res.stdout
