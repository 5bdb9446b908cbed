"""Multi-GPU parity: torchrun over 2 (or more) B200 with the NCCL
transposition; every rank compares its local slice with the 1-rank oracle."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = Path(__file__).resolve().parents[1]


def _ngpu():
    import torch

    return torch.cuda.device_count()


@pytest.mark.parametrize("nproc", [2, 4])
def test_torchrun_parity(nproc):
    if _ngpu() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={29600 + nproc}", str(ROOT / "tools" / "mp_check.py"),
           "79", "6", "319", "5", "639", "4"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    sys.stdout.write(res.stdout[-4000:])
    sys.stderr.write(res.stderr[-4000:])
    assert res.returncode == 0
    assert "MP_OK" in res.stdout
