"""Multi-GPU parity and failure handling: torchrun over 2 / 4 B200.

* parity: every rank compares its local slice of K >= 4 back-to-back
  inverse + direct pairs (distinct inputs, no host sync in between) with the
  1-rank oracle (tools/mp_check.py), for both transports of the
  grid <-> spectral transposition -- p2p (kernels store into the peers'
  buffers over NVLink, flag handshakes) and NCCL grouped send/recv in the
  reference's rotated order (collectives.py:85-86) -- and for the recompute
  Legendre mode, and for both Fourier-row layouts (classic, field-blocked);
* failure: one rank dies after plan creation; the survivors must raise
  ProtocolError from their bounded wait instead of hanging
  (tools/mp_fail_check.py; the reference's first-error abort,
  halo/router.py:124-126, 199-205).
"""

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


def _torchrun(nproc, script, args, env_extra, port, timeout=900):
    env = dict(os.environ, **env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "tools" / script), *args]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)
    sys.stdout.write(res.stdout[-4000:])
    sys.stderr.write(res.stderr[-4000:])
    return res


@pytest.mark.parametrize("nproc,transport,recompute,layout", [
    (2, "p2p", 0, ""), (2, "nccl", 0, ""), (2, "p2p", 1, ""), (4, "p2p", 0, ""), (4, "nccl", 0, ""),
    # field-blocked Fourier rows (chosen automatically past the remote-store cliff, sht_internal.h)
    (2, "p2p", 0, "blocked"), (4, "p2p", 0, "blocked"), (4, "p2p", 1, "blocked")])
def test_torchrun_parity(nproc, transport, recompute, layout):
    if _ngpu() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    port = 29600 + 10 * nproc + (transport == "nccl") + 2 * recompute + 4 * (layout == "blocked")
    env = {"SHT_TRANSPORT": transport, "SHT_RECOMPUTE": str(recompute), "MP_PAIRS": "4"}
    if layout:
        env["SHT_ROW_LAYOUT"] = layout
    res = _torchrun(nproc, "mp_check.py", ["79", "6", "319", "70", "639", "4"], env, port)
    assert res.returncode == 0
    assert "MP_OK" in res.stdout


@pytest.mark.parametrize("nproc,gp", [(2, "2,1"), (2, "1,2"), (4, "2,2")])
def test_torchrun_parity_gridpoint_layout(nproc, gp):
    """2-D grid-point layout (latitude bands x longitude segments) with the ring <-> grid-point
    transposition: every rank's grid-point slice of inv_trans, and dir_trans from grid-point
    slices, vs the oracle."""
    if _ngpu() < nproc:
        pytest.skip(f"needs {nproc} GPUs")
    port = 29640 + 10 * nproc + (1 if gp.startswith("1") else 0)
    res = _torchrun(nproc, "mp_check.py", ["79", "6", "639", "4"], {"MP_GP": gp, "MP_PAIRS": "2"}, port)
    assert res.returncode == 0
    assert "MP_OK" in res.stdout


@pytest.mark.parametrize("transport", ["p2p", "nccl"])
def test_dead_peer_raises_protocol_error(transport):
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    res = _torchrun(2, "mp_fail_check.py", ["79", "4"],
                    {"SHT_TRANSPORT": transport, "SHT_COMM_TIMEOUT_MS": "5000", "TORCH_NCCL_ASYNC_ERROR_HANDLING": "0"},
                    29680 + (transport == "nccl"), timeout=300)
    assert "FAIL_OK" in res.stdout, res.stdout[-2000:]
