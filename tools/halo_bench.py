"""Halo engine measurement: neighbourhood-mean steps of a periodic
nx x ny quad mesh (degree 4) on 1 or more B200 (torchrun for > 1), device-timed with CUDA
events over K steps after W warm-ups, max over ranks.  The stencil kernel's algorithmic HBM
bytes per owned element and step: 8 B member index + 4 x 8 B neighbour indices + 8 B value
read (its 4 neighbours' values are the same array, L2-resident between them) + 8 B output +
16 B copy back = 72 B; reported against the measured HBM copy peak.

usage: [torchrun --nproc-per-node N] python tools/halo_bench.py [nx] [ny] [steps]
"""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1908_06097_b200.halo import HaloEngine, derive_ghosts, negotiate_plan, partition_block, stencil_groups  # noqa: E402


def quad_csr(nx, ny):
    idx = np.arange(nx * ny, dtype=np.int64)
    x, y = idx % nx, idx // nx
    nb = np.stack([((x - 1) % nx) + y * nx, ((x + 1) % nx) + y * nx, x + ((y - 1) % ny) * nx,
                   x + ((y + 1) % ny) * nx], axis=1)
    nb.sort(axis=1)
    return np.arange(0, 4 * nx * ny + 1, 4, dtype=np.int64), nb.ravel()


def main():
    nx = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    ny = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 20
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    indptr, indices = quad_csr(nx, ny)
    owner, owned = partition_block(nx * ny, world)
    ghosts = derive_ghosts(indptr, indices, owner, owned[rank], rank)
    plan = negotiate_plan(owned[rank], ghosts, rank, world)
    eng = HaloEngine(plan, stencil_groups(indptr, indices, owned[rank], ghosts))
    v = torch.rand(plan.n_local, dtype=torch.float64, device="cuda")
    for _ in range(3):
        eng.stencil_step(v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        eng.stencil_step(v)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
    hbm = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() else 6650.0
    nsend, nrecv = eng.counts()
    gbs = 72.0 * plan.n_owned / (ms * 1e-3) / 1e9
    if rank == 0:
        print(json.dumps({"tool": "halo_bench", "grid": f"quad {nx}x{ny}", "ranks": world, "ms_per_step": ms,
                          "elements_per_rank": plan.n_owned, "halo_sent_per_rank": nsend,
                          "achieved_gbs_per_gpu": gbs, "hbm_frac": gbs / hbm,
                          "note": "72 algorithmic B per owned element per step"}), flush=True)
    eng.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
