"""Multi-rank GPU halo engine vs the reference's own halo engine (run under torchrun):
every rank builds its block partition, ghosts, plan (negotiated over NCCL) and stencil
groups, runs the fixture's steps on its GPU, and rank 0 compares the gathered owned values
and the per-step global checksums with tests/golden/halo_*.npz bit for bit.

usage: torchrun --nproc-per-node N tools/halo_check.py
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1908_06097_b200.halo import HaloEngine, derive_ghosts, negotiate_plan, partition_block, stencil_groups  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, P = dist.get_rank(), dist.get_world_size()
    ok = True
    for name in ("quad20x12", "rand300"):
        d = dict(np.load(ROOT / "tests" / "golden" / f"halo_{name}.npz"))
        n = len(d["init"])
        owner, owned = partition_block(n, P)
        ghosts = derive_ghosts(d["indptr"], d["indices"], owner, owned[rank], rank)
        plan = negotiate_plan(owned[rank], ghosts, rank, P)
        eng = HaloEngine(plan, stencil_groups(d["indptr"], d["indices"], owned[rank], ghosts))
        v = torch.zeros(plan.n_local, dtype=torch.float64, device="cuda")
        v[: plan.n_owned] = torch.from_numpy(d["init"][owned[rank]]).cuda()
        checks = []
        for _ in range(int(d["steps"])):
            eng.stencil_step(v)
            parts = [None] * P
            dist.all_gather_object(parts, v[: plan.n_owned].cpu().numpy())
            glob = np.empty(n)
            for r in range(P):
                glob[owned[r]] = parts[r]
            total = 0.0
            for x in glob:
                total += float(x)
            checks.append(total)
        good = np.array_equal(glob, d[f"final_{P}"]) and checks == list(d[f"checksums_{P}"])
        if rank == 0:
            print(f"{name} P={P}: values {'bit-identical' if np.array_equal(glob, d[f'final_{P}']) else 'DIFFER'}, "
                  f"checksums {'equal' if checks == list(d[f'checksums_{P}']) else 'DIFFER'}, "
                  f"sent/recv per exchange {eng.counts()}", flush=True)
        ok = ok and good
        eng.close()
    t = torch.tensor([0.0 if ok else 1.0], device="cuda")
    dist.all_reduce(t)
    if rank == 0:
        print("HALO_OK" if t.item() == 0 else "HALO_FAIL", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if t.item() == 0 else 1)


if __name__ == "__main__":
    main()
