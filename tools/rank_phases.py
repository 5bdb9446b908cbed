"""Per-rank phase breakdown of the transform pair (run under torchrun).
usage: torchrun --nproc-per-node N tools/rank_phases.py [T] [nfld] [pairs]
Prints one line per rank: ms/pair and the seven phase times, plus the
all-to-all bytes that rank sends per direction."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_06097_b200 import SHTransform  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 639
    nf = int(sys.argv[2]) if len(sys.argv) > 2 else 548
    K = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    sh = SHTransform(T, nfld=nf, group=dist.group.WORLD, profile=True)
    spec = torch.randn(nf, sh.nspec_local, dtype=torch.float64, device="cuda") * 1e-3
    grid = torch.empty(nf, sh.npts_local, dtype=torch.float64, device="cuda")
    for _ in range(3):
        sh.inv_trans(spec, out=grid)
        sh.dir_trans(grid, out=spec)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(K):
        sh.inv_trans(spec, out=grid)
        sh.dir_trans(grid, out=spec)
    e1.record()
    torch.cuda.synchronize()
    ph = sh.phase_ms(K)
    w = sh.work()
    line = (f"rank {rank}/{world} {e0.elapsed_time(e1) / K:.2f} ms/pair rings={len(sh.ring_list)} m={len(sh.m_list)} "
            + " ".join(f"{k}={v:.2f}" for k, v in ph.items()) + f" work={ {k: float(v) for k, v in w.items()} }")
    out = [None] * world
    dist.all_gather_object(out, line)
    if rank == 0:
        print("\n".join(out), flush=True)
    sh.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
