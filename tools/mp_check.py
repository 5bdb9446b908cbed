"""Multi-rank parity check (run under torchrun): each rank's local slice of
inv_trans / dir_trans / round trip vs the 1-rank CPU oracle.

Every configuration enqueues K >= 4 inverse + direct pairs on DISTINCT inputs
back to back with no host synchronisation in between (the p2p transport's
epoch handshakes -- arrived / drained -- then run under overlap, as in the
bench), synchronises once (bounded, SHTransform.synchronize) and compares
every output with the oracle.  The transport comes from SHT_TRANSPORT (p2p
default, nccl), the Legendre mode from SHT_RECOMPUTE=1.

usage: torchrun --nproc-per-node N tools/mp_check.py T nfld [T nfld ...]
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.sht_oracle import SHTransformOracle, random_grid, random_spectral  # noqa: E402
from oracle.transposition import Layout, gp_local  # noqa: E402
from paper_1908_06097_b200 import SHTransform  # noqa: E402

K = int(os.environ.get("MP_PAIRS", "4"))


def rel(x, ref):
    return float(np.max(np.max(np.abs(x - ref), axis=1) / np.max(np.abs(ref), axis=1)))


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    args = [int(x) for x in sys.argv[1:]]
    recompute = bool(int(os.environ.get("SHT_RECOMPUTE", "0")))
    gp = tuple(int(x) for x in os.environ["MP_GP"].split(",")) if os.environ.get("MP_GP") else None
    worst = 0.0
    for T, nf in zip(args[0::2], args[1::2]):
        o = SHTransformOracle(T, nfld=nf)
        lay = Layout(o, world)
        sh = SHTransform(T, nfld=nf, group=dist.group.WORLD, recompute_legendre=recompute, gp_layout=gp)
        assert list(sh.m_list) == list(lay.M[rank]), "m partition differs from the restatement"
        assert list(sh.ring_list) == lay.local_rings(rank), "ring partition differs"
        want = os.environ.get("SHT_TRANSPORT", "p2p")
        assert sh.transport == want, (sh.transport, want)
        specs = [random_spectral(T, nf, seed=1000 * T + k) for k in range(K)]
        grids = [random_grid(T, nf, o.npts, seed=2000 * T + k) for k in range(K)]
        la = [torch.from_numpy(np.ascontiguousarray(lay.local_spec(a, rank))).cuda() for a in specs]
        if gp:  # grid side in the 2-D grid-point layout
            local_grid = lambda x: gp_local(x, o.nloen, rank, gp[0], gp[1])  # noqa: E731
        else:
            local_grid = lambda x: lay.local_grid(x, rank)  # noqa: E731
        lg = [torch.from_numpy(np.ascontiguousarray(local_grid(g))).cuda() for g in grids]
        torch.cuda.synchronize()
        gi, sd, rt = [], [], []
        for k in range(K):  # no host sync between the pairs
            gi.append(sh.inv_trans(la[k]))
            sd.append(sh.dir_trans(lg[k]))
            rt.append(sh.dir_trans(gi[k]))
        sh.synchronize(timeout_ms=600000)
        e = [0.0, 0.0, 0.0]
        for k in range(K):
            e[0] = max(e[0], rel(gi[k].cpu().numpy(), local_grid(o.inv_trans(specs[k]))))
            e[1] = max(e[1], rel(sd[k].cpu().numpy(), lay.local_spec(o.dir_trans(grids[k]), rank)))
            e[2] = max(e[2], rel(rt[k].cpu().numpy(), lay.local_spec(specs[k], rank)))
        print(f"rank {rank}/{world} T={T} nfld={nf} transport={sh.transport} recompute={recompute} gp={gp} pairs={K}: "
              f"inv {e[0]:.2e} dir {e[1]:.2e} rt {e[2]:.2e}", flush=True)
        worst = max(worst, *e)
        sh.close()
    t = torch.tensor([worst], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print("MP_OK" if t.item() <= 1e-10 else f"MP_FAIL {t.item()}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if t.item() <= 1e-10 else 1)


if __name__ == "__main__":
    main()
