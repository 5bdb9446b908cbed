"""Peer-failure check (run under torchrun, >= 2 GPUs): the last rank dies
right after plan creation; every other rank must get ProtocolError from its
next bounded wait (SHTransform.synchronize) within SHT_COMM_TIMEOUT_MS plus
slack, instead of hanging (the reference's first-error abort,
halo/router.py:124-126, 199-205).  Prints FAIL_OK on rank 0.

usage: SHT_COMM_TIMEOUT_MS=3000 torchrun --nproc-per-node 2 tools/mp_fail_check.py [T nfld]
"""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1908_06097_b200 import ProtocolError, SHTransform  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 79
    nf = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    sh = SHTransform(T, nfld=nf, group=dist.group.WORLD)
    spec = torch.zeros(nf, sh.nspec_local, dtype=torch.float64, device="cuda")
    grid = torch.empty(nf, sh.npts_local, dtype=torch.float64, device="cuda")
    sh.inv_trans(spec, out=grid)  # one healthy transform first
    sh.synchronize(timeout_ms=60000)
    dist.barrier()
    if rank == world - 1:
        print(f"rank {rank}: dying now", flush=True)
        os._exit(0)
    t0 = time.time()
    dbg = os.environ.get("MP_FAIL_DEBUG") == "1"
    try:
        for i in range(3):
            if dbg:
                print(f"rank {rank}: pair {i} inv", flush=True)
            sh.inv_trans(spec, out=grid)
            if dbg:
                print(f"rank {rank}: pair {i} dir", flush=True)
            sh.dir_trans(grid, out=spec)
        if dbg:
            print(f"rank {rank}: synchronize", flush=True)
        sh.synchronize()
        print(f"rank {rank}: no error after {time.time() - t0:.1f}s", flush=True)
        ok = False
    except ProtocolError as e:
        dt = time.time() - t0
        print(f"rank {rank}: ProtocolError after {dt:.1f}s: {e}", flush=True)
        limit = float(os.environ.get("SHT_COMM_TIMEOUT_MS", "60000")) / 1e3 + 30.0
        ok = dt <= limit
    try:  # the second call must fail at once (the plan stays failed)
        sh.inv_trans(spec, out=grid)
        ok = False
        print(f"rank {rank}: call after the failure was accepted", flush=True)
    except ProtocolError:
        pass
    if rank == 0:
        print("FAIL_OK" if ok else "FAIL_BAD", flush=True)
    sys.stdout.flush()
    os._exit(0 if ok else 1)  # the process group is broken: no collective teardown


if __name__ == "__main__":
    main()
