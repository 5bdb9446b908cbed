"""Generate the committed golden fixtures under tests/golden/.

Run in the build container (needs /root/reference for the schedule fixture):

    python tests/golden/make_golden.py

* tco79_f4.npz, tco15_f3.npz -- oracle inverse/direct outputs on the seeded
  synthetic inputs of SURVEY.md 8d (spectral seed T, grid seed T+1).  The
  transform has no reference implementation, so these pin the
  oracle (itself pinned by analytic KATs + scipy in tests/test_oracle.py)
  against accidental drift, and let GPU tests run without the oracle.
* halo_*.npz -- the reference's own halo engine (run_stencil: block partition,
  negotiated plan, 5 neighbourhood-mean steps) on a periodic quad mesh and a
  random grid for 1 / 2 / 4 ranks: final values, checksums and every rank's
  send_index / recv_slot, pinning the GPU halo engine (csrc/sht_halo.cu).
* schedules.json -- the reference's own all-to-all schedules, produced by
  importing haloflow from /root/reference: build_alltoall(kind, sizes) flow
  order for P = 1..8 (collectives.py:96-117) and, for the TCo639 transposition
  size matrix of this build, the reference netsim makespan of each schedule
  on an inline 8 x B200 NVSwitch topology (topology.py:536-599,
  netsim.py:347-398).
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from oracle.sht_oracle import SHTransformOracle, random_grid, random_spectral  # noqa: E402
from oracle.transposition import Layout  # noqa: E402


def transform_fixture(T: int, nfld: int) -> None:
    o = SHTransformOracle(T, nfld=nfld)
    a = random_spectral(T, nfld)
    g = random_grid(T, nfld, o.npts)
    np.savez_compressed(HERE / f"tco{T}_f{nfld}.npz", spec=a, grid=g, inv=o.inv_trans(a), dir=o.dir_trans(g),
                        mu=o.mu, w=o.w)


def schedule_fixture() -> None:
    sys.path.insert(0, "/root/reference/pkg/src")
    from haloflow.collectives import ScheduleKind, build_alltoall, compare_schedules, uniform_sizes
    from haloflow.topology import from_spec

    out = {"rotated_order": {}, "tco639": {}}
    for P in range(1, 9):
        flows = build_alltoall(ScheduleKind.ROTATED_CONCURRENT, uniform_sizes(P, 1))
        out["rotated_order"][str(P)] = [[f.src_rank, f.dst_rank] for f in flows]
    nfld = 548
    o = SHTransformOracle(639, nfld=1)
    topo = from_spec({
        "name": "b200_nvswitch_8",
        "nodes": [f"device:{i}" for i in range(8)] + ["switch:0"],
        "links": [{"a": f"device:{i}", "b": "switch:0", "gbps_per_dir": 50, "lanes": 18} for i in range(8)],
        "device_mem_bw_gbps": 3216.8,
    })
    for P in (2, 4, 8):
        rows = Layout(o, P).rows()
        sizes = (rows * 32 * nfld).tolist()
        res = compare_schedules(topo, list(range(P)), sizes)
        out["tco639"][str(P)] = {
            "rows": rows.tolist(),
            "bytes": sizes,
            "makespan_s": {k.value: v.makespan for k, v in res.items()},
        }
    (HERE / "schedules.json").write_text(json.dumps(out, indent=1, sort_keys=True))


HALO_GRIDS = {"quad20x12": ("quad_mesh", (20, 12)), "rand300": ("random_grid", (300, 6, 5))}
HALO_STEPS = 5


def halo_init(n: int) -> np.ndarray:
    g = np.arange(n, dtype=np.float64)
    return np.sin(0.37 * g) + 0.01 * g


def halo_fixture() -> None:
    """The reference's own halo engine (haloflow.halo, run_stencil with the block
    partition and the negotiated plan) on two grids for 1, 2 and 4 ranks: the grid
    (CSR), the initial field, the gathered owned values and global checksums after
    each of HALO_STEPS neighbourhood-mean steps, and every rank's plan."""
    sys.path.insert(0, "/root/reference/pkg/src")
    from haloflow.halo import grid as hg
    from haloflow.halo.engine import gather_global, run_stencil

    for name, (gen, args) in HALO_GRIDS.items():
        grid = getattr(hg, gen)(*args)
        indptr = np.zeros(grid.n + 1, dtype=np.int64)
        indptr[1:] = np.cumsum([len(a) for a in grid.adjacency])
        indices = np.asarray([j for a in grid.adjacency for j in a], dtype=np.int64)
        init = halo_init(grid.n)
        out = {"indptr": indptr, "indices": indices, "init": init, "steps": np.int64(HALO_STEPS)}
        for P in (1, 2, 4):
            fields, part, plan, checks = run_stencil(grid, P, HALO_STEPS, init)
            out[f"final_{P}"] = gather_global(fields, part)
            out[f"checksums_{P}"] = np.asarray(checks)
            for r, rp in enumerate(plan.ranks):
                for q in range(P):
                    if q in rp.send_index:
                        out[f"send_{P}_{r}_{q}"] = rp.send_index[q]
                    if q in rp.recv_slot:
                        out[f"recv_{P}_{r}_{q}"] = rp.recv_slot[q]
        np.savez_compressed(HERE / f"halo_{name}.npz", **out)


if __name__ == "__main__":
    transform_fixture(79, 4)
    transform_fixture(15, 3)
    schedule_fixture()
    halo_fixture()
    print("wrote", sorted(p.name for p in HERE.iterdir()))
