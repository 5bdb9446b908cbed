"""Generate the committed golden fixtures under tests/golden/.

Run in the build container (needs /root/reference for the schedule fixture):

    python tests/golden/make_golden.py

* tco79_f4.npz, tco15_f3.npz -- oracle inverse/direct outputs on the seeded
  synthetic inputs of SURVEY.md 8d (spectral seed T, grid seed T+1).  The
  transform has no reference implementation, so these pin the
  oracle (itself pinned by analytic KATs + scipy in tests/test_oracle.py)
  against accidental drift, and let GPU tests run without the oracle.
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


if __name__ == "__main__":
    transform_fixture(79, 4)
    transform_fixture(15, 3)
    schedule_fixture()
    print("wrote", sorted(p.name for p in HERE.iterdir()))
