"""Host logic of the multi-GPU path on CPU: the P-rank layout emulated in
process must equal the 1-rank oracle (the reference's oracle-equivalence
pattern, test_acceptance.py:60-80), and the same pack / all-to-all / unpack
run across real processes over gloo (world_size 2)."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.sht_oracle import SHTransformOracle, random_spectral
from oracle.transposition import Layout, emulate_inv


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_emulated_ranks_equal_one_rank(P):
    T, nf = 31, 3
    o = SHTransformOracle(T, nfld=nf)
    a = random_spectral(T, nf)
    ref = o.inv_trans(a)
    grids, lay = emulate_inv(o, a, P)
    for r in range(P):
        assert np.max(np.abs(grids[r] - lay.local_grid(ref, r))) <= 1e-13
    # every grid point is owned exactly once
    assert sum(g.shape[1] for g in grids) == o.npts


def _worker(rank, world, port, T, nf, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = SHTransformOracle(T, nfld=nf)
    lay = Layout(o, world)
    a = random_spectral(T, nf)
    blocks = lay.pack_inv(lay.local_spec(a, rank), rank)
    rows = lay.rows()
    send = torch.from_numpy(np.concatenate(blocks))
    recv = torch.empty(int(rows[:, rank].sum()) * nf * 4, dtype=torch.float64)
    # rotated issue order (collectives.py:85-86) realised as one all_to_all_single
    dist.all_to_all_single(recv, send, output_split_sizes=[int(x) * nf * 4 for x in rows[:, rank]],
                           input_split_sizes=[int(x) * nf * 4 for x in rows[rank, :]])
    splits = np.cumsum([0] + [int(x) * nf * 4 for x in rows[:, rank]])
    recv_blocks = [recv.numpy()[splits[s]: splits[s + 1]] for s in range(world)]
    grid = lay.unpack_inv(recv_blocks, rank)
    err = float(np.max(np.abs(grid - lay.local_grid(o.inv_trans(a), rank))))
    q.put((rank, err))
    dist.destroy_process_group()


def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 23, 3, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r for r, _ in res) == [0, 1]
    assert max(e for _, e in res) <= 1e-13


def test_gp_bands_match_restatement(lib):
    """libsht's latitude bands of the 2-D grid-point layout == the restatement."""
    import numpy as np

    from oracle.sht_oracle import octahedral_nloen
    from oracle.transposition import gp_bands, gp_local
    from paper_1908_06097_b200 import _lib

    for T, nA in [(79, 1), (79, 2), (79, 3), (639, 2), (639, 4), (1279, 8)]:
        out = np.zeros(nA + 1, dtype=np.int32)
        _lib.check(lib.sht_gp_bands(T, 0, None, nA, out.ctypes.data_as(_lib.i32p)))
        assert list(out) == gp_bands(octahedral_nloen(T), nA)
    # the grid-point slices of all ranks partition the global grid
    T, nA, nB = 31, 2, 3
    nl = octahedral_nloen(T)
    g = np.arange(int(nl.sum()), dtype=float)[None, :]
    got = np.sort(np.concatenate([gp_local(g, nl, r, nA, nB)[0] for r in range(nA * nB)]))
    assert np.array_equal(got, g[0])
