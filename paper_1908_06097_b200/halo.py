"""GPU halo engine: the reference's unstructured-grid
halo exchange and neighbourhood-mean stencil, on device-resident fields.

The reference (/root/reference/pkg/src/haloflow/halo/) runs a rank program per
partition in one Python process: ``partition_block`` (partition.py:65-82) owns
contiguous global blocks, ghosts are the remote neighbours sorted by (owner,
global) (partition.py:46-62), ``build_plan`` negotiates per-peer send indices and
receive slots in two collective rounds (plan.py:75-144), ``exchange`` packs,
moves and unpacks them (engine.py:115-220) and ``stencil_step`` replaces every
owned value by the mean of its neighbours (engine.py:274-327).

Here one process per GPU holds one rank's field as a float64 CUDA tensor
(owned elements, then ghosts: the reference's local layout), the plan is
negotiated over ``torch.distributed`` (any backend: gloo on the CPU test-suite,
NCCL on the GPU), and ``HaloEngine`` executes exchange / stencil steps in
libsht.so (csrc/sht_halo.cu): a gather kernel, grouped NCCL send/recv in the
rotated order, a scatter kernel and the degree-grouped mean kernel, bit-identical
to the reference's numpy arithmetic.  The host-side pieces (partition, ghosts,
plan negotiation, stencil groups) are plain restatements with the reference's
ordering rules, so the local layout and plan are the reference's.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ConfigurationError, ProtocolError

__all__ = ["csr_adjacency", "partition_block", "derive_ghosts", "negotiate_plan", "stencil_groups",
           "RankPlan", "HaloEngine"]


def csr_adjacency(adjacency) -> tuple[np.ndarray, np.ndarray]:
    """(indptr, indices) of an adjacency list (``GlobalGrid.adjacency``: ascending, unique)."""
    indptr = np.zeros(len(adjacency) + 1, dtype=np.int64)
    indptr[1:] = np.cumsum([len(a) for a in adjacency])
    indices = np.fromiter((j for a in adjacency for j in a), dtype=np.int64, count=int(indptr[-1]))
    return indptr, indices


def partition_block(n: int, nranks: int):
    """Rank r owns globals [r B, (r+1) B), B = ceil(n / nranks) (partition.py:65-82).
    Returns (owner[n], owned list per rank)."""
    if nranks < 1:
        raise ConfigurationError("nranks must be >= 1")
    if nranks > n:
        raise ConfigurationError(f"cannot split {n} elements across {nranks} ranks")
    block = -(-n // nranks)
    owner = np.empty(n, dtype=np.int64)
    owned = []
    for r in range(nranks):
        lo = min(r * block, n)
        hi = min(lo + block, n)
        owner[lo:hi] = r
        owned.append(np.arange(lo, hi, dtype=np.int64))
    return owner, owned


def derive_ghosts(indptr: np.ndarray, indices: np.ndarray, owner: np.ndarray, owned: np.ndarray, rank: int):
    """Remote neighbours of this rank's owned elements as (global, owner), sorted by
    (owner, global) -- the ghost-slot order of partition.py:46-62."""
    owned = np.asarray(owned, dtype=np.int64)
    if len(owned) == 0:
        return []
    starts, lens = indptr[owned], indptr[owned + 1] - indptr[owned]
    first = np.concatenate([[0], np.cumsum(lens)[:-1]])              # CSR rows of the owned elements
    nb = indices[np.repeat(starts - first, lens) + np.arange(int(lens.sum()))]
    remote = np.unique(nb[owner[nb] != rank])
    order = np.lexsort((remote, owner[remote]))
    return [(int(g), int(owner[g])) for g in remote[order]]


@dataclass
class RankPlan:
    """One rank's exchange plan (plan.py:33-55)."""

    rank: int
    nranks: int
    n_owned: int
    n_local: int
    send_index: dict
    recv_slot: dict


def negotiate_plan(owned: np.ndarray, ghosts, rank: int, nranks: int, group=None) -> RankPlan:
    """The reference's plan protocol (plan.py:75-144) over torch.distributed: every rank
    publishes, per owner, the globals it needs (ascending, from the (owner, global)-sorted
    ghost list) and learns what the others need from it; a request for an element the rank
    does not own is a corrupt partition (ProtocolError)."""
    needs: dict[int, list[int]] = {}
    slots: dict[int, list[int]] = {}
    base = len(owned)
    for slot, (gid, own) in enumerate(ghosts):
        needs.setdefault(own, []).append(int(gid))
        slots.setdefault(own, []).append(base + slot)
    if nranks > 1:
        import torch.distributed as dist

        everyone = [None] * nranks
        dist.all_gather_object(everyone, needs, group=group)
    else:
        everyone = [needs]
    send_index = {}
    for src in range(nranks):
        if src == rank:
            continue
        wanted = everyone[src].get(rank, [])
        if not wanted:
            continue
        w = np.asarray(wanted, dtype=np.int64)
        locs = np.searchsorted(owned, w)
        bad = (locs >= len(owned)) | (owned[np.minimum(locs, max(len(owned) - 1, 0))] != w) if len(owned) else \
            np.ones(len(w), dtype=bool)
        if bad.any():
            raise ProtocolError(f"corrupt partition: rank {src} asked rank {rank} for element {int(w[bad][0])} "
                                "it does not own")
        send_index[src] = locs.astype(np.int64)
    recv_slot = {p: np.asarray(sl, dtype=np.int64) for p, sl in slots.items()}
    return RankPlan(rank, nranks, len(owned), base + len(ghosts), send_index, recv_slot)


def stencil_groups(indptr: np.ndarray, indices: np.ndarray, owned: np.ndarray, ghosts):
    """Degree groups of the neighbourhood mean (engine._stencil_ws, engine.py:237-271):
    [(degree, members (owned locals, ascending), neighbours [count, degree] as local
    indices in ascending global order per row)], degrees ascending."""
    owned = np.asarray(owned, dtype=np.int64)
    gg = np.asarray([g for g, _ in ghosts], dtype=np.int64)
    keys = np.concatenate([owned, gg])
    locs = np.arange(len(keys), dtype=np.int64)
    srt = np.argsort(keys, kind="stable")
    keys_s, locs_s = keys[srt], locs[srt]
    deg = indptr[owned + 1] - indptr[owned]
    out = []
    for d in np.unique(deg):
        mem = np.flatnonzero(deg == d).astype(np.int64)
        rows = indices[indptr[owned[mem]][:, None] + np.arange(d)[None, :]]
        pos = np.searchsorted(keys_s, rows)
        out.append((int(d), mem, locs_s[pos].reshape(len(mem), int(d))))
    return out


class HaloEngine:
    """Exchange / stencil executor of one rank on its CUDA device (libsht.so, csrc/sht_halo.cu).

    ``values`` passed to ``exchange`` / ``stencil_step`` is this rank's float64 CUDA tensor
    of ``plan.n_local`` elements (owned, then ghosts); both are stream-ordered on the current
    stream.  Collective over ``group`` (an NCCL process group when nranks > 1)."""

    def __init__(self, plan: RankPlan, groups=None, group=None, device=None):
        import torch

        lib = _lib.load()
        self.plan = plan
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        P = plan.nranks
        send_counts = np.zeros(P, dtype=np.int64)
        recv_counts = np.zeros(P, dtype=np.int64)
        sidx, rslot = [], []
        for p in range(P):
            s = plan.send_index.get(p)
            r = plan.recv_slot.get(p)
            if s is not None:
                send_counts[p] = len(s)
                sidx.append(np.asarray(s, dtype=np.int64))
            if r is not None:
                recv_counts[p] = len(r)
                rslot.append(np.asarray(r, dtype=np.int64))
        send_index = np.concatenate(sidx) if sidx else np.zeros(1, dtype=np.int64)
        recv_slot = np.concatenate(rslot) if rslot else np.zeros(1, dtype=np.int64)
        groups = groups or []
        deg = np.asarray([g[0] for g in groups] or [1], dtype=np.int32)
        cnt = np.asarray([len(g[1]) for g in groups] or [0], dtype=np.int64)
        mem = np.concatenate([g[1] for g in groups]) if groups else np.zeros(1, dtype=np.int64)
        nbr = np.concatenate([g[2].ravel() for g in groups]) if groups else np.zeros(1, dtype=np.int64)
        uid = None
        if P > 1:
            import torch.distributed as dist

            buf = C.create_string_buffer(128)
            if plan.rank == 0:
                _lib.check(lib.sht_nccl_get_unique_id(buf))
            obj = [bytes(buf.raw)]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            uid = C.create_string_buffer(obj[0], 128)
        h = C.c_void_p()
        arrs = [np.ascontiguousarray(a) for a in (send_counts, send_index, recv_counts, recv_slot, deg, cnt, mem, nbr)]
        with torch.cuda.device(self.device):
            _lib.check(lib.sht_halo_create(
                plan.rank, P, uid, plan.n_local, plan.n_owned,
                arrs[0].ctypes.data_as(_lib.i64p), arrs[1].ctypes.data_as(_lib.i64p),
                arrs[2].ctypes.data_as(_lib.i64p), arrs[3].ctypes.data_as(_lib.i64p),
                len(groups), arrs[4].ctypes.data_as(_lib.i32p), arrs[5].ctypes.data_as(_lib.i64p),
                arrs[6].ctypes.data_as(_lib.i64p), arrs[7].ctypes.data_as(_lib.i64p), C.byref(h)))
        self._h = h
        self._lib = lib

    def _check(self, values):
        import torch

        if self._h is None:
            raise ConfigurationError("the halo engine is closed")
        if not isinstance(values, torch.Tensor) or values.dtype != torch.float64 or values.device != self.device:
            raise ConfigurationError(f"values must be a float64 tensor on {self.device}")
        if values.numel() != self.plan.n_local or not values.is_contiguous():
            raise ConfigurationError(f"values must be contiguous with {self.plan.n_local} elements")

    def exchange(self, values) -> None:
        """Refresh every ghost with its owner's value (engine.exchange)."""
        import torch

        self._check(values)
        with torch.cuda.device(self.device):
            s = torch.cuda.current_stream(self.device)
            _lib.check(self._lib.sht_halo_exchange(self._h, C.c_void_p(values.data_ptr()), C.c_void_p(s.cuda_stream)))

    def stencil_step(self, values) -> None:
        """One neighbourhood-mean step, OverlapMode.NONE (engine.stencil_step)."""
        import torch

        self._check(values)
        with torch.cuda.device(self.device):
            s = torch.cuda.current_stream(self.device)
            _lib.check(self._lib.sht_halo_stencil_step(self._h, C.c_void_p(values.data_ptr()),
                                                      C.c_void_p(s.cuda_stream)))

    def counts(self) -> tuple[int, int]:
        a, b = C.c_int64(), C.c_int64()
        _lib.check(self._lib.sht_halo_counts(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def close(self) -> None:
        import torch

        h, self._h = getattr(self, "_h", None), None
        if h:
            with torch.cuda.device(self.device):
                self._lib.sht_halo_destroy(h)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
