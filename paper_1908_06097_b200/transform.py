"""The drop-in transform API: ``SHTransform(truncation, grid, nfld)`` with
``inv_trans`` (spectral -> grid) and ``dir_trans`` (grid -> spectral).

This is the "CPU reference's Python transform API (setup with truncation,
grid and field count; inv_trans/dir_trans on field batches)" named by the
north star (BASELINE.json).  The reference has no such code, so
the names, argument meaning and error behaviour follow SURVEY.md section 8b;
``oracle.sht_oracle.SHTransformOracle`` is the CPU restatement with the same
signature that the tests compare against.

Every call goes through libsht.so (include/sht.h): hand-written sm_100a
kernels for the Legendre GEMMs (DMMA), the ring FFTs and the Legendre
polynomial table, plus NCCL for the grid <-> spectral transposition when a
process group with more than one rank is given.  There is no CPU path.

Array conventions:
  spectral  float64 [nfld, nspec_local]  m-major, n ascending, re/im interleaved
            (nspec_local = (T+1)(T+2) on one rank)
  grid      float64 [nfld, npts_local]   rings north -> south, 2 pi k / NLOEN longitudes
On more than one rank each rank holds the spectral coefficients of
``m_list`` and the grid points of ``ring_list`` (see ``local_layout``).
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np

from . import _lib
from .errors import ConfigurationError


def octahedral_nloen(truncation: int) -> np.ndarray:
    """NLOEN of the octahedral TCo grid: 4i+16 points on northern ring i (1-based), mirrored south."""
    T = int(truncation)
    north = 4 * np.arange(1, T + 2, dtype=np.int32) + 16
    return np.concatenate([north, north[::-1]])


def nspec_real(truncation: int) -> int:
    T = int(truncation)
    return (T + 1) * (T + 2)


class SHTransform:
    """Spherical-harmonics transform plan on the current CUDA device.

    Parameters
    ----------
    truncation : spectral truncation T (TCo T).
    grid       : "octahedral" (TCo grid, NDGL = 2(T+1)) or an array of NDGL ring
                 lengths (north first, north/south symmetric).
    nfld       : number of fields per batch.
    group      : torch.distributed process group (NCCL) to shard over, or None
                 for one GPU.
    recompute_legendre : do not store the P_n^m table; regenerate it chunk by
                 chunk of wavenumbers (bounded 2 GB scratch) right before the
                 GEMM tiles that use it, every transform (TCo1999 memory mode).
    profile    : record CUDA events around every phase (see ``phase_ms``).
    gp_layout  : (nA, nB) with nA * nB = ranks: the grid side in a 2-D grid-point
                 layout (nA latitude bands x nB longitude segments, see
                 ``local_layout``) instead of whole ring pairs; inv_trans / dir_trans
                 then add the ring <-> grid-point transposition (TRGTOL / TRLTOG role).
    """

    def __init__(self, truncation: int, grid="octahedral", nfld: int = 1, *, group=None,
                 recompute_legendre: bool = False, profile: bool = False, device=None, gp_layout=None):
        import torch

        lib = _lib.load()
        self.T = int(truncation)
        self.nfld = int(nfld)
        if self.T < 1:
            raise ConfigurationError("truncation must be >= 1")
        if self.nfld < 1:
            raise ConfigurationError("nfld must be >= 1")
        if isinstance(grid, str):
            if grid != "octahedral":
                raise ConfigurationError(f"unknown grid {grid!r} (use 'octahedral' or an NLOEN array)")
            self.nloen = octahedral_nloen(self.T)
            nloen_p = None
        else:
            self.nloen = np.ascontiguousarray(np.asarray(grid, dtype=np.int32))
            if self.nloen.ndim != 1:
                raise ConfigurationError("grid must be 1-D ring lengths")
            nloen_p = self.nloen.ctypes.data_as(_lib.i32p)
        self.ndgl = int(self.nloen.size)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if self.device.type != "cuda":
            raise ConfigurationError("SHTransform runs on a CUDA device only (no CPU fallback)")

        self.group = group
        if group is not None:
            import torch.distributed as dist

            self.rank = dist.get_rank(group)
            self.nranks = dist.get_world_size(group)
        else:
            self.rank, self.nranks = 0, 1
        uid = None
        if self.nranks > 1:
            import torch.distributed as dist

            buf = C.create_string_buffer(128)
            if self.rank == 0:
                _lib.check(lib.sht_nccl_get_unique_id(buf))
            obj = [bytes(buf.raw)]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0), group=group)
            uid = C.create_string_buffer(obj[0], 128)
        flags = 0
        if recompute_legendre:
            flags |= _lib.SHT_FLAG_RECOMPUTE_LEGENDRE
        if profile:
            flags |= _lib.SHT_FLAG_PROFILE_PHASES
        self.profile = bool(profile)
        plan = C.c_void_p()
        with torch.cuda.device(self.device):
            _lib.check(lib.sht_plan_create(self.T, self.ndgl, nloen_p, self.nfld, self.rank, self.nranks,
                                           uid, flags, C.byref(plan)))
        self._plan = plan
        self._lib = lib

        nspec = C.c_int64()
        npts = C.c_int64()
        nm = C.c_int32()
        nr = C.c_int32()
        mlist = (C.c_int32 * (self.T + 1))()
        rlist = (C.c_int32 * self.ndgl)()
        _lib.check(lib.sht_local_layout(plan, C.byref(nspec), C.byref(npts), mlist, C.byref(nm), rlist, C.byref(nr)))
        self.nspec_local = int(nspec.value)
        self.npts_local = int(npts.value)
        self.m_list = np.array(mlist[: nm.value], dtype=np.int64)
        self.ring_list = np.array(rlist[: nr.value], dtype=np.int64)
        self.gp = None
        if gp_layout is not None:
            nA, nB = (int(x) for x in gp_layout)
            with torch.cuda.device(self.device):
                _lib.check(lib.sht_plan_set_gp_layout(plan, nA, nB))
            npg, lo, hi, seg, nseg = C.c_int64(), C.c_int32(), C.c_int32(), C.c_int32(), C.c_int32()
            _lib.check(lib.sht_gp_layout(plan, C.byref(npg), C.byref(lo), C.byref(hi), C.byref(seg), C.byref(nseg)))
            self.gp = {"nA": nA, "nB": nB, "npts_gp_local": int(npg.value), "band_rings": (lo.value, hi.value),
                       "segment": seg.value, "nsegments": nseg.value}
            self.npts_grid = int(npg.value)
        else:
            self.npts_grid = self.npts_local

    # ------------------------------------------------------------------ helpers
    def local_layout(self) -> dict:
        """This rank's spectral wavenumbers and ring pairs; with a grid-point layout also its
        latitude band (global rings [lo, hi)) and longitude segment (points
        [floor(N_j s / nB), floor(N_j (s+1) / nB)) of each ring)."""
        out = {"nspec_local": self.nspec_local, "npts_local": self.npts_local,
               "m_list": self.m_list.copy(), "ring_list": self.ring_list.copy()}
        if self.gp:
            out["gp"] = dict(self.gp)
        return out

    def work(self) -> dict:
        """Algorithmic work of this rank per inverse+direct pair."""
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        _lib.check(self._lib.sht_work(self._plan, C.byref(a), C.byref(b), C.byref(c)))
        return {"legendre_flops": a.value, "fft_bytes": b.value, "a2a_bytes": c.value}

    def kernel_launches(self) -> int:
        """libsht kernel launches issued by one inv_trans + dir_trans pair."""
        n = C.c_int32()
        _lib.check(self._lib.sht_kernel_launches(self._plan, C.byref(n)))
        return int(n.value)

    @property
    def transport(self) -> str:
        """'p2p' (rows stored into the peers' buffers by the kernels over NVLink),
        'nccl' (grouped send/recv) or 'local' (one rank)."""
        n = C.c_int32()
        _lib.check(self._lib.sht_transport(self._plan, C.byref(n)))
        return "p2p" if n.value & 1 else ("nccl" if self.nranks > 1 else "local")

    @property
    def row_layout(self) -> str:
        """'classic' (a Fourier row holds every field) or 'field-blocked' (64-field
        blocks; the p2p transposition past the remote-store cliff), sht_internal.h."""
        n = C.c_int32()
        _lib.check(self._lib.sht_transport(self._plan, C.byref(n)))
        return "field-blocked" if n.value & 2 else "classic"

    def phase_ms(self, npairs: int = 1) -> dict:
        """Device times (ms) per phase, averaged over the last ``npairs`` (<= 64)
        inv_trans + dir_trans pairs (plan created with profile=True)."""
        import torch

        v = (C.c_float * 7)()
        with torch.cuda.device(self.device):
            _lib.check(self._lib.sht_phase_ms_avg(self._plan, int(npairs), v, 7))
        keys = ("legendre_poly_setup", "inv_legendre", "inv_alltoall", "inv_fft", "dir_fft", "dir_alltoall",
                "dir_legendre")
        return dict(zip(keys, [float(x) for x in v]))

    def _check(self, x, ncols: int, what: str):
        import torch

        if not isinstance(x, torch.Tensor):
            raise ConfigurationError(f"{what} must be a torch.Tensor or numpy array")
        if x.dtype != torch.float64:
            raise ConfigurationError(f"{what} must be float64, got {x.dtype}")
        if x.device != self.device:
            raise ConfigurationError(f"{what} must live on {self.device}, got {x.device}")
        if tuple(x.shape) != (self.nfld, ncols):
            raise ConfigurationError(f"{what} must have shape ({self.nfld}, {ncols}), got {tuple(x.shape)}")
        if not x.is_contiguous():
            raise ConfigurationError(f"{what} must be contiguous")
        if x.data_ptr() % 16:
            raise ConfigurationError(f"{what} must be 16-byte aligned")

    def _run(self, fn, x, ncols_in: int, ncols_out: int, out, stream):
        import torch

        if getattr(self, "_plan", None) is None:
            raise ConfigurationError("the plan is closed")
        with torch.cuda.device(self.device):
            s = stream if stream is not None else torch.cuda.current_stream(self.device)
            host = isinstance(x, np.ndarray)
            if host:  # copy in on the transform's stream, so it is ordered before the kernels
                xt = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).pin_memory()
                with torch.cuda.stream(s):
                    xt = xt.to(self.device, non_blocking=True)
            else:
                xt = x
            self._check(xt, ncols_in, "input")
            if out is None:
                with torch.cuda.stream(s):
                    out = torch.empty((self.nfld, ncols_out), dtype=torch.float64, device=self.device)
            else:
                self._check(out, ncols_out, "out")
            _lib.check(fn(self._plan, C.c_void_p(xt.data_ptr()), C.c_void_p(out.data_ptr()),
                          C.c_void_p(s.cuda_stream)))
            if host:  # bounded wait (peer failure -> ProtocolError), then the copy back on the same stream
                self.synchronize(s)
                with torch.cuda.stream(s):
                    res = out.cpu()
                return res.numpy()
        return out

    def synchronize(self, stream=None, timeout_ms: int = 0) -> None:
        """Wait for the transforms enqueued on ``stream`` (default: the current
        stream) with failure detection: raises ``ProtocolError`` when a peer
        rank died or desynchronised (handshake timeout, NCCL asynchronous
        error) or the wait exceeded ``timeout_ms`` (<= 0: SHT_COMM_TIMEOUT_MS,
        default 60 s)."""
        import torch

        with torch.cuda.device(self.device):
            s = stream if stream is not None else torch.cuda.current_stream(self.device)
            _lib.check(self._lib.sht_wait(self._plan, C.c_void_p(s.cuda_stream), int(timeout_ms)))

    # ------------------------------------------------------------------ API
    def inv_trans(self, spec, out=None, stream=None):
        """Spectral [nfld, nspec_local] -> grid [nfld, npts_local] (float64).

        ``spec`` may be a CUDA tensor (result stays on the device, stream-ordered
        on ``stream`` / the current stream) or a host numpy array (copied in and
        the result copied back to a numpy array).
        """
        fn = self._lib.sht_inv_trans_gp if self.gp else self._lib.sht_inv_trans
        return self._run(fn, spec, self.nspec_local, self.npts_grid, out, stream)

    def dir_trans(self, grid, out=None, stream=None):
        """Grid [nfld, npts_local] -> spectral [nfld, nspec_local] (float64)."""
        fn = self._lib.sht_dir_trans_gp if self.gp else self._lib.sht_dir_trans
        return self._run(fn, grid, self.npts_grid, self.nspec_local, out, stream)

    def pairs_pipelined(self, host_in, host_out) -> None:
        """inv_trans + dir_trans of a stream of host batches: host_in[i] (pinned
        float64 [nfld, nspec_local]) -> round trip -> host_out[i].  The copy of
        batch i+1 to the GPU and of batch i-1 back to the host run on their own
        streams under the transforms of batch i (double-buffered device
        buffers), so PCIe in, PCIe out and the transform overlap.  Returns when
        the work is enqueued; the caller's current stream waits for every copy
        back (synchronize it before reading host_out)."""
        import torch

        with torch.cuda.device(self.device):
            self._pairs_pipelined(host_in, host_out)

    def _pairs_pipelined(self, host_in, host_out) -> None:
        import torch

        dev = self.device
        if getattr(self, "_pipe", None) is None:
            mk = lambda n: torch.empty((self.nfld, n), dtype=torch.float64, device=dev)  # noqa: E731
            self._pipe = {"din": [mk(self.nspec_local) for _ in range(2)],
                          "dout": [mk(self.nspec_local) for _ in range(2)], "grid": mk(self.npts_local),
                          "h2d": torch.cuda.Stream(dev), "d2h": torch.cuda.Stream(dev)}
        P = self._pipe
        cs = torch.cuda.current_stream(dev)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        P["h2d"].wait_stream(cs)
        P["d2h"].wait_stream(cs)
        for i, (hi, ho) in enumerate(zip(host_in, host_out)):
            b = i % 2
            if i >= 2:
                P["h2d"].wait_event(ev_done[b])   # batch i-2 no longer reads din[b]
            with torch.cuda.stream(P["h2d"]):
                P["din"][b].copy_(hi, non_blocking=True)
            ev_in[b].record(P["h2d"])
            cs.wait_event(ev_in[b])
            if i >= 2:
                cs.wait_event(ev_out[b])          # batch i-2's result has left dout[b]
            self.inv_trans(P["din"][b], out=P["grid"])
            self.dir_trans(P["grid"], out=P["dout"][b])
            ev_done[b].record(cs)
            P["d2h"].wait_event(ev_done[b])
            with torch.cuda.stream(P["d2h"]):
                ho.copy_(P["dout"][b], non_blocking=True)
            ev_out[b].record(P["d2h"])
        cs.wait_stream(P["d2h"])

    def close(self) -> None:
        """Release the plan.  Collective when the plan spans several ranks (a
        bounded barrier, so no peer still stores into this rank's buffers);
        raises ``ProtocolError`` if a peer does not arrive."""
        import torch

        self._pipe = None
        plan, self._plan = getattr(self, "_plan", None), None
        if plan:
            with torch.cuda.device(self.device):
                _lib.check(self._lib.sht_plan_close(plan))

    def __del__(self):
        # local release only: a collective in a destructor hangs every peer
        # when one rank raised or never collects its plan
        plan = getattr(self, "_plan", None)
        if not plan:
            return
        self._plan = None
        try:
            if self.nranks > 1:
                import warnings

                warnings.warn("SHTransform spanning several ranks was not close()d; releasing it locally",
                              ResourceWarning)
            import torch

            with torch.cuda.device(self.device):
                self._lib.sht_plan_destroy(plan)
        except Exception:
            pass


def gauss_nodes(ndgl: int):
    """Northern Gaussian nodes (mu, cos(lat), w) as computed by the plan (host-only call)."""
    lib = _lib.load()
    nh = int(ndgl) // 2
    mu, s, w = np.empty(nh), np.empty(nh), np.empty(nh)
    _lib.check(lib.sht_gauss_nodes(int(ndgl), mu.ctypes.data_as(_lib.f64p), s.ctypes.data_as(_lib.f64p),
                                   w.ctypes.data_as(_lib.f64p)))
    return mu, s, w


def partition(truncation: int, nranks: int, grid="octahedral"):
    """(m_owner[T+1], ring_owner[NDGL/2]) the plan uses for ``nranks`` ranks (host-only call)."""
    lib = _lib.load()
    T = int(truncation)
    if isinstance(grid, str):
        nloen_p, ndgl = None, 2 * (T + 1)
    else:
        arr = np.ascontiguousarray(np.asarray(grid, dtype=np.int32))
        nloen_p, ndgl = arr.ctypes.data_as(_lib.i32p), int(arr.size)
    mo = np.empty(T + 1, dtype=np.int32)
    ro = np.empty(ndgl // 2, dtype=np.int32)
    _lib.check(lib.sht_partition(T, ndgl, nloen_p, int(nranks), mo.ctypes.data_as(_lib.i32p),
                                 ro.ctypes.data_as(_lib.i32p)))
    return mo, ro


def _nloen_arg(truncation: int, grid):
    T = int(truncation)
    if isinstance(grid, str):
        return None, 2 * (T + 1), None
    arr = np.ascontiguousarray(np.asarray(grid, dtype=np.int32))
    return arr.ctypes.data_as(_lib.i32p), int(arr.size), arr


def plan_validate(truncation: int, nfld: int, nranks: int = 1, grid="octahedral") -> None:
    """Build every rank's plan tables on the host (no GPU); raise ConfigurationError if unsupported."""
    lib = _lib.load()
    ptr, ndgl, _keep = _nloen_arg(truncation, grid)
    _lib.check(lib.sht_plan_validate(int(truncation), ndgl, ptr, int(nfld), int(nranks)))


def alltoall_rows(truncation: int, nranks: int, grid="octahedral") -> np.ndarray:
    """[P, P] Fourier rows rank r sends to rank d in the inverse transposition (host-only call).

    Multiply by 32 * nfld for bytes: this is the ``sizes`` matrix of the
    reference's ``collectives.build_alltoall`` (collectives.py:96) for this path.
    """
    lib = _lib.load()
    ptr, ndgl, _keep = _nloen_arg(truncation, grid)
    P = int(nranks)
    rows = np.empty(P * P, dtype=np.int64)
    _lib.check(lib.sht_alltoall_rows(int(truncation), ndgl, ptr, P, rows.ctypes.data_as(_lib.i64p)))
    return rows.reshape(P, P)


def alltoall_order(nranks: int, rank: int) -> list:
    """Peers in the order rank ``rank`` issues its transfers (rotated, collectives.py:85-86)."""
    lib = _lib.load()
    out = np.empty(int(nranks), dtype=np.int32)
    _lib.check(lib.sht_alltoall_order(int(nranks), int(rank), out.ctypes.data_as(_lib.i32p)))
    return [int(x) for x in out]


def fft_plan_info(n: int) -> dict:
    lib = _lib.load()
    rad = (C.c_int32 * 32)()
    ns, L, blue = C.c_int32(), C.c_int32(), C.c_int32()
    _lib.check(lib.sht_fft_plan_info(int(n), rad, C.byref(ns), C.byref(L), C.byref(blue)))
    return {"radices": list(rad[: ns.value]), "length": L.value, "bluestein": bool(blue.value)}
