"""CPU restatement of the distributed data path -- TEST INFRASTRUCTURE ONLY.

Restates, independently of libsht's C++ plan (paper_1908_06097_b200/csrc/
sht_plan.cu), how the transform is sharded over P ranks and how the
grid <-> spectral transposition moves Fourier rows, so the CPU test-suite can
check the partition, the size matrix and the pack/unpack index math without a
GPU, in process (the reference's oracle-equivalence pattern,
/root/reference/pkg/tests/test_acceptance.py:60-80: a P-rank run must equal
the 1-rank oracle) and across real processes over gloo.

* Ownership: snake (boustrophedon) dealing of the zonal wavenumbers m
  (SURVEY.md section 8e); the northern ring pairs i go longest-first to the
  least-loaded rank under a ring-FFT cost model (ring_fft_cost below).
* Issue order: rank r sends to (r + k) % P for k = 0..P-1, the reference's
  ROTATED_CONCURRENT schedule (/root/reference/pkg/src/haloflow/
  collectives.py:85-86).
* Fourier rows: one row per (ring pair i, m <= M_i) holding nfld x
  (S.re, S.im, A.re, A.im); rank r's send block for rank d lists d's rings
  ascending and, per ring, r's wavenumbers ascending.
"""

from __future__ import annotations

import numpy as np

from .sht_oracle import SHTransformOracle


def snake(n: int, P: int) -> np.ndarray:
    k = np.arange(n)
    blk, pos = k // P, k % P
    return np.where(blk % 2 == 0, pos, P - 1 - pos).astype(np.int64)


def _factor(n: int, maxp: int):
    primes, m, p = [], n, 2
    while p <= maxp and m > 1:
        while m % p == 0:
            primes.append(p)
            m //= p
        p += 1
    return primes, m == 1


def _pencils(primes):
    """Pencil radices: primes > 16 alone, the rest first-fit-decreasing into factors <= 16."""
    big = [p for p in primes if p > 16]
    bins = []
    for p in sorted((p for p in primes if p <= 16), reverse=True):
        for j, b in enumerate(bins):
            if b * p <= 16:
                bins[j] = b * p
                break
        else:
            bins.append(p)
    return big + bins


_CODELET = {2: 4, 3: 12, 4: 16, 5: 36, 6: 44, 7: 66, 8: 55, 9: 88, 10: 108, 11: 150, 12: 128, 13: 204, 14: 184,
            15: 200, 16: 165}


def _bluestein_cost(L: int, rad) -> int:
    c = 0
    for j, R in enumerate(rad):
        pen = L // R
        c += pen * (2 * _CODELET[R] + 16 * R)
        if j < len(rad) - 1:
            c += pen * 2 * (8 * R - 8)
    return c


def _bluestein_len(lo: int, lmax: int = 1 << 30):
    """Least modelled-cost 13-smooth length in [lo, min(lmax, 1.5 lo)] with <= 4 pencil steps,
    else the shortest up to min(lmax, 4 lo + 64) (libsht's fft_bluestein_len)."""
    best = None
    for cand in range(lo, min(lmax, lo + lo // 2) + 1):
        primes, ok = _factor(cand, 13)
        if ok:
            rad = _pencils(primes)
            if len(rad) <= 4:
                c = _bluestein_cost(cand, rad)
                if best is None or c < best[0]:
                    best = (c, cand, rad)
    if best is not None:
        return best[1], best[2]
    for cand in range(lo, min(lmax, 4 * lo + 64) + 1):
        primes, ok = _factor(cand, 13)
        if ok and len(_pencils(primes)) <= 4:
            return cand, _pencils(primes)
    return -1, []


def ring_fft_cost(n: int, mcap: int) -> int:
    """Cost of one ring pair's FFTs per field: 3 per element-step + grid and row bytes.

    Plans (libsht's fft_plan_ring): pencils <= 16 plus at most one prime 17..127 as a DMMA
    prime step (~p/16 element-steps per point), <= 4 steps; else whole-ring Bluestein (pruned for
    even n) when it fits one CTA, else factor-local Bluestein steps (~6 extra element-steps)."""
    primes, _ = _factor(n, n)
    small = [p for p in primes if p <= 16]
    mid = [p for p in primes if 16 < p <= 127]
    big = [p for p in primes if p > 127]
    if not big and len(mid) <= 1:
        rad = _pencils(small) + mid
        if not rad:
            rad = [n]
        if len(rad) <= 4 and (not mid or len(rad) >= 2):
            dp = mid[0] if mid else 0
            return 3 * n * (len(rad) + dp // 16) + 16 * n + 32 * (mcap + 1)
    # whole-ring Bluestein; even n keeping |k| <= mcap needs only n + 2 mcap lags
    pruned = n % 2 == 0 and n + 2 * mcap < 2 * n - 1
    lo = n + 2 * mcap if pruned else 2 * n - 1
    L, rad = _bluestein_len(lo, 6022)
    if L < 0:
        L, rad = _bluestein_len(lo, 12288)
    if 0 < L <= 12288:
        return 3 * 2 * L * len(rad) + 16 * n + 32 * (mcap + 1)
    rad = _pencils(small) + sorted(mid + big)
    return 3 * n * (len(rad) + 6) + 16 * n + 32 * (mcap + 1)


def ring_partition(nloen_north, mcap_north, P: int) -> np.ndarray:
    """Longest-processing-time dealing of the ring pairs over P ranks."""
    cost = [ring_fft_cost(int(n), int(m)) for n, m in zip(nloen_north, mcap_north)]
    order = sorted(range(len(cost)), key=lambda i: (-cost[i], i))
    load = [0] * P
    owner = np.zeros(len(cost), dtype=np.int64)
    for i in order:
        r = min(range(P), key=lambda q: (load[q], q))
        owner[i] = r
        load[r] += cost[i]
    return owner


class Layout:
    """Ownership and row layout of a P-rank plan (restated)."""

    def __init__(self, o: SHTransformOracle, P: int):
        self.o, self.P = o, P
        self.m_owner = snake(o.T + 1, P)
        self.mcap = o.mcap[: o.nh]
        self.ring_owner = ring_partition(o.nloen[: o.nh], self.mcap, P)
        self.M = [np.flatnonzero(self.m_owner == r) for r in range(P)]
        self.R = [np.flatnonzero(self.ring_owner == r) for r in range(P)]

    def rows(self) -> np.ndarray:
        """rows[r, d]: Fourier rows r sends to d in the inverse transposition."""
        P = self.P
        out = np.zeros((P, P), dtype=np.int64)
        for r in range(P):
            for d in range(P):
                out[r, d] = sum(int(np.sum(self.M[r] <= self.mcap[i])) for i in self.R[d])
        return out

    def local_spec(self, spec: np.ndarray, r: int) -> np.ndarray:
        soff = self.o.soff
        return np.concatenate([spec[:, 2 * soff[m]: 2 * soff[m + 1]] for m in self.M[r]], axis=1)

    def local_rings(self, r: int) -> list:
        """Global ring indices in local storage order (north asc, then south mirrors)."""
        north = list(self.R[r])
        return north + [self.o.ndgl - 1 - i for i in reversed(north)]

    def local_grid(self, grid: np.ndarray, r: int) -> np.ndarray:
        roff = self.o.roff
        return np.concatenate([grid[:, roff[j]: roff[j + 1]] for j in self.local_rings(r)], axis=1)

    # -- inverse transform, split at the transposition -------------------------
    def pack_inv(self, spec_local: np.ndarray, r: int) -> list:
        """Legendre side of rank r: per destination d, the flat float64 send block."""
        o, T, nf = self.o, self.o.T, self.o.nfld
        rows = {}  # (i, m) -> [nfld, 4]
        off = 0
        for m in self.M[r]:
            K = T - m + 1
            i0, P = o.tables[m]
            am = spec_local[:, 2 * off: 2 * (off + K)].reshape(nf, K, 2)
            off += K
            if i0 >= o.nh:
                continue
            bs = am[:, 0::2, :].transpose(1, 0, 2).reshape(-1, 2 * nf)
            ba = am[:, 1::2, :].transpose(1, 0, 2).reshape(-1, 2 * nf)
            S = (P[:, 0::2] @ bs).reshape(-1, nf, 2)
            A = (P[:, 1::2] @ ba).reshape(-1, nf, 2)
            for k, i in enumerate(range(i0, o.nh)):
                rows[(i, m)] = np.concatenate([S[k], A[k]], axis=1)  # S.re S.im A.re A.im
        blocks = []
        for d in range(self.P):
            parts = [rows[(i, m)] for i in self.R[d] for m in self.M[r] if m <= self.mcap[i]]
            blocks.append(np.concatenate([p.reshape(-1) for p in parts]) if parts else np.zeros(0))
        return blocks

    def unpack_inv(self, recv: list, r: int) -> np.ndarray:
        """FFT side of rank r: receive blocks (per source s) -> local grid."""
        o, nf = self.o, self.o.nfld
        four = {}
        for s in range(self.P):
            buf = recv[s].reshape(-1, nf, 4)
            k = 0
            for i in self.R[r]:
                for m in self.M[s]:
                    if m <= self.mcap[i]:
                        four[(i, m)] = buf[k]
                        k += 1
            assert k == buf.shape[0]
        cols = []
        for j in self.local_rings(r):
            i = j if j < o.nh else o.ndgl - 1 - j
            sgn = 1.0 if j < o.nh else -1.0
            M = int(self.mcap[i])
            n = int(o.nloen[j])
            c = np.zeros((nf, n // 2 + 1), dtype=np.complex128)
            for m in range(M + 1):
                row = four[(i, m)]
                f = row[:, 0:2] + sgn * row[:, 2:4]
                c[:, m] = f[:, 0] + 1j * f[:, 1]
            cols.append(np.fft.irfft(c, n=n, axis=1) * n)
        return np.concatenate(cols, axis=1)


def emulate_inv(o: SHTransformOracle, spec: np.ndarray, P: int):
    """In-process P-rank inverse transform; returns the list of local grids."""
    lay = Layout(o, P)
    send = [lay.pack_inv(lay.local_spec(spec, r), r) for r in range(P)]
    return [lay.unpack_inv([send[s][r] for s in range(P)], r) for r in range(P)], lay


# ------------------------------------------------------------------ 2-D grid-point layout
def gp_bands(nloen, nA: int):
    """First global ring of every latitude band (+ NDGL): contiguous rings, split where the
    cumulative point count crosses a / nA of the total (libsht's gp_bands)."""
    nloen = [int(n) for n in nloen]
    tot = sum(nloen)
    lo = [len(nloen)] * (nA + 1)
    lo[0] = 0
    cum, a = 0, 1
    for j, n in enumerate(nloen):
        if a >= nA:
            break
        cum += n
        while a < nA and cum * nA >= tot * a:
            lo[a] = j + 1
            a += 1
    return lo


def gp_local(grid: np.ndarray, nloen, rank: int, nA: int, nB: int) -> np.ndarray:
    """Rank a nB + b's grid-point-layout slice of a global grid [nfld, NPTS]: segment b
    (points [floor(N_j b / nB), floor(N_j (b+1) / nB))) of every ring j of band a."""
    nloen = np.asarray(nloen, dtype=np.int64)
    off = np.concatenate([[0], np.cumsum(nloen)])
    lo = gp_bands(nloen, nA)
    a, b = rank // nB, rank % nB
    cols = []
    for j in range(lo[a], lo[a + 1]):
        k0, k1 = nloen[j] * b // nB, nloen[j] * (b + 1) // nB
        cols.append(np.arange(off[j] + k0, off[j] + k1))
    idx = np.concatenate(cols) if cols else np.zeros(0, dtype=np.int64)
    return grid[:, idx]
