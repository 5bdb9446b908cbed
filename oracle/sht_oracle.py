"""CPU ORACLE for the spherical-harmonics transform step -- TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import it.  The product path
(``paper_1908_06097_b200``) never imports anything under ``oracle/``.

What it restates
----------------
The north star (BASELINE.json) names "the CPU reference's Python transform
API (setup with truncation, grid and field count; inv_trans/dir_trans on
field batches)".  That API does not exist in /root/reference: the reference
package (``haloflow``) explicitly puts "spectral-transform ... numerical
mathematics" OUT OF SCOPE and only *models* the
SH dwarf's all-to-all transposition (collectives.py:96-117, netsim.py:347-398).
The transform mathematics therefore follows SURVEY.md Appendix A (the IFS /
ecTrans conventions of the ESCAPE SH dwarf described at
/root/reference/PAPER.md:193-199), restated here from scratch in NumPy:

* octahedral TCo grid: NH = T+1 rings per hemisphere, ring i (1-based, pole
  to equator) has 4i+16 points (SURVEY.md App. A "Grid");
* Gaussian latitudes by Newton iteration (App. A; SURVEY.md section 7 shows
  ``numpy.polynomial.legendre.leggauss`` is not accurate enough for NDGL>=160);
* orthonormal associated Legendre functions, no Condon-Shortley phase, with
  an X-number (mantissa, base-2 exponent) recurrence so TCo1999 does not
  underflow (App. A; SURVEY.md section 7 "Legendre recurrence range");
* per-ring wavenumber cap M_i = min(T, floor((N_i-1)/2));
* spectral storage: m-major, n ascending, re/im interleaved, length (T+1)(T+2);
* inverse: F_m(mu_j) = sum_n a_n^m P_n^m(mu_j), f = Re F_0 + 2 sum_m Re(F_m e^{i m lambda});
* direct:  F_m = (1/N) sum_k f_k e^{-i m lambda_k}, a_n^m = sum_j w_j P_n^m(mu_j) F_m(mu_j).

Parity status: the transform has NO reference implementation, so the oracle
is pinned by (a) analytic known-answer tests (Y_0^0, Y_1^0, Y_1^1), (b)
orthonormality of the discrete Legendre operator on the Gauss grid, (c)
``scipy.special`` (an independent implementation) for Gauss nodes/weights and
normalised associated Legendre values, and (d) the dir(inv(a)) = a round trip.
The golden fixtures under tests/golden/ are generated from this module by
tests/golden/make_golden.py.  "Parity pinned to analytic KATs + scipy; no
reference transform exists" is what DESIGN.md states.
"""

from __future__ import annotations

import os

import numpy as np
import scipy.fft as _sfft

__all__ = [
    "octahedral_nloen",
    "ring_mcap",
    "gauss_nodes",
    "legendre_diag",
    "legendre_table",
    "spec_offsets",
    "nspec_real",
    "ring_offsets",
    "SHTransformOracle",
    "random_spectral",
    "random_grid",
]

_TWO400 = 2.0 ** 400
_TWOM400 = 2.0 ** -400


# --------------------------------------------------------------------------- grid


def octahedral_nloen(T: int) -> np.ndarray:
    """Ring lengths of the octahedral TCo grid, all NDGL = 2(T+1) rings, north first.

    SURVEY.md App. A: northern ring i = 1..NH has 4i+16 points; the southern
    ring NDGL+1-i mirrors it.
    """
    nh = T + 1
    north = 4 * np.arange(1, nh + 1, dtype=np.int64) + 16
    return np.concatenate([north, north[::-1]])


def ring_mcap(T: int, nloen: np.ndarray) -> np.ndarray:
    """Per-ring wavenumber cap M_j = min(T, floor((N_j - 1)/2)) (never the Nyquist mode)."""
    nloen = np.asarray(nloen, dtype=np.int64)
    return np.minimum(T, (nloen - 1) // 2)


def ring_offsets(nloen: np.ndarray) -> np.ndarray:
    """Start of each ring in the flattened grid (length NDGL+1, last = NPTS)."""
    return np.concatenate([[0], np.cumsum(np.asarray(nloen, dtype=np.int64))])


def gauss_nodes(ndgl: int, iters: int = 8):
    """Northern-hemisphere Gaussian nodes by Newton iteration on theta.

    Returns (mu, sintheta, w) as float64 for the NH = ndgl/2 northern rings
    ordered pole to equator (mu descending).  Newton runs in x87 extended
    precision (``np.longdouble``; the C++ plan does the same in ``long
    double`` with the identical operation order) on the colatitude theta with
    f(theta) = P_ndgl(cos theta), f'(theta) = -sin(theta) P'_ndgl(cos theta),
    starting from theta_k = pi(4k-1)/(4 ndgl + 2).  The
    result is rounded once to double.  Working in extended precision matters:
    a 1-ulp node shift moves P_n^m by ~n^2 * 1e-16, i.e. ~4e-11 at TCo639,
    which would eat most of the 1e-10 parity budget if the GPU plan and the
    oracle rounded their nodes differently.
    Weights w = 2 sin^2(theta) / (ndgl P_{ndgl-1}(mu))^2 (= 2/((1-mu^2) P'^2) at a root).
    """
    if ndgl < 2 or ndgl % 2:
        raise ValueError("ndgl must be even and >= 2")
    n = ndgl
    LD = np.longdouble
    nld = LD(n)
    k = np.arange(1, n // 2 + 1).astype(LD)
    pi = LD("3.14159265358979323846264338327950288")
    theta = pi * (LD(4) * k - LD(1)) / (LD(4) * nld + LD(2))

    def pn(x):
        p0 = np.ones_like(x)
        p1 = x.copy()
        for j in range(2, n + 1):
            jl = LD(j)
            p0, p1 = p1, ((LD(2) * jl - LD(1)) * x * p1 - (jl - LD(1)) * p0) / jl
        return p1, p0

    for _ in range(iters):
        x = np.cos(theta)
        s = np.sin(theta)
        p1, p0 = pn(x)
        dp = nld * (x * p1 - p0) / (x * x - LD(1))
        theta = theta + p1 / (s * dp)
    x = np.cos(theta)
    s = np.sin(theta)
    _, p0 = pn(x)
    w = LD(2) * s * s / ((nld * p0) * (nld * p0))
    return x.astype(np.float64), s.astype(np.float64), w.astype(np.float64)


# --------------------------------------------------------------------- Legendre


def legendre_diag(T: int, sint: np.ndarray):
    """Sectoral values P_m^m for m = 0..T as X-numbers (mant[m, i], expo[m, i]).

    P_0^0 = 1/sqrt(2); P_m^m = sqrt((2m+1)/(2m)) sin(theta) P_{m-1}^{m-1}.
    The mantissa is renormalised by 2^400 whenever it falls below 2^-400
    (SURVEY.md App. A X-number rule), so nothing underflows before the
    n-recurrence has grown the value back into range.
    """
    sint = np.asarray(sint, dtype=np.float64)
    mant = np.empty((T + 1, sint.size))
    expo = np.zeros((T + 1, sint.size), dtype=np.int64)
    cur = np.full(sint.size, 1.0 / np.sqrt(2.0))
    e = np.zeros(sint.size, dtype=np.int64)
    mant[0] = cur
    for m in range(1, T + 1):
        cur = cur * (np.sqrt((2.0 * m + 1.0) / (2.0 * m)) * sint)
        small = cur < _TWOM400
        cur = np.where(small, cur * _TWO400, cur)
        e = np.where(small, e - 400, e)
        mant[m] = cur
        expo[m] = e
    return mant, expo


def _eps(n: np.ndarray | float, m: int):
    n = np.asarray(n, dtype=np.float64)
    return np.sqrt((n * n - m * m) / (4.0 * n * n - 1.0))


def legendre_m(T: int, m: int, mu: np.ndarray, mant_mm: np.ndarray, expo_mm: np.ndarray) -> np.ndarray:
    """P_n^m(mu_i) for n = m..T on the given rings -> array [ring, n-m].

    Three-term recurrence in n on the mantissa with a shared per-ring
    exponent; the mantissa pair is renormalised by 2^-400 when it exceeds
    2^400 and values are emitted with ldexp.
    """
    mu = np.asarray(mu, dtype=np.float64)
    nr = mu.size
    K = T - m + 1
    out = np.empty((nr, K))
    e = np.array(expo_mm, dtype=np.int64)
    q2 = np.array(mant_mm, dtype=np.float64)          # P_m^m mantissa
    out[:, 0] = np.ldexp(q2, e)
    if K == 1:
        return out
    q1 = np.sqrt(2.0 * m + 3.0) * mu * q2              # P_{m+1}^m
    out[:, 1] = np.ldexp(q1, e)
    for n in range(m + 2, T + 1):
        q = (mu * q1 - _eps(n - 1, m) * q2) / _eps(n, m)
        big = np.abs(q) > _TWO400
        if big.any():
            q = np.where(big, q * _TWOM400, q)
            q1 = np.where(big, q1 * _TWOM400, q1)
            e = np.where(big, e + 400, e)
        q2, q1 = q1, q
        out[:, n - m] = np.ldexp(q, e)
    return out


def legendre_table(T: int, mu: np.ndarray, sint: np.ndarray, mcap_north: np.ndarray, m_subset=None):
    """All P_n^m on the northern rings that need them.

    Returns a list over m of (i0, P) where rings i0..NH-1 are the rings with
    M_i >= m (M is non-decreasing toward the equator) and P has shape
    [NH - i0, T - m + 1].  With ``m_subset`` only those wavenumbers get a
    table (the others are None): a TCo1999 table is 27 GB, a few m are not.
    """
    mant, expo = legendre_diag(T, sint)
    tables = []
    for m in range(T + 1):
        if m_subset is not None and m not in m_subset:
            tables.append(None)
            continue
        i0 = int(np.searchsorted(mcap_north, m, side="left"))
        tables.append((i0, legendre_m(T, m, mu[i0:], mant[m, i0:], expo[m, i0:])))
    return tables


# ---------------------------------------------------------------- spectral layout


def spec_offsets(T: int) -> np.ndarray:
    """Complex offset of (m, n=m) for m = 0..T+1: m(2T - m + 3)/2."""
    m = np.arange(T + 2, dtype=np.int64)
    return m * (2 * T - m + 3) // 2


def nspec_real(T: int) -> int:
    return (T + 1) * (T + 2)


def random_spectral(T: int, nfld: int, seed: int | None = None) -> np.ndarray:
    """Seeded synthetic spectral fields [nfld, (T+1)(T+2)].

    a = (g1 + i g2)/sqrt(2), g ~ N(0,1), PCG64 ``default_rng(seed=T)``; Im a_n^0 = 0.
    """
    rng = np.random.default_rng(T if seed is None else seed)
    ncplx = (T + 1) * (T + 2) // 2
    a = rng.standard_normal((nfld, ncplx, 2)) / np.sqrt(2.0)
    a[:, : T + 1, 1] = 0.0
    return a.reshape(nfld, 2 * ncplx)


def random_grid(T: int, nfld: int, npts: int, seed: int | None = None) -> np.ndarray:
    """Seeded synthetic grid fields [nfld, npts], N(0,1), ``default_rng(seed=T+1)``."""
    rng = np.random.default_rng(T + 1 if seed is None else seed)
    return rng.standard_normal((nfld, npts))


# ---------------------------------------------------------------- the transform


class SHTransformOracle:
    """CPU restatement of the SH transform API: setup(truncation, grid, nfld), inv/dir.

    ``grid`` is "octahedral" (TCo) or an explicit array of NDGL ring lengths
    (north first, north/south symmetric).
    """

    def __init__(self, truncation: int, grid="octahedral", nfld: int = 1, workers: int | None = None,
                 m_subset=None):
        T = int(truncation)
        self.workers = int(workers) if workers else (os.cpu_count() or 1)
        if T < 1:
            raise ValueError("truncation must be >= 1")
        self.T = T
        self.nfld = int(nfld)
        if isinstance(grid, str):
            if grid != "octahedral":
                raise ValueError(f"unknown grid {grid!r}")
            nloen = octahedral_nloen(T)
        else:
            nloen = np.asarray(grid, dtype=np.int64)
        self.nloen = nloen
        self.ndgl = nloen.size
        if self.ndgl % 2 or not np.array_equal(nloen, nloen[::-1]):
            raise ValueError("grid must have an even, north/south-symmetric ring list")
        self.nh = self.ndgl // 2
        self.mcap = ring_mcap(T, nloen)
        if np.any(np.diff(self.mcap[: self.nh]) < 0):
            raise ValueError("ring lengths must be non-decreasing from pole to equator")
        self.roff = ring_offsets(nloen)
        self.npts = int(self.roff[-1])
        self.mu, self.sint, self.w = gauss_nodes(self.ndgl)
        # m_subset: restrict the transform to these zonal wavenumbers (inv_trans
        # ignores the other coefficients, dir_trans returns zeros for them)
        self.m_subset = None if m_subset is None else {int(m) for m in m_subset}
        self.tables = legendre_table(T, self.mu, self.sint, self.mcap[: self.nh], self.m_subset)
        self.soff = spec_offsets(T)
        self.nspec = nspec_real(T)

    # -- helpers ---------------------------------------------------------------
    def _fourier_inv(self, spec: np.ndarray):
        """Legendre synthesis: Fourier coefficients per ring, list of [nfld, M_j+1] complex.

        Per m the S (even n-m) and A (odd n-m) sums are real GEMMs over the
        re/im-interleaved coefficients; F_north = S + A, F_south = S - A.
        """
        T, nh, nf = self.T, self.nh, self.nfld
        four = [np.zeros((nf, int(self.mcap[j]) + 1), dtype=np.complex128) for j in range(self.ndgl)]
        for m in range(T + 1):
            if self.tables[m] is None:
                continue
            i0, P = self.tables[m]
            if i0 >= nh:
                continue
            K = T - m + 1
            am = spec[:, 2 * self.soff[m]: 2 * self.soff[m + 1]].reshape(nf, K, 2)
            bs = am[:, 0::2, :].transpose(1, 0, 2).reshape(-1, 2 * nf)       # [K_S, nfld*2]
            ba = am[:, 1::2, :].transpose(1, 0, 2).reshape(-1, 2 * nf)
            S = (P[:, 0::2] @ bs).reshape(-1, nf, 2)                          # [rings, nfld, 2]
            A = (P[:, 1::2] @ ba).reshape(-1, nf, 2)
            fn = (S + A)[..., 0] + 1j * (S + A)[..., 1]
            fs = (S - A)[..., 0] + 1j * (S - A)[..., 1]
            for r, i in enumerate(range(i0, nh)):
                four[i][:, m] = fn[r]
                four[self.ndgl - 1 - i][:, m] = fs[r]
        return four

    def inv_trans(self, spec: np.ndarray) -> np.ndarray:
        """Spectral [nfld, (T+1)(T+2)] -> grid [nfld, NPTS] (float64)."""
        spec = np.asarray(spec, dtype=np.float64).reshape(self.nfld, self.nspec)
        four = self._fourier_inv(spec)
        grid = np.empty((self.nfld, self.npts))
        for j in range(self.ndgl):
            n = int(self.nloen[j])
            c = np.zeros((self.nfld, n // 2 + 1), dtype=np.complex128)
            c[:, : four[j].shape[1]] = four[j]
            grid[:, self.roff[j]: self.roff[j + 1]] = _sfft.irfft(c, n=n, axis=1, workers=self.workers) * n
        return grid

    def fourier_dir(self, grid: np.ndarray):
        """Ring DFTs: list over rings of [nfld, M_j+1] complex, scaled 1/N_j."""
        out = []
        for j in range(self.ndgl):
            n = int(self.nloen[j])
            z = _sfft.rfft(grid[:, self.roff[j]: self.roff[j + 1]], axis=1, workers=self.workers) / n
            out.append(z[:, : int(self.mcap[j]) + 1])
        return out

    def dir_trans(self, grid: np.ndarray) -> np.ndarray:
        """Grid [nfld, NPTS] -> spectral [nfld, (T+1)(T+2)] (float64)."""
        grid = np.asarray(grid, dtype=np.float64).reshape(self.nfld, self.npts)
        four = self.fourier_dir(grid)
        T, nh, nf = self.T, self.nh, self.nfld
        spec = np.zeros((nf, self.nspec))
        for m in range(T + 1):
            if self.tables[m] is None:
                continue
            i0, P = self.tables[m]
            if i0 >= nh:
                continue
            K = T - m + 1
            fn = np.stack([four[i][:, m] for i in range(i0, nh)])                 # [rings, nfld]
            fs = np.stack([four[self.ndgl - 1 - i][:, m] for i in range(i0, nh)])
            w = self.w[i0:nh, None]
            gs, ga = w * (fn + fs), w * (fn - fs)
            gs = np.stack([gs.real, gs.imag], axis=-1).reshape(-1, 2 * nf)        # [rings, nfld*2]
            ga = np.stack([ga.real, ga.imag], axis=-1).reshape(-1, 2 * nf)
            out = np.empty((K, nf, 2))
            out[0::2] = (P[:, 0::2].T @ gs).reshape(-1, nf, 2)
            out[1::2] = (P[:, 1::2].T @ ga).reshape(-1, nf, 2)
            spec[:, 2 * self.soff[m]: 2 * self.soff[m + 1]] = out.transpose(1, 0, 2).reshape(nf, 2 * K)
        return spec
