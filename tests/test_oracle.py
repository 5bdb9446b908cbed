"""The CPU oracle pinned to analytic known answers, scipy and its golden fixtures.

The transform has no reference implementation,
so parity is anchored on (a) the analytic KATs of SURVEY.md App. A, (b)
orthonormality of the discrete Legendre operator on the Gauss grid, (c)
scipy.special as an independent implementation of the Gauss rule and of the
normalised associated Legendre functions, and (d) dir(inv(a)) = a.
"""

from pathlib import Path

import numpy as np
import pytest
import scipy.special as sp

from oracle.sht_oracle import (SHTransformOracle, gauss_nodes, legendre_diag, legendre_m, octahedral_nloen,
                               random_grid, random_spectral, ring_mcap)

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def o79():
    return SHTransformOracle(79, nfld=4)


def test_grid_geometry():
    nl = octahedral_nloen(79)
    assert nl.size == 160 and nl[0] == 20 and nl[79] == 336 and np.array_equal(nl, nl[::-1])
    assert int(nl.sum()) == 28480
    assert int(octahedral_nloen(639).sum()) == 1661440
    m = ring_mcap(639, octahedral_nloen(639))
    assert m[0] == 9 and m.max() == 639


@pytest.mark.parametrize("ndgl", [2, 16, 160, 320, 1280])
def test_gauss_nodes_vs_scipy(ndgl):
    mu, s, w = gauss_nodes(ndgl)
    x, ws = sp.roots_legendre(ndgl)
    nh = ndgl // 2
    assert np.max(np.abs(mu - x[::-1][:nh])) <= 4e-16
    # scipy's polar weights are only ~1e-10 accurate (checked against mpmath below)
    assert np.max(np.abs(w - ws[::-1][:nh]) / ws[::-1][:nh]) <= 1e-7
    assert abs(2 * w.sum() - 2.0) <= 1e-14
    assert np.max(np.abs(mu * mu + s * s - 1.0)) <= 4e-16


@pytest.mark.parametrize("ndgl", [16, 320])
def test_gauss_weights_vs_mpmath(ndgl):
    mpmath = pytest.importorskip("mpmath")
    mpmath.mp.dps = 40
    mu, _, w = gauss_nodes(ndgl)

    def pn(t):
        p0, p1 = mpmath.mpf(1), t
        for j in range(2, ndgl + 1):
            p0, p1 = p1, ((2 * j - 1) * t * p1 - (j - 1) * p0) / j
        return p1, p0

    for j in sorted({0, 1, ndgl // 4, ndgl // 2 - 1}):
        x = mpmath.mpf(mu[j])
        for _ in range(6):
            a, b = pn(x)
            x = x - a / (ndgl * (x * a - b) / (x * x - 1))
        a, b = pn(x)
        wr = 2 / ((1 - x * x) * (ndgl * (x * a - b) / (x * x - 1)) ** 2)
        assert abs(float(mpmath.mpf(mu[j]) - x)) <= 1.2e-16
        assert abs(float((mpmath.mpf(w[j]) - wr) / wr)) <= 1e-12


def test_legendre_vs_scipy():
    T = 40
    mu, s, _ = gauss_nodes(2 * T + 2)
    mant, expo = legendre_diag(T, s)
    ref = sp.assoc_legendre_p_all(T, T, mu, norm=True)[0]   # [n, m, ring], orthonormal, includes (-1)^m
    for m in range(T + 1):
        P = legendre_m(T, m, mu, mant[m], expo[m])           # [ring, n-m]
        r = ref[m:, m, :].T * (-1.0) ** m                      # drop the Condon-Shortley phase
        assert np.max(np.abs(P - r)) <= 1e-13 * max(1.0, np.max(np.abs(r)))


def test_xnumber_recurrence_no_underflow():
    # TCo1999-size start values underflow double without the exponent
    T = 1999
    mu, s, _ = gauss_nodes(4000)
    mant, expo = legendre_diag(T, s[:50])
    assert np.all(mant[T] > 0) and expo[T].min() < -1000
    P = legendre_m(T, 735, mu[:50], mant[735], expo[735])
    assert np.all(np.isfinite(P))


def test_kats(o79):
    o = o79
    spec = np.zeros((4, o.nspec))
    spec[0, 0] = 1.0                       # a_0^0 = 1       -> 1/sqrt(2)
    spec[1, 2] = 1.0                       # a_1^0 = 1       -> sqrt(3/2) mu
    spec[2, 2 * o.soff[1]] = 1.0           # a_1^1 = 1       -> sqrt(3) cos(lat) cos(lon)
    spec[3, 2 * o.soff[1] + 1] = 1.0       # a_1^1 = i       -> -sqrt(3) cos(lat) sin(lon)
    g = o.inv_trans(spec)
    mu = np.repeat(np.concatenate([o.mu, -o.mu[::-1]]), o.nloen)
    cl = np.repeat(np.concatenate([o.sint, o.sint[::-1]]), o.nloen)
    lam = np.concatenate([2 * np.pi * np.arange(n) / n for n in o.nloen])
    assert np.max(np.abs(g[0] - 1 / np.sqrt(2))) <= 1e-15
    assert np.max(np.abs(g[1] - np.sqrt(1.5) * mu)) <= 1e-14
    assert np.max(np.abs(g[2] - np.sqrt(3) * cl * np.cos(lam))) <= 1e-14
    assert np.max(np.abs(g[3] + np.sqrt(3) * cl * np.sin(lam))) <= 1e-14
    back = o.dir_trans(g)
    assert np.max(np.abs(back - spec)) <= 1e-13


def test_orthonormality(o79):
    o = o79
    worst = 0.0
    for m in range(o.T + 1):
        i0, P = o.tables[m]
        G = 2 * (P.T * o.w[i0:]) @ P
        K = o.T - m + 1
        par = (np.arange(K)[:, None] + np.arange(K)[None, :]) % 2
        G[par == 1] = 0.0
        worst = max(worst, float(np.abs(G - np.eye(K)).max()))
    assert worst <= 5e-12          # limited by double-rounded nodes (n^2 * 1e-16)


@pytest.mark.parametrize("T", [15, 79])
def test_roundtrip(T):
    o = SHTransformOracle(T, nfld=3)
    a = random_spectral(T, 3)
    b = o.dir_trans(o.inv_trans(a))
    assert np.max(np.abs(b - a)) / np.max(np.abs(a)) <= 1e-11


def test_linearity(o79):
    o = o79
    a, b = random_spectral(79, 4, seed=1), random_spectral(79, 4, seed=2)
    lhs = o.inv_trans(2.0 * a - b)
    rhs = 2.0 * o.inv_trans(a) - o.inv_trans(b)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(lhs))


@pytest.mark.parametrize("name,T,nfld", [("tco79_f4", 79, 4), ("tco15_f3", 15, 3)])
def test_golden(name, T, nfld):
    d = np.load(GOLD / f"{name}.npz")
    o = SHTransformOracle(T, nfld=nfld)
    assert np.array_equal(d["spec"], random_spectral(T, nfld))
    assert np.array_equal(d["grid"], random_grid(T, nfld, o.npts))
    assert np.max(np.abs(o.inv_trans(d["spec"]) - d["inv"])) <= 1e-13 * np.abs(d["inv"]).max()
    assert np.max(np.abs(o.dir_trans(d["grid"]) - d["dir"])) <= 1e-13 * np.abs(d["dir"]).max()


def test_custom_grid_regular_gaussian():
    # full (regular) Gaussian grid: every ring has 2T+2 points, caps all equal T
    T = 21
    nloen = np.full(2 * (T + 1), 2 * T + 2)
    o = SHTransformOracle(T, grid=nloen, nfld=2)
    a = random_spectral(T, 2)
    assert np.max(np.abs(o.dir_trans(o.inv_trans(a)) - a)) <= 1e-12


def test_bad_grid():
    with pytest.raises(ValueError):
        SHTransformOracle(10, grid=np.array([20, 24, 20]), nfld=1)


# ---------------------------------------------------------------- brute-force pins (no FFT, no recurrence)
from oracle.brute import brute_analysis, brute_synthesis  # noqa: E402


@pytest.mark.parametrize("T", [23, 31])
def test_oracle_vs_brute_force(T):
    """The oracle's inverse and direct transforms equal pointwise synthesis / quadrature by explicit
    sums over all (n, m) with scipy's Pbar -- no FFT and no shared recurrence (pins the conventions
    beyond the l <= 1 KATs)."""
    o = SHTransformOracle(T, nfld=3)
    mu, _, w = gauss_nodes(2 * T + 2)
    mu_all = np.concatenate([mu, -mu[::-1]])
    w_all = np.concatenate([w, w[::-1]])
    a = random_spectral(T, 3, seed=7)
    g = random_grid(T, 3, o.npts, seed=8)
    fb = brute_synthesis(T, a, o.nloen, mu_all)
    assert np.max(np.abs(o.inv_trans(a) - fb)) <= 1e-12 * np.max(np.abs(fb))
    sb = brute_analysis(T, g, o.nloen, mu_all, w_all)
    assert np.max(np.abs(o.dir_trans(g) - sb)) <= 1e-12 * np.max(np.abs(sb))


def test_oracle_m_subset_matches_full():
    """m_subset restricts the oracle to a few wavenumbers (the TCo1999 parity tests use it)."""
    T, S = 47, [0, 1, 5, 30, 47]
    full = SHTransformOracle(T, nfld=2)
    sub = SHTransformOracle(T, nfld=2, m_subset=S)
    a = random_spectral(T, 2, seed=3)
    soff = np.arange(T + 2) * (2 * T - np.arange(T + 2) + 3) // 2
    keep = np.zeros(a.shape[1], dtype=bool)
    for m in S:
        keep[2 * soff[m]: 2 * soff[m + 1]] = True
    a[:, ~keep] = 0.0
    assert np.max(np.abs(sub.inv_trans(a) - full.inv_trans(a))) <= 1e-15 * np.max(np.abs(full.inv_trans(a)))
    g = random_grid(T, 2, full.npts, seed=4)
    ds, df = sub.dir_trans(g), full.dir_trans(g)
    assert np.array_equal(ds[:, keep], df[:, keep]) and not ds[:, ~keep].any()
