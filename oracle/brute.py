"""Brute-force spherical-harmonic synthesis and quadrature -- TEST INFRASTRUCTURE ONLY.

Pins the oracle (and the GPU path directly) beyond the l <= 1 analytic KATs:
every (n, m) term is evaluated pointwise with scipy.special's normalised
associated Legendre functions (Condon-Shortley phase removed), at every ring's
own latitude (south rings at -mu, not through the hemispheric symmetry), and
the Fourier sums are explicit exponential matrices -- no FFT and no shared
recurrence.  O(T^4): for T <= ~40 only.  Conventions: SURVEY.md App. A.
"""

import numpy as np
import scipy.special as sp

def brute_synthesis(T, a, nloen, mu_all):
    """f(lambda_k, mu_j) = sum_m c_m Re(sum_n a_n^m Pbar_n^m(mu_j) e^{i m lambda_k}), pointwise.

    Pbar from scipy.special.assoc_legendre_p_all (normalised, Condon-Shortley
    phase removed) evaluated at every ring's own mu (south rings at -mu, not
    through the hemispheric symmetry), the Fourier sum as an explicit
    exponential matrix: independent of the oracle's recurrence and scipy.fft."""
    nf = a.shape[0]
    soff = np.arange(T + 2) * (2 * T - np.arange(T + 2) + 3) // 2
    ac = a.reshape(nf, -1, 2)[..., 0] + 1j * a.reshape(nf, -1, 2)[..., 1]       # [nf, ncplx]
    Pall = sp.assoc_legendre_p_all(T, T, mu_all, norm=True)[0]                   # [n, m, ring]
    out = []
    for j, N in enumerate(nloen):
        M = min(T, (int(N) - 1) // 2)
        lam = 2 * np.pi * np.arange(N) / N
        F = np.zeros((nf, M + 1), dtype=complex)
        for m in range(M + 1):
            Pm = Pall[m:, m, j] * (-1.0) ** m
            F[:, m] = ac[:, soff[m]: soff[m + 1]] @ Pm
        c = np.full(M + 1, 2.0)
        c[0] = 1.0
        E = np.exp(1j * np.outer(np.arange(M + 1), lam))                           # [M+1, N]
        out.append(np.real((F * c) @ E))
    return np.concatenate(out, axis=1)


def brute_analysis(T, g, nloen, mu_all, w_all):
    """a_n^m = sum_j w_j Pbar_n^m(mu_j) (1/N_j) sum_k f_jk e^{-i m lambda_k}: the quadrature
    adjoint of brute_synthesis, by explicit sums over every ring."""
    nf = g.shape[0]
    soff = np.arange(T + 2) * (2 * T - np.arange(T + 2) + 3) // 2
    Pall = sp.assoc_legendre_p_all(T, T, mu_all, norm=True)[0]
    spec = np.zeros((nf, soff[-1]), dtype=complex)
    off = 0
    for j, N in enumerate(nloen):
        N = int(N)
        M = min(T, (N - 1) // 2)
        lam = 2 * np.pi * np.arange(N) / N
        F = g[:, off: off + N] @ np.exp(-1j * np.outer(lam, np.arange(M + 1))) / N  # [nf, M+1]
        off += N
        for m in range(M + 1):
            Pm = Pall[m:, m, j] * (-1.0) ** m
            spec[:, soff[m]: soff[m + 1]] += w_all[j] * F[:, m: m + 1] * Pm[None, :]
    out = np.stack([spec.real, spec.imag], axis=-1).reshape(nf, -1)
    return out
