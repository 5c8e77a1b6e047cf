"""B-spline basis by the Cox-de Boor recursion (§5.1).

Test infrastructure only (see oracle/__init__.py)."""
from __future__ import annotations

import numpy as np


def open_uniform_knots(p: int, n: int) -> np.ndarray:
    """Open knot vector xi_1=...=xi_{p+1}=0 < ... < xi_{m+1}=...=xi_{m+p+1}=1
     with n uniform elements and maximal regularity:
    interior knots i/n, each of multiplicity 1.  Length m+p+1, m = n+p."""
    return np.concatenate([np.zeros(p), np.linspace(0.0, 1.0, n + 1), np.ones(p)])


def _last_nonempty_span(t: np.ndarray) -> int:
    return max(i for i in range(len(t) - 1) if t[i] < t[i + 1])


def basis(t: np.ndarray, p: int, x) -> np.ndarray:
    """All m = len(t)-p-1 degree-p B-splines at points x, shape (len(x), m).

    Cox-de Boor: b_{i,0} = 1 on [xi_i, xi_{i+1}), and
    b_{i,p} = (x-xi_i)/(xi_{i+p}-xi_i) b_{i,p-1} + (xi_{i+p+1}-x)/(xi_{i+p+1}-xi_{i+1}) b_{i+1,p-1}
    with 0/0 = 0.  The right end x = 1 is assigned to the last non-empty span
    so that partition of unity holds on the closed interval."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    nb = len(t) - 1
    B = np.zeros((x.size, nb))
    for i in range(nb):
        B[:, i] = ((t[i] <= x) & (x < t[i + 1])).astype(np.float64)
    B[x == t[-1], _last_nonempty_span(t)] = 1.0
    for q in range(1, p + 1):
        nbq = len(t) - q - 1
        Bq = np.zeros((x.size, nbq))
        for i in range(nbq):
            d1 = t[i + q] - t[i]
            d2 = t[i + q + 1] - t[i + 1]
            left = (x - t[i]) / d1 * B[:, i] if d1 > 0 else 0.0
            right = (t[i + q + 1] - x) / d2 * B[:, i + 1] if d2 > 0 else 0.0
            Bq[:, i] = left + right
        B = Bq
    return B


def basis_deriv(t: np.ndarray, p: int, x) -> np.ndarray:
    """First derivatives of all degree-p B-splines at x, shape (len(x), m).

    Textbook derivative of the Cox-de Boor recursion:
    b'_{i,p} = p/(xi_{i+p}-xi_i) b_{i,p-1} - p/(xi_{i+p+1}-xi_{i+1}) b_{i+1,p-1}, 0/0 = 0."""
    x = np.atleast_1d(np.asarray(x, dtype=np.float64))
    if p == 0:
        return np.zeros((x.size, len(t) - 1))
    Bm = basis(t, p - 1, x)  # (npts, len(t)-p)
    m = len(t) - p - 1
    D = np.zeros((x.size, m))
    for i in range(m):
        d1 = t[i + p] - t[i]
        d2 = t[i + p + 1] - t[i + 1]
        if d1 > 0:
            D[:, i] += p / d1 * Bm[:, i]
        if d2 > 0:
            D[:, i] -= p / d2 * Bm[:, i + 1]
    return D


def gauss_legendre(npts: int):
    """Gauss-Legendre nodes/weights on [-1, 1] (library routine)."""
    return np.polynomial.legendre.leggauss(npts)


def quadrature_1d(p: int, n: int):
    """(p+1)-point Gauss rule on each of the n uniform elements.

    Returns (points, weights) of length n(p+1), element-major."""
    xg, wg = gauss_legendre(p + 1)
    h = 1.0 / n
    pts = np.concatenate([(e + 0.5) * h + 0.5 * h * xg for e in range(n)])
    wts = np.concatenate([0.5 * h * wg for _ in range(n)])
    return pts, wts
