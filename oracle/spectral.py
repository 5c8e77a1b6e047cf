"""Amplification matrix of the scheme on a single mode (§3.2, §4.1).

Test infrastructure only (see oracle/__init__.py).

For M = 1, K = lambda, tau = 1 (so Theta = tau^2 lambda) one step of
oracle.integrator.step is a linear map of the 3k-vector
[U, tau V, tau^2 A, tau^3 L^1(A), ...]; G(Theta) is built column by
column by stepping unit vectors (not from the printed A, B of P:196-215,
which carry typos, reading R5)."""
from __future__ import annotations

import numpy as np

from .integrator import step
from .params import scheme_params


def amplification(theta: float, k: int, rho: float, param_set: int = 0, rho_s=None):
    al, be, ga, _ = scheme_params(k, rho, param_set, rho_s)
    K = np.array([[theta]])
    G = np.zeros((3 * k, 3 * k))
    for col in range(3 * k):
        c = [np.zeros(1) for _ in range(3 * k)]
        c[col][0] = 1.0
        new = step(c, k, 1.0, al, be, ga, lambda b: b, K)
        G[:, col] = [v[0] for v in new]
    return G


def spectral_radius(theta, k, rho, param_set=0, rho_s=None):
    return float(np.max(np.abs(np.linalg.eigvals(amplification(theta, k, rho, param_set, rho_s)))))


def theta_max_scan(k, rho, param_set=0, hi=6.0, npts=60000, tol=1e-9):
    """First Theta on a uniform grid of (0, hi] where rho(G) > 1 + tol, refined
    by bisection."""
    grid = np.linspace(hi / npts, hi, npts)
    prev = grid[0]
    for th in grid:
        if spectral_radius(th, k, rho, param_set) > 1.0 + tol:
            lo, up = prev, th
            for _ in range(60):
                mid = 0.5 * (lo + up)
                if spectral_radius(mid, k, rho, param_set) > 1.0 + tol:
                    up = mid
                else:
                    lo = mid
            return 0.5 * (lo + up)
        prev = th
    return np.inf
