"""Generalized-alpha parameters of the explicit order-2k scheme.

Test infrastructure only (see oracle/__init__.py).

Block k (the last block, K acting on the old displacement) uses the printed
closed forms P:497-499, alpha_fk = 0.  Blocks j < k (alpha_fj = 1,
P:515) come in two readings (reading R2 = SURVEY.md §8c G2):
  param_set 0 (default, "isospectral"): re-derived from the root target
    (lambda + rho_b)^2 (lambda + rho_s) that P:328 states;
  param_set 1: the formulas as printed in P:494-496.
gamma_j = 1/2 - alpha_fj + alpha_j for every block."""
from __future__ import annotations

import numpy as np


def block_k(rho_b: float, rho_s: float):
    """alpha_k, beta_k, gamma_k (P:497-499, P:477 with alpha_fk = 0)."""
    rb, rs = rho_b, rho_s
    alpha = (2.0 + (1.0 - rb) * rs) / ((1.0 + rb) * (1.0 + rs))
    beta = ((-5.0 - 3.0 * rb - 4.0 * rs + 2.0 * rb * rs + 2.0 * rb ** 2 * rs - rs ** 2 + rb * rs ** 2)
            / ((1.0 + rb) ** 2 * (-2.0 - 3.0 * rs + rb * rs - rs ** 2 + rb * rs ** 2)))
    gamma = 0.5 - 0.0 + alpha
    return alpha, beta, gamma


def block_j_printed(rho_b: float, rho_s: float):
    """alpha_j, beta_j, gamma_j as printed in P:494-496 (alpha_fj = 1).
    Undefined (division by zero) at rho = 1."""
    rb, rs = rho_b, rho_s
    alpha = (2.0 - (1.0 + rb) * rs) / ((-1.0 + rb) * (-1.0 + rs))
    beta = ((1.0 + rb) * (-1.0 + rb * rs) ** 2
            / ((-1.0 + rb) ** 2 * (-1.0 + rs) * (-2.0 + rs + rb * rs)))
    gamma = 0.5 - 1.0 + alpha
    return alpha, beta, gamma


def block_j_isospectral(rho_b: float, rho_s: float):
    """alpha_j, beta_j, gamma_j solving det(lambda I - Lambda_j) proportional to
    (lambda + rho_b)^2 (lambda + rho_s) for the Lambda_1-type block
     with alpha_fj = 1.  Pinned by tests (roots at Omega_b)."""
    rb, rs = rho_b, rho_s
    alpha = (2.0 + rs - rb * rs) / ((1.0 + rb) * (1.0 + rs))
    beta = ((1.0 - rb) * (1.0 - rb * rs) ** 2
            / ((1.0 + rb) ** 2 * (1.0 + rs) * (2.0 + rs - rb * rs)))
    gamma = 0.5 - 1.0 + alpha
    return alpha, beta, gamma


def omega_b_k(rho_b, rho_s):
    """Bifurcation limit of block k."""
    return 2.0 + 2.0 * rho_b + rho_s - rho_s * rho_b ** 2


def scheme_params(k: int, rho: float, param_set: int = 0, rho_s: float | None = None):
    """Arrays alpha[j], beta[j], gamma[j], alpha_f[j], j = 0..k-1 (block j+1).

    rho_b = rho_s = rho for every block unless rho_s is given."""
    rs = rho if rho_s is None else rho_s
    al, be, ga, af = [], [], [], []
    for j in range(1, k + 1):
        if j < k:
            a, b, g = (block_j_isospectral if param_set == 0 else block_j_printed)(rho, rs)
            f = 1.0
        else:
            a, b, g = block_k(rho, rs)
            f = 0.0
        al.append(a); be.append(b); ga.append(g); af.append(f)
    return np.array(al), np.array(be), np.array(ga), np.array(af)


def theta_max_closed_form(rho: float) -> float:
    """lambda = -1 crossing of the Lambda_k-type block with rho_b = rho_s = rho:
    Theta_max = (4 alpha - 2)/(2 beta - gamma) = 12(2-rho)(1+rho)/(rho^2-5rho+10)
    (replaces the inexact printed Omega_s of P:505-511)."""
    return 12.0 * (2.0 - rho) * (1.0 + rho) / (rho * rho - 5.0 * rho + 10.0)


def omega_s_printed_k(rho_b, rho_s):
    """Printed critical value Omega_sk, P:509-510 (kept for the G3 pin)."""
    rb, rs = rho_b, rho_s
    num = 4 * (1 + rb) * (2 - rb * rs + rs) * (3 - rb + rs - 3 * rb * rs)
    den = 2 * (5 - rb ** 2) + (5 - 13 * rb - rb ** 2 + rb ** 3) * rs - (1 - rb) ** 3 * rs ** 2
    return num / den
