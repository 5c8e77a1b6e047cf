"""Explicit order-2k generalized-alpha integrator (§3-§4).

Test infrastructure only (see oracle/__init__.py).

State chain c_0 .. c_{3k-1}:  c_0 = U, c_1 = V, c_2 = A, c_{m} = L^{m-2}(A)
(P:123).  Block j (1-based) owns disp = 3j-3, vel = 3j-2,
acc = 3j-1.  Taylor predictor T_m(c) = sum_{i=0}^{3k-1-m} tau^i/i! c_{m+i}.

One step (P:398-431 with the jump [[.]] = Delta of P:113; reading R1 =
SURVEY.md §8c G1 for the K-term of blocks j < k; F = C = 0):
  s_j  = T_disp(c)   (j < k)      s_k = c_{3k-3}
  y_j  = M^{-1}(-K s_j)           (= T_acc + alpha_j P_j, P:424/428/429)
  P_j  = (y_j - T_acc(c)) / alpha_j
  c'_disp = T_disp + beta_j tau^2 P_j   c'_vel = T_vel + gamma_j tau P_j
  c'_acc  = T_acc + P_j
All k blocks read only old-step data.

Initial chain (P:119-121, P:155-162 generalised, reading R3):
  c_0 = U_0, c_1 = V_0, c_m = M^{-1}(-K c_{m-2}), m = 2 .. 3k-1.

Forcing (eq:ho1 P:398-404): block j's right-hand side is
F^{(3j-3)}(t_n + alpha_fj tau) - K s_j, and the initial chain is
c_m = M^{-1}(F^{(m-2)}(t_0) - K c_{m-2}) (the ODE differentiated m-2 times at t_0).
Here F(t) = G h(t) with h a sum of sinusoids, whose derivatives are closed form.

Damping C (eq:ho1's C L^{3j-4}(A_n) term, reading R16 = SURVEY G8 resolved like R1): block j
subtracts C w_j with w_j = T_{3j-2}(c) (j < k, the Taylor predictor of its velocity-level
entry) and w_k = c_{3k-2}; the initial chain c_m = M^{-1}(F^{(m-2)} - K c_{m-2} - C c_{m-1}).
The literal old value c_{3j-2} for j < k is first order (test_damped_scalar_ode_order_2k)."""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .params import scheme_params


class DirectMassSolver:
    """Sparse LU of M (SuperLU) plus one step of iterative refinement
    x += M^{-1}(b - M x) reusing the factorisation."""

    def __init__(self, M):
        self.M = sp.csc_matrix(M)
        # minimum-degree ordering on A^T+A (SPD M): same factorisation up to rounding, ~8x faster than COLAMD
        self.lu = spla.splu(self.M, permc_spec="MMD_AT_PLUS_A")

    def __call__(self, b):
        b = np.asarray(b, dtype=np.float64)
        if not np.any(b):
            return np.zeros_like(b)
        x = self.lu.solve(b)
        x += self.lu.solve(b - self.M @ x)
        return x


def taylor(c, m: int, tau: float):
    """T_m(c) = sum_{i=0}^{len(c)-1-m} tau^i / i! c_{m+i}."""
    out = np.array(c[m], dtype=np.float64, copy=True)
    for i in range(1, len(c) - m):
        out = out + (tau ** i / math.factorial(i)) * c[m + i]
    return out


class Forcing:
    """F(t) = G h(t), h(t) = sum_i a_i cos(w_i t + phi_i); F^{(m)}(t) = G h^{(m)}(t) with
    h^{(m)}(t) = sum_i a_i w_i^m cos(w_i t + phi_i + m pi / 2)."""

    def __init__(self, G, terms):
        self.G = np.asarray(G, dtype=np.float64)
        self.terms = [(float(a), float(w), float(ph)) for a, w, ph in terms]

    def h(self, m: int, t: float) -> float:
        return sum(a * w ** m * math.cos(w * t + ph + m * math.pi / 2) for a, w, ph in self.terms)

    def __call__(self, m: int, t: float):
        return self.h(m, t) * self.G


class ForcingSum:
    """Sum of Forcing terms (e.g. a load plus the Dirichlet lifting pairs)."""

    def __init__(self, parts):
        self.parts = [f for f in parts if f is not None]

    def __call__(self, m: int, t: float):
        out = None
        for f in self.parts:
            v = f(m, t)
            out = v if out is None else out + v
        return out


def sinusoid_derivative_terms(terms, order: int, scale: float = 1.0):
    """Terms of scale * h^{(order)} for h = sum a cos(w t + phi): a w^order, w, phi + order pi/2."""
    return [(scale * a * w ** order, w, ph + order * math.pi / 2) for a, w, ph in terms]


def initial_chain(u0, v0, k: int, solve, Kop, F=None, t0: float = 0.0, Cop=None):
    """c_0 = U_0, c_1 = V_0, c_m = M^{-1}(F^{(m-2)}(t_0) - K c_{m-2} - C c_{m-1}), m = 2..3k-1."""
    c = [np.array(u0, dtype=np.float64), np.array(v0, dtype=np.float64)]
    for m in range(2, 3 * k):
        rhs = -(Kop @ c[m - 2])
        if Cop is not None:
            rhs = rhs - Cop @ c[m - 1]
        if F is not None:
            rhs = rhs + F(m - 2, t0)
        c.append(solve(rhs))
    return c


def step(c, k: int, tau: float, alpha, beta, gamma, solve, Kop, F=None, t: float = 0.0, alpha_f=None, Cop=None):
    """One explicit step of the order-2k scheme from time t; returns the new chain."""
    new = [None] * (3 * k)
    for j in range(1, k + 1):
        d, v, a = 3 * j - 3, 3 * j - 2, 3 * j - 1
        Td, Tv, Ta = taylor(c, d, tau), taylor(c, v, tau), taylor(c, a, tau)
        s = Td if j < k else c[d]
        rhs = -(Kop @ s)
        if Cop is not None:  # C w_j, w_j = T_vel(c) for j < k, c_vel for j = k (reading R16)
            rhs = rhs - Cop @ (Tv if j < k else c[v])
        if F is not None:  # F^{(3j-3)} at t_n + alpha_fj tau (eq:ho1)
            rhs = rhs + F(3 * j - 3, t + alpha_f[j - 1] * tau)
        y = solve(rhs)
        P = (y - Ta) / alpha[j - 1]
        new[d] = Td + beta[j - 1] * tau * tau * P
        new[v] = Tv + gamma[j - 1] * tau * P
        new[a] = Ta + P
    return new


class Integrator:
    """Convenience driver: M, K (free-DoF sparse matrices), k, rho, dt."""

    def __init__(self, M, K, k: int, rho: float, dt: float, param_set: int = 0, solver=None, forcing=None,
                 t0: float = 0.0, C=None):
        self.M, self.K = sp.csr_matrix(M), sp.csr_matrix(K)
        self.k, self.dt = k, dt
        self.alpha, self.beta, self.gamma, self.alpha_f = scheme_params(k, rho, param_set)
        self.solve = solver if solver is not None else DirectMassSolver(self.M)
        self.F, self.t0, self.n = forcing, t0, 0
        self.C = None if C is None else sp.csr_matrix(C)

    def init(self, u0, v0):
        self.n = 0
        return initial_chain(u0, v0, self.k, self.solve, self.K, self.F, self.t0, self.C)

    def step(self, c):
        out = step(c, self.k, self.dt, self.alpha, self.beta, self.gamma, self.solve, self.K, self.F,
                   self.t0 + self.n * self.dt, self.alpha_f, self.C)
        self.n += 1
        return out

    def run(self, u0, v0, nsteps: int, chain=None):
        c = self.init(u0, v0) if chain is None else chain
        for _ in range(nsteps):
            c = self.step(c)
        return c
