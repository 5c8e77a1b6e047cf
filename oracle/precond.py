"""Mass preconditioner and PCG (§5.4-5.6).

Test infrastructure only (see oracle/__init__.py).

Single patch:  calM = D^{1/2} Dh^{-1/2} Mh Dh^{-1/2} D^{1/2},
  Mh = parametric mass (identity map), Mh = Mh_z (x) Mh_y (x) Mh_x on the free
  indices, Dh = diag(Mh), D = diag(M).
  calM^{-1} r = s o Mh^{-1} (s o r),  s = sqrt(Dh / D).
Multi-patch additive Schwarz:
  calM_ad^{-1} = sum_r R^(r)T calM^(r)^{-1} R^(r),
  with D^(r) = restriction of the global diag(M) and, where the patch's free
  set is not a tensor product (re-entrant corner), zero-extension to its
  bounding box (reading R6 = SURVEY.md §8c G14(a)).
Mh^{-1} is applied by banded Cholesky line solves along each direction
(library routine scipy.linalg.cho_solve_banded)."""
from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from .assembly import tables_1d


def param_mass_1d(p: int, n: int) -> np.ndarray:
    """Dense 1D parametric mass matrix Mh_1D[i,j] = int_0^1 b_i b_j, all m indices."""
    B, _, w = tables_1d(p, n)
    return B.T @ (w[:, None] * B)


def _banded_lower(A: np.ndarray, p: int) -> np.ndarray:
    nn = A.shape[0]
    ab = np.zeros((p + 1, nn))
    for d in range(p + 1):
        ab[d, : nn - d] = np.diagonal(A, -d)
    return ab


class KronFactor:
    """Cholesky factors of Mh restricted to a box [lo_d, hi_d] of local indices."""

    def __init__(self, p, n, lo, hi):
        full = param_mass_1d(p, n)
        self.p = p
        self.dims = [h - l + 1 for l, h in zip(lo, hi)]
        self.fac = []
        self.diag = []
        for l, h in zip(lo, hi):
            A = full[l:h + 1, l:h + 1]
            self.diag.append(np.diag(A).copy())
            self.fac.append(sla.cholesky_banded(_banded_lower(A, p), lower=True))
        dh = self.diag[0]
        for dd in self.diag[1:]:
            dh = np.kron(dd, dh)
        self.Dhat = dh  # co-lex (x fastest)

    def solve(self, v: np.ndarray) -> np.ndarray:
        """Mh^{-1} v for v in co-lex order over the box."""
        dim = len(self.dims)
        T = v.reshape(self.dims[::-1])  # axes (z, y, x)
        for d in range(dim):
            ax = dim - 1 - d
            Tm = np.moveaxis(T, ax, 0)
            sh = Tm.shape
            sol = sla.cho_solve_banded((self.fac[d], True), Tm.reshape(sh[0], -1))
            T = np.moveaxis(sol.reshape(sh), 0, ax)
        return T.reshape(-1)


class SchwarzPreconditioner:
    """calM_ad^{-1} for a Discretization (single patch: one term, calM^{-1})."""

    def __init__(self, disc):
        self.disc = disc
        m, dim, p, n = disc.m, disc.dim, disc.p, disc.n
        diagM = disc.M.diagonal()[: disc.nfree]  # component 0 block (density-scaled scalar M)
        self.terms = []
        idx = np.indices((m,) * dim).reshape(dim, -1)[::-1]  # local multi-index per control point
        for r, G in enumerate(disc.G):
            loc = np.nonzero(G >= 0)[0]
            if loc.size == 0:
                continue
            mi = idx[:, loc]
            lo, hi = mi.min(axis=1), mi.max(axis=1)
            fac = KronFactor(p, n, lo, hi)
            dims = fac.dims
            boxpos = np.zeros(loc.size, dtype=np.int64)
            stride = 1
            for d in range(dim):
                boxpos += (mi[d] - lo[d]) * stride
                stride *= dims[d]
            glob = G[loc]
            s = np.sqrt(fac.Dhat[boxpos] / diagM[glob])
            self.terms.append((fac, boxpos, glob, s, int(np.prod(dims))))

    def __call__(self, r: np.ndarray) -> np.ndarray:
        nf, nc = self.disc.nfree, self.disc.ncomp
        R = r.reshape(nc, nf)
        Z = np.zeros_like(R)
        for c in range(nc):
            for fac, boxpos, glob, s, nbox in self.terms:
                t = np.zeros(nbox)
                t[boxpos] = s * R[c, glob]
                t = fac.solve(t)
                np.add.at(Z[c], glob, s * t[boxpos])
        return Z.reshape(-1)


def pcg(apply_M, b, apply_Pinv, tol=1e-13, maxit=500, x0=None):
    """Textbook preconditioned conjugate gradients, stop when
    ||r||_2 <= tol ||b||_2 (recursive residual), zero initial guess.
    Returns (x, iterations, history of ||r||/||b||)."""
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
    if nb == 0.0:
        return x, 0, [0.0]
    r = b - apply_M(x) if x0 is not None else b.copy()
    hist = [np.linalg.norm(r) / nb]
    it = 0
    z = apply_Pinv(r)
    p = z.copy()
    rz = r @ z
    while hist[-1] > tol and it < maxit:
        q = apply_M(p)
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        it += 1
        hist.append(np.linalg.norm(r) / nb)
        if hist[-1] <= tol:
            break
        z = apply_Pinv(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, it, hist
