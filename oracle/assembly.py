"""Galerkin operators of a single patch or a conforming multi-patch domain.

Test infrastructure only (see oracle/__init__.py).

Definitions written out as sparse matrix products over the Gauss points:
  M_ij = sum_q w_q |J(q)| B_i(q) B_j(q)
  K_ij = sum_q w_q |J(q)| omega^2 grad B_i(q) . grad B_j(q)     (weak form of P:57)
  elastic K_(i,a),(j,b) = sum_q w|J| [lam d_aB_i d_bB_j + mu d_bB_i d_aB_j
                                       + mu delta_ab grad B_i . grad B_j]
with grad B = J^{-T} grad_xi B (isoparametric push-forward).
The quadrature rule is (p+1) Gauss points per element per direction
(the rule defines M and K on deformed maps)."""
from __future__ import annotations

import itertools

import numpy as np
import scipy.sparse as sp

from . import splines


def tables_1d(p: int, n: int):
    """Basis values / derivatives at the 1D Gauss points: (B, dB, w), B is (n(p+1), m)."""
    t = splines.open_uniform_knots(p, n)
    x, w = splines.quadrature_1d(p, n)
    return splines.basis(t, p, x), splines.basis_deriv(t, p, x), w


def _kron_all(mats):
    """kron(..., kron(A_z, kron(A_y, A_x))) so that the x index is fastest
    (co-lexicographic order).  mats = [A_x, A_y(, A_z)]."""
    out = sp.csr_matrix(mats[0])
    for A in mats[1:]:
        out = sp.kron(sp.csr_matrix(A), out, format="csr")
    return out


class PatchQuad:
    """Tensor-product quadrature data of one patch: basis matrices mapping the
    m^d control coefficients to the (n(p+1))^d Gauss points, Jacobians, weights."""

    def __init__(self, ctrl: np.ndarray, p: int, n: int, dim: int, reverse_points: bool = False):
        """reverse_points: enumerate the Gauss points in reverse order, which
        changes only the summation order of every quadrature sum (used by the
        tests to measure the fp64 assembly-order floor)."""
        B1, dB1, w1 = tables_1d(p, n)
        self.p, self.n, self.dim, self.m = p, n, dim, n + p
        self.B = _kron_all([B1] * dim)
        self.D = []  # parametric derivative matrices, D[c] = d/dxi_c
        for c in range(dim):
            mats = [dB1 if a == c else B1 for a in range(dim)]
            self.D.append(_kron_all(mats))
        w = w1
        for _ in range(dim - 1):
            w = np.kron(w1, w)
        if reverse_points:
            rev = np.arange(self.B.shape[0])[::-1]
            self.B = sp.csr_matrix(self.B[rev])
            self.D = [sp.csr_matrix(Dc[rev]) for Dc in self.D]
            w = w[rev]
        self.w = w
        # J[q, a, b] = dF_a/dxi_b = sum_i C_i[a] dB_i/dxi_b
        J = np.empty((self.B.shape[0], dim, dim))
        for a in range(dim):
            for b in range(dim):
                J[:, a, b] = self.D[b] @ ctrl[:, a]
        self.J = J
        self.detJ = np.linalg.det(J)
        self.Jinv = np.linalg.inv(J)
        # physical derivative matrices: d_a B = sum_c Jinv[c, a] d_xi_c B
        self.PD = []
        for a in range(dim):
            acc = None
            for c in range(dim):
                term = sp.diags(self.Jinv[:, c, a]) @ self.D[c]
                acc = term if acc is None else acc + term
            self.PD.append(sp.csr_matrix(acc))

    def min_detJ(self) -> float:
        return float(self.detJ.min())


def patch_operators(ctrl, p, n, dim, ncomp=1, omega=1.0, lam=1.0, mu=1.0, density=1.0, reverse_points=False):
    """Unreduced (all m^d control points) M and K of one patch.

    ncomp = 1: scalar wave; ncomp = dim: linear elasticity, component-major
    unknown ordering [u_x (all points), u_y, (u_z)].  Raises ValueError when
    |J| <= 0 at a Gauss point (Assumption P:699-701)."""
    Q = PatchQuad(ctrl, p, n, dim, reverse_points)
    if Q.min_detJ() <= 0.0:
        raise ValueError("non-positive Jacobian determinant")
    W = sp.diags(Q.w * Q.detJ)
    M = sp.csr_matrix(Q.B.T @ W @ Q.B)
    if ncomp == 1:
        K = None
        for a in range(dim):
            t = Q.PD[a].T @ W @ Q.PD[a]
            K = t if K is None else K + t
        K = sp.csr_matrix(omega ** 2 * K)
        return M, K
    assert ncomp == dim
    lap = None
    for f in range(dim):
        t = Q.PD[f].T @ W @ Q.PD[f]
        lap = t if lap is None else lap + t
    blocks = [[None] * dim for _ in range(dim)]
    for a in range(dim):
        for b in range(dim):
            blk = lam * (Q.PD[a].T @ W @ Q.PD[b]) + mu * (Q.PD[b].T @ W @ Q.PD[a])
            if a == b:
                blk = blk + mu * lap
            blocks[a][b] = blk
    K = sp.csr_matrix(sp.bmat(blocks))
    Mel = sp.csr_matrix(sp.block_diag([density * M] * dim))
    return Mel, K


def interior_mask(m: int, dim: int) -> np.ndarray:
    """Free (non-boundary) control points of a single patch, co-lex order:
    homogeneous Dirichlet on every face removes index 0 and m-1."""
    idx = np.indices((m,) * dim).reshape(dim, -1)[::-1]
    return np.all((idx > 0) & (idx < m - 1), axis=0)


class Discretization:
    """Reduced (free-DoF) operators of a single- or multi-patch problem.

    Multi-patch gluing: the global index map G^(r) identifies two
    local functions iff they coincide on the interface, which for conforming
    patches with matching knot vectors means coincident control points; a
    patch face is an interface iff its control points match another patch's
    face.  A global function is Dirichlet iff any of its local copies lies on
    a face that is not an interface (homogeneous BC on the outer boundary).

    Attributes
      M, K          free-DoF matrices (scipy CSR), scalar or component-major
      nfree         number of free scalar DoFs (per component)
      local_of      list over free DoFs of (patch, local control index) (first copy)
      G             per patch: array local index -> global index (or -1 if Dirichlet)
    """

    def __init__(self, patches, p, n, dim, ncomp=1, reverse_points=False, **mat):
        self.p, self.n, self.dim, self.ncomp = p, n, dim, ncomp
        m = n + p
        self.m = m
        npatch = len(patches)
        ctrls = [c for _, c in patches]
        # --- faces and interface detection --------------------------------
        idx = np.indices((m,) * dim).reshape(dim, -1)[::-1]
        faces = {}
        for r in range(npatch):
            for a in range(dim):
                for side in (0, m - 1):
                    sel = np.nonzero(idx[a] == side)[0]
                    key = frozenset(map(tuple, ctrls[r][sel]))
                    faces[(r, a, side)] = (sel, key)
        is_iface = {}
        for f, (sel, key) in faces.items():
            is_iface[f] = any(g != f and g[0] != f[0] and k2 == key
                              for g, (s2, k2) in faces.items())
        # --- global numbering by coincident control points -----------------
        coord_id = {}
        glob_of = []  # per patch: local -> global (all points, incl. Dirichlet)
        for r in range(npatch):
            gl = np.empty(m ** dim, dtype=np.int64)
            for i, pt in enumerate(map(tuple, ctrls[r])):
                if pt not in coord_id:
                    coord_id[pt] = len(coord_id)
                gl[i] = coord_id[pt]
            glob_of.append(gl)
        nglob = len(coord_id)
        dirichlet = np.zeros(nglob, dtype=bool)
        for (r, a, side), (sel, _) in faces.items():
            if not is_iface[(r, a, side)]:
                dirichlet[glob_of[r][sel]] = True
        free_ids = np.nonzero(~dirichlet)[0]
        # canonical order of free DoFs: by (patch, local index) of first copy
        first = {}
        for r in range(npatch):
            for i, g in enumerate(glob_of[r]):
                if not dirichlet[g] and g not in first:
                    first[g] = (r, i)
        order = sorted(first.keys(), key=lambda g: first[g])
        renum = -np.ones(nglob, dtype=np.int64)
        renum[np.array(order, dtype=np.int64)] = np.arange(len(order))
        self.nfree = len(order)
        assert self.nfree == len(free_ids)
        self.local_of = [first[g] for g in order]
        self.G = [renum[gl] for gl in glob_of]
        self.nadj = np.bincount(np.concatenate([g[g >= 0] for g in self.G]),
                                minlength=self.nfree).max() if self.nfree else 0
        # --- assembly: scatter-sum of patch contributions -------
        Mg = sp.csr_matrix((nglob * ncomp, nglob * ncomp))
        Kg = sp.csr_matrix((nglob * ncomp, nglob * ncomp))
        self.min_detJ = np.inf
        for r in range(npatch):
            Mr, Kr = patch_operators(ctrls[r], p, n, dim, ncomp, reverse_points=reverse_points, **mat)
            self.min_detJ = min(self.min_detJ, PatchQuad(ctrls[r], p, n, dim).min_detJ())
            rows = np.concatenate([glob_of[r] + c * nglob for c in range(ncomp)])
            Pr = sp.csr_matrix((np.ones(rows.size), (rows, np.arange(rows.size))),
                               shape=(nglob * ncomp, rows.size))
            Mg = Mg + Pr @ Mr @ Pr.T
            Kg = Kg + Pr @ Kr @ Pr.T
        self.M_full, self.K_full = sp.csr_matrix(Mg), sp.csr_matrix(Kg)
        sel = np.concatenate([np.array(order, dtype=np.int64) + c * nglob for c in range(ncomp)])
        self.M = sp.csr_matrix(Mg[sel][:, sel])
        self.K = sp.csr_matrix(Kg[sel][:, sel])
        self.nglob = nglob
        self._order = np.array(order, dtype=np.int64)

    def restrict_local(self, per_patch_values):
        """Free-DoF vector from per-patch control-point values (m^d, ncomp)
        (first copy wins; conforming data agree on interfaces)."""
        out = np.empty((self.ncomp, self.nfree))
        for f, (r, i) in enumerate(self.local_of):
            out[:, f] = per_patch_values[r][i]
        return out.reshape(-1)


def _element_point_data(ctrl, t, p, n, dim, elem, xg, wg):
    """Local quadrature data of one element (same definitions as PatchQuad, restricted to the
    (p+1)^d Gauss points of `elem` and its (p+1)^d non-zero bases, both co-lex, x fastest):
    weights w|J| (nq,), values B (nq, nloc), physical gradients PD (dim, nq, nloc), and the
    local basis multi-indices."""
    h = 1.0 / n
    V, Dd = [], []
    for d in range(dim):
        pts = (elem[d] + 0.5) * h + 0.5 * h * xg
        sl = slice(elem[d], elem[d] + p + 1)
        V.append(splines.basis(t, p, pts)[:, sl])
        Dd.append(splines.basis_deriv(t, p, pts)[:, sl])

    def kron_dirs(mats):  # kron(A_z, kron(A_y, A_x)): x fastest in both points and bases
        out = mats[0]
        for A in mats[1:]:
            out = np.kron(A, out)
        return out

    B = kron_dirs(V)
    D = [kron_dirs([Dd[a] if a == c else V[a] for a in range(dim)]) for c in range(dim)]
    loc = list(itertools.product(*[range(elem[d], elem[d] + p + 1) for d in reversed(range(dim))]))
    loc = [j[::-1] for j in loc]  # (x, y(, z)), x fastest
    m = n + p
    lin = np.array([j[0] + m * (j[1] + (m * j[2] if dim == 3 else 0)) for j in loc])
    # J[q, a, b] = sum_j C_j[a] dB_j/dxi_b
    J = np.einsum("ja,bqj->qab", ctrl[lin], np.array(D))
    det = np.linalg.det(J)
    Ji = np.linalg.inv(J)
    PD = np.einsum("qca,cqj->aqj", Ji, np.array(D))  # d_a B = sum_c Jinv[c, a] d_xi_c B
    wq = wg
    for _ in range(dim - 1):
        wq = np.kron(wg, wq)
    return 0.5 ** dim * h ** dim * wq * det, B, PD, loc


def operator_rows(ctrl, p, n, dim, rows, omega=1.0):
    """Rows of the unreduced scalar M and K of one patch, computed one by one
    by local quadrature over the support elements of each row (same
    definitions as patch_operators).  rows: control-point multi-indices
    (x, y(, z)).  Returns dict row -> (cols(list of multi-index), Mvals, Kvals).

    Used for full-size sampled checks; pinned against patch_operators."""
    t = splines.open_uniform_knots(p, n)
    xg, wg = splines.gauss_legendre(p + 1)
    out = {}
    for row in rows:
        row = tuple(int(v) for v in row)
        # elements whose support contains B_row: e_d in [row_d - p, row_d] ∩ [0, n)
        ranges = [range(max(0, r - p), min(n, r + 1)) for r in row]
        acc_M, acc_K = {}, {}
        for elem in itertools.product(*ranges):
            wd, B, PD, loc = _element_point_data(ctrl, t, p, n, dim, elem, xg, wg)
            me = loc.index(row)
            mrow = (wd * B[:, me]) @ B
            krow = omega ** 2 * sum((wd * PD[a][:, me]) @ PD[a] for a in range(dim))
            for jj, j in enumerate(loc):
                acc_M[j] = acc_M.get(j, 0.0) + mrow[jj]
                acc_K[j] = acc_K.get(j, 0.0) + krow[jj]
        cols = sorted(acc_M.keys(), key=lambda j: j[::-1])
        out[row] = (cols, np.array([acc_M[c] for c in cols]), np.array([acc_K[c] for c in cols]))
    return out


def elastic_operator_rows(ctrl, p, n, rows, lam=1.0, mu=1.0):
    """Rows of the unreduced elastic K of one 3D patch (component-major unknowns), one by one
    by local quadrature (same definition as patch_operators, ncomp = 3):
      K_(i,a),(j,b) = sum_q w|J| [lam d_aB_i d_bB_j + mu d_bB_i d_aB_j + mu delta_ab grad B_i . grad B_j].
    rows: control-point multi-indices (x, y, z).  Returns dict row -> (cols, vals) with
    vals[c][a][b] = K_(row,a),(cols[c],b).  Used for full-size sampled checks (C4); pinned
    against patch_operators."""
    dim = 3
    t = splines.open_uniform_knots(p, n)
    xg, wg = splines.gauss_legendre(p + 1)
    out = {}
    for row in rows:
        row = tuple(int(v) for v in row)
        ranges = [range(max(0, r - p), min(n, r + 1)) for r in row]
        acc = {}
        for elem in itertools.product(*ranges):
            wd, B, PD, loc = _element_point_data(ctrl, t, p, n, dim, elem, xg, wg)
            me = loc.index(row)
            gi = wd[None, :] * PD[:, :, me]                 # w|J| d_a B_row at the points (a, q)
            G = np.einsum("aq,bqj->abj", gi, PD)              # G[a, b, j] = sum_q w|J| d_aB_row d_bB_j
            lap = np.einsum("aaj->j", G)
            blk = lam * G + mu * np.transpose(G, (1, 0, 2)) + mu * np.eye(dim)[:, :, None] * lap[None, None, :]
            for jj, j in enumerate(loc):
                acc[j] = acc.get(j, 0.0) + blk[:, :, jj]
        cols = sorted(acc.keys(), key=lambda j: j[::-1])
        out[row] = (cols, np.array([acc[c] for c in cols]))
    return out


def dirichlet_lift(ctrl, p, n, dim, g_full, hD_terms, a0=0.0, a1=0.0, omega=1.0):
    """Non-homogeneous Dirichlet data by lifting, single patch,
    scalar wave: the boundary control coefficients are U_b(t) = g_b h_D(t) (g_full: all m^d
    control values, only the boundary entries are used; h_D = sum a cos(w t + phi)).  The free
    equations M_ff U_f'' + C_ff U_f' + K_ff U_f = F_f - M_fb U_b'' - C_fb U_b' - K_fb U_b with
    C = a0 M + a1 K become two forcing pairs: (-M_fb g_b) (h_D'' + a0 h_D') and
    (-K_fb g_b) (h_D + a1 h_D').  Returns (GM, termsM, GK, termsK) for integrator.Forcing."""
    from .integrator import sinusoid_derivative_terms
    M, K = patch_operators(ctrl, p, n, dim, omega=omega)
    m = n + p
    free = interior_mask(m, dim)
    bnd = ~free
    gb = np.asarray(g_full, dtype=np.float64)[bnd]
    GM = -(M[free][:, bnd] @ gb)
    GK = -(K[free][:, bnd] @ gb)
    termsM = sinusoid_derivative_terms(hD_terms, 2) + sinusoid_derivative_terms(hD_terms, 1, a0)
    termsK = list(hD_terms) + sinusoid_derivative_terms(hD_terms, 1, a1)
    return GM, termsM, GK, termsK
