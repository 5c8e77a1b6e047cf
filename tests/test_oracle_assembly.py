"""Pins for oracle/assembly.py: textbook stencils, integrals the domain fixes,
kernels of the operators, Kronecker structure of the identity map, elasticity
rigid-body modes, multi-patch gluing counts."""
import json
import os

import numpy as np
import pytest
import scipy.linalg as sla

import synth
from oracle import assembly, precond

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def test_p1_1d_stencils():
    n = 10
    h = 1.0 / n
    ctrl = synth.control_net(1, 1, n)
    M, K = assembly.patch_operators(ctrl, 1, n, 1)
    M, K = M.toarray(), K.toarray()
    g = GOLD["fem_p1_1d"]
    i = 5
    np.testing.assert_allclose(M[i, i - 1:i + 2], h * np.array(g["mass"]), rtol=1e-14)
    np.testing.assert_allclose(K[i, i - 1:i + 2], np.array(g["stiff"]) / h, rtol=1e-13)


@pytest.mark.parametrize("dim,p,n,noise", [(2, 2, 6, 0.2), (2, 3, 5, 0.2), (3, 2, 3, 0.15), (3, 3, 2, 0.15)])
def test_integrals_and_kernels(dim, p, n, noise):
    ctrl = synth.control_net(dim, p, n, noise, seed=11)
    M, K = assembly.patch_operators(ctrl, p, n, dim)
    # boundary control points are unperturbed, so F maps onto the unit square/cube
    # (p+1)-point Gauss is exact for degree 2p+1 per direction; |J| has degree
    # dim*p-1 per direction and x_a |J| p more, so check exactly only then.
    exact_vol = dim * p - 1 <= 2 * p + 1
    exact_mom = (dim + 1) * p - 1 <= 2 * p + 1
    assert abs(M.sum() - 1.0) < (1e-13 if exact_vol else 1e-5)          # |Omega| = 1
    # int x_a dOmega = 1/2: isoparametric map reproduces x_a = sum C_i[a] B_i
    one = np.ones(M.shape[0])
    for a in range(dim):
        assert abs(one @ (M @ ctrl[:, a]) - 0.5) < (1e-13 if exact_mom else 1e-5)
    assert np.abs(K @ one).max() < 1e-12 * np.abs(K).max()   # constants in ker K
    # linear field u = x_a: K u vanishes on rows whose support avoids the boundary
    m = n + p
    idx = np.indices((m,) * dim).reshape(dim, -1)[::-1]
    far = np.all((idx > p) & (idx < m - 1 - p), axis=0)
    if far.any():
        for a in range(dim):
            assert np.abs((K @ ctrl[:, a])[far]).max() < 1e-11 * np.abs(K).max()
    Md, Kd = M.toarray(), K.toarray()
    assert np.abs(Md - Md.T).max() < 1e-16 * 100
    assert np.abs(Kd - Kd.T).max() < 1e-13 * np.abs(Kd).max()
    assert sla.eigvalsh(Md).min() > 0


@pytest.mark.parametrize("dim,p,n", [(2, 2, 5), (2, 3, 4), (3, 2, 3), (3, 4, 2)])
def test_identity_map_is_kronecker(dim, p, n):
    # Greville control points => F = identity => M = Mh_z (x) Mh_y (x) Mh_x
    ctrl = synth.control_net(dim, p, n)
    M, _ = assembly.patch_operators(ctrl, p, n, dim)
    M1 = precond.param_mass_1d(p, n)
    Mk = M1
    for _ in range(dim - 1):
        Mk = np.kron(M1, Mk)
    np.testing.assert_allclose(M.toarray(), Mk, atol=1e-16 * 50)


def test_affine_map_scales_mass():
    # affine F(xi) = A xi + b: |J| = det A constant => M = det(A) * Mh (x) Mh
    p, n = 3, 4
    ctrl = synth.control_net(2, p, n)
    A = np.array([[1.3, 0.4], [-0.2, 0.9]])
    M, K = assembly.patch_operators(ctrl @ A.T + np.array([0.3, -1.0]), p, n, 2)
    M1 = precond.param_mass_1d(p, n)
    np.testing.assert_allclose(M.toarray(), np.linalg.det(A) * np.kron(M1, M1), atol=1e-15)


def test_identity_map_spectrum_separable():
    # identity map: eigenvalues of (K, M) in 2D are sums of 1D eigenvalues
    p, n = 2, 8
    c1 = synth.control_net(1, p, n)
    c2 = synth.control_net(2, p, n)
    d1 = assembly.Discretization([((0,), c1)], p, n, 1)
    d2 = assembly.Discretization([((0, 0), c2)], p, n, 2)
    e1 = sla.eigh(d1.K.toarray(), d1.M.toarray(), eigvals_only=True)
    e2 = sla.eigh(d2.K.toarray(), d2.M.toarray(), eigvals_only=True)
    np.testing.assert_allclose(np.sort(e2), np.sort((e1[:, None] + e1[None, :]).ravel()), rtol=1e-10)
    # lowest eigenvalue -> d pi^2 (continuous Dirichlet Laplacian), error O(h^2p)
    assert abs(e2[0] - 2 * np.pi ** 2) / (2 * np.pi ** 2) < 1e-4


def test_elasticity_rigid_body_modes_and_symmetry():
    p, n = 2, 3
    ctrl = synth.control_net(3, p, n, 0.15, seed=4)
    M, K = assembly.patch_operators(ctrl, p, n, 3, ncomp=3, lam=1.0, mu=1.0, density=1.0)
    Kd = K.toarray()
    nrm = np.abs(Kd).max()
    assert np.abs(Kd - Kd.T).max() < 1e-13 * nrm
    npt = ctrl.shape[0]
    modes = []
    for a in range(3):  # translations
        v = np.zeros((3, npt)); v[a] = 1.0; modes.append(v.ravel())
    for w in np.eye(3):  # rotations u = w x X (isoparametric: coefficients w x C_i)
        modes.append(np.cross(w[None, :], ctrl).T.ravel())
    for v in modes:
        assert np.abs(K @ v).max() < 1e-12 * nrm * np.abs(v).max()
    # a pure strain mode is not in the kernel
    v = np.zeros((3, npt)); v[0] = ctrl[:, 0]
    assert np.abs(K @ v.ravel()).max() > 1e-3 * nrm


def test_lshape_gluing():
    p, n = 2, 4
    m = n + p
    patches = synth.lshape_patches(p, n, 0.1, seed=5)
    d = assembly.Discretization(patches, p, n, 2)
    assert d.nfree == 3 * m * m - 10 * m + 8          # SURVEY.md §8c (3 patches, C0 gluing)
    assert d.nglob == 3 * m * m - 2 * m
    assert d.nadj == 2                               # N_adj: no triple points among free DoFs
    assert abs(d.M_full.sum() - 3.0) < 1e-13         # |L-shape| = 3
    one = np.ones(d.nglob)
    assert np.abs(d.K_full @ one).max() < 1e-12 * np.abs(d.K_full).max()
    Md = d.M.toarray()
    assert np.abs(Md - Md.T).max() == 0.0 or np.abs(Md - Md.T).max() < 1e-17
    assert sla.eigvalsh(Md).min() > 0


def test_operator_rows_match_assembly():
    p, n, dim = 2, 3, 3
    ctrl = synth.control_net(dim, p, n, 0.15, seed=9)
    M, K = assembly.patch_operators(ctrl, p, n, dim)
    m = n + p
    rows = [(1, 2, 3), (0, 0, 0), (4, 1, 2)]
    res = assembly.operator_rows(ctrl, p, n, dim, rows)
    for row in rows:
        L = row[0] + m * (row[1] + m * row[2])
        cols, mv, kv = res[row]
        cl = [c[0] + m * (c[1] + m * c[2]) for c in cols]
        np.testing.assert_allclose(mv, M.toarray()[L, cl], rtol=1e-12, atol=1e-18)
        np.testing.assert_allclose(kv, K.toarray()[L, cl], rtol=1e-11, atol=1e-14)
        assert np.count_nonzero(M.toarray()[L]) == len(cols)


def _bspline_1d_matrices(p, n):
    """1D parametric matrices on [0, 1] from scipy's B-splines (an independent library):
    M1 = int b_i b_j, K1 = int b_i' b_j', C1 = int b_i' b_j, by dense Gauss-Legendre per element."""
    from scipy.interpolate import BSpline
    t = np.concatenate([np.zeros(p), np.linspace(0.0, 1.0, n + 1), np.ones(p)])
    m = n + p
    xg, wg = np.polynomial.legendre.leggauss(p + 4)
    M1, K1, C1 = np.zeros((m, m)), np.zeros((m, m)), np.zeros((m, m))
    for e in range(n):
        a, b = e / n, (e + 1) / n
        x = 0.5 * (a + b) + 0.5 * (b - a) * xg
        w = 0.5 * (b - a) * wg
        V = np.array([BSpline(t, np.eye(m)[i], p, extrapolate=False)(x) for i in range(m)])
        Dv = np.array([BSpline(t, np.eye(m)[i], p, extrapolate=False).derivative()(x) for i in range(m)])
        V, Dv = np.nan_to_num(V), np.nan_to_num(Dv)
        M1 += (V * w) @ V.T
        K1 += (Dv * w) @ Dv.T
        C1 += (Dv * w) @ V.T
    return M1, K1, C1


def test_elasticity_kronecker_identities_lambda_ne_mu():
    # identity map (Greville control points): G_cd = int d_cB_i d_dB_j is a Kronecker product of 1D
    # matrices, and the elastic blocks are K_(a,a) = (lam + 2mu) G_aa + mu sum_{c != a} G_cc,
    # K_(a,b) = lam G_ab + mu G_ba.  lam != mu makes a lam <-> mu swap or a
    # mu-for-2mu slip visible.  The exact 1D Gauss rule is exact here.
    p, n, lam, mu = 2, 3, 2.0, 0.5
    ctrl = synth.control_net(3, p, n)
    _, K = assembly.patch_operators(ctrl, p, n, 3, ncomp=3, lam=lam, mu=mu, density=1.0)
    M1, K1, C1 = _bspline_1d_matrices(p, n)
    m = n + p
    N = m ** 3

    def kr(ax, ay, az):  # kron(z, kron(y, x)): x fastest (co-lex)
        return np.kron(az, np.kron(ay, ax))

    def G(c, d):
        facs = []
        for dirn in range(3):
            if dirn == c and dirn == d:
                facs.append(K1)
            elif dirn == c:
                facs.append(C1)          # d/dx on B_i only: int b_i' b_j
            elif dirn == d:
                facs.append(C1.T)        # d/dx on B_j only: int b_i b_j'
            else:
                facs.append(M1)
        return kr(*facs)

    Kd = K.toarray()
    for a in range(3):
        for b in range(3):
            blk = Kd[a * N:(a + 1) * N, b * N:(b + 1) * N]
            if a == b:
                ref = (lam + 2 * mu) * G(a, a) + mu * sum(G(c, c) for c in range(3) if c != a)
            else:
                ref = lam * G(a, b) + mu * G(b, a)
            np.testing.assert_allclose(blk, ref, atol=1e-13 * np.abs(ref).max(), err_msg=f"block {a}{b}")
    # the swapped parameters give a different operator (the pin discriminates lam from mu)
    _, Ks = assembly.patch_operators(ctrl, p, n, 3, ncomp=3, lam=mu, mu=lam, density=1.0)
    assert np.abs(Ks.toarray() - Kd).max() > 0.1 * np.abs(Kd).max()


@pytest.mark.parametrize("p,n,lam,mu", [(2, 3, 1.0, 1.0), (3, 2, 2.0, 0.5), (4, 2, 0.7, 1.3)])
def test_elastic_operator_rows_match_assembly(p, n, lam, mu):
    ctrl = synth.control_net(3, p, n, 0.15, seed=4)
    _, K = assembly.patch_operators(ctrl, p, n, 3, ncomp=3, lam=lam, mu=mu, density=1.0)
    Kd = K.toarray()
    m = n + p
    N = m ** 3
    rows = [(1, 2, 1), (0, 0, 0), (m - 1, 1, m - 2)]
    res = assembly.elastic_operator_rows(ctrl, p, n, rows, lam=lam, mu=mu)
    for row in rows:
        L = row[0] + m * (row[1] + m * row[2])
        cols, vals = res[row]
        cl = np.array([c[0] + m * (c[1] + m * c[2]) for c in cols])
        for a in range(3):
            for b in range(3):
                np.testing.assert_allclose(vals[:, a, b], Kd[a * N + L, b * N + cl], rtol=1e-11,
                                           atol=1e-13 * np.abs(Kd).max())
        assert np.count_nonzero(Kd[L, :N]) <= len(cols)


@pytest.mark.parametrize("dim,p,n", [(2, 3, 5), (3, 4, 2)])
def test_operator_rows_match_assembly_2d_and_high_p(dim, p, n):
    ctrl = synth.control_net(dim, p, n, 0.15, seed=9)
    M, K = assembly.patch_operators(ctrl, p, n, dim)
    Md, Kd = M.toarray(), K.toarray()
    m = n + p
    rows = [(1,) * dim, (m - 1,) * dim, tuple([2, m - 2, 1][:dim])]
    res = assembly.operator_rows(ctrl, p, n, dim, rows)
    for row in rows:
        L = row[0] + m * (row[1] + (m * row[2] if dim == 3 else 0))
        cols, mv, kv = res[row]
        cl = [c[0] + m * (c[1] + (m * c[2] if dim == 3 else 0)) for c in cols]
        np.testing.assert_allclose(mv, Md[L, cl], rtol=1e-12, atol=1e-18)
        np.testing.assert_allclose(kv, Kd[L, cl], rtol=1e-11, atol=1e-13 * np.abs(Kd).max())
        assert np.count_nonzero(Md[L]) == len(cols)
