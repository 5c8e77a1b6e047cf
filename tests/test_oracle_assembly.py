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
