"""Pins for oracle/precond.py: on the identity map the preconditioner is M
itself (P:703-713 with D = Dh), so PCG converges in one iteration; diag(calM)
= diag(M); the Schwarz preconditioner is SPD and PCG converges with counts
that do not grow under refinement (Tables)."""
import numpy as np
import pytest
import scipy.linalg as sla

import synth
from oracle import assembly, precond


def _disc(dim, p, n, noise=0.0, seed=0):
    ctrl = synth.control_net(dim, p, n, noise, seed)
    return assembly.Discretization([((0,) * dim, ctrl)], p, n, dim)


@pytest.mark.parametrize("dim,p,n", [(2, 2, 8), (2, 3, 9), (3, 2, 4), (3, 3, 3), (3, 4, 3), (3, 6, 3)])
def test_identity_map_one_iteration(dim, p, n):
    d = _disc(dim, p, n)
    P = precond.SchwarzPreconditioner(d)
    # right-hand side in the range of an operator, as on the hot path (b = -K s);
    # a raw random b amplifies the rounding of M by kappa(M) (~1e9 at p=6)
    b = d.M @ np.random.default_rng(1).standard_normal(d.nfree)
    x, it, hist = precond.pcg(lambda v: d.M @ v, b, P, tol=1e-13)
    assert it == 1, hist
    assert np.linalg.norm(b - d.M @ x) / np.linalg.norm(b) < 1e-13


def _dense_prec(d):
    P = precond.SchwarzPreconditioner(d)
    N = d.nfree * d.ncomp
    return np.stack([P(e) for e in np.eye(N)], axis=1)


def test_preconditioner_diagonal_equals_mass_diagonal():
    d = _disc(2, 3, 5, 0.2, seed=3)
    Pinv = _dense_prec(d)
    calM = np.linalg.inv(Pinv)
    np.testing.assert_allclose(np.diag(calM), d.M.diagonal(), rtol=1e-10)
    assert np.abs(Pinv - Pinv.T).max() < 1e-12 * np.abs(Pinv).max()


def test_schwarz_spd_and_converges_lshape():
    patches = synth.lshape_patches(2, 4, 0.1, seed=5)
    d = assembly.Discretization(patches, 2, 4, 2)
    Pinv = _dense_prec(d)
    assert np.abs(Pinv - Pinv.T).max() < 1e-12 * np.abs(Pinv).max()
    assert sla.eigvalsh(0.5 * (Pinv + Pinv.T)).min() > 0
    P = precond.SchwarzPreconditioner(d)
    b = np.random.default_rng(2).standard_normal(d.nfree)
    x, it, _ = precond.pcg(lambda v: d.M @ v, b, P, tol=1e-13)
    assert it <= 40
    assert np.linalg.norm(b - d.M @ x) / np.linalg.norm(b) < 1e-12


def test_iterations_do_not_grow_under_refinement():
    # robustness in h: counts at n and 2n within +2
    its = []
    for n in (8, 16):
        d = _disc(2, 3, n, 0.2, seed=7)
        P = precond.SchwarzPreconditioner(d)
        b = d.M @ np.random.default_rng(3).standard_normal(d.nfree)
        its.append(precond.pcg(lambda v: d.M @ v, b, P, tol=1e-13)[1])
    assert its[1] <= its[0] + 2, its
    assert its[0] <= 25


def test_elastic_preconditioner_blockwise():
    ctrl = synth.control_net(3, 2, 2, 0.15, seed=4)
    d = assembly.Discretization([((0, 0, 0), ctrl)], 2, 2, 3, ncomp=3)
    P = precond.SchwarzPreconditioner(d)
    b = np.random.default_rng(5).standard_normal(3 * d.nfree)
    x, it, _ = precond.pcg(lambda v: d.M @ v, b, P, tol=1e-13)
    assert np.linalg.norm(b - d.M @ x) / np.linalg.norm(b) < 1e-12
    assert it < 20
