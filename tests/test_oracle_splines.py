"""Pins for oracle/splines.py (§5.1) against closed forms and an
independent library implementation."""
import json
import os

import numpy as np
import pytest
from scipy.interpolate import BSpline

from oracle import splines

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7])
def test_partition_of_unity_and_nonnegativity(p):
    # non-negative, sum to one on [0,1]
    t = splines.open_uniform_knots(p, 9)
    x = np.concatenate([np.linspace(0, 1, 301), [1.0]])
    B = splines.basis(t, p, x)
    assert B.shape == (x.size, 9 + p)
    assert B.min() >= 0.0
    np.testing.assert_allclose(B.sum(axis=1), 1.0, atol=1e-14)
    D = splines.basis_deriv(t, p, x[:-1])
    np.testing.assert_allclose(D.sum(axis=1), 0.0, atol=1e-11)


@pytest.mark.parametrize("p,n", [(1, 4), (2, 7), (3, 5), (5, 11), (7, 10)])
def test_matches_scipy_bspline(p, n):
    # independent library routine (de Boor evaluation in scipy)
    t = splines.open_uniform_knots(p, n)
    x = np.random.default_rng(p).uniform(0, 1, 200)
    ours = splines.basis(t, p, x)
    ref = BSpline.design_matrix(x, t, p).toarray()
    np.testing.assert_allclose(ours, ref, atol=1e-14)
    d_ours = splines.basis_deriv(t, p, x)
    m = n + p
    d_ref = np.stack([BSpline(t, np.eye(m)[i], p).derivative()(x) for i in range(m)], axis=1)
    np.testing.assert_allclose(d_ours, d_ref, atol=1e-10 * max(1.0, np.abs(d_ref).max()))


def test_quadratic_midpoint_values():
    vals = GOLD["quadratic_bspline_midpoint"]["values"]
    n = 8
    t = splines.open_uniform_knots(2, n)
    e = 4  # interior element [4/8, 5/8]; supports basis e..e+2
    B = splines.basis(t, 2, [(e + 0.5) / n])[0]
    np.testing.assert_allclose(B[e:e + 3], vals, atol=1e-15)
    assert abs(B.sum() - 1.0) < 1e-15


def test_hat_functions_p1():
    # p = 1: b_i are the piecewise-linear hats at the nodes i/n
    n = 5
    t = splines.open_uniform_knots(1, n)
    x = np.linspace(0, 1, 51)
    B = splines.basis(t, 1, x)
    for i in range(n + 1):
        np.testing.assert_allclose(B[:, i], np.maximum(0, 1 - np.abs(x * n - i)), atol=1e-14)


@pytest.mark.parametrize("p", [1, 2, 3, 6])
def test_gauss_rule_exactness(p):
    # (p+1)-point Gauss integrates degree 2p+1 exactly on each element
    x, w = splines.quadrature_1d(p, 7)
    deg = 2 * p + 1
    np.testing.assert_allclose((w * x ** deg).sum(), 1.0 / (deg + 1), rtol=1e-13)
    np.testing.assert_allclose(w.sum(), 1.0, rtol=1e-14)
