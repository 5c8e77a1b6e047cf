"""Pins for oracle/params.py and oracle/spectral.py against what PAPER.md
prints: the Lambda_j / Lambda_k blocks, the characteristic
polynomials, the root target, the Theta -> 0 eigenvalues
(P:301), the order condition and the k-independent CFL limit
(P:29)."""
import json
import os

import numpy as np
import pytest

from oracle import params, spectral

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def printed_lambda_j(a, b, g, th):
    """Lambda_j, j < k, as printed in P:455-459."""
    return np.array([[a - b * th, a - b * th, 0.5 * (a - b * (th + 2))],
                     [-g * th, a - g * th, a - g / 2 * (th + 2)],
                     [-th, -th, a - 1 - th / 2]]) / a


def printed_lambda_k(a, b, g, th):
    """Lambda_k as printed in P:460-464."""
    return np.array([[a - b * th, a, a / 2 - b],
                     [-g * th, a, a - g],
                     [-th, 0.0, a - 1]]) / a


def test_rho0_values():
    g = GOLD["rho0_params"]
    for ps in (0, 1):
        al, be, ga, af = params.scheme_params(2, 0.0, ps)
        np.testing.assert_allclose([al[0], be[0], ga[0]], [g["alpha_j"], g["beta_j"], g["gamma_j"]], rtol=1e-15)
        np.testing.assert_allclose([al[1], be[1], ga[1]], [g["alpha_k"], g["beta_k"], g["gamma_k"]], rtol=1e-15)
    assert params.omega_b_k(0.0, 0.0) == g["omega_bk"]
    assert abs(params.omega_s_printed_k(0.0, 0.0) - g["omega_sk"]) < 1e-15


@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("rho", [0.0, 0.3, 0.5, 0.9, 1.0])
def test_order_condition_and_alpha_bound(k, rho):
    al, be, ga, af = params.scheme_params(k, rho, 0)
    np.testing.assert_allclose(ga - al + af, 0.5, atol=1e-15)
    assert np.all(al >= GOLD["alpha_lower_bound"]["value"] - 1e-15)
    assert af[-1] == 0.0 and np.all(af[:-1] == 1.0)


@pytest.mark.parametrize("k", [2, 3])
@pytest.mark.parametrize("rho", [0.0, 0.5, 1.0])
@pytest.mark.parametrize("th", [0.05, 0.7, 2.3])
def test_stepped_blocks_equal_printed_lambdas(k, rho, th):
    # reading R1 (K on the full Taylor predictor) reproduces the printed blocks
    al, be, ga, _ = params.scheme_params(k, rho, 0)
    G = spectral.amplification(th, k, rho, 0)
    for j in range(k):
        blk = G[3 * j:3 * j + 3, 3 * j:3 * j + 3]
        ref = (printed_lambda_j if j < k - 1 else printed_lambda_k)(al[j], be[j], ga[j], th)
        np.testing.assert_allclose(blk, ref, atol=1e-14)
        assert np.abs(G[3 * j + 3:, 3 * j:3 * j + 3]).max(initial=0.0) == 0.0  # block upper triangular


def test_k1_is_hulbert_chung_block():
    # k = 1: the single block is of Lambda_k type (eq:galpha)
    al, be, ga, _ = params.scheme_params(1, 0.4, 0)
    G = spectral.amplification(0.9, 1, 0.4)
    np.testing.assert_allclose(G, printed_lambda_k(al[0], be[0], ga[0], 0.9), atol=1e-15)


@pytest.mark.parametrize("rho", [0.0, 0.25, 0.5, 0.8])
def test_characteristic_polynomials_match_print(rho):
    # P:311-313, written with Theta (reading R7: the Theta^2 of eq:char is Theta)
    th = 1.37
    for ps in (0, 1):
        al, be, ga, _ = params.scheme_params(2, rho, ps)
        a, b, g = al[0], be[0], ga[0]
        p1 = np.array([2 * a, th * (2 * b + 2 * g + 1) - 6 * a + 2, th * (-4 * b - 2 * g + 1) + 6 * a - 4, 2 * b * th - 2 * a + 2])
        np.testing.assert_allclose(2 * a * np.poly(printed_lambda_j(a, b, g, th)), p1, atol=1e-13)
        a, b, g = al[1], be[1], ga[1]
        p2 = np.array([2 * a, 2 * th * b - 6 * a + 2, th * (-4 * b + 2 * g + 1) + 6 * a - 4, th * (2 * b + 1 - 2 * g) - 2 * a + 2])
        np.testing.assert_allclose(2 * a * np.poly(printed_lambda_k(a, b, g, th)), p2, atol=1e-13)


@pytest.mark.parametrize("rb,rs", [(0.0, 0.0), (0.5, 0.5), (0.6, 0.2), (0.3, 0.3), (0.9, 0.4)])
def test_root_target_at_bifurcation(rb, rs):
    # at the bifurcation limit the block polynomial is (l + rb)^2 (l + rs)
    target = np.poly([-rb, -rb, -rs])
    # block k: printed alpha_k, beta_k, Omega_bk
    a, b, g = params.block_k(rb, rs)
    blk = printed_lambda_k(a, b, g, params.omega_b_k(rb, rs))
    np.testing.assert_allclose(np.poly(blk), target, atol=1e-13)
    # blocks j < k, isospectral reading R2: Theta_b = (1+rb)(2+rs-rb rs)
    a, b, g = params.block_j_isospectral(rb, rs)
    blk = printed_lambda_j(a, b, g, (1 + rb) * (2 + rs - rb * rs))
    np.testing.assert_allclose(np.poly(blk), target, atol=1e-13)


@pytest.mark.parametrize("rb,rs", [(0.5, 0.5), (0.6, 0.2)])
def test_printed_jk_parameters_put_roots_at_plus_rho(rb, rs):
    # documents reading R2: the printed P:494-496 set is the P:328 solution with rho -> -rho
    a, b, g = params.block_j_printed(rb, rs)
    th = 2 - 2 * rb - rs + rs * rb ** 2  # printed Omega_bj
    np.testing.assert_allclose(np.poly(printed_lambda_j(a, b, g, th)), np.poly([rb, rb, rs]), atol=1e-12)


@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("rho", [0.0, 0.5, 0.9])
def test_theta_to_zero_eigenvalues(k, rho):
    # eigenvalues 1 (twice per block) and 1 - 1/alpha_j as Theta -> 0
    al, _, _, _ = params.scheme_params(k, rho, 0)
    G = spectral.amplification(0.0, k, rho, 0)
    ev = np.sort_complex(np.linalg.eigvals(G))
    ref = np.sort_complex(np.array([1.0] * (2 * k) + [1 - 1 / a for a in al], dtype=complex))
    np.testing.assert_allclose(ev, ref, atol=1e-6)  # defective eigenvalue 1: perturbation ~ sqrt(eps)


@pytest.mark.parametrize("rho", [0.0, 0.3, 0.5])
def test_cfl_limit_independent_of_k(rho):
    # the stability region does not depend on the order
    ref = params.theta_max_closed_form(rho)
    for k in (1, 2, 3):
        th = spectral.theta_max_scan(k, rho, npts=1200, tol=1e-9 if k < 3 else 1e-7)
        assert abs(th - ref) < 2e-6 * ref, (k, th, ref)


def test_cfl_limit_tends_to_four():
    # rho -> 1 gives the central-difference limit Theta = 4
    assert abs(params.theta_max_closed_form(1.0) - GOLD["theta_max_rho_to_1"]["value"]) < 1e-15
    assert abs(params.theta_max_closed_form(0.99) - 4.0) < 1e-3
    th = spectral.theta_max_scan(1, 0.99, npts=1200)
    assert abs(th - params.theta_max_closed_form(0.99)) < 1e-5


def test_printed_set_shrinks_cfl_for_k2():
    # reading R2 evidence: with the printed j<k set the k=2 limit falls below k=1's
    th1 = spectral.theta_max_scan(1, 0.5, npts=1200)
    th2 = spectral.theta_max_scan(2, 0.5, param_set=1, npts=1200)
    assert th2 < 0.5 * th1


@pytest.mark.parametrize("k", [1, 2])
@pytest.mark.parametrize("rho", [0.0, 0.5, 0.8])
def test_dissipation_and_radius_at_bifurcation(k, rho):
    # rho(G(Theta)) <= 1 on (0, Theta_max) (stable), < 1 in the interior of the
    # range for rho < 1 (dissipative), and equals rho at Theta = Omega_b
    thmax = params.theta_max_closed_form(rho)
    for th in np.linspace(0.01, 0.999 * thmax, 40):
        assert spectral.spectral_radius(th, k, rho) < 1.0
    thb = params.omega_b_k(rho, rho)
    assert abs(spectral.spectral_radius(thb, k, rho) - rho) < 1e-4  # triple root: eig error ~ eps^(1/3)
