"""Pins for oracle/integrator.py: temporal order 2k,
exact modal decomposition through the amplification matrix, spatial order
p+1 against the closed-form wave solution (BASELINE.json configs[0]),
dissipation / stability behaviour."""
import math

import numpy as np
import pytest
import scipy.linalg as sla

import synth
from oracle import assembly, integrator, params, spectral


def _orders(errs):
    e = np.asarray(errs)
    return np.log2(e[:-1] / e[1:])


@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("rho", [0.0, 0.5, 1.0])
def test_scalar_ode_order_2k(k, rho):
    # u'' = -w^2 u, u(0)=1, v(0)=0: exact u = cos(w t), v = -w sin(w t)
    w, T = 1.0, 4.0
    K = np.array([[w * w]])
    errs_u, errs_v = [], []
    taus = [0.2 / 2 ** i for i in range(5)] if k < 3 else [0.4 / 2 ** i for i in range(4)]
    for tau in taus:
        it = integrator.Integrator(np.eye(1), K, k, rho, tau, solver=lambda b: b)
        c = it.init(np.array([1.0]), np.array([0.0]))
        eu = ev = 0.0  # max error over the trajectory (robust to sign changes)
        for n in range(1, int(round(T / tau)) + 1):
            c = it.step(c)
            eu = max(eu, abs(c[0][0] - math.cos(w * n * tau)))
            ev = max(ev, abs(c[1][0] + w * math.sin(w * n * tau)))
        errs_u.append(eu)
        errs_v.append(ev)
    ou, ov = _orders(errs_u), _orders(errs_v)
    assert ou[-1] > 2 * k - 0.35, (ou, errs_u)
    assert ov[-1] > 2 * k - 0.35, (ov, errs_v)


@pytest.fixture(scope="module")
def c1_disc():
    cfg = synth.config("c1")
    prob = synth.make_problem(cfg)
    d = assembly.Discretization(prob["patches"], cfg["p"], cfg["n"], cfg["dim"])
    ev, Phi = sla.eigh(d.K.toarray(), d.M.toarray())
    return cfg, prob, d, ev, Phi


def _mnorm(M, x):
    return math.sqrt(x @ (M @ x))


def test_c1_lambda_max_and_cfl(c1_disc):
    cfg, prob, d, ev, Phi = c1_disc
    # identity map p=2: lambda_max h^2 = d * 10, i.e. 5120 for h = 1/16
    assert abs(ev[-1] - 5120.0) < 1e-8 * 5120
    dt = 0.5 * math.sqrt(params.theta_max_closed_form(0.5) / ev[-1])
    assert abs(dt - 0.0130427) < 1e-6


@pytest.mark.parametrize("k", [1, 2])
def test_c1_temporal_order_vs_semidiscrete_exact(c1_disc, k):
    # BASELINE.json configs[0]: dt = 0.5 CFL, 200 steps, then dt/2, /4, /8
    cfg, prob, d, ev, Phi = c1_disc
    M = d.M
    u0 = d.restrict_local([u[:, 0] for u in prob["u0"]])
    dt0 = 0.5 * math.sqrt(params.theta_max_closed_form(0.5) / ev[-1])
    T = 200 * dt0
    # U(t) = Phi cos(sqrt(Lambda) t) Phi^T M U0 (Phi M-orthonormal)
    coef = Phi.T @ (M @ u0)
    U_ex = Phi @ (np.cos(np.sqrt(ev) * T) * coef)
    V_ex = Phi @ (-np.sqrt(ev) * np.sin(np.sqrt(ev) * T) * coef)
    eu, evv = [], []
    for lvl in range(4):
        dt = dt0 / 2 ** lvl
        it = integrator.Integrator(M, d.K, k, 0.5, dt)
        c = it.run(u0, np.zeros_like(u0), 200 * 2 ** lvl)
        eu.append(_mnorm(M, c[0] - U_ex) / _mnorm(M, U_ex))
        evv.append(_mnorm(M, c[1] - V_ex) / _mnorm(M, V_ex))
    ou = _orders(eu)
    assert np.all(ou > 2 * k - 0.2), (ou, eu)
    assert _orders(evv)[-1] > 2 * k - 0.3


@pytest.mark.parametrize("k", [1, 2, 3])
@pytest.mark.parametrize("rho", [0.5, 1.0])
def test_c1_modal_exactness(c1_disc, k, rho):
    # n steps of the stepper equal the modal map sum_i phi_i G(tau^2 lambda_i)^n
    cfg, prob, d, ev, Phi = c1_disc
    M = d.M
    u0 = d.restrict_local([u[:, 0] for u in prob["u0"]])
    v0 = 0.3 * u0
    dt = 0.5 * math.sqrt(params.theta_max_closed_form(rho) / ev[-1])
    it = integrator.Integrator(M, d.K, k, rho, dt)
    chain = it.init(u0, v0)
    nst = 60
    c = it.run(None, None, nst, chain=chain)
    Md = M.toarray()
    # modal coordinates of the chain, scaled as [U, tau V, tau^2 A, ...]
    Z = np.stack([dt ** m * (Phi.T @ (Md @ chain[m])) for m in range(3 * k)])  # (3k, N)
    out = np.zeros_like(Z)
    for i in range(len(ev)):
        G = spectral.amplification(dt * dt * ev[i], k, rho)
        out[:, i] = np.linalg.matrix_power(G, nst) @ Z[:, i]
    for m in range(3):
        ref = Phi @ (out[m] / dt ** m)
        assert _mnorm(M, c[m] - ref) / _mnorm(M, ref) < 1e-10, m


def test_c1_spatial_convergence_closed_form():
    # exact u = cos(sqrt(2) pi t) sin(pi x) sin(pi y) (BASELINE.json configs[0]);
    # L2 projection of u0; error O(h^{p+1}) in L2
    errs = {}
    for p in (2, 3):
        for n in (4, 8, 16):
            ctrl = synth.control_net(2, p, n)
            d = assembly.Discretization([((0, 0), ctrl)], p, n, 2)
            Q = assembly.PatchQuad(ctrl, p, n, 2)
            free = assembly.interior_mask(n + p, 2)
            Bf = Q.B[:, free]
            xq = Q.B @ ctrl
            W = Q.w * Q.detJ
            u0q = np.sin(np.pi * xq[:, 0]) * np.sin(np.pi * xq[:, 1])
            U0 = integrator.DirectMassSolver(d.M)(Bf.T @ (W * u0q))
            T, dt = 0.5, 2.5e-3 / (n / 4)
            it = integrator.Integrator(d.M, d.K, 2, 0.5, dt)
            c = it.run(U0, np.zeros_like(U0), int(round(T / dt)))
            ex = math.cos(math.sqrt(2) * math.pi * T) * u0q
            e = Bf @ c[0] - ex
            errs[(p, n)] = math.sqrt((W * e * e).sum() / (W * ex * ex).sum())
    for p in (2, 3):
        r = _orders([errs[(p, n)] for n in (4, 8, 16)])
        assert r[-1] > p + 1 - 0.3, (p, r)
    assert 3e-5 < errs[(2, 16)] < 8e-5  # ~5.2e-5


@pytest.mark.parametrize("k", [1, 2])
def test_c1_energy_and_top_mode_dissipation(c1_disc, k):
    # Reading R4: the physical energy is not monotone, but on
    # smooth data its drift is bounded and the highest mode is damped (rho<1)
    cfg, prob, d, ev, Phi = c1_disc
    M, K = d.M, d.K
    dt = 0.5 * math.sqrt(params.theta_max_closed_form(0.5) / ev[-1])
    E = lambda c: 0.5 * (c[1] @ (M @ c[1]) + c[0] @ (K @ c[0]))
    u0 = d.restrict_local([u[:, 0] for u in prob["u0"]])
    it = integrator.Integrator(M, K, k, 0.5, dt)
    c = it.run(u0, np.zeros_like(u0), 200)
    E0 = E(it.init(u0, np.zeros_like(u0)))
    assert abs(E(c) / E0 - 1) < (5e-3 if k == 1 else 1e-5)
    top = Phi[:, -1]
    c = it.run(top, np.zeros_like(top), 200)
    assert E(c) / E(it.init(top, np.zeros_like(top))) < (0.01 if k == 1 else 0.95)


def test_c1_instability_above_cfl(c1_disc):
    # beyond Theta_max the top mode grows without bound (CFL condition)
    cfg, prob, d, ev, Phi = c1_disc
    top = Phi[:, -1]
    for fac, grows in ((0.97, False), (1.03, True)):
        dt = fac * math.sqrt(params.theta_max_closed_form(0.5) / ev[-1])
        it = integrator.Integrator(d.M, d.K, 2, 0.5, dt)
        c = it.run(top, np.zeros_like(top), 400)
        assert (np.abs(c[0]).max() > 1e3) == grows


def test_e1_closed_form_solves_the_wave_equation():
    # E1 (reading G24): u = sin(10 pi x) sin(10 pi y)[cos + sin](10 sqrt2 pi t) must
    # solve u_tt = Laplace(u) (omega = 1, f = 0) with u = 0 on the boundary of the unit square,
    # and the second return value must be u_t; checked by centred differences at random points
    rng = np.random.default_rng(3)
    pts = rng.uniform(0.0, 1.0, (50, 2))
    h, ht = 1e-4, 1e-5
    for t in (0.0, 0.037, 0.1):
        u, ut = synth.e1_exact(pts, t)
        up, _ = synth.e1_exact(pts, t + ht)
        um, _ = synth.e1_exact(pts, t - ht)
        np.testing.assert_allclose((up - um) / (2 * ht), ut, rtol=0, atol=1e-6 * np.abs(ut).max())
        utt = (up - 2 * u + um) / ht ** 2
        lap = 0.0
        for dx in (np.array([h, 0.0]), np.array([0.0, h])):
            lap = lap + (synth.e1_exact(pts + dx, t)[0] - 2 * u + synth.e1_exact(pts - dx, t)[0]) / h ** 2
        scale = 200 * np.pi ** 2 * np.abs(u).max()
        assert np.abs(utt - lap).max() < 1e-3 * scale
    edge = np.array([[0.0, 0.3], [1.0, 0.7], [0.4, 0.0], [0.6, 1.0]])
    assert np.abs(synth.e1_exact(edge, 0.05)[0]).max() < 1e-12


@pytest.mark.parametrize("k", [1, 2, 3])
def test_forced_scalar_ode_order_2k(k):
    # Forcing (eq:ho1, F^{(3j-3)} at t_n + alpha_fj tau; initial chain with F^{(m-2)}(0)):
    # u'' + w^2 u = cos(2t) + 0.5 cos(3t + 0.4), u(0) = 1, v(0) = 0.3, closed-form solution.
    # Evaluating the forcing at t_n instead of t_n + alpha_f tau (or dropping its derivatives
    # from the chain) breaks order 2k for k >= 2 -- this pins the reading.
    w, T, rho = 1.3, 4.0, 0.5
    terms = [(1.0, 2.0, 0.0), (0.5, 3.0, 0.4)]
    part = lambda t, d=0: sum(a / (w * w - om * om) * om ** d * math.cos(om * t + ph + d * math.pi / 2)
                              for a, om, ph in terms)
    A = 1.0 - part(0.0)
    B = (0.3 - part(0.0, 1)) / w
    ue = lambda t: A * math.cos(w * t) + B * math.sin(w * t) + part(t)
    ve = lambda t: -A * w * math.sin(w * t) + B * w * math.cos(w * t) + part(t, 1)
    F = integrator.Forcing(np.array([1.0]), terms)
    errs_u, errs_v = [], []
    taus = [0.2 / 2 ** i for i in range(5)] if k < 3 else [0.4 / 2 ** i for i in range(4)]
    for tau in taus:
        it = integrator.Integrator(np.eye(1), np.array([[w * w]]), k, rho, tau, solver=lambda b: b, forcing=F)
        c = it.init(np.array([1.0]), np.array([0.3]))
        eu = ev = 0.0
        for n in range(1, int(round(T / tau)) + 1):
            c = it.step(c)
            eu = max(eu, abs(c[0][0] - ue(n * tau)))
            ev = max(ev, abs(c[1][0] - ve(n * tau)))
        errs_u.append(eu)
        errs_v.append(ev)
    ou, ov = _orders(errs_u), _orders(errs_v)
    assert ou[-1] > 2 * k - 0.35, (ou, errs_u)
    assert ov[-1] > 2 * k - 0.35, (ov, errs_v)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_damped_scalar_ode_order_2k(k):
    # Damping (eq:ho1's C term, reading R16): u'' + 2 zeta w u' + w^2 u = 0, u(0) = 1, v(0) = 0,
    # exact u = e^{-zeta w t}(cos(wd t) + zeta w / wd sin(wd t)).  C acting on the old
    # velocity-level entry instead of its Taylor predictor drops the order to 1 for k >= 2.
    w, zeta, T, rho = 1.0, 0.15, 4.0, 0.5
    wd = w * math.sqrt(1 - zeta ** 2)
    ue = lambda t: math.exp(-zeta * w * t) * (math.cos(wd * t) + zeta * w / wd * math.sin(wd * t))
    errs = []
    taus = [0.2 / 2 ** i for i in range(5)] if k < 3 else [0.4 / 2 ** i for i in range(4)]
    for tau in taus:
        it = integrator.Integrator(np.eye(1), np.array([[w * w]]), k, rho, tau, solver=lambda b: b,
                                   C=np.array([[2 * zeta * w]]))
        c = it.init(np.array([1.0]), np.array([0.0]))
        e = 0.0
        for n in range(1, int(round(T / tau)) + 1):
            c = it.step(c)
            e = max(e, abs(c[0][0] - ue(n * tau)))
        errs.append(e)
    o = _orders(errs)
    assert o[-1] > 2 * k - 0.35, (o, errs)


@pytest.mark.parametrize("k", [1, 2])
def test_dirichlet_lift_exact_in_space(k):
    # Lifting: u = L(x, y) cos(2t), L = 1 + x + 2y, solves u_tt - Laplace u = f with
    # f = -4 L cos(2t) and u = L cos(2t) on the boundary.  On the identity map L lies in the spline
    # space (Greville control values reproduce linear functions), so the semi-discrete solution is
    # exact and the error is the time discretisation only: order 2k (with Rayleigh damping too).
    p, n = 2, 6
    ctrl = synth.control_net(2, p, n)
    Lc = 1.0 + ctrl[:, 0] + 2.0 * ctrl[:, 1]
    d = assembly.Discretization([((0, 0), ctrl)], p, n, 2)
    free = assembly.interior_mask(n + p, 2)
    Mfull, _ = assembly.patch_operators(ctrl, p, n, 2)
    hD = [(1.0, 2.0, 0.0)]
    for a0, a1 in ((0.0, 0.0), (0.7, 0.01)):
        # f = u_tt + C-term - Laplace u: with damping C = a0 M + a1 K the exact u needs
        # f = L (-4 cos 2t) + a0 L (-2 sin 2t) (K L = 0 up to the boundary: lifting handles it)
        GM, tM, GK, tK = assembly.dirichlet_lift(ctrl, p, n, 2, Lc, hD, a0, a1)
        Gf = (Mfull @ Lc)[free]  # int L B_i over free i (M applied to the exact coefficients)
        tf = [(-4.0, 2.0, 0.0), (2.0 * a0, 2.0, math.pi / 2)]
        F = integrator.ForcingSum([integrator.Forcing(Gf, tf), integrator.Forcing(GM, tM), integrator.Forcing(GK, tK)])
        C = a0 * d.M + a1 * d.K if (a0 or a1) else None
        errs = []
        for tau in (0.04, 0.02, 0.01):
            it = integrator.Integrator(d.M, d.K, k, 0.5, tau, forcing=F, C=C)
            c = it.run(Lc[free], np.zeros(d.nfree), int(round(1.0 / tau)))
            errs.append(np.abs(c[0] - Lc[free] * math.cos(2.0)).max())
        o = _orders(errs)
        assert o[-1] > 2 * k - 0.3, (a0, a1, o, errs)
