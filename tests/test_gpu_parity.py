"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Operators and the preconditioner element by element;
solves and trajectories in the relative M-norm (= L2(Omega), DESIGN.md
"Parity metric") with the bar of BASELINE.json (1e-10)."""
import math

import numpy as np
import pytest

import synth
from oracle import integrator, precond

from _helpers import Case, mnorm_rel, oracle_with_floor, record_parity

pytestmark = pytest.mark.gpu

OP_CASES = {
    "2d_p2_identity": synth.config("c1", n=8),
    "2d_p3_deformed": synth.config("c2", n=10),
    "2d_p1": synth.config("c2", p=1, n=9),
    "3d_p2": synth.config("c3", p=2, n=4),
    "3d_p3": synth.config("c3", p=3, n=3),
    "3d_p5": synth.config("c3", p=5, n=2),
    "elastic_p2": synth.config("c4", p=2, n=3),
    # C4's configured degree, and lam != mu (a lam <-> mu swap or a mu-for-2mu slip would show)
    "elastic_p4": synth.config("c4", p=4, n=2),
    "elastic_p3_lam2_mu05": synth.config("c4", p=3, n=2, lam=2.0, mu=0.5),
    "lshape_p2": synth.config("c5", p=2, n=4),
    "lshape_p3": synth.config("c5", p=3, n=5),
}


@pytest.fixture(scope="module", params=sorted(OP_CASES))
def case(request):
    return Case(OP_CASES[request.param])


def test_operators_elementwise(case):
    d = case.disc
    rng = np.random.default_rng(7)
    for which, A in (("M", d.M), ("K", d.K)):
        x = rng.standard_normal(A.shape[0])
        y = case.from_lib(case.ctx.apply(which, case.to_lib(x)))
        ref = A @ x
        scale = np.abs(A).max() * np.abs(x).max()
        assert np.abs(y - ref).max() <= 1e-13 * scale, which
    # unit vectors: exact columns
    for col in [0, d.M.shape[0] // 2, d.M.shape[0] - 1]:
        e = np.zeros(d.M.shape[0]); e[col] = 1.0
        y = case.from_lib(case.ctx.apply("M", case.to_lib(e)))
        np.testing.assert_allclose(y, d.M[:, col].toarray().ravel(), rtol=1e-13, atol=1e-15 * abs(d.M[col, col]))


def test_preconditioner_elementwise(case):
    P = precond.SchwarzPreconditioner(case.disc)
    x = np.random.default_rng(8).standard_normal(case.disc.M.shape[0])
    y = case.from_lib(case.ctx.apply("Pinv", case.to_lib(x)))
    ref = P(x)
    assert np.abs(y - ref).max() <= 1e-11 * np.abs(ref).max()


def test_mass_solve(case):
    d = case.disc
    b = d.K @ case.u0()
    x, its = case.ctx.solve_mass(case.to_lib(b))
    x = case.from_lib(x)
    ref = integrator.DirectMassSolver(d.M)(b)
    # ||r|| <= 1e-13 ||b|| bounds the relative M-norm error by 1e-13 sqrt(kappa(M));
    # kappa(M) reaches ~1e7 at 3D p=5, hence the looser bar there
    assert mnorm_rel(d.M, x, ref) < (1e-12 if case.cfg["p"] <= 4 else 2e-11)
    assert np.linalg.norm(b - d.M @ x) <= 1.01e-13 * np.linalg.norm(b)
    if case.cfg["noise"] == 0.0 and not case.cfg.get("lshape"):
        assert its == 1  # identity map: calM = M


def test_initial_chain(case):
    d = case.disc
    u0 = case.u0()
    v0 = 0.5 * u0
    case.ctx.set_state(case.to_lib(u0), case.to_lib(v0))
    it = integrator.Integrator(d.M, d.K, case.cfg["k"], case.cfg["rho"], case.dt)
    ref = it.init(u0, v0)
    for m in range(3 * case.cfg["k"]):
        got = case.from_lib(case.ctx.get_chain(m))
        # conditioning of M at high p (kappa ~1e7 at 3D p=5) amplifies rounding per solve
        assert mnorm_rel(d.M, got, ref[m]) < (1e-11 if case.cfg["p"] <= 4 else 1e-9), m
    assert case.ctx.stats().status == 0


def _trajectory(cfg, nsteps, tol=1e-10, v0fac=0.0, **kw):
    """Bar: relative M-norm
    <= max(tol, 10 F), F = the oracle-vs-oracle rounding floor: max of (LU + refinement
    vs dense Cholesky) and (Gauss points summed in reverse order) on the same case."""
    c = Case(cfg, **kw)
    d = c.disc
    u0 = c.u0()
    v0 = v0fac * u0
    c.ctx.set_state(c.to_lib(u0), c.to_lib(v0) if v0fac else None)
    c.ctx.advance(nsteps)
    st = c.ctx.stats()
    assert st.status == 0, st.status
    assert st.steps == nsteps
    u, v, a = (c.from_lib(t) for t in c.ctx.get_state())
    ps = kw.get("param_set", 0)
    ref, floor = oracle_with_floor(d, cfg["k"], cfg["rho"], c.dt, u0, v0, nsteps, ps, case=c)
    errs = [mnorm_rel(d.M, x, y) for x, y in zip((u, v, a), ref[:3])]
    bar = [max(tol, 10 * f) for f in floor]
    record_parity(errs, floor, bar, n_free=int(d.nfree * d.ncomp), steps=nsteps, p=cfg["p"], k=cfg["k"],
                  rho=cfg["rho"], operator_mode=c.ctx.operator_mode())
    assert all(e < b for e, b in zip(errs, bar)), (errs, floor)
    return c, errs, st


@pytest.mark.parametrize("k", [1, 2])
def test_c1_full(k):
    # BASELINE.json configs[0] at full size: 2D p=2 n=16, rho=0.5, 0.5 CFL, 200 steps
    _trajectory(synth.config("c1", k=k), 200)


def test_c2_reduced():
    _trajectory(synth.config("c2", n=24), 100)


@pytest.mark.parametrize("p,k,rho", [(2, 1, 0.0), (2, 2, 0.5), (2, 3, 1.0), (3, 2, 0.0), (3, 3, 0.5),
                                     (4, 2, 0.5), (4, 3, 0.0), (5, 1, 1.0), (6, 2, 0.0)])
def test_c3_reduced(p, k, rho):
    n = {2: 6, 3: 5, 4: 4, 5: 3, 6: 3}[p]
    _trajectory(synth.config("c3", p=p, n=n, k=k, rho=rho), 40)


def test_c4_reduced():
    _trajectory(synth.config("c4", p=2, n=3), 20)


@pytest.mark.parametrize("p,n,lam,mu", [(4, 3, 1.0, 1.0), (4, 2, 2.0, 0.5), (3, 4, 0.7, 1.3)],
                         ids=["p4_n3", "p4_n2_lam2_mu05", "p3_n4_lam07_mu13"])
def test_c4_configured_degree_and_lame(p, n, lam, mu):
    # BASELINE configs[3] at its configured p = 4 (reduced n), and with lam != mu
    _trajectory(synth.config("c4", p=p, n=n, lam=lam, mu=mu), 20)


@pytest.mark.parametrize("p,n,k,rho", [(2, 16, 2, 0.0), (3, 12, 2, 0.5), (4, 8, 3, 0.0), (4, 8, 2, 1.0)])
def test_c3_larger_grids(p, n, k, rho):
    # C3 trajectories on grids of 1e3-4e3 DoFs per direction product (n = 8-32)
    _trajectory(synth.config("c3", p=p, n=n, k=k, rho=rho), 40)


def test_c5_reduced():
    _trajectory(synth.config("c5", p=3, n=8), 50)


def test_nonzero_velocity_and_k4():
    _trajectory(synth.config("c2", n=8, k=4, rho=0.5), 30, v0fac=0.7)


def test_printed_parameter_set():
    _trajectory(synth.config("c1", k=2, rho=0.3), 50, param_set=1)


def test_zero_steps_and_checkpoint_resume():
    c = Case(synth.config("c2", n=10))
    u0 = c.u0()
    c.ctx.set_state(c.to_lib(u0))
    c.ctx.advance(0)
    u, _, _ = c.ctx.get_state()
    np.testing.assert_array_equal(c.from_lib(u), u0)
    c.ctx.advance(7)
    chain = [c.ctx.get_chain(m).clone() for m in range(3 * c.cfg["k"])]
    c.ctx.advance(5)
    u12 = c.from_lib(c.ctx.get_state()[0])
    for m, t in enumerate(chain):
        c.ctx.set_chain(m, t)
    c.ctx.advance(5)
    np.testing.assert_array_equal(c.from_lib(c.ctx.get_state()[0]), u12)  # deterministic resume


def test_lambda_max():
    c = Case(synth.config("c1"))
    lam = c.ctx.lambda_max(200)
    assert abs(lam - 5120.0) / 5120.0 < 1e-9  # Lanczos (C1 closed form)


def test_noconv_reported():
    c = Case(synth.config("c2", n=10), pcg_maxit=2)
    c.ctx.set_state(c.to_lib(c.u0()))
    c.ctx.advance(3)
    st = c.ctx.stats()
    assert st.status == -5 and st.fail_block >= 0


def test_geometry_error():
    from paper_2102_11536_b200 import GAError, make_desc, Context
    p, n = 2, 4
    ctrl = synth.control_net(2, p, n)
    m = n + p
    ctrl = ctrl.copy()
    # fold the map: swap two interior columns of control points
    a, b = 2 + m * 2, 3 + m * 2
    ctrl[[a, b]] = ctrl[[b, a]]
    ctrl[a, 0] += 0.4
    with pytest.raises(GAError) as ei:
        Context(make_desc([((0, 0), ctrl)], p, n, 2, k=1, rho=0.5, dt=1e-3))
    assert ei.value.code == -3
