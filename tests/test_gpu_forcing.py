"""GPU parity of the forcing term (eq:ho1 P:398-404, reading: block j takes
F^{(3j-3)} at t_n + alpha_fj tau, the initial chain F^{(m-2)}(t0)): F(x, t) = G(x) h(t) with a
sinusoidal h, set through ga_set_forcing, against the oracle (whose reading is pinned by
test_oracle_integrator.py::test_forced_scalar_ode_order_2k).  Plus a manufactured forced
solution u = sin(pi x) sin(pi y) h(t) on the GPU alone: order-2k self-convergence and a small
error against the closed form."""
import math

import numpy as np
import pytest

import synth
from oracle import assembly, integrator

from _helpers import Case, mnorm_rel

pytestmark = pytest.mark.gpu
TERMS = [(1.0, 30.0, 0.1), (0.3, 55.0, -0.7)]


@pytest.mark.parametrize("cfg,op_mode", [
    (synth.config("c2", n=10, k=2, rho=0.5), 0),
    (synth.config("c2", n=10, k=1, rho=0.0), 0),
    (synth.config("c3", p=2, n=5, k=3, rho=1.0), 0),
    (synth.config("c3", p=3, n=4, k=2, rho=0.5), 2),
    (synth.config("c3", p=3, n=4, k=2, rho=0.5), 3),
    (synth.config("c4", p=2, n=3), 0),
    (synth.config("c5", p=2, n=4), 0),
], ids=["2d_k2", "2d_k1", "3d_k3_rho1", "3d_matrix_free", "3d_half", "elastic", "lshape"])
def test_forcing_parity(cfg, op_mode):
    c = Case(cfg, op_mode=op_mode)
    d = c.disc
    u0 = c.u0()
    v0 = 0.3 * u0
    G = d.M @ np.cos(np.arange(d.M.shape[0]) * 0.37)  # any load vector; smooth-ish
    t0, nsteps = 0.2, 25
    c.ctx.set_forcing(c.to_lib(G), TERMS, t0)
    c.ctx.set_state(c.to_lib(u0), c.to_lib(v0))
    c.ctx.advance(nsteps)
    st = c.ctx.stats()
    assert st.status == 0 and st.steps == nsteps
    got = [c.from_lib(t) for t in c.ctx.get_state()]
    it = integrator.Integrator(d.M, d.K, cfg["k"], cfg["rho"], c.dt, forcing=integrator.Forcing(G, TERMS), t0=t0)
    ref = it.run(u0, v0, nsteps)
    errs = [mnorm_rel(d.M, x, y) for x, y in zip(got, ref[:3])]
    assert max(errs) < 1e-10, errs
    # removing the forcing restores the homogeneous step
    c.ctx.set_forcing(None)
    c.ctx.set_state(c.to_lib(u0), c.to_lib(v0))
    c.ctx.advance(5)
    ref0 = integrator.Integrator(d.M, d.K, cfg["k"], cfg["rho"], c.dt).run(u0, v0, 5)
    assert mnorm_rel(d.M, c.from_lib(c.ctx.get_state()[0]), ref0[0]) < 1e-10


def test_forced_manufactured_solution_order():
    # u = sin(pi x) sin(pi y) h(t), h = cos(3t) + 0.5 cos(5t + 0.3): u_tt - Laplace u =
    # sin sin (h'' + 2 pi^2 h) -> F = G h_F with G_i = int sin sin B_i, h_F terms a (2 pi^2 - w^2)
    import torch

    from paper_2102_11536_b200 import Context, make_desc
    p, n, k, rho, T = 3, 12, 2, 0.5, 0.3
    ctrl = synth.control_net(2, p, n)
    d = assembly.Discretization([((0, 0), ctrl)], p, n, 2)
    Q = assembly.PatchQuad(ctrl, p, n, 2)
    free = assembly.interior_mask(n + p, 2)
    Bf = Q.B[:, free]
    xq = Q.B @ ctrl
    W = Q.w * Q.detJ
    g = np.sin(np.pi * xq[:, 0]) * np.sin(np.pi * xq[:, 1])
    G = Bf.T @ (W * g)
    hterms = [(1.0, 3.0, 0.0), (0.5, 5.0, 0.3)]
    fterms = [(a * (2 * np.pi ** 2 - w * w), w, ph) for a, w, ph in hterms]
    h = lambda t, m=0: sum(a * w ** m * math.cos(w * t + ph + m * math.pi / 2) for a, w, ph in hterms)
    solve = integrator.DirectMassSolver(d.M)
    Pg = solve(G)  # L2 projection of sin sin
    sols = {}
    for N in (60, 120, 240):
        desc = make_desc([((0, 0), ctrl)], p, n, 2, k=k, rho=rho, dt=T / N)
        ctx = Context(desc)
        ctx.set_forcing(torch.tensor(G, device="cuda"), fterms, 0.0)
        ctx.set_state(torch.tensor(Pg * h(0.0), device="cuda"), torch.tensor(Pg * h(0.0, 1), device="cuda"))
        ctx.advance(N)
        assert ctx.stats().status == 0
        sols[N] = ctx.get_state()[0].cpu().numpy()
    M = d.M
    rel = lambda x, y: math.sqrt((x - y) @ (M @ (x - y)) / (y @ (M @ y)))
    d1, d2 = rel(sols[60], sols[120]), rel(sols[120], sols[240])
    assert math.log2(d1 / d2) > 2 * k - 0.4, (d1, d2)
    ex = g * h(T)
    e = Bf @ sols[240] - ex
    assert math.sqrt((W * e * e).sum() / (W * ex * ex).sum()) < 1e-4


@pytest.mark.parametrize("cfg,op_mode,forced", [
    (synth.config("c2", n=10, k=2, rho=0.5), 0, False),
    (synth.config("c2", n=10, k=3, rho=0.0), 0, True),
    (synth.config("c2", n=10, k=1, rho=0.5), 0, True),
    (synth.config("c3", p=2, n=5, k=2, rho=0.5), 0, True),
    (synth.config("c3", p=3, n=4, k=2, rho=0.5), 3, False),
    (synth.config("c3", p=3, n=4, k=2, rho=0.5), 2, True),
    (synth.config("c4", p=2, n=3), 0, False),
    (synth.config("c5", p=2, n=4), 0, True),
], ids=["2d_k2", "2d_k3_forced", "2d_k1_forced", "3d_forced", "3d_half", "3d_matrix_free_forced", "elastic",
        "lshape_forced"])
def test_rayleigh_damping_parity(cfg, op_mode, forced):
    # C = a0 M + a1 K (reading R16, pinned by test_oracle_integrator.py::test_damped_scalar_ode_order_2k)
    base = Case(cfg, op_mode=op_mode)
    lam = base.lam_max
    a0, a1 = 0.8 * math.sqrt(lam) * 0.05, 0.3 / math.sqrt(lam)
    c = Case(cfg, op_mode=op_mode, dt=base.dt, damp_a0=a0, damp_a1=a1)
    d = c.disc
    u0 = c.u0()
    v0 = -0.2 * u0
    F = None
    if forced:
        G = d.M @ np.cos(np.arange(d.M.shape[0]) * 0.37)
        c.ctx.set_forcing(c.to_lib(G), TERMS, 0.1)
        F = integrator.Forcing(G, TERMS)
    c.ctx.set_state(c.to_lib(u0), c.to_lib(v0))
    nsteps = 25
    c.ctx.advance(nsteps)
    st = c.ctx.stats()
    assert st.status == 0 and st.steps == nsteps
    got = [c.from_lib(t) for t in c.ctx.get_state()]
    it = integrator.Integrator(d.M, d.K, cfg["k"], cfg["rho"], c.dt, forcing=F, t0=0.1, C=a0 * d.M + a1 * d.K)
    ref = it.run(u0, v0, nsteps)
    errs = [mnorm_rel(d.M, x, y) for x, y in zip(got, ref[:3])]
    assert max(errs) < 1e-10, errs


def _lift_case(p, n, k, rho, dt, a0=0.0, a1=0.0, noise=0.0, seed=3):
    import torch

    from paper_2102_11536_b200 import Context, make_desc
    ctrl = synth.control_net(2, p, n, noise=noise, seed=seed)
    desc = make_desc([((0, 0), ctrl)], p, n, 2, k=k, rho=rho, dt=dt, damp_a0=a0, damp_a1=a1)
    return ctrl, Context(desc), torch


@pytest.mark.parametrize("a0,a1,forced", [(0.0, 0.0, False), (0.5, 0.002, True)])
def test_dirichlet_lifting_parity(a0, a1, forced):
    # S:230-239 lifting on a deformed patch: boundary values g_b h_D(t); GPU = oracle (dirichlet_lift)
    p, n, k, rho, dt, nsteps = 3, 10, 2, 0.5, 2e-3, 20
    ctrl, ctx, torch = _lift_case(p, n, k, rho, dt, a0, a1, noise=0.2)
    m = n + p
    g = np.cos(1.3 * ctrl[:, 0]) + ctrl[:, 1] ** 2  # any boundary data (interior entries unused)
    hD = [(1.0, 4.0, 0.2), (0.4, 7.0, -1.0)]
    d = assembly.Discretization([((0, 0), ctrl)], p, n, 2)
    free = assembly.interior_mask(m, 2)
    parts = []
    if forced:
        G = d.M @ np.cos(np.arange(d.nfree) * 0.37)
        ctx.set_forcing(torch.tensor(G, device="cuda"), TERMS, 0.0)
        parts.append(integrator.Forcing(G, TERMS))
    ctx.set_dirichlet(g, hD)
    GM, tM, GK, tK = assembly.dirichlet_lift(ctrl, p, n, 2, g, hD, a0, a1)
    parts += [integrator.Forcing(GM, tM), integrator.Forcing(GK, tK)]
    u0 = np.sin(np.arange(d.nfree) * 0.1)
    ctx.set_state(torch.tensor(u0, device="cuda"))
    ctx.advance(nsteps)
    assert ctx.stats().status == 0
    got = [t.cpu().numpy() for t in ctx.get_state()]
    C = a0 * d.M + a1 * d.K if (a0 or a1) else None
    ref = integrator.Integrator(d.M, d.K, k, rho, dt, forcing=integrator.ForcingSum(parts), C=C).run(
        u0, np.zeros(d.nfree), nsteps)
    errs = [mnorm_rel(d.M, x, y) for x, y in zip(got, ref[:3])]
    assert max(errs) < 1e-10, errs
    # removing the lifting restores the homogeneous problem (forcing kept)
    ctx.set_dirichlet(None)
    ctx.set_state(torch.tensor(u0, device="cuda"))
    ctx.advance(3)
    ref2 = integrator.Integrator(d.M, d.K, k, rho, dt, forcing=parts[0] if forced else None, C=C).run(
        u0, np.zeros(d.nfree), 3)
    assert mnorm_rel(d.M, ctx.get_state()[0].cpu().numpy(), ref2[0]) < 1e-10


def test_dirichlet_lifting_exact_in_space_order():
    # u = (1 + x + 2y) cos(2t) lies in the spline space on the identity map: the GPU error at
    # t = 1 is the time discretisation only, order 2k = 4 (k = 2)
    p, n, k = 2, 8, 2
    errs = []
    for tau in (0.04, 0.02, 0.01):
        ctrl, ctx, torch = _lift_case(p, n, k, 0.5, tau)
        free = assembly.interior_mask(n + p, 2)
        L = 1.0 + ctrl[:, 0] + 2.0 * ctrl[:, 1]
        Mfull, _ = assembly.patch_operators(ctrl, p, n, 2)
        ctx.set_forcing(torch.tensor((Mfull @ L)[free], device="cuda"), [(-4.0, 2.0, 0.0)], 0.0)
        ctx.set_dirichlet(L, [(1.0, 2.0, 0.0)])
        ctx.set_state(torch.tensor(L[free], device="cuda"))
        ctx.advance(int(round(1.0 / tau)))
        assert ctx.stats().status == 0
        errs.append(np.abs(ctx.get_state()[0].cpu().numpy() - L[free] * math.cos(2.0)).max())
    o = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert o[-1] > 2 * k - 0.3, (o, errs)
