"""GPU tests of the state-keeping parts of the C ABI (include/genalpha.h): the instability
detector's reference for runs that start from rest, the forcing clock across a checkpoint /
resume (ga_set_chain + ga_set_time, eq:ho1 P:398-404: block j takes F^{(3j-3)} at
t_n + alpha_fj tau, so t_n must survive a resume), ga_lambda_max leaving the statistics and the
predictors untouched, and ga_profile_op doing real work on an active PCG state."""
import numpy as np
import pytest

import synth
from oracle import integrator

from _helpers import Case, mnorm_rel

pytestmark = pytest.mark.gpu
TERMS = [(1.0, 30.0, 0.1), (0.3, 55.0, -0.7)]


def test_start_from_rest_with_velocity_is_not_unstable():
    # U0 = 0, V0 != 0: the old detector compared ||U_n||^2 with 1e12 * ||U0||^2 = 0 and failed
    # at step 1; the reference is now ||U0||^2 + dt^2 ||V0||^2
    cfg = synth.config("c2", n=10, k=2, rho=0.5)
    c = Case(cfg)
    d = c.disc
    v0 = c.u0() * 3.0
    u0 = np.zeros_like(v0)
    c.ctx.set_state(c.to_lib(u0), c.to_lib(v0))
    c.ctx.advance(30)
    st = c.ctx.stats()
    assert st.status == 0 and st.steps == 30, (st.status, st.steps)
    ref = integrator.Integrator(d.M, d.K, cfg["k"], cfg["rho"], c.dt).run(u0, v0, 30)
    got = [c.from_lib(t) for t in c.ctx.get_state()]
    assert max(mnorm_rel(d.M, x, y) for x, y in zip(got, ref[:3])) < 1e-10


def test_forced_run_from_rest_is_not_unstable():
    # U0 = V0 = 0 and F != 0: the reference is 0 until the first non-zero ||U_n||^2 is adopted
    cfg = synth.config("c2", n=10, k=2, rho=0.5)
    c = Case(cfg)
    d = c.disc
    G = d.M @ np.cos(np.arange(d.nfree) * 0.37)
    z = np.zeros(d.nfree)
    c.ctx.set_forcing(c.to_lib(G), TERMS, 0.0)
    c.ctx.set_state(c.to_lib(z), c.to_lib(z))
    c.ctx.advance(25)
    st = c.ctx.stats()
    assert st.status == 0 and st.steps == 25, (st.status, st.steps)
    ref = integrator.Integrator(d.M, d.K, cfg["k"], cfg["rho"], c.dt, forcing=integrator.Forcing(G, TERMS)).run(
        z, z, 25)
    got = [c.from_lib(t) for t in c.ctx.get_state()]
    assert max(mnorm_rel(d.M, x, y) for x, y in zip(got, ref[:3])) < 1e-10


def test_instability_still_detected_from_rest():
    # the adopted reference still catches a blow-up: dt well above the CFL limit
    cfg = synth.config("c2", n=10, k=2, rho=0.5)
    base = Case(cfg)
    c = Case(cfg, dt=base.dt * 3.0)
    d = c.disc
    G = d.M @ np.cos(np.arange(d.nfree) * 0.37)
    z = np.zeros(d.nfree)
    c.ctx.set_forcing(c.to_lib(G), TERMS, 0.0)
    c.ctx.set_state(c.to_lib(z), c.to_lib(z))
    c.ctx.advance(400)
    assert c.ctx.stats().status == -6  # GA_ERR_UNSTABLE


@pytest.mark.parametrize("fresh", [False, True], ids=["same_context", "fresh_context"])
def test_checkpoint_resume_with_forcing(fresh):
    cfg = synth.config("c2", n=10, k=2, rho=0.5)
    c = Case(cfg)
    d = c.disc
    G = d.M @ np.cos(np.arange(d.nfree) * 0.37)
    u0 = c.u0()
    v0 = 0.3 * u0
    t0, n1, n2 = 0.2, 12, 13
    c.ctx.set_forcing(c.to_lib(G), TERMS, t0)
    c.ctx.set_state(c.to_lib(u0), c.to_lib(v0))
    c.ctx.advance(n1)
    chain = [c.ctx.get_chain(m).clone() for m in range(3 * cfg["k"])]
    assert c.ctx.stats().step_index == n1
    if fresh:
        r = Case(cfg, dt=c.dt)
        r.ctx.set_forcing(r.to_lib(G), TERMS, t0)
        tgt = r
    else:
        c.ctx.advance(7)  # move on, then roll back to the checkpoint
        tgt = c
    for m, x in enumerate(chain):
        tgt.ctx.set_chain(m, x)
    if fresh:
        assert tgt.ctx.stats().step_index == 0
        tgt.ctx.set_time(n1)
    else:
        # set_chain keeps the clock of the state it was on: put it back to the checkpoint's
        tgt.ctx.set_time(n1)
    tgt.ctx.advance(n2)
    st = tgt.ctx.stats()
    assert st.status == 0 and st.steps == n2 and st.step_index == n1 + n2
    ref = integrator.Integrator(d.M, d.K, cfg["k"], cfg["rho"], c.dt, forcing=integrator.Forcing(G, TERMS),
                                t0=t0).run(u0, v0, n1 + n2)
    got = [tgt.from_lib(t) for t in tgt.ctx.get_state()]
    assert max(mnorm_rel(d.M, x, y) for x, y in zip(got, ref[:3])) < 1e-10


def test_set_chain_keeps_the_clock():
    cfg = synth.config("c2", n=8, k=2, rho=0.5)
    c = Case(cfg)
    c.ctx.set_state(c.to_lib(c.u0()))
    c.ctx.advance(5)
    x = c.ctx.get_chain(0).clone()
    c.ctx.set_chain(0, x)
    st = c.ctx.stats()
    assert st.steps == 0 and st.step_index == 5


def test_lambda_max_leaves_stats_and_state():
    cfg = synth.config("c2", n=10, k=2, rho=0.5)
    c = Case(cfg)
    c.ctx.set_state(c.to_lib(c.u0()))
    c.ctx.advance(4)
    before = c.ctx.stats()
    chain = [c.ctx.get_chain(m).cpu().numpy() for m in range(6)]
    lam = c.ctx.lambda_max(40)
    after = c.ctx.stats()
    assert abs(lam - c.lam_max) < 1e-6 * c.lam_max
    for f in ("steps", "solves", "status", "loop_iters", "step_index"):
        assert getattr(after, f) == getattr(before, f), f
    assert list(after.pcg_iters) == list(before.pcg_iters)
    for m in range(6):
        assert np.array_equal(c.ctx.get_chain(m).cpu().numpy(), chain[m])
    # stepping continues exactly as without the Lanczos call
    ref = Case(cfg, dt=c.dt)
    ref.ctx.set_state(ref.to_lib(ref.u0()))
    ref.ctx.advance(7)
    c.ctx.advance(3)
    assert np.array_equal(c.ctx.get_state()[0].cpu().numpy(), ref.ctx.get_state()[0].cpu().numpy())


def test_lambda_max_noconv_not_latched():
    # pcg_maxit = 1 makes every Lanczos solve fail: the call reports NOCONV, the context's status
    # stays clean (the time stepping was never run)
    from paper_2102_11536_b200 import GAError
    cfg = synth.config("c2", n=10, k=2, rho=0.5)
    c = Case(cfg, pcg_maxit=1)
    with pytest.raises(GAError) as e:
        c.ctx.lambda_max(5)
    assert e.value.code == -5
    assert c.ctx.stats().status == 0


@pytest.mark.parametrize("op", [2, 5])
def test_profile_op_leaves_stepping_intact(op):
    # ops 2 (preconditioner) and 5 (p = z + beta p) run on an active profiling PcgState (their
    # full work, for the bench's per-kernel timing); the PcgState is zeroed afterwards, so the
    # next step is the same as without profiling
    import torch
    cfg = synth.config("c3", p=2, n=6, k=2, rho=0.0)
    c = Case(cfg)
    c.ctx.set_state(c.to_lib(c.u0()))
    c.ctx.advance(1)
    torch.cuda.synchronize()
    c0 = c.ctx.stats().kernel_launches
    c.ctx.profile_op(op, 3)
    torch.cuda.synchronize()
    assert c.ctx.stats().kernel_launches > c0
    c.ctx.advance(1)
    assert c.ctx.stats().status == 0
    ref = Case(cfg, dt=c.dt)
    ref.ctx.set_state(ref.to_lib(ref.u0()))
    ref.ctx.advance(2)
    assert np.array_equal(c.ctx.get_state()[0].cpu().numpy(), ref.ctx.get_state()[0].cpu().numpy())
