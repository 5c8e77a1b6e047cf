"""GPU edge cases of the hot path (degenerate sizes and data, error reporting):
* the smallest grids (one free DoF in 2D and 3D; p = 1 with n = 2) against the oracle,
  with every operator representation (full / half-symmetric stencils, matrix-free);
* zero initial data: every right-hand side is zero, the solves are skipped, the state
  stays exactly zero;
* a time step above the stability limit (Theta_max of R9): GA_ERR_UNSTABLE with
  the failing step reported, and further stepping refused until ga_set_state;
* non-conforming multi-patch interfaces: GA_ERR_CONFORMITY;
* op_mode validation (GA_ERR_ARG)."""
import math

import numpy as np
import pytest

import synth
from oracle import params

from _helpers import Case, mnorm_rel, oracle_with_floor

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("op_mode", [1, 2, 3])
@pytest.mark.parametrize("cfg", [synth.config("c2", p=2, n=1), synth.config("c3", p=2, n=1),
                                 synth.config("c2", p=1, n=2), synth.config("c3", p=3, n=1, k=3)],
                         ids=["2d_one_dof", "3d_one_dof", "2d_p1_n2", "3d_p3_n1_k3"])
def test_smallest_grids(cfg, op_mode):
    c = Case(cfg, op_mode=op_mode)
    d = c.disc
    u0 = c.u0()
    if not np.any(u0):
        u0 = np.ones_like(u0)
    c.ctx.set_state(c.to_lib(u0))
    c.ctx.advance(10)
    st = c.ctx.stats()
    assert st.status == 0
    u, v, a = (c.from_lib(t) for t in c.ctx.get_state())
    ref, floor = oracle_with_floor(d, cfg["k"], cfg["rho"], c.dt, u0, np.zeros_like(u0), 10, case=c)
    errs = [mnorm_rel(d.M, x, y) for x, y in zip((u, v, a), ref[:3])]
    assert all(e < max(1e-10, 10 * f) for e, f in zip(errs, floor)), (errs, floor)


def test_zero_data_stays_zero():
    c = Case(synth.config("c2", n=12))
    z = np.zeros(c.disc.nfree)
    c.ctx.set_state(c.to_lib(z))
    c.ctx.advance(5)
    st = c.ctx.stats()
    assert st.status == 0
    for t in c.ctx.get_state():
        assert not np.any(t.cpu().numpy())


def test_unstable_time_step_reported():
    cfg = synth.config("c2", n=10, rho=0.5)
    base = Case(cfg)
    lam = base.lam_max
    dt = 1.5 * math.sqrt(params.theta_max_closed_form(0.5) / lam)  # 1.5x the stability limit
    c = Case(cfg, dt=dt, unstable_factor=1e3)
    c.ctx.set_state(c.to_lib(c.u0()))
    c.ctx.advance(400)
    st = c.ctx.stats()
    assert st.status == -6 and 0 < st.fail_step < 400, (st.status, st.fail_step)
    steps = st.steps
    c.ctx.advance(5)  # refused: no further steps after a device-side failure
    assert c.ctx.stats().steps == steps
    c.ctx.set_state(c.to_lib(c.u0()))  # reset clears the failure
    assert c.ctx.stats().status == 0


def test_nonconforming_interfaces_rejected():
    from paper_2102_11536_b200 import Context, GAError, make_desc
    cfg = synth.config("c5", p=2, n=4)
    prob = synth.make_problem(cfg)
    patches = [(cell, ctrl.copy()) for cell, ctrl in prob["patches"]]
    m = cfg["n"] + cfg["p"]
    cell, ctrl = patches[1]
    # move one control point on patch 1's interface (local x index 0) off the shared edge
    ctrl[0 + m * (m // 2), 1] += 1e-3
    with pytest.raises(GAError) as ei:
        Context(make_desc(patches, cfg["p"], cfg["n"], 2, k=2, rho=0.3, dt=1e-4))
    assert ei.value.code == -4


def test_op_mode_validation():
    from paper_2102_11536_b200 import Context, GAError, make_desc
    cfg = synth.config("c2", n=6)
    prob = synth.make_problem(cfg)
    with pytest.raises(GAError) as ei:
        Context(make_desc(prob["patches"], cfg["p"], cfg["n"], 2, k=2, rho=0.0, dt=1e-4, op_mode=7))
    assert ei.value.code == -1


@pytest.mark.parametrize("cfg", [synth.config("c1"), synth.config("c2", n=12), synth.config("c3", p=3, n=4),
                                 synth.config("c4", p=2, n=3), synth.config("c5", p=2, n=4)],
                         ids=["c1", "2d_deformed", "3d_p3", "elastic", "lshape"])
def test_lambda_max_lanczos(cfg):
    # ga_lambda_max (Lanczos in the M inner product) against the oracle's
    # generalized eigensolver; the time-stepping state must be left unchanged
    c = Case(cfg)
    u0 = c.u0()
    c.ctx.set_state(c.to_lib(u0))
    c.ctx.advance(2)
    before = [t.clone() for t in c.ctx.get_state()]
    lam = c.ctx.lambda_max(80)
    assert abs(lam - c.lam_max) <= 1e-8 * c.lam_max, (lam, c.lam_max)
    after = c.ctx.get_state()
    for x, y in zip(before, after):
        assert bool((x == y).all())
    c.ctx.advance(1)
    assert c.ctx.stats().status == 0
