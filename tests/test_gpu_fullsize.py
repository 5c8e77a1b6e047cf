"""Full-size GPU checks, in the configuration bench.py times.

* C2 (BASELINE configs[1]) end to end: 500 steps on the GPU against the
  stored oracle trajectory (tests/golden/make_c2_reference.py, oracle only),
  relative M-norm <= 1e-10 in u, v, a.
* C3 p=2 n=192 (7.1 M DoFs): sampled rows of M and K recomputed one by one by
  the oracle (assembly.operator_rows) against the GPU operators, and one GPU
  step checked at sampled rows through the step relations of P:408-431:
  M y_j = -K s_j with y_j = T_acc + alpha_j P_j, P_j recovered from the new
  acceleration, and the displacement/velocity updates elementwise."""
import math
import os

import numpy as np
import pytest

import synth
from oracle import assembly, params
from oracle.integrator import taylor

from _helpers import mnorm_rel

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _ctx(cfg, dt, op_mode=0):
    from paper_2102_11536_b200 import Context, make_desc
    prob = synth.make_problem(cfg)
    desc = make_desc(prob["patches"], cfg["p"], cfg["n"], cfg["dim"], k=cfg["k"], rho=cfg["rho"], dt=dt,
                     op_mode=op_mode)
    return prob, Context(desc)


def test_c2_full_size_500_steps():
    path = os.path.join(HERE, "golden", "c2_full_oracle.npz")
    if not os.path.exists(path):
        pytest.skip("run tests/golden/make_c2_reference.py first")
    import torch
    ref = np.load(path)
    cfg = synth.config("c2")
    prob, ctx = _ctx(cfg, float(ref["dt"]))
    d = assembly.Discretization(prob["patches"], cfg["p"], cfg["n"], cfg["dim"])
    u0 = d.restrict_local(prob["u0"])  # single patch: library order = oracle order
    ctx.set_state(torch.tensor(u0, device="cuda"))
    ctx.advance(int(ref["steps"]))
    st = ctx.stats()
    assert st.status == 0 and st.steps == int(ref["steps"])
    u, v, a = (t.cpu().numpy() for t in ctx.get_state())
    errs = [mnorm_rel(d.M, x, y) for x, y in zip((u, v, a), (ref["u"], ref["v"], ref["a"]))]
    assert max(errs) < 1e-10, errs


@pytest.mark.parametrize("op_mode", [1, 3, 2], ids=["stencil", "half_symmetric", "matrix_free"])
def test_c3_p2_n192_sampled_rows_and_one_step(op_mode):
    # every operator representation at the bench's largest grid (7.1 M DoFs)
    import torch
    cfg = synth.config("c3", p=2, n=192, k=2, rho=0.5)
    p, n, dim = cfg["p"], cfg["n"], 3
    m = n + p
    nf = m - 2
    dt = 2e-4
    prob, ctx = _ctx(cfg, dt, op_mode)
    assert ctx.operator_mode() == op_mode
    ctrl = prob["patches"][0][1]
    rng = np.random.default_rng(11)
    # free multi-indices: interior (1..m-2)^3; include faces/edges/corners of the free box
    picks = [(1, 1, 1), (nf, nf, nf), (1, nf // 2, nf), (nf // 2, 1, 2)] + [tuple(rng.integers(1, nf + 1, 3)) for _ in range(4)]
    rows = assembly.operator_rows(ctrl, p, n, dim, picks)
    fidx = lambda ijk: (ijk[0] - 1) + nf * ((ijk[1] - 1) + nf * (ijk[2] - 1))
    # --- operators
    x = torch.tensor(rng.standard_normal(nf ** 3), device="cuda")
    yM = ctx.apply("M", x).cpu().numpy()
    yK = ctx.apply("K", x).cpu().numpy()
    xn = x.cpu().numpy()
    for ijk in picks:
        cols, mv, kv = rows[ijk]
        free = [(c, mm, kk) for c, mm, kk in zip(cols, mv, kv) if all(1 <= c[q] <= nf for q in range(3))]
        idx = np.array([fidx(c) for c, _, _ in free])
        refM = sum(mm * xn[i] for (_, mm, _), i in zip(free, idx))
        refK = sum(kk * xn[i] for (_, _, kk), i in zip(free, idx))
        sM = sum(abs(mm * xn[i]) for (_, mm, _), i in zip(free, idx))
        sK = sum(abs(kk * xn[i]) for (_, _, kk), i in zip(free, idx))
        assert abs(yM[fidx(ijk)] - refM) <= 1e-13 * sM, ijk
        assert abs(yK[fidx(ijk)] - refK) <= 1e-12 * sK, ijk
    # --- one step from a smooth state
    u0 = prob["u0"][0][:, 0].reshape(m, m, m)[1:-1, 1:-1, 1:-1].reshape(-1)
    ctx.set_state(torch.tensor(u0, device="cuda"))
    k = cfg["k"]
    c_old = [ctx.get_chain(q).cpu().numpy() for q in range(3 * k)]
    ctx.advance(1)
    assert ctx.stats().status == 0
    c_new = [ctx.get_chain(q).cpu().numpy() for q in range(3 * k)]
    al, be, ga, _ = params.scheme_params(k, cfg["rho"], 0)
    for j in range(1, k + 1):
        dsp, vel, acc = 3 * j - 3, 3 * j - 2, 3 * j - 1
        Td, Tv, Ta = (taylor(c_old, q, dt) for q in (dsp, vel, acc))
        P = c_new[acc] - Ta
        np.testing.assert_allclose(c_new[dsp], Td + be[j - 1] * dt * dt * P, rtol=0, atol=1e-13 * np.abs(Td).max())
        np.testing.assert_allclose(c_new[vel], Tv + ga[j - 1] * dt * P, rtol=0, atol=1e-13 * np.abs(Tv).max())
        y = Ta + al[j - 1] * P            # the mass-solve result
        s = Td if j < k else c_old[dsp]    # reading R1
        for ijk in picks:
            cols, mv, kv = rows[ijk]
            free = [(c, mm, kk) for c, mm, kk in zip(cols, mv, kv) if all(1 <= c[q] <= nf for q in range(3))]
            idx = np.array([fidx(c) for c, _, _ in free])
            lhs = sum(mm * y[i] for (_, mm, _), i in zip(free, idx))
            rhs = -sum(kk * s[i] for (_, _, kk), i in zip(free, idx))
            scale = sum(abs(kk * s[i]) for (_, _, kk), i in zip(free, idx))
            # PCG at 1e-13 relative residual (2-norm over 7 M DoFs) bounds a single row loosely
            assert abs(lhs - rhs) <= 1e-9 * scale, (j, ijk, lhs, rhs, scale)
