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

from _helpers import Case, mnorm_rel, record_parity

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
    record_parity(errs, None, [1e-10] * 3, n_free=int(d.nfree), steps=int(ref["steps"]), full_size=True)
    assert max(errs) < 1e-10, errs


def test_c5_full_size_200_steps():
    # BASELINE configs[4] at full size (3 patches p=3 n=512, 790,533 DoFs, additive Schwarz,
    # P:737-783): 200 GPU steps against the stored oracle trajectory
    # (tests/golden/make_c5_reference.py, oracle only), relative M-norm <= 1e-10 in u, v, a
    path = os.path.join(HERE, "golden", "c5_full_oracle.npz")
    if not os.path.exists(path):
        pytest.skip("run tests/golden/make_c5_reference.py first")
    ref = np.load(path)
    cfg = synth.config("c5")
    c = Case(cfg, dt=float(ref["dt"]))  # the library context + the oracle's DoF order mapping
    d = c.disc
    assert d.nfree == int(ref["nfree"]) == 790533
    c.ctx.set_state(c.to_lib(c.u0()))
    c.ctx.advance(int(ref["steps"]))
    st = c.ctx.stats()
    assert st.status == 0 and st.steps == int(ref["steps"])
    got = [c.from_lib(t) for t in c.ctx.get_state()]
    errs = [mnorm_rel(d.M, x, y) for x, y in zip(got, (ref["u"], ref["v"], ref["a"]))]
    record_parity(errs, None, [1e-10] * 3, n_free=int(d.nfree), steps=int(ref["steps"]), full_size=True,
                  pcg_iters_per_solve=float(sum(st.pcg_iters) / max(1, st.solves)))
    assert max(errs) < 1e-10, errs
    c.ctx.close()


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


def _sampled_rows_and_one_step(cfg, op_mode, picks_extra, dt, tol_step=1e-9):
    """Sampled rows of M and K recomputed one by one by the oracle (assembly.operator_rows)
    against the GPU operators, then one GPU step checked at the sampled rows through the step
    relations of P:408-431 (M y_j = -K s_j, displacement / velocity updates elementwise)."""
    import torch
    p, n, dim = cfg["p"], cfg["n"], 3
    m = n + p
    nf = m - 2
    prob, ctx = _ctx(cfg, dt, op_mode)
    ctrl = prob["patches"][0][1]
    rng = np.random.default_rng(11)
    picks = [(1, 1, 1), (nf, nf, nf), (1, nf // 2, nf)] + picks_extra
    rows = assembly.operator_rows(ctrl, p, n, dim, picks)
    fidx = lambda ijk: (ijk[0] - 1) + nf * ((ijk[1] - 1) + nf * (ijk[2] - 1))
    x = torch.tensor(rng.standard_normal(nf ** 3), device="cuda")
    yM = ctx.apply("M", x).cpu().numpy()
    yK = ctx.apply("K", x).cpu().numpy()
    xn = x.cpu().numpy()
    worst = 0.0
    for ijk in picks:
        cols, mv, kv = rows[ijk]
        free = [(c, mm, kk) for c, mm, kk in zip(cols, mv, kv) if all(1 <= c[q] <= nf for q in range(3))]
        idx = np.array([fidx(c) for c, _, _ in free])
        refM = sum(mm * xn[i] for (_, mm, _), i in zip(free, idx))
        refK = sum(kk * xn[i] for (_, _, kk), i in zip(free, idx))
        sM = sum(abs(mm * xn[i]) for (_, mm, _), i in zip(free, idx))
        sK = sum(abs(kk * xn[i]) for (_, _, kk), i in zip(free, idx))
        worst = max(worst, abs(yM[fidx(ijk)] - refM) / sM, abs(yK[fidx(ijk)] - refK) / sK)
        assert abs(yM[fidx(ijk)] - refM) <= 1e-13 * sM, ijk
        assert abs(yK[fidx(ijk)] - refK) <= 1e-12 * sK, ijk
    u0 = prob["u0"][0][:, 0].reshape(m, m, m)[1:-1, 1:-1, 1:-1].reshape(-1)
    ctx.set_state(torch.tensor(u0, device="cuda"))
    k = cfg["k"]
    c_old = [ctx.get_chain(q).cpu().numpy() for q in range(3 * k)]
    ctx.advance(1)
    assert ctx.stats().status == 0
    c_new = [ctx.get_chain(q).cpu().numpy() for q in range(3 * k)]
    al, be, ga, _ = params.scheme_params(k, cfg["rho"], 0)
    wstep = 0.0
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
            if scale > 0:
                wstep = max(wstep, abs(lhs - rhs) / scale)
            assert abs(lhs - rhs) <= tol_step * scale, (j, ijk, lhs, rhs, scale)
    record_parity([worst, wstep, 0.0], None, None, kind="sampled rows (operator rel err, step-relation rel err)",
                  p=p, n=n, operator_mode=ctx.operator_mode(), full_size=True)
    ctx.close()
    del ctx
    torch.cuda.empty_cache()


def test_c3_p6_n192_half_symmetric_sampled_rows_and_one_step():
    # the bench's headline workload (BASELINE configs[2] at "~7.5M DoFs": p = 6, n = 192,
    # 7,529,536 DoFs), in the representation op_mode 0 picks there (half-symmetric stencils,
    # single-read SpMV); rows spread over x-segments (incl. the partial last one), y-tiles, z-chunks
    cfg = synth.config("c3", p=6, n=192, k=2, rho=0.0)
    nf = cfg["n"] + cfg["p"] - 2
    extra = [(nf // 2, 37, 101), (193, 5, 64), (33, 190, 2)]
    _sampled_rows_and_one_step(cfg, 0, extra, dt=2.5e-4)


def test_c4_full_size_elastic_stiffness_sampled_rows():
    # BASELINE configs[3] grid (p = 4, n = 96, 3 x 98^3 DoFs): rows of the elastic 3x3-block K
    # recomputed one by one by the oracle (assembly.elastic_operator_rows, lam = mu = 1)
    import torch

    from paper_2102_11536_b200 import Context, make_desc
    p, n = 4, 96
    cfg = synth.config("c4", p=p, n=n)
    prob = synth.make_problem(cfg)
    ctx = Context(make_desc(prob["patches"], p, n, 3, ncomp=3, k=2, rho=cfg["rho"], dt=1e-4, lam=cfg["lam"],
                            mu=cfg["mu"], density=cfg["density"]))
    nf = n + p - 2
    N = nf ** 3
    ctrl = prob["patches"][0][1]
    rng = np.random.default_rng(13)
    picks = [(1, 1, 1), (nf, nf, nf), (nf, 1, nf // 2), (33, 17, 2)] + [tuple(rng.integers(1, nf + 1, 3))
                                                                       for _ in range(3)]
    rows = assembly.elastic_operator_rows(ctrl, p, n, picks, lam=cfg["lam"], mu=cfg["mu"])
    fidx = lambda ijk: (ijk[0] - 1) + nf * ((ijk[1] - 1) + nf * (ijk[2] - 1))
    x = torch.tensor(rng.standard_normal(3 * N), device="cuda")
    y = ctx.apply("K", x).cpu().numpy()
    xn = x.cpu().numpy().reshape(3, N)
    worst = 0.0
    for ijk in picks:
        cols, vals = rows[ijk]
        keep = [q for q, c in enumerate(cols) if all(1 <= c[t] <= nf for t in range(3))]
        idx = np.array([fidx(cols[q]) for q in keep])
        V = vals[keep]                               # (ncols, 3, 3)
        for a in range(3):
            ref = sum(V[:, a, b] @ xn[b, idx] for b in range(3))
            sc = sum(np.abs(V[:, a, b]) @ np.abs(xn[b, idx]) for b in range(3))
            err = abs(y[a * N + fidx(ijk)] - ref)
            worst = max(worst, err / sc)
            assert err <= 1e-12 * sc, (ijk, a, err, sc)
    record_parity([worst], None, None, kind="sampled rows of the elastic K (rel err)", p=p, n=n, full_size=True)
    ctx.close()
