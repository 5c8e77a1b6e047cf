"""GPU parity of the elastic mass SpMV (M = density * scalar M per component) on
grids where the register-blocked row-tile kernel runs (k_spmv_rt: nx >= 32, ny >= 16, 3D;
DESIGN.md "Elastic mass SpMV"): full and ragged x / y tiles, one right-hand side (ga_apply) and
the k = 1..4 lock-stepped right-hand sides of the step's PCG, and sampled rows at C4's full size.

The oracle side is the scalar M of the same control net (oracle.assembly), applied per component;
the elastic K of the step relation comes from the library's own K apply, which the small-grid
parity tests (test_gpu_parity.py, elastic_p2) pin to the oracle."""
import numpy as np
import pytest

import synth
from oracle import assembly, params

pytestmark = pytest.mark.gpu


def _setup(p, n, k=2, dt=1e-3):
    import torch

    from paper_2102_11536_b200 import Context, make_desc
    cfg = synth.config("c4", p=p, n=n, k=k)
    prob = synth.make_problem(cfg)
    desc = make_desc(prob["patches"], p, n, 3, ncomp=3, k=k, rho=cfg["rho"], dt=dt, op_mode=1)
    return cfg, prob, Context(desc), torch


def _taylor(c, m, dt):
    out = np.zeros_like(c[m])
    f = 1.0
    for i in range(len(c) - m):
        out += f * c[m + i]
        f *= dt / (i + 1)
    return out


_MCACHE = {}


def _oracle_mass(prob, p, n):
    # scalar oracle M on the same (single-patch) control net: free DoFs in co-lexicographic
    # order = library order per component
    if n not in _MCACHE:
        _MCACHE[n] = assembly.Discretization(prob["patches"], p, n, 3).M.tocsr()
    return _MCACHE[n]


# k = number of lock-stepped right-hand sides of the PCG (KK template of the kernel: even KK
# stages 16-byte pairs, odd KK single doubles)
# free DoFs per direction n + p - 2: nx mod 32 = 0 (full x tiles), 2, 3, 6 (ragged last x tile)
@pytest.mark.parametrize("n,k", [(32, 2), (34, 2), (34, 1), (34, 4), (35, 3), (38, 2)],
                         ids=["full_tiles_k2", "rag2_k2", "rag2_k1", "rag2_k4", "rag3_k3", "rag6_k2"])
def test_elastic_mass_rowtiles_vs_oracle(n, k):
    p = 2
    cfg, prob, ctx, torch = _setup(p, n, k=k)
    M = _oracle_mass(prob, p, n)
    N = M.shape[0]
    rng = np.random.default_rng(21)
    x = rng.standard_normal(3 * N)
    y = ctx.apply("M", torch.tensor(x, device="cuda")).cpu().numpy()
    for c in range(3):
        ref = M @ x[c * N:(c + 1) * N]
        scale = abs(M).max() * np.abs(x).max()
        assert np.abs(y[c * N:(c + 1) * N] - ref).max() <= 1e-13 * scale, c
    # one step: the k lock-stepped mass solves (KK = k row tiles inside the PCG) solve
    # M y_j = -K s_j with the oracle's M (reading R1 for s_j)
    dt = 1e-3
    u0 = np.concatenate([prob["u0"][0][:, c].reshape((n + p,) * 3)[1:-1, 1:-1, 1:-1].reshape(-1) for c in range(3)])
    ctx.set_state(torch.tensor(u0, device="cuda"))
    c_old = [ctx.get_chain(q).cpu().numpy() for q in range(3 * k)]
    ctx.advance(1)
    assert ctx.stats().status == 0
    c_new = [ctx.get_chain(q).cpu().numpy() for q in range(3 * k)]
    al, be, ga, _ = params.scheme_params(k, cfg["rho"], 0)
    for j in range(1, k + 1):
        dsp, acc = 3 * j - 3, 3 * j - 1
        Ta = _taylor(c_old, acc, dt)
        y = Ta + al[j - 1] * (c_new[acc] - Ta)
        s = _taylor(c_old, dsp, dt) if j < k else c_old[dsp]
        Ks = ctx.apply("K", torch.tensor(s, device="cuda")).cpu().numpy()
        My = np.concatenate([M @ y[c * N:(c + 1) * N] for c in range(3)])
        assert np.linalg.norm(My + Ks) <= 1e-12 * np.linalg.norm(Ks), j


def test_elastic_mass_c4_full_size_sampled_rows():
    # BASELINE configs[3] grid: p = 4, n = 96, 3 x 98^3 DoFs; rows recomputed one by one
    p, n = 4, 96
    cfg, prob, ctx, torch = _setup(p, n)
    nf = n + p - 2
    N = nf ** 3
    ctrl = prob["patches"][0][1]
    rng = np.random.default_rng(12)
    picks = [(1, 1, 1), (nf, nf, nf), (nf, 1, nf // 2), (33, 17, 2), (32, 16, nf)] + \
        [tuple(rng.integers(1, nf + 1, 3)) for _ in range(3)]
    rows = assembly.operator_rows(ctrl, p, n, 3, picks)
    fidx = lambda ijk: (ijk[0] - 1) + nf * ((ijk[1] - 1) + nf * (ijk[2] - 1))
    x = torch.tensor(rng.standard_normal(3 * N), device="cuda")
    y = ctx.apply("M", x).cpu().numpy()
    xn = x.cpu().numpy()
    for ijk in picks:
        cols, mv, _ = rows[ijk]
        free = [(cc, mm) for cc, mm in zip(cols, mv) if all(1 <= cc[q] <= nf for q in range(3))]
        idx = np.array([fidx(cc) for cc, _ in free])
        for c in range(3):
            ref = sum(mm * xn[c * N + i] for (_, mm), i in zip(free, idx))
            sc = sum(abs(mm * xn[c * N + i]) for (_, mm), i in zip(free, idx))
            assert abs(y[c * N + fidx(ijk)] - ref) <= 1e-13 * sc, (ijk, c)
