"""Memory and race checks of every kernel family without compute-sanitizer (closed on the GPU
pool, profiles/r02_sanitizer_closed.txt): the workspace is placed between 1 MiB canary regions
(a write outside the workspace's ends is caught), and every case is run twice from fresh contexts
and compared - bitwise for the deterministic paths (a data race shows up as run-to-run noise),
to 1e-10 (the parity bar) for the single-read symmetric SpMV (its L2 reductions round in
run-dependent order, and the PCG solves amplify the last bits by the conditioning).  The cases are those of tools/sanitize_cases.py: persistent cooperative solver,
graph PCG with the chunked tiles, the multi-patch Schwarz path and the 3D paths of the whole-line
solver, symmetric SpMV, elastic row tiles and the matrix-free operators."""
import math

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu

CASES = {
    "c1": (synth.config("c1"), 0, 3, True),
    "c2": (synth.config("c2", n=16), 0, 3, True),
    "c5": (synth.config("c5", p=3, n=8), 0, 3, True),
    "c5_k3": (synth.config("c5", p=2, n=9, k=3), 0, 2, True),
    "c3_full": (synth.config("c3", p=3, n=10), 1, 2, True),
    "c3_sym": (synth.config("c3", p=4, n=36), 3, 1, False),
    "c3_sym_k3": (synth.config("c3", p=2, n=34, k=3), 3, 1, False),
    "c3_lines": (synth.config("c3", p=2, n=99), 1, 1, True),   # 99 free per direction: whole-line solver, 3D
    "c4_rt": (synth.config("c4", p=2, n=34), 1, 1, True),
    "c3_mf": (synth.config("c3", p=3, n=8), 2, 1, True),
    "c2_mf": (synth.config("c2", n=12), 2, 1, True),
}


def _run(name):
    import torch
    from paper_2102_11536_b200 import Context, make_desc
    cfg, op_mode, steps, _ = CASES[name]
    prob = synth.make_problem(cfg)
    nc = cfg.get("ncomp", 1)
    mat = dict(lam=cfg.get("lam", 1.0), mu=cfg.get("mu", 1.0), density=cfg.get("density", 1.0)) if nc > 1 else {}
    lam_est = 1.2 * cfg["dim"] * 60.0 * cfg["n"] ** 2
    dt = 0.3 * math.sqrt(2.4 / lam_est)
    ctx = Context(make_desc(prob["patches"], cfg["p"], cfg["n"], cfg["dim"], ncomp=nc, k=cfg["k"], rho=cfg["rho"],
                            dt=dt, op_mode=op_mode, **mat), guard_bytes=1 << 20)
    fmap = ctx.free_dof_map()
    mp = (cfg["n"] + cfg["p"]) ** cfg["dim"]
    u0 = np.concatenate([np.array([prob["u0"][int(v // mp)][int(v % mp), c] for v in fmap]) for c in range(nc)])
    ctx.set_state(torch.tensor(u0, device="cuda"))
    ctx.advance(steps)
    out = [t.cpu().numpy() for t in ctx.get_state()]
    x = torch.tensor(np.random.default_rng(1).standard_normal(ctx.n_free), device="cuda")
    for which in ("M", "K", "Pinv"):
        out.append(ctx.apply(which, x).cpu().numpy())
    st = ctx.stats()
    assert st.status == 0
    assert ctx.guards_intact(), "a kernel wrote outside the workspace"
    ctx.close()
    return out


@pytest.mark.parametrize("name", list(CASES))
def test_guards_and_repeatability(name):
    a = _run(name)
    b = _run(name)
    bitwise = CASES[name][3]
    for x, y in zip(a, b):
        assert np.all(np.isfinite(x))
        if bitwise:
            assert np.array_equal(x, y)
        else:
            assert np.abs(x - y).max() <= 1e-10 * np.abs(x).max()
