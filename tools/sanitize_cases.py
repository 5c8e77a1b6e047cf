"""Small invocations of every hot-path kernel family for compute-sanitizer (memcheck, racecheck,
synccheck): persistent cooperative solver (C1, C2 reduced), graph PCG with the 2D tile line
solves, the multi-patch Schwarz path (C5 reduced), the 3D line-solve modes (tiles / streamed /
whole-line, forced by GA_LINE_MODE in separate processes), the single-read symmetric SpMV (3D
half-symmetric), the elastic row tiles and the matrix-free operators.  Usage:
  compute-sanitizer --tool memcheck python tools/sanitize_cases.py <case>"""
import math
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch

import synth
from paper_2102_11536_b200 import Context, make_desc

CASES = {
    "c1": (synth.config("c1"), 0, 3),
    "c2": (synth.config("c2", n=16), 0, 3),
    "c5": (synth.config("c5", p=3, n=8), 0, 3),
    "c3_full": (synth.config("c3", p=3, n=10), 1, 2),
    "c3_sym": (synth.config("c3", p=4, n=36), 3, 1),
    "c3_sym_k3": (synth.config("c3", p=2, n=34, k=3), 3, 1),
    "c4_rt": (synth.config("c4", p=2, n=34), 1, 1),
    "c3_mf": (synth.config("c3", p=3, n=8), 2, 1),
    "c2_mf": (synth.config("c2", n=12), 2, 1),
}


def run(name):
    cfg, op_mode, steps = CASES[name]
    prob = synth.make_problem(cfg)
    nc = cfg.get("ncomp", 1)
    mat = dict(lam=cfg.get("lam", 1.0), mu=cfg.get("mu", 1.0), density=cfg.get("density", 1.0)) if nc > 1 else {}
    lam_est = 1.2 * cfg["dim"] * 60.0 * cfg["n"] ** 2
    dt = 0.3 * math.sqrt(2.4 / lam_est)
    ctx = Context(make_desc(prob["patches"], cfg["p"], cfg["n"], cfg["dim"], ncomp=nc, k=cfg["k"], rho=cfg["rho"],
                            dt=dt, op_mode=op_mode, **mat))
    fmap = ctx.free_dof_map()
    m = cfg["n"] + cfg["p"]
    mp = m ** cfg["dim"]
    u0 = np.concatenate([np.array([prob["u0"][int(v // mp)][int(v % mp), c] for v in fmap]) for c in range(nc)])
    ctx.set_state(torch.tensor(u0, device="cuda"))
    ctx.advance(steps)
    x = torch.tensor(np.random.default_rng(1).standard_normal(ctx.n_free), device="cuda")
    for which in ("M", "K", "Pinv"):
        ctx.apply(which, x)
    st = ctx.stats()
    torch.cuda.synchronize()
    print(f"{name}: status {st.status} steps {st.steps} launches {st.kernel_launches} op_mode {ctx.operator_mode()}")
    assert st.status == 0


if __name__ == "__main__":
    run(sys.argv[1])
