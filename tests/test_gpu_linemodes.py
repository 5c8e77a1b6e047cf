"""GPU parity of every line-solve implementation of the Kronecker preconditioner
(P:703-713): the chunked shared-memory tiles ('t'), the streamed thread-per-line
sweeps ('s') and the whole-line sequential sweeps from shared memory ('q', line_seq.cu).  The automatic choice depends
on the grid size, so each mode is forced through GA_LINE_MODE in a fresh
process (the mode is read once per process) on small 3D cases with ragged
tiles (free lines not a multiple of 32 slots), k = 1..3, and the elastic
(3-component) layout; calM^{-1} is compared with the oracle element by element
and a short trajectory in the relative M-norm."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import synth
from oracle import precond
from _helpers import Case, mnorm_rel, oracle_with_floor
cfg = synth.config(*{cfg!r}[:1], **{cfg!r}[1])
c = Case(cfg)
d = c.disc
P = precond.SchwarzPreconditioner(d)
x = np.random.default_rng(5).standard_normal(d.M.shape[0])
y = c.from_lib(c.ctx.apply("Pinv", c.to_lib(x)))
ref = P(x)
pre = float(np.abs(y - ref).max() / np.abs(ref).max())
u0 = c.u0()
c.ctx.set_state(c.to_lib(u0))
c.ctx.advance(8)
st = c.ctx.stats()
u, v, a = (c.from_lib(t) for t in c.ctx.get_state())
tr, floor = oracle_with_floor(d, cfg["k"], cfg["rho"], c.dt, u0, np.zeros_like(u0), 8, case=c)
errs = [mnorm_rel(d.M, p, q) for p, q in zip((u, v, a), tr[:3])]
print(json.dumps(dict(pre=pre, errs=errs, floor=floor, status=st.status)))
"""

CASES = [
    ("c3", dict(p=3, n=7, k=2)),           # 8 free per direction: ragged tiles
    ("c3", dict(p=2, n=11, k=3, rho=1.0)),  # 11 free, 3 rhs (10 x lines = 30 slots per tile)
    ("c3", dict(p=4, n=5, k=1)),
    ("c4", dict(p=2, n=4)),                 # elastic: 3 components
    ("c3", dict(p=5, n=4, k=2)),            # p >= 5: batches of 4 in the whole-line sweeps, 64-byte factor rows
    ("c3", dict(p=1, n=9, k=4)),            # p = 1, 4 right-hand sides
]


@pytest.mark.parametrize("mode", ["t", "s", "q"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}_" + "_".join(f"{k}{v}" for k, v in c[1].items()))
def test_line_mode_parity(mode, case):
    code = SCRIPT.format(root=ROOT, tests=os.path.join(ROOT, "tests"), cfg=(case[0], case[1]))
    env = dict(os.environ, GA_LINE_MODE=mode)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["status"] == 0
    assert r["pre"] <= 1e-11, r
    assert all(e < max(1e-10, 10 * f) for e, f in zip(r["errs"], r["floor"])), r
