"""3D multi-patch (block-structured cells glued by coincident control points) through the
masked global grid and the additive Schwarz preconditioner: two cubes and a 3D
L-shaped block of three cubes against the oracle - operators row by row, calM^{-1} element by
element, a mass solve and a short trajectory in the relative M-norm; and the same for linear
elastodynamics (3 components, 9-block K) on two glued cubes.  (BASELINE's multi-patch
config C5 is 2D; this covers the same path in 3D: masked row blocks, boxes with interfaces on
faces and edges, the whole-line solver on boxes with three directions.)"""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

import synth
from oracle import precond

from _helpers import Case, mnorm_rel, oracle_with_floor

pytestmark = pytest.mark.gpu

LAYOUTS = {
    "two_cubes": [(0, 0, 0), (1, 0, 0)],
    "l_block": [(0, 0, 0), (1, 0, 0), (0, 1, 0)],
    "stack_z": [(0, 0, 0), (0, 0, 1)],
}


@pytest.mark.parametrize("layout,p,n,k", [("two_cubes", 2, 5, 2), ("l_block", 3, 4, 2), ("stack_z", 2, 6, 3)])
def test_3d_multipatch_against_oracle(layout, p, n, k):
    cfg = synth.config("c3", p=p, n=n, k=k, cells=LAYOUTS[layout], noise=0.1)
    c = Case(cfg)
    d = c.disc
    rng = np.random.default_rng(21)
    x = rng.standard_normal(d.nfree)
    P = precond.SchwarzPreconditioner(d)
    for which, ref in (("M", d.M @ x), ("K", d.K @ x), ("Pinv", P(x))):
        y = c.from_lib(c.ctx.apply(which, c.to_lib(x)))
        if which == "Pinv":
            assert np.abs(y - ref).max() <= 1e-11 * np.abs(ref).max(), which
        else:
            A = d.M if which == "M" else d.K
            assert np.all(np.abs(y - ref) <= 1e-13 * (abs(A) @ np.abs(x)) + 1e-300), which
    b = d.M @ rng.standard_normal(d.nfree)
    xs, _ = c.ctx.solve_mass(c.to_lib(b))
    assert mnorm_rel(d.M, c.from_lib(xs), spla.spsolve(d.M.tocsc(), b)) < 1e-11
    u0 = c.u0()
    c.ctx.set_state(c.to_lib(u0))
    c.ctx.advance(10)
    assert c.ctx.stats().status == 0
    u, v, a = (c.from_lib(t) for t in c.ctx.get_state())
    tr, floor = oracle_with_floor(d, cfg["k"], cfg["rho"], c.dt, u0, np.zeros_like(u0), 10, case=c)
    for got, want, f in zip((u, v, a), tr[:3], floor):
        assert mnorm_rel(d.M, got, want) < max(1e-10, 10 * f)


def test_3d_multipatch_elasticity():
    cfg = synth.config("c4", p=2, n=4, cells=LAYOUTS["two_cubes"], noise=0.1, lam=2.0, mu=0.5)
    c = Case(cfg)
    d = c.disc
    rng = np.random.default_rng(22)
    x = rng.standard_normal(d.M.shape[0])
    P = precond.SchwarzPreconditioner(d)
    for which, ref in (("M", d.M @ x), ("K", d.K @ x), ("Pinv", P(x))):
        y = c.from_lib(c.ctx.apply(which, c.to_lib(x)))
        if which == "Pinv":
            assert np.abs(y - ref).max() <= 1e-11 * np.abs(ref).max(), which
        else:
            A = d.M if which == "M" else d.K
            assert np.all(np.abs(y - ref) <= 1e-13 * (abs(A) @ np.abs(x)) + 1e-300), which
    u0 = c.u0()
    c.ctx.set_state(c.to_lib(u0))
    c.ctx.advance(10)
    assert c.ctx.stats().status == 0
    u, v, a = (c.from_lib(t) for t in c.ctx.get_state())
    tr, floor = oracle_with_floor(d, cfg["k"], cfg["rho"], c.dt, u0, np.zeros_like(u0), 10, case=c)
    for got, want, f in zip((u, v, a), tr[:3], floor):
        assert mnorm_rel(d.M, got, want) < max(1e-10, 10 * f)
