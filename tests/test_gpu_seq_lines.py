"""GPU parity of the whole-line sequential line solver (csrc/line_seq.cu; the Kronecker factor
Mh_d^{-1} of calM^{-1}) on the shapes its staging paths distinguish:

* a 3D single patch large enough that the library selects it by itself (> 148 x 128 line-slots
  per direction: 32-slot tiles, bulk copies for the x lines, 16-byte cp.async for y and z lines),
  on the undeformed cube, where calM^{-1} = Mh^{-1} (x) Mh^{-1} (x) Mh^{-1} EXACTLY (P:703-713:
  identity map => M is the Kronecker product and the scaling is 1), so the reference is three
  dense 1D solves with the parametric mass matrix - a textbook identity, independent of the
  oracle's assembly;
* L-shapes (additive Schwarz) with k = 1, 3, 4 right-hand sides and odd box sizes
  (8-byte cp.async staging, ragged tiles, lines that are not 16-byte multiples) against the
  oracle's Schwarz preconditioner, element by element."""
import numpy as np
import pytest

import synth
from oracle import precond

from _helpers import Case

pytestmark = pytest.mark.gpu


# (p, n, k): even and odd free counts x k = 1..4 (bulk copies need 16-byte lines: odd n_f k falls back
# to 8-byte cp.async), every batch size of the sweeps (p <= 4: 8, p >= 5: 4), p = 1 and p = 7
@pytest.mark.parametrize("p,n,k", [(3, 100, 2), (2, 140, 1), (5, 80, 3), (2, 139, 1), (3, 81, 3), (1, 73, 4),
                                   (4, 101, 2), (7, 94, 2), (6, 99, 1)])
def test_kronecker_identity_on_the_cube(p, n, k):
    import torch
    from paper_2102_11536_b200 import Context, make_desc
    cfg = synth.config("c3", p=p, n=n, k=k, noise=0.0)
    prob = synth.make_problem(cfg)
    ctx = Context(make_desc(prob["patches"], p, n, 3, k=k, rho=cfg["rho"], dt=1e-3))
    nf = n + p - 2
    assert ctx.n_free == nf ** 3
    Mh = precond.param_mass_1d(p, n)[1:-1, 1:-1]
    Mi = np.linalg.inv(Mh)
    x = np.random.default_rng(11).standard_normal(nf ** 3)
    X = x.reshape(nf, nf, nf)  # [z][y][x], x fastest (the library's free-DoF order of one patch)
    ref = np.einsum("ai,bj,ck,ijk->abc", Mi, Mi, Mi, X, optimize=True).reshape(-1)
    y = ctx.apply("Pinv", torch.tensor(x, device="cuda")).cpu().numpy()
    assert np.abs(y - ref).max() <= 1e-11 * np.abs(ref).max()


@pytest.mark.parametrize("p,n,k", [(2, 5, 1), (3, 6, 3), (3, 9, 4), (2, 12, 3)])
def test_lshape_schwarz_other_rhs_counts(p, n, k):
    c = Case(synth.config("c5", p=p, n=n, k=k), dt=1e-3)
    d = c.disc
    P = precond.SchwarzPreconditioner(d)
    x = np.random.default_rng(7).standard_normal(d.nfree)
    y = c.from_lib(c.ctx.apply("Pinv", c.to_lib(x)))
    ref = P(x)
    assert np.abs(y - ref).max() <= 1e-11 * np.abs(ref).max()
    # and a mass solve through it (PCG, the other k - 1 slots idle)
    b = d.M @ np.random.default_rng(8).standard_normal(d.nfree)
    xs, its = c.ctx.solve_mass(c.to_lib(b))
    import scipy.sparse.linalg as spla
    xr = spla.spsolve(d.M.tocsc(), b)
    e = c.from_lib(xs) - xr
    assert np.sqrt(e @ (d.M @ e)) <= 1e-11 * np.sqrt(xr @ (d.M @ xr))
