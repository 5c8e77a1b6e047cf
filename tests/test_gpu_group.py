"""GPU parity of the partitioned multi-patch mode (patch-per-GPU): one
subdomain context per patch (its LOCAL operators on the bounding box of its free control
points), stepped together by a ga_group (dist.cu) whose exchanges sum the interface copies.
Against the oracle's glued discretization and global additive-Schwarz preconditioner
(P:763-783): operators and preconditioner element by element, mass solves, trajectories; the
L-shape also against the single-context masked-grid path; the NCCL transport (a one-rank
communicator: ncclAllReduce + the host-driven PCG loop) against the single-process group.
All subdomains run on one GPU in ONE process (no kernel waits on another process)."""
import math

import numpy as np
import pytest

import synth
from oracle import assembly, integrator, params, precond

from _helpers import mnorm_rel, record_parity

pytestmark = pytest.mark.gpu


class GroupCase:
    """Subdomain contexts + group for the patches of cfg; loc[r][f] = oracle free index of the
    library free DoF f of subdomain r."""

    def __init__(self, cfg, dt, nccl=False, **over):
        import torch

        import paper_2102_11536_b200.genalpha as ga
        self.ga, self.torch = ga, torch
        self.cfg = cfg
        self.prob = synth.make_problem(cfg)
        dim, p, n = cfg["dim"], cfg["p"], cfg["n"]
        patches = self.prob["patches"]
        self.d = assembly.Discretization(patches, p, n, dim)
        self.plan = ga.PartitionPlan([c for _, c in patches], p, n, dim)
        self.ctxs = []
        self.loc = []
        mp = (n + p) ** dim
        for r, (cell, ctrl) in enumerate(patches):
            desc = ga.make_desc([((0,) * dim, ctrl)], p, n, dim, k=cfg["k"], rho=cfg["rho"], dt=dt,
                                sub=self.plan.sub[r], **over)
            c = ga.Context(desc)
            fmap = c.free_dof_map()
            assert np.all(fmap < mp)
            self.loc.append(self.d.G[r][fmap])
            assert np.all(self.loc[-1] >= 0)
            self.ctxs.append(c)
        self.comm = None
        if nccl:
            uid = ga.nccl_unique_id()
            self.comm = ga.nccl_comm_init(1, uid, 0)
        self.grp = ga.Group(self.ctxs, nccl_comm=self.comm)

    def split(self, x):
        return [self.torch.tensor(np.asarray(x)[l], dtype=self.torch.float64, device="cuda") for l in self.loc]

    def join(self, ts, check_consistent=True):
        out = np.full(self.d.nfree, np.nan)
        for l, t in zip(self.loc, ts):
            v = t.cpu().numpy()
            if check_consistent:
                seen = ~np.isnan(out[l])
                assert np.array_equal(out[l][seen], v[seen]), "interface copies differ"
            out[l] = v
        assert not np.any(np.isnan(out))
        return out

    def close(self):
        self.grp.close()
        for c in self.ctxs:
            c.close()
        if self.comm is not None:
            self.ga.nccl_comm_destroy(self.comm)


def _cfg(name):
    if name == "lshape":
        return synth.config("c5", n=8)
    if name == "lshape_p2":
        return synth.config("c5", p=2, n=6, k=1, rho=0.5)
    if name == "fan2d":
        return synth.config("fan2d", n=6)
    if name == "fan2d_p2":
        return synth.config("fan2d", p=2, n=5, k=3, rho=0.0)
    if name == "fan3d":
        return synth.config("fan3d", n=3)
    if name == "fan3d_p3":
        return synth.config("fan3d", p=3, n=3, k=1, rho=1.0)
    raise KeyError(name)


CASES = ["lshape", "lshape_p2", "fan2d", "fan2d_p2", "fan3d", "fan3d_p3"]


def _dt(cfg, d):
    import scipy.linalg as sla
    lam = sla.eigh(d.K.toarray(), d.M.toarray(), eigvals_only=True)[-1]
    return cfg["cfl_frac"] * math.sqrt(params.theta_max_closed_form(cfg["rho"]) / lam)


@pytest.mark.parametrize("name", CASES)
def test_group_operators_elementwise(name):
    cfg = _cfg(name)
    g = GroupCase(cfg, dt=1e-3)
    d = g.d
    rng = np.random.default_rng(1)
    x = rng.standard_normal(d.nfree)
    Pinv = precond.SchwarzPreconditioner(d)
    for which, ref in (("M", d.M @ x), ("K", d.K @ x), ("Pinv", Pinv(x))):
        y = g.join(g.grp.apply(which, g.split(x)))
        if which == "Pinv":
            scale = np.max(np.abs(ref))
            assert np.max(np.abs(y - ref)) <= 1e-12 * scale, which
        else:
            A = d.M if which == "M" else d.K
            absx = abs(A) @ np.abs(x)
            assert np.all(np.abs(y - ref) <= 1e-13 * absx + 1e-300), which
    g.close()


@pytest.mark.parametrize("name", CASES)
def test_group_mass_solve(name):
    import scipy.sparse.linalg as spla
    cfg = _cfg(name)
    g = GroupCase(cfg, dt=1e-3)
    d = g.d
    rng = np.random.default_rng(2)
    b = d.M @ rng.standard_normal(d.nfree)
    xs, its = g.grp.solve_mass(g.split(b))
    x = g.join(xs)
    xr = spla.spsolve(d.M.tocsc(), b)
    _, itg, _ = precond.pcg(lambda v: d.M @ v, b, precond.SchwarzPreconditioner(d), tol=1e-13)
    assert mnorm_rel(d.M, x, xr) < 1e-11
    assert abs(its - itg) <= 2, (its, itg)
    g.close()


@pytest.mark.parametrize("name", CASES)
def test_group_trajectory_vs_oracle(name):
    cfg = _cfg(name)
    prob = synth.make_problem(cfg)
    d = assembly.Discretization(prob["patches"], cfg["p"], cfg["n"], cfg["dim"])
    dt = _dt(cfg, d)
    g = GroupCase(cfg, dt=dt)
    u0 = d.restrict_local(prob["u0"])
    nsteps = 30
    g.grp.set_state(g.split(u0))
    g.grp.advance(nsteps)
    for st in g.grp.stats():
        assert st.status == 0 and st.steps == nsteps
    got = [g.join([s[m] for s in g.grp.get_state()]) for m in range(3)]
    ref = integrator.Integrator(d.M, d.K, cfg["k"], cfg["rho"], dt).run(u0, np.zeros_like(u0), nsteps)
    errs = [mnorm_rel(d.M, x, y) for x, y in zip(got, ref)]
    record_parity(errs, None, [1e-10] * 3, n_free=int(d.nfree), steps=nsteps, npatch=len(prob["patches"]),
                  p=cfg["p"], dim=cfg["dim"], mode="group")
    assert max(errs) < 1e-10, errs
    g.close()


def test_group_lshape_equals_single_context_path():
    # the L-shape is block-structured: the masked-grid single context steps the same problem
    from _helpers import Case
    cfg = _cfg("lshape")
    c = Case(cfg)
    g = GroupCase(cfg, dt=c.dt)
    u0 = c.u0()
    c.ctx.set_state(c.to_lib(u0))
    g.grp.set_state(g.split(u0))
    c.ctx.advance(20)
    g.grp.advance(20)
    a = [c.from_lib(t) for t in c.ctx.get_state()]
    b = [g.join([s[m] for s in g.grp.get_state()]) for m in range(3)]
    for x, y in zip(a, b):
        assert mnorm_rel(c.disc.M, y, x) < 1e-12
    st1, st2 = c.ctx.stats(), g.grp.stats()[0]
    assert list(st1.pcg_iters) == list(st2.pcg_iters)  # same PCG, same iteration counts
    g.close()
    c.ctx.close()


@pytest.mark.parametrize("name", ["lshape", "fan3d"])
def test_group_nccl_transport_one_rank(name):
    # ncclAllReduce on a one-rank communicator + the host-driven PCG loop (the multi-process
    # code path) against the single-process group graph
    cfg = _cfg(name)
    prob = synth.make_problem(cfg)
    d = assembly.Discretization(prob["patches"], cfg["p"], cfg["n"], cfg["dim"])
    dt = _dt(cfg, d)
    u0 = d.restrict_local(prob["u0"])
    out = []
    for nccl in (False, True):
        g = GroupCase(cfg, dt=dt, nccl=nccl)
        g.grp.set_state(g.split(u0))
        g.grp.advance(10)
        out.append(([g.join([s[m] for s in g.grp.get_state()]) for m in range(3)],
                    [list(s.pcg_iters) for s in g.grp.stats()]))
        g.close()
    for x, y in zip(out[0][0], out[1][0]):
        assert mnorm_rel(d.M, y, x) < 1e-13
    assert out[0][1] == out[1][1]


def test_group_rejects_bad_use():
    import paper_2102_11536_b200.genalpha as ga
    cfg = _cfg("lshape")
    g = GroupCase(cfg, dt=1e-3)
    with pytest.raises(ga.GAError):   # a subdomain is stepped only through its group
        g.ctxs[0].advance(1)
    with pytest.raises(ga.GAError):   # one group per context
        ga.Group(g.ctxs[:1])
    g.close()
