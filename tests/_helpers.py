"""Shared helpers of the GPU parity tests: build an oracle discretization and
the matching library context on the same seeded inputs, and map vectors
between the oracle's free-DoF order and the library's."""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import synth
from oracle import assembly, params


class Case:
    """cfg-driven case; `perm[f]` = oracle index of library free DoF f (per component)."""

    def __init__(self, cfg, dt=None, lam_max=None, param_set=0, **desc_over):
        import torch

        from paper_2102_11536_b200 import Context, make_desc
        self.cfg = cfg
        self.prob = synth.make_problem(cfg)
        dim, p, n, nc = cfg["dim"], cfg["p"], cfg["n"], cfg.get("ncomp", 1)
        mat = dict(lam=cfg.get("lam", 1.0), mu=cfg.get("mu", 1.0), density=cfg.get("density", 1.0)) if nc > 1 else {}
        self.disc = assembly.Discretization(self.prob["patches"], p, n, dim, ncomp=nc, **mat)
        d = self.disc
        if dt is None:
            if lam_max is None:
                if d.M.shape[0] <= 3000:
                    lam_max = sla.eigh(d.K.toarray(), d.M.toarray(), eigvals_only=True)[-1]
                else:
                    lam_max = spla.eigsh(d.K, k=1, M=d.M.tocsc(), which="LA", return_eigenvectors=False)[0]
            self.lam_max = lam_max
            thmax = params.theta_max_closed_form(cfg["rho"])
            dt = cfg["cfl_frac"] * math.sqrt(thmax / lam_max)
        self.dt = dt
        self.desc = make_desc(self.prob["patches"], p, n, dim, ncomp=nc, k=cfg["k"], rho=cfg["rho"], dt=dt,
                              param_set=param_set, lam=mat.get("lam", 1.0), mu=mat.get("mu", 1.0),
                              density=mat.get("density", 1.0), **desc_over)
        self.ctx = Context(self.desc)
        m = n + p
        mpow = m ** dim
        fmap = self.ctx.free_dof_map()
        self.perm = np.array([d.G[int(v // mpow)][int(v % mpow)] for v in fmap], dtype=np.int64)
        assert np.all(self.perm >= 0) and len(set(self.perm.tolist())) == d.nfree
        nf = d.nfree
        self.full_perm = np.concatenate([self.perm + c * nf for c in range(nc)])
        self.torch = torch

    # oracle vector (oracle order) -> library tensor, and back
    def to_lib(self, x):
        return self.torch.tensor(np.asarray(x)[self.full_perm], dtype=self.torch.float64, device="cuda")

    def from_lib(self, t):
        out = np.empty(len(self.full_perm))
        out[self.full_perm] = t.detach().cpu().numpy()
        return out

    def u0(self):
        return self.disc.restrict_local(self.prob["u0"])


def record_parity(errs, floor=None, bar=None, **extra):
    """Append one parity result (relative M-norm errors of u, v, a against the oracle, the
    oracle-vs-oracle floor F, the bar max(1e-10, 10 F)) to the JSON-lines record
    GA_PARITY_RECORD (default gpurun_out/parity_record.jsonl), committed from the GPU run under
    profiles/ so the cases that meet 1e-10 outright and those on a widened bar are visible."""
    import json
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    path = os.environ.get("GA_PARITY_RECORD", os.path.join(root, "gpurun_out", "parity_record.jsonl"))
    os.makedirs(os.path.dirname(path), exist_ok=True)
    rec = {"test": os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0],
           "errs_uva": [float(e) for e in errs],
           "floor_uva": None if floor is None else [float(f) for f in floor],
           "bar_uva": None if bar is None else [float(b) for b in bar],
           "meets_1e-10": bool(all(e <= 1e-10 for e in errs))}
    rec.update(extra)
    with open(path, "a") as f:
        f.write(json.dumps(rec) + "\n")


def mnorm_rel(M, x, ref):
    e = x - ref
    den = math.sqrt(max(ref @ (M @ ref), 1e-300))
    return math.sqrt(max(e @ (M @ e), 0.0)) / den


class _CholSolver:
    """Second, independent fp64 direct solver: dense Cholesky, no refinement."""

    def __init__(self, M):
        self.f = sla.cho_factor(M.toarray())

    def __call__(self, b):
        return sla.cho_solve(self.f, b)


def oracle_with_floor(d, k, rho, dt, u0, v0, nsteps, param_set=0, case=None):
    """Oracle trajectory (LU + refinement) and the relative M-norm distance F
    to a second oracle run with another direct solver, per output u, v, a."""
    from oracle import integrator
    it = integrator.Integrator(d.M, d.K, k, rho, dt, param_set=param_set)
    ref = it.run(u0, v0, nsteps)
    if d.M.shape[0] <= 4000:
        alt_solver = _CholSolver(d.M)
    else:
        lu = spla.splu(d.M.tocsc())
        alt_solver = lu.solve
    it2 = integrator.Integrator(d.M, d.K, k, rho, dt, param_set=param_set, solver=alt_solver)
    alt = it2.run(u0, v0, nsteps)
    floor = [mnorm_rel(d.M, alt[m], ref[m]) for m in range(3)]
    # assembly-order floor: the same trajectory with M and K assembled by the
    # same definitions but the Gauss points summed in reverse order.  Both are
    # valid fp64 evaluations of the quadrature sums; kappa(M) ~ 1e8 at 3D p=6
    # amplifies their ~1e-14 entry differences far above the solver floor
    #
    if case is not None:
        c = case.cfg
        mat = dict(lam=c.get("lam", 1.0), mu=c.get("mu", 1.0), density=c.get("density", 1.0)) if d.ncomp > 1 else {}
        d2 = assembly.Discretization(case.prob["patches"], d.p, d.n, d.dim, ncomp=d.ncomp, reverse_points=True,
                                     **mat)
        it3 = integrator.Integrator(d2.M, d2.K, k, rho, dt, param_set=param_set)
        rev = it3.run(u0, v0, nsteps)
        floor = [max(f, mnorm_rel(d.M, rev[m], ref[m])) for m, f in enumerate(floor)]
    return ref, floor
