"""Writes tests/golden/c5_full_oracle.npz: the CPU oracle (oracle/ only) run of
BASELINE.json configs[4] at full size (2D L-shape of 3 C^0-glued patches, p=3,
512x512 elements each, +-0.1h interior noise, 790,533 free DoFs, k=2, rho=0.3,
dt = 0.5 CFL, 200 steps), used by the full-size GPU parity test of the multi-patch
additive-Schwarz path.  lambda_max from scipy eigsh on the oracle's
(K, M); U0 = control-point interpolation (synth); vectors in the oracle's free-DoF
order.  Run: python tests/golden/make_c5_reference.py"""
import math
import os
import sys
import time

import numpy as np
import scipy.sparse.linalg as spla

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
import synth  # noqa: E402
from oracle import assembly, integrator, params  # noqa: E402

cfg = synth.config("c5")
prob = synth.make_problem(cfg)
t0 = time.time()
d = assembly.Discretization(prob["patches"], cfg["p"], cfg["n"], cfg["dim"])
print(f"assembled {d.nfree} DoFs in {time.time() - t0:.0f}s", flush=True)
lam = spla.eigsh(d.K, k=1, M=d.M.tocsc(), which="LA", return_eigenvectors=False, tol=1e-12)[0]
dt = cfg["cfl_frac"] * math.sqrt(params.theta_max_closed_form(cfg["rho"]) / lam)
print(f"lambda_max {lam:.10e} in {time.time() - t0:.0f}s", flush=True)
u0 = d.restrict_local(prob["u0"])
it = integrator.Integrator(d.M, d.K, cfg["k"], cfg["rho"], dt)
c = it.run(u0, np.zeros_like(u0), cfg["steps"])
np.savez_compressed(os.path.join(HERE, "c5_full_oracle.npz"), u=c[0], v=c[1], a=c[2], dt=dt, lam=lam,
                    steps=cfg["steps"], nfree=d.nfree)
print(f"lambda_max {lam:.10e} dt {dt:.10e} steps {cfg['steps']} wall {time.time() - t0:.0f}s")
