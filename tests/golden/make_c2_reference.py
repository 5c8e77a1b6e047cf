"""Writes tests/golden/c2_full_oracle.npz: the CPU oracle (oracle/ only) run of
BASELINE.json configs[1] at full size (2D p=3, 256x256 elements, +-0.2h, k=2,
rho=0, dt = 0.8 CFL, 500 steps), used by the full-size GPU parity test.
lambda_max from scipy eigsh on the oracle's (K, M); U0 = control-point
interpolation (synth).  Run: python tests/golden/make_c2_reference.py"""
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

cfg = synth.config("c2")
prob = synth.make_problem(cfg)
t0 = time.time()
d = assembly.Discretization(prob["patches"], cfg["p"], cfg["n"], cfg["dim"])
lam = spla.eigsh(d.K, k=1, M=d.M.tocsc(), which="LA", return_eigenvectors=False, tol=1e-12)[0]
dt = cfg["cfl_frac"] * math.sqrt(params.theta_max_closed_form(cfg["rho"]) / lam)
u0 = d.restrict_local(prob["u0"])
it = integrator.Integrator(d.M, d.K, cfg["k"], cfg["rho"], dt)
c = it.run(u0, np.zeros_like(u0), cfg["steps"])
np.savez_compressed(os.path.join(HERE, "c2_full_oracle.npz"), u=c[0], v=c[1], a=c[2], dt=dt, lam=lam,
                    steps=cfg["steps"])
print(f"lambda_max {lam:.10e} dt {dt:.10e} steps {cfg['steps']} wall {time.time() - t0:.0f}s")
