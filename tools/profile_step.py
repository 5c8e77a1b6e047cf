"""Run a few explicit steps of a config (for ncu launch lists / captures).
Use GA_NO_GRAPH=1 so the kernels are launched directly (ncu cannot profile
kernel nodes of graphs with conditional nodes)."""
import math
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch

import synth
from paper_2102_11536_b200 import Context, ga_params, make_desc

args = dict(a.split("=") for a in sys.argv[2:])
steps = int(args.pop("steps", 3))
cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "c2", **{k: (float(v) if "." in v else int(v)) for k, v in args.items()})
prob = synth.make_problem(cfg)
nc = cfg.get("ncomp", 1)
_, _, _, _, th = ga_params(cfg["k"], cfg["rho"])
# dt from the C2-like estimate lambda_max ~ 1.09 * d * c_p / h^2 (only timing matters here)
cp = {1: 12.0, 2: 10.0, 3: 14.56, 4: 24.49, 5: 39.3, 6: 59.5, 7: 88.0}[cfg["p"]]
lam = 1.2 * cfg["dim"] * cp * cfg["n"] ** 2 * (1.73 if nc > 1 else 1.0)
dt = cfg["cfl_frac"] * math.sqrt(th / lam)
desc = make_desc(prob["patches"], cfg["p"], cfg["n"], cfg["dim"], ncomp=nc, k=cfg["k"], rho=cfg["rho"], dt=dt)
ctx = Context(desc)
fmap = ctx.free_dof_map()
m = cfg["n"] + cfg["p"]
mp = m ** cfg["dim"]
u0 = np.concatenate([np.array([prob["u0"][int(v // mp)][int(v % mp), c] for v in fmap]) for c in range(nc)])
ctx.set_state(torch.tensor(u0, device="cuda"))
ctx.advance(steps)
torch.cuda.synchronize()
st = ctx.stats()
print("status", st.status, "steps", st.steps, "loop_iters", st.loop_iters, "launches", st.kernel_launches)
