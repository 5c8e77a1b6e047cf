import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import synth
from _helpers import Case
import numpy as np
cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "c2", **{k: int(v) for k, v in (a.split("=") for a in sys.argv[2:])})
c = Case(cfg)
x = np.random.default_rng(0).standard_normal(c.disc.M.shape[0])
y = c.from_lib(c.ctx.apply("Pinv", c.to_lib(x)))
from oracle import precond
ref = precond.SchwarzPreconditioner(c.disc)(x)
print("prec err", np.abs(y - ref).max() / np.abs(ref).max())
