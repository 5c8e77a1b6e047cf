import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np, synth
from _helpers import Case, mnorm_rel
from oracle import integrator
cfg = synth.config(sys.argv[1], **{k: (float(v) if "." in v else int(v)) for k, v in (a.split("=") for a in sys.argv[2:])})
c = Case(cfg)
d = c.disc
b = d.K @ c.u0()
for rep in range(3):
    x, its = c.ctx.solve_mass(c.to_lib(b))
    x = c.from_lib(x)
    ref = integrator.DirectMassSolver(d.M)(b)
    st = c.ctx.stats()
    print("rep", rep, "its", its, "err", mnorm_rel(d.M, x, ref), "status", st.status, "solves", st.solves, "loop", st.loop_iters, "launches", st.kernel_launches)
c.ctx.set_state(c.to_lib(c.u0())); c.ctx.advance(3); st = c.ctx.stats()
print("after 3 steps: steps", st.steps, "status", st.status, "solves", st.solves, "iters", list(st.pcg_iters))
