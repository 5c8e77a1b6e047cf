import sys, os, math
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np, scipy.sparse as sp
import synth
from oracle import integrator
from _helpers import Case, mnorm_rel
p = int(sys.argv[1]) if len(sys.argv) > 1 else 6
c = Case(synth.config("c3", p=p, n=3, k=2, rho=0.0))
d = c.disc
N = d.M.shape[0]
def extract(which):
    cols = []
    for j in range(N):
        e = np.zeros(N); e[j] = 1
        cols.append(c.from_lib(c.ctx.apply(which, c.to_lib(e))))
    return np.stack(cols, axis=1)
Mg, Kg = extract("M"), extract("K")
Mo, Ko = d.M.toarray(), d.K.toarray()
nz = Mo != 0
print("M rel entry err max", np.max(np.abs(Mg - Mo)[nz] / np.abs(Mo)[nz]), "K rel err (scaled by row max)", np.max(np.abs(Kg - Ko) / np.abs(Ko).max(axis=1, keepdims=True)))
print("K entry rel err max", np.max(np.abs(Kg - Ko)[Ko != 0] / np.abs(Ko)[Ko != 0]))
print("Mg sym", np.abs(Mg - Mg.T).max() / np.abs(Mg).max(), "Kg sym", np.abs(Kg - Kg.T).max() / np.abs(Kg).max())
u0 = c.u0()
c.ctx.set_state(c.to_lib(u0)); c.ctx.advance(40)
u, v, a = (c.from_lib(t) for t in c.ctx.get_state())
ref = integrator.Integrator(d.M, d.K, 2, 0.0, c.dt).run(u0, np.zeros_like(u0), 40)
refg = integrator.Integrator(sp.csr_matrix(Mg), sp.csr_matrix(Kg), 2, 0.0, c.dt).run(u0, np.zeros_like(u0), 40)
for nm, x, y, z in (("u", u, ref[0], refg[0]), ("v", v, ref[1], refg[1]), ("a", a, ref[2], refg[2])):
    print(nm, "gpu-vs-oracle", mnorm_rel(d.M, x, y), "gpu-vs-oracle(gpu ops)", mnorm_rel(d.M, x, z), "oracle(gpu ops)-vs-oracle", mnorm_rel(d.M, z, y))
st = c.ctx.stats(); print("iters", list(st.pcg_iters), "solves", st.solves, "maxit", st.max_iters, "relres", st.max_rel_residual)
