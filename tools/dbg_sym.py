"""Debug: single-read 3D SpMV (op_mode 3) vs the full stencil SpMV (op_mode 1), error locations."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import synth
from paper_2102_11536_b200 import Context, make_desc
p, n, k = (int(v) for v in sys.argv[1:4])
cfg = synth.config("c3", p=p, n=n, k=k)
prob = synth.make_problem(cfg)
cs = [Context(make_desc(prob["patches"], p, n, 3, k=k, rho=0.0, dt=1e-4, op_mode=om)) for om in (1, 3)]
nf = n + p - 2
x = torch.tensor(np.random.default_rng(1).standard_normal(cs[0].n_free), device="cuda")
for which in ("M", "K"):
    a, b = (c.apply(which, x).cpu().numpy() for c in cs)
    e = np.abs(a - b).reshape(nf, nf, nf)
    rel = e.max() / np.abs(a).max()
    print(which, "rel err", rel)
    if rel > 1e-13:
        bad = np.argwhere(e > 1e-10 * np.abs(a).max())
        print("  bad count", len(bad), "of", nf ** 3)
        for ax, nm in ((2, "x"), (1, "y"), (0, "z")):
            vals, cnt = np.unique(bad[:, ax], return_counts=True)
            print("  ", nm, dict(zip(vals.tolist()[:40], cnt.tolist()[:40])))
