"""Per-kernel timing (CUDA events) of the hot-path ops through ga_profile_op,
warm (back-to-back launches, as inside a step) and cold (L2 flushed before
each launch), plus the graph step time.  Usage: kbench.py c2 [p=.. n=.. k=..]"""
import math
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch

import synth
from paper_2102_11536_b200 import Context, ga_params, make_desc

args = dict(a.split("=") for a in sys.argv[2:])
reps = int(args.pop("reps", 50))
op_mode = int(args.pop("op", 0))
cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "c2", **{k: (float(v) if "." in v else int(v)) for k, v in args.items()})
prob = synth.make_problem(cfg)
nc = cfg.get("ncomp", 1)
_, _, _, _, th = ga_params(cfg["k"], cfg["rho"])
cp = {1: 12.0, 2: 10.0, 3: 14.56, 4: 24.49, 5: 39.3, 6: 59.5, 7: 88.0}[cfg["p"]]
lam = 1.2 * cfg["dim"] * cp * cfg["n"] ** 2 * (1.73 if nc > 1 else 1.0)
dt = cfg["cfl_frac"] * math.sqrt(th / lam)
desc = make_desc(prob["patches"], cfg["p"], cfg["n"], cfg["dim"], ncomp=nc, k=cfg["k"], rho=cfg["rho"], dt=dt, op_mode=op_mode)
ctx = Context(desc)
fmap = ctx.free_dof_map()
m = cfg["n"] + cfg["p"]
mp = m ** cfg["dim"]
u0 = np.concatenate([np.array([prob["u0"][int(v // mp)][int(v % mp), c] for v in fmap]) for c in range(nc)])
ctx.set_state(torch.tensor(u0, device="cuda"))
ctx.advance(3)
torch.cuda.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = ctx.stream


def timed(fn, n, cold):
    ts = []
    for _ in range(n):
        if cold:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return np.median(ts)


names = ["spmv_M(PQ)", "spmv_K(NEGB)", "precond", "predict", "spmv_M(APPLY)", "p_update"]
print(f"config {cfg['name']} p={cfg['p']} n={cfg['n']} k={cfg['k']} N={ctx.n_free} matrix_free={ctx.matrix_free()}")
for op in range(6):
    warm_batch = timed(lambda: ctx.profile_op(op, reps), 3, False) / reps
    cold = timed(lambda: ctx.profile_op(op, 1), 10, True)
    print(f"  {names[op]:22s} warm(batched) {warm_batch:8.2f} us   cold {cold:8.2f} us")
st0 = ctx.stats()
step = timed(lambda: ctx.advance(1), 20, False)
st1 = ctx.stats()
print(f"  step (graph, warm)     {step:8.2f} us   lockstep iters/step {(st1.loop_iters - st0.loop_iters) / 20:.2f}  launches/step {(st1.kernel_launches - st0.kernel_launches) / 20:.1f}")
