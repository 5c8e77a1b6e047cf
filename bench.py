"""Benchmark of the explicit order-2k generalized-alpha hot path on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config c2] [--p P] [--n N] [--k K] [--rho R]

A "step" is one explicit step of the integrator: the K stencil
apply on the k predictors, k lock-stepped PCG mass solves (with refinement)
and the 3k-variable stage update, on one synthetic problem resident in HBM.
Default workload: the largest single-GPU configuration of BASELINE.json,
configs[2] at its top size (3D scalar wave, p=6, 192^3 elements, 7,529,536 free
DoFs, +-0.15h deformed cube, k=2, rho=0, dt = 0.5 CFL; half-symmetric stencils
applied by the single-read SpMV).  Other configs (--config c2 ... ) print their
own line.

Metric: DoF-updates/s = N_free x steps / device time.  Timing: W untimed
warm-up steps, then K steps each bracketed by CUDA events on the launching
stream, with L2 flushed (256 MiB write) between steps, barrier + synchronize
on both sides, max over ranks.  Multi-GPU: independent replicas (the path
does not shard), value = sum of all ranks' DoF-updates
/ max time.  --impl reference times the CPU oracle (oracle/, as it stands) on
rank 0 instead.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DoF-updates/s per explicit step (fp64, k PCG solves)"
UNIT = "DoF-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--p", type=int)
    ap.add_argument("--n", type=int)
    ap.add_argument("--k", type=int)
    ap.add_argument("--rho", type=float)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kernel-reps", type=int, default=20)
    ap.add_argument("--lam-iters", type=int, default=40, help="Lanczos steps for lambda_max (dt)")
    ap.add_argument("--op-mode", type=int, default=0, choices=[0, 1, 2, 3],
                    help="0 auto (measured-faster / capacity), 1 stencil, 2 matrix-free, 3 half-symmetric")
    return ap.parse_args()


# the headline workload (BASELINE.json configs[2] at its largest size, "up to ~7.5M DoFs")
HEADLINE = {"c3": dict(p=6, n=192, k=2, rho=0.0)}


def make_cfg(args):
    import synth
    over = dict(HEADLINE.get(args.config, {}))
    over.update({k: getattr(args, k) for k in ("p", "n", "k", "rho") if getattr(args, k) is not None})
    return synth.config(args.config, **over)


def oracle_sample_cfg(cfg):
    """The bounded sample of a workload the CPU oracle is timed on: the same configuration
    (geometry recipe, p, k, rho) at the largest n whose oracle assembly stays within ~2e10
    multiply-adds (the sparse products B^T W B over the Gauss points, ~30 s on one core);
    the full size where that is feasible.  Returns (cfg_sample, extrapolated)."""
    import synth
    d, p = cfg["dim"], cfg["p"]
    nmax = int((2e10 / ((p + 1) ** (2 * d) * 7)) ** (1.0 / d) / (p + 1))
    nmax = max(2 if p >= 3 else 3, nmax)
    if cfg["n"] <= nmax:
        return cfg, False
    return synth.config(cfg["name"], **{k: cfg[k] for k in ("p", "k", "rho")}, n=nmax), True


def workload_name(cfg):
    shape = "L-shape 3 patches" if cfg.get("lshape") else ("unit square" if cfg["dim"] == 2 else "unit cube")
    kind = "elasticity" if cfg.get("ncomp", 1) > 1 else "scalar wave"
    return (f"{cfg['name']}: {cfg['dim']}D {kind}, {shape}, p={cfg['p']}, n={cfg['n']} elements/dir, "
            f"+-{cfg['noise']}h control-point noise (seed {cfg['seed']}), k={cfg['k']}, rho={cfg['rho']}, "
            f"dt={cfg['cfl_frac']} CFL")


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([c.strip() for c in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)
        sms = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# --------------------------------------------------------------------------- CPU oracle timing
def oracle_timing(cfg, nsteps, warmup=0, budget_s=None):
    """Time the oracle (oracle/, as it stands) on this host: setup excluded,
    then `warmup` untimed and `nsteps` timed steps (fewer if `budget_s` seconds
    of stepping run out first; at least one).  Single-threaded SciPy."""
    import numpy as np

    import synth
    from oracle import assembly, integrator
    prob = synth.make_problem(cfg)
    nc = cfg.get("ncomp", 1)
    mat = dict(lam=cfg.get("lam", 1.0), mu=cfg.get("mu", 1.0), density=cfg.get("density", 1.0)) if nc > 1 else {}
    t0 = time.perf_counter()
    d = assembly.Discretization(prob["patches"], cfg["p"], cfg["n"], cfg["dim"], ncomp=nc, **mat)
    it = integrator.Integrator(d.M, d.K, cfg["k"], cfg["rho"], 1e-4)
    t_setup = time.perf_counter() - t0
    u0 = d.restrict_local(prob["u0"])
    c = it.init(u0, np.zeros_like(u0))
    tw = time.perf_counter()
    done_w = 0
    for _ in range(warmup):
        c = it.step(c)
        done_w += 1
        if budget_s is not None and time.perf_counter() - tw > 0.2 * budget_s:
            break
    t0 = time.perf_counter()
    done = 0
    for _ in range(nsteps):
        c = it.step(c)
        done += 1
        if budget_s is not None and time.perf_counter() - t0 > budget_s:
            break
    t = time.perf_counter() - t0
    return dict(n_free=d.nfree * nc, seconds=t, setup_s=t_setup, steps=done, warmup=done_w)


def full_n_free(cfg):
    """Free DoFs of a single-patch configuration: (n + p - 2)^dim per component."""
    return (cfg["n"] + cfg["p"] - 2) ** cfg["dim"] * cfg.get("ncomp", 1)


def cpu_cores_used():
    return 1  # SuperLU triangular solves and SciPy CSR matvec are single-threaded


# --------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return
    full = make_cfg(args)
    cfg, extrap = oracle_sample_cfg(full)
    steps, warm = args.steps, args.warmup
    # bound the run to a few minutes: time K steps only if they fit, else a prefix
    r = oracle_timing(cfg, steps, warm, budget_s=150.0)
    w_eff = r["warmup"]
    value = r["n_free"] * r["steps"] / r["seconds"]
    sample = (f"{r['steps']} timed steps (+{w_eff} warm-up) of the {cfg['name']} workload after "
              f"{r['setup_s']:.1f}s untimed setup (assembly + sparse LU); steps requested {steps}")
    if extrap:
        sample += (f"; at n={cfg['n']} ({r['n_free']} DoFs, same p, k, rho and geometry recipe): the oracle "
                   f"cannot assemble M, K at n={full['n']} (sparse products over the Gauss points, > 200 GB), "
                   "so the per-DoF rate is extrapolated to the full size (an upper bound for the oracle there)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": r["steps"], "warmup": w_eff, "ms_per_step": 1e3 * r["seconds"] / r["steps"],
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(full),
                   "n_free": full_n_free(full) if extrap else r["n_free"], "sample_n_free": r["n_free"]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu_cores_used(), "kind": "oracle",
                         "sample": sample, "host_cpus": os.cpu_count(), "extrapolated": extrap},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- replicas
def aggregate_replicas(local_ms, local_units, world, device=None):
    """Multi-GPU = independent replicas: the job time is
    the MAX of the ranks' device times, the work is the SUM of their units.
    Returns (t_max_ms, total_units).  Only scalars cross ranks."""
    if world <= 1:
        return float(local_ms), float(local_units)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(local_ms)], dtype=torch.float64, device=device)
    u = torch.tensor([float(local_units)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(u, op=dist.ReduceOp.SUM)
    return float(t.item()), float(u.item())


# --------------------------------------------------------------------------- our arm
def algorithmic_bytes(op, ctx_info):
    """Algorithmic (compulsory) bytes per launch, DESIGN.md "Roofline":
    op 0 M SpMV + p.q: S coefficients per row (shared by the k RHS), read p, write q.
    op 1 K SpMV: S (x9 elastic) coefficients per row, read s, write b.
    op 2 preconditioner: read r, write z, read s twice, d line passes of read+write.
    op 3 predictor pass: read 3k chain values, write k predictors."""
    N, S, nv, k, d = ctx_info["npts"], ctx_info["S"], ctx_info["nvec"], ctx_info["k"], ctx_info["dim"]
    if op == 0:
        return 8 * S * N + 16 * nv * k * N
    if op == 1:
        return 8 * S * N * (9 if nv == 3 else 1) + 16 * nv * k * N
    if op == 2:
        return 16 * nv * k * N * (1 + d) + 16 * N
    return 8 * nv * N * (3 * k + k)


# B200 fp64: 148 SMs x 64 DFMA/clk/SM x 2 flop x 1.965 GHz (sm_max_mhz) = 37.2 TFLOP/s
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def matfree_flops(op, cfg, nf):
    """Algorithmic flops of one matrix-free apply (op 0 = M, op 1 = scalar K) over the k
    right-hand sides: the non-redundant global sum factorisation,
    forward contractions z, x, y (free bases -> Gauss points), the pointwise W product and
    the mirrored backward contractions; 2 flops per FMA."""
    p, n, d, k = cfg["p"], cfg["n"], cfg["dim"], cfg["k"]
    q = n * (p + 1)
    if d == 3:
        stages = [nf * nf * q, nf * q * q, q * q * q]
    else:
        stages = [nf * q, q * q]
    if op == 0:
        fwd = sum(stages) * (p + 1)
        return k * (2 * 2 * fwd + q ** d) * cfg.get("ncomp", 1)
    fields = [2, 3, 3] if d == 3 else [2, 2]
    fwd = sum(f * st for f, st in zip(fields, stages)) * (p + 1)
    wprod = (d * d) * 2 * q ** d
    return k * (2 * 2 * fwd + wprod)


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_2102_11536_b200 import Context, ga_params, make_desc
    import synth

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cfg = make_cfg(args)
    prob = synth.make_problem(cfg)
    nc = cfg.get("ncomp", 1)
    mat = dict(lam=cfg.get("lam", 1.0), mu=cfg.get("mu", 1.0), density=cfg.get("density", 1.0)) if nc > 1 else {}
    _, _, _, _, thmax = ga_params(cfg["k"], cfg["rho"])
    # dt from the GPU's own lambda_max estimate (power iteration through the library)
    probe = Context(make_desc(prob["patches"], cfg["p"], cfg["n"], cfg["dim"], ncomp=nc, k=cfg["k"], rho=cfg["rho"],
                              dt=1e-6, op_mode=args.op_mode, **mat), device=dev)
    lam = probe.lambda_max(args.lam_iters)
    probe.close()
    del probe
    dt = cfg["cfl_frac"] * math.sqrt(thmax / lam)
    desc = make_desc(prob["patches"], cfg["p"], cfg["n"], cfg["dim"], ncomp=nc, k=cfg["k"], rho=cfg["rho"], dt=dt,
                     op_mode=args.op_mode, **mat)
    ctx = Context(desc, device=dev)
    stream = ctx.stream
    fmap = ctx.free_dof_map()
    m = cfg["n"] + cfg["p"]
    mpow = m ** cfg["dim"]
    u0_np = np.concatenate([np.array([prob["u0"][int(v // mpow)][int(v % mpow), c] for v in fmap])
                            for c in range(nc)])
    u0 = torch.tensor(u0_np, dtype=torch.float64, device=dev)
    v0 = None
    if prob.get("v0") is not None:  # E1: V0 != 0 (initial chain with a velocity, R3)
        v0 = torch.tensor(np.concatenate([np.array([prob["v0"][int(v // mpow)][int(v % mpow), c] for v in fmap])
                                          for c in range(nc)]), dtype=torch.float64, device=dev)
    ctx.set_state(u0, v0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(args.warmup):
        ctx.advance(1)
        flush.zero_()
    torch.cuda.synchronize()
    st0 = ctx.stats()
    if st0.status != 0:
        raise RuntimeError(f"warm-up failed: status {st0.status}")
    sampler = ClockSampler(local_rank)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    sampler.start()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for e0, e1 in evs:
        e0.record(stream)
        ctx.advance(1)
        e1.record(stream)
        flush.zero_()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = sampler.stop()
    ms = sum(e0.elapsed_time(e1) for e0, e1 in evs)
    st1 = ctx.stats()
    if st1.status != 0:
        raise RuntimeError(f"timed run failed: status {st1.status}")
    launches = st1.kernel_launches - st0.kernel_launches
    loop_iters = st1.loop_iters - st0.loop_iters
    solves = st1.solves - st0.solves
    its = sum(st1.pcg_iters[j] - st0.pcg_iters[j] for j in range(4))
    n_free = ctx.n_free
    t_max, units = aggregate_replicas(ms, n_free * args.steps, world, dev)
    value = units / (t_max * 1e-3)

    # ---- per-kernel timing (events on the launching stream, L2 flushed before each launch)
    info = dict(npts=n_free // nc if not cfg.get("lshape") else None, S=(2 * cfg["p"] + 1) ** cfg["dim"], nvec=nc,
                k=cfg["k"], dim=cfg["dim"])
    # grid points (incl. masked) for the multi-patch layout
    G = [(max(c[d] for c, _ in prob["patches"]) + 1) * (m - 1) - 1 for d in range(cfg["dim"])]
    info["npts"] = int(np.prod(G))
    kern = {}
    names = {0: "k_spmv_sm(M)+p.q", 1: "k_spmv_sm(K)", 2: "preconditioner (Kronecker line solves x d, scaling, PCG update, dots)",
             3: "k_stage(predictor pass)", 5: "k_p_update"}
    persistent = ctx.persistent()
    mfree = ctx.matrix_free()
    opmode = ctx.operator_mode()  # 1 full stencils, 2 matrix-free, 3 half-symmetric stencils
    if opmode == 3:  # compulsory coefficient bytes of the half layout: (S + 1) / 2 per row
        info["S"] = (info["S"] + 1) // 2
        sym = cfg["dim"] == 3 and nc == 1  # single-read SpMV (spmv_sym.cu)
        names[0] = "k_spmv_sym(M)+p.q" if sym else "k_spmv_half(M)+p.q"
        if nc == 1:
            names[1] = "k_spmv_sym(K)" if sym else "k_spmv_half(K)"
    if mfree:
        names[0] = "k_mf3/k_mf2(M, matrix-free)+p.q"
        if nc == 1:
            names[1] = "k_mf3/k_mf2(K, matrix-free)"
    ops = [0, 1, 2, 3, 5] + ([6] if persistent else [])
    steps = args.steps
    L = loop_iters / steps  # lock-stepped PCG iterations per step (one solve set per step)
    nsolve_phases = 2 if True else 1  # main phase + refinement restart
    info_bytes = {op: algorithmic_bytes(op, info) for op in (0, 1, 2, 3)}
    if cfg.get("lshape"):  # masked grid: only the free rows have coefficients to read (masked row blocks are skipped)
        for op in (0, 1):
            info_bytes[op] = algorithmic_bytes(op, dict(info, npts=n_free // nc))
    if opmode == 3 and nc == 3:  # the elastic K stays a full 3x3-block stencil
        info_bytes[1] = algorithmic_bytes(1, dict(info, S=(2 * cfg["p"] + 1) ** cfg["dim"]))
    info_bytes[5] = 24 * info["nvec"] * info["k"] * info["npts"]
    # whole solve: L SpMV + 1 true-residual SpMV, L + 2 preconditioner applications, L direction updates
    info_bytes[6] = (L + 1) * info_bytes[0] + (L + 2) * info_bytes[2] + L * info_bytes[5]
    names[6] = "k_pcg_persist (one cooperative kernel = whole lock-stepped solve)"
    for op in ops:
        durs = []
        for _ in range(args.kernel_reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            ctx.profile_op(op, 1)
            e1.record(stream)
            torch.cuda.synchronize()
            durs.append(e0.elapsed_time(e1))
        avg = sum(durs) / len(durs)
        kern[op] = dict(name=names[op], ms=avg, bytes=info_bytes[op])
        if mfree and op == 0 and cfg["dim"] == 3:
            # multi-pass mass (matfree_mp.cu, HBM streams): Gauss weights once + per DoF and rhs the
            # intermediates 2 + 2(p+1) + 2(p+1)^2 doubles
            qd, p1 = cfg["n"] * (cfg["p"] + 1), cfg["p"] + 1
            kern[op]["bytes"] = 8 * qd ** 3 + 8 * nc * cfg["k"] * info["npts"] * (2 + 2 * p1 + 2 * p1 * p1)
            names[0] = "k_mp_* (M, matrix-free multi-pass)+p.q"
            kern[op]["name"] = names[0]
        elif mfree and (op == 0 or (op == 1 and nc == 1)):
            nfd = G[0]  # free bases per direction (single patch)
            qd = cfg["n"] * (cfg["p"] + 1)
            # compulsory bytes: Gauss-point data once (1 or d(d+1)/2 values), read x, write y
            kern[op]["bytes"] = 8 * qd ** cfg["dim"] * (1 if op == 0 else cfg["dim"] * (cfg["dim"] + 1) // 2) + \
                16 * nc * cfg["k"] * info["npts"]
            kern[op]["flops"] = matfree_flops(op, cfg, nfd)
    if persistent:
        per_step_launches = {0: 0.0, 1: 1.0, 2: 0.0, 3: 1.0, 5: 0.0, 6: 1.0}
    else:
        per_step_launches = {0: L + 1, 1: 1.0, 2: L + 2, 3: 1.0, 5: L, 6: 0.0}
    share = {op: kern[op]["ms"] * per_step_launches[op] / (ms / steps) for op in kern}
    dom = max(share, key=lambda o: share[o])
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = peaks.get("hbm_gbs", 6650.0)
    achieved = kern[dom]["bytes"] / (kern[dom]["ms"] * 1e-3) / 1e9
    alu = "flops" in kern[dom]
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            traffic = json.load(open(tf)).get(f"{cfg['name']}_p{cfg['p']}_n{cfg['n']}_k{cfg['k']}", {}).get(str(dom))
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic, "kernel": kern[dom]["name"], "kernel_ms": kern[dom]["ms"],
                "algorithmic_bytes": kern[dom]["bytes"],
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)" if "hbm_gbs" in peaks else "fallback",
                "timing": "CUDA events on the launching stream, L2 flushed before each launch, "
                          f"mean of {args.kernel_reps} launches after the timed region",
                "kernels": {kern[o]["name"]: {"ms": kern[o]["ms"], "GB/s": kern[o]["bytes"] / kern[o]["ms"] / 1e6,
                                              "frac": kern[o]["bytes"] / kern[o]["ms"] / 1e6 / peak,
                                              "launches_per_step": per_step_launches[o],
                                              "est_share_of_step": share[o]} for o in kern},
                "note": ("persistent solver: the whole lock-stepped solve is one launch; its 'achieved' counts the "
                         "algorithmic bytes of all its SpMVs, preconditioner applications and updates" if persistent
                         else "separate kernels per PCG phase inside a CUDA graph")}
    if alu:  # matrix-free operator: fp64-ALU bound
        tf = kern[dom]["flops"] / (kern[dom]["ms"] * 1e-3) / 1e12
        roofline.update({"bound": "alu", "achieved": tf, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": tf / FP64_PEAK_TFLOPS, "algorithmic_flops": kern[dom]["flops"],
                         "hbm_GB/s": achieved,
                         "peak_source": "derived: 148 SMs x 64 DFMA/clk x 2 x 1.965 GHz (DESIGN.md)"})
    for o in kern:
        if "flops" in kern[o]:
            roofline["kernels"][kern[o]["name"]]["TFLOP/s"] = kern[o]["flops"] / kern[o]["ms"] / 1e9

    # ---- end to end through the public API with host buffers
    u0_host = torch.tensor(u0_np, dtype=torch.float64).pin_memory()
    u_host = torch.empty(n_free, dtype=torch.float64).pin_memory()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    u0_dev = torch.empty(n_free, dtype=torch.float64, device=dev)
    u0_dev.copy_(u0_host, non_blocking=True)
    ctx.set_state(u0_dev)
    u_dev = ctx.vec()
    for _ in range(args.steps):
        ctx.advance(1)
        ctx.get_state_into(u_dev)
        u_host.copy_(u_dev, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms, e2e_units = aggregate_replicas(e0.elapsed_time(e1), n_free * args.steps, world, dev)
    e2e = {"value": e2e_units / (e2e_ms * 1e-3), "unit": UNIT,
           "h2d_bytes_per_step": 8 * n_free / args.steps, "d2h_bytes_per_step": 8 * n_free,
           "note": "one job through the C ABI: pinned H2D of U0, ga_set_state (initial chain, "
                   f"{3 * cfg['k'] - 2} solves), then per step ga_advance(1) + D2H of U into pinned memory"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload_name(cfg), "n_free": n_free, "dt": dt, "lambda_max": lam,
                           "pcg_rtol": 1e-13, "pcg_iters_per_solve": its / max(1, solves),
                           "lockstep_iters_per_step": loop_iters / steps,
                           "l2": "flushed between timed steps (256 MiB write), working set "
                                 f"{ctx.workspace.numel() / 2**20:.0f} MiB",
                           "parallelism": f"replicas x{world}" if world > 1 else "single GPU",
                           "operators": {1: "stencil", 2: "matrix-free", 3: "half-symmetric stencil"}[opmode]},
                "roofline": roofline, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": {k: clocks[k] for k in ("sm_mhz", "sm_max_mhz", "reasons")}}
        if world == 1 and not args.no_cpu_baseline:
            ref_steps = 3
            scfg, extrap = oracle_sample_cfg(cfg)
            r = oracle_timing(scfg, ref_steps, 0)
            sample = (f"{ref_steps} steps of the same workload after {r['setup_s']:.1f}s untimed oracle setup "
                      "(assembly + sparse LU)")
            if extrap:
                sample = (f"{ref_steps} steps at n={scfg['n']} ({r['n_free']} DoFs; same p, k, rho and geometry "
                          f"recipe) after {r['setup_s']:.1f}s untimed setup: the oracle cannot assemble M, K at "
                          f"n={cfg['n']} (> 200 GB of sparse products), so its per-DoF rate is extrapolated "
                          "(an upper bound for the oracle at full size)")
            line["cpu_baseline"] = {"value": r["n_free"] * r["steps"] / r["seconds"], "unit": UNIT,
                                    "cores": cpu_cores_used(), "kind": "oracle", "sample": sample,
                                    "host_cpus": os.cpu_count(), "extrapolated": extrap}
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # --gpus N outside torchrun: relaunch as N ranks (one process per GPU) on this node
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", os.environ.get("MASTER_PORT", "29517"),
               os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    if args.gpus != world:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "ours":
            torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
