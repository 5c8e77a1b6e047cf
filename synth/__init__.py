"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no basis functions, no
quadrature, no operators, no time stepping).  It only produces the inputs a
user hands to the library: control-point nets, initial coefficient vectors and
the configuration table of BASELINE.json.  Both the CPU oracle (`oracle/`) and
the CUDA path (`paper_2102_11536_b200`) consume these arrays; neither imports
the other.

Recipe:
  * control points sit at the Greville abscissae (xi_{i+1}+...+xi_{i+p})/p of
    the open uniform knot vector, which makes the undeformed map the identity;
  * patch-interior control points get independent uniform noise
    U(-a*h, a*h) per coordinate, h = 1/n, from numpy PCG64(seed); points on a
    patch boundary are never moved (keeps the map onto the square/cube and the
    multi-patch interfaces conforming);
  * initial displacement coefficients are the control-point interpolation of
    u0(x) = sum_{m=1..8} a_m prod_d sin(m pi x_d), a_m ~ N(0,1)/m^2 (seeded),
    v0 = 0.
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "greville_1d", "control_net", "lshape_patches", "fan_patches", "sine_modes", "eval_modes",
    "sinpi_product", "e1_exact", "CONFIGS", "config", "make_problem",
]


def greville_1d(p: int, n: int) -> np.ndarray:
    """Greville abscissae of the open uniform knot vector with n elements, degree p.

    The knot vector is {0^(p+1), 1/n, ..., (n-1)/n, 1^(p+1)} (PAPER.md:529-536,
    uniform, maximal regularity PAPER.md:811).  Returned array has m = n+p
    entries.  Used only to *place* control points (input generation)."""
    inner = np.arange(1, n) / n
    knots = np.concatenate([np.zeros(p + 1), inner, np.ones(p + 1)])
    m = n + p
    g = np.array([knots[i + 1:i + p + 1].sum() / p for i in range(m)])
    g[0], g[-1] = 0.0, 1.0
    return g


def control_net(dim: int, p: int, n: int, noise: float = 0.0, seed: int = 0,
                origin=None, rng: np.random.Generator | None = None) -> np.ndarray:
    """Control-point net of one patch, shape (m**dim, dim), co-lexicographic
    (x fastest), xyz interleaved per point.

    noise = a: interior points (not on any patch face) move by U(-a h, a h) per
    coordinate with h = 1/n.  origin shifts the patch (unit square/cube cell)."""
    m = n + p
    g = greville_1d(p, n)
    axes = [g] * dim
    grids = np.meshgrid(*axes[::-1], indexing="ij")[::-1]  # x fastest
    pts = np.stack([gg.reshape(-1) for gg in grids], axis=1).astype(np.float64)
    if origin is not None:
        pts = pts + np.asarray(origin, dtype=np.float64)[None, :]
    if noise > 0.0:
        if rng is None:
            rng = np.random.default_rng(seed)
        idx = np.indices((m,) * dim).reshape(dim, -1)[::-1]  # idx[0] = x index
        interior = np.all((idx > 0) & (idx < m - 1), axis=0)
        h = 1.0 / n
        delta = rng.uniform(-noise * h, noise * h, size=pts.shape)
        pts[interior] += delta[interior]
    return pts


def lshape_patches(p: int, n: int, noise: float, seed: int):
    """Three unit-square patches tiling the L-shape [0,2]^2 minus (1,2]^2.

    Returns a list of (cell, ctrl) with cell = (cx, cy) the position of the
    patch in the coarse patch grid: A=(0,0), B=(1,0), C=(0,1).  One PCG64
    stream perturbs the patches in that order."""
    rng = np.random.default_rng(seed)
    out = []
    for cell in [(0, 0), (1, 0), (0, 1)]:
        ctrl = control_net(2, p, n, noise=noise, origin=cell, rng=rng)
        out.append((cell, ctrl))
    return out


def fan_patches(dim: int, p: int, n: int, npatch: int = 7, noise: float = 0.0, seed: int = 0,
                radius: float = 1.0, height: float = 1.0):
    """A fan of npatch (>= 3) kite-shaped patches around the origin (a
    generator standing in for the paper's seven-blade fan, whose CAD is not available).

    Patch r has the corners O = 0 (xi = eta = 0), A = R e(theta_r) (xi = 1), B = R e(theta_r +
    pi / npatch) (xi = eta = 1) and C = R e(theta_{r+1}) (eta = 1), theta_j = 2 pi j / npatch: its
    control points are the bilinear map of the Greville grid.  Neighbours share a ray edge with
    rotated parameter directions (patch r's eta axis = patch r+1's xi axis), all npatch patches
    share the centre vertex.  dim 3: the fan extruded over z in [0, height] (Greville in z), all
    patches share the centre axis.  Ray edges / faces are evaluated by one expression in both
    patches (bitwise-equal control points, conformity P:645-652); interior points get U(-a h, a h)
    noise per coordinate (h = radius / n), one PCG64 stream in patch order.  Returns
    [((r, 0, 0)[:dim], ctrl)]."""
    assert npatch >= 3
    m = n + p
    g = greville_1d(p, n)
    ray = [radius * np.array([np.cos(2 * np.pi * j / npatch), np.sin(2 * np.pi * j / npatch)])
           for j in range(npatch)]
    rng = np.random.default_rng(seed)
    h = radius / n
    out = []
    for r in range(npatch):
        A, C = ray[r], ray[(r + 1) % npatch]
        tb = 2 * np.pi * (r + 0.5) / npatch
        B = radius * np.array([np.cos(tb), np.sin(tb)])
        xi, eta = np.meshgrid(g, g, indexing="xy")  # [eta][xi], xi fastest
        xy = (xi * (1 - eta))[..., None] * A + (xi * eta)[..., None] * B + ((1 - xi) * eta)[..., None] * C
        xy[0, :, :] = g[:, None] * A[None, :]      # eta = 0 edge: shared with patch r-1
        xy[:, 0, :] = g[:, None] * C[None, :]      # xi = 0 edge: shared with patch r+1
        xy[0, 0, :] = 0.0
        pts2 = xy.reshape(-1, 2)
        if dim == 2:
            pts = pts2.copy()
            idx = np.indices((m, m)).reshape(2, -1)[::-1]
        else:
            gz = g * height
            pts = np.concatenate([np.tile(pts2, (m, 1)), np.repeat(gz, m * m)[:, None]], axis=1)
            idx = np.indices((m, m, m)).reshape(3, -1)[::-1]
        interior = np.all((idx > 0) & (idx < m - 1), axis=0)
        delta = rng.uniform(-noise * h, noise * h, size=pts.shape)
        pts[interior] += delta[interior]
        out.append(((r, 0, 0)[:dim], np.ascontiguousarray(pts)))
    return out


def sine_modes(seed: int, nmodes: int = 8) -> np.ndarray:
    """Amplitudes a_m ~ N(0,1)/m^2, m = 1..nmodes."""
    rng = np.random.default_rng(seed)
    a = rng.standard_normal(nmodes)
    return a / (np.arange(1, nmodes + 1, dtype=np.float64) ** 2)


def eval_modes(amp: np.ndarray, pts: np.ndarray) -> np.ndarray:
    """u0(x) = sum_m a_m prod_d sin(m pi x_d) at the points pts (npts, dim)."""
    u = np.zeros(pts.shape[0])
    for mi, a in enumerate(amp, start=1):
        u += a * np.prod(np.sin(mi * np.pi * pts), axis=1)
    return u


def sinpi_product(pts: np.ndarray) -> np.ndarray:
    """u0 = prod_d sin(pi x_d) (BASELINE.json configs[0])."""
    return np.prod(np.sin(np.pi * pts), axis=1)


# ---------------------------------------------------------------------------
# BASELINE.json configurations.  dt is NOT stored: it is
# cfl_frac * sqrt(Theta_max(rho) / lambda_max), computed by the harness.
CONFIGS = {
    "c1": dict(name="c1", dim=2, ncomp=1, p=2, n=16, noise=0.0, seed=1, init="sinpi",
               init_seed=101, k=2, rho=0.5, steps=200, cfl_frac=0.5, lshape=False),
    "c2": dict(name="c2", dim=2, ncomp=1, p=3, n=256, noise=0.2, seed=2, init="modes",
               init_seed=102, k=2, rho=0.0, steps=500, cfl_frac=0.8, lshape=False),
    "c3": dict(name="c3", dim=3, ncomp=1, p=2, n=32, noise=0.15, seed=3, init="modes",
               init_seed=103, k=2, rho=0.0, steps=100, cfl_frac=0.5, lshape=False),
    "c4": dict(name="c4", dim=3, ncomp=3, p=4, n=96, noise=0.15, seed=4, init="modes",
               init_seed=104, k=2, rho=0.5, steps=50, cfl_frac=0.5, lshape=False,
               lam=1.0, mu=1.0, density=1.0),
    "c5": dict(name="c5", dim=2, ncomp=1, p=3, n=512, noise=0.1, seed=5, init="modes",
               init_seed=105, k=2, rho=0.3, steps=200, cfl_frac=0.5, lshape=True),
    # the paper's own order-4 experiment (§6.1), unit square,
    # p=7, C^6, 100x100 elements, T = 0.1, u = sin(10 pi x) sin(10 pi y)[cos + sin](10 sqrt2 pi t)
    # (P:831 read as sin(10 pi y)); u0 = sin sin, v0 = 10 sqrt2 pi sin sin
    "e1": dict(name="e1", dim=2, ncomp=1, p=7, n=100, noise=0.0, seed=1, init="e1",
               init_seed=0, k=2, rho=0.0, steps=100, cfl_frac=0.5, lshape=False, T=0.1),
    # SURVEY §8f NEXT-4 (patch-per-GPU multi-patch): seven-patch fans, rotated interfaces, seven
    # patches at the centre vertex (2D) / axis (3D); stand-ins for the paper's fan
    "fan2d": dict(name="fan2d", dim=2, ncomp=1, p=3, n=256, noise=0.1, seed=6, init="modes",
                  init_seed=106, k=2, rho=0.3, steps=100, cfl_frac=0.5, lshape=False, fan=7),
    "fan3d": dict(name="fan3d", dim=3, ncomp=1, p=2, n=48, noise=0.1, seed=7, init="modes",
                  init_seed=107, k=2, rho=0.3, steps=50, cfl_frac=0.5, lshape=False, fan=7),
}


def e1_exact(pts: np.ndarray, t: float):
    """(u, u_t) of the E1 closed form (reading G24) at points pts (N, 2), time t."""
    w = 10.0 * np.sqrt(2.0) * np.pi
    sp = np.sin(10.0 * np.pi * pts[:, 0]) * np.sin(10.0 * np.pi * pts[:, 1])
    return sp * (np.cos(w * t) + np.sin(w * t)), sp * w * (np.cos(w * t) - np.sin(w * t))


def config(name: str, **over) -> dict:
    c = dict(CONFIGS[name])
    c.update(over)
    return c


def make_problem(cfg: dict):
    """Patches and per-patch initial displacement at every control point.

    Returns dict(patches=[(cell, ctrl)], u0=[per-patch array (m^dim, ncomp)]).
    Values at Dirichlet control points are returned too; consumers drop them."""
    dim, p, n = cfg["dim"], cfg["p"], cfg["n"]
    if cfg.get("cells"):
        # block-structured multi-patch domain: unit cells of the coarse patch grid (any dimension),
        # one PCG64 stream perturbs the interior points of the patches in the listed order
        rng = np.random.default_rng(cfg["seed"])
        patches = [(tuple(c), control_net(dim, p, n, noise=cfg["noise"], origin=tuple(c), rng=rng))
                   for c in cfg["cells"]]
    elif cfg.get("lshape"):
        patches = lshape_patches(p, n, cfg["noise"], cfg["seed"])
    elif cfg.get("fan"):
        patches = fan_patches(dim, p, n, cfg["fan"], cfg["noise"], cfg["seed"])
    else:
        patches = [((0,) * dim, control_net(dim, p, n, cfg["noise"], cfg["seed"]))]
    ncomp = cfg.get("ncomp", 1)
    u0 = []
    v0 = None
    if cfg["init"] == "sinpi":
        for _, ctrl in patches:
            u0.append(np.stack([sinpi_product(ctrl)] * ncomp, axis=1))
    elif cfg["init"] == "e1":
        v0 = []
        for _, ctrl in patches:
            uu, vv = e1_exact(ctrl, 0.0)
            u0.append(uu[:, None])
            v0.append(vv[:, None])
    else:
        amps = [sine_modes(cfg["init_seed"] + 1000 * c) for c in range(ncomp)]
        for _, ctrl in patches:
            u0.append(np.stack([eval_modes(a, ctrl) for a in amps], axis=1))
    return dict(patches=patches, u0=u0, v0=v0)
