"""ctypes binding of libgenalpha.so (include/genalpha.h).

Argument marshalling only: every step of the hot path runs in the CUDA
library.  PyTorch supplies device memory (workspace, scratch, vectors) and the
stream.  Importing this module on a machine without the built library raises:
there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, byref, c_double, c_int, c_longlong, c_size_t, c_void_p

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgenalpha.so")

GA_OK, GA_ERR_ARG, GA_ERR_PARAM, GA_ERR_GEOMETRY, GA_ERR_CONFORMITY = 0, -1, -2, -3, -4
GA_ERR_NOCONV, GA_ERR_UNSTABLE, GA_ERR_CUDA, GA_ERR_OOM = -5, -6, -7, -8
STATUS_NAMES = {0: "GA_OK", -1: "GA_ERR_ARG", -2: "GA_ERR_PARAM", -3: "GA_ERR_GEOMETRY",
                -4: "GA_ERR_CONFORMITY", -5: "GA_ERR_NOCONV", -6: "GA_ERR_UNSTABLE",
                -7: "GA_ERR_CUDA", -8: "GA_ERR_OOM"}

EXPORTED = ["ga_params", "ga_spectral_scan", "ga_query", "ga_create", "ga_set_state", "ga_set_forcing", "ga_set_time", "ga_set_dirichlet", "ga_advance", "ga_get_state",
            "ga_get_chain", "ga_set_chain", "ga_get_stats", "ga_apply", "ga_solve_mass",
            "ga_lambda_max", "ga_free_dof_map", "ga_profile_op", "ga_uses_persistent_solver", "ga_uses_matrix_free", "ga_operator_mode", "ga_destroy",
            "ga_last_error", "ga_partition_plan", "ga_group_create", "ga_group_set_state", "ga_group_advance",
            "ga_group_apply", "ga_group_solve_mass", "ga_group_set_forcing", "ga_group_destroy", "ga_group_last_error",
            "ga_nccl_unique_id", "ga_nccl_comm_init", "ga_nccl_comm_destroy"]


class ga_patch(ctypes.Structure):
    _fields_ = [("cell", c_int * 3), ("ctrl", POINTER(c_double))]


class ga_subdomain(ctypes.Structure):
    _fields_ = [("free_mask", POINTER(ctypes.c_ubyte)), ("owned", POINTER(ctypes.c_ubyte)),
                ("iface", POINTER(c_longlong)), ("n_iface", c_longlong)]


class ga_desc(ctypes.Structure):
    _fields_ = [("dim", c_int), ("ncomp", c_int), ("p", c_int), ("n", c_int), ("npatch", c_int),
                ("patches", POINTER(ga_patch)), ("omega", c_double), ("lame_lambda", c_double),
                ("lame_mu", c_double), ("density", c_double), ("k", c_int), ("rho_b", c_double),
                ("rho_s", c_double), ("param_set", c_int), ("dt", c_double), ("pcg_rtol", c_double),
                ("pcg_maxit", c_int), ("pcg_refine", c_int), ("pcg_refine_rtol", c_double),
                ("unstable_factor", c_double), ("op_mode", c_int), ("damp_a0", c_double),
                ("damp_a1", c_double), ("sub", POINTER(ga_subdomain))]


class ga_stats(ctypes.Structure):
    _fields_ = [("steps", c_longlong), ("solves", c_longlong), ("pcg_iters", c_longlong * 4),
                ("last_iters", c_int * 4), ("max_iters", c_int), ("max_rel_residual", c_double),
                ("status", c_int), ("fail_step", c_longlong), ("fail_block", c_int),
                ("kernel_launches", c_longlong), ("loop_iters", c_longlong), ("step_index", c_longlong)]


class GAError(RuntimeError):
    def __init__(self, code, msg=""):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2102_11536_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, D = POINTER(c_double), POINTER(ga_desc)
    sig = {
        "ga_params": (c_int, [c_int, c_double, c_double, c_int, P, P, P, P, P]),
        "ga_spectral_scan": (c_int, [c_int, c_double, c_double, c_int, c_void_p, c_int, c_void_p, c_void_p]),
        "ga_query": (c_int, [D, POINTER(c_size_t), POINTER(c_size_t), POINTER(c_size_t), POINTER(c_size_t)]),
        "ga_create": (c_int, [D, c_void_p, c_size_t, c_void_p, c_size_t, c_void_p, POINTER(c_void_p)]),
        "ga_set_state": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
        "ga_advance": (c_int, [c_void_p, c_int, c_void_p]),
        "ga_set_forcing": (c_int, [c_void_p, c_void_p, c_int, P, P, P, c_double, c_void_p]),
        "ga_set_time": (c_int, [c_void_p, c_longlong, c_void_p]),
        "ga_set_dirichlet": (c_int, [c_void_p, P, c_int, P, P, P, c_void_p, c_size_t, c_void_p]),
        "ga_get_state": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
        "ga_get_chain": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
        "ga_set_chain": (c_int, [c_void_p, c_int, c_void_p, c_void_p]),
        "ga_get_stats": (c_int, [c_void_p, POINTER(ga_stats), c_void_p]),
        "ga_apply": (c_int, [c_void_p, c_int, c_void_p, c_void_p, c_void_p]),
        "ga_solve_mass": (c_int, [c_void_p, c_void_p, c_void_p, POINTER(c_int), c_void_p]),
        "ga_lambda_max": (c_int, [c_void_p, c_int, P, c_void_p]),
        "ga_free_dof_map": (c_int, [c_void_p, POINTER(c_longlong)]),
        "ga_profile_op": (c_int, [c_void_p, c_int, c_int, c_void_p]),
        "ga_uses_persistent_solver": (c_int, [c_void_p]),
        "ga_uses_matrix_free": (c_int, [c_void_p]),
        "ga_operator_mode": (c_int, [c_void_p]),
        "ga_destroy": (None, [c_void_p]),
        "ga_last_error": (ctypes.c_char_p, [c_void_p]),
        "ga_partition_plan": (c_int, [c_int, c_int, c_int, c_int, POINTER(P), c_void_p, c_void_p, c_void_p,
                                      POINTER(c_longlong), POINTER(c_longlong)]),
        "ga_group_create": (c_int, [POINTER(c_void_p), c_int, c_void_p, c_void_p, POINTER(c_void_p)]),
        "ga_group_set_state": (c_int, [c_void_p, POINTER(c_void_p), POINTER(c_void_p), c_void_p]),
        "ga_group_advance": (c_int, [c_void_p, c_int, c_void_p]),
        "ga_group_apply": (c_int, [c_void_p, c_int, POINTER(c_void_p), POINTER(c_void_p), c_void_p]),
        "ga_group_solve_mass": (c_int, [c_void_p, POINTER(c_void_p), POINTER(c_void_p), POINTER(c_int), c_void_p]),
        "ga_group_set_forcing": (c_int, [c_void_p, c_int, c_void_p, c_int, P, P, P, c_double, c_void_p]),
        "ga_group_destroy": (None, [c_void_p]),
        "ga_group_last_error": (ctypes.c_char_p, [c_void_p]),
        "ga_nccl_unique_id": (c_int, [c_void_p]),
        "ga_nccl_comm_init": (c_int, [c_int, c_void_p, c_int, POINTER(c_void_p)]),
        "ga_nccl_comm_destroy": (None, [c_void_p]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype, f.argtypes = res, args
    return lib


lib = _load()


def _err(ctx=None):
    return lib.ga_last_error(ctx).decode(errors="replace")


def _check(code, ctx=None):
    if code != GA_OK:
        raise GAError(code, _err(ctx))


# --------------------------------------------------------------------------- raw calls
def ga_params(k, rho_b, rho_s=None, param_set=0):
    """(alpha, beta, gamma, alpha_f, theta_max) of the k blocks (host only)."""
    rho_s = rho_b if rho_s is None else rho_s
    arr = [(c_double * 4)() for _ in range(4)]
    th = c_double()
    _check(lib.ga_params(k, rho_b, rho_s, param_set, *arr, byref(th)))
    return tuple(np.array(a[:k]) for a in arr) + (th.value,)


def spectral_scan(theta, k, rho_b, rho_s=None, param_set=0):
    """rho(G(Theta)) for a CUDA float64 tensor of Theta values (ga_spectral_scan)."""
    import torch
    rho_s = rho_b if rho_s is None else rho_s
    th = theta.contiguous()
    out = torch.empty_like(th)
    _check(lib.ga_spectral_scan(int(k), float(rho_b), float(rho_s), int(param_set), c_void_p(th.data_ptr()),
                                th.numel(), c_void_p(out.data_ptr()), c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out


def make_desc(patches, p, n, dim, *, ncomp=1, k=2, rho=0.5, rho_s=None, dt=1e-3, param_set=0,
              omega=1.0, lam=1.0, mu=1.0, density=1.0, pcg_rtol=1e-13, pcg_maxit=500,
              pcg_refine=None, pcg_refine_rtol=None, unstable_factor=1e6, op_mode=0, damp_a0=0.0, damp_a1=0.0,
              sub=None):
    """ga_desc from [(cell, ctrl ndarray (m^dim, dim))].  Keeps the ctrl arrays
    alive on the returned object (`_keep`).  sub: a Subdomain of a PartitionPlan (one patch)
    for the partitioned (patch-per-GPU) mode, stepped through a Group."""
    arr = (ga_patch * len(patches))()
    keep = []
    for i, (cell, ctrl) in enumerate(patches):
        c = np.ascontiguousarray(ctrl, dtype=np.float64)
        keep.append(c)
        cc = list(cell) + [0] * (3 - len(cell))
        arr[i].cell = (c_int * 3)(*cc)
        arr[i].ctrl = c.ctypes.data_as(POINTER(c_double))
    d = ga_desc(dim=dim, ncomp=ncomp, p=p, n=n, npatch=len(patches), patches=arr, omega=omega,
                lame_lambda=lam, lame_mu=mu, density=density, k=k, rho_b=rho,
                rho_s=rho if rho_s is None else rho_s, param_set=param_set, dt=dt,
                pcg_rtol=pcg_rtol, pcg_maxit=pcg_maxit,
                # refinement restart (R8): needed where kappa(M) ~1e7-1e8 (3D p >= 5)
                pcg_refine=(1 if p >= 5 else 0) if pcg_refine is None else pcg_refine,
                pcg_refine_rtol=(1e-3 if p >= 5 else 0.0) if pcg_refine_rtol is None else pcg_refine_rtol,
                unstable_factor=unstable_factor, op_mode=op_mode, damp_a0=damp_a0, damp_a1=damp_a1)
    sd = None
    if sub is not None:
        sd = ga_subdomain(free_mask=sub.free_mask.ctypes.data_as(POINTER(ctypes.c_ubyte)),
                          owned=sub.owned.ctypes.data_as(POINTER(ctypes.c_ubyte)),
                          iface=sub.iface.ctypes.data_as(POINTER(c_longlong)), n_iface=int(sub.n_iface))
        d.sub = ctypes.pointer(sd)
    d._keep = (arr, keep, sd, sub)
    return d


def ga_query(desc):
    nf, ws, sc, sm = c_size_t(), c_size_t(), c_size_t(), c_size_t()
    _check(lib.ga_query(byref(desc), byref(nf), byref(ws), byref(sc), byref(sm)))
    return nf.value, ws.value, sc.value, sm.value


# --------------------------------------------------------------------------- torch-backed context
class Context:
    """Owns the torch-allocated workspace of one ga_ctx.  All vectors are
    torch float64 CUDA tensors of length n_free (free-DoF order)."""

    def __init__(self, desc, device="cuda", scratch_bytes=None, stream=None, guard_bytes=0):
        """guard_bytes > 0: the workspace handed to ga_create sits between two guard regions of
        that many bytes filled with a canary pattern (guards_intact() checks them: the memory
        checks of tests/test_gpu_guards.py; compute-sanitizer is not available on the GPU pool)."""
        import torch
        self.torch = torch
        self.desc = desc
        self.n_free, ws, sc, smin = ga_query(desc)
        if scratch_bytes is not None:
            sc = max(smin, scratch_bytes)
        g = (int(guard_bytes) + 255) // 256 * 256
        self._guard = g
        self._ws_bytes = ws
        self.workspace = torch.empty(ws + 512 + 2 * g, dtype=torch.uint8, device=device)
        if g:
            self.workspace.fill_(0xA5)
        base = _aligned(self.workspace).value + g
        self._ws_off = base - self.workspace.data_ptr()
        scratch = torch.empty(sc + 256, dtype=torch.uint8, device=device)
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        ctx = c_void_p()
        code = lib.ga_create(byref(desc), c_void_p(base), ws, _aligned(scratch), sc,
                             c_void_p(self.stream.cuda_stream), byref(ctx))
        del scratch
        if code != GA_OK:
            raise GAError(code, _err(None))
        self.ctx = ctx
        self.k = desc.k

    def _s(self):
        return c_void_p(self.stream.cuda_stream)

    def guards_intact(self):
        """True if no byte of the guard regions around the workspace was overwritten."""
        self.torch.cuda.synchronize()
        w = self.workspace
        lo = w[:self._ws_off]
        hi = w[self._ws_off + (self._ws_bytes + 255) // 256 * 256:]
        return bool((lo == 0xA5).all().item()) and bool((hi == 0xA5).all().item())

    def close(self):
        if getattr(self, "ctx", None):
            lib.ga_destroy(self.ctx)
            self.ctx = None

    __del__ = close

    def vec(self):
        return self.torch.zeros(self.n_free, dtype=self.torch.float64, device=self.workspace.device)

    def set_state(self, u0, v0=None):
        _check(lib.ga_set_state(self.ctx, _ptr(u0), _ptr(v0) if v0 is not None else None, self._s()), self.ctx)

    def set_forcing(self, G=None, terms=(), t0=0.0):
        """F(x, t) = G h(t), h(t) = sum a cos(w t + phi) for (a, w, phi) in terms; G: free-DoF
        tensor of the load integrals (None removes the forcing).  Call before set_state."""
        n = len(terms) if G is not None else 0
        arr = [(c_double * max(1, n))(*[t[i] for t in terms]) for i in range(3)]
        _check(lib.ga_set_forcing(self.ctx, _ptr(G) if G is not None else None, n, arr[0], arr[1], arr[2],
                                  float(t0), self._s()), self.ctx)

    def set_dirichlet(self, g=None, terms=()):
        """Boundary values U_b(t) = g_b h_D(t), h_D = sum a cos(w t + phi) for (a, w, phi) in terms;
        g: numpy array of all (n+p)^dim control values of the (single) patch, None removes it."""
        import numpy as _np
        torch = self.torch
        n = len(terms) if g is not None else 0
        arr = [(c_double * max(1, n))(*[t[i] for t in terms]) for i in range(3)]
        gp = None
        if g is not None:
            gc = _np.ascontiguousarray(g, dtype=_np.float64)
            gp = gc.ctypes.data_as(POINTER(c_double))
        _, _, sc, smin = ga_query(self.desc)
        sc += 8 * (self.desc.n + self.desc.p) ** self.desc.dim + 512  # + the uploaded control values
        scratch = torch.empty(sc + 256, dtype=torch.uint8, device=self.workspace.device)
        _check(lib.ga_set_dirichlet(self.ctx, gp, n, arr[0], arr[1], arr[2], _aligned(scratch), sc, self._s()),
               self.ctx)
        del scratch

    def set_time(self, step_index):
        """Simulation step index n of the state (t_n = t0 + n dt of the forcing), e.g. after
        ga_set_chain into a fresh context."""
        _check(lib.ga_set_time(self.ctx, int(step_index), self._s()), self.ctx)

    def advance(self, nsteps):
        _check(lib.ga_advance(self.ctx, int(nsteps), self._s()), self.ctx)

    def get_state(self):
        u, v, a = self.vec(), self.vec(), self.vec()
        _check(lib.ga_get_state(self.ctx, _ptr(u), _ptr(v), _ptr(a), self._s()), self.ctx)
        return u, v, a

    def get_state_into(self, u=None, v=None, a=None):
        _check(lib.ga_get_state(self.ctx, _ptr(u), _ptr(v), _ptr(a), self._s()), self.ctx)

    def get_chain(self, m):
        out = self.vec()
        _check(lib.ga_get_chain(self.ctx, m, _ptr(out), self._s()), self.ctx)
        return out

    def set_chain(self, m, x):
        _check(lib.ga_set_chain(self.ctx, m, _ptr(x), self._s()), self.ctx)

    def stats(self):
        st = ga_stats()
        _check(lib.ga_get_stats(self.ctx, byref(st), self._s()), self.ctx)
        return st

    def apply(self, which, x):
        y = self.vec()
        _check(lib.ga_apply(self.ctx, {"M": 0, "K": 1, "Pinv": 2}.get(which, which), _ptr(x), _ptr(y),
                            self._s()), self.ctx)
        return y

    def solve_mass(self, b, want_iters=True):
        x = self.vec()
        it = c_int(-1)
        code = lib.ga_solve_mass(self.ctx, _ptr(b), _ptr(x), byref(it) if want_iters else None, self._s())
        _check(code, self.ctx)
        return x, it.value

    def lambda_max(self, iters=50):
        lam = c_double()
        _check(lib.ga_lambda_max(self.ctx, iters, byref(lam), self._s()), self.ctx)
        return lam.value

    def profile_op(self, op, reps=1):
        _check(lib.ga_profile_op(self.ctx, int(op), int(reps), self._s()), self.ctx)

    def persistent(self):
        return bool(lib.ga_uses_persistent_solver(self.ctx))

    def matrix_free(self):
        return bool(lib.ga_uses_matrix_free(self.ctx))

    def operator_mode(self):
        """1 full stencils, 2 matrix-free, 3 half-symmetric stencils."""
        return int(lib.ga_operator_mode(self.ctx))

    def free_dof_map(self):
        ncomp = self.desc.ncomp
        out = (c_longlong * (self.n_free // ncomp))()
        _check(lib.ga_free_dof_map(self.ctx, out))
        return np.frombuffer(out, dtype=np.int64).copy()


# --------------------------------------------------------------------------- partitioned multi-patch
class Subdomain:
    """ga_subdomain arrays of one patch (host numpy, (n+p)^dim entries, co-lex)."""

    def __init__(self, free_mask, owned, iface, n_iface):
        self.free_mask = np.ascontiguousarray(free_mask, dtype=np.uint8)
        self.owned = np.ascontiguousarray(owned, dtype=np.uint8)
        self.iface = np.ascontiguousarray(iface, dtype=np.int64)
        self.n_iface = int(n_iface)


class PartitionPlan:
    """ga_partition_plan of a conforming multi-patch domain: .sub[r] (Subdomain of patch r),
    .n_iface, .n_free (global free DoFs)."""

    def __init__(self, ctrls, p, n, dim):
        m = n + p
        mp = m ** dim
        cs = [np.ascontiguousarray(c, dtype=np.float64).reshape(-1) for c in ctrls]
        for c in cs:
            assert c.size == mp * dim
        arr = (POINTER(c_double) * len(cs))(*[c.ctypes.data_as(POINTER(c_double)) for c in cs])
        fm = np.zeros(len(cs) * mp, dtype=np.uint8)
        ow = np.zeros(len(cs) * mp, dtype=np.uint8)
        it = np.zeros(len(cs) * mp, dtype=np.int64)
        ni, nf = c_longlong(), c_longlong()
        _check(lib.ga_partition_plan(int(dim), int(p), int(n), len(cs), arr, c_void_p(fm.ctypes.data),
                                     c_void_p(ow.ctypes.data), c_void_p(it.ctypes.data), byref(ni), byref(nf)))
        self.n_iface, self.n_free = ni.value, nf.value
        self.sub = [Subdomain(fm[r * mp:(r + 1) * mp], ow[r * mp:(r + 1) * mp], it[r * mp:(r + 1) * mp], ni.value)
                    for r in range(len(cs))]


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib.ga_nccl_unique_id(ctypes.cast(buf, c_void_p)))
    return buf.raw


def nccl_comm_init(nranks, uid: bytes, rank):
    buf = ctypes.create_string_buffer(uid, 128)
    comm = c_void_p()
    _check(lib.ga_nccl_comm_init(int(nranks), ctypes.cast(buf, c_void_p), int(rank), byref(comm)))
    return comm


def nccl_comm_destroy(comm):
    lib.ga_nccl_comm_destroy(comm)


def _gerr(g):
    return lib.ga_group_last_error(g).decode(errors="replace")


def _gcheck(code, g=None):
    if code != GA_OK:
        raise GAError(code, _gerr(g))


class Group:
    """ga_group over subdomain Contexts of this process (one NCCL communicator for the other
    processes of a multi-GPU run, None on one process).  Vectors are lists (one torch tensor
    per context, its free-DoF order)."""

    def __init__(self, contexts, nccl_comm=None, stream=None):
        import torch
        self.torch = torch
        self.ctxs = list(contexts)
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        arr = (c_void_p * len(self.ctxs))(*[c.ctx for c in self.ctxs])
        g = c_void_p()
        _gcheck(lib.ga_group_create(arr, len(self.ctxs), nccl_comm, c_void_p(self.stream.cuda_stream), byref(g)))
        self.g = g

    def _s(self):
        return c_void_p(self.stream.cuda_stream)

    @staticmethod
    def _arr(ts):
        return (c_void_p * len(ts))(*[None if t is None else _ptr(t) for t in ts])

    def close(self):
        if getattr(self, "g", None):
            lib.ga_group_destroy(self.g)
            self.g = None

    __del__ = close

    def set_state(self, u0s, v0s=None):
        _gcheck(lib.ga_group_set_state(self.g, self._arr(u0s), self._arr(v0s) if v0s is not None else None,
                                       self._s()), self.g)

    def set_forcing(self, i, G=None, terms=(), t0=0.0):
        """Forcing of context i: G its LOCAL load integrals (free-DoF tensor), terms (a, w, phi)."""
        n = len(terms) if G is not None else 0
        arr = [(c_double * max(1, n))(*[t[q] for t in terms]) for q in range(3)]
        _gcheck(lib.ga_group_set_forcing(self.g, int(i), _ptr(G) if G is not None else None, n, arr[0], arr[1],
                                         arr[2], float(t0), self._s()), self.g)

    def advance(self, nsteps):
        _gcheck(lib.ga_group_advance(self.g, int(nsteps), self._s()), self.g)

    def apply(self, which, xs):
        ys = [c.vec() for c in self.ctxs]
        _gcheck(lib.ga_group_apply(self.g, {"M": 0, "K": 1, "Pinv": 2}.get(which, which), self._arr(xs),
                                   self._arr(ys), self._s()), self.g)
        return ys

    def solve_mass(self, bs):
        xs = [c.vec() for c in self.ctxs]
        it = c_int(-1)
        _gcheck(lib.ga_group_solve_mass(self.g, self._arr(bs), self._arr(xs), byref(it), self._s()), self.g)
        return xs, it.value

    def get_state(self):
        return [c.get_state() for c in self.ctxs]

    def stats(self):
        return [c.stats() for c in self.ctxs]


def _aligned(t):
    base = t.data_ptr()
    return c_void_p((base + 255) & ~255)


def _ptr(t):
    if t is None:
        return None
    assert t.is_cuda and t.dtype.__str__() == "torch.float64" and t.is_contiguous()
    return c_void_p(t.data_ptr())
