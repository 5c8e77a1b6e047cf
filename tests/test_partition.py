"""CPU tests of the partitioned multi-patch mode (patch-per-GPU):

* the library's partition plan (ga_partition_plan, C++ host code) against the oracle's gluing of
  the same patches by coincident control points (oracle/assembly.py Discretization):
  free DoFs, one owner per global DoF, interface slots shared by exactly the copies;
* the exchange protocol of ga_group (dist.cu) on two gloo ranks: a host model of the group PCG
  -- local patch operators M^(r) (oracle.patch_operators), local additive-Schwarz terms (oracle
  KronFactor), the plan's interface slots and owned masks, one all-reduce of [interface values |
  partial sums] per exchange -- must reproduce the oracle's global PCG solve with the global
  Schwarz preconditioner: same iteration count, same solution.  This checks the
  plan and the algebra of the exchanges (p.q and r.z from unassembled local products, owned
  norms, global diag(M) in the scaling); the GPU kernels of the same protocol are compared with
  the oracle in tests/test_gpu_group.py.
"""
import os
import socket

import numpy as np
import pytest

import synth
from oracle import assembly, precond

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ga():
    from paper_2102_11536_b200 import build
    build.build()
    import paper_2102_11536_b200.genalpha as g
    return g


def _cases():
    return [
        ("lshape_p3_n4", synth.lshape_patches(3, 4, 0.1, 5), 3, 4, 2),
        ("fan2d_p2_n3", synth.fan_patches(2, 2, 3, 7, 0.1, 6), 2, 3, 2),
        ("fan2d_p3_n5", synth.fan_patches(2, 3, 5, 7, 0.1, 6), 3, 5, 2),
        ("fan3d_p2_n3", synth.fan_patches(3, 2, 3, 7, 0.1, 7), 2, 3, 3),
        ("fan5_3d_p1_n2", synth.fan_patches(3, 1, 2, 5, 0.0, 7), 1, 2, 3),
    ]


@pytest.mark.parametrize("name,patches,p,n,dim", _cases(), ids=[c[0] for c in _cases()])
def test_plan_matches_oracle_gluing(ga, name, patches, p, n, dim):
    d = assembly.Discretization(patches, p, n, dim)
    plan = ga.PartitionPlan([c for _, c in patches], p, n, dim)
    assert plan.n_free == d.nfree
    owners = np.zeros(d.nfree, dtype=int)
    copies = np.zeros(d.nfree, dtype=int)
    for r, G in enumerate(d.G):
        sub = plan.sub[r]
        np.testing.assert_array_equal(sub.free_mask.astype(bool), G >= 0)
        np.add.at(owners, G[sub.owned.astype(bool)], 1)
        np.add.at(copies, G[G >= 0], 1)
        assert not np.any(sub.owned[G < 0])
    assert np.all(owners == 1)  # every global free DoF is counted by exactly one subdomain
    # interface slots: exactly the DoFs with >= 2 copies, one slot per global DoF, shared
    slot_of = {}
    for r, G in enumerate(d.G):
        it = plan.sub[r].iface
        for loc in np.nonzero(G >= 0)[0]:
            g = int(G[loc])
            if copies[g] >= 2:
                assert it[loc] >= 0
                assert slot_of.setdefault(g, int(it[loc])) == int(it[loc])
            else:
                assert it[loc] == -1
        assert np.all(it[G < 0] == -1)
    assert plan.n_iface == len(slot_of) == int(np.sum(copies >= 2))
    assert sorted(slot_of.values()) == list(range(plan.n_iface))
    if name.startswith("fan"):
        assert copies.max() == len(patches)  # all patches meet at the centre vertex / axis


def test_plan_rejects_nonconforming(ga):
    patches = synth.lshape_patches(2, 3, 0.0, 5)
    m = 5
    ctrl_b = patches[1][1].copy()
    # move one point of B's left face (the A-B interface) off A's right face
    i = 0 + m * 2
    ctrl_b[i, 0] += 1e-3
    with pytest.raises(ga.GAError) as e:
        ga.PartitionPlan([patches[0][1], ctrl_b, patches[2][1]], 2, 3, 2)
    assert e.value.code == ga.GA_ERR_CONFORMITY


# ------------------------------------------------------------------------------------------
# host model of the group PCG on two gloo ranks
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class _Sub:
    """One subdomain of the model: local operators on the patch's free local points, the
    plan's exchange lists, the local Schwarz term with the scaling from the global diagonal."""

    def __init__(self, ctrl, p, n, dim, sub):
        M, K = assembly.patch_operators(ctrl, p, n, dim)
        self.free = np.nonzero(sub.free_mask)[0]
        self.M = M[self.free][:, self.free].tocsr()
        self.K = K[self.free][:, self.free].tocsr()
        self.own = sub.owned[self.free].astype(float)
        it = sub.iface[self.free]
        self.xl = np.nonzero(it >= 0)[0]        # held interface DoFs (local free index)
        self.xs = it[self.xl]                   # their slots
        m = n + p
        idx = np.indices((m,) * dim).reshape(dim, -1)[::-1][:, self.free]
        lo, hi = idx.min(axis=1), idx.max(axis=1)
        self.fac = precond.KronFactor(p, n, lo, hi)
        dims = self.fac.dims
        self.boxpos = np.zeros(self.free.size, dtype=np.int64)
        stride = 1
        for a in range(dim):
            self.boxpos += (idx[a] - lo[a]) * stride
            stride *= dims[a]
        self.nbox = int(np.prod(dims))

    def set_scaling(self, diag_global):
        self.s = np.sqrt(self.fac.Dhat[self.boxpos] / diag_global)

    def schwarz(self, r):
        t = np.zeros(self.nbox)
        t[self.boxpos] = self.s * r
        return self.s * self.fac.solve(t)[self.boxpos]


def _exchange(dist, torch, subs, n_iface, vals, scal):
    """One group exchange: [interface values | scalars] summed over all subdomains."""
    buf = np.zeros(n_iface + len(scal))
    for sd, v in zip(subs, vals):
        if v is not None:
            buf[sd.xs] += v[sd.xl]
    buf[n_iface:] = scal
    t = torch.tensor(buf)
    dist.all_reduce(t)
    out = t.numpy()
    if vals[0] is not None:
        for sd, v in zip(subs, vals):
            v[sd.xl] = out[sd.xs]
    return out[n_iface:]


def _group_pcg_worker(rank, world, port, case, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2102_11536_b200.genalpha as ga
    name, patches, p, n, dim = [c for c in _cases() if c[0] == case][0]
    plan = ga.PartitionPlan([c for _, c in patches], p, n, dim)
    mine = [r for r in range(len(patches)) if r % world == rank]  # round-robin patch-per-rank
    subs = [_Sub(patches[r][1], p, n, dim, plan.sub[r]) for r in mine]
    d = assembly.Discretization(patches, p, n, dim)
    ni = plan.n_iface
    # global diag(M): sum of the local diagonals over the copies
    diags = [sd.M.diagonal().copy() for sd in subs]
    _exchange(dist, torch, subs, ni, diags, [])
    for sd, dg in zip(subs, diags):
        sd.set_scaling(dg)
    # right-hand side: b = -K u0 of a smooth field (consistent), by the group K apply
    u0 = [synth.eval_modes(synth.sine_modes(3), patches[r][1])[sd.free] for r, sd in zip(mine, subs)]
    b = [-(sd.K @ u) for sd, u in zip(subs, u0)]
    _exchange(dist, torch, subs, ni, b, [])
    # group PCG, the sequence of dist.cu: init (||b||^2 owned) | precond + exchange (r.z, r.r)
    # | loop { p = z + beta p ; q = M p + exchange (p.q) ; x, r update ; precond + exchange }
    x = [np.zeros_like(v) for v in b]
    r = [v.copy() for v in b]
    (bb,) = _exchange(dist, torch, subs, ni, [None] * len(subs), [sum(float(sd.own @ (v * v)) for sd, v in zip(subs, b))])
    z = [sd.schwarz(v) for sd, v in zip(subs, r)]
    rz, rr = _exchange(dist, torch, subs, ni, z, [sum(float(a @ c) for a, c in zip(r, z)),
                                                   sum(float(sd.own @ (v * v)) for sd, v in zip(subs, r))])
    pv = [v.copy() for v in z]
    it = 0
    while rr > 1e-26 * bb and it < 500:
        q = [sd.M @ v for sd, v in zip(subs, pv)]
        (pq,) = _exchange(dist, torch, subs, ni, q, [sum(float(a @ c) for a, c in zip(pv, q))])
        al = rz / pq
        x = [a + al * c for a, c in zip(x, pv)]
        r = [a - al * c for a, c in zip(r, q)]
        it += 1
        z = [sd.schwarz(v) for sd, v in zip(subs, r)]
        rz_new, rr = _exchange(dist, torch, subs, ni, z, [sum(float(a @ c) for a, c in zip(r, z)),
                                                           sum(float(sd.own @ (v * v)) for sd, v in zip(subs, r))])
        if rr <= 1e-26 * bb:
            break
        pv = [zz + (rz_new / rz) * pp for zz, pp in zip(z, pv)]
        rz = rz_new
    # the oracle: global assembly, global Schwarz preconditioner, textbook PCG
    ug = d.restrict_local([synth.eval_modes(synth.sine_modes(3), c)[:, None] for _, c in patches])
    bg = -(d.K @ ug)
    xg, itg, _ = precond.pcg(lambda v: d.M @ v, bg, precond.SchwarzPreconditioner(d), tol=1e-13)
    err = 0.0
    for rr_, sd, xx in zip(mine, subs, x):
        g = d.G[rr_][sd.free]
        err = max(err, float(np.max(np.abs(xx - xg[g]))) / float(np.max(np.abs(xg))))
    out[rank] = (it, itg, err)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("case", ["lshape_p3_n4", "fan2d_p3_n5", "fan3d_p2_n3"])
def test_group_pcg_protocol_two_gloo_ranks(ga, case):
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_group_pcg_worker, args=(2, _free_port(), case, out), nprocs=2, join=True)
    for rank in (0, 1):
        it, itg, err = out[rank]
        assert abs(it - itg) <= 1, (it, itg)
        assert err < 1e-11, err
