"""Partitioned PCG + V-cycle (paper_2506_08284_b200/distributed.py) on CPU
with the gloo backend, world_size 2 and 3.

The distributed layer's partitioning, halo plans, halo exchanges,
all_reduce'd inner products and the replicated coarsest solve are the code
under test; the six local kernels are provided by a scipy implementation
here (the product injects CudaOps). The result must match the single-process
oracle solve on the same hierarchy.
"""

import os
import pickle
import socket
import tempfile
from types import SimpleNamespace

import numpy as np
import pytest
import scipy.sparse as sp
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hcurl_oracle as O
from paper_2506_08284_b200 import distributed as D
from paper_2506_08284_b200.inputs import discretize_hex


class ScipyOps:
    """Reference local kernels (test double for CudaOps)."""

    def _m(self, A):
        m = getattr(A, "_sp", None)
        if m is None:
            m = sp.csr_matrix((A.val.numpy(), A.col.numpy(), A.rowptr.numpy()), shape=A.shape)
            A._sp = m
        return m

    def spmv(self, A, x, y, alpha=1.0, beta=0.0, z=None):
        v = alpha * (self._m(A) @ x.numpy())
        if z is not None:
            v = v + beta * z.numpy()
        y.copy_(torch.from_numpy(v))

    def cheb(self, A, dinv, b, x_ext, x_out, d, cd, cr, x_zero):
        n = A.shape[0]
        ax = np.zeros(n) if x_zero else self._m(A) @ x_ext.numpy()
        dn = cd * d.numpy() + cr * (dinv.numpy() * (b.numpy() - ax))
        d.copy_(torch.from_numpy(dn))
        x0 = np.zeros(n) if x_zero else x_ext.numpy()[:n]
        x_out.copy_(torch.from_numpy(x0 + dn))

    def dot(self, x, y, out):
        out.fill_(float(x.numpy() @ y.numpy()))

    def gemv(self, M, x, y):
        y.copy_(M @ x)

    def gather(self, idx, x, out):
        out.copy_(x[idx])

    def copy(self, dst, src):
        dst.copy_(src)

    def pcg_update(self, sc, p, Ap, x, r, flag):
        pAp = float(sc[0])
        if not pAp > 0.0:
            return
        a = float(sc[2]) / pAp
        xn = x + a * p
        flag.fill_(int(bool((xn != x).any())))
        x.copy_(xn)
        r.sub_(a * Ap)

    def pcg_direction(self, sc, z, p):
        p.copy_(z + (float(sc[3]) / float(sc[2])) * p)

    def pcg_rotate(self, sc):
        sc[2] = sc[3]


def _levels(h):
    out = []
    for li, lv in enumerate(h.levels):
        last = li == len(h.levels) - 1
        out.append(SimpleNamespace(
            A_e=lv.A_e, nodal_aux=lv.nodal_aux, D=lv.D, Dt=O.canonical(lv.D.T),
            P_e=None if last else lv.P_e, R_e=None if last else O.canonical(lv.P_e.T),
            edge_sweeper=SimpleNamespace(dinv=lv.edge_sweeper.dinv,
                                         coefs=lv.edge_sweeper.coefficients()),
            aux_sweeper=SimpleNamespace(dinv=lv.aux_sweeper.dinv,
                                        coefs=lv.aux_sweeper.coefficients())))
    return out


def _problem():
    s = discretize_hex(6, 1.0, True)
    h = O.build_hierarchy(s.A_e, s.S, s.A_n, s.D, coarse_size=40, smoother="cheb")
    b = np.random.default_rng(0).uniform(-1, 1, s.A_e.shape[0])
    inv = np.linalg.inv(h.levels[-1].A_e.toarray())
    return h, b, inv


def _replicated(h, inv):
    def vcycle(level, b):
        return torch.from_numpy(_vc(h, inv, b.numpy(), level))
    return vcycle


def _worker(rank, world, port, out_path, agglomerate):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.set_num_threads(1)
    h, b, inv = _problem()
    dh = D.distribute(_levels(h), _replicated(h, inv), D.TorchComm(), ScipyOps(),
                      torch.device("cpu"), agglomerate=agglomerate)
    part = dh.levels[0].edge_part
    res = D.dist_pcg_solve(dh, torch.from_numpy(b[part.lo(rank):part.hi(rank)]).clone())
    xs = [None] * world
    dist.all_gather_object(xs, res.x.numpy())
    if rank == 0:
        with open(out_path, "wb") as f:
            pickle.dump(dict(x=np.concatenate(xs), its=res.iterations, status=res.status,
                             hist=res.residual_history, n_part=len(dh.levels)), f)
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_partition_and_halo_plan_sizes():
    p = D.Partition.balanced(10, 3)
    assert p.offsets.tolist() == [0, 3, 6, 10]
    assert p.owner(np.array([0, 2, 3, 5, 6, 9])).tolist() == [0, 0, 1, 1, 2, 2]
    plan = D.HaloPlan(4, 3, torch.zeros(0), [0, 2, 0, 5], [1, 0, 2, 0])
    assert plan.peers() == ([(1, 0, 2), (3, 2, 5)], [(0, 0, 1), (2, 1, 2)])


def test_halo_neighbours_of_a_slab_partition():
    """Contiguous row blocks of the edge operator are slabs: each rank's halo
    comes from its (at most two) neighbouring blocks, so the exchange is
    point-to-point with <= 2 peers. Virtual ranks (threads) on CPU."""
    h, b, inv = _problem()
    A = h.levels[0].A_e
    world = 4

    def fn(comm):
        part = D.Partition.balanced(A.shape[0], world)
        op = D.make_op(A, part, part, comm, torch.device("cpu"))
        x = torch.arange(part.lo(comm.rank), part.hi(comm.rank), dtype=torch.float64)
        xe = D.halo(op, ScipyOps(), x, comm)
        return [q for q, _ in op.recvs], xe.numpy().copy(), op.plan
    outs = D.run_virtual(world, fn)
    for r, (peers, xe, plan) in enumerate(outs):
        assert 0 < len(peers) <= 2 and all(abs(q - r) == 1 for q in peers)
        # halo values are the owners' entries: the global column ids here
        halo_vals = xe[plan.n_own:]
        assert np.all(np.diff(halo_vals) > 0)
        assert not np.any((halo_vals >= D.Partition.balanced(A.shape[0], world).lo(r)) &
                          (halo_vals < D.Partition.balanced(A.shape[0], world).hi(r)))


def test_virtual_ranks_solve_cpu():
    """The ThreadComm virtual ranks (the communicator of the single-GPU
    multi-rank tests) reproduce the gloo result on CPU."""
    h, b, inv = _problem()
    ref = O.pcg(h.levels[0].A_e, b, lambda r: _vc(h, inv, r))

    def fn(comm):
        dh = D.distribute(_levels(h), _replicated(h, inv), comm, ScipyOps(),
                          torch.device("cpu"), agglomerate=0)
        part = dh.levels[0].edge_part
        res = D.dist_pcg_solve(dh, torch.from_numpy(b[part.lo(comm.rank):part.hi(comm.rank)]))
        return res
    outs = D.run_virtual(3, fn)
    x = np.concatenate([o.x.numpy() for o in outs])
    assert all(o.iterations == outs[0].iterations for o in outs)
    assert abs(outs[0].iterations - ref.iterations) <= 1
    assert np.max(np.abs(x - ref.x)) <= 1e-8 * np.max(np.abs(ref.x))


@pytest.mark.parametrize("world,agglomerate", [(2, 0), (3, 0), (3, 10 ** 9)])
def test_distributed_solve_matches_single_process(world, agglomerate):
    """Partitioned levels with point-to-point neighbour halos; the levels
    below ``agglomerate`` edges run replicated after one all-gather
    (10**9: only level 0 is partitioned; 0: all but the coarsest)."""
    h, b, inv = _problem()
    # single-process reference: the same V-cycle with the dense coarse inverse
    ref = O.pcg(h.levels[0].A_e, b, lambda r: _vc(h, inv, r))
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "res.pkl")
        mp.spawn(_worker, args=(world, _free_port(), out, agglomerate), nprocs=world,
                 join=True)
        with open(out, "rb") as f:
            got = pickle.load(f)
    assert got["n_part"] == (len(h.levels) - 1 if agglomerate == 0 else 1)
    assert got["status"] == "converged"
    assert abs(got["its"] - ref.iterations) <= 1
    assert np.max(np.abs(got["x"] - ref.x)) <= 1e-8 * np.max(np.abs(ref.x))
    np.testing.assert_allclose(got["hist"][:len(ref.residual_history)],
                               ref.residual_history[:len(got["hist"])], rtol=1e-6)


def _vc(h, inv, b, level=0):
    lv = h.levels[level]
    if level == len(h.levels) - 1:
        return inv @ b
    x = O.hiptmair(lv, np.zeros(b.size), b)
    rc = lv.P_e.T @ (b - lv.A_e @ x)
    x = x + lv.P_e @ _vc(h, inv, rc, level + 1)
    return O.hiptmair(lv, x, b)
