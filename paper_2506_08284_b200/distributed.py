"""Row-block partitioned PCG + Hiptmair V-cycle.

The solve shards by contiguous row blocks: edge ids follow the lexicographic
mesh order, so a block is a slab and its halo is about one node plane, owned
by at most two neighbouring ranks. Every level whose edge count is at least
``agglomerate`` is partitioned across the ranks of a communicator (one
process per GPU), with a halo plan per operator; the levels below it are
AGGLOMERATED: the restricted residual is all-gathered once and every rank
runs the rest of the V-cycle on its replicated copy of those levels (the
single-GPU kernels, no halos), keeping its own block of the correction. On
the partitioned levels:

* a halo exchange precedes every SpMV-type application: point-to-point
  sends / receives with the neighbours that actually share entries
  (``batch_isend_irecv``; NCCL over NVLink on B200 boxes), no group-wide
  collective; the local rows keep the global entry order, so every local
  SpMV row is bit-identical to the single-GPU row;
* PCG inner products are local partial sums + an all-reduce on the device
  scalar array (the only other data that crosses ranks).

The setup is replicated or row-block sharded (``sharding.py``): every rank
holds the whole hierarchy, partitioned here by views of its row blocks.

The collective layer is a communicator object:

* ``TorchComm(group)``: torch.distributed (NCCL on the GPU, gloo on CPU);
* ``ThreadComm``: W virtual ranks as W threads of one process, each with
  its own CUDA stream, exchanging through host-synchronised device copies
  (every transfer waits for the sender's stream on the host, then copies):
  the CUDA path with real, non-empty halos runs on ONE GPU without any
  kernel waiting on another rank's kernel (tests/test_gpu_distributed.py).

Local kernels come from an ops object: ``CudaOps`` (libsphcurl, the
product); the CPU gloo tests inject a scipy implementation of the same
calls to exercise the partitioning, plans and collectives without a GPU.
"""

import contextlib
import math
import os
import threading
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist

AGGLOMERATE_EDGES = int(os.environ.get("SPHC_AGGLOMERATE_EDGES", "250000"))


# ---------------------------------------------------------------------------
# communicators


class TorchComm:
    """torch.distributed process group (NCCL / gloo)."""

    def __init__(self, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def all_to_all(self, out, inp, out_splits, in_splits):
        """Setup only (halo plans): variable-size all-to-all."""
        dist.all_to_all_single(out, inp, list(out_splits), list(in_splits), group=self.group)

    def exchange(self, sends, recvs):
        """Point-to-point: sends = [(peer, tensor)], recvs = [(peer, tensor)];
        only the ranks that share halo entries talk to each other."""
        ops = [dist.P2POp(dist.isend, t, self._global(q), self.group) for q, t in sends]
        ops += [dist.P2POp(dist.irecv, t, self._global(q), self.group) for q, t in recvs]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def _global(self, q):
        return q if self.group is None else dist.get_global_rank(self.group, q)

    def all_reduce_(self, t):
        dist.all_reduce(t, group=self.group)

    def all_gather_(self, out, t):
        dist.all_gather_into_tensor(out, t, group=self.group)

    def replicated(self):
        return contextlib.nullcontext()


class VirtualWorld:
    """Shared state of W virtual ranks (ThreadComm)."""

    def __init__(self, world):
        self.world = int(world)
        self.barrier = threading.Barrier(self.world)
        self.slots = [None] * self.world
        self.lock = threading.Lock()


class ThreadComm:
    """Rank ``rank`` of a VirtualWorld: every transfer posts the sender's
    tensors after a host sync of its stream, waits at a barrier, copies on
    the receiver's stream, syncs, and waits again before buffers are
    reused. No device-side waiting between ranks."""

    def __init__(self, vw, rank):
        self.vw, self.rank, self.world = vw, int(rank), vw.world
        self.group = None

    def _sync(self):
        if torch.cuda.is_available():
            torch.cuda.current_stream().synchronize()

    def _post(self, obj):
        self._sync()
        self.vw.slots[self.rank] = obj
        self.vw.barrier.wait()

    def _done(self):
        self._sync()
        self.vw.barrier.wait()

    def all_to_all(self, out, inp, out_splits, in_splits):
        ioff = np.concatenate([[0], np.cumsum(in_splits)]).astype(np.int64)
        self._post((inp, ioff))
        o = 0
        for q in range(self.world):
            src, qoff = self.vw.slots[q]
            k = int(out_splits[q])
            if k:
                out[o:o + k].copy_(src[int(qoff[self.rank]):int(qoff[self.rank]) + k])
            o += k
        self._done()

    def exchange(self, sends, recvs):
        self._post({q: t for q, t in sends})
        for q, t in recvs:
            t.copy_(self.vw.slots[q][self.rank])
        self._done()

    def all_reduce_(self, t):
        self._post(t.clone())
        t.copy_(self.vw.slots[0])
        for q in range(1, self.world):
            t.add_(self.vw.slots[q])
        self._done()

    def all_gather_(self, out, t):
        self._post(t.clone())
        m = t.numel()
        for q in range(self.world):
            out[q * m:(q + 1) * m].copy_(self.vw.slots[q])
        self._done()

    @contextlib.contextmanager
    def replicated(self):
        """The agglomerated levels' buffers are shared by the virtual ranks
        of one process: one rank at a time."""
        with self.vw.lock:
            yield
            self._sync()


def run_virtual(world, fn, *args):
    """fn(comm, *args) on ``world`` virtual ranks (threads, one CUDA stream
    each); returns the per-rank results. Exceptions are re-raised."""
    vw = VirtualWorld(world)
    out, errs = [None] * world, []
    dev = torch.cuda.current_device() if torch.cuda.is_available() else None

    def body(r):
        try:
            if dev is not None:
                torch.cuda.set_device(dev)
                with torch.cuda.stream(torch.cuda.Stream()):
                    out[r] = fn(ThreadComm(vw, r), *args)
                    torch.cuda.current_stream().synchronize()
            else:
                out[r] = fn(ThreadComm(vw, r), *args)
        except BaseException as e:     # noqa: BLE001 - re-raised below
            errs.append(e)
            vw.barrier.abort()

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    real = [e for e in errs if not isinstance(e, threading.BrokenBarrierError)]
    if real or errs:
        raise (real or errs)[0]
    return out


# ---------------------------------------------------------------------------
# partitions and halo plans


@dataclass
class Partition:
    """Contiguous blocks of [0, n) over `world` ranks."""

    offsets: np.ndarray

    @staticmethod
    def balanced(n, world):
        return Partition(np.array([(n * r) // world for r in range(world + 1)], dtype=np.int64))

    @property
    def n(self):
        return int(self.offsets[-1])

    def lo(self, r):
        return int(self.offsets[r])

    def hi(self, r):
        return int(self.offsets[r + 1])

    def size(self, r):
        return self.hi(r) - self.lo(r)

    def owner(self, idx):
        return np.searchsorted(self.offsets, idx, side="right") - 1


@dataclass
class CSRLocal:
    """Owned rows of a distributed operator; columns index the extended
    vector [owned block of the column partition | halo]."""

    rowptr: torch.Tensor
    col: torch.Tensor
    val: torch.Tensor
    shape: tuple                 # (n_rows_owned, n_own_cols + n_halo)

    @property
    def nnz(self):
        return int(self.col.numel())

    def lanes(self):
        m = self.nnz / max(self.shape[0], 1)
        for L, lim in ((2, 3), (4, 6), (8, 14), (16, 40)):
            if m <= lim:
                return L
        return 32


@dataclass
class HaloPlan:
    n_own: int
    n_halo: int
    send_idx: torch.Tensor       # owned indices to send, grouped by destination rank
    send_counts: list
    recv_counts: list

    def peers(self):
        """[(peer, start, count)] of the sends and of the receives (halo
        entries are sorted, hence grouped by owner in rank order)."""
        def runs(counts):
            out, o = [], 0
            for q, k in enumerate(counts):
                if k:
                    out.append((q, o, int(k)))
                o += int(k)
            return out
        return runs(self.send_counts), runs(self.recv_counts)


def localize(rp, ci, val, row_lo, row_hi, col_part, comm, device):
    """Owned rows [row_lo, row_hi) of a global CSR (torch tensors on
    `device`: the GPU in the product, CPU under the gloo tests) ->
    (CSRLocal with remapped columns, HaloPlan). Collective over `comm`
    (every rank calls it for every operator). Everything stays on the
    device: the slice, the sorted halo set (unique of the off-block
    columns), the column remap (searchsorted) and the owner counts; the only
    host reads are the block's CSR bounds and the per-neighbour counts."""
    world, rank = comm.world, comm.rank
    bounds = rp[[row_lo, row_hi]].cpu().tolist()
    s, e = int(bounds[0]), int(bounds[1])
    lrp = (rp[row_lo:row_hi + 1] - s).to(torch.int64)
    cols = ci[s:e].to(torch.int64)
    lo, hi = col_part.lo(rank), col_part.hi(rank)
    own = (cols >= lo) & (cols < hi)
    halo_ids = torch.unique(cols[~own])                 # sorted
    n_own = hi - lo
    lcol = torch.where(own, cols - lo, n_own + torch.searchsorted(halo_ids, cols))
    offs = torch.as_tensor(col_part.offsets, dtype=torch.int64, device=cols.device)
    owners = torch.searchsorted(offs, halo_ids, right=True) - 1
    recv_counts = torch.bincount(owners, minlength=world).cpu().tolist()
    if world > 1:
        rc = torch.tensor(recv_counts, dtype=torch.int64, device=device)
        sc = torch.empty_like(rc)
        comm.all_to_all(sc, rc, [1] * world, [1] * world)
        send_counts = sc.cpu().tolist()
        got = torch.empty(int(sum(send_counts)), dtype=torch.int64, device=device)
        comm.all_to_all(got, halo_ids, send_counts, recv_counts)
    else:
        send_counts, got = [0], torch.empty(0, dtype=torch.int64, device=device)
    send_idx = (got - lo).to(torch.int64)
    A = CSRLocal(lrp, lcol.to(torch.int32), val[s:e].contiguous(),
                 (row_hi - row_lo, n_own + int(halo_ids.numel())))
    return A, HaloPlan(n_own, int(halo_ids.numel()), send_idx, send_counts, recv_counts)


@dataclass
class DistOp:
    A: CSRLocal
    plan: HaloPlan
    xbuf: torch.Tensor = None    # extended input [owned | halo]
    sbuf: torch.Tensor = None    # send staging
    sends: list = None           # [(peer, view of sbuf)]
    recvs: list = None           # [(peer, view of xbuf's halo part)]


def make_op(M, row_part, col_part, comm, device):
    """M: global operator (DeviceCSR / anything with rowptr, col, val
    tensors, or a scipy CSR), replicated on every rank."""
    if hasattr(M, "rowptr"):
        rp, ci, v = M.rowptr, M.col, M.val
    else:
        rp, ci, v = (torch.from_numpy(np.ascontiguousarray(a))
                     for a in (M.indptr.astype(np.int64), M.indices, M.data))
    rp, ci, v = (t.to(device) for t in (rp, ci, v))
    A, plan = localize(rp, ci, v, row_part.lo(comm.rank), row_part.hi(comm.rank), col_part,
                       comm, device)
    op = DistOp(A, plan)
    op.xbuf = torch.zeros(plan.n_own + plan.n_halo, dtype=torch.float64, device=device)
    op.sbuf = torch.empty(plan.send_idx.numel(), dtype=torch.float64, device=device)
    sp_, rp_ = plan.peers()
    op.sends = [(q, op.sbuf[o:o + k]) for q, o, k in sp_]
    op.recvs = [(q, op.xbuf[plan.n_own + o:plan.n_own + o + k]) for q, o, k in rp_]
    return op


def halo(op, ops, x_own, comm):
    """Extended input of op: [x_own | halo values from the owners]."""
    p = op.plan
    xb = op.xbuf
    if x_own is not None:
        ops.copy(xb[:p.n_own], x_own)
    if p.send_idx.numel():
        ops.gather(p.send_idx, xb, op.sbuf)
    if comm.world > 1:
        comm.exchange(op.sends, op.recvs)
    return xb


# ---------------------------------------------------------------------------
# local kernels of the product: libsphcurl on the rank's GPU


class CudaOps:
    """The local operations, on libsphcurl kernels."""

    def __init__(self):
        from . import device as dv
        from ._lib import call
        self.dv, self.call = dv, call

    def spmv(self, A, x, y, alpha=1.0, beta=0.0, z=None):
        # SELL mirror for the smoothed square operators (built in prepare)
        self.dv.spmv(A, x, y, alpha, beta, z)

    def cheb(self, A, dinv, b, x_ext, x_out, d, cd, cr, x_zero):
        m = self.dv.sell(A)      # SELL-32 mirror of the local rows (cached on A)
        if m.d16 is not None and not x_zero:
            # delta-coded columns (a lower neighbour's halo columns come first
            # in a row and sit above the owned ones: those rows restart from
            # a further 32-bit base, csrc/sell.cu)
            self.call("sphc_sell_cheb_step16", A.shape[0], m.slice_ptr, m.d16, m.c0, m.val,
                      dinv, b, x_ext, x_out, d, cd, cr, m.nbase)
            return
        self.call("sphc_sell_cheb_step", A.shape[0], m.slice_ptr, m.col, m.val, dinv, b,
                  None if x_zero else x_ext, x_out, d, cd, cr, int(x_zero), m.padded)

    def prepare(self, dl):
        """SELL-32 mirrors of the level's smoothed operators (csrc/sell.cu)."""
        self.dv.sell(dl.A.A)
        self.dv.sell(dl.aux.A)

    def dot(self, x, y, out):
        self.call("sphc_dot", x.numel(), x, y, out)

    def gather(self, idx, x, out):
        self.call("sphc_gather", idx.numel(), idx, x, out)

    def copy(self, dst, src):
        dst.copy_(src)

    def pcg_update(self, sc, p, Ap, x, r, flag):
        self.call("sphc_pcg_update", x.numel(), sc, p, Ap, x, r, flag)

    def pcg_direction(self, sc, z, p):
        self.call("sphc_pcg_direction", p.numel(), sc, z, p)

    def pcg_rotate(self, sc):
        self.call("sphc_pcg_rotate", sc)


# ---------------------------------------------------------------------------
# distributed hierarchy


@dataclass
class DistLevel:
    A: DistOp
    aux: DistOp
    D: DistOp
    Dt: DistOp
    P: DistOp = None
    R: DistOp = None
    dinv_A: torch.Tensor = None
    dinv_aux: torch.Tensor = None
    coefs_A: list = None
    coefs_aux: list = None
    edge_part: Partition = None
    node_part: Partition = None
    work: dict = field(default_factory=dict)


@dataclass
class DistHierarchy:
    levels: list                 # the partitioned levels
    n_levels: int                # of the whole hierarchy
    agg_part: Partition          # edge partition of the first agglomerated level
    replicated_vcycle: object    # (level, b_full) -> x_full on the replicated levels
    comm: object
    ops: object

    @property
    def rank(self):
        return self.comm.rank

    @property
    def world(self):
        return self.comm.world


def _own(t, part, rank):
    return t[part.lo(rank):part.hi(rank)].clone()


def distribute_hierarchy(h, comm=None, agglomerate=None):
    """Partition a product ``multigrid.Hierarchy`` (identical on every rank:
    replicated or sharded setup) over ``comm`` (default: the default
    torch.distributed group) for ``dist_pcg_solve``."""
    from . import multigrid as mg
    comm = comm or TorchComm()

    def vcycle(level, b):
        return mg.v_cycle(h, None, b, level)
    return distribute(h.levels, vcycle, comm, CudaOps(), agglomerate=agglomerate)


def distribute(levels, replicated_vcycle, comm, ops=None, device=None, agglomerate=None):
    """Partition a replicated hierarchy. ``levels``: objects with A_e,
    nodal_aux, D, Dt, P_e, R_e (global operators; P_e / R_e None on the
    coarsest) and edge / aux sweepers exposing dinv and coefs.
    ``replicated_vcycle(level, b_full)`` runs the V-cycle from ``level``
    down on the replicated levels. Levels with fewer than ``agglomerate``
    edges (and the coarsest) are agglomerated; level 0 is always
    partitioned."""
    ops = ops or CudaOps()
    agglomerate = AGGLOMERATE_EDGES if agglomerate is None else int(agglomerate)
    device = device or (torch.device("cuda", torch.cuda.current_device())
                        if isinstance(ops, CudaOps) else torch.device("cpu"))
    world, rank = comm.world, comm.rank
    n_part = 1
    while (n_part < len(levels) - 1 and levels[n_part].A_e.shape[0] >= agglomerate):
        n_part += 1
    parts = [Partition.balanced(lv.A_e.shape[0], world) for lv in levels[:n_part + 1]]
    out = []
    for li, lv in enumerate(levels[:n_part]):
        ep = parts[li]
        npart = Partition.balanced(lv.D.shape[1], world)
        if not hasattr(lv.edge_sweeper, "coefs"):
            raise ValueError("the partitioned solve needs the Chebyshev smoother "
                             "(Gauss-Seidel is sequential across rows)")
        cp = parts[li + 1]
        dl = DistLevel(A=make_op(lv.A_e, ep, ep, comm, device),
                       aux=make_op(lv.nodal_aux, npart, npart, comm, device),
                       D=make_op(lv.D, ep, npart, comm, device),
                       Dt=make_op(lv.Dt, npart, ep, comm, device),
                       P=make_op(lv.P_e, ep, cp, comm, device),
                       R=make_op(lv.R_e, cp, ep, comm, device),
                       edge_part=ep, node_part=npart)
        dl.dinv_A = _own(torch.as_tensor(lv.edge_sweeper.dinv).to(device), ep, rank)
        dl.dinv_aux = _own(torch.as_tensor(lv.aux_sweeper.dinv).to(device), npart, rank)
        dl.coefs_A = list(lv.edge_sweeper.coefs)
        dl.coefs_aux = list(lv.aux_sweeper.coefs)
        if hasattr(ops, "prepare"):
            ops.prepare(dl)
        ne, nn = ep.size(rank), npart.size(rank)
        z = lambda k: torch.zeros(k, dtype=torch.float64, device=device)  # noqa: E731
        dl.work = dict(x=[z(ne), z(ne)], d=z(ne), r=z(ne), bn=z(nn), c=[z(nn), z(nn)],
                       dn=z(nn), rc=z(cp.size(rank)))
        out.append(dl)
    ap = parts[n_part]
    m = max(ap.size(r) for r in range(world))
    z = lambda k: torch.zeros(k, dtype=torch.float64, device=device)  # noqa: E731
    dh = DistHierarchy(out, len(levels), ap, replicated_vcycle, comm, ops)
    dh.agg_work = dict(send=z(m), all=z(m * world), full=z(ap.n), out=z(ap.size(rank)))
    return dh


def _cheb(dh, op, dinv, coefs, b, x_own, bufs, d, x_zero):
    """Chebyshev polynomial with halo exchanges; returns the buffer holding x."""
    ops = dh.ops
    cur = x_own
    for step, (cd, cr) in enumerate(coefs):
        out = bufs[0] if cur is not bufs[0] else bufs[1]
        z = x_zero and step == 0
        xe = None if z else halo(op, ops, cur, dh.comm)
        ops.cheb(op.A, dinv, b, xe, out, d, cd, cr, z)
        cur = out
    return cur


def _hiptmair(dh, dl, x, b, x_zero):
    ops, c_ = dh.ops, dh.comm
    w = dl.work
    x = _cheb(dh, dl.A, dl.dinv_A, dl.coefs_A, b, x, w["x"], w["d"], x_zero)
    ops.spmv(dl.A.A, halo(dl.A, ops, x, c_), w["r"], -1.0, 1.0, b)
    ops.spmv(dl.Dt.A, halo(dl.Dt, ops, w["r"], c_), w["bn"])
    c = _cheb(dh, dl.aux, dl.dinv_aux, dl.coefs_aux, w["bn"], None, w["c"], w["dn"], True)
    ops.spmv(dl.D.A, halo(dl.D, ops, c, c_), x, 1.0, 1.0, x)
    return _cheb(dh, dl.A, dl.dinv_A, dl.coefs_A, b, x, w["x"], w["d"], False)


def _agglomerated(dh, b, level):
    """All-gather the restricted residual of the first agglomerated level,
    run the replicated V-cycle from there, keep the owned block."""
    part, comm, aw = dh.agg_part, dh.comm, dh.agg_work
    m = aw["send"].numel()
    dh.ops.copy(aw["send"][:b.numel()], b)
    comm.all_gather_(aw["all"], aw["send"])
    for r in range(comm.world):
        dh.ops.copy(aw["full"][part.lo(r):part.hi(r)], aw["all"][r * m:r * m + part.size(r)])
    with comm.replicated():
        y = dh.replicated_vcycle(level, aw["full"])
        dh.ops.copy(aw["out"], y[part.lo(comm.rank):part.hi(comm.rank)])
    return aw["out"]


def dist_v_cycle(dh, b, level=0):
    if level == len(dh.levels):
        return _agglomerated(dh, b, level)
    dl = dh.levels[level]
    ops, c_ = dh.ops, dh.comm
    x = _hiptmair(dh, dl, None, b, True)
    w = dl.work
    ops.spmv(dl.A.A, halo(dl.A, ops, x, c_), w["r"], -1.0, 1.0, b)
    ops.spmv(dl.R.A, halo(dl.R, ops, w["r"], c_), w["rc"])
    ec = dist_v_cycle(dh, w["rc"], level + 1)
    ops.spmv(dl.P.A, halo(dl.P, ops, ec, c_), x, 1.0, 1.0, x)
    return _hiptmair(dh, dl, x, b, False)


@dataclass
class DistPcgResult:
    x: torch.Tensor              # owned block of the solution
    iterations: int
    residual_history: list
    precond_history: list
    status: str
    relative_residual: float


def dist_pcg_solve(dh, b_own, rtol=1e-8, maxit=500):
    """PCG (multigrid.py:220-274 semantics) on the partitioned hierarchy."""
    ops, comm = dh.ops, dh.comm
    dl0 = dh.levels[0]
    dev = b_own.device
    n = b_own.numel()
    sc = torch.zeros(6, dtype=torch.float64, device=dev)
    flag = sc.view(torch.int32)[8:9]
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    r = b_own.clone()
    Ap = torch.empty_like(r)

    def allsum(lo, hi):
        comm.all_reduce_(sc[lo:hi])

    ops.dot(b_own, b_own, sc[1:2])
    allsum(1, 2)
    nb = math.sqrt(float(sc[1].item()))
    if nb == 0.0:
        return DistPcgResult(x, 0, [0.0], [0.0], "converged", 0.0)
    z = dist_v_cycle(dh, r)
    p = z.clone()
    ops.dot(r, z, sc[2:3])
    allsum(2, 3)
    rz0 = float(sc[2].item())
    hist, phist = [nb], [math.sqrt(max(rz0, 0.0))]
    status, its = "maxit", 0
    for k in range(maxit):
        # the whole iteration is queued without a host decision: alpha and
        # beta live in sc, the update is a no-op when p.Ap <= 0, and the
        # scalars of the tests come back in ONE readback per iteration
        ops.spmv(dl0.A.A, halo(dl0.A, ops, p, comm), Ap)
        ops.dot(p, Ap, sc[0:1])
        allsum(0, 1)
        sc[4] = 0.0
        ops.pcg_update(sc, p, Ap, x, r, flag)
        ops.dot(r, r, sc[1:2])
        # the stagnation flag is an OR over ranks: sum of 0/1 as doubles
        sc[5:6].copy_((flag != 0).to(torch.float64))
        allsum(1, 2)
        allsum(5, 6)
        z = dist_v_cycle(dh, r)
        ops.dot(r, z, sc[3:4])
        allsum(3, 4)
        # next direction queued speculatively (unused if this iteration ends)
        ops.pcg_direction(sc, z, p)
        ops.pcg_rotate(sc)
        h = sc.cpu().numpy()
        pAp = float(h[0])
        if pAp <= 0.0:
            status = "indefinite"
            break
        its = k + 1
        if float(h[5]) == 0.0:
            status = "stagnated"
            ops.spmv(dl0.A.A, halo(dl0.A, ops, x, comm), Ap, -1.0, 1.0, b_own)
            ops.dot(Ap, Ap, sc[0:1])
            allsum(0, 1)
            hist.append(math.sqrt(float(sc[0].item())))
            phist.append(phist[-1])
            break
        res = math.sqrt(float(h[1]))
        hist.append(res)
        phist.append(math.sqrt(max(float(h[3]), 0.0)))
        if res <= rtol * nb:
            status = "converged"
            break
    return DistPcgResult(x, its, hist, phist, status, hist[-1] / nb)
