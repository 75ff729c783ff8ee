"""Row-block partitioned PCG + Hiptmair V-cycle over torch.distributed.

SURVEY.md 8(e): the solve shards by contiguous row blocks (edge ids follow
the lexicographic mesh order, so a block is a slab and its halo is about one
node plane). This module partitions every level of a hierarchy across the
ranks of a process group (one process per GPU), builds per-operator halo
plans, and runs the same V-cycle / PCG as ``multigrid`` with

* halo exchange before every SpMV-type application (``all_to_all_single``
  with per-neighbour splits; NCCL over NVLink on B200 boxes), the local rows
  keeping the global entry order, so every local SpMV row is bit-identical to
  the single-GPU row;
* PCG inner products as local partial sums + ``all_reduce`` on the device
  scalar array (the only data that crosses ranks besides halos);
* the coarsest level replicated: ``all_gather`` of the restricted residual
  and the dense inverse applied redundantly.

The setup is replicated in round 1 (every rank builds the bit-identical
hierarchy on its own GPU). Local kernels come from an ops
object: ``CudaOps`` (libsphcurl, the product) -- the CPU gloo tests inject a
scipy implementation of the same six calls to exercise the partitioning,
halo plans and collectives without a GPU.
"""

import math
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist


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


def _exchange_counts(counts, group, device):
    t = torch.tensor(counts, dtype=torch.int64, device=device)
    out = torch.empty_like(t)
    dist.all_to_all_single(out, t, group=group)
    return out.cpu().tolist()


def localize(rp, ci, val, row_lo, row_hi, col_part, rank, group, device):
    """Owned rows [row_lo, row_hi) of a global CSR (torch tensors on
    `device`: the GPU in the product, CPU under the gloo tests) ->
    (CSRLocal with remapped columns, HaloPlan). Collective over `group`.
    Everything stays on the device: the slice, the sorted halo set
    (unique of the off-block columns), the column remap (searchsorted) and
    the owner counts; the only host reads are the block's CSR bounds and the
    per-neighbour counts."""
    world = col_part.offsets.size - 1
    bounds = rp[[row_lo, row_hi]].cpu().tolist()
    s, e = int(bounds[0]), int(bounds[1])
    lrp = (rp[row_lo:row_hi + 1] - s).to(torch.int64)
    cols = ci[s:e].to(torch.int64)
    lo, hi = col_part.lo(rank), col_part.hi(rank)
    own = (cols >= lo) & (cols < hi)
    halo = torch.unique(cols[~own])                     # sorted
    n_own = hi - lo
    lcol = torch.where(own, cols - lo, n_own + torch.searchsorted(halo, cols))
    offs = torch.as_tensor(col_part.offsets, dtype=torch.int64, device=cols.device)
    owners = torch.searchsorted(offs, halo, right=True) - 1
    recv_counts = torch.bincount(owners, minlength=world).cpu().tolist()
    if world > 1:
        send_counts = _exchange_counts(recv_counts, group, device)
        got = torch.empty(int(sum(send_counts)), dtype=torch.int64, device=device)
        dist.all_to_all_single(got, halo, send_counts, recv_counts, group=group)
    else:
        send_counts, got = [0], torch.empty(0, dtype=torch.int64, device=device)
    send_idx = (got - lo).to(torch.int64)
    A = CSRLocal(lrp, lcol.to(torch.int32), val[s:e].contiguous(),
                 (row_hi - row_lo, n_own + int(halo.numel())))
    return A, HaloPlan(n_own, int(halo.numel()), send_idx, send_counts, recv_counts)


@dataclass
class DistOp:
    A: CSRLocal
    plan: HaloPlan
    xbuf: torch.Tensor = None    # extended input [owned | halo]
    sbuf: torch.Tensor = None    # send staging


def make_op(M, row_part, col_part, rank, group, device):
    """M: global operator (DeviceCSR / anything with rowptr, col, val
    tensors, or a scipy CSR), replicated on every rank."""
    if hasattr(M, "rowptr"):
        rp, ci, v = M.rowptr, M.col, M.val
    else:
        rp, ci, v = (torch.from_numpy(np.ascontiguousarray(a))
                     for a in (M.indptr.astype(np.int64), M.indices, M.data))
    rp, ci, v = (t.to(device) for t in (rp, ci, v))
    A, plan = localize(rp, ci, v, row_part.lo(rank), row_part.hi(rank), col_part, rank,
                       group, device)
    op = DistOp(A, plan)
    op.xbuf = torch.zeros(plan.n_own + plan.n_halo, dtype=torch.float64, device=device)
    op.sbuf = torch.empty(plan.send_idx.numel(), dtype=torch.float64, device=device)
    return op


def halo(op, ops, x_own, group):
    """Extended input of op: [x_own | halo values from the owners]."""
    p = op.plan
    xb = op.xbuf
    if x_own is not None:
        ops.copy(xb[:p.n_own], x_own)
    if p.send_idx.numel():
        ops.gather(p.send_idx, xb, op.sbuf)
    if sum(p.send_counts) or p.n_halo:
        dist.all_to_all_single(xb[p.n_own:], op.sbuf, p.recv_counts, p.send_counts,
                               group=group)
    return xb


# ---------------------------------------------------------------------------
# local kernels of the product: libsphcurl on the rank's GPU


class CudaOps:
    """The six local operations, on libsphcurl kernels."""

    def __init__(self):
        from . import device as dv
        from ._lib import call
        self.dv, self.call = dv, call

    def spmv(self, A, x, y, alpha=1.0, beta=0.0, z=None):
        # SELL mirror for the smoothed square operators (built in cheb)
        self.dv.spmv(A, x, y, alpha, beta, z)

    def cheb(self, A, dinv, b, x_ext, x_out, d, cd, cr, x_zero):
        m = self.dv.sell(A)      # SELL-32 mirror of the local rows (cached on A)
        self.call("sphc_sell_cheb_step", A.shape[0], m.slice_ptr, m.col, m.val, dinv, b,
                  None if x_zero else x_ext, x_out, d, cd, cr, int(x_zero), m.padded)

    def prepare(self, dl):
        """SELL-32 mirrors of the level's smoothed operators (csrc/sell.cu)."""
        self.dv.sell(dl.A.A)
        self.dv.sell(dl.aux.A)

    def dot(self, x, y, out):
        self.call("sphc_dot", x.numel(), x, y, out)

    def gemv(self, M, x, y):
        self.call("sphc_dense_gemv", M.shape[0], M, x, y)

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
    levels: list
    coarse_inverse: torch.Tensor
    coarse_part: Partition
    rank: int
    world: int
    group: object
    ops: object


def _own(t, part, rank):
    return t[part.lo(rank):part.hi(rank)].clone()


def distribute_hierarchy(h, group=None):
    """Partition a product ``multigrid.Hierarchy`` (built identically on every
    rank) over the ranks of `group` for ``dist_pcg_solve``."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    return distribute(h.levels, h.coarse_factorization, rank, world, group, CudaOps())


def distribute(levels, coarse_inverse, rank, world, group=None, ops=None, device=None):
    """Partition a replicated hierarchy. `levels`: sequence of objects with
    A_e, nodal_aux, D, Dt, P_e, R_e (global operators; P_e/R_e None on the
    coarsest) and edge/aux sweepers exposing dinv and coefs."""
    ops = ops or CudaOps()
    device = device or (coarse_inverse.device if isinstance(coarse_inverse, torch.Tensor)
                        else torch.device("cpu"))
    out = []
    parts = [Partition.balanced(lv.A_e.shape[0], world) for lv in levels]
    nparts = [Partition.balanced(lv.D.shape[1], world) for lv in levels]
    for li, lv in enumerate(levels):
        ep, npart = parts[li], nparts[li]
        dl = DistLevel(A=make_op(lv.A_e, ep, ep, rank, group, device),
                       aux=make_op(lv.nodal_aux, npart, npart, rank, group, device),
                       D=make_op(lv.D, ep, npart, rank, group, device),
                       Dt=make_op(lv.Dt, npart, ep, rank, group, device),
                       edge_part=ep, node_part=npart)
        if li + 1 < len(levels):
            if not hasattr(lv.edge_sweeper, "coefs"):
                raise ValueError("the partitioned solve needs the Chebyshev smoother "
                                 "(Gauss-Seidel is sequential across rows)")
            cp = parts[li + 1]
            dl.P = make_op(lv.P_e, ep, cp, rank, group, device)
            dl.R = make_op(lv.R_e, cp, ep, rank, group, device)
            dl.dinv_A = _own(torch.as_tensor(lv.edge_sweeper.dinv).to(device), ep, rank)
            dl.dinv_aux = _own(torch.as_tensor(lv.aux_sweeper.dinv).to(device), npart, rank)
            dl.coefs_A = list(lv.edge_sweeper.coefs)
            dl.coefs_aux = list(lv.aux_sweeper.coefs)
        if hasattr(ops, "prepare"):
            ops.prepare(dl)
        ne, nn = ep.size(rank), npart.size(rank)
        z = lambda k: torch.zeros(k, dtype=torch.float64, device=device)  # noqa: E731
        dl.work = dict(x=[z(ne), z(ne)], d=z(ne), r=z(ne), bn=z(nn), c=[z(nn), z(nn)],
                       dn=z(nn), rc=z(parts[li + 1].size(rank)) if li + 1 < len(levels) else None)
        out.append(dl)
    inv = torch.as_tensor(coarse_inverse, dtype=torch.float64).to(device)
    return DistHierarchy(out, inv, parts[-1], rank, world, group, ops)


def _cheb(dh, op, dinv, coefs, b, x_own, bufs, d, x_zero):
    """Chebyshev polynomial with halo exchanges; returns the buffer holding x."""
    ops = dh.ops
    cur = x_own
    for step, (cd, cr) in enumerate(coefs):
        out = bufs[0] if cur is not bufs[0] else bufs[1]
        z = x_zero and step == 0
        xe = None if z else halo(op, ops, cur, dh.group)
        ops.cheb(op.A, dinv, b, xe, out, d, cd, cr, z)
        cur = out
    return cur


def _hiptmair(dh, dl, x, b, x_zero):
    ops, g = dh.ops, dh.group
    w = dl.work
    x = _cheb(dh, dl.A, dl.dinv_A, dl.coefs_A, b, x, w["x"], w["d"], x_zero)
    ops.spmv(dl.A.A, halo(dl.A, ops, x, g), w["r"], -1.0, 1.0, b)
    ops.spmv(dl.Dt.A, halo(dl.Dt, ops, w["r"], g), w["bn"])
    c = _cheb(dh, dl.aux, dl.dinv_aux, dl.coefs_aux, w["bn"], None, w["c"], w["dn"], True)
    ops.spmv(dl.D.A, halo(dl.D, ops, c, g), x, 1.0, 1.0, x)
    return _cheb(dh, dl.A, dl.dinv_A, dl.coefs_A, b, x, w["x"], w["d"], False)


def dist_v_cycle(dh, b, level=0):
    dl = dh.levels[level]
    ops, g = dh.ops, dh.group
    if level == len(dh.levels) - 1:
        part = dh.coarse_part
        m = max(part.size(r) for r in range(dh.world))
        send = torch.zeros(m, dtype=torch.float64, device=b.device)
        ops.copy(send[:b.numel()], b)
        allb = torch.empty(m * dh.world, dtype=torch.float64, device=b.device)
        dist.all_gather_into_tensor(allb, send, group=g)
        full = torch.cat([allb[r * m:r * m + part.size(r)] for r in range(dh.world)])
        y = torch.empty_like(full)
        ops.gemv(dh.coarse_inverse, full, y)
        out = dl.work["r"]
        ops.copy(out, y[part.lo(dh.rank):part.hi(dh.rank)])
        return out
    x = _hiptmair(dh, dl, None, b, True)
    w = dl.work
    ops.spmv(dl.A.A, halo(dl.A, ops, x, g), w["r"], -1.0, 1.0, b)
    ops.spmv(dl.R.A, halo(dl.R, ops, w["r"], g), w["rc"])
    ec = dist_v_cycle(dh, w["rc"], level + 1)
    ops.spmv(dl.P.A, halo(dl.P, ops, ec, g), x, 1.0, 1.0, x)
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
    ops, g = dh.ops, dh.group
    dl0 = dh.levels[0]
    dev = b_own.device
    n = b_own.numel()
    sc = torch.zeros(6, dtype=torch.float64, device=dev)
    flag = sc.view(torch.int32)[8:9]
    x = torch.zeros(n, dtype=torch.float64, device=dev)
    r = b_own.clone()
    Ap = torch.empty_like(r)

    def allsum(lo, hi):
        dist.all_reduce(sc[lo:hi], group=g)

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
        # scalars of the tests come back in ONE readback at the end (the
        # single-GPU path's scheme, multigrid.pcg_solve)
        ops.spmv(dl0.A.A, halo(dl0.A, ops, p, g), Ap)
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
            ops.spmv(dl0.A.A, halo(dl0.A, ops, x, g), Ap, -1.0, 1.0, b_own)
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
