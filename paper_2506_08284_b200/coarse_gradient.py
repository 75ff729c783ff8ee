"""Coarse discrete gradients from nodal grid transfers, on the B200.

Mirror of the reference's coarse_gradient.py (same names and signatures:
``gen_piecewise_const(P) -> P_const``, ``build_coarse_gradient(D_h, P_const)``,
``augment_dirichlet_edges(cg, D_h, P_const)``, ``append_edge(cg, i, j)``).
Algorithm 1 runs on the device as cooperative fixed-point claiming passes
(csrc/pconst.cu), bit-identical to the reference's ordered loops; the coarse
edge set, the Dirichlet single-node edges and D_H are built by libsphcurl
kernels (bucket by lower aggregate, segmented sort, unique, scan). The
hierarchy itself uses the assignment-vector forms
(``piecewise_const_assignment``, ``coarse_gradient_from_assignment``): P_const
is exactly that vector.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import device as dv
from .device import checked, DeviceCSR, Status, as_device_csr, call


@dataclass
class CoarseGradient:
    """Coarse edge-to-node incidence plus its edge bookkeeping
    (coarse_gradient.py:19-33)."""

    D_H: DeviceCSR
    n_interior: int               # interior edges come first, sorted (a, b)
    n_single: int                 # then single-node edges, sorted by node
    adj: DeviceCSR                # upper adjacency: row a -> b's, edge id = position
    ep_a: torch.Tensor            # int32 [n_edges] tail node (-1 single-node)
    ep_b: torch.Tensor            # int32 [n_edges] head / single node
    single_id: torch.Tensor       # int32 [n_nodes] single-node edge id or -1
    augmented_edges: list = None

    @property
    def n_edges(self):
        return self.D_H.shape[0]

    @property
    def n_nodes(self):
        return self.D_H.shape[1]

    @property
    def edge_endpoints(self):
        a = self.ep_a.cpu().numpy()
        b = self.ep_b.cpu().numpy()
        return [(int(x), int(y)) if x >= 0 else (int(y),) for x, y in zip(a, b)]


def coarse_gradient_from_edges(pairs, singles, n_nodes):
    """CoarseGradient from explicit edge lists: interior pairs (a < b, sorted)
    then single-node edges (sorted) -- the layout build_coarse_gradient
    produces (used by tests that feed reference-side edge sets)."""
    pairs = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    singles = np.asarray(singles, dtype=np.int64)
    n_int, n_single = pairs.shape[0], singles.size
    dev = dv.device()
    adj_rp = np.zeros(n_nodes + 1, dtype=np.int64)
    np.add.at(adj_rp, pairs[:, 0] + 1, 1)
    adj_rp = np.cumsum(adj_rp)
    soff = np.zeros(n_nodes + 1, dtype=np.int64)
    soff[singles + 1] = 1
    soff = np.cumsum(soff)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)  # noqa: E731
    n_edges = n_int + n_single
    dh_rp = torch.empty(n_edges + 1, dtype=torch.int64, device=dev)
    dh_ci = torch.empty(2 * n_int + n_single, dtype=torch.int32, device=dev)
    dh_v = torch.empty(2 * n_int + n_single, dtype=torch.float64, device=dev)
    ep_a = torch.empty(n_edges, dtype=torch.int32, device=dev)
    ep_b = torch.empty(n_edges, dtype=torch.int32, device=dev)
    sid = torch.empty(n_nodes, dtype=torch.int32, device=dev)
    arp, acol, so = t(adj_rp, np.int64), t(pairs[:, 1], np.int32), t(soff, np.int64)
    call("sphc_build_coarse_gradient", n_nodes, n_int, arp, acol, so, n_single, dh_rp, dh_ci,
         dh_v, ep_a, ep_b, sid)
    return CoarseGradient(D_H=DeviceCSR(dh_rp, dh_ci, dh_v, (n_edges, n_nodes)),
                          n_interior=n_int, n_single=n_single,
                          adj=DeviceCSR(arp, acol, None, (n_nodes, n_nodes)),
                          ep_a=ep_a, ep_b=ep_b, single_id=sid, augmented_edges=[])


@checked
def gen_piecewise_const(P, n_passes=2):
    """Algorithm 1 (coarse_gradient.py:36-103): P_const, one unit entry per
    row at the column Algorithm 1 assigns it (a DeviceCSR)."""
    assign = piecewise_const_assignment(P, n_passes)
    n, m = P.shape
    dev = assign.device
    return DeviceCSR(torch.arange(n + 1, dtype=torch.int64, device=dev),
                     assign.to(torch.int32), torch.ones(n, dtype=torch.float64, device=dev),
                     (n, m))


def _assignment_of(P_const):
    """The assignment vector of a P_const matrix (one entry per row)."""
    P = as_device_csr(P_const)
    if P.nnz != P.shape[0]:
        raise ValueError("P_const must hold exactly one entry per row")
    return P.col.to(torch.int64), P.shape[1]


@checked
def piecewise_const_assignment(P, n_passes=2):
    """Algorithm 1 (coarse_gradient.py:36-103): the column assigned to every
    row (int64, device) -- P_const as a vector. Runs on the device
    (csrc/pconst.cu), bit-identical to the reference's ordered loops."""
    P = as_device_csr(P)
    m_h, m_H = P.shape
    dev = P.rowptr.device
    Pc = dv.transpose(P)
    st = Status()
    i64 = dict(dtype=torch.int64, device=dev)
    m = max(m_h, m_H) + 1
    target, counts = torch.empty(m_H, **i64), torch.empty(m_H, **i64)
    flags, pos, lst = torch.empty(m, **i64), torch.empty(m, **i64), torch.empty(m, **i64)
    srow = torch.empty(P.nnz, dtype=torch.int32, device=dev)
    owner = torch.empty(2 * m_h, dtype=torch.int32, device=dev)
    changed = torch.empty(2, dtype=torch.int32, device=dev)
    assign = torch.empty(m_h, **i64)
    call("sphc_piecewise_const", m_h, m_H, P.rowptr, P.col, P.val, Pc.rowptr, Pc.col, Pc.val,
         int(n_passes), target, counts, srow, owner, changed, flags, pos, lst, assign, st.t)

    def check(rows):
        if "PC_EMPTY_COLUMN" in rows:
            raise ValueError(f"empty column {rows['PC_EMPTY_COLUMN']} cannot be assigned "
                             "any row")
        if "PC_EMPTY_ROW" in rows:
            raise ValueError(f"row {rows['PC_EMPTY_ROW']} has no entries to assign")
        if "PC_NO_DONOR" in rows:
            raise ValueError(f"empty column {rows['PC_NO_DONOR']} cannot be assigned any row")
        if "PC_NO_FIXPOINT" in rows:
            raise RuntimeError("piecewise_const: claiming pass did not reach its fixed point")
    st.defer(check)
    return assign


def gen_piecewise_const_host(P, n_passes=2):
    """``piecewise_const_assignment`` computed by the sequential host C++
    loop (kept as a cross-check for the device version)."""
    P = as_device_csr(P)
    m_h, m_H = P.shape
    rp = P.rowptr.cpu().numpy()
    ci = P.col.cpu().numpy()
    v = P.val.cpu().numpy()
    assign = np.empty(m_h, dtype=np.int64)
    err = np.zeros(2, dtype=np.int64)
    rc = call("sphc_host_piecewise_const", m_h, m_H, rp, ci, v, int(n_passes), assign, err)
    if rc != 0:
        kind, idx = int(err[0]), int(err[1])
        if kind == 2:
            raise ValueError(f"row {idx} has no entries to assign")
        raise ValueError(f"empty column {idx} cannot be assigned any row")
    return torch.from_numpy(assign).to(P.rowptr.device)


@checked
def build_coarse_gradient(D_h, P_const):
    """Coarse edges from the projected node-graph Laplacian
    (coarse_gradient.py:106-120): one edge (i, j), i < j, per pair of
    aggregates joined by a fine edge with two free ends, sorted."""
    assign, n_agg = _assignment_of(P_const)
    return coarse_gradient_from_assignment(D_h, assign, n_agg, dirichlet=False)


@checked
def augment_dirichlet_edges(cg, D_h, P_const):
    """Append one single-node coarse edge per coarse node owning the free end
    of a one-entry fine gradient row (coarse_gradient.py:139-160). The edges
    already present are kept in place (build_coarse_gradient's output: they
    are recomputed identically on the device)."""
    assign, n_agg = _assignment_of(P_const)
    if cg.augmented_edges:
        raise NotImplementedError("augment_dirichlet_edges after append_edge: the device "
                                  "layout keeps single-node edges before appended ones")
    return coarse_gradient_from_assignment(D_h, assign, n_agg, dirichlet=True)


def append_edge(cg, i, j):
    """Append interior coarse edge (min, max), recorded as augmented
    (coarse_gradient.py:163-171); duplicates of an existing pair allowed."""
    i, j = int(min(i, j)), int(max(i, j))
    D = cg.D_H
    dev = D.rowptr.device
    rp = torch.cat([D.rowptr, (D.rowptr[-1:] + 2)])
    ci = torch.cat([D.col, torch.tensor([i, j], dtype=torch.int32, device=dev)])
    v = torch.cat([D.val, torch.tensor([-1.0, 1.0], dtype=torch.float64, device=dev)])
    return CoarseGradient(
        D_H=DeviceCSR(rp, ci, v, (D.shape[0] + 1, D.shape[1])),
        n_interior=cg.n_interior, n_single=cg.n_single, adj=cg.adj,
        ep_a=torch.cat([cg.ep_a, torch.tensor([i], dtype=torch.int32, device=dev)]),
        ep_b=torch.cat([cg.ep_b, torch.tensor([j], dtype=torch.int32, device=dev)]),
        single_id=cg.single_id, augmented_edges=list(cg.augmented_edges or []) + [(i, j)])


@checked
def coarse_gradient_from_assignment(D_h, assignment, n_agg, dirichlet=True):
    """Coarse edges from the projected node-graph Laplacian plus (dirichlet)
    the single-node edges (coarse_gradient.py:106-160, build_coarse_gradient
    followed by augment_dirichlet_edges), from the assignment vector."""
    D = as_device_csr(D_h)
    n_e = D.shape[0]
    dev = D.rowptr.device
    cnt = torch.zeros(n_agg, dtype=torch.int64, device=dev)
    call("sphc_coarse_pairs_count", n_e, D.rowptr, D.col, assignment, cnt)
    brp, nb = dv.scan(cnt)
    bcol = torch.empty(nb, dtype=torch.int32, device=dev)
    cursor = torch.zeros(n_agg, dtype=torch.int64, device=dev)
    call("sphc_coarse_pairs_fill", n_e, D.rowptr, D.col, assignment, brp, cursor, bcol)
    st = Status()
    call("sphc_csr_sort_rows", n_agg, brp, bcol, None, st.t)
    st.defer(dv.capacity_check)
    call("sphc_unique_count", n_agg, brp, bcol, cnt)
    flags = torch.zeros(n_agg, dtype=torch.int64, device=dev)
    if dirichlet:
        call("sphc_single_flags", n_e, D.rowptr, D.col, assignment, flags)
    (arp, n_int), (soff, n_single) = dv.scan_many(cnt, flags)
    acol = torch.empty(n_int, dtype=torch.int32, device=dev)
    call("sphc_unique_fill", n_agg, brp, bcol, arp, acol)
    n_edges = n_int + n_single
    dh_rp = torch.empty(n_edges + 1, dtype=torch.int64, device=dev)
    dh_ci = torch.empty(2 * n_int + n_single, dtype=torch.int32, device=dev)
    dh_v = torch.empty(2 * n_int + n_single, dtype=torch.float64, device=dev)
    ep_a = torch.empty(n_edges, dtype=torch.int32, device=dev)
    ep_b = torch.empty(n_edges, dtype=torch.int32, device=dev)
    sid = torch.empty(n_agg, dtype=torch.int32, device=dev)
    call("sphc_build_coarse_gradient", n_agg, n_int, arp, acol, soff, n_single, dh_rp, dh_ci,
         dh_v, ep_a, ep_b, sid)
    return CoarseGradient(D_H=DeviceCSR(dh_rp, dh_ci, dh_v, (n_edges, n_agg)),
                          n_interior=n_int, n_single=n_single,
                          adj=DeviceCSR(arp, acol, None, (n_agg, n_agg)),
                          ep_a=ep_a, ep_b=ep_b, single_id=sid, augmented_edges=[])
