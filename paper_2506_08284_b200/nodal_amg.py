"""Smoothed aggregation for the auxiliary nodal problem, on the B200.

Mirror of the reference's nodal_amg.py (same names, signatures and
results). Every row is bit-identical to the reference (SURVEY.md Hazard 1 /
Appendix A): the strength pattern, the power-method norms (Haswell-ddot
order), the Jacobi-smoothed prolongator and its row normalisation run as
libsphcurl kernels with explicit round-to-nearest arithmetic; the greedy
aggregation runs on the device as a distance-2 wavefront in index order
(csrc/aggregate.cu), bit-identical to the reference's sequential loops.
"""

from dataclasses import dataclass

import numpy as np
import torch

from . import device as dv
from .device import checked, DeviceCSR, Status, as_device_csr, call


@dataclass
class Aggregation:
    """Partition of fine nodes into aggregates (nodal_amg.py:17-23)."""

    n_fine: int
    n_agg: int
    membership: torch.Tensor     # int64 aggregate id per fine node (device)


@dataclass
class NodalProlongator:
    P: DeviceCSR
    omega_used: float
    rho_estimate: float


@checked
def strength_graph(A_n, drop_tol):
    """Symmetric strength pattern incl. the diagonal (nodal_amg.py:33-56)."""
    A = as_device_csr(A_n)
    n = A.shape[0]
    st = Status()
    d = dv.diagonal(A)
    cnt = torch.empty(n, dtype=torch.int64, device=A.rowptr.device)
    call("sphc_strength_count", n, A.rowptr, A.col, A.val, d, float(drop_tol), cnt, st.t)

    def check(rows):
        if "NONPOS_DIAG" in rows:
            raise ValueError(f"nonpositive diagonal entry in row {rows['NONPOS_DIAG']}")
    st.defer(check)
    frp, nnz = dv.scan(cnt)
    fci = torch.empty(nnz, dtype=torch.int32, device=A.rowptr.device)
    call("sphc_strength_fill", n, A.rowptr, A.col, A.val, d, float(drop_tol), frp, fci)
    F = DeviceCSR(frp, fci, None, A.shape)
    Ft = dv.transpose(F)
    call("sphc_pattern_union_count", n, F.rowptr, F.col, Ft.rowptr, Ft.col, cnt)
    srp, snnz = dv.scan(cnt)
    sci = torch.empty(snnz, dtype=torch.int32, device=A.rowptr.device)
    call("sphc_pattern_union_fill", n, F.rowptr, F.col, Ft.rowptr, Ft.col, srp, sci)
    return DeviceCSR(srp, sci, None, A.shape)


@checked
def aggregate(strength):
    """Greedy two-phase root aggregation (nodal_amg.py:59-88) on the device
    (csrc/aggregate.cu), bit-identical to the reference's ordered loops."""
    n = strength.shape[0]
    dev = strength.rowptr.device
    i64 = dict(dtype=torch.int64, device=dev)
    state = torch.empty(n, dtype=torch.int32, device=dev)
    ticket = torch.empty(1, dtype=torch.int32, device=dev)
    flags, pos, lst = (torch.empty(n + 1, **i64) for _ in range(3))
    memb = torch.empty(n, **i64)
    st = Status()
    call("sphc_aggregate", n, strength.rowptr, strength.col, state, ticket, flags, pos, lst,
         memb, st.t)

    def check(rows):
        if "AGG_CAPACITY" in rows:
            raise RuntimeError(f"node {rows['AGG_CAPACITY']}: more assigned neighbours than "
                               "the device aggregation buffer holds (256)")
    st.defer(check)
    n_agg = int(dv.readback(lst[n:n + 1])[0][0]) if n else 0
    return Aggregation(n_fine=n, n_agg=n_agg, membership=memb)


def aggregate_host(strength):
    """The same aggregation by the sequential host C++ loop (cross-check)."""
    n = strength.shape[0]
    rp = strength.rowptr.cpu().numpy()
    ci = strength.col.cpu().numpy()
    memb = np.empty(n, dtype=np.int64)
    n_agg = np.zeros(1, dtype=np.int64)
    call("sphc_host_aggregate", n, rp, ci, memb, n_agg)
    return Aggregation(n_fine=n, n_agg=int(n_agg[0]),
                       membership=torch.from_numpy(memb).to(strength.rowptr.device))


def tentative_prolongator(agg):
    """Piecewise-constant transfer, one unit entry per row at the node's
    aggregate (nodal_amg.py:91-96), built in place from the membership."""
    n = agg.n_fine
    dev = agg.membership.device
    rp = torch.arange(n + 1, dtype=torch.int64, device=dev)
    ci = agg.membership.to(torch.int32)
    v = torch.ones(n, dtype=torch.float64, device=dev)
    return DeviceCSR(rp, ci, v, (n, agg.n_agg))


_START = {}


def _power_start(n):
    # the reference's deterministic start vector, formed by numpy on the host
    # (nodal_amg.py:106; numpy's sin, bit for bit) and uploaded once per size
    # (a constant of n, kept like a lookup table; callers only read it)
    v = _START.get(n)
    if v is None:
        if len(_START) > 64:
            _START.clear()
        v = _START[n] = torch.from_numpy(
            1.0 + 0.01 * np.sin(np.arange(n, dtype=np.float64))).to(dv.device())
    return v


def _power_iterations(n, spmv, iterations):
    """The power method's loop (nodal_amg.py:104-116) with ``spmv(v, w)``
    computing w = A_scaled v; norms in the OpenBLAS-Haswell ddot order."""
    v0 = _power_start(n)           # shared constant: never written
    v = dv.empty_f64(n)
    sq = dv.empty_f64(1)
    norms = dv.empty_f64(iterations + 1)
    call("sphc_hsw_dot", n, v0, v0, sq)
    call("sphc_scale_by_norm", n, v0, sq, v, norms[0:1])
    w = dv.empty_f64(n)
    for it in range(iterations):
        spmv(v, w)
        call("sphc_hsw_dot", n, w, w, sq)
        call("sphc_scale_by_norm", n, w, sq, v, norms[it + 1:it + 2])
    h = dv.readback(norms)[0]
    rho = 1.0
    for it in range(iterations):
        if h[it + 1] == 0.0:
            return 0.0
        rho = float(h[it + 1])
    return rho


def _stored_order_csr(A):
    """A on the device with each row's entries in the caller's storage order
    (no canonical sort): scipy's csr_matvec sums in that order."""
    if isinstance(A, DeviceCSR):
        return A
    import scipy.sparse as sp
    A = A if sp.issparse(A) and A.format == "csr" else sp.csr_matrix(A)
    return DeviceCSR(dv.upload(A.indptr, np.int64), dv.upload(A.indices, np.int32),
                     dv.upload(A.data, np.float64), tuple(int(x) for x in A.shape))


@checked
def estimate_rho(A_scaled, iterations=10):
    """Power-method estimate of the spectral radius of a scaled operator
    (nodal_amg.py:99-116), same signature: the deterministic start vector
    1 + 0.01 sin(i), ``iterations`` steps, rho = the last norm (0.0 if a norm
    vanishes). Row sums in the matrix's storage order, norms in the
    OpenBLAS-Haswell ddot order: bit-identical to the reference."""
    A = _stored_order_csr(A_scaled)
    n = A.shape[0]
    return _power_iterations(
        n, lambda v, w: call("sphc_spmv_stored_order", n, A.rowptr, A.col, A.val, v, w),
        iterations)


def _estimate_rho_scaled(A, dinv, iterations=10):
    """estimate_rho(diags(dinv) @ A) without forming the scaled matrix: rows
    summed in DESCENDING column order, the storage scipy's ``diags @ A``
    produces (what smooth_and_normalize passes the reference's estimate_rho)."""
    n = A.shape[0]
    return _power_iterations(
        n, lambda v, w: call("sphc_nodal_powmv", n, A.rowptr, A.col, A.val, dinv, v, w),
        iterations)


def _dinv(A):
    st = Status()
    d = dv.diagonal(A, st)

    def check(rows):
        if "ZERO_DIAG" in rows:
            raise ValueError("zero diagonal in nodal operator")
    st.defer(check)
    return dv.reciprocal(d)


def _membership_of(P_tent):
    """(membership, n_agg) of a tentative prolongator: an Aggregation, or a
    matrix with exactly one unit entry per row (tentative_prolongator)."""
    if isinstance(P_tent, Aggregation):
        return P_tent.membership, P_tent.n_agg, P_tent.n_fine
    P = as_device_csr(P_tent)
    n, m = P.shape
    ok = P.nnz == n and bool(dv.readback(
        ((P.rowptr == torch.arange(n + 1, device=P.rowptr.device)).all()
         & (P.val == 1.0).all()).reshape(1))[0][0])
    if not ok:
        raise ValueError("smooth_and_normalize expects the tentative prolongator "
                         "(one unit entry per row)")
    return P.col.to(torch.int64), m, n


@checked
def smooth_and_normalize(A_n, P_tent):
    """P = normalize((I - omega D^-1 A_n) P_tent), omega = 4 / (3 rho)
    (nodal_amg.py:138-155), same signature: ``P_tent`` is the tentative
    prolongator (tentative_prolongator(agg)) or, equivalently, the
    Aggregation itself (no matrix needed: P_tent is the membership array)."""
    A = as_device_csr(A_n)
    memb, n_agg, n_fine = _membership_of(P_tent)
    n = A.shape[0]
    if A.shape[1] != n_fine:
        raise ValueError(f"incompatible shapes {A.shape} and {(n_fine, n_agg)}")
    dinv = _dinv(A)
    rho = _estimate_rho_scaled(A, dinv)
    omega = 4.0 / (3.0 * rho)
    st = Status()
    cnt = torch.empty(n, dtype=torch.int64, device=A.rowptr.device)
    call("sphc_nodal_smooth_count", n, A.rowptr, A.col, A.val, dinv, memb, omega, cnt, st.t)
    prp, nnz = dv.scan(cnt)
    pci = torch.empty(nnz, dtype=torch.int32, device=A.rowptr.device)
    pv = dv.empty_f64(nnz)
    call("sphc_nodal_smooth_fill", n, A.rowptr, A.col, A.val, dinv, memb, omega, prp, pci, pv,
         st.t)

    def check(rows):
        if "SPGEMM_CAPACITY" in rows:
            raise RuntimeError(f"nodal row {rows['SPGEMM_CAPACITY']} exceeds the kernel "
                               "capacity")
        if "ZERO_ROWSUM" in rows:
            raise ValueError(f"zero row sum before scaling in row {rows['ZERO_ROWSUM']}")
    st.defer(check)
    P = DeviceCSR(prp, pci, pv, (n, n_agg))
    return NodalProlongator(P=P, omega_used=omega, rho_estimate=rho)


@checked
def normalize_rows(P):
    """Scale every row to sum exactly one (nodal_amg.py:119-135): the row sum
    is numpy's ``np.add.reduceat`` (a_0 + pairwise(a_1..)), a vanishing sum
    (|s| <= 1e-13 max(1, sum |a|)) raises the reference's ValueError, values
    are fl(fl(1 / s) a) and exact zeros are dropped, as ``diags(1/s) @ P``
    does. Bit-identical to the reference."""
    P = as_device_csr(P)
    n = P.shape[0]
    st = Status()
    out = dv.empty_f64(P.nnz)
    call("sphc_normalize_rows", n, P.rowptr, P.val, out, st.t)

    def check(rows):
        if "SPGEMM_CAPACITY" in rows:
            raise RuntimeError(f"row {rows['SPGEMM_CAPACITY']} longer than the "
                               "normalize_rows kernel holds (257)")
        if "ZERO_ROWSUM" in rows:
            raise ValueError(f"zero row sum before scaling in row {rows['ZERO_ROWSUM']}")
    st.defer(check)
    return dv.drop_zeros(DeviceCSR(P.rowptr, P.col, out, P.shape))
