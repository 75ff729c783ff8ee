"""Smoothed aggregation for the auxiliary nodal problem, on the B200.

Mirror of the reference's nodal_amg.py (same names and results). Every row is
bit-identical to the reference (SURVEY.md Hazard 1 / Appendix A): the
strength pattern, the power-method norms (Haswell-ddot order), the Jacobi-
smoothed prolongator and its row normalisation run as libsphcurl kernels with
explicit round-to-nearest arithmetic; the greedy aggregation is the host C++
pass of libsphcurl (sequential by definition).
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


@checked
def estimate_rho(A, dinv, iterations=10):
    """Ten-step power method on diag(1/d) A (nodal_amg.py:99-116). The norms
    run in the OpenBLAS-Haswell ddot order, so rho is bit-identical."""
    n = A.shape[0]
    v0 = _power_start(n)           # shared constant: never written
    v = dv.empty_f64(n)
    sq = dv.empty_f64(1)
    norms = dv.empty_f64(iterations + 1)
    call("sphc_hsw_dot", n, v0, v0, sq)
    call("sphc_scale_by_norm", n, v0, sq, v, norms[0:1])
    w = dv.empty_f64(n)
    for it in range(iterations):
        call("sphc_nodal_powmv", n, A.rowptr, A.col, A.val, dinv, v, w)
        call("sphc_hsw_dot", n, w, w, sq)
        call("sphc_scale_by_norm", n, w, sq, v, norms[it + 1:it + 2])
    h = dv.readback(norms)[0]
    rho = 1.0
    for it in range(iterations):
        if h[it + 1] == 0.0:
            return 0.0
        rho = float(h[it + 1])
    return rho


def _dinv(A):
    st = Status()
    d = dv.diagonal(A, st)

    def check(rows):
        if "ZERO_DIAG" in rows:
            raise ValueError("zero diagonal in nodal operator")
    st.defer(check)
    return dv.reciprocal(d)


@checked
def smooth_and_normalize(A_n, agg):
    """P = normalize((I - omega D^-1 A_n) P_tent), omega = 4 / (3 rho)
    (nodal_amg.py:138-155). ``agg`` replaces the reference's P_tent argument
    (the tentative prolongator is exactly the membership array)."""
    A = as_device_csr(A_n)
    n = A.shape[0]
    if n != agg.n_fine:
        raise ValueError(f"incompatible shapes {A.shape} and {(agg.n_fine, agg.n_agg)}")
    dinv = _dinv(A)
    rho = estimate_rho(A, dinv)
    omega = 4.0 / (3.0 * rho)
    st = Status()
    cnt = torch.empty(n, dtype=torch.int64, device=A.rowptr.device)
    call("sphc_nodal_smooth_count", n, A.rowptr, A.col, A.val, dinv, agg.membership, omega,
         cnt, st.t)
    prp, nnz = dv.scan(cnt)
    pci = torch.empty(nnz, dtype=torch.int32, device=A.rowptr.device)
    pv = dv.empty_f64(nnz)
    call("sphc_nodal_smooth_fill", n, A.rowptr, A.col, A.val, dinv, agg.membership, omega,
         prp, pci, pv, st.t)

    def check(rows):
        if "SPGEMM_CAPACITY" in rows:
            raise RuntimeError(f"nodal row {rows['SPGEMM_CAPACITY']} exceeds the kernel "
                               "capacity")
        if "ZERO_ROWSUM" in rows:
            raise ValueError(f"zero row sum before scaling in row {rows['ZERO_ROWSUM']}")
    st.defer(check)
    P = DeviceCSR(prp, pci, pv, (n, agg.n_agg))
    return NodalProlongator(P=P, omega_used=omega, rho_estimate=rho)
