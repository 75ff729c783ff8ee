"""Per-edge commutator subproblems on the B200 (mirror of emin_setup.py).

The reference loops over fine edges in Python building a dense block, a
union-find irreducibility test and a Householder QR per row
(emin_setup.py:256-336; 87% of its setup time). Here two libsphcurl launches
(count, fill) do the whole pass, one warp per fine edge, and nothing per row
is stored except the pattern rows T (= J, with the commutator right-hand side
D_h P_n on it) and N (= I, the prolongator pattern) and the feasible guess;
the Gram-Cholesky factor is recomputed on chip where needed.
"""

from collections import Counter
from dataclasses import dataclass

import numpy as np
import torch

from . import device as dv
from .device import checked, DeviceCSR, Status, as_device_csr, call
from .trace import phase


@dataclass
class EminSetup:
    """Everything the energy minimisation needs (emin_setup.py:51-59)."""

    T: DeviceCSR            # fine edge x coarse node, values = R_dp on the pattern
    pattern: DeviceCSR      # prolongator pattern N; values = feasible guess
    cg: object              # CoarseGradient
    subproblem_dims: Counter
    rdp_scale: float
    n_augmented: int = 0
    over: torch.Tensor = None   # device count of rows in the wide capacity class

    @property
    def R_dp(self):
        """The commutator right-hand side D_h P_n (emin_setup.py:268): T's
        values (T's pattern also keeps the exactly-cancelled entries)."""
        return self.T


def _checker(D):
    """Deferred check of the emin kernels' status slots (Status.defer)."""
    def check(rows):
        if "MALFORMED_GRAD" in rows:
            b = rows["MALFORMED_GRAD"]
            rp = D.rowptr[b:b + 2].cpu().numpy()
            raise ValueError(f"malformed gradient: row {b} has {int(rp[1] - rp[0])} nonzeros")
        if "EMPTY_J" in rows:
            raise ValueError(f"fine edge {rows['EMPTY_J']} has an empty constraint "
                             "pattern (isolated edge or pattern bug)")
        if "EMIN_CAPACITY" in rows:
            raise RuntimeError(f"fine edge {rows['EMIN_CAPACITY']}: constraint block exceeds "
                               f"the device kernels' wide class (|J| <= 32, |I| <= 592)")
        if "REDUCIBLE" in rows:
            # only reachable if a block is still reducible after the repair pass
            raise RuntimeError(
                f"fine edge {rows['REDUCIBLE']}: constraint block reducible after the "
                "make_irreducible pass (internal error)")
        if "RANK_LOW" in rows:
            raise ValueError(f"fine edge {rows['RANK_LOW']}: numerical rank below the "
                             "expected rank (topology bug)")
    return check


# Capacity of the default (on-chip, 4 rows per CTA) class of the emin kernels:
# rows with |J| or |I| above it are re-run through the wide class (|J| <= 32).
# (0, 0) = the compiled capacity (16, 128); tests lower it to drive ordinary
# rows through the wide kernels.
DEFAULT_CLASS_CAPS = (0, 0)
_TABLE = (129, 17)      # SPHC_DIMS_I, SPHC_DIMS_J


def _raise(st, D):
    _checker(D)(st.rows())


def _view(t, lo):
    return None if t is None else t[lo:]


def _count(D, P, cg, xrp, xeid, flags, shard=None):
    n_e = D.shape[0]
    dev = D.rowptr.device
    st = Status()
    icount = torch.empty(n_e, dtype=torch.int64, device=dev)
    jcount = torch.empty(n_e, dtype=torch.int64, device=dev)
    rmax2 = torch.zeros(2, dtype=torch.float64, device=dev)
    dims = torch.zeros(129 * 17, dtype=torch.int64, device=dev)
    rowflag = torch.zeros(n_e, dtype=torch.uint8, device=dev) if flags else None
    rowmax = torch.empty(n_e, dtype=torch.float64, device=dev) if flags else None
    over = dv.zeros_i64(1)
    jcap, icap = DEFAULT_CLASS_CAPS
    for _, lo, hi in (shard.blocks(n_e) if shard else [(0, 0, n_e)]):
        call("sphc_emin_count", hi - lo, D.rowptr[lo:], D.col, D.val, P.rowptr, P.col, P.val,
             cg.adj.rowptr, cg.adj.col, cg.n_interior, cg.single_id, _view(xrp, lo), xeid,
             cg.ep_a, cg.ep_b, icount[lo:], jcount[lo:], rmax2, dims, _view(rowflag, lo),
             _view(rowmax, lo), jcap, icap, over, st.t)
    if shard is not None:
        b = shard.bounds(n_e)
        for t in (icount, jcount, rowflag, rowmax):
            if t is not None:
                shard.gather_ranges(t, b)
        shard.max_(rmax2)
        shard.sum_(dims)
        shard.sum_(over)
        shard.min_(st.t)
    return st, icount, jcount, rmax2, dims, rowflag, rowmax, over


def _fill(D, P, cg, icount, jcount, xrp, xeid, st, over, rowflag=None, shard=None):
    n_e = D.shape[0]
    dev = D.rowptr.device
    (trp, tnnz), (erp, ennz) = dv.scan_many(jcount, icount)
    tci = torch.empty(tnnz, dtype=torch.int32, device=dev)
    tv = torch.empty(tnnz, dtype=torch.float64, device=dev)
    eci = torch.empty(ennz, dtype=torch.int32, device=dev)
    ev = torch.empty(ennz, dtype=torch.float64, device=dev)
    jcap, icap = DEFAULT_CLASS_CAPS
    for _, lo, hi in (shard.blocks(n_e) if shard else [(0, 0, n_e)]):
        call("sphc_emin_fill", hi - lo, D.rowptr[lo:], D.col, D.val, P.rowptr, P.col, P.val,
             cg.adj.rowptr, cg.adj.col, cg.n_interior, cg.single_id, _view(xrp, lo), xeid,
             cg.ep_a, cg.ep_b, trp[lo:], tci, tv, erp[lo:], eci, ev, _view(rowflag, lo),
             jcap, icap, over, st.t)
    if shard is not None:
        b = shard.bounds(n_e)
        if shard.collective:
            from .sharding import host_offsets
            toff, eoff = host_offsets(trp, b), host_offsets(erp, b)
            for t in (tci, tv):
                shard.gather_ranges(t, toff)
            for t in (eci, ev):
                shard.gather_ranges(t, eoff)
        if rowflag is not None:
            shard.gather_ranges(rowflag, b)
        shard.min_(st.t)
    return (DeviceCSR(trp, tci, tv, (n_e, P.shape[1])),
            DeviceCSR(erp, eci, ev, (n_e, cg.n_edges)))


@checked
def setup_constraints(D_h, P_n, cg, shard=None):
    """Pattern, irreducibility, factor checks and feasible guess for every
    fine edge (emin_setup.py:256-336 + edge_prolongator.py:104-126).

    Rows whose constraint block is reducible, or whose pattern is empty while
    their commutator row is not, are flagged by the device pass and repaired
    on the host with the reference's make_irreducible semantics
    (``repair.make_irreducible_pass``); the coarse edges it appends are fed
    back to the device kernels as per-row extras."""
    D = as_device_csr(D_h)
    P = as_device_csr(P_n)
    n_e = D.shape[0]
    check = _checker(D)
    with phase("emin.count"):
        st, icount, jcount, rmax2, dims, rowflag, rowmax, over = _count(D, P, cg, None, None,
                                                                        True, shard)
    # the count pass's checks ride on the fill pass's scan readback
    st.defer(check)
    # the fill pass factors every block and flags the reducible ones
    with phase("emin.fill"):
        T, pattern = _fill(D, P, cg, icount, jcount, None, None, st, over, rowflag, shard)
    flags = rowflag
    # reducible rows, and empty-pattern rows whose commutator row exceeds
    # 1e-12 rdp_scale (rdp_scale = max(1, max|R_dp|)); decided on the device
    scale = torch.clamp(rmax2[0:1], min=1.0)
    need = (flags & 1).bool() | ((rmax2[1:2] > 1e-12 * scale)
                                 & (flags & 2).bool() & (rowmax > 1e-12 * scale))
    st.defer(check)
    rm, any_need, h, ov = dv.readback(rmax2, need.any(), dims, over)
    rdp_scale = max(1.0, float(rm[0]))
    n_aug = 0
    if bool(any_need[0]):
        from . import repair
        cg0 = cg
        with phase("emin.repair"):
            cg, xrp, xeid, n_aug, post = repair.make_irreducible_pass(
                need, flags, rowmax, rdp_scale, T, pattern, cg)
        with phase("emin.refill"):
            # the refill flags the post-pass rows that are still reducible
            # (instead of raising); the host repairs just those, then refills
            track = post is not None
            st, icount, jcount, rmax2, dims, rowflag, _, over = _count(D, P, cg, xrp, xeid,
                                                                       track, shard)
            st.defer(check)
            T, pattern = _fill(D, P, cg, icount, jcount, xrp, xeid, st, over,
                               rowflag=rowflag, shard=shard)
            st.defer(check)
            if track:
                red = torch.nonzero(rowflag & 1).flatten()    # (syncs: sized output)
                h, ov = dv.readback(dims, over)
                if red.numel():
                    with phase("emin.repair"):
                        cg, xrp, xeid, n_aug = repair.finish_post_pass(
                            post, red.cpu().numpy(), cg0, n_e)
                    st, icount, jcount, rmax2, dims, _, _, over = _count(D, P, cg, xrp, xeid,
                                                                         False, shard)
                    st.defer(check)
                    T, pattern = _fill(D, P, cg, icount, jcount, xrp, xeid, st, over,
                                       shard=shard)
                    st.defer(check)
                    h, ov = dv.readback(dims, over)
            else:
                h, ov = dv.readback(dims, over)
    h = h.reshape(*_TABLE)
    nz = np.argwhere(h)
    counter = Counter({(int(i), int(j)): int(h[i, j]) for i, j in nz})
    if int(ov[0]):
        # wide-class rows beyond the device histogram's table (rare: sized gather)
        big = torch.nonzero((icount >= _TABLE[0]) | (jcount >= _TABLE[1])).flatten()
        ij = torch.stack((icount[big], jcount[big]), 1).cpu().numpy()
        counter.update((int(i), int(j)) for i, j in ij if i > 0)
    return EminSetup(T=T, pattern=pattern, cg=cg, subproblem_dims=counter,
                     rdp_scale=rdp_scale, n_augmented=n_aug, over=over)
