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
from .device import DeviceCSR, Status, as_device_csr, call


@dataclass
class EminSetup:
    """Everything the energy minimisation needs (emin_setup.py:51-59)."""

    T: DeviceCSR            # fine edge x coarse node, values = R_dp on the pattern
    pattern: DeviceCSR      # prolongator pattern N; values = feasible guess
    cg: object              # CoarseGradient
    subproblem_dims: Counter
    rdp_scale: float
    n_augmented: int = 0


def _raise(st, D):
    rows = st.rows()
    if "MALFORMED_GRAD" in rows:
        b = rows["MALFORMED_GRAD"]
        rp = D.rowptr[b:b + 2].cpu().numpy()
        raise ValueError(f"malformed gradient: row {b} has {int(rp[1] - rp[0])} nonzeros")
    if "EMPTY_J" in rows:
        raise ValueError(f"fine edge {rows['EMPTY_J']} has an empty constraint "
                         "pattern (isolated edge or pattern bug)")
    if "EMIN_CAPACITY" in rows:
        raise RuntimeError(f"fine edge {rows['EMIN_CAPACITY']}: constraint block exceeds "
                           f"the device kernel capacity (|J| <= 16, |I| <= 64)")
    if "REDUCIBLE" in rows:
        # reference: make_irreducible (emin_setup.py:183-217); never fired on
        # any measured configuration and not ported.
        raise NotImplementedError(
            f"fine edge {rows['REDUCIBLE']}: reducible constraint block needs the "
            "make_irreducible repair, which the device path does not implement")
    if "RANK_LOW" in rows:
        raise ValueError(f"fine edge {rows['RANK_LOW']}: numerical rank below the "
                         "expected rank (topology bug)")


def setup_constraints(D_h, P_n, cg):
    """Pattern, irreducibility, factor checks and feasible guess for every
    fine edge (emin_setup.py:256-336 + edge_prolongator.py:104-126)."""
    D = as_device_csr(D_h)
    P = as_device_csr(P_n)
    n_e = D.shape[0]
    dev = D.rowptr.device
    st = Status()
    icount = torch.empty(n_e, dtype=torch.int64, device=dev)
    jcount = torch.empty(n_e, dtype=torch.int64, device=dev)
    rmax2 = torch.zeros(2, dtype=torch.float64, device=dev)
    dims = torch.zeros(65 * 17, dtype=torch.int64, device=dev)
    call("sphc_emin_count", n_e, D.rowptr, D.col, D.val, P.rowptr, P.col, P.val,
         cg.adj.rowptr, cg.adj.col, cg.n_interior, cg.single_id, icount, jcount, rmax2, dims,
         st.t)
    _raise(st, D)
    rm = rmax2.cpu().numpy()
    rdp_scale = max(1.0, float(rm[0]))
    if rm[1] > 1e-12 * rdp_scale:
        # reference: _empty_shell + make_irreducible (emin_setup.py:292-302)
        raise NotImplementedError(
            "a fine edge with an empty prolongator pattern has a nonzero commutator "
            "row; the make_irreducible repair is not implemented on the device path")
    trp, tnnz = dv.scan(jcount)
    erp, ennz = dv.scan(icount)
    tci = torch.empty(tnnz, dtype=torch.int32, device=dev)
    tv = torch.empty(tnnz, dtype=torch.float64, device=dev)
    eci = torch.empty(ennz, dtype=torch.int32, device=dev)
    ev = torch.empty(ennz, dtype=torch.float64, device=dev)
    call("sphc_emin_fill", n_e, D.rowptr, D.col, D.val, P.rowptr, P.col, P.val,
         cg.adj.rowptr, cg.adj.col, cg.n_interior, cg.single_id, trp, tci, tv, erp, eci, ev,
         st.t)
    _raise(st, D)
    h = dims.cpu().numpy().reshape(65, 17)
    nz = np.argwhere(h)
    counter = Counter({(int(i), int(j)): int(h[i, j]) for i, j in nz})
    return EminSetup(T=DeviceCSR(trp, tci, tv, (n_e, P.shape[1])),
                     pattern=DeviceCSR(erp, eci, ev, (n_e, cg.n_edges)),
                     cg=cg, subproblem_dims=counter, rdp_scale=rdp_scale)
