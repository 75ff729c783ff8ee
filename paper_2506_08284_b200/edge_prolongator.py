"""Edge interpolation by constrained energy minimisation, on the B200.

Mirror of the reference's edge_prolongator.py (EminConfig, EdgeProlongator,
build_edge_prolongator). The projected damped-Jacobi sweep is one libsphcurl
launch per iteration: masked S P on the fixed pattern (warp per fine edge,
sequential ascending-k sums), Jacobi scaling, projection onto the null space
of the row's constraint block, update, the energy of the input iterate and
the commutator residual of the output -- fused.
"""

from collections import Counter
from dataclasses import dataclass, field

import torch

from . import coarse_gradient as cgrad
from . import device as dv
from . import emin_setup as es
from . import nodal_amg as na
from .device import checked, DeviceCSR, Status, as_device_csr, call
from .trace import phase


@dataclass
class EminConfig:
    """Knobs of the prolongator energy minimisation (edge_prolongator.py:28-44)."""

    omega: float = 0.5
    iterations: int = 1
    mode: str = "sphcurl"          # "sphcurl" or "rsamg" (the paper's baseline)
    n_passes: int = 2
    drop_tol: float = 0.0

    def __post_init__(self):
        if not 0.0 < self.omega < 2.0:
            raise ValueError(f"omega must be in (0, 2), got {self.omega}")
        if self.iterations < 0:
            raise ValueError("iterations must be >= 0")
        if self.mode not in ("sphcurl", "rsamg"):
            raise ValueError(f"unknown mode {self.mode!r}")


@dataclass
class EdgeProlongator:
    P_e: DeviceCSR
    energy_history: list
    commutator_residual: float
    subproblem_dims: Counter = field(default_factory=Counter)
    n_augmented: int = 0


@checked
def jacobi_diag_inverse(S):
    """1 / diag(S) with zeros replaced by 1e-12 max (edge_prolongator.py:159-167)."""
    d = dv.diagonal(S)
    # diag(S) >= 0 for the PSD curl-curl operator, so max d = max |d|
    top = dv.zeros_f64(1)
    if d.numel():
        dv.maxabs(d, top)
    sub = top * 1e-12
    # flag "all zero" in a status slot on the device (no host sync here)
    st = Status()
    k = dv.ST["ZERO_DIAG"]
    st.t[k:k + 1].masked_fill_(top <= 0.0, 0)

    def check(rows):
        if "ZERO_DIAG" in rows:
            raise ValueError("curl-curl diagonal is entirely zero")
    st.defer(check)
    return dv.reciprocal(d, sub)


@checked
def emin_sweeps(S, setup, omega, iterations, shard=None, final_energy=True):
    """Projected damped-Jacobi sweeps; returns (values, energies, residual).
    ``final_energy=False`` (build_hierarchy): the energy of the last iterate,
    trace(P^T S P), is left to the caller, who forms P^T S P anyway -- that
    saves the masked S P pass that only measures it (the last sweep already
    reports the commutator residual of its output).
    With ``shard`` every rank sweeps its block of fine edges and the value
    ranges are all-gathered after each sweep (the next sweep's masked S P
    reads neighbouring rows)."""
    S = as_device_csr(S)
    n_e = setup.pattern.shape[0]
    T, Pp, cg = setup.T, setup.pattern, setup.cg
    st = Status()
    e_row = dv.empty_f64(n_e)
    res = torch.zeros(1, dtype=torch.float64, device=e_row.device)
    esum = dv.empty_f64(iterations + 1)
    vals = Pp.val
    jcap, icap = es.DEFAULT_CLASS_CAPS
    over = setup.over if setup.over is not None else dv.zeros_i64(1)
    blocks = shard.blocks(n_e) if shard is not None else [(0, 0, n_e)]
    if shard is not None and shard.collective:
        from .sharding import host_offsets
        rbounds = shard.bounds(n_e)
        voff = host_offsets(Pp.rowptr, rbounds)

    def gather(v_out):
        if shard is not None and shard.collective:
            if v_out is not None:
                shard.gather_ranges(v_out, voff)
            shard.gather_ranges(e_row, rbounds)
            shard.max_(res)

    if iterations:
        dinv = jacobi_diag_inverse(S)
        for it in range(iterations):
            out = torch.empty_like(vals)
            res.zero_()
            for _, lo, hi in blocks:
                call("sphc_emin_step", lo, hi, S.rowptr, S.col, S.val, dinv, T.rowptr, T.col,
                     T.val, Pp.rowptr, Pp.col, vals, out, cg.ep_a, cg.ep_b, float(omega), 1,
                     e_row, res, jcap, icap, over, st.t)
            gather(out)
            dv.vsum(e_row, esum[it:it + 1])
            vals = out
    last = final_energy or not iterations
    if last:
        # energy of the final iterate and its commutator residual
        res.zero_()
        for _, lo, hi in blocks:
            call("sphc_emin_step", lo, hi, S.rowptr, S.col, S.val, None, T.rowptr, T.col,
                 T.val, Pp.rowptr, Pp.col, vals, None, cg.ep_a, cg.ep_b, float(omega), 0,
                 e_row, res, jcap, icap, over, st.t)
        gather(None)
        dv.vsum(e_row, esum[iterations:iterations + 1])
    if shard is not None:
        shard.min_(st.t)
    st.defer(es._checker(S))
    eh, rh = dv.readback(esum, res)
    energies = [float(x) for x in eh[:iterations + (1 if last else 0)]] if iterations else []
    return vals, energies, float(rh[0])


@checked
def build_edge_prolongator(A_n, A_e, S, D_h, cfg=None, shard=None, final_energy=True):
    """Edge prolongator and coarse gradient for one level
    (edge_prolongator.py:184-228). Returns
    (EdgeProlongator, CoarseGradient, NodalProlongator). ``shard`` (a
    sharding.Sharding) splits the emin rows over ranks; the nodal chain and
    the coarse topology stay replicated.

    cfg.mode == "rsamg" (edge_prolongator.py:200-213): the nodal transfer is
    the tentative prolongator itself (omega = rho = 0) and no emin sweeps
    run, so P_e is the feasible initial guess (entries +-1, 0 and the
    least-norm fractions of Dirichlet rows; many empty rows).

    ``final_energy=False``: energy_history lacks its last entry, the energy of
    the returned P_e, which equals trace(P_e^T S P_e) (see emin_sweeps)."""
    cfg = cfg or EminConfig()
    rsamg = cfg.mode == "rsamg"
    with phase("setup.strength"):
        strength = na.strength_graph(A_n, cfg.drop_tol)
    with phase("setup.aggregate"):
        agg = na.aggregate(strength)
    with phase("setup.smooth_and_normalize"):
        if rsamg:
            nod = na.NodalProlongator(P=na.tentative_prolongator(agg), omega_used=0.0,
                                      rho_estimate=0.0)
        else:
            nod = na.smooth_and_normalize(A_n, agg)
    with phase("setup.piecewise_const"):
        assign = cgrad.piecewise_const_assignment(nod.P, cfg.n_passes)
    with phase("setup.coarse_gradient"):
        cg = cgrad.coarse_gradient_from_assignment(D_h, assign, agg.n_agg)
    with phase("setup.emin_constraints"):
        setup = es.setup_constraints(D_h, nod.P, cg, shard=shard)
        cg = setup.cg                      # with any edges make_irreducible appended
    with phase("setup.emin_sweeps"):
        vals, energy, res = emin_sweeps(S, setup, cfg.omega, 0 if rsamg else cfg.iterations,
                                        shard=shard, final_energy=final_energy)
    P = setup.pattern
    P_e = DeviceCSR(P.rowptr, P.col, vals, P.shape)
    prol = EdgeProlongator(P_e=P_e, energy_history=energy, commutator_residual=res,
                           subproblem_dims=setup.subproblem_dims,
                           n_augmented=setup.n_augmented)
    prol.membership = agg.membership
    prol.assignment = assign
    return prol, cg, nod


# ---------------------------------------------------------------------------
# reference-signature pieces of Alg. 3 (edge_prolongator.py:104-181), over the
# same kernels build_edge_prolongator runs


def initial_feasible_guess(setup, structure=None):
    """All-ones seed corrected row by row to satisfy the commutator
    constraints (edge_prolongator.py:104-126). Returns (structure, values):
    the prolongator pattern (a value-less DeviceCSR) and the feasible guess,
    which the constraint pass already formed on the device (fused)."""
    P = setup.pattern
    if structure is None:
        structure = DeviceCSR(P.rowptr, P.col, None, P.shape)
    return structure, P.val.clone()


@checked
def emin_step(S, values, setup, structure, omega):
    """One projected damped-Jacobi sweep on the prolongator values
    (edge_prolongator.py:170-176): masked S P / diag(S) on the pattern,
    projection onto each row's constraint null space, values - omega dP.
    One fused launch (sphc_emin_step)."""
    S = as_device_csr(S)
    n_e = structure.shape[0]
    T, cg = setup.T, setup.cg
    st = Status()
    e_row = dv.empty_f64(n_e)
    res = torch.zeros(1, dtype=torch.float64, device=e_row.device)
    out = torch.empty_like(values)
    jcap, icap = es.DEFAULT_CLASS_CAPS
    over = setup.over if setup.over is not None else dv.zeros_i64(1)
    call("sphc_emin_step", 0, n_e, S.rowptr, S.col, S.val, jacobi_diag_inverse(S), T.rowptr,
         T.col, T.val, structure.rowptr, structure.col, values, out, cg.ep_a, cg.ep_b,
         float(omega), 1, e_row, res, jcap, icap, over, st.t)
    st.defer(es._checker(S))
    return out


@checked
def commutator_residual(P_e, D_H, R_dp):
    """max |P_e D_H - R_dp|, the feasibility defect (edge_prolongator.py:
    179-181): device SpGEMM, union-pattern difference, max reduction."""
    P, Dh, R = as_device_csr(P_e), as_device_csr(D_H), as_device_csr(R_dp)
    C = dv.spgemm(P, Dh, drop=False)
    if C.shape != R.shape:
        raise ValueError(f"shape mismatch: P_e D_H {C.shape} vs R_dp {R.shape}")
    Df = dv.csr_add(C, R, 1.0, -1.0)
    m = dv.zeros_f64(1)
    if Df.nnz:
        dv.maxabs(Df.val, m)
    return float(dv.readback(m)[0][0])
