"""Inputs on which the reference raises, written once against the API names the
reference and this package share, so the same callable runs
on both: tests/golden/make_golden.py executes it on the unmodified reference
and records (exception type, message) in tests/golden/error_inputs.json; the
GPU test executes it on the device package and compares.

``m`` is a namespace of modules (na = nodal_amg, cgm = coarse_gradient,
es = emin_setup, epm = edge_prolongator, mg = multigrid); ``s`` the 4^3-cell
hex system with natural BC, sigma = 1 (scipy CSR A_e, S, A_n, D)."""

import numpy as np
import scipy.sparse as sp


def _sp(X):
    return X.to_scipy() if hasattr(X, "to_scipy") else sp.csr_matrix(X)


def _with_entry(A, i, j, v):
    A = sp.lil_matrix(A)
    A[i, j] = v
    A = sp.csr_matrix(A)
    A.sort_indices()
    return A


def _nodal(m, s):
    agg = m.na.aggregate(m.na.strength_graph(s.A_n, 0.0))
    P_tent = m.na.tentative_prolongator(agg)
    nod = m.na.smooth_and_normalize(s.A_n, P_tent)
    return P_tent, nod


def _coarse(m, s):
    P_tent, nod = _nodal(m, s)
    Pc = m.cgm.gen_piecewise_const(nod.P, 2)
    cg = m.cgm.augment_dirichlet_edges(m.cgm.build_coarse_gradient(s.D, Pc), s.D, Pc)
    return nod, cg


def _gradient_three(m, s):
    nod, cg = _coarse(m, s)
    D = _sp(s.D)
    free = [c for c in range(D.shape[1]) if D[5, c] == 0][0]
    return m.es.setup_constraints(_with_entry(D, 5, free, 1.0), nod.P, cg)


def _gradient_empty_row(m, s):
    nod, cg = _coarse(m, s)
    D = sp.lil_matrix(_sp(s.D))
    D[7, :] = 0
    D = sp.csr_matrix(D)
    D.eliminate_zeros()
    return m.es.setup_constraints(D, nod.P, cg)


def _nullspace_fine(m, s):
    S = _sp(s.S).copy()
    S.data[S.indptr[3]] += 1.0          # row 3 no longer annihilates gradients
    return m.mg.build_hierarchy(s.A_e, S, s.A_n, s.D,
                                m.mg.SolverConfig(coarse_size=20))


def _zero_curl(m, s):
    S = _sp(s.S) * 0.0
    return m.mg.build_hierarchy(s.A_e, S, s.A_n, s.D, m.mg.SolverConfig(coarse_size=20))


def _edge_zero_diag(m, s):
    A = sp.lil_matrix(_sp(s.A_e))
    A[3, 3] = 0.0
    A = sp.csr_matrix(A)
    A.eliminate_zeros()
    return m.mg.build_hierarchy(A, s.S, s.A_n, s.D, m.mg.SolverConfig(coarse_size=20))


def _normalize_zero_rowsum(m, s):
    _, nod = _nodal(m, s)
    P = _sp(nod.P).copy()
    lo, hi = P.indptr[2], P.indptr[3]
    P.data[lo:hi] = 0.0
    P.data[lo] = 1.0
    if hi - lo > 1:
        P.data[lo + 1] = -1.0
    else:
        P.data[lo] = 0.0
    return m.na.normalize_rows(P)


def _smooth_shapes(m, s):
    P_tent, _ = _nodal(m, s)
    return m.na.smooth_and_normalize(s.A_n, _sp(P_tent)[:-1])


def _smooth_zero_diag(m, s):
    P_tent, _ = _nodal(m, s)
    A = sp.lil_matrix(_sp(s.A_n))
    A[4, 4] = 0.0
    A = sp.csr_matrix(A)
    A.eliminate_zeros()
    return m.na.smooth_and_normalize(A, P_tent)


def _pc_empty_row(m, s):
    _, nod = _nodal(m, s)
    P = sp.lil_matrix(_sp(nod.P))
    P[6, :] = 0
    P = sp.csr_matrix(P)
    P.eliminate_zeros()
    return m.cgm.gen_piecewise_const(P, 2)


def _pc_empty_column(m, s):
    _, nod = _nodal(m, s)
    P = sp.lil_matrix(_sp(nod.P))
    P[:, 1] = 0
    P = sp.csr_matrix(P)
    P.eliminate_zeros()
    return m.cgm.gen_piecewise_const(P, 2)


def _strength_diag(m, s):
    A = _with_entry(_sp(s.A_n), 7, 7, -1.0)
    return m.na.strength_graph(A, 0.0)


CASES = {
    "emin_cfg_omega": lambda m, s: m.epm.EminConfig(omega=2.0),
    "emin_cfg_omega_low": lambda m, s: m.epm.EminConfig(omega=0.0),
    "emin_cfg_iterations": lambda m, s: m.epm.EminConfig(iterations=-1),
    "emin_cfg_mode": lambda m, s: m.epm.EminConfig(mode="amg"),
    "strength_nonpositive_diagonal": _strength_diag,
    "gradient_row_of_three": _gradient_three,
    "gradient_empty_row": _gradient_empty_row,
    "nullspace_on_fine_level": _nullspace_fine,
    "zero_curl_curl": _zero_curl,
    "edge_operator_zero_diagonal": _edge_zero_diag,
    "normalize_zero_row_sum": _normalize_zero_rowsum,
    "smooth_incompatible_shapes": _smooth_shapes,
    "smooth_zero_diagonal": _smooth_zero_diag,
    "piecewise_const_empty_row": _pc_empty_row,
    "piecewise_const_empty_column": _pc_empty_column,
}


def run(m, s, name):
    """(type name, message) of the exception the case raises, or None."""
    try:
        CASES[name](m, s)
    except Exception as e:      # noqa: BLE001 -- the type is part of the result
        return [type(e).__name__, str(e)]
    return None
