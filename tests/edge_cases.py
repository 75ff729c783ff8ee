"""Degenerate but valid inputs, written once against the API names the
reference and this package share: zero right-hand side, a hierarchy that is
only its coarsest level, max_levels = 1 / 2, maxit = 0, a loose tolerance and
the smallest meshes. tests/golden/make_golden.py runs them on the unmodified
reference (tests/golden/edge_cases.json); the GPU test runs them on the device
package with the reference's smoother and compares.

``m.mg`` is the multigrid module, ``m.config(**kw)`` its SolverConfig with the
reference's Gauss-Seidel smoother, ``m.system(N, sigma, dirichlet)`` the hex
model problem."""

import numpy as np


def _rhs(n, seed=0):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def _solve(m, s, cfg, b=None, **kw):
    h = m.mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, cfg)
    A = h.levels[0].A_e
    n = A.shape[0]
    b = _rhs(n) if b is None else b
    r = m.mg.pcg_solve(A, b, m.mg.v_cycle_preconditioner(h), **kw)
    x = np.asarray(r.x)
    return {"n_levels": h.n_levels, "n_edges": [int(lv.A_e.shape[0]) for lv in h.levels],
            "operator_complexity": float(h.operator_complexity),
            "iterations": int(r.iterations), "status": r.status,
            "residual_history": [float(v) for v in r.residual_history],
            "precond_history": [float(v) for v in r.precond_history],
            "relative_residual": float(r.relative_residual),
            "x_norm": float(np.linalg.norm(x)), "x_size": int(x.size)}


CASES = {
    "zero_rhs": lambda m: _solve(m, m.system(4, 1.0, False), m.config(coarse_size=20),
                                 b=np.zeros(m.system(4, 1.0, False).A_e.shape[0])),
    "coarsest_only": lambda m: _solve(m, m.system(3, 1.0, True), m.config(coarse_size=200)),
    "max_levels_1": lambda m: _solve(m, m.system(4, 1.0, False),
                                     m.config(coarse_size=20, max_levels=1)),
    "max_levels_2": lambda m: _solve(m, m.system(8, 1.0, True),
                                     m.config(coarse_size=20, max_levels=2)),
    "maxit_0": lambda m: _solve(m, m.system(4, 1.0, False), m.config(coarse_size=20), maxit=0),
    "maxit_1": lambda m: _solve(m, m.system(4, 1.0, False), m.config(coarse_size=20), maxit=1),
    "loose_rtol": lambda m: _solve(m, m.system(6, 1.0, True), m.config(coarse_size=50),
                                   rtol=0.5),
    "smallest_mesh_natural": lambda m: _solve(m, m.system(2, 1.0, False),
                                              m.config(coarse_size=10)),
    "smallest_mesh_dirichlet": lambda m: _solve(m, m.system(2, 1.0, True),
                                                m.config(coarse_size=2)),
    "tiny_sigma": lambda m: _solve(m, m.system(4, 1e-8, True), m.config(coarse_size=20)),
    "large_sigma": lambda m: _solve(m, m.system(4, 1e6, False), m.config(coarse_size=20)),
}


def run(m, name):
    try:
        return CASES[name](m)
    except Exception as e:      # noqa: BLE001 -- an error is a result too
        return {"error": [type(e).__name__, str(e)]}
