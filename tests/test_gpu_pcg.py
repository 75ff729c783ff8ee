"""PCG exits on the device loop (WHILE-graph, multigrid.PcgLoop) and on the
host loop, against the reference's own non-converged results
(tests/golden/pcg_status.json, multigrid.py:244-264): maxit, stagnated
(rtol=0, x frozen at round-off; last history entry = true residual) and
indefinite (negated operator). Also the reference's preconditioner
contract: a numpy callable."""

import json
import os

import numpy as np
import pytest

from golden_util import GOLDEN

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")


def _golden():
    with open(os.path.join(GOLDEN, "pcg_status.json")) as f:
        meta = json.load(f)
    return meta, dict(np.load(os.path.join(GOLDEN, "pcg_status.npz")))


def _setup(g, smoother):
    from paper_2506_08284_b200 import multigrid as mg
    from paper_2506_08284_b200.inputs import discretize_hex
    s = discretize_hex(g["N"], 1.0, g["dirichlet"])
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D,
                           mg.SolverConfig(coarse_size=g["coarse_size"], smoother=smoother))
    b = np.random.default_rng(0).uniform(-1, 1, s.A_e.shape[0])
    return mg, s, h, b


def _neg(dv, A):
    return dv.DeviceCSR(A.rowptr, A.col, -A.val, A.shape)


@pytest.mark.parametrize("kind", ["maxit", "stagnated", "indefinite"])
@pytest.mark.parametrize("case", ["N4n", "N6d"])
def test_pcg_exit_gauss_seidel_vs_reference(case, kind):
    """Reference smoother (exact symmetric Gauss-Seidel): same status, the
    reference's iteration count (stagnation +-1: the frozen iterate depends
    on last-bit rounding), histories to 1e-6."""
    from paper_2506_08284_b200 import device as dv
    meta, arrays = _golden()
    g = meta[f"{case}_{kind}"]
    mg, s, h, b = _setup(g, "gauss_seidel")
    A = h.levels[0].A_e if kind != "indefinite" else _neg(dv, h.levels[0].A_e)
    kw = {"maxit": dict(maxit=3), "stagnated": dict(rtol=0.0), "indefinite": {}}[kind]
    r = mg.pcg_solve(A, b, mg.v_cycle_preconditioner(h), **kw)
    assert r.status == g["status"] == kind
    if kind == "stagnated":
        assert abs(r.iterations - g["iterations"]) <= 1
        assert r.residual_history[-1] <= 1e-11 * g["residual_history"][0]
        assert r.precond_history[-1] == r.precond_history[-2]
        return
    assert r.iterations == g["iterations"]
    np.testing.assert_allclose(r.residual_history, g["residual_history"], rtol=1e-6)
    np.testing.assert_allclose(r.precond_history, g["precond_history"], rtol=1e-6)
    x = arrays[f"{case}_{kind}_x"]
    assert np.max(np.abs(r.x - x)) <= 1e-6 * max(np.max(np.abs(x)), 1e-300)


@pytest.mark.parametrize("kind", ["maxit", "stagnated", "indefinite"])
def test_pcg_exit_chebyshev_vs_oracle(kind):
    """Performance smoother, graph loop vs host loop vs the oracle's PCG with
    the same Chebyshev sweeper: identical exits."""
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200 import device as dv
    meta, _ = _golden()
    g = meta[f"N6d_{kind}"]
    mg, s, h, b = _setup(g, "chebyshev")
    A = h.levels[0].A_e if kind != "indefinite" else _neg(dv, h.levels[0].A_e)
    kw = {"maxit": dict(maxit=3), "stagnated": dict(rtol=0.0), "indefinite": {}}[kind]
    r = mg.pcg_solve(A, b, mg.v_cycle_preconditioner(h), **kw)
    # host loop: the same preconditioner without graph capture
    M = mg.v_cycle_preconditioner(h)
    M.graph_safe = False
    rh = mg.pcg_solve(A, b, M, **kw)
    ho = O.build_hierarchy(s.A_e, s.S, s.A_n, s.D, coarse_size=g["coarse_size"],
                           smoother="cheb")
    Ao = ho.levels[0].A_e if kind != "indefinite" else -ho.levels[0].A_e
    ro = O.pcg(Ao, b, lambda v: O.v_cycle(ho, v), **kw)
    assert r.status == rh.status == ro.status == kind
    assert r.iterations == rh.iterations
    if kind == "stagnated":
        assert abs(r.iterations - ro.iterations) <= 2
    else:
        assert r.iterations == ro.iterations
        np.testing.assert_allclose(r.residual_history, ro.residual_history, rtol=1e-6)
    np.testing.assert_allclose(r.residual_history, rh.residual_history, rtol=1e-12)


def test_pcg_numpy_preconditioner():
    """A reference-style preconditioner (numpy in, numpy out) runs through
    the host loop: Jacobi on C1's edge operator, against the oracle."""
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200 import multigrid as mg
    from paper_2506_08284_b200.inputs import discretize_hex
    s = discretize_hex(8, 1.0, True)
    b = np.random.default_rng(1).uniform(-1, 1, s.A_e.shape[0])
    dinv = 1.0 / s.A_e.diagonal()

    def jacobi(r):
        assert isinstance(r, np.ndarray)
        return dinv * r
    r = mg.pcg_solve(s.A_e, b, jacobi, maxit=40)
    ro = O.pcg(s.A_e, b, jacobi, maxit=40)
    assert r.status == ro.status
    assert r.iterations == ro.iterations
    np.testing.assert_allclose(r.residual_history, ro.residual_history, rtol=1e-8)
    assert isinstance(r.x, np.ndarray)


def test_coarse_lu_matches_scipy_lu_solve():
    """SolverConfig(coarse_solver="lu"): the coarsest solve is the
    reference's partial-pivoting LU (multigrid.py:156-157,180-181); its
    action equals scipy's lu_solve of the same matrix to rounding, also on a
    nearly singular operator; on a well-conditioned hierarchy it solves like
    the default equilibrated Cholesky inverse."""
    import scipy.linalg as la
    from paper_2506_08284_b200 import multigrid as mg
    from paper_2506_08284_b200.inputs import discretize_hex
    s = discretize_hex(8, 1.0, True)
    b = np.random.default_rng(0).uniform(-1, 1, s.A_e.shape[0])
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D,
                           mg.SolverConfig(coarse_size=200, coarse_solver="lu"))
    Ac = h.levels[-1].A_e.to_scipy().toarray()
    rng = np.random.default_rng(1)
    v = rng.standard_normal(Ac.shape[0])
    got = h.coarse_factorization.cpu().numpy() @ v
    ref = la.lu_solve(la.lu_factor(Ac), v)
    assert np.max(np.abs(got - ref)) <= 1e-10 * np.max(np.abs(ref))
    # nearly singular SPD (cond ~ 1e13): same inverse action as LAPACK's LU
    Q, _ = np.linalg.qr(rng.standard_normal((60, 60)))
    M = (Q * np.logspace(0, -13, 60)) @ Q.T
    inv, _ = mg._coarse_lu_inverse(torch.from_numpy(M).cuda())
    ref = la.lu_solve(la.lu_factor(M), v[:60])
    got = inv.cpu().numpy() @ v[:60]
    assert np.max(np.abs(got - ref)) <= 1e-2 * np.max(np.abs(ref))
    r = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    rc = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(
        mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D,
                           mg.SolverConfig(coarse_size=200, coarse_solver="cholesky"))))
    assert r.status == rc.status == "converged" and abs(r.iterations - rc.iterations) <= 1


def test_coarse_inverse_breakdown_fallbacks():
    """The coarsest solve's fallbacks (multigrid._coarse_inverse_finish): a
    numerically singular SPD operator (the Galerkin operator of a
    rank-deficient prolongator) breaks the Cholesky factorisation (or leaves
    a round-off pivot) -> pseudo-inverse by eigendecomposition (small
    operators) or shifted factorisation (large ones: an explicit inverse with
    entries ~1 / shift, good to ~1e-3 on the range); a slightly indefinite
    one breaks the shifted factorisation too -> eigendecomposition. Every
    inverse must be symmetric positive semidefinite and solve A x = b for b
    in the range of A."""
    from paper_2506_08284_b200 import multigrid as mg
    rng = np.random.default_rng(7)
    n, r = 60, 52
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.concatenate([rng.uniform(1.0, 100.0, r), np.zeros(n - r)])
    A = (Q * lam) @ Q.T                             # rank 52 of 60: exactly semidefinite
    A = 0.5 * (A + A.T)
    for kind, Ad, tol, eigh_max in (("pseudo-inverse", A, 1e-9, 2048),
                                    ("shifted", A, 1e-2, 0),
                                    ("eigen after shifted", A - 1e-7 * np.abs(A).max()
                                     * np.eye(n), 1e-5, 0)):
        At = torch.from_numpy(Ad).cuda()
        inv, info, state = mg._coarse_inverse_start(At)
        assert int(info) != 0, kind                # a breakdown or a round-off pivot
        old = mg.COARSE_EIGH_MAX
        try:
            mg.COARSE_EIGH_MAX = eigh_max
            inv = mg._coarse_inverse_finish(inv, int(info), state)
        finally:
            mg.COARSE_EIGH_MAX = old
        assert torch.isfinite(inv).all(), kind
        assert float((inv - inv.T).abs().max()) == 0.0
        lo = float(torch.linalg.eigvalsh(inv)[0])
        assert lo > -1e-9 * float(inv.abs().max()), (kind, lo)     # positive semidefinite
        y = rng.standard_normal(n)
        b = A @ y                                  # in the range
        x = (inv @ torch.from_numpy(b).cuda()).cpu().numpy()
        res = np.linalg.norm(A @ x - b) / np.linalg.norm(b)
        assert res < tol, (kind, res)
