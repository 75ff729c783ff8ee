"""The paper's comparison modes on the B200 path vs the reference's goldens
(run with pytest -m gpu):

* RSAMG (EminConfig(mode="rsamg"), edge_prolongator.py:200-213): tentative
  nodal transfer, no emin sweeps. BIT: aggregates, P_n, piecewise-constant
  map, coarse edges, P_e pattern, level sizes. TOL: P_e and the coarse
  operators (1e-10 of max on the union pattern). The coarse PATTERNS keep or
  drop entries by exact cancellation of values that carry LAPACK QR
  round-off in the reference, so they are compared modulo entries of
  magnitude <= 1e-12 max (tests/golden_util.roundoff_pattern_diff).
  Iterations: within +-1 of the reference's sym-GS PCG with our
  Gauss-Seidel smoother, and of the oracle's Chebyshev PCG with ours.
* relaxation-only (fine_level + hiptmair_preconditioner,
  multigrid.py:198-207): iterations within +-1 of the reference (GS) and of
  the oracle (Chebyshev), residual history and solution close.
"""

import numpy as np
import pytest

from golden_util import (csr_hash, golden_csr, load_case, load_relax, rel_max_diff,
                         roundoff_pattern_diff, sha)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

RSAMG = ["R8d", "R12n", "R16d"]
RELAX = ["X8d", "X12n"]


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    from paper_2506_08284_b200.build import build_library
    build_library()


def _system(N, sigma, dirichlet):
    from paper_2506_08284_b200.inputs import discretize_hex
    return discretize_hex(N, sigma, dirichlet)


def _rsamg_cfg(meta, smoother="chebyshev"):
    from paper_2506_08284_b200 import multigrid as mg
    from paper_2506_08284_b200.edge_prolongator import EminConfig
    return mg.SolverConfig(coarse_size=meta["coarse_size"], emin=EminConfig(mode="rsamg"),
                           smoother=smoother)


@pytest.mark.parametrize("name", RSAMG)
def test_rsamg_hierarchy_vs_reference(name):
    from paper_2506_08284_b200 import multigrid as mg
    meta, arrays = load_case(name)
    assert meta["mode"] == "rsamg"
    s = _system(meta["N"], meta["sigma"], meta["dirichlet"])
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, _rsamg_cfg(meta))
    assert [lv.A_e.shape[0] for lv in h.levels] == meta["n_edges"]
    for li, (lv, L) in enumerate(zip(h.levels[:-1], meta["levels"])):
        assert csr_hash(lv.D.to_scipy()) == L["D"]
        assert sha(lv.membership.cpu().numpy().astype(np.int64)) == L["membership"]
        assert float(lv.omega).hex() == L["omega_hex"]
        assert float(lv.rho).hex() == L["rho_hex"]
        assert csr_hash(lv.P_n.to_scipy()) == L["P_n"]
        assert sha(lv.assignment.cpu().numpy().astype(np.int64)) == L["assignment"]
        P = lv.P_e.to_scipy()
        assert sha(P.indptr.astype(np.int64), P.indices.astype(np.int64)) == L["P_e_pattern"]
        dims = sorted([list(k) + [v] for k, v in lv.subproblem_dims.items()])
        assert dims == L["subproblem_dims"]
        assert rel_max_diff(P, golden_csr(arrays, f"L{li}_P_e", P.shape)) <= 1e-10
        assert lv.emin_energy == L["emin_energy"] == []
        assert lv.commutator_residual <= 1e-12
        nxt = h.levels[li + 1]
        for key, M in (("A_e", nxt.A_e), ("S_e", nxt.S_e)):
            Mg = M.to_scipy()
            G = golden_csr(arrays, f"L{li + 1}_{key}", Mg.shape)
            assert rel_max_diff(Mg, G) <= 1e-10, (li, key)
            _, mag = roundoff_pattern_diff(Mg, G)
            assert mag <= 1e-12, (li, key, mag)
        assert csr_hash(nxt.D.to_scipy()) == meta["levels"][li + 1]["D"]


@pytest.mark.parametrize("name", RSAMG)
def test_rsamg_solve_vs_reference(name):
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200 import multigrid as mg
    meta, arrays = load_case(name)
    s = _system(meta["N"], meta["sigma"], meta["dirichlet"])
    b = np.random.default_rng(meta["seed"]).uniform(-1, 1, s.A_e.shape[0])
    # the reference's own smoother
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, _rsamg_cfg(meta, "gauss_seidel"))
    res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    assert res.status == meta["gs"]["status"] == "converged"
    assert abs(res.iterations - meta["gs"]["iterations"]) <= 1
    xr = arrays["gs_x"]
    assert np.abs(res.x - xr).max() <= 1e-6 * np.abs(xr).max()
    # the performance smoother against the reference hierarchy with the same
    # polynomial in its sweeper seam
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, _rsamg_cfg(meta))
    res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    assert res.status == "converged"
    assert abs(res.iterations - meta["cheb"]["iterations"]) <= 1
    assert np.linalg.norm(b - s.A_e @ res.x) <= 1.5e-8 * np.linalg.norm(b)
    ho = O.build_hierarchy(s.A_e, s.S, s.A_n, s.D, coarse_size=meta["coarse_size"],
                           mode="rsamg", smoother="cheb")
    assert abs(res.iterations - O.solve(ho, b).iterations) <= 1


@pytest.mark.parametrize("name", RELAX)
def test_relaxation_only_vs_reference(name):
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200 import multigrid as mg
    meta, arrays = load_relax(name)
    s = _system(meta["N"], meta["sigma"], meta["dirichlet"])
    b = np.random.default_rng(meta["seed"]).uniform(-1, 1, s.A_e.shape[0])
    lv = mg.fine_level(s.A_e, s.S, s.D, mg.SolverConfig(smoother="gauss_seidel"))
    # D^T A D: TOL, pattern modulo exactly-cancelling round-off entries (the
    # reference stores 6565 at X8d, scipy's summation order leaves 55 more
    # 1e-16 residues than ours)
    aux_ref = O.fine_level(s.A_e, s.S, s.D).nodal_aux
    assert aux_ref.nnz == meta["nodal_aux_nnz"]
    aux = lv.nodal_aux.to_scipy()
    assert rel_max_diff(aux, aux_ref) <= 1e-10
    assert roundoff_pattern_diff(aux, aux_ref)[1] <= 1e-12
    res = mg.pcg_solve(lv.A_e, b, mg.hiptmair_preconditioner(lv))
    assert res.status == meta["status"]
    assert abs(res.iterations - meta["iterations"]) <= 1
    k = min(4, len(meta["residual_history"]))
    np.testing.assert_allclose(res.residual_history[:k], meta["residual_history"][:k],
                               rtol=1e-6)
    assert np.abs(res.x - arrays["x"]).max() <= 1e-6 * np.abs(arrays["x"]).max()
    # a second solve replays the captured iteration kept on the level
    res2 = mg.pcg_solve(lv.A_e, b, mg.hiptmair_preconditioner(lv))
    assert res2.iterations == res.iterations
    np.testing.assert_array_equal(res2.x, res.x)
    # Chebyshev-3 sweeps against the oracle's
    lv = mg.fine_level(s.A_e, s.S, s.D)
    res = mg.pcg_solve(lv.A_e, b, mg.hiptmair_preconditioner(lv))
    ro = O.relax_solve(O.fine_level(s.A_e, s.S, s.D, smoother="cheb"), b)
    assert res.status == ro.status == "converged"
    assert abs(res.iterations - ro.iterations) <= 1


def test_relaxation_only_slower_than_amg():
    """SPEC.md:660's ordering at desk scale (hex here): relaxation-only PCG
    needs at least twice the AMG-preconditioned iterations."""
    from paper_2506_08284_b200 import multigrid as mg
    s = _system(16, 1e-2, True)
    b = np.random.default_rng(1).uniform(-1, 1, s.A_e.shape[0])
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=1000))
    amg = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    lv = mg.fine_level(s.A_e, s.S, s.D)
    rel = mg.pcg_solve(lv.A_e, b, mg.hiptmair_preconditioner(lv))
    assert rel.iterations >= 2 * amg.iterations


def test_reuse_hierarchy_reprojects_new_operators():
    """Setup reuse (PAPER.md setup-cost remarks): transfers kept, operators
    re-projected. Every level equals scipy's P^T A P of the new operators
    through the kept P_e (TOL), null-space identity holds, and the solve
    converges close to a fresh setup's iteration count."""
    from golden_util import rel_max_diff
    from paper_2506_08284_b200 import multigrid as mg
    s1 = _system(12, 1e-2, True)
    s2 = _system(12, 1.0, True)              # same mesh, new sigma
    cfg = mg.SolverConfig(coarse_size=200)
    h = mg.build_hierarchy(s1.A_e, s1.S, s1.A_n, s1.D, cfg)
    h2 = mg.reuse_hierarchy(h, s2.A_e, s2.S, cfg)
    assert [lv.A_e.shape for lv in h2.levels] == [lv.A_e.shape for lv in h.levels]
    A, S = s2.A_e.tocsr(), s2.S.tocsr()
    for lv, lv2 in zip(h.levels[:-1], h2.levels[:-1]):
        assert lv2.P_e is lv.P_e and lv2.R_e is lv.R_e
        assert rel_max_diff(lv2.A_e.to_scipy(), A) <= 1e-10
        P = lv.P_e.to_scipy()
        A, S = (P.T @ A @ P).tocsr(), (P.T @ S @ P).tocsr()
    assert rel_max_diff(h2.levels[-1].A_e.to_scipy(), A) <= 1e-10
    assert rel_max_diff(h2.levels[-1].S_e.to_scipy(), S) <= 1e-10
    b = np.random.default_rng(1).uniform(-1, 1, s2.A_e.shape[0])
    r2 = mg.pcg_solve(h2.levels[0].A_e, b, mg.v_cycle_preconditioner(h2))
    fresh = mg.build_hierarchy(s2.A_e, s2.S, s2.A_n, s2.D, cfg)
    rf = mg.pcg_solve(fresh.levels[0].A_e, b, mg.v_cycle_preconditioner(fresh))
    assert r2.status == rf.status == "converged"
    assert r2.iterations <= rf.iterations + 5
    assert np.linalg.norm(b - s2.A_e @ r2.x) <= 1.5e-8 * np.linalg.norm(b)
    # the original hierarchy is untouched and still solves its own system
    r1 = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    assert r1.status == "converged"
    with pytest.raises(ValueError, match="do not match"):
        mg.reuse_hierarchy(h, _system(8, 1.0, True).A_e, _system(8, 1.0, True).S, cfg)


def test_matrix_market_import_feeds_the_device_path(tmp_path):
    """SPEC.md:618 import workflow: exported (A_e, S, A_n, D) -> MatrixMarket
    -> load_system -> build_hierarchy: the same hierarchy bit for bit as the
    in-memory inputs (C1 golden case), and the reference's iterations."""
    from paper_2506_08284_b200 import mmio, multigrid as mg
    meta, _ = load_case("C1")
    s = _system(meta["N"], meta["sigma"], meta["dirichlet"])
    paths = []
    for name in ("A_e", "S", "A_n", "D"):
        paths.append(str(tmp_path / f"{name}.mtx"))
        mmio.write_matrix_market(getattr(s, name), paths[-1])
    A_e, S, A_n, D = mmio.load_system(*paths)
    cfg = mg.SolverConfig(coarse_size=meta["coarse_size"])
    h = mg.build_hierarchy(A_e, S, A_n, D, cfg)
    assert [lv.A_e.shape[0] for lv in h.levels] == meta["n_edges"]
    assert [lv.A_e.nnz for lv in h.levels] == meta["nnz_A_e"]
    for lv, L in zip(h.levels[:-1], meta["levels"]):
        assert sha(lv.membership.cpu().numpy().astype(np.int64)) == L["membership"]
        assert csr_hash(lv.P_n.to_scipy()) == L["P_n"]
    b = np.random.default_rng(meta["seed"]).uniform(-1, 1, s.A_e.shape[0])
    res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    assert abs(res.iterations - meta["cheb"]["iterations"]) <= 1
