"""CUDA path vs oracle / reference goldens (run on a B200: pytest -m gpu).

Parity classes: BIT for aggregates, omega/rho, P_n, the
piecewise-constant map, coarse edges, patterns and coarse counts; TOL (1e-10
relative to the matrix max) for P_e and coarse operators; commutator residual
<= 1e-12; PCG iterations within +-1 of the same-smoother oracle.
"""

import numpy as np
import pytest
import scipy.sparse as sp

from golden_util import (check_values, csr_hash, golden_csr, load_case, pattern_sha,
                         rel_max_diff, sha)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    from paper_2506_08284_b200.build import build_library
    build_library()


def _dev():
    from paper_2506_08284_b200 import device as dv
    return dv


def _rand_csr(n, m, density, seed, dtype=np.float64):
    rng = np.random.default_rng(seed)
    A = sp.random(n, m, density=density, random_state=rng, format="csr")
    A.data = rng.standard_normal(A.nnz) * np.exp(2 * rng.standard_normal(A.nnz))
    A.sum_duplicates()
    A.sort_indices()
    return A


def test_scan_and_reductions():
    dv = _dev()
    rng = np.random.default_rng(0)
    for n in (0, 1, 5, 2047, 2048, 2049, 5_000_001):
        c = rng.integers(0, 7, n).astype(np.int64)
        rp, tot = dv.scan(torch.from_numpy(c).cuda())
        ref = np.concatenate([[0], np.cumsum(c)])
        assert tot == ref[-1]
        assert np.array_equal(rp.cpu().numpy(), ref)
    x = rng.standard_normal(1_000_003)
    y = rng.standard_normal(x.size)
    xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    assert abs(dv.dot(xt, yt).item() - x @ y) <= 1e-12 * np.abs(x * y).sum()
    assert dv.maxabs(xt).item() == np.abs(x).max()
    assert abs(dv.vsum(xt).item() - x.sum()) <= 1e-12 * np.abs(x).sum()


def test_hsw_dot_bitwise():
    """Device Haswell-order ddot == oracle restatement (== pinned numpy)."""
    from oracle.hcurl_oracle import hsw_dot
    from paper_2506_08284_b200.device import call
    rng = np.random.default_rng(1)
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    for n in list(range(0, 40)) + [1000, 65537, 2_000_003]:
        x = rng.standard_normal(n) * np.exp(3 * rng.standard_normal(n))
        xt = torch.from_numpy(x).cuda()
        call("sphc_hsw_dot", n, xt, xt, out)
        assert out.item() == hsw_dot(x, x), n
    # two different vectors; tile boundaries of the TMA pipeline (1024-element
    # tiles, 4 stages); a source that is only 8-byte aligned takes the
    # plain-load variant of the kernel
    for n in (1023, 1024, 1040, 4096, 4097 + 16, 5 * 1024 + 7, 300_001):
        x = rng.standard_normal(n + 1)
        y = rng.standard_normal(n + 1) * np.exp(rng.standard_normal(n + 1))
        xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        call("sphc_hsw_dot", n, xt, yt, out)
        assert out.item() == hsw_dot(x[:n], y[:n]), n
        call("sphc_hsw_dot", n, xt[1:], yt[1:], out)          # misaligned by 8 bytes
        assert out.item() == hsw_dot(x[1:n + 1], y[1:n + 1]), n


@pytest.mark.parametrize("lanes", [1, 2, 4, 8, 16, 32])
def test_spmv(lanes):
    dv = _dev()
    A = _rand_csr(3000, 2000, 0.01, 2)
    x = np.random.default_rng(3).standard_normal(2000)
    z = np.random.default_rng(4).standard_normal(3000)
    Ad = dv.DeviceCSR.from_scipy(A)
    y = torch.empty(3000, dtype=torch.float64, device="cuda")
    dv.spmv(Ad, torch.from_numpy(x).cuda(), y, alpha=-1.0, beta=2.0,
            z=torch.from_numpy(z).cuda(), lanes=lanes)
    ref = -(A @ x) + 2.0 * z
    assert np.max(np.abs(y.cpu().numpy() - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_sell_spmv_and_cheb_match_csr():
    """SELL-32 mirror: same y as scipy; fused Chebyshev step same as CSR's."""
    dv = _dev()
    from paper_2506_08284_b200.device import call
    rng = np.random.default_rng(7)
    for n in (1, 31, 33, 1000, 4097):
        A = _rand_csr(n, n, min(1.0, 12.0 / n), 50 + n) + sp.eye(n)
        A = sp.csr_matrix(A)
        A.sort_indices()
        Ad = dv.DeviceCSR.from_scipy(A)
        x, z, dinv, b = (rng.standard_normal(n) for _ in range(4))
        X, Z, DI, B = (torch.from_numpy(v).cuda() for v in (x, z, dinv, b))
        m = dv.sell(Ad)
        assert m.padded >= A.nnz
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        dv.spmv(Ad, X, y, alpha=-1.0, beta=0.5, z=Z)
        ref = -(A @ x) + 0.5 * z
        assert np.max(np.abs(y.cpu().numpy() - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))
        d1 = torch.from_numpy(rng.standard_normal(n)).cuda()
        d2 = d1.clone()
        o1 = torch.empty_like(X)
        o2 = torch.empty_like(X)
        call("sphc_sell_cheb_step", n, m.slice_ptr, m.col, m.val, DI, B, X, o1, d1, 0.3, 0.7, 0,
             m.padded)
        call("sphc_cheb_step", n, Ad.rowptr, Ad.col, Ad.val, 8, DI, B, X, o2, d2, 0.3, 0.7, 0)
        assert torch.allclose(o1, o2, rtol=1e-13, atol=1e-13)
        assert torch.allclose(d1, d2, rtol=1e-13, atol=1e-13)


def test_spgemm_matches_scipy_bitwise():
    """Sequential ascending-k sums: identical bits to scipy's csr_matmat."""
    dv = _dev()
    for seed, (n, k, m, d1, d2) in enumerate([(500, 400, 300, 0.02, 0.03),
                                               (2000, 2000, 2000, 0.005, 0.005),
                                               (50, 3000, 40, 0.1, 0.05)]):
        A = _rand_csr(n, k, d1, 10 + seed)
        B = _rand_csr(k, m, d2, 20 + seed)
        C = dv.spgemm(dv.DeviceCSR.from_scipy(A), dv.DeviceCSR.from_scipy(B), ordered=True).to_scipy()
        ref = A @ B
        ref.sort_indices()
        assert np.array_equal(C.indptr, ref.indptr)
        assert np.array_equal(C.indices, ref.indices)
        assert np.array_equal(C.data.view(np.uint64), ref.data.view(np.uint64))


def test_spgemm_unordered_tol_and_deterministic():
    """All-lanes variant: same pattern, values within 1e-13, bitwise rerun."""
    dv = _dev()
    for seed, (n, k, m, d1, d2) in enumerate([(500, 400, 300, 0.02, 0.03),
                                               (300, 20000, 200, 0.05, 0.02),
                                               (3000, 3000, 3000, 0.003, 0.004)]):
        A = _rand_csr(n, k, d1, 30 + seed)
        B = _rand_csr(k, m, d2, 40 + seed)
        Ad, Bd = dv.DeviceCSR.from_scipy(A), dv.DeviceCSR.from_scipy(B)
        C1 = dv.spgemm(Ad, Bd).to_scipy()
        C2 = dv.spgemm(Ad, Bd).to_scipy()
        ref = A @ B
        ref.sort_indices()
        assert np.array_equal(C1.indptr, ref.indptr)
        assert np.array_equal(C1.indices, ref.indices)
        assert rel_max_diff(C1, ref) <= 1e-13
        assert np.array_equal(C1.data.view(np.uint64), C2.data.view(np.uint64))


def test_spgemm_long_rows_cta_kernel():
    """CTA-per-row kernels (A rows >= 64 entries on average: the R (A P)
    Galerkin shape): pattern identical to scipy, values TOL, bitwise rerun,
    pair = two single products, B rows longer than a warp, capacity flag."""
    dv = _dev()
    for seed, (n, k, m, d1, d2) in enumerate([(200, 5000, 150, 0.03, 0.02),
                                               (64, 3000, 250, 0.05, 0.05),   # B rows ~12
                                               (40, 2000, 256, 0.1, 0.2)]):   # B rows ~51
        A = _rand_csr(n, k, d1, 60 + seed)
        B = _rand_csr(k, m, d2, 70 + seed)
        A2, B2 = A.copy(), B.copy()
        A2.data = np.cos(A.data)
        B2.data = np.sin(B.data)
        Ad, Bd = dv.DeviceCSR.from_scipy(A), dv.DeviceCSR.from_scipy(B)
        assert dv._long_rows(Ad)
        C1 = dv.spgemm(Ad, Bd).to_scipy()
        C1b = dv.spgemm(Ad, Bd).to_scipy()
        ref = A @ B
        ref.sort_indices()
        assert np.array_equal(C1.indptr, ref.indptr)
        assert np.array_equal(C1.indices, ref.indices)
        assert rel_max_diff(C1, ref) <= 1e-13
        assert np.array_equal(C1.data.view(np.uint64), C1b.data.view(np.uint64))
        P1, P2 = dv.spgemm_pair(Ad, dv.DeviceCSR.from_scipy(A2), Bd,
                                dv.DeviceCSR.from_scipy(B2), drop=False)
        assert np.array_equal(P1.to_scipy().data.view(np.uint64), C1.data.view(np.uint64))
        ref2 = A2 @ B2
        ref2.sort_indices()
        assert rel_max_diff(P2.to_scipy(), ref2) <= 1e-13
    # more than 256 distinct columns in a row: beyond the on-chip hash, the
    # global-memory row path takes over (tests/test_gpu_capacity.py)
    A = _rand_csr(8, 400, 0.5, 80)
    B = _rand_csr(400, 2000, 0.05, 81)
    C = dv.spgemm(dv.DeviceCSR.from_scipy(A), dv.DeviceCSR.from_scipy(B)).to_scipy()
    ref = A @ B
    ref.sort_indices()
    assert np.array_equal(C.indptr, ref.indptr)
    assert np.array_equal(C.indices, ref.indices)
    assert rel_max_diff(C, ref) <= 1e-13


def test_transpose():
    dv = _dev()
    A = _rand_csr(4000, 700, 0.01, 5)
    T = dv.transpose(dv.DeviceCSR.from_scipy(A)).to_scipy()
    ref = sp.csr_matrix(A.T)
    ref.sort_indices()
    assert np.array_equal(T.indptr, ref.indptr)
    assert np.array_equal(T.indices, ref.indices)
    assert np.array_equal(T.data, ref.data)


# ---------------------------------------------------------------------------
# per-level parity against the oracle


def _system(N, sigma, dirichlet):
    from paper_2506_08284_b200.inputs import discretize_hex
    return discretize_hex(N, sigma, dirichlet)


@pytest.mark.parametrize("N,sigma,dirichlet", [(4, 1.0, False), (6, 1.0, True),
                                               (10, 1e-4, False), (16, 1.0, True)])
def test_nodal_chain_and_topology_bitwise(N, sigma, dirichlet):
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200 import coarse_gradient as cg
    from paper_2506_08284_b200 import nodal_amg as na
    s = _system(N, sigma, dirichlet)
    Sg = na.strength_graph(s.A_n, 0.0).to_scipy()
    So = O.strength_pattern(s.A_n)
    assert np.array_equal(Sg.indptr, So.indptr) and np.array_equal(Sg.indices, So.indices)
    agg = na.aggregate(na.strength_graph(s.A_n, 0.0))
    memb_o, nagg_o = O.aggregate(So)
    assert agg.n_agg == nagg_o
    assert np.array_equal(agg.membership.cpu().numpy(), memb_o)
    nod = na.smooth_and_normalize(s.A_n, agg)
    Po, wo, ro = O.smoothed_prolongator(s.A_n, memb_o, nagg_o)
    assert nod.rho_estimate == ro and nod.omega_used == wo
    assert csr_hash(nod.P.to_scipy()) == csr_hash(Po)
    assign = cg.piecewise_const_assignment(nod.P, 2).cpu().numpy()
    assert np.array_equal(assign, O.piecewise_const(Po, 2))
    cgd = cg.coarse_gradient_from_assignment(s.D, torch.from_numpy(assign).cuda(), nagg_o)
    ceo = O.coarse_edges(s.D, assign, nagg_o)
    assert cgd.n_interior == ceo.pairs.shape[0] and cgd.n_single == ceo.singles.size
    DH = cgd.D_H.to_scipy()
    assert csr_hash(DH) == csr_hash(ceo.D_H())


@pytest.mark.parametrize("N,sigma,dirichlet", [(4, 1.0, False), (6, 1.0, True),
                                               (10, 1e-4, False), (16, 1.0, True)])
def test_edge_prolongator_vs_oracle(N, sigma, dirichlet):
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200 import edge_prolongator as ep
    s = _system(N, sigma, dirichlet)
    prol, cgd, nod = ep.build_edge_prolongator(s.A_n, s.A_e, s.S, s.D)
    memb, nagg = O.aggregate(O.strength_pattern(s.A_n))
    Po, _, _ = O.smoothed_prolongator(s.A_n, memb, nagg)
    ce = O.coarse_edges(s.D, O.piecewise_const(Po, 2), nagg)
    em = O.emin_prolongator(s.D, Po, ce, s.S)
    P = prol.P_e.to_scipy()
    # STRUCT
    assert np.array_equal(P.indptr, em.P_e.indptr)
    assert np.array_equal(P.indices, em.P_e.indices)
    assert dict(prol.subproblem_dims) == dict(em.subproblem_dims)
    # TOL
    assert rel_max_diff(P, em.P_e) <= 1e-10
    assert np.allclose(prol.energy_history, em.energy_history, rtol=1e-10, atol=0)
    assert prol.commutator_residual <= 1e-12


def test_make_irreducible_repair_vs_reference():
    """Reducible constraint blocks (a reduced coarse gradient) are repaired with
    the reference's make_irreducible semantics: same appended coarse edges,
    same prolongator pattern, same feasible guess (golden from the reference's
    own setup_constraints, tests/golden/make_golden.py repair_case)."""
    import json
    import os
    from golden_util import GOLDEN
    from paper_2506_08284_b200 import coarse_gradient as cg_mod
    from paper_2506_08284_b200 import emin_setup as es
    from paper_2506_08284_b200 import nodal_amg as na
    with open(os.path.join(GOLDEN, "repair_N10d.json")) as f:
        meta = json.load(f)
    arr = dict(np.load(os.path.join(GOLDEN, "repair_N10d.npz")))
    s = _system(10, 1.0, True)
    agg = na.aggregate(na.strength_graph(s.A_n, 0.0))
    nod = na.smooth_and_normalize(s.A_n, agg)
    cg = cg_mod.coarse_gradient_from_edges(arr["pairs"], arr["singles"], meta["n_nodes"])
    setup = es.setup_constraints(s.D, nod.P, cg)
    assert setup.n_augmented == meta["n_augmented"]
    aug = [list(e) for e in setup.cg.augmented_edges]
    assert aug == meta["augmented"]
    P = setup.pattern.to_scipy()
    assert np.array_equal(P.indptr, arr["P_indptr"])
    assert np.array_equal(P.indices, arr["P_indices"])
    ref = sp.csr_matrix((arr["P_data"], arr["P_indices"], arr["P_indptr"]), shape=P.shape)
    assert rel_max_diff(P, ref) <= 1e-10
    dims = sorted([list(k) + [v] for k, v in setup.subproblem_dims.items()])
    assert dims == meta["dims"]


GOLDEN_CASES = ["N4n", "N6d", "N8d", "N10n", "C1", "N16n", "C2"]


@pytest.mark.parametrize("name", GOLDEN_CASES)
def test_hierarchy_vs_reference_golden(name):
    """Full build_hierarchy on the device vs the reference's own outputs."""
    from paper_2506_08284_b200 import multigrid as mg
    meta, arrays = load_case(name)
    s = _system(meta["N"], meta["sigma"], meta["dirichlet"])
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=meta["coarse_size"]))
    assert [lv.A_e.shape[0] for lv in h.levels] == meta["n_edges"]
    assert [lv.A_e.nnz for lv in h.levels] == meta["nnz_A_e"]
    assert abs(h.operator_complexity - meta["operator_complexity"]) < 1e-14
    for li, (lv, L) in enumerate(zip(h.levels, meta["levels"])):
        assert csr_hash(lv.D.to_scipy()) == L["D"], li
        if lv.P_e is None:
            continue
        assert sha(lv.membership.cpu().numpy().astype(np.int64)) == L["membership"]
        assert float(lv.omega).hex() == L["omega_hex"]
        assert float(lv.rho).hex() == L["rho_hex"]
        assert csr_hash(lv.P_n.to_scipy()) == L["P_n"]
        assert sha(lv.assignment.cpu().numpy().astype(np.int64)) == L["assignment"]
        P = lv.P_e.to_scipy()
        assert sha(P.indptr.astype(np.int64), P.indices.astype(np.int64)) == L["P_e_pattern"]
        dims = sorted([list(k) + [v] for k, v in lv.subproblem_dims.items()])
        assert dims == L["subproblem_dims"]
        rows = arrays[f"L{li}_Pe_sample_rows"]
        ref = golden_csr(arrays, f"L{li}_Pe_sample", (rows.size, P.shape[1]))
        assert rel_max_diff(P[rows], ref) <= 1e-10
        if f"L{li}_Pe_vals" in arrays:
            # every P_e entry (values-only goldens of the large cases)
            check_values(P, arrays, f"L{li}_Pe", L["P_e_fro"])
        assert np.allclose(lv.emin_energy, L["emin_energy"], rtol=1e-10, atol=0)
        assert lv.commutator_residual <= 1e-12
        if f"L{li + 1}_A_e_vals" in arrays:
            nxt = h.levels[li + 1]
            for key, M in (("A_e", nxt.A_e), ("S_e", nxt.S_e)):
                Ms = M.to_scipy()
                assert pattern_sha(Ms) == L[f"next_{key}_pattern"], (li, key)
                check_values(Ms, arrays, f"L{li + 1}_{key}")
        if f"L{li + 1}_A_e_data" in arrays:
            nxt = h.levels[li + 1]
            n1 = nxt.A_e.shape[0]
            Aref = golden_csr(arrays, f"L{li + 1}_A_e", (n1, n1))
            Ag = nxt.A_e.to_scipy()
            assert np.array_equal(Ag.indptr, Aref.indptr)
            assert np.array_equal(Ag.indices, Aref.indices)
            assert rel_max_diff(Ag, Aref) <= 1e-10


@pytest.mark.parametrize("name", ["N6d", "N10n", "C1", "N16n", "C2"])
def test_solve_iterations_vs_reference(name):
    """PCG iterations within +-1 of the reference hierarchy with the same
    Chebyshev sweeper, and within +-1 of the reference's Gauss-Seidel."""
    from paper_2506_08284_b200 import multigrid as mg
    meta, _ = load_case(name)
    s = _system(meta["N"], meta["sigma"], meta["dirichlet"])
    b = np.random.default_rng(meta["seed"]).uniform(-1, 1, s.A_e.shape[0])
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=meta["coarse_size"]))
    res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    assert res.status == "converged"
    assert abs(res.iterations - meta["cheb"]["iterations"]) <= 1
    assert res.relative_residual <= 1e-8
    # true residual of the returned x
    x = res.x
    assert np.linalg.norm(b - s.A_e @ x) <= 1.5e-8 * np.linalg.norm(b)


def _tie_heavy_P(m_h, m_H, seed, dense_col=None):
    """Random prolongator-like matrix with many magnitude ties (values from a
    tiny set), optionally one very long column (device long-column path)."""
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for r in range(m_h):
        k = int(rng.integers(1, 7))
        c = rng.choice(m_H, size=k, replace=False)
        rows += [r] * k
        cols += list(c)
    if dense_col is not None:
        extra = np.setdiff1d(np.arange(m_h), np.array(rows)[np.array(cols) == dense_col])
        rows += list(extra)
        cols += [dense_col] * len(extra)
    vals = rng.choice([-1.0, -0.5, 0.25, 0.5, 1.0, 2.0], size=len(rows))
    P = sp.csr_matrix((vals, (rows, cols)), shape=(m_h, m_H))
    P.sum_duplicates()
    P.sort_indices()
    # every column needs an entry (else the reference raises)
    assert np.all(np.diff(P.tocsc().indptr) > 0)
    return P


@pytest.mark.parametrize("case", ["mesh6d", "mesh10n", "mesh16d", "ties", "ties_long", "ties_1pass",
                                  "ties_3pass"])
def test_piecewise_const_device_bitwise(case):
    """Device Algorithm 1 (sync-free column passes, parallel + ordered
    leftovers, safeguard) == the reference's sequential loops."""
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200.coarse_gradient import piecewise_const_assignment as gen_piecewise_const
    from paper_2506_08284_b200.inputs import discretize_hex
    passes = {"ties_1pass": 1, "ties_3pass": 3}.get(case, 2)
    if case.startswith("mesh"):
        N, sig, dr = {"mesh6d": (6, 1.0, True), "mesh10n": (10, 1e-4, False),
                      "mesh16d": (16, 1.0, True)}[case]
        s = discretize_hex(N, sig, dr)
        S = O.strength_pattern(s.A_n)
        mo, nao = O.aggregate(S)
        P, _, _ = O.smoothed_prolongator(s.A_n, mo, nao)
    elif case == "ties_long":
        P = _tie_heavy_P(3000, 200, 7, dense_col=17)
    else:
        P = _tie_heavy_P(2000, 300, 3)
    got = gen_piecewise_const(P, passes).cpu().numpy()
    ref = O.piecewise_const(P, passes)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("case", ["mesh6d", "mesh10n", "mesh16d", "path", "random"])
def test_aggregate_device_bitwise(case):
    """Device aggregation (sync-free distance-2 MIS + ordered leftovers) ==
    the reference's two sequential loops."""
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200.device import DeviceCSR
    from paper_2506_08284_b200.inputs import discretize_hex
    from paper_2506_08284_b200.nodal_amg import aggregate
    if case.startswith("mesh"):
        N, sig, dr = {"mesh6d": (6, 1.0, True), "mesh10n": (10, 1e-4, False),
                      "mesh16d": (16, 1.0, True)}[case]
        S = O.strength_pattern(discretize_hex(N, sig, dr).A_n)
    elif case == "path":
        n = 9
        A = sp.diags([np.ones(n - 1), np.ones(n), np.ones(n - 1)], [-1, 0, 1], format="csr")
        S = sp.csr_matrix(A)
    else:   # irregular symmetric graph: many leftovers and ties
        R = _rand_csr(3000, 3000, 0.002, 11)
        S = sp.csr_matrix(((abs(R) + abs(R.T) + sp.eye(3000)) > 0).astype(np.float64))
    S.sort_indices()
    mo, nao = O.aggregate(S)
    agg = aggregate(DeviceCSR.from_scipy(S))
    assert agg.n_agg == nao
    assert np.array_equal(agg.membership.cpu().numpy(), mo)


def test_piecewise_const_device_errors():
    from paper_2506_08284_b200.coarse_gradient import piecewise_const_assignment as gen_piecewise_const
    P = sp.csr_matrix(np.array([[1.0, 0.0, 0.0], [0.5, 0.0, 2.0]]))
    with pytest.raises(ValueError, match="empty column 1 cannot be assigned any row"):
        gen_piecewise_const(P)


def test_gauss_seidel_half_sweeps_match_scipy():
    """Sync-free tril/triu substitution == x + spsolve_triangular(T, b - A x)
    (multigrid.py:45-59), on an edge operator and its nodal auxiliary."""
    from scipy.sparse.linalg import spsolve_triangular
    from paper_2506_08284_b200.device import DeviceCSR, Status, call
    from paper_2506_08284_b200.inputs import discretize_hex
    s = discretize_hex(6, sigma=0.3, dirichlet=False)
    rng = np.random.default_rng(5)
    for A in (s.A_e, sp.csr_matrix(s.D.T @ s.A_e @ s.D)):
        A = sp.csr_matrix(A)
        A.sort_indices()
        n = A.shape[0]
        x = rng.standard_normal(n)
        b = rng.standard_normal(n)
        Ad = DeviceCSR.from_scipy(A)
        X, B = torch.from_numpy(x).cuda(), torch.from_numpy(b).cuda()
        y = torch.empty(n, dtype=torch.float64, device="cuda")
        out = torch.empty_like(y)
        tk = torch.zeros(1, dtype=torch.int32, device="cuda")
        st = Status()
        for lower, T in ((1, sp.tril(A, format="csr")), (0, sp.triu(A, format="csr"))):
            ref = x + spsolve_triangular(T, b - A @ x, lower=bool(lower))
            call("sphc_gs_half_sweep", n, Ad.rowptr, Ad.col, Ad.val, B, X, out, y, tk, lower, st.t)
            got = out.cpu().numpy()
            assert np.abs(got - ref).max() <= 1e-11 * np.abs(ref).max()
            ref0 = spsolve_triangular(T, b, lower=bool(lower))
            call("sphc_gs_half_sweep", n, Ad.rowptr, Ad.col, Ad.val, B, None, out, y, tk, lower, st.t)
            assert np.abs(out.cpu().numpy() - ref0).max() <= 1e-11 * np.abs(ref0).max()
        assert st.rows() == {}


@pytest.mark.parametrize("name", ["N6d", "N10n", "C1", "C2"])
def test_gauss_seidel_solve_vs_reference(name):
    """The reference's own smoother on the B200 hierarchy: iterations within
    +-1 of the reference's sym-GS PCG, residual history close while far from
    round-off, solution within the solver tolerance."""
    from paper_2506_08284_b200 import multigrid as mg
    meta, arrays = load_case(name)
    s = _system(meta["N"], meta["sigma"], meta["dirichlet"])
    b = np.random.default_rng(meta["seed"]).uniform(-1, 1, s.A_e.shape[0])
    cfg = mg.SolverConfig(coarse_size=meta["coarse_size"], smoother="gauss_seidel")
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, cfg)
    res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    ref = meta["gs"]
    assert res.status == "converged"
    assert abs(res.iterations - ref["iterations"]) <= 1
    k = min(4, len(ref["residual_history"]))
    np.testing.assert_allclose(res.residual_history[:k], ref["residual_history"][:k], rtol=1e-6)
    if "gs_x" in arrays:
        xr = arrays["gs_x"]
        assert np.abs(res.x - xr).max() <= 1e-6 * np.abs(xr).max()


def test_error_case_matches_reference():
    import json
    import os
    from golden_util import GOLDEN
    from paper_2506_08284_b200 import multigrid as mg
    with open(os.path.join(GOLDEN, "errors.json")) as f:
        msg = json.load(f)["N8d_cs100"]
    s = _system(8, 1.0, True)
    with pytest.raises(ValueError) as e:
        mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=100))
    assert str(e.value).split(":")[0] == msg.split(":")[0]


def test_piecewise_const_safeguard_error_matches_reference():
    """Algorithm 1's safeguard failing inside build_hierarchy (a strength
    threshold that leaves a coarse node without a donor row,
    coarse_gradient.py:90-96): the reference's ValueError, same column."""
    import json
    import os
    from golden_util import GOLDEN
    from paper_2506_08284_b200 import multigrid as mg
    from paper_2506_08284_b200.edge_prolongator import EminConfig
    with open(os.path.join(GOLDEN, "errors.json")) as f:
        msg = json.load(f)["N8d_droptol025"]
    s = _system(8, 1.0, True)
    with pytest.raises(ValueError) as e:
        mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D,
                           mg.SolverConfig(coarse_size=100, emin=EminConfig(drop_tol=0.25)))
    assert str(e.value) == msg


def test_partitioned_solve_single_rank_nccl():
    """distributed.py on the GPU with CudaOps and an NCCL group of one rank:
    the partitioned V-cycle / PCG equals the single-GPU solve."""
    import os
    import socket
    import torch.distributed as dist
    from paper_2506_08284_b200 import distributed as D
    from paper_2506_08284_b200 import multigrid as mg
    s = _system(16, 1.0, True)
    b = np.random.default_rng(0).uniform(-1, 1, s.A_e.shape[0])
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=200))
    ref = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        dh = D.distribute_hierarchy(h)
        res = D.dist_pcg_solve(dh, torch.from_numpy(b).cuda())
    finally:
        dist.destroy_process_group()
    assert res.status == "converged"
    assert abs(res.iterations - ref.iterations) <= 1
    x = res.x.cpu().numpy()
    assert np.max(np.abs(x - ref.x)) <= 1e-8 * np.max(np.abs(ref.x))
