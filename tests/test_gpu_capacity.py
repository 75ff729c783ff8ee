"""Capacity fallbacks: inputs whose rows exceed the on-chip kernels'
buffers degrade to global-memory paths instead of raising (imported
MatrixMarket systems, mmio.py, have no structural bound).

* SpGEMM rows of > 256 distinct columns, or with a B row longer than a
  staging window: one CTA per row, hash tables in global memory
  (sphc_spgemm_global), same ascending-k sums -- bitwise scipy for the
  ordered product;
* a whole hierarchy driven through that path (every row of more than 8
  output columns) equals the on-chip one;
* aggregation of nodes with > 256 aggregated neighbours;
* emin constraint blocks beyond the default class (|J| > 16 or |I| > 128)
  re-run through the wide class (one lane per coarse node, |J| <= 32): a
  whole hierarchy and the make_irreducible flow driven through it are bitwise
  the default ones, genuinely wide blocks match the oracle, and blocks
  beyond the wide class raise.
"""

import numpy as np
import pytest
import scipy.sparse as sp

from golden_util import csr_hash, rel_max_diff

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")


def _rand(n, m, per_row, seed, dense_rows=(), dense_len=0):
    rng = np.random.default_rng(seed)
    rows, cols = [], []
    for r in range(n):
        k = dense_len if r in dense_rows else per_row
        c = rng.choice(m, size=min(k, m), replace=False)
        rows += [r] * c.size
        cols += list(c)
    A = sp.csr_matrix((rng.standard_normal(len(rows)), (rows, cols)), shape=(n, m))
    A.sum_duplicates()
    A.sort_indices()
    return A


def test_spgemm_long_rows_global_path():
    from paper_2506_08284_b200 import device as dv
    A = _rand(3000, 2500, 6, 0, dense_rows=(5, 17, 2999), dense_len=900)
    B = _rand(2500, 4000, 4, 1, dense_rows=(7,), dense_len=1200)   # a long B row too
    A2, B2 = A.copy(), B.copy()
    A2.data = A2.data * 0.5 + 1.0
    B2.data = B2.data - 2.0
    ref = (A @ B).tocsr()
    ref.sort_indices()
    assert np.diff(ref.indptr).max() > 2000
    before = dv.STATS["spgemm_global_rows"]
    dA, dB = dv.DeviceCSR.from_scipy(A), dv.DeviceCSR.from_scipy(B)
    C = dv.spgemm(dA, dB, ordered=True).to_scipy()
    assert dv.STATS["spgemm_global_rows"] > before
    assert csr_hash(C) == csr_hash(ref)              # bitwise scipy (ordered sums)
    Cu = dv.spgemm(dA, dB).to_scipy()
    assert rel_max_diff(Cu, ref) <= 1e-14
    C1, C2 = dv.spgemm_pair(dA, dv.DeviceCSR.from_scipy(A2), dB, dv.DeviceCSR.from_scipy(B2))
    assert rel_max_diff(C1.to_scipy(), ref) <= 1e-14
    assert rel_max_diff(C2.to_scipy(), A2 @ B2) <= 1e-14


def test_hierarchy_through_global_spgemm_path():
    from paper_2506_08284_b200 import device as dv
    from paper_2506_08284_b200 import multigrid as mg
    from paper_2506_08284_b200.inputs import discretize_hex
    s = discretize_hex(10, 1.0, False)
    cfg = mg.SolverConfig(coarse_size=100)
    h0 = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, cfg)
    old = dv.GLOBAL_ROWS_ABOVE
    dv.GLOBAL_ROWS_ABOVE = 8
    try:
        before = dv.STATS["spgemm_global_rows"]
        h1 = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, cfg)
        assert dv.STATS["spgemm_global_rows"] - before > 5000
    finally:
        dv.GLOBAL_ROWS_ABOVE = old
    assert [lv.A_e.shape[0] for lv in h0.levels] == [lv.A_e.shape[0] for lv in h1.levels]
    for a, b in zip(h0.levels, h1.levels):
        A0, A1 = a.A_e.to_scipy(), b.A_e.to_scipy()
        assert np.array_equal(A0.indptr, A1.indptr) and np.array_equal(A0.indices, A1.indices)
        assert rel_max_diff(A1, A0) <= 1e-12
        if a.P_n is not None:      # the ordered nodal Galerkin: bitwise either way
            assert csr_hash(a.P_n.to_scipy()) == csr_hash(b.P_n.to_scipy())
    b = np.random.default_rng(0).uniform(-1, 1, s.A_e.shape[0])
    r0 = mg.pcg_solve(h0.levels[0].A_e, b, mg.v_cycle_preconditioner(h0))
    r1 = mg.pcg_solve(h1.levels[0].A_e, b, mg.v_cycle_preconditioner(h1))
    assert r0.iterations == r1.iterations


def test_aggregation_high_degree_nodes():
    """Aggregation (nodal_amg.py:59-88) of a graph whose leftover nodes have
    > 256 aggregated neighbours: bitwise the reference's loops (oracle)."""
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200 import nodal_amg as na
    n = 3001
    rng = np.random.default_rng(3)
    rows, cols = [], []
    for i in range(n - 1):                # a path 0..n-2 ...
        if i + 2 < n:
            rows += [i, i + 1]
            cols += [i + 1, i]
    # ... plus a hub (node n-1) joined to 700 path nodes that phase 1 claims
    # before visiting them (i = 1 mod 3): the hub is a leftover with 700
    # aggregated neighbours
    nb = rng.choice(np.arange(1, n - 1, 3), size=700, replace=False)
    rows += [n - 1] * nb.size + list(nb)
    cols += list(nb) + [n - 1] * nb.size
    G = sp.csr_matrix((np.ones(len(rows)), (rows, cols)), shape=(n, n))
    G = G + sp.identity(n) * 4.0
    G.sum_duplicates()
    G.sort_indices()
    S = na.strength_graph(G, 0.0)
    agg = na.aggregate(S)
    memb, n_agg = O.aggregate(O.strength_pattern(G))
    assert agg.n_agg == n_agg
    assert np.array_equal(agg.membership.cpu().numpy(), memb)


def test_thin_spgemm_is_bitwise_scipy():
    """The thread-per-row kernels (sphc_spgemm_*_thin: products with few
    multiplications per row, <= 32 distinct columns) walk their products in
    scipy's csr_matmat order, so even the unordered entry points are bitwise
    scipy; rows beyond 32 columns fall to the warp kernels (TOL there), rows
    with no entries and empty B rows included. Pair product likewise."""
    from paper_2506_08284_b200 import device as dv
    # a gradient-like B (<= 2 entries per row, some rows empty)
    rng = np.random.default_rng(11)
    n, m = 5000, 1800
    A = _rand(n, 4000, 9, 2)
    A.data[A.indptr[17]:A.indptr[18]] = 0.0      # an empty A row
    A.eliminate_zeros()
    bi, bj, bv = [], [], []
    for r in range(4000):
        k = rng.integers(0, 3)
        c = rng.choice(m, size=k, replace=False)
        bi += [r] * k
        bj += list(c)
        bv += list(rng.choice([-1.0, 1.0], size=k))
    B = sp.csr_matrix((bv, (bi, bj)), shape=(4000, m))
    B.sort_indices()
    assert dv._thin_rows(dv.DeviceCSR.from_scipy(A), dv.DeviceCSR.from_scipy(B))
    ref = (A @ B).tocsr()
    ref.sort_indices()
    dA, dB = dv.DeviceCSR.from_scipy(A), dv.DeviceCSR.from_scipy(B)
    C = dv.spgemm(dA, dB, drop=False).to_scipy()
    assert csr_hash(C) == csr_hash(ref)
    A2 = A.copy()
    A2.data = A2.data * 0.25 - 3.0
    C1, C2 = dv.spgemm_pair(dA, dv.DeviceCSR.from_scipy(A2), dB, dB, drop=False)
    ref2 = (A2 @ B).tocsr()
    ref2.sort_indices()
    assert csr_hash(C1.to_scipy()) == csr_hash(ref) and csr_hash(C2.to_scipy()) == csr_hash(ref2)
    # mixed: a few A rows reach > 32 distinct columns -> warp kernels for those
    Ab = _rand(3000, 4000, 9, 5, dense_rows=(3, 1500, 2999), dense_len=60)
    dAb = dv.DeviceCSR.from_scipy(Ab)
    assert dv._thin_rows(dAb, dB)
    refb = (Ab @ B).tocsr()
    refb.sort_indices()
    assert np.diff(refb.indptr).max() > 32
    Cb = dv.spgemm(dAb, dB, drop=False).to_scipy()
    assert np.array_equal(Cb.indptr, refb.indptr) and np.array_equal(Cb.indices, refb.indices)
    assert rel_max_diff(Cb, refb) <= 1e-14
    Co = dv.spgemm(dAb, dB, drop=False, ordered=True).to_scipy()
    assert csr_hash(Co) == csr_hash(refb)


def _same_csr(A, B):
    return (torch.equal(A.rowptr, B.rowptr) and torch.equal(A.col, B.col)
            and torch.equal(A.val, B.val))


@pytest.mark.parametrize("N,sigma,dirichlet,coarse", [(10, 1.0, False, 100), (12, 1e-2, True, 200)])
def test_hierarchy_through_wide_emin_class(N, sigma, dirichlet, coarse):
    """Every constraint block with |J| > 6 or |I| > 12 driven through the wide
    capacity class of the emin kernels (count, fill, sweeps): the hierarchy is
    bit for bit the default one (same arithmetic in the same order)."""
    from paper_2506_08284_b200 import emin_setup as es
    from paper_2506_08284_b200 import multigrid as mg
    from paper_2506_08284_b200.inputs import discretize_hex
    s = discretize_hex(N, sigma, dirichlet)
    cfg = mg.SolverConfig(coarse_size=coarse)
    h0 = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, cfg)
    old = es.DEFAULT_CLASS_CAPS
    es.DEFAULT_CLASS_CAPS = (6, 12)
    try:
        h1 = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, cfg)
    finally:
        es.DEFAULT_CLASS_CAPS = old
    assert h0.n_levels == h1.n_levels
    for a, b in zip(h0.levels, h1.levels):
        assert _same_csr(a.A_e, b.A_e) and _same_csr(a.S_e, b.S_e)
        if a.P_e is None:
            continue
        assert _same_csr(a.P_e, b.P_e)
        assert a.subproblem_dims == b.subproblem_dims
        assert a.emin_energy == b.emin_energy
        assert a.commutator_residual == b.commutator_residual
        assert max(k[1] for k in a.subproblem_dims) > 6      # the wide class did run


def test_make_irreducible_through_wide_emin_class():
    """The repair flow (flagged rows, appended coarse edges, refill) with the
    blocks in the wide class: same result as the default class, which
    test_gpu_parity.py pins to the reference's make_irreducible."""
    import json
    import os
    from golden_util import GOLDEN
    from paper_2506_08284_b200 import coarse_gradient as cg_mod
    from paper_2506_08284_b200 import emin_setup as es
    from paper_2506_08284_b200 import nodal_amg as na
    from paper_2506_08284_b200.inputs import discretize_hex
    with open(os.path.join(GOLDEN, "repair_N10d.json")) as f:
        meta = json.load(f)
    arr = dict(np.load(os.path.join(GOLDEN, "repair_N10d.npz")))
    s = discretize_hex(10, 1.0, True)
    agg = na.aggregate(na.strength_graph(s.A_n, 0.0))
    nod = na.smooth_and_normalize(s.A_n, agg)

    def run():
        cg = cg_mod.coarse_gradient_from_edges(arr["pairs"], arr["singles"], meta["n_nodes"])
        return es.setup_constraints(s.D, nod.P, cg)
    s0 = run()
    old = es.DEFAULT_CLASS_CAPS
    es.DEFAULT_CLASS_CAPS = (5, 10)
    try:
        s1 = run()
    finally:
        es.DEFAULT_CLASS_CAPS = old
    assert s0.n_augmented == s1.n_augmented == meta["n_augmented"] > 0
    assert [list(e) for e in s1.cg.augmented_edges] == meta["augmented"]
    assert _same_csr(s0.pattern, s1.pattern) and _same_csr(s0.T, s1.T)
    assert s0.subproblem_dims == s1.subproblem_dims


def test_wide_constraint_blocks_vs_oracle():
    """Blocks that really exceed the default class: the C4 recipe at 10^3 with
    drop_tol = 0.08 shrinks the aggregates until 1387 fine edges see 17-28
    coarse nodes (|I| up to 118). First level against the oracle (which has no
    capacity): STRUCT, subproblem dims, TOL 1e-10; then the whole hierarchy
    builds and PCG converges. drop_tol = 0.09 gives |J| = 34: beyond the wide
    class too, which must raise, not truncate."""
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200 import edge_prolongator as ep
    from paper_2506_08284_b200 import multigrid as mg
    from paper_2506_08284_b200.assembly import make_device_config
    s, rhs, cfg = make_device_config("C4", 10)
    A_e, S, A_n, D = (M.to_scipy() for M in (s.A_e, s.S, s.A_n, s.D))
    prol, cgd, nod = ep.build_edge_prolongator(s.A_n, s.A_e, s.S, s.D,
                                               ep.EminConfig(drop_tol=0.08))
    memb, nagg = O.aggregate(O.strength_pattern(A_n, 0.08))
    Po, _, _ = O.smoothed_prolongator(A_n, memb, nagg)
    ce = O.coarse_edges(D, O.piecewise_const(Po, 2), nagg)
    em = O.emin_prolongator(D, Po, ce, S)
    assert max(k[1] for k in em.subproblem_dims) > 16
    assert dict(prol.subproblem_dims) == dict(em.subproblem_dims)
    P = prol.P_e.to_scipy()
    assert np.array_equal(P.indptr, em.P_e.indptr)
    assert np.array_equal(P.indices, em.P_e.indices)
    assert rel_max_diff(P, em.P_e) <= 1e-10
    assert np.allclose(prol.energy_history, em.energy_history, rtol=1e-10, atol=0)
    assert prol.commutator_residual <= 1e-12
    assert prol.n_augmented == em.n_augmented
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D,
                           mg.SolverConfig(coarse_size=200, emin=ep.EminConfig(drop_tol=0.08)))
    r = mg.pcg_solve(h.levels[0].A_e, rhs, mg.v_cycle_preconditioner(h))
    assert r.status == "converged"
    with pytest.raises(RuntimeError, match="wide class"):
        ep.build_edge_prolongator(s.A_n, s.A_e, s.S, s.D, ep.EminConfig(drop_tol=0.09))
