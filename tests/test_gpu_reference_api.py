"""The reference's finer-grained API on the device,
same signatures as hcurlamg's, each against the oracle through the C ABI:

* nodal_amg: estimate_rho(A_scaled) and normalize_rows(P) BIT (rho hex and
  every value), smooth_and_normalize(A_n, P_tent) BIT;
* coarse_gradient: gen_piecewise_const(P) -> P_const BIT,
  build_coarse_gradient(D_h, P_const) / augment_dirichlet_edges /
  append_edge BIT on D_H;
* edge_prolongator: initial_feasible_guess / emin_step / commutator_residual
  TOL 1e-10 against the oracle's Alg. 3;
* multigrid: symmetric_gauss_seidel TOL.
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


def _sys(N=6, sigma=1.0, dirichlet=True):
    from paper_2506_08284_b200.inputs import discretize_hex
    return discretize_hex(N, sigma, dirichlet)


@pytest.mark.parametrize("N,dirichlet", [(6, True), (9, False)])
def test_estimate_rho_bitwise(N, dirichlet):
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200 import nodal_amg as na
    s = _sys(N, 1e-2, dirichlet)
    d = s.A_n.diagonal()
    scaled = sp.diags(1.0 / d) @ s.A_n            # the reference's Dinv_A (rows descending)
    for A_scaled in (scaled, O.canonical(scaled)):
        for it in (10, 3):
            assert na.estimate_rho(A_scaled, it).hex() == O.power_rho(A_scaled, it).hex()


def test_normalize_rows_bitwise():
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200 import nodal_amg as na
    rng = np.random.default_rng(4)
    P = sp.random(300, 40, density=0.15, random_state=rng, format="csr")
    P.data = rng.standard_normal(P.nnz) * np.exp(2 * rng.standard_normal(P.nnz))
    P.data[::17] = 0.0                             # stored zeros are dropped
    P.data[P.indptr[5]:P.indptr[6]] = 1.0 / 3.0     # exact-ish sums
    P[7, 3] = 5.0
    P = O.canonical(P)
    rows = np.diff(P.indptr)
    P = P[rows > 0]
    got = na.normalize_rows(P).to_scipy()
    ref = O.normalize_rows(P)
    assert csr_hash(got) == csr_hash(ref)
    Z = sp.csr_matrix(np.array([[1.0, -1.0, 0.0], [0.5, 0.25, 0.0]]))
    with pytest.raises(ValueError, match="zero row sum before scaling in row 0"):
        na.normalize_rows(Z)


def test_smooth_and_normalize_reference_signature():
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200 import nodal_amg as na
    s = _sys(8, 1.0, True)
    agg = na.aggregate(na.strength_graph(s.A_n, 0.0))
    P_tent = na.tentative_prolongator(agg)
    nod = na.smooth_and_normalize(s.A_n, P_tent)
    memb, n_agg = O.aggregate(O.strength_pattern(s.A_n))
    Po, w, rho = O.smoothed_prolongator(s.A_n, memb, n_agg)
    assert csr_hash(nod.P.to_scipy()) == csr_hash(Po)
    assert nod.omega_used.hex() == w.hex() and nod.rho_estimate.hex() == rho.hex()
    # scipy tentative prolongator too
    Pt = sp.csr_matrix((np.ones(memb.size), memb, np.arange(memb.size + 1)),
                       shape=(memb.size, n_agg))
    assert csr_hash(na.smooth_and_normalize(s.A_n, Pt).P.to_scipy()) == csr_hash(Po)
    with pytest.raises(ValueError, match="incompatible shapes"):
        na.smooth_and_normalize(s.A_n, Pt[:-1])


def test_coarse_gradient_reference_signatures():
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200 import coarse_gradient as cgm
    from paper_2506_08284_b200 import nodal_amg as na
    s = _sys(8, 1.0, True)
    nod = na.smooth_and_normalize(s.A_n, na.aggregate(na.strength_graph(s.A_n, 0.0)))
    P_const = cgm.gen_piecewise_const(nod.P, 2)
    memb, n_agg = O.aggregate(O.strength_pattern(s.A_n))
    Po, _, _ = O.smoothed_prolongator(s.A_n, memb, n_agg)
    assign = O.piecewise_const(Po, 2)
    Pc = P_const.to_scipy()
    assert np.array_equal(Pc.indices, assign) and np.all(Pc.data == 1.0)
    ce = O.coarse_edges(s.D, assign, n_agg)
    cg = cgm.build_coarse_gradient(s.D, P_const)
    interior = O.CoarseEdges(pairs=ce.pairs, singles=np.zeros(0, np.int64), n_nodes=n_agg)
    assert csr_hash(cg.D_H.to_scipy()) == csr_hash(interior.D_H())
    cg = cgm.augment_dirichlet_edges(cg, s.D, P_const)
    assert ce.singles.size > 0
    assert csr_hash(cg.D_H.to_scipy()) == csr_hash(ce.D_H())
    cg2 = cgm.append_edge(cg, 5, 2)
    assert cg2.augmented_edges == [(2, 5)]
    aug = O.CoarseEdges(pairs=ce.pairs, singles=ce.singles, n_nodes=n_agg,
                        augmented=np.array([[2, 5]]))
    assert csr_hash(cg2.D_H.to_scipy()) == csr_hash(aug.D_H())
    assert cg2.edge_endpoints[-1] == (2, 5)


def test_alg3_pieces_vs_oracle():
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200 import coarse_gradient as cgm
    from paper_2506_08284_b200 import edge_prolongator as ep
    from paper_2506_08284_b200 import emin_setup as es
    from paper_2506_08284_b200 import nodal_amg as na
    s = _sys(8, 1e-2, False)
    nod = na.smooth_and_normalize(s.A_n, na.aggregate(na.strength_graph(s.A_n, 0.0)))
    P_const = cgm.gen_piecewise_const(nod.P, 2)
    cg = cgm.augment_dirichlet_edges(cgm.build_coarse_gradient(s.D, P_const), s.D, P_const)
    setup = es.setup_constraints(s.D, nod.P, cg)
    structure, v0 = ep.initial_feasible_guess(setup)
    v1 = ep.emin_step(s.S, v0, setup, structure, 0.5)
    memb, n_agg = O.aggregate(O.strength_pattern(s.A_n))
    Po, _, _ = O.smoothed_prolongator(s.A_n, memb, n_agg)
    ce = O.coarse_edges(s.D, O.piecewise_const(Po, 2), n_agg)
    e0 = O.emin_prolongator(s.D, Po, ce, s.S, iterations=0)
    e1 = O.emin_prolongator(s.D, Po, ce, s.S, iterations=1)
    ind = structure.col.cpu().numpy()
    assert np.array_equal(ind, e0.P_e.indices)
    scale = np.abs(e1.P_e.data).max()
    assert np.max(np.abs(v0.cpu().numpy() - e0.P_e.data)) <= 1e-10 * scale
    assert np.max(np.abs(v1.cpu().numpy() - e1.P_e.data)) <= 1e-10 * scale
    from paper_2506_08284_b200.device import DeviceCSR
    P1 = DeviceCSR(structure.rowptr, structure.col, v1, structure.shape)
    res = ep.commutator_residual(P1, cg.D_H, setup.R_dp)
    assert res <= 1e-12
    assert abs(res - e1.commutator_residual) <= 1e-13
    # a perturbed prolongator: the defect is what scipy computes
    v2 = v1.clone()
    v2[3] += 1e-3
    P2 = DeviceCSR(structure.rowptr, structure.col, v2, structure.shape)
    ref = O.max_abs(O.canonical(P2.to_scipy() @ ce.D_H() - e1.R_dp))
    assert abs(ep.commutator_residual(P2, cg.D_H, setup.R_dp) - ref) <= 1e-15 * ref


def test_symmetric_gauss_seidel_vs_oracle():
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200 import multigrid as mg
    s = _sys(6, 1.0, True)
    rng = np.random.default_rng(2)
    x = rng.standard_normal(s.A_e.shape[0])
    b = rng.standard_normal(s.A_e.shape[0])
    got = mg.symmetric_gauss_seidel(s.A_e, x, b, sweeps=2)
    ref = O.GaussSeidelSweeper(s.A_e).symmetric(x, b, sweeps=2)
    assert isinstance(got, np.ndarray)
    assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))
