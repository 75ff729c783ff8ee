"""Randomised parity: seeded draws of the mesh size, boundary condition,
jitter, per-element sigma (lognormal spreads up to 8 decades, jumps) and
EminConfig knobs, each built on the device and by the oracle (the CPU
restatement pinned to the reference's goldens, tests/test_oracle.py) on the
same matrices. BIT: aggregates, rho / omega, P_n, Algorithm-1 assignment, D_H,
level sizes; STRUCT: P_e and coarse patterns (up to exact-cancellation
entries of round-off size); TOL 1e-10: P_e, coarse A_e / S_e, energies;
commutator residual <= 1e-12; ITER: PCG (Chebyshev seam) within +-1.
A draw on which the oracle raises must raise the same error on the device."""

import numpy as np
import pytest

from golden_util import csr_hash, rel_max_diff

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")


def _draw(seed):
    rng = np.random.default_rng(1000 + seed)
    N = int(rng.integers(5, 17))
    dirichlet = bool(rng.integers(0, 2))
    h = 1.0 / N
    jitter = rng.uniform(-0.2 * h, 0.2 * h, ((N - 1) ** 3, 3)) if rng.integers(0, 2) else None
    kind = int(rng.integers(0, 3))
    if kind == 0:
        sigma = float(10.0 ** rng.uniform(-6, 2))
    elif kind == 1:
        sigma = rng.lognormal(np.log(10.0 ** rng.uniform(-4, 0)), rng.uniform(0.5, 2.5), N ** 3)
    else:
        sigma = np.where(rng.random(N ** 3) < 0.3, 10.0 ** rng.uniform(-6, -2), 1.0)
    emin = dict(omega=float(rng.choice([0.5, 0.7, 1.0])), iterations=int(rng.choice([0, 1, 1, 2])),
                n_passes=int(rng.choice([1, 2, 2, 3])))
    coarse = int(rng.choice([30, 100, 300]))
    return N, dirichlet, jitter, sigma, emin, coarse, rng.uniform(-1, 1, 1)


@pytest.mark.parametrize("seed", range(30))
def test_random_config_vs_oracle(seed):
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200 import multigrid as mg
    from paper_2506_08284_b200.assembly import assemble_hex
    from paper_2506_08284_b200.edge_prolongator import EminConfig
    N, dirichlet, jitter, sigma, emin, coarse, _ = _draw(seed)
    s = assemble_hex(N, sigma, dirichlet, jitter)
    A_e, S, A_n, D = (M.to_scipy() for M in (s.A_e, s.S, s.A_n, s.D))
    rhs = np.random.default_rng(seed).uniform(-1, 1, A_e.shape[0])
    try:
        ho = O.build_hierarchy(A_e, S, A_n, D, coarse_size=coarse, smoother="cheb", **emin)
    except ValueError as e:
        # e.g. a coarse curl-curl operator that is pure round-off: same error
        with pytest.raises(ValueError) as got:
            mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D,
                               mg.SolverConfig(coarse_size=coarse, emin=EminConfig(**emin)))
        head = str(e).split(": max|S D|")[0]
        assert str(got.value).startswith(head), (str(got.value), str(e))
        return
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D,
                           mg.SolverConfig(coarse_size=coarse, emin=EminConfig(**emin)))
    assert [lv.A_e.shape[0] for lv in h.levels] == [lv.A_e.shape[0] for lv in ho.levels]
    for li, (lv, lo) in enumerate(zip(h.levels, ho.levels)):
        assert csr_hash(lv.D.to_scipy()) == csr_hash(lo.D), li
        A = lv.A_e.to_scipy()
        if li > 0:
            for got, want in ((A, lo.A_e), (lv.S_e.to_scipy(), lo.S_e)):
                scale = abs(want).max()
                if got.nnz == want.nnz:
                    assert np.array_equal(got.indptr, want.indptr), li
                    assert np.array_equal(got.indices, want.indices), li
                # entries only one side keeps are exact cancellations on the other
                assert abs(got - want).max() <= 1e-10 * scale, li
        if lv.P_e is None:
            continue
        assert np.array_equal(lv.membership.cpu().numpy(), lo.membership), li
        assert lv.omega == lo.omega and lv.rho == lo.rho, li
        assert csr_hash(lv.P_n.to_scipy()) == csr_hash(lo.P_n), li
        assert np.array_equal(lv.assignment.cpu().numpy(), lo.assignment), li
        P = lv.P_e.to_scipy()
        assert np.array_equal(P.indptr, lo.P_e.indptr) and np.array_equal(P.indices, lo.P_e.indices)
        assert rel_max_diff(P, lo.P_e) <= 1e-10, li
        assert dict(lv.subproblem_dims) == dict(lo.emin.subproblem_dims), li
        assert lv.n_augmented == lo.emin.n_augmented, li
        assert np.allclose(lv.emin_energy, lo.emin.energy_history, rtol=1e-9, atol=0), li
        assert lv.commutator_residual <= 1e-12, li
    r = mg.pcg_solve(h.levels[0].A_e, rhs, mg.v_cycle_preconditioner(h), maxit=200)
    ro = O.solve(ho, rhs, maxit=200)
    assert r.status == ro.status
    if r.status == "converged":
        assert abs(r.iterations - ro.iterations) <= 1
        k = min(len(r.residual_history), len(ro.residual_history), 6)
        np.testing.assert_allclose(r.residual_history[:k], ro.residual_history[:k], rtol=1e-5)
