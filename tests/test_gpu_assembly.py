"""Device input generator (csrc/assemble.cu) vs the host generator and the
independent isoparametric checker (tests/iso_assembly.py)."""

import numpy as np
import pytest
import scipy.sparse as sp

import iso_assembly as ISO
from paper_2506_08284_b200.inputs import discretize_hex

torch = pytest.importorskip("torch")


def _cmp(dev, ref, tol, name):
    X = dev.to_scipy() if not sp.issparse(dev) else dev
    assert X.shape == ref.shape, name
    assert np.array_equal(X.indptr, ref.indptr), f"{name}: row pointers differ"
    assert np.array_equal(X.indices, ref.indices), f"{name}: columns differ"
    err = np.abs(X.data - ref.data).max() / np.abs(ref.data).max()
    assert err <= tol, f"{name}: rel diff {err:.2e}"


def _jitter(N, seed, amp=0.2):
    rng = np.random.default_rng(seed)
    h = 1.0 / N
    return rng.uniform(-amp * h, amp * h, ((N - 1) ** 3, 3))


# CPU: the checker itself is pinned to the reference-faithful host generator
@pytest.mark.parametrize("N,dirichlet", [(3, False), (4, True)])
def test_iso_checker_matches_host_generator_at_zero_jitter(N, dirichlet):
    sig = np.random.default_rng(N).lognormal(0.0, 1.0, N ** 3)
    A, S, An, D = ISO.assemble(N, sig, dirichlet)
    h = discretize_hex(N, sig, dirichlet)
    _cmp(A, h.A_e, 1e-14, "A_e")
    _cmp(S, h.S, 1e-14, "S")
    _cmp(An, h.A_n, 1e-14, "A_n")
    _cmp(D, h.D, 0.0, "D")


def test_iso_checker_curl_of_gradient_vanishes():
    N = 4
    A, S, An, D = ISO.assemble(N, 1.0, False, _jitter(N, 1))
    assert np.abs(S @ D).max() <= 1e-13 * np.abs(S).max()


@pytest.fixture(scope="module")
def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    from paper_2506_08284_b200.build import build_library
    build_library()


@pytest.mark.gpu
@pytest.mark.parametrize("N,dirichlet,sigma", [(1, False, 1.0), (2, True, 1.0), (6, False, 1e-2),
                                               (7, True, 1e-4), (5, False, "lognormal"),
                                               (6, True, "lognormal")])
def test_device_assembly_uniform_vs_host(_gpu, N, dirichlet, sigma):
    from paper_2506_08284_b200.assembly import assemble_hex
    if sigma == "lognormal":
        sigma = np.random.default_rng(7).lognormal(np.log(1e-3), 2.0, N ** 3)
    if dirichlet and N < 3:
        pytest.skip("no free edges")
    d = assemble_hex(N, sigma, dirichlet)
    h = discretize_hex(N, sigma, dirichlet)
    _cmp(d.A_e, h.A_e, 2e-15, "A_e")
    _cmp(d.S, h.S, 2e-15, "S")
    _cmp(d.A_n, h.A_n, 2e-15, "A_n")
    _cmp(d.D, h.D, 0.0, "D")


@pytest.mark.gpu
@pytest.mark.parametrize("N,dirichlet", [(4, False), (5, True), (8, False)])
def test_device_assembly_jittered_vs_checker(_gpu, N, dirichlet):
    from paper_2506_08284_b200.assembly import assemble_hex
    jit = _jitter(N, N)
    sig = np.random.default_rng(N).lognormal(np.log(1e-3), 2.0, N ** 3)
    d = assemble_hex(N, sig, dirichlet, jit)
    A, S, An, D = ISO.assemble(N, sig, dirichlet, jit)
    _cmp(d.A_e, A, 1e-13, "A_e")
    _cmp(d.S, S, 1e-13, "S")
    _cmp(d.A_n, An, 1e-13, "A_n")
    _cmp(d.D, D, 0.0, "D")


@pytest.mark.gpu
def test_device_assembly_exact_symmetry_and_curl_grad(_gpu):
    from paper_2506_08284_b200.assembly import assemble_hex
    N = 9
    d = assemble_hex(N, np.random.default_rng(2).lognormal(0, 2, N ** 3), False, _jitter(N, 3))
    for M in (d.A_e, d.S, d.A_n):
        X = M.to_scipy()
        assert (X != X.T).nnz == 0          # bitwise symmetric
    S, D = d.S.to_scipy(), d.D.to_scipy()
    assert np.abs(S @ D).max() <= 1e-12 * np.abs(S).max()
    assert d.A_e.rowptr is d.S.rowptr and d.A_e.col is d.S.col   # one shared pattern


@pytest.mark.gpu
def test_device_config_c4_small_hierarchy_vs_oracle(_gpu):
    """C4's recipe (jittered hexes, lognormal sigma, one rng) at N=8 through
    setup + solve, against the oracle on the downloaded inputs."""
    from oracle import hcurl_oracle as O
    from paper_2506_08284_b200 import multigrid as mg
    from paper_2506_08284_b200.assembly import make_device_config
    sysd, rhs, cfg = make_device_config("C4", 8)
    assert cfg["N"] == 8 and sysd.coords is not None
    h = mg.build_hierarchy(sysd.A_e, sysd.S, sysd.A_n, sysd.D, mg.SolverConfig(coarse_size=50))
    res = mg.pcg_solve(h.levels[0].A_e, rhs, mg.v_cycle_preconditioner(h))
    A_e, S, A_n, D = (M.to_scipy() for M in (sysd.A_e, sysd.S, sysd.A_n, sysd.D))
    ho = O.build_hierarchy(A_e, S, A_n, D, coarse_size=50, smoother="cheb")
    ro = O.solve(ho, rhs)
    assert [lv.A_e.shape[0] for lv in h.levels] == [lv.A_e.shape[0] for lv in ho.levels]
    for lv, lo in zip(h.levels, ho.levels):
        if lo.membership is not None:
            assert np.array_equal(lv.membership.cpu().numpy(), lo.membership)
    assert res.status == "converged"
    assert abs(res.iterations - ro.iterations) <= 1, (res.iterations, ro.iterations)


@pytest.mark.gpu
@pytest.mark.parametrize("config,N", [("C4", 12), ("C3", 16), ("C2", 8), ("C5", 10)])
def test_device_assembly_equals_host_build_bitwise(config, N):
    """The device generator and its host build (oracle/host_assembly.py, the
    input source of the reference goldens for the device configs) produce the
    same bits: same per-row source, explicit IEEE rounding."""
    from golden_util import csr_hash
    from oracle.host_assembly import config_host
    from paper_2506_08284_b200.assembly import make_device_config
    s, rhs, _ = make_device_config(config, N)
    A_e, S, A_n, D, rhs_h, _ = config_host(config, N)
    assert np.array_equal(rhs, rhs_h)
    for M, H in ((s.A_e, A_e), (s.S, S), (s.A_n, A_n), (s.D, D)):
        assert csr_hash(M.to_scipy()) == csr_hash(H)
