"""Device hierarchy vs the UNMODIFIED reference on the benchmark recipes
(row X1 of the round-1 verdict: parity where the performance is claimed).

Goldens ``hier_C4s`` (C4 recipe at 16^3), ``hier_C3`` (64^3, sigma jump),
``hier_C5s`` (C5 recipe at 64^3) and ``hier_C4rh`` (the C4 recipe at 128^3,
the smallest size where ``make_irreducible`` fires: 154 coarse edges appended
on level 2) were made by running the reference on the host build of the
device assembly (oracle/host_assembly.py, tests/golden/make_golden.py BIG).
Goldens ``hier_V*`` run non-default EminConfig / SolverConfig knobs (omega,
iterations, n_passes, drop_tol, max_levels) on small hex meshes.
Goldens ``hier_T9n`` / ``hier_T8d`` (tet meshes), ``hier_Q41d`` (2-D quads)
and ``hier_R33n`` (2-D triangles) are the reference on its own other element
families (meshing.py:15), inputs stored with the golden.
Each test assembles the same config on the B200, proves the inputs identical
(sha256 of A_e, S, A_n, D and of the RHS), builds the hierarchy through the
public API and checks:

* BIT: aggregates, rho / omega (hex), P_n, piecewise-constant assignment,
  coarse edge lists, D_H per level (incl. the appended coarse edges, their
  endpoints and the reference's duplicates), level sizes and nnz, operator
  complexity, subproblem dims;
* STRUCT: P_e and every coarse A_e / S_e pattern (sha256); a coarse S_e may
  lack a handful of the reference's entries that cancel to an exact zero in
  the device's summation order (both sides drop exact zeros): it must then
  equal the reference on the reference's pattern with zeros restored;
* TOL 1e-10 (relative to the matrix max): P_e and coarse A_e / S_e values --
  every entry where the golden holds them all, else every k-th row
  (``<key>_stride``) plus the Frobenius norm of the whole matrix; emin
  energies rtol 1e-10; commutator residual <= 1e-12;
* ITER: PCG iterations within +-1 of the reference hierarchy with the same
  Chebyshev sweeper in its seam: C4s, C3 and the headline C4 at 128^3 (the
  reference converges in 81 iterations there; so does the device, with its
  default equilibrated-Cholesky coarsest solve). On the C5 recipe at 64^3
  (sigma = 1e-4, coarse_size 1000) the reference itself does not converge
  (its LU coarsest solve on a numerically singular operator: maxit = 500 at
  7.7e-7 with the Chebyshev seam, 2.2e-5 with its own Gauss-Seidel): the
  device's LU mode (``coarse_solver="lu"``) reproduces that exit, and the
  default coarsest solve converges (the documented deviation).
"""

import os

import numpy as np
import pytest

from golden_util import (GOLDEN, MESH, MESH_SINGULAR, VARIANTS, check_coarse_operator, check_values, csr_hash, embed_in_pattern, load_case,
                         pattern_sha, sha, stored_inputs)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CASES = ["C4s", "C5s", "C3", "C4rh"]


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.fail("GPU tests need a CUDA device (no CPU fallback exists)")
    from paper_2506_08284_b200.build import build_library
    build_library()


def _case(name):
    if not os.path.exists(os.path.join(GOLDEN, f"hier_{name}.json")):
        pytest.fail(f"golden hier_{name} missing (tests/golden/make_golden.py {name})")
    return load_case(name)


@pytest.mark.parametrize("name", CASES + MESH + MESH_SINGULAR + VARIANTS)
def test_device_config_vs_reference(name):
    from types import SimpleNamespace
    from paper_2506_08284_b200 import multigrid as mg, device as dv
    from paper_2506_08284_b200.assembly import make_device_config
    meta, arrays = _case(name)
    if "mesh" in meta:
        # the reference's own tet / quad / tri system (meshing.py:15), stored
        # with the golden: the path only sees (A_e, S, A_n, D)
        A_e, S, A_n, D, rhs = stored_inputs(arrays)
        s = SimpleNamespace(A_e=dv.DeviceCSR.from_scipy(A_e), S=dv.DeviceCSR.from_scipy(S),
                            A_n=dv.DeviceCSR.from_scipy(A_n), D=dv.DeviceCSR.from_scipy(D))
    else:
        s, rhs, cfg = make_device_config(meta["config"], meta["N"])
    # identical inputs: the device assembly is the reference run's input
    for k, M in (("A_e", s.A_e), ("S", s.S), ("A_n", s.A_n), ("D", s.D)):
        assert csr_hash(M.to_scipy()) == meta["inputs"][k], k
    assert sha(rhs) == meta["rhs"]

    from paper_2506_08284_b200.edge_prolongator import EminConfig
    scfg = mg.SolverConfig(coarse_size=meta["coarse_size"],
                           max_levels=meta.get("max_levels", 10),
                           emin=EminConfig(**meta.get("emin", {})))
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, scfg)
    assert [lv.A_e.shape[0] for lv in h.levels] == meta["n_edges"]
    assert [lv.A_e.nnz for lv in h.levels] == meta["nnz_A_e"]
    assert abs(h.operator_complexity - meta["operator_complexity"]) < 1e-14
    for li, (lv, L) in enumerate(zip(h.levels, meta["levels"])):
        assert csr_hash(lv.D.to_scipy()) == L["D"], li
        if li > 0:
            # STRUCT + TOL; an exact cancellation that differs by summation
            # order (two entries of 25.9M at 128^3) is accepted as round-off
            # (golden_util.check_coarse_operator)
            As = lv.A_e.to_scipy()
            check_coarse_operator(As, L, arrays, li, "A_e")
            check_coarse_operator(lv.S_e.to_scipy(), L, arrays, li, "S_e", A_struct=As)
        if lv.P_e is None:
            continue
        assert sha(lv.membership.cpu().numpy().astype(np.int64)) == L["membership"], li
        assert float(lv.omega).hex() == L["omega_hex"], li
        assert float(lv.rho).hex() == L["rho_hex"], li
        assert csr_hash(lv.P_n.to_scipy()) == L["P_n"], li
        assert sha(lv.assignment.cpu().numpy().astype(np.int64)) == L["assignment"], li
        assert lv.n_augmented == L["n_augmented"], li
        P = lv.P_e.to_scipy()
        assert pattern_sha(P) == L["P_e_pattern"], li
        check_values(P, arrays, f"L{li}_Pe", L["P_e_fro"])
        dims = sorted([list(k) + [v] for k, v in lv.subproblem_dims.items()])
        assert dims == L["subproblem_dims"], li
        assert np.allclose(lv.emin_energy, L["emin_energy"], rtol=1e-10, atol=0), li
        assert lv.commutator_residual <= 1e-12, li
        if L["n_augmented"]:
            # the appended coarse edges: the last rows of the next level's D
            Dn = h.levels[li + 1].D.to_scipy()
            got = [Dn.indices[Dn.indptr[r]:Dn.indptr[r + 1]].tolist()
                   for r in range(Dn.shape[0] - L["n_augmented"], Dn.shape[0])]
            assert got == L["augmented"], li

    if "cheb" not in meta:
        # the hierarchy goldens are written before the reference's solves
        # (hours on one core at 128^3); every hierarchy check above has run
        pytest.skip(f"golden hier_{name} holds the hierarchy only (no reference solve)")
    b = torch.from_numpy(rhs).cuda()
    ref = meta["cheb"]
    res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    if ref["status"] == "converged":
        assert res.status == "converged"
        assert abs(res.iterations - ref["iterations"]) <= 1, (res.iterations,
                                                              ref["iterations"])
    else:
        # the reference's LU coarsest solve fails here; so does ours in LU
        # mode, while the default coarsest solve converges
        assert res.status == "converged"
        hl = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D,
                                mg.SolverConfig(coarse_size=meta["coarse_size"],
                                                coarse_solver="lu"))
        rl = mg.pcg_solve(hl.levels[0].A_e, b, mg.v_cycle_preconditioner(hl),
                          maxit=ref.get("maxit", 500))
        assert rl.status == ref["status"], (rl.status, ref["status"])
