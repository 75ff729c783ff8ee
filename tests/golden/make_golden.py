"""Generate the golden fixtures from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

The script re-executes itself with ``OPENBLAS_CORETYPE=Haswell
OPENBLAS_NUM_THREADS=1`` (the reference's hierarchy depends on
the BLAS kernel behind np.linalg.norm) and imports the unmodified reference
from /root/reference/pkg/src. Nothing under tests/ reads /root/reference at
test time; the tests only read the files written here:

* ``inputs.json``  -- sha256 of the reference-assembled (A_e, S, A_n, D) arrays
  for a grid of (N, dirichlet, sigma) cases;
* ``hier_<case>.npz`` / ``hier_<case>.json`` -- per-level hierarchy outputs of
  ``build_hierarchy`` (membership, omega/rho bits, P_n, P_const assignment,
  coarse edges, P_e, energies, commutator residual, subproblem dims, coarse
  operators) and PCG results with the reference's Gauss-Seidel sweeper and with
  the oracle's Chebyshev sweeper installed in the reference hierarchy's own
  sweeper slots (multigrid.py:79-80). Large cases store hashes + samples.
"""

import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))

if os.environ.get("OPENBLAS_CORETYPE") != "Haswell" or \
        os.environ.get("OPENBLAS_NUM_THREADS") != "1":
    env = dict(os.environ, OPENBLAS_CORETYPE="Haswell", OPENBLAS_NUM_THREADS="1")
    os.execve(sys.executable, [sys.executable] + sys.argv, env)

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import scipy.sparse as sp  # noqa: E402

from hcurlamg.assembly import discretize  # noqa: E402
from hcurlamg.meshing import build_structured_mesh  # noqa: E402
from hcurlamg import multigrid as mg  # noqa: E402

from oracle.hcurl_oracle import ChebyshevSweeper  # noqa: E402


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def csr_hash(A):
    A = sp.csr_matrix(A)
    return sha(A.indptr.astype(np.int64), A.indices.astype(np.int64),
               A.data.astype(np.float64))


def inputs_table():
    out = {}
    for N in (2, 3, 4, 6, 8, 16, 32):
        for dirichlet in (False, True):
            for sigma in (1.0, 1e-2, 1e-4):
                m = build_structured_mesh(3, "hex", N + 1, dirichlet)
                s = discretize(m, sigma)
                out[f"{N}_{int(dirichlet)}_{sigma!r}"] = {
                    k: csr_hash(getattr(s, k)) for k in ("A_e", "S", "A_n", "D")}
    return out


CASES = {
    # name: (N, dirichlet, sigma, coarse_size, rhs_seed, full arrays?)
    "N4n": (4, False, 1.0, 40, 0, True),
    "N6d": (6, True, 1.0, 40, 0, True),
    "N8d": (8, True, 1.0, 200, 0, True),
    "N10n": (10, False, 1e-4, 100, 5, True),
    "C1": (16, True, 1.0, 1000, 0, True),
    "N16n": (16, False, 1e-2, 200, 1, False),
    "C2": (32, True, 1e-2, 1000, 1, False),
    # RSAMG baseline mode (EminConfig(mode="rsamg"), edge_prolongator.py:200-213)
    "R8d": (8, True, 1.0, 100, 0, True, "rsamg"),
    "R12n": (12, False, 1e-2, 100, 2, True, "rsamg"),
    "R16d": (16, True, 1.0, 200, 0, True, "rsamg"),
}

# relaxation-only mode (multigrid.py:198-207): PCG preconditioned by one
# stand-alone Hiptmair sweep on the fine level; (N, dirichlet, sigma, seed)
RELAX = {
    "X8d": (8, True, 1e-2, 0),
    "X12n": (12, False, 1.0, 3),
}


def run_case(name, N, dirichlet, sigma, coarse_size, seed, full, mode="sphcurl"):
    from hcurlamg.edge_prolongator import EminConfig
    m = build_structured_mesh(3, "hex", N + 1, dirichlet)
    s = discretize(m, sigma)
    cfg = mg.SolverConfig(coarse_size=coarse_size, emin=EminConfig(mode=mode))
    t0 = time.perf_counter()
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, cfg)
    t_setup = time.perf_counter() - t0
    b = np.random.default_rng(seed).uniform(-1.0, 1.0, s.A_e.shape[0])
    t0 = time.perf_counter()
    res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    t_solve = time.perf_counter() - t0

    meta = {"N": N, "dirichlet": dirichlet, "sigma": sigma,
            "coarse_size": coarse_size, "seed": seed, "mode": mode,
            "t_setup_ref": t_setup, "t_solve_ref": t_solve,
            "n_levels": h.n_levels,
            "n_edges": [lv.A_e.shape[0] for lv in h.levels],
            "nnz_A_e": [int(lv.A_e.nnz) for lv in h.levels],
            "operator_complexity": h.operator_complexity,
            "gs": {"iterations": res.iterations, "status": res.status,
                   "residual_history": res.residual_history,
                   "precond_history": res.precond_history,
                   "relative_residual": res.relative_residual},
            "levels": []}
    arrays = {}
    if full:
        arrays["gs_x"] = res.x
    for li, lv in enumerate(h.levels):
        L = {"n_edges": lv.A_e.shape[0], "n_nodes": lv.D.shape[1],
             "A_e": csr_hash(lv.A_e), "S_e": csr_hash(lv.S_e),
             "D": csr_hash(lv.D), "nodal_aux_nnz": int(lv.nodal_aux.nnz),
             "A_e_nnz": int(lv.A_e.nnz), "S_e_nnz": int(lv.S_e.nnz)}
        if lv.P_e is not None:
            L.update({
                "P_e_nnz": int(lv.P_e.nnz),
                "P_e_pattern": sha(lv.P_e.indptr.astype(np.int64),
                                   lv.P_e.indices.astype(np.int64)),
                "P_e_fro": float(np.linalg.norm(lv.P_e.data)),
                "P_n": csr_hash(lv.P_n), "P_n_nnz": int(lv.P_n.nnz),
                "emin_energy": lv.emin_energy,
                "commutator_residual": lv.commutator_residual,
                "subproblem_dims": sorted([list(k) + [v] for k, v in
                                           lv.subproblem_dims.items()]),
                "n_augmented": lv.n_augmented,
            })
            # P_e sample rows (TOL check on big cases)
            step = max(1, lv.P_e.shape[0] // 500)
            rows = np.arange(0, lv.P_e.shape[0], step)
            sub = lv.P_e[rows]
            arrays[f"L{li}_Pe_sample_rows"] = rows
            arrays[f"L{li}_Pe_sample_indptr"] = sub.indptr
            arrays[f"L{li}_Pe_sample_indices"] = sub.indices
            arrays[f"L{li}_Pe_sample_data"] = sub.data
            if full:
                for key, M in (("P_n", lv.P_n), ("P_e", lv.P_e)):
                    arrays[f"L{li}_{key}_indptr"] = M.indptr
                    arrays[f"L{li}_{key}_indices"] = M.indices
                    arrays[f"L{li}_{key}_data"] = M.data
        nxt = h.levels[li + 1] if li + 1 < h.n_levels else None
        if not full and lv.P_e is not None:
            # values only (the patterns are pinned by sha256): every entry of
            # the prolongator and of the next level's coarse operators
            _store_values(arrays, f"L{li}_Pe", lv.P_e, None)
            _store_values(arrays, f"L{li + 1}_A_e", nxt.A_e, None)
            _store_values(arrays, f"L{li + 1}_S_e", nxt.S_e, None)
            L["next_A_e_pattern"] = sha(nxt.A_e.indptr.astype(np.int64),
                                        nxt.A_e.indices.astype(np.int64))
            L["next_S_e_pattern"] = sha(nxt.S_e.indptr.astype(np.int64),
                                        nxt.S_e.indices.astype(np.int64))
        if full:
            if nxt is not None:
                for key, M in (("A_e", nxt.A_e), ("S_e", nxt.S_e), ("D", nxt.D)):
                    arrays[f"L{li + 1}_{key}_indptr"] = M.indptr
                    arrays[f"L{li + 1}_{key}_indices"] = M.indices
                    arrays[f"L{li + 1}_{key}_data"] = M.data
        meta["levels"].append(L)

    # discrete decisions of each prolongator build, recomputed with the
    # reference's own module functions on the level's inputs
    from hcurlamg import nodal_amg as na, coarse_gradient as cgm
    for li, lv in enumerate(h.levels[:-1]):
        strength = na.strength_graph(_an(h, li, s), 0.0)
        agg = na.aggregate(strength)
        if mode == "rsamg":
            nod = na.NodalProlongator(P=na.tentative_prolongator(agg), omega_used=0.0,
                                      rho_estimate=0.0)
        else:
            nod = na.smooth_and_normalize(_an(h, li, s), na.tentative_prolongator(agg))
        assert (nod.P != lv.P_n).nnz == 0
        Pc = cgm.gen_piecewise_const(nod.P, 2)
        assign = Pc.indices[Pc.indptr[:-1]].astype(np.int64)
        cg = cgm.build_coarse_gradient(lv.D, Pc)
        cg = cgm.augment_dirichlet_edges(cg, lv.D, Pc)
        pairs = np.array([e for e in cg.edge_endpoints if len(e) == 2],
                         dtype=np.int64).reshape(-1, 2)
        singles = np.array([e[0] for e in cg.edge_endpoints if len(e) == 1],
                           dtype=np.int64)
        Lm = meta["levels"][li]
        Lm.update({"n_agg": agg.n_agg, "membership": sha(agg.membership.astype(np.int64)),
                   "omega_hex": float(nod.omega_used).hex(),
                   "rho_hex": float(nod.rho_estimate).hex(),
                   "assignment": sha(assign), "pairs": sha(pairs),
                   "singles": sha(singles), "n_pairs": int(pairs.shape[0]),
                   "n_singles": int(singles.size)})
        arrays[f"L{li}_membership"] = agg.membership.astype(np.int32)
        arrays[f"L{li}_assignment"] = assign.astype(np.int32)
        arrays[f"L{li}_pairs"] = pairs.astype(np.int32)
        arrays[f"L{li}_singles"] = singles.astype(np.int32)

    # Chebyshev-3 sweeper in the reference hierarchy's own seam
    for lv in h.levels[:-1]:
        lv.edge_sweeper = ChebyshevSweeper(lv.A_e, 3)
        lv.aux_sweeper = ChebyshevSweeper(lv.nodal_aux, 3)
    t0 = time.perf_counter()
    rc = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    meta["cheb"] = {"iterations": rc.iterations, "status": rc.status,
                    "residual_history": rc.residual_history,
                    "precond_history": rc.precond_history,
                    "relative_residual": rc.relative_residual,
                    "t_solve_ref": time.perf_counter() - t0}
    if full:
        arrays["cheb_x"] = rc.x
    return meta, arrays


_AN_CACHE = {}


def _an(h, li, s):
    """A_n of level li (the reference does not keep it; recompute)."""
    key = id(h)
    if key not in _AN_CACHE:
        An = [sp.csr_matrix(s.A_n)]
        for lv in h.levels[:-1]:
            P = lv.P_n
            C = sp.csr_matrix(P.T @ (An[-1] @ P))
            C.sum_duplicates()
            C.sort_indices()
            C.eliminate_zeros()
            An.append(C)
        _AN_CACHE[key] = An
    return _AN_CACHE[key][li]


def relax_case(N, dirichlet, sigma, seed):
    """Relaxation-only PCG: hiptmair_preconditioner(fine_level(A_e, S, D))
    (multigrid.py:198-207) with the reference's Gauss-Seidel sweeps."""
    m = build_structured_mesh(3, "hex", N + 1, dirichlet)
    s = discretize(m, sigma)
    lv = mg.fine_level(s.A_e, s.S, s.D)
    b = np.random.default_rng(seed).uniform(-1.0, 1.0, s.A_e.shape[0])
    res = mg.pcg_solve(lv.A_e, b, mg.hiptmair_preconditioner(lv))
    meta = {"N": N, "dirichlet": dirichlet, "sigma": sigma, "seed": seed,
            "n_edges": int(s.A_e.shape[0]), "nodal_aux_nnz": int(lv.nodal_aux.nnz),
            "iterations": res.iterations, "status": res.status,
            "residual_history": res.residual_history,
            "precond_history": res.precond_history,
            "relative_residual": res.relative_residual}
    return meta, {"x": res.x}


def error_cases():
    """Reference raising on a degenerate coarse level."""
    out = {}
    m = build_structured_mesh(3, "hex", 9, True)
    s = discretize(m, 1.0)
    try:
        mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=100))
        out["N8d_cs100"] = None
    except ValueError as e:
        out["N8d_cs100"] = str(e)
    # Algorithm 1's safeguard failing (coarse_gradient.py:90-96): a strength
    # threshold that leaves a coarse node with no donor row
    from hcurlamg.edge_prolongator import EminConfig
    try:
        mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D,
                           mg.SolverConfig(coarse_size=100, emin=EminConfig(drop_tol=0.25)))
        out["N8d_droptol025"] = None
    except ValueError as e:
        out["N8d_droptol025"] = str(e)
    return out


def error_input_cases():
    """Every case of tests/error_inputs.py on the unmodified reference."""
    from types import SimpleNamespace
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import error_inputs
    from hcurlamg import nodal_amg as na, coarse_gradient as cgm, emin_setup as es
    from hcurlamg import edge_prolongator as epm
    m = SimpleNamespace(na=na, cgm=cgm, es=es, epm=epm, mg=mg)
    s = discretize(build_structured_mesh(3, "hex", 5, False), 1.0)
    return {name: error_inputs.run(m, s, name) for name in error_inputs.CASES}


def edge_case_results():
    """Every case of tests/edge_cases.py on the unmodified reference."""
    from types import SimpleNamespace
    sys.path.insert(0, os.path.join(REPO, "tests"))
    import edge_cases
    m = SimpleNamespace(
        mg=mg, config=lambda **kw: mg.SolverConfig(**kw),
        system=lambda N, sigma, dirichlet: discretize(
            build_structured_mesh(3, "hex", N + 1, dirichlet), sigma))
    return {name: edge_cases.run(m, name) for name in edge_cases.CASES}


def repair_case():
    """make_irreducible exercised through the reference's own setup_constraints:
    level-0 inputs of N=10 Dirichlet with every 17th interior coarse edge
    removed from the coarse gradient, so some constraint blocks are reducible
    (or empty) and the reference appends coarse edges (emin_setup.py:183-336)."""
    from hcurlamg import nodal_amg as na, coarse_gradient as cgm, emin_setup as es
    from hcurlamg import edge_prolongator as epm
    m = build_structured_mesh(3, "hex", 11, True)
    s = discretize(m, 1.0)
    agg = na.aggregate(na.strength_graph(s.A_n, 0.0))
    nod = na.smooth_and_normalize(s.A_n, na.tentative_prolongator(agg))
    Pc = cgm.gen_piecewise_const(nod.P, 2)
    cg = cgm.augment_dirichlet_edges(cgm.build_coarse_gradient(s.D, Pc), s.D, Pc)
    pairs = [e for e in cg.edge_endpoints if len(e) == 2]
    singles = [e for e in cg.edge_endpoints if len(e) == 1]
    keep = [p for k, p in enumerate(pairs) if k % 17 != 3]
    eps = keep + singles
    cg_r = cgm.CoarseGradient(D_H=cgm._gradient_from_endpoints(eps, cg.n_nodes),
                              edge_endpoints=eps)
    setup = es.setup_constraints(s.D, nod.P, cg_r)
    structure, values = epm.initial_feasible_guess(setup)
    P = structure.matrix(values)
    dims = epm.Counter((r.coarse_edges.size, r.coarse_nodes.size)
                       for r in setup.rows if r is not None)
    meta = {"n_nodes": cg.n_nodes, "n_augmented": setup.n_augmented,
            "augmented": [list(e) for e in setup.cg.edge_endpoints[len(eps):]],
            "dims": sorted([list(k) + [v] for k, v in dims.items()])}
    arrays = {"pairs": np.array(keep, dtype=np.int64), "singles":
              np.array([e[0] for e in singles], dtype=np.int64),
              "P_indptr": P.indptr, "P_indices": P.indices, "P_data": P.data}
    return meta, arrays


# Device-generated configs: the inputs are
# built by the host build of the device assembly rows (oracle/host_assembly.py,
# bit-identical to assembly.make_device_config on the B200, recorded by sha256),
# and the UNMODIFIED reference is run on them. Values of the prolongators and
# coarse operators are stored in full up to ``limit`` entries per matrix, else
# on every k-th row (k = ceil(nnz / limit)); patterns by sha256.
BIG = {
    # name: (config, N, coarse_size, value limit per matrix, run GS solve
    #        [, maxit of the Chebyshev-seam solve])
    "C4s": ("C4", 16, 200, None, True),
    "C3": ("C3", 64, 1000, 1_000_000, True),
    "C5s": ("C5", 64, 1000, 1_000_000, True),
    "C4r": ("C4", 128, 1000, 500_000, True),
    # the C4 recipe again without the Gauss-Seidel solve and with the
    # Chebyshev-seam solve capped at 250 iterations (the reference's LU
    # coarsest solve does not converge there: one V-cycle PCG iteration is
    # ~30 s on one core)
    "C4rh": ("C4", 128, 1000, 500_000, False, 250),
}


def _store_values(arrays, key, M, limit):
    M = sp.csr_matrix(M)
    k = 1 if limit is None else max(1, -(-int(M.nnz) // int(limit)))
    rows = np.arange(0, M.shape[0], k)
    arrays[key + "_stride"] = np.array(k, dtype=np.int64)
    if k == 1:
        arrays[key + "_vals"] = M.data
    else:
        ln = np.diff(M.indptr)[rows]
        idx = np.repeat(M.indptr[rows], ln) + (np.arange(int(ln.sum()))
                                               - np.repeat(np.cumsum(ln) - ln, ln))
        arrays[key + "_vals"] = M.data[idx]


def _write_case(name, meta, arrays):
    with open(os.path.join(HERE, f"hier_{name}.json"), "w") as f:
        json.dump(meta, f, indent=1)
    np.savez_compressed(os.path.join(HERE, f"hier_{name}.npz"), **arrays)


# Other element families of the reference (meshing.py:15 SUPPORTED: quad, tri,
# hex, tet): the unmodified reference on its own meshes and assembly. The hot
# path only sees (A_e, S, A_n, D), so the INPUTS are stored with the golden
# (the repo's generators are hex only) and the tests upload them as they are.
MESH = {
    # name: (dim, kind, nodal shape, dirichlet, sigma, coarse_size, rhs seed)
    "T9n": (3, "tet", 9, False, 1.0, 100, 11),
    "T8d": (3, "tet", 8, True, 1e-2, 100, 12),
    "Q41d": (2, "quad", 41, True, 1.0, 500, 13),
    "R33n": (2, "tri", 33, False, 1e-2, 100, 14),
    # Q41d coarsened once more: the 64-edge coarsest operator is singular in
    # exact arithmetic (the reference's LU meets a round-off pivot and still
    # converges; the oracle's meets an exact zero) -- the device's coarsest
    # solve takes its breakdown fallback here
    "Q41s": (2, "quad", 41, True, 1.0, 100, 13),
}


# Non-default knobs of the path (EminConfig: omega, iterations, n_passes,
# drop_tol -- edge_prolongator.py:28-44; SolverConfig.max_levels --
# multigrid.py:23-30) on small hex meshes, inputs stored like MESH.
VARIANTS = {
    # name: (nodal shape, dirichlet, sigma, coarse_size, seed, emin kwargs, max_levels)
    "V9a": (9, False, 1e-2, 100, 21, dict(iterations=3, omega=0.7), 10),
    "V9b": (9, True, 1.0, 100, 22, dict(drop_tol=0.05), 10),
    "V9e": (9, False, 1.0, 100, 25, dict(n_passes=1), 10),
    "V11c": (11, False, 1.0, 100, 23, dict(n_passes=3, iterations=0), 10),
    "V9d": (9, True, 1e-4, 50, 24, dict(iterations=2, omega=1.2), 2),
}


def run_variant_case(name, shape, dirichlet, sigma, coarse_size, seed, emin, max_levels):
    m = build_structured_mesh(3, "hex", shape, dirichlet)
    sysm = discretize(m, sigma)
    rhs = np.random.default_rng(seed).uniform(-1.0, 1.0, sysm.A_e.shape[0])
    inputs = (sp.csr_matrix(sysm.A_e), sp.csr_matrix(sysm.S), sp.csr_matrix(sysm.A_n),
              sp.csr_matrix(sysm.D), rhs,
              {"dirichlet": dirichlet, "dim": 3, "kind": "hex", "shape": shape,
               "sigma": sigma, "seed": seed})
    return run_device_case(name, "hex3d", shape, coarse_size, None, True, inputs=inputs,
                           emin=emin, max_levels=max_levels)


def run_mesh_case(name, dim, kind, shape, dirichlet, sigma, coarse_size, seed):
    m = build_structured_mesh(dim, kind, shape, dirichlet)
    sysm = discretize(m, sigma)
    rhs = np.random.default_rng(seed).uniform(-1.0, 1.0, sysm.A_e.shape[0])
    inputs = (sp.csr_matrix(sysm.A_e), sp.csr_matrix(sysm.S), sp.csr_matrix(sysm.A_n),
              sp.csr_matrix(sysm.D), rhs,
              {"dirichlet": dirichlet, "dim": dim, "kind": kind, "shape": shape,
               "sigma": sigma, "seed": seed})
    return run_device_case(name, f"{kind}{dim}d", shape, coarse_size, None, True,
                           inputs=inputs)


def run_device_case(name, config, N, coarse_size, limit, with_gs, cheb_maxit=500,
                    inputs=None, emin=None, max_levels=10):
    from types import SimpleNamespace
    from hcurlamg import nodal_amg as na, coarse_gradient as cgm
    from hcurlamg.edge_prolongator import EminConfig
    emin = dict(emin or {})
    ecfg = EminConfig(**emin)
    if inputs is None:
        from oracle.host_assembly import config_host
        A_e, S, A_n, D, rhs, cfg = config_host(config, N)
    else:
        A_e, S, A_n, D, rhs, cfg = inputs
    s = SimpleNamespace(A_e=A_e, S=S, A_n=A_n, D=D)
    meta = {"config": config, "N": N, "dirichlet": bool(cfg["dirichlet"]),
            "coarse_size": coarse_size, "limit": limit,
            "inputs": {k: csr_hash(getattr(s, k)) for k in ("A_e", "S", "A_n", "D")},
            "rhs": sha(rhs), "levels": []}
    if inputs is not None:
        meta["mesh"] = cfg
    meta["emin"] = emin
    meta["max_levels"] = max_levels
    t0 = time.perf_counter()
    h = mg.build_hierarchy(A_e, S, A_n, D, mg.SolverConfig(coarse_size=coarse_size,
                                                           max_levels=max_levels, emin=ecfg))
    meta["t_setup_ref"] = time.perf_counter() - t0
    print(name, "setup", meta["t_setup_ref"], "levels", [lv.A_e.shape[0] for lv in h.levels],
          flush=True)
    meta.update({"n_levels": h.n_levels, "operator_complexity": h.operator_complexity,
                 "n_edges": [lv.A_e.shape[0] for lv in h.levels],
                 "nnz_A_e": [int(lv.A_e.nnz) for lv in h.levels]})
    arrays = {}
    if inputs is not None:
        for k in ("A_e", "S", "A_n", "D"):
            M = sp.csr_matrix(getattr(s, k))
            arrays[f"in_{k}_indptr"] = M.indptr.astype(np.int64)
            arrays[f"in_{k}_indices"] = M.indices.astype(np.int32)
            arrays[f"in_{k}_data"] = M.data.astype(np.float64)
            arrays[f"in_{k}_shape"] = np.array(M.shape, dtype=np.int64)
        arrays["in_rhs"] = rhs
    for li, lv in enumerate(h.levels):
        L = {"n_edges": lv.A_e.shape[0], "n_nodes": lv.D.shape[1],
             "A_e": csr_hash(lv.A_e), "S_e": csr_hash(lv.S_e), "D": csr_hash(lv.D),
             "A_e_pattern": sha(lv.A_e.indptr.astype(np.int64),
                                lv.A_e.indices.astype(np.int64)),
             "S_e_pattern": sha(lv.S_e.indptr.astype(np.int64),
                                lv.S_e.indices.astype(np.int64)),
             "A_e_nnz": int(lv.A_e.nnz), "S_e_nnz": int(lv.S_e.nnz),
             "nodal_aux_nnz": int(lv.nodal_aux.nnz)}
        if li > 0:
            _store_values(arrays, f"L{li}_A_e", lv.A_e, limit)
            _store_values(arrays, f"L{li}_S_e", lv.S_e, limit)
            if limit is None:
                # small cases: the patterns themselves, for the rule "equal up to
                # round-off-sized entries" when an exact cancellation differs
                for key, M in (("A_e", lv.A_e), ("S_e", lv.S_e)):
                    M = sp.csr_matrix(M)
                    arrays[f"L{li}_{key}_indptr"] = M.indptr.astype(np.int64)
                    arrays[f"L{li}_{key}_indices"] = M.indices.astype(np.int32)
            L["A_e_fro"] = float(np.linalg.norm(lv.A_e.data))
            L["S_e_fro"] = float(np.linalg.norm(lv.S_e.data))
        if lv.P_e is not None:
            nxt = h.levels[li + 1]
            n_aug = int(lv.n_augmented)
            Dn = sp.csr_matrix(nxt.D)
            aug = [Dn.indices[Dn.indptr[r]:Dn.indptr[r + 1]].tolist()
                   for r in range(Dn.shape[0] - n_aug, Dn.shape[0])]
            L.update({
                "P_e_nnz": int(lv.P_e.nnz),
                "P_e_pattern": sha(lv.P_e.indptr.astype(np.int64),
                                   lv.P_e.indices.astype(np.int64)),
                "P_e_fro": float(np.linalg.norm(lv.P_e.data)),
                "P_n": csr_hash(lv.P_n), "P_n_nnz": int(lv.P_n.nnz),
                "emin_energy": lv.emin_energy,
                "commutator_residual": lv.commutator_residual,
                "subproblem_dims": sorted([list(k) + [v] for k, v in
                                           lv.subproblem_dims.items()]),
                "n_augmented": n_aug, "augmented": aug,
            })
            _store_values(arrays, f"L{li}_Pe", lv.P_e, limit)
        meta["levels"].append(L)

    for li, lv in enumerate(h.levels[:-1]):
        An = _an(h, li, s)
        agg = na.aggregate(na.strength_graph(An, ecfg.drop_tol))
        nod = na.smooth_and_normalize(An, na.tentative_prolongator(agg))
        assert (nod.P != lv.P_n).nnz == 0
        Pc = cgm.gen_piecewise_const(nod.P, ecfg.n_passes)
        assign = Pc.indices[Pc.indptr[:-1]].astype(np.int64)
        cg = cgm.augment_dirichlet_edges(cgm.build_coarse_gradient(lv.D, Pc), lv.D, Pc)
        pairs = np.array([e for e in cg.edge_endpoints if len(e) == 2],
                         dtype=np.int64).reshape(-1, 2)
        singles = np.array([e[0] for e in cg.edge_endpoints if len(e) == 1],
                           dtype=np.int64)
        meta["levels"][li].update({
            "n_agg": agg.n_agg, "membership": sha(agg.membership.astype(np.int64)),
            "omega_hex": float(nod.omega_used).hex(), "rho_hex": float(nod.rho_estimate).hex(),
            "assignment": sha(assign), "pairs": sha(pairs), "singles": sha(singles),
            "n_pairs": int(pairs.shape[0]), "n_singles": int(singles.size)})
    print(name, "decisions recorded", flush=True)
    # the hierarchy goldens are complete: write them before the solves
    _write_case(name, meta, arrays)

    b = rhs
    if with_gs:
        t0 = time.perf_counter()
        res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
        meta["t_solve_ref"] = time.perf_counter() - t0
        meta["gs"] = {"iterations": res.iterations, "status": res.status,
                      "residual_history": res.residual_history,
                      "relative_residual": res.relative_residual}
        print(name, "gs its", res.iterations, meta["t_solve_ref"], flush=True)
    for lv in h.levels[:-1]:
        lv.edge_sweeper = ChebyshevSweeper(lv.A_e, 3)
        lv.aux_sweeper = ChebyshevSweeper(lv.nodal_aux, 3)
    t0 = time.perf_counter()
    rc = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h), maxit=cheb_maxit)
    meta["cheb"] = {"iterations": rc.iterations, "status": rc.status,
                    "residual_history": rc.residual_history,
                    "relative_residual": rc.relative_residual, "maxit": cheb_maxit,
                    "t_solve_ref": time.perf_counter() - t0}
    print(name, "cheb its", rc.iterations, flush=True)
    return meta, arrays


def pcg_status_cases():
    """The reference's non-converged PCG exits (multigrid.py:244-264) on
    small hierarchies: maxit (maxit=3), stagnated (rtol=0: x stops changing
    at round-off; the last history entry is the true residual) and
    indefinite (the negated operator: p.Ap <= 0 on the first iteration)."""
    out, arrays = {}, {}
    for name, (N, dirich, cs) in {"N4n": (4, False, 40), "N6d": (6, True, 40)}.items():
        s = discretize(build_structured_mesh(3, "hex", N + 1, dirich), 1.0)
        h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=cs))
        b = np.random.default_rng(0).uniform(-1, 1, s.A_e.shape[0])
        M = mg.v_cycle_preconditioner(h)
        for kind, (A, kw) in {"maxit": (h.levels[0].A_e, dict(maxit=3)),
                              "stagnated": (h.levels[0].A_e, dict(rtol=0.0)),
                              "indefinite": (-h.levels[0].A_e, {})}.items():
            r = mg.pcg_solve(A, b, M, **kw)
            out[f"{name}_{kind}"] = {"N": N, "dirichlet": dirich, "coarse_size": cs,
                                     "status": r.status, "iterations": r.iterations,
                                     "residual_history": r.residual_history,
                                     "precond_history": r.precond_history,
                                     "relative_residual": r.relative_residual}
            arrays[f"{name}_{kind}_x"] = r.x
    return out, arrays


def main(which):
    if "repair" in which:
        meta, arrays = repair_case()
        with open(os.path.join(HERE, "repair_N10d.json"), "w") as f:
            json.dump(meta, f, indent=1)
        np.savez_compressed(os.path.join(HERE, "repair_N10d.npz"), **arrays)
        print("repair case: n_augmented", meta["n_augmented"])
    if "pcg_status" in which:
        meta, arrays = pcg_status_cases()
        with open(os.path.join(HERE, "pcg_status.json"), "w") as f:
            json.dump(meta, f, indent=1)
        np.savez_compressed(os.path.join(HERE, "pcg_status.npz"), **arrays)
        print("pcg status cases", {k: (v["status"], v["iterations"]) for k, v in meta.items()})
    if "edge_cases" in which:
        with open(os.path.join(HERE, "edge_cases.json"), "w") as f:
            json.dump(edge_case_results(), f, indent=1)
    if "error_inputs" in which:
        with open(os.path.join(HERE, "error_inputs.json"), "w") as f:
            json.dump(error_input_cases(), f, indent=1)
    if "errors" in which:
        with open(os.path.join(HERE, "errors.json"), "w") as f:
            json.dump(error_cases(), f, indent=1)
    for name, spec in RELAX.items():
        if which and name not in which:
            continue
        meta, arrays = relax_case(*spec)
        with open(os.path.join(HERE, f"relax_{name}.json"), "w") as f:
            json.dump(meta, f, indent=1)
        np.savez_compressed(os.path.join(HERE, f"relax_{name}.npz"), **arrays)
        print(name, "relaxation-only its", meta["iterations"], flush=True)
    if "inputs" in which:
        with open(os.path.join(HERE, "inputs.json"), "w") as f:
            json.dump(inputs_table(), f, indent=1, sort_keys=True)
        print("inputs.json written")
    for name, spec in MESH.items():
        if which and name not in which:
            continue
        meta, arrays = run_mesh_case(name, *spec)
        _write_case(name, meta, arrays)
        print(name, "levels", meta["n_edges"], "gs", meta["gs"]["iterations"],
              meta["gs"]["status"], "cheb", meta["cheb"]["iterations"], meta["cheb"]["status"],
              flush=True)
    for name, spec in VARIANTS.items():
        if which and name not in which:
            continue
        meta, arrays = run_variant_case(name, *spec)
        _write_case(name, meta, arrays)
        print(name, "levels", meta["n_edges"], "gs", meta["gs"]["iterations"],
              meta["gs"]["status"], "cheb", meta["cheb"]["iterations"], meta["cheb"]["status"],
              flush=True)
    for name, spec in BIG.items():
        if name not in which:           # only on request (minutes to hours)
            continue
        meta, arrays = run_device_case(name, *spec)
        _write_case(name, meta, arrays)
        print(name, "written", flush=True)
    for name, spec in CASES.items():
        if which and name not in which:
            continue
        t0 = time.perf_counter()
        meta, arrays = run_case(name, *spec)
        with open(os.path.join(HERE, f"hier_{name}.json"), "w") as f:
            json.dump(meta, f, indent=1)
        np.savez_compressed(os.path.join(HERE, f"hier_{name}.npz"), **arrays)
        print(name, "levels", meta["n_edges"], "gs its", meta["gs"]["iterations"],
              "cheb its", meta["cheb"]["iterations"],
              f"{time.perf_counter() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main(set(sys.argv[1:]) or set(["inputs", "errors", "error_inputs", "edge_cases", "repair", "pcg_status"] + list(CASES) + list(RELAX)
                                  + list(MESH) + list(VARIANTS)))
