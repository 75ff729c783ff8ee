"""B200-native (sm_100a) SpHcurlAMG hot path: structure-preserving H(curl)
algebraic multigrid setup (constrained energy minimisation of the edge
prolongator, Galerkin products, coarse discrete gradient) and the PCG +
Hiptmair V-cycle solve, behind the reference's Python API.

    from paper_2506_08284_b200 import multigrid as mg
    h = mg.build_hierarchy(A_e, S_e, A_n, D, mg.SolverConfig(coarse_size=1000))
    res = mg.pcg_solve(A_e, b, mg.v_cycle_preconditioner(h), rtol=1e-8)

All numerics run in libsphcurl.so (include/sphcurl.h); there is no CPU path.
"""

__version__ = "0.1.0"
