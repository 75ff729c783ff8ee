"""Iteration counts of the device-assembled C4 under different smoothers."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_08284_b200 import multigrid as mg
from paper_2506_08284_b200.assembly import make_device_config
N = int(sys.argv[1])
s, rhs, cfg = make_device_config("C4", N)
b = torch.from_numpy(rhs).cuda()
for sm, deg, safety in (("chebyshev", 3, 1.1), ("chebyshev", 4, 1.1), ("chebyshev", 2, 1.1)):
    mg.CHEB_SAFETY = safety
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=1000, smoother=sm, cheb_degree=deg))
    r = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h), maxit=800)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    his = r.residual_history
    print(N, sm, deg, safety, "its", r.iterations, r.status, f"{1e3*(t1-t0):.0f} ms",
          [f"{x:.1e}" for x in his[::max(1, len(his)//10)]], flush=True)
    if sm == "chebyshev":
        print("   bounds", [(round(lv.edge_sweeper.hi, 3), round(lv.aux_sweeper.hi, 3)) for lv in h.levels[:-1]], flush=True)
