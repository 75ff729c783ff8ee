"""Coarsest solve: the reference's LU vs the equilibrated Cholesky inverse,
on the device-generated recipes (iterations, status, time)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_08284_b200 import multigrid as mg
from paper_2506_08284_b200.assembly import make_device_config
for spec in sys.argv[1:]:
    cfgname, N, cs = spec.split(":")
    s, rhs, cfg = make_device_config(cfgname, int(N))
    b = torch.from_numpy(rhs).cuda()
    for solver in ("lu", "cholesky"):
        t0 = time.perf_counter()
        h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D,
                               mg.SolverConfig(coarse_size=int(cs), coarse_solver=solver))
        r = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
        torch.cuda.synchronize()
        print(spec, solver, "levels", [lv.A_e.shape[0] for lv in h.levels], "its", r.iterations,
              r.status, f"relres {r.relative_residual:.2e}", f"{time.perf_counter()-t0:.2f}s",
              flush=True)
        del h
    del s
    torch.cuda.empty_cache()
