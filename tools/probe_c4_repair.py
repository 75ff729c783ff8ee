"""Where does make_irreducible fire on the C4 recipe (jittered hexes,
lognormal sigma, default_rng(3))?  Prints level sizes and n_augmented per
level for a range of N on the device path."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_08284_b200 import multigrid as mg
from paper_2506_08284_b200.assembly import make_device_config
for N in [int(x) for x in sys.argv[1:]]:
    s, rhs, cfg = make_device_config("C4", N)
    b = torch.from_numpy(rhs).cuda()
    t0 = time.perf_counter()
    try:
        h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=1000))
        r = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
        print(N, "levels", [lv.A_e.shape[0] for lv in h.levels],
              "n_aug", [lv.n_augmented for lv in h.levels[:-1]],
              "its", r.iterations, r.status, f"{time.perf_counter()-t0:.2f}s", flush=True)
    except Exception as e:
        print(N, "ERROR", type(e).__name__, e, flush=True)
    del s
    torch.cuda.empty_cache()
