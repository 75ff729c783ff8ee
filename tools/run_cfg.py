"""Setup + solve of a named config at several sizes on the GPU (iterations, times)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_08284_b200 import multigrid as mg
from paper_2506_08284_b200.inputs import make_config
name = sys.argv[1]
for N in [int(a) for a in sys.argv[2:]]:
    s, rhs, cfg = make_config(name, N)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=1000))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    r = mg.pcg_solve(h.levels[0].A_e, rhs, mg.v_cycle_preconditioner(h))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    naug = [lv.n_augmented for lv in h.levels]
    print("peak GB", torch.cuda.max_memory_allocated() / 1e9, "reserved GB", torch.cuda.max_memory_reserved() / 1e9)
    print(name, N, [lv.A_e.shape[0] for lv in h.levels], "aug", naug, "its", r.iterations, r.status,
          f"relres {r.relative_residual:.2e}", f"setup {1e3*(t1-t0):.0f} ms solve {1e3*(t2-t1):.0f} ms",
          "hist", [f"{x:.2e}" for x in r.residual_history[::max(1, len(r.residual_history)//8)]], flush=True)
