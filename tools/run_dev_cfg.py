"""Device-assembled config: assembly time, setup + solve (iterations, times, memory)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_08284_b200 import multigrid as mg
from paper_2506_08284_b200.assembly import make_device_config
name = sys.argv[1]
for N in [int(a) for a in sys.argv[2:]]:
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s, rhs, cfg = make_device_config(name, N)
    torch.cuda.synchronize(); ta = time.perf_counter()
    print(name, N, "n_e", s.n_edges, "nnz(A_e)", s.A_e.nnz, "nnz(A_n)", s.A_n.nnz,
          f"assembly+draws {1e3*(ta-t0):.0f} ms", "mem GB", torch.cuda.memory_allocated() / 1e9, flush=True)
    b = torch.from_numpy(rhs).cuda()
    for rep in range(int(os.environ.get("REPS", "2"))):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=1000))
        torch.cuda.synchronize(); t1 = time.perf_counter()
        r = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
        torch.cuda.synchronize(); t2 = time.perf_counter()
        print(name, N, [lv.A_e.shape[0] for lv in h.levels], "aug", [lv.n_augmented for lv in h.levels],
              "its", r.iterations, r.status, f"relres {r.relative_residual:.2e}",
              f"setup {1e3*(t1-t0):.0f} ms solve {1e3*(t2-t1):.0f} ms",
              "peak GB", torch.cuda.max_memory_allocated() / 1e9, flush=True)
        del h, r
