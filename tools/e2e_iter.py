"""Per-iteration e2e times (host scipy inputs -> host solution) at C2."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_08284_b200 import multigrid as mg
from paper_2506_08284_b200.inputs import make_config
s, rhs, cfg = make_config("C2")
sc = mg.SolverConfig(coarse_size=1000)
import gc
if os.environ.get("NOGC"):
    gc.disable()
ts = []
for k in range(8):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, sc)
    t1 = time.perf_counter()
    r = mg.pcg_solve(h.levels[0].A_e, rhs, mg.v_cycle_preconditioner(h))
    torch.cuda.synchronize(); t2 = time.perf_counter()
    ts.append((round(1e3 * (t1 - t0), 2), round(1e3 * (t2 - t0), 2)))
print(os.environ.get("SPHC_ASYNC_UPLOAD", "1"), "nogc" if os.environ.get("NOGC") else "gc", ts)
