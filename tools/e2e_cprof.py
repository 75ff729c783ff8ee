"""Host-side profile (cProfile) of one e2e step at C2: build_hierarchy from
scipy inputs + pcg_solve with a numpy RHS, after warm-up."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_08284_b200 import multigrid as mg
from paper_2506_08284_b200.inputs import make_config
s, rhs, cfg = make_config("C2")
sc = mg.SolverConfig(coarse_size=1000)
for _ in range(3):
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, sc); r = mg.pcg_solve(h.levels[0].A_e, rhs, mg.v_cycle_preconditioner(h)); h = r = None
torch.cuda.synchronize()
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, sc)
    t1 = time.perf_counter()
    r = mg.pcg_solve(h.levels[0].A_e, rhs, mg.v_cycle_preconditioner(h))
    torch.cuda.synchronize()
    ts.append(((t1 - t0) * 1e3, (time.perf_counter() - t1) * 1e3))
    h = r = None
print("e2e setup/solve ms:", [(round(a, 2), round(b, 2)) for a, b in ts])
pr = cProfile.Profile()
pr.enable()
h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, sc)
r = mg.pcg_solve(h.levels[0].A_e, rhs, mg.v_cycle_preconditioner(h))
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
