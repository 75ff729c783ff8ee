import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_08284_b200 import multigrid as mg
from paper_2506_08284_b200.inputs import discretize_hex
N = int(sys.argv[1]) if len(sys.argv) > 1 else 4
dirich = bool(int(sys.argv[2])) if len(sys.argv) > 2 else False
cs = int(sys.argv[3]) if len(sys.argv) > 3 else 40
s = discretize_hex(N, 1.0, dirich)
h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=cs))
torch.cuda.synchronize()
print("levels", [lv.A_e.shape[0] for lv in h.levels])
b = np.random.default_rng(0).uniform(-1, 1, s.A_e.shape[0])
r = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
print(r.iterations, r.status)
