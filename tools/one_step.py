"""One warm-up + one measured setup+solve step (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_08284_b200 import multigrid as mg, device as dv, _lib
from paper_2506_08284_b200.inputs import make_config
cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
N = int(sys.argv[2]) if len(sys.argv) > 2 else None
s, rhs, cfg = make_config(cfgname, N)
A_e, S, A_n, D = (dv.DeviceCSR.from_scipy(M) for M in (s.A_e, s.S, s.A_n, s.D))
b = torch.from_numpy(rhs).cuda()
sc = mg.SolverConfig(coarse_size=1000)
for rep in range(2):
    l0 = _lib.launch_count()
    h = mg.build_hierarchy(A_e, S, A_n, D, sc)
    l1 = _lib.launch_count()
    res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    torch.cuda.synchronize()
    print(f"rep {rep}: setup launches {l1-l0}, solve launches {_lib.launch_count()-l1}, its {res.iterations}", flush=True)
