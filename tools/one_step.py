"""One warm-up + one measured setup+solve step (for ncu launch lists and
captures). Device-assembled inputs for C3-C5, host (reference-identical)
inputs uploaded for C1/C2."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_08284_b200 import multigrid as mg, device as dv, _lib
cfgname = sys.argv[1] if len(sys.argv) > 1 else "C4"
N = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
if cfgname in ("C3", "C4", "C5"):
    from paper_2506_08284_b200.assembly import make_device_config
    s, rhs, cfg = make_device_config(cfgname, N)
    A_e, S, A_n, D = s.A_e, s.S, s.A_n, s.D
else:
    from paper_2506_08284_b200.inputs import make_config
    s, rhs, cfg = make_config(cfgname, N)
    A_e, S, A_n, D = (dv.DeviceCSR.from_scipy(M) for M in (s.A_e, s.S, s.A_n, s.D))
b = torch.from_numpy(rhs).cuda()
sc = mg.SolverConfig(coarse_size=cfg.get("coarse_size", 1000))
for rep in range(reps):
    h = res = None
    l0 = _lib.launch_count()
    h = mg.build_hierarchy(A_e, S, A_n, D, sc)
    l1 = _lib.launch_count()
    res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    torch.cuda.synchronize()
    print(f"rep {rep}: setup launches {l1-l0}, solve launches {_lib.launch_count()-l1}, "
          f"its {res.iterations}, levels {[lv.A_e.shape[0] for lv in h.levels]}", flush=True)
