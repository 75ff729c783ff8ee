"""Does a setup+solve step leave device memory behind once its hierarchy is
dropped? Prints allocated / reserved after each step (and with the PCG
graph disabled)."""
import gc, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_08284_b200 import multigrid as mg, device as dv
from paper_2506_08284_b200.inputs import make_config
s, rhs, cfg = make_config("C2")
A_e, S, A_n, D = (dv.DeviceCSR.from_scipy(M) for M in (s.A_e, s.S, s.A_n, s.D))
b = torch.from_numpy(rhs).cuda()
sc = mg.SolverConfig(coarse_size=1000)
for mode in ("setup", "setup+solve"):
    for k in range(6):
        h = mg.build_hierarchy(A_e, S, A_n, D, sc)
        if mode != "setup":
            res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
            res = None
        h = None
        gc.collect()
        torch.cuda.synchronize()
        print(mode, k, "allocated", torch.cuda.memory_allocated(), "reserved",
              torch.cuda.memory_reserved(), flush=True)
