import os, sys, cProfile, pstats, io
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_08284_b200 import multigrid as mg, device as dv
from paper_2506_08284_b200.inputs import make_config
cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
s, rhs, cfg = make_config(cfgname)
A_e, S, A_n, D = (dv.DeviceCSR.from_scipy(M) for M in (s.A_e, s.S, s.A_n, s.D))
b = torch.from_numpy(rhs).cuda()
sc = mg.SolverConfig(coarse_size=1000)
for _ in range(3):
    h = mg.build_hierarchy(A_e, S, A_n, D, sc); r = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for _ in range(3):
    h = mg.build_hierarchy(A_e, S, A_n, D, sc)
    torch.cuda.synchronize()
pr.disable()
st = io.StringIO(); pstats.Stats(pr, stream=st).sort_stats("tottime").print_stats(25); print(st.getvalue()[:6000])
