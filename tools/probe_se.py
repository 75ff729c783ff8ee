import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np
from paper_2506_08284_b200 import multigrid as mg, device as dv
from paper_2506_08284_b200.assembly import make_device_config
s, rhs, cfg = make_device_config("C4", None)
h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=1000))
for li, lv in enumerate(h.levels):
    v = lv.S_e.val
    mx = float(v.abs().max())
    print(li, lv.A_e.nnz, lv.S_e.nnz, "zeros", int((v == 0).sum()), "tiny<1e-12max", int((v.abs() < 1e-12 * mx).sum()), "max", mx)
