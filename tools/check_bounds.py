"""Compare the Chebyshev upper bound (15 power steps x 1.1) with a long power
iteration on every smoothed operator of a config's hierarchy."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_08284_b200 import multigrid as mg, device as dv
from paper_2506_08284_b200.inputs import make_config
name, N = sys.argv[1], int(sys.argv[2])
s, rhs, cfg = make_config(name, N)
h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=1000))
def lam(A, dinv, its):
    n = A.shape[0]
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
    x /= x.norm()
    y = torch.empty_like(x)
    l = 0.0
    for _ in range(its):
        dv.spmv(A, x, y); y *= dinv
        l = float(y.norm()); x = y / l
    return l
for li, lv in enumerate(h.levels[:-1]):
    for nm, sw in (("edge", lv.edge_sweeper), ("aux", lv.aux_sweeper)):
        print(li, nm, sw.A.shape[0], "hi", sw.hi, "lam300", lam(sw.A, sw.dinv, 300), flush=True)
