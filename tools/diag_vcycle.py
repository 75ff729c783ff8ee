"""V-cycle symmetry / definiteness diagnostics on a config's GPU hierarchy."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_08284_b200 import multigrid as mg, device as dv
from paper_2506_08284_b200.inputs import make_config
name, N = sys.argv[1], int(sys.argv[2])
s, rhs, cfg = make_config(name, N)
h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=1000))
Ac = dv.to_dense(h.levels[-1].A_e)
print("coarsest n", Ac.shape[0], "cond", float(torch.linalg.cond(Ac)), "asym", float((Ac - Ac.T).abs().max() / Ac.abs().max()))
ev = torch.linalg.eigvalsh(0.5 * (Ac + Ac.T))
print("coarse eig min/max", float(ev.min()), float(ev.max()))
inv = h.coarse_factorization
print("inv asym", float((inv - inv.T).abs().max() / inv.abs().max()))
for li, lv in enumerate(h.levels):
    A = lv.A_e.to_scipy()
    print("level", li, "A asym", abs(A - A.T).max() / abs(A).max(), "S asym", abs(lv.S_e.to_scipy() - lv.S_e.to_scipy().T).max() / abs(lv.S_e.to_scipy()).max())
pre = mg.v_cycle_preconditioner(h)
n = s.A_e.shape[0]
g = torch.Generator(device="cuda").manual_seed(0)
for t in range(3):
    b1 = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) - 0.5
    b2 = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) - 0.5
    v1 = pre(b1).clone(); v2 = pre(b2).clone()
    print("sym", float(v1 @ b2), float(b1 @ v2), "pd", float(v1 @ b1), float(v2 @ b2))
# level-wise: two-level check with exact coarse solve replaced by numpy LU
import scipy.linalg as la
lu = la.lu_factor(Ac.cpu().numpy())
x = np.random.default_rng(0).standard_normal(Ac.shape[0])
y_inv = (inv.cpu().numpy() @ x); y_lu = la.lu_solve(lu, x)
print("inv vs lu rel", np.abs(y_inv - y_lu).max() / np.abs(y_lu).max())
