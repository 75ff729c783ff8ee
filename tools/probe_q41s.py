import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from golden_util import load_case, stored_inputs
from paper_2506_08284_b200 import multigrid as mg, device as dv
meta, arrays = load_case("Q41s")
A_e, S, A_n, D, rhs = stored_inputs(arrays)
h = mg.build_hierarchy(A_e, S, A_n, D, mg.SolverConfig(coarse_size=meta["coarse_size"]))
Ac = h.levels[-1].A_e.to_scipy().toarray()
lam = np.linalg.eigvalsh(0.5 * (Ac + Ac.T))
print("coarsest n", Ac.shape, "eig min/max", lam[:4], lam[-1])
d = np.diag(Ac); sc = 1 / np.sqrt(d); As = sc[:, None] * Ac * sc[None, :]
ls = np.linalg.eigvalsh(0.5 * (As + As.T)); print("equilibrated eigs lowest", ls[:5], "max", ls[-1])
inv = h.coarse_factorization.cpu().numpy()
print("inv finite", np.isfinite(inv).all(), "max|inv|", np.abs(inv).max(), "sym defect", np.abs(inv - inv.T).max())
li = np.linalg.eigvalsh(0.5 * (inv + inv.T)); print("inv eigs min/max", li[0], li[-1])
b = torch.from_numpy(rhs).cuda()
res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h), maxit=60)
print("device default:", res.status, res.iterations, res.residual_history[:6], res.precond_history[:4])
# replace the coarse inverse by the pseudo-inverse
pin = np.linalg.pinv(0.5 * (Ac + Ac.T), rcond=1e-12, hermitian=True)
h.coarse_factorization = torch.from_numpy(pin).cuda()
h._pcg_ws = None
res2 = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h), maxit=60)
print("pinv coarse:", res2.status, res2.iterations)
hl = mg.build_hierarchy(A_e, S, A_n, D, mg.SolverConfig(coarse_size=meta["coarse_size"], coarse_solver="lu"))
res3 = mg.pcg_solve(hl.levels[0].A_e, b, mg.v_cycle_preconditioner(hl), maxit=60)
print("device lu:", res3.status, res3.iterations)
