"""Convergence diagnostics of a device-assembled config: sizes, iterations,
coarsest spectrum (raw and Jacobi-scaled), rank of the small prolongators."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_08284_b200 import multigrid as mg, device as dv
from paper_2506_08284_b200.assembly import make_device_config
name = sys.argv[1]
for spec in sys.argv[2:]:
    N, cs = (int(x) for x in spec.split(":"))
    s, rhs, cfg = make_device_config(name, N)
    b = torch.from_numpy(rhs).cuda()
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=cs))
    Ad = dv.to_dense(h.levels[-1].A_e)
    A = 0.5 * (Ad + Ad.T)
    Ds = torch.diagonal(A).rsqrt()
    lam = torch.linalg.eigvalsh(Ds[:, None] * A * Ds[None, :]) if A.shape[0] < 12000 else torch.zeros(2, dtype=A.dtype)
    print("   coarsest zero diag", int((torch.diagonal(A) == 0).sum()), "n_aug", [lv.n_augmented for lv in h.levels], flush=True)
    r = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h), maxit=300)
    his = r.residual_history
    print(name, N, "coarse_size", cs, [lv.A_e.shape[0] for lv in h.levels], "its", r.iterations, r.status,
          f"relres {r.relative_residual:.2e}", f"scaled coarse eig [{lam[0].item():.2e}, {lam[-1].item():.2e}]",
          "bounds", [(round(lv.edge_sweeper.hi, 2), round(lv.aux_sweeper.hi, 2)) for lv in h.levels[:-1]], flush=True)
    for i, lv in enumerate(h.levels[:-1]):
        if lv.P_e.shape[1] <= 5000:
            sv = torch.linalg.svdvals(dv.to_dense(lv.P_e))
            Pd = dv.to_dense(lv.P_e)
            zc = int((Pd.abs().sum(0) == 0).sum())
            nsmall = int((sv < 1e-10 * sv[0]).sum())
            print(f"   P_e[{i}] {tuple(lv.P_e.shape)} sv [{sv[-1].item():.2e}, {sv[0].item():.2e}] #sv<1e-10: {nsmall} zero cols {zc} max|P| {lv.P_e.val.abs().max().item():.2f}", flush=True)
    print("   hist", [f"{x:.1e}" for x in his[::max(1, len(his)//12)]], flush=True)
    del h
