"""Probe (GPU): the device V-cycle's linearity defect in units of the fine
level's rounding, C4 recipe over N (compare tools/probe_vlin_oracle.py)."""
import sys
import torch
from paper_2506_08284_b200 import multigrid as mg
from paper_2506_08284_b200.assembly import make_device_config


def sp(A, absval=False):
    return torch.sparse_csr_tensor(A.rowptr, A.col.to(torch.int64), A.val.abs() if absval else A.val, size=A.shape)


def mv(A, x):
    return (A @ x.unsqueeze(1)).squeeze(1)


def rand(n, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1


for N in [int(a) for a in sys.argv[1:]] or [16]:
    s, rhs, cfg = make_device_config("C4", N)
    for solver in ("cholesky", "lu"):
        h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=1000 if N > 16 else 200, coarse_solver=solver))
        A, Aabs = sp(h.levels[0].A_e), sp(h.levels[0].A_e, True)
        n = h.levels[0].n_edges
        b1, b2 = rand(n, 1), rand(n, 2)
        a, c = 0.37, -2.25
        b12 = a * b1 + c * b2
        V = mg.v_cycle_preconditioner(h)
        v1, v2, v12 = V(b1).clone(), V(b2).clone(), V(b12).clone()
        d = v12 - (a * v1 + c * v2)
        unit = 2.0 ** -53 * float(mv(Aabs, v12.abs()).norm())
        print("device N", N, solver, "levels", [l.n_edges for l in h.levels], "lin max rel", float(d.abs().max() / v12.abs().max()),
              "|A d|/unit", float(mv(A, d).norm()) / unit, flush=True)
        del h
