import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from paper_2506_08284_b200 import multigrid as mg, device as dv
from paper_2506_08284_b200.assembly import make_device_config
from paper_2506_08284_b200.inputs import make_config
from golden_util import load_case, stored_inputs
orig = mg._coarse_inverse_start
def spy(Ad, solver="cholesky"):
    A = 0.5 * (Ad + Ad.T); d = torch.diagonal(A); sc = torch.where(d > 0, d.rsqrt(), torch.ones_like(d))
    As = sc[:, None] * A * sc[None, :]; As = 0.5 * (As + As.T)
    L, info = torch.linalg.cholesky_ex(As)
    dl = torch.diagonal(L)
    lam = torch.linalg.eigvalsh(As)
    print(f"   n={A.shape[0]} info={int(info)} min pivot^2={float(dl.min())**2:.3e} eig min={float(lam[0]):.3e} 2nd={float(lam[1]):.3e} max={float(lam[-1]):.3e} n*eps={A.shape[0]*2.2e-16:.2e}", flush=True)
    return orig(Ad, solver)
mg._coarse_inverse_start = spy
for name, N, cs in (("C4", None, 1000), ("C4", 32, 1000), ("C5", 64, 1000), ("C5", 128, 2000), ("C3", None, 1000)):
    s, rhs, cfg = make_device_config(name, N)
    print(name, N, cs)
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=cs)); del h
for name in ("C1", "C2"):
    s, rhs, cfg = make_config(name)
    print(name)
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=1000)); del h
for name in ("Q41s", "Q41d", "T9n", "T8d", "R33n"):
    meta, arrays = load_case(name)
    A_e, S, A_n, D, rhs = stored_inputs(arrays)
    print(name)
    h = mg.build_hierarchy(A_e, S, A_n, D, mg.SolverConfig(coarse_size=meta["coarse_size"])); del h
