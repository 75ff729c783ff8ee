"""Phase breakdown of one setup + solve (SPHC_TRACE=1 adds syncs)."""
import os, sys, time
os.environ.setdefault("SPHC_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_08284_b200 import multigrid as mg, device as dv, trace
from paper_2506_08284_b200.inputs import make_config

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
N = int(sys.argv[2]) if len(sys.argv) > 2 else None
if cfgname in ("C3", "C4", "C5"):
    from paper_2506_08284_b200.assembly import make_device_config
    s, rhs, cfg = make_device_config(cfgname, N)
    A_e, S, A_n, D = s.A_e, s.S, s.A_n, s.D
else:
    s, rhs, cfg = make_config(cfgname, N)
    A_e, S, A_n, D = (dv.DeviceCSR.from_scipy(M) for M in (s.A_e, s.S, s.A_n, s.D))
b = torch.from_numpy(rhs).cuda()
sc = mg.SolverConfig(coarse_size=cfg.get("coarse_size", 1000))
h = res = None
for rep in range(int(os.environ.get("REPS", "3"))):
    h = res = None
    torch.cuda.synchronize(); t0 = time.perf_counter()
    with trace.phase("TOTAL.setup"):
        h = mg.build_hierarchy(A_e, S, A_n, D, sc)
    with trace.phase("TOTAL.solve"):
        res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    rep_txt = trace.report()
print(f"{cfgname} n_e={s.A_e.shape[0]} levels={[lv.A_e.shape[0] for lv in h.levels]} its={res.iterations} wall={1e3*(t1-t0):.1f} ms")
print(rep_txt)
# untraced timing
trace.ENABLED = False
for rep in range(int(os.environ.get("UREPS", "2"))):
    h = res = None
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = mg.build_hierarchy(A_e, S, A_n, D, sc)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"untraced: setup {1e3*(t1-t0):.1f} ms, solve {1e3*(t2-t1):.1f} ms")
