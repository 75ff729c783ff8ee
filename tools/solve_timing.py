"""pcg_solve wall time on one C2 hierarchy: first solve (includes the loop
graph capture) and steady-state repeats."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_08284_b200 import multigrid as mg, device as dv
from paper_2506_08284_b200.inputs import make_config
s, rhs, cfg = make_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
A_e, S, A_n, D = (dv.DeviceCSR.from_scipy(M) for M in (s.A_e, s.S, s.A_n, s.D))
b = torch.from_numpy(rhs).cuda()
sc = mg.SolverConfig(coarse_size=1000)
for rep in range(3):
    h = mg.build_hierarchy(A_e, S, A_n, D, sc)
    torch.cuda.synchronize()
    ts = []
    for k in range(5):
        t0 = time.perf_counter()
        r = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print("solve ms:", " ".join(f"{t:.2f}" for t in ts), "its", r.iterations, flush=True)
# capture + instantiate cost: a plain graph of one V-cycle vs the loop graph
pre = mg.v_cycle_preconditioner(h)
pre(b)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(cap):
        g = mg.PcgGraph(lambda: pre(b))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    del g
    ws = h._pcg_ws
    with torch.cuda.stream(cap):
        lp = mg.PcgLoop(lambda: mg._pcg_iteration(ws["A"], ws["A"].lanes(), pre, ws["x"], ws["r"],
                                                  ws["p"], ws["Ap"], ws["sc"], ws["flag"], None,
                                                  rotate=False),
                        ws["sc"], ws["ctl"], ws["hist"])
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    del lp
    print(f"capture+instantiate: V-cycle graph {1e3*(t1-t0):.2f} ms, PCG loop graph {1e3*(t2-t1):.2f} ms")
