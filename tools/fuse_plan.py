"""Fusion plan (steps per pass, bandwidth in blocks) of every level's smoothers
for a device config, and the V-cycle time (graph replay)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_08284_b200 import multigrid as mg
from paper_2506_08284_b200.assembly import make_device_config
s, rhs, cfg = make_device_config(sys.argv[1] if len(sys.argv) > 1 else "C4")
b = torch.from_numpy(rhs).cuda()
h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=cfg.get("coarse_size", 1000)))
for i, lv in enumerate(h.levels[:-1]):
    for nm in ("edge_sweeper", "aux_sweeper"):
        sw = getattr(lv, nm)
        print(i, nm, "n", sw.A.shape[0], "fuse", sw.fuse, "L", getattr(sw, "fuse_L", None))
pre = mg.v_cycle_preconditioner(h)
pre(b)
cap = torch.cuda.Stream(); cap.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(cap):
    g = mg.PcgGraph(lambda: pre(b))
torch.cuda.current_stream().wait_stream(cap)
for _ in range(3): g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): g.replay()
e1.record(); torch.cuda.synchronize()
print("V-cycle ms", e0.elapsed_time(e1) / 10)
t0 = time.perf_counter()
r = mg.pcg_solve(h.levels[0].A_e, b, pre)
torch.cuda.synchronize()
print("solve ms", (time.perf_counter() - t0) * 1e3, "its", r.iterations, r.status)
