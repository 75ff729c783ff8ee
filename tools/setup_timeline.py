"""Stream timeline of one device-resident setup (torch.profiler / CUPTI):
every kernel longer than MIN_MS with its start, duration and stream, to see
what overlaps what. Usage: python tools/setup_timeline.py [C4] [N]"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2506_08284_b200 import multigrid as mg
from paper_2506_08284_b200.assembly import make_device_config
cfgname = sys.argv[1] if len(sys.argv) > 1 else "C4"
N = int(sys.argv[2]) if len(sys.argv) > 2 else None
s, rhs, cfg = make_device_config(cfgname, N)
sc = mg.SolverConfig(coarse_size=cfg.get("coarse_size", 1000))
for _ in range(2):
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, sc)
torch.cuda.synchronize()
h = None
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    torch.cuda.synchronize()
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, sc)
    torch.cuda.synchronize()
path = "gpurun_out/setup_timeline.json"
os.makedirs("gpurun_out", exist_ok=True)
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
k = sorted([(e["ts"], e["dur"], e["args"].get("stream"), e["name"]) for e in ev
            if e.get("ph") == "X" and e.get("cat") == "kernel"])
t0 = k[0][0]
tend = max(a + d for a, d, _, _ in k)
busy, cur = 0.0, t0
for a, d, st, n in k:
    busy += max(0.0, a + d - max(a, cur)); cur = max(cur, a + d)
print(f"setup GPU span {(tend - t0) / 1e3:.1f} ms, busy (union) {busy / 1e3:.1f} ms, "
      f"sum of kernel times {sum(d for _, d, _, _ in k) / 1e3:.1f} ms")
# idle gaps (GPU waiting for the host) with the kernels around them
gaps, cur, prev = [], t0, None
for a, d, st, n in k:
    if a > cur:
        gaps.append((a - cur, prev, n, cur - t0))
    if a + d > cur:
        cur, prev = a + d, n
gaps.sort(reverse=True)
print(f"{len(gaps)} gaps, total {sum(g[0] for g in gaps) / 1e3:.1f} ms; largest:")
for g, p_, n_, at in gaps[:int(os.environ.get("TOPGAPS", "12"))]:
    print(f"   {g / 1e3:6.2f} ms at {at / 1e3:7.1f}: {str(p_)[:38]} -> {n_[:38]}")
mn = float(os.environ.get("MIN_MS", "0.4")) * 1e3
for a, d, st, n in k:
    if d >= mn:
        print(f"{(a - t0) / 1e3:8.2f} +{d / 1e3:7.2f} ms  s{st}  {n[:70]}")
os.remove(path)
