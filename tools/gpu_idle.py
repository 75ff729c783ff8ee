"""GPU busy vs idle during one setup + solve (torch.profiler / CUPTI kernel
timeline): where the wall time goes when kernels are small."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2506_08284_b200 import multigrid as mg, device as dv
from paper_2506_08284_b200.inputs import make_config
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
if name in ("C3", "C4", "C5"):
    from paper_2506_08284_b200.assembly import make_device_config
    s, rhs, cfg = make_device_config(name)
    A_e, S, A_n, D = s.A_e, s.S, s.A_n, s.D
else:
    s, rhs, cfg = make_config(name)
    A_e, S, A_n, D = (dv.DeviceCSR.from_scipy(M) for M in (s.A_e, s.S, s.A_n, s.D))
b = torch.from_numpy(rhs).cuda()
sc = mg.SolverConfig(coarse_size=cfg.get("coarse_size", 1000))
for _ in range(int(os.environ.get("WARM", "3"))):
    h = None
    h = mg.build_hierarchy(A_e, S, A_n, D, sc)
    if os.environ.get("SETUP_ONLY") != "1":
        r = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
h = None
torch.cuda.synchronize()
marks = {}
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    torch.cuda.synchronize(); marks["t0"] = time.perf_counter()
    h = mg.build_hierarchy(A_e, S, A_n, D, sc)
    torch.cuda.synchronize(); marks["t1"] = time.perf_counter()
    if os.environ.get("SETUP_ONLY") != "1":
        r = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    torch.cuda.synchronize(); marks["t2"] = time.perf_counter()
prof.export_chrome_trace("/tmp/trace.json")
ev = json.load(open("/tmp/trace.json"))["traceEvents"]
kern = sorted([(e["ts"], e["ts"] + e["dur"], e["name"]) for e in ev if e.get("cat") == "kernel"])
memc = [(e["ts"], e["ts"] + e["dur"]) for e in ev if e.get("cat") in ("gpu_memcpy", "gpu_memset")]
allg = sorted([(a, b) for a, b, _ in kern] + memc)
t0, t1 = allg[0][0], allg[-1][1]
busy = 0.0; cur_s, cur_e = allg[0]
for a, b_ in allg[1:]:
    if a > cur_e:
        busy += cur_e - cur_s; cur_s, cur_e = a, b_
    else:
        cur_e = max(cur_e, b_)
busy += cur_e - cur_s
print(f"wall setup {1e3*(marks['t1']-marks['t0']):.2f} ms, solve {1e3*(marks['t2']-marks['t1']):.2f} ms")
print(f"GPU span {1e-3*(t1-t0):.2f} ms, busy {1e-3*busy:.2f} ms ({100*busy/(t1-t0):.0f}%), kernels {len(kern)}")
# split at the largest gap between setup and solve is hard; report by name
import collections
agg = collections.defaultdict(float)
cnt = collections.Counter()
for a, b_, n in kern:
    agg[n.split("(")[0][:50]] += b_ - a
    cnt[n.split("(")[0][:50]] += 1
for n, v in sorted(agg.items(), key=lambda kv: -kv[1])[:int(os.environ.get("TOPK", "25"))]:
    print(f"{v/1e3:8.3f} ms  x{cnt[n]:4d}  {n}")
# gaps histogram
gaps = [allg[i+1][0] - allg[i][1] for i in range(len(allg)-1)]
gaps = [g for g in gaps if g > 0]
print("idle gaps: n", len(gaps), "total ms", sum(gaps)/1e3, ">50us", sum(1 for g in gaps if g > 50), "sum>50us ms", sum(g for g in gaps if g > 50)/1e3)
named = sorted([(a, b_, n.split("(")[0][:40]) for a, b_, n in kern] + [(a, b_, "memcpy/set") for a, b_ in memc])
gl = [(named[i+1][0] - named[i][1], named[i][2], named[i+1][2], i) for i in range(len(named)-1)]
print("largest gaps (us): after -> before")
for g, a, b_, i in sorted(gl, reverse=True)[:40]:
    print(f"{g:8.1f}  #{i:5d} {a} -> {b_}")
show = os.environ.get("SHOW")
if show:
    import re
    pat = re.compile(show)
    for e in sorted((e for e in ev if e.get("cat") == "kernel"), key=lambda e: e["ts"]):
        if pat.search(e["name"]):
            a = e.get("args", {})
            print(f"{e['dur']:9.1f} us  {e['name'].split('(')[0][:40]:40s} grid {a.get('grid')} block {a.get('block')} smem {a.get('shared memory')}")
