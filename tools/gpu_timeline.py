"""GPU busy time vs wall time of one C2 setup (+ solve) from a torch.profiler
(CUPTI) trace: union of kernel / memcpy intervals, and the largest idle gaps
with the kernels around them. Usage: python tools/gpu_timeline.py [C2] [out.json]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import profile, ProfilerActivity
from paper_2506_08284_b200 import multigrid as mg, device as dv
from paper_2506_08284_b200.inputs import make_config

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
s, rhs, cfg = make_config(cfgname)
if os.environ.get("E2E") == "1":
    # the public API from host inputs (scipy CSR, numpy RHS), as bench.py's e2e
    A_e, S, A_n, D, b = s.A_e, s.S, s.A_n, s.D, rhs
else:
    A_e, S, A_n, D = (dv.DeviceCSR.from_scipy(M) for M in (s.A_e, s.S, s.A_n, s.D))
    b = torch.from_numpy(rhs).cuda()
sc = mg.SolverConfig(coarse_size=1000)
for _ in range(3):
    h = mg.build_hierarchy(A_e, S, A_n, D, sc)
    r = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
torch.cuda.synchronize()
h = r = None
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA],
             with_stack=os.environ.get("STACK") == "1") as prof:
    torch.cuda.synchronize()
    with torch.profiler.record_function("SETUP"):
        h = mg.build_hierarchy(A_e, S, A_n, D, sc)
        torch.cuda.synchronize()
    with torch.profiler.record_function("SOLVE"):
        r = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
        torch.cuda.synchronize()
path = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/timeline.json"
prof.export_chrome_trace(path)
ev = json.load(open(path))["traceEvents"]
win = {e["name"]: (e["ts"], e["ts"] + e["dur"]) for e in ev
       if e.get("ph") == "X" and e.get("name") in ("SETUP", "SOLVE") and e.get("cat") == "user_annotation"}
gpu = sorted([(e["ts"], e["ts"] + e["dur"], e["name"]) for e in ev
              if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")])
rt = sorted([(e["ts"], e["ts"] + e["dur"], e["name"]) for e in ev
             if e.get("ph") == "X" and e.get("cat") == "cuda_runtime"])
py = [(e["ts"], e["ts"] + e["dur"], e["name"]) for e in ev
      if e.get("ph") == "X" and e.get("cat") == "python_function" and "paper_2506" in e["name"]]
for name, (t0, t1) in sorted(win.items(), key=lambda kv: kv[1][0]):
    g = [x for x in gpu if x[0] >= t0 and x[1] <= t1]
    busy, cur_end = 0.0, t0
    gaps = []
    prev = None
    for a, z, n in g:
        if a > cur_end:
            gaps.append((a - cur_end, prev, n, cur_end, a))
        busy += max(0.0, z - max(a, cur_end))
        cur_end = max(cur_end, z)
        prev = n
    print(f"{name}: wall {(t1 - t0) / 1e3:.2f} ms, GPU busy {busy / 1e3:.2f} ms, "
          f"{len(g)} GPU ops, idle {(t1 - t0 - busy) / 1e3:.2f} ms")
    gaps.sort(reverse=True)
    for d, p, n, ga, gz in gaps[:int(os.environ.get("TOPGAPS", "25"))]:
        calls = {}
        for a, z, rn in rt:
            if a >= ga - 5 and a <= gz:
                calls[rn] = calls.get(rn, 0) + 1
        print(f"  gap {d:7.1f} us after {str(p)[:38]:38s} before {n[:38]:38s} "
              + " ".join(f"{k}x{v}" for k, v in sorted(calls.items(), key=lambda kv: -kv[1])[:3]))
        if py:
            # our python frames overlapping the gap, by overlap time
            ov = {}
            for a, z, fn in py:
                o = min(z, gz) - max(a, ga)
                if o > 0:
                    ov[fn] = ov.get(fn, 0) + o
            for fn, o in sorted(ov.items(), key=lambda kv: (-kv[1], kv[0]))[:6]:
                print(f"      {o:6.1f} us {fn.split('paper_2506_08284_b200/')[-1][:90]}")
    # gap histogram
    tot = sum(x[0] for x in gaps)
    small = sum(x[0] for x in gaps if x[0] < 10)
    print(f"  gaps: {len(gaps)} total {tot / 1e3:.2f} ms; < 10 us: {small / 1e3:.2f} ms")
    # kernels by GPU time inside the window
    agg = {}
    for a, z, n in g:
        k = n.split("(")[0][:70]
        c, d = agg.get(k, (0, 0.0))
        agg[k] = (c + 1, d + z - a)
    for k, (c, d) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:int(os.environ.get("TOPK", "12"))]:
        print(f"  {d:8.1f} us x{c:4d} {k}")
