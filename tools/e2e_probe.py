"""Where the host-input (e2e) step spends its time beyond the device-resident
step: upload bandwidths (sync single arrays, AsyncUpload), build_hierarchy
from host vs device inputs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_08284_b200 import multigrid as mg, device as dv
from paper_2506_08284_b200.assembly import make_device_config
cfgname = sys.argv[1] if len(sys.argv) > 1 else "C4"
N = int(sys.argv[2]) if len(sys.argv) > 2 else None
s, rhs, cfg = make_device_config(cfgname, N)
host = {k: getattr(s, k).to_scipy() for k in ("A_e", "S", "A_n", "D")}
sc = mg.SolverConfig(coarse_size=cfg.get("coarse_size", 1000))
def sync(): torch.cuda.synchronize()
def gb(M): return (M.data.nbytes + M.indices.size * 4 + M.indptr.size * 8) / 1e9
for rep in range(3):
    sync(); t0 = time.perf_counter()
    An = dv.DeviceCSR.from_scipy(host["A_n"]); Dd = dv.DeviceCSR.from_scipy(host["D"])
    sync(); t1 = time.perf_counter()
    up = dv.AsyncUpload([host["S"], host["A_e"]])
    Sd = up.get(0); sync(); t2 = time.perf_counter()
    Ad = up.get(1); sync(); t3 = time.perf_counter()
    print(f"rep {rep}: A_n+D sync upload {gb(host['A_n'])+gb(host['D']):.2f} GB {1e3*(t1-t0):.1f} ms; "
          f"S {gb(host['S']):.2f} GB landed {1e3*(t2-t1):.1f} ms; A_e {1e3*(t3-t1):.1f} ms", flush=True)
    del An, Dd, Sd, Ad, up
for rep in range(3):
    sync(); t0 = time.perf_counter()
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, sc); sync(); t1 = time.perf_counter()
    del h
    h = mg.build_hierarchy(host["A_e"], host["S"], host["A_n"], host["D"], sc); sync()
    t2 = time.perf_counter()
    r = mg.pcg_solve(h.levels[0].A_e, rhs, mg.v_cycle_preconditioner(h)); sync()
    t3 = time.perf_counter()
    bd = torch.from_numpy(rhs).cuda(); sync(); t4 = time.perf_counter()
    r2 = mg.pcg_solve(h.levels[0].A_e, bd, mg.v_cycle_preconditioner(h)); sync()
    t5 = time.perf_counter()
    print(f"rep {rep}: setup device {1e3*(t1-t0):.1f} ms, host inputs {1e3*(t2-t1):.1f} ms; "
          f"solve host rhs {1e3*(t3-t2):.1f} ms, device rhs {1e3*(t5-t4):.1f} ms", flush=True)
    del h, r, r2
if os.environ.get("SPHC_TRACE"):
    from paper_2506_08284_b200 import trace

# host timeline of the host-input setup (readbacks keep the host within a
# kernel or two of the device, so host stamps are a fair picture)
import paper_2506_08284_b200.multigrid as M
stamps = []
def stamp(tag): stamps.append((tag, time.perf_counter()))
_own, _bep, _cn = M.own_csr, M.build_edge_prolongator, M._check_nullspace
def own(A):
    r = _own(A); stamp("own_csr"); return r
def bep(*a, **k):
    stamp("bep.start"); r = _bep(*a, **k); stamp("bep.end"); return r
def cn(*a, **k):
    stamp("nullspace.start"); r = _cn(*a, **k); stamp("nullspace.end"); return r
M.own_csr, M.build_edge_prolongator, M._check_nullspace = own, bep, cn
import paper_2506_08284_b200.edge_prolongator as EP
_es = EP.emin_sweeps
def es_(*a, **k):
    stamp("emin_sweeps.start"); r = _es(*a, **k); stamp("emin_sweeps.end"); return r
EP.emin_sweeps = es_
for inputs in ("host", "device"):
    stamps.clear(); sync(); t0 = time.perf_counter()
    if inputs == "host":
        h = mg.build_hierarchy(host["A_e"], host["S"], host["A_n"], host["D"], sc)
    else:
        h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, sc)
    sync(); t1 = time.perf_counter()
    print(inputs, f"total {1e3*(t1-t0):.1f} ms:", " ".join(f"{t}@{1e3*(x-t0):.0f}" for t, x in stamps[:14]))
    del h
