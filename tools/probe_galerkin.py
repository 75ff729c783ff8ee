import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2506_08284_b200 import multigrid as mg, device as dv
from paper_2506_08284_b200.assembly import make_device_config
s, rhs, cfg = make_device_config("C4", None)
sc = mg.SolverConfig(coarse_size=1000)
times = {}
def wrap(mod, name):
    f = getattr(mod, name)
    def g(*a, **k):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = f(*a, **k)
        torch.cuda.synchronize(); times.setdefault(name, []).append((time.perf_counter() - t0) * 1e3)
        return r
    setattr(mod, name, g)
for rep in range(3):
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, sc); del h
wrap(mg, "_galerkin_edge"); wrap(dv, "spgemm_pair"); wrap(dv, "drop_zeros_many"); wrap(dv, "transpose")
torch.cuda.synchronize(); t0 = time.perf_counter()
h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, sc)
torch.cuda.synchronize(); print("setup with syncs", (time.perf_counter() - t0) * 1e3)
for k, v in times.items():
    print(k, [round(x, 1) for x in v])
print(torch.cuda.max_memory_allocated() / 1e9, "GB peak", torch.cuda.memory_reserved() / 1e9, "reserved")
