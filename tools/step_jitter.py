"""Per-step time of C2 setup+solve with the allocator / GC activity of
each step: where do the outlier steps come from?"""
import gc, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_08284_b200 import multigrid as mg, device as dv
from paper_2506_08284_b200.inputs import make_config
s, rhs, cfg = make_config("C2")
A_e, S, A_n, D = (dv.DeviceCSR.from_scipy(M) for M in (s.A_e, s.S, s.A_n, s.D))
b = torch.from_numpy(rhs).cuda()
sc = mg.SolverConfig(coarse_size=1000)
if os.environ.get("NOGC") == "1":
    gc.disable()
h = res = None
flush = torch.empty(32 * 2**20, dtype=torch.float64, device="cuda") if os.environ.get("FLUSH") else None
for k in range(30):
    if flush is not None:
        flush.fill_(float(k))
    st0 = torch.cuda.memory_stats()
    g0 = [x["collections"] for x in gc.get_stats()]
    h = res = None
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h = mg.build_hierarchy(A_e, S, A_n, D, sc)
    res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
    torch.cuda.synchronize(); t1 = time.perf_counter()
    st1 = torch.cuda.memory_stats()
    g1 = [x["collections"] for x in gc.get_stats()]
    print(f"{k:2d} {1e3*(t1-t0):7.2f} ms  cudaMalloc +{st1['num_device_alloc']-st0['num_device_alloc']:3d}"
          f" cudaFree +{st1['num_device_free']-st0['num_device_free']:3d}"
          f" gc {[a-b for a,b in zip(g1,g0)]} reserved {st1['reserved_bytes.all.current']/1e6:.0f} MB", flush=True)
