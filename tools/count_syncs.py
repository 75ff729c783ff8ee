"""Count host<->device synchronisations in one C2 build_hierarchy, by call site."""
import os, sys, collections, traceback, warnings
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_08284_b200 import multigrid as mg, device as dv
from paper_2506_08284_b200.inputs import make_config
s, rhs, cfg = make_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
A_e, S, A_n, D = (dv.DeviceCSR.from_scipy(M) for M in (s.A_e, s.S, s.A_n, s.D))
sc = mg.SolverConfig(coarse_size=1000)
h = mg.build_hierarchy(A_e, S, A_n, D, sc)
torch.cuda.synchronize()
sites = collections.Counter()
def hook(message, category, filename, lineno, file=None, line=None):
    st = traceback.extract_stack()[:-2]
    fr = [f for f in st if "paper_2506_08284_b200" in f.filename]
    fr = [f for f in fr if f.name not in ("readback", "scan", "scan_many", "wrap",
                                           "drop_zeros_many", "rows", "flush_checks")]
    key = " <- ".join(f"{os.path.basename(f.filename)}:{f.lineno} {f.name}"
                      for f in fr[-1:-3:-1]) if fr else "?"
    sites[key] += 1
warnings.showwarning = hook
warnings.simplefilter("always")
torch.cuda.set_sync_debug_mode("warn")
h = mg.build_hierarchy(A_e, S, A_n, D, sc)
torch.cuda.set_sync_debug_mode(0)
print("total syncs", sum(sites.values()))
for k, v in sites.most_common(60):
    print(f"{v:5d} {k}")
