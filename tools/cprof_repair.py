"""cProfile of one C4 (device inputs) setup, restricted to the repair pass."""
import os, sys, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_08284_b200 import multigrid as mg, repair
from paper_2506_08284_b200.assembly import make_device_config
s, rhs, cfg = make_device_config("C4", int(sys.argv[1]) if len(sys.argv) > 1 else 128)
sc = mg.SolverConfig(coarse_size=1000)
h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, sc)
orig = repair.make_irreducible_pass
pr = cProfile.Profile()
def wrapped(*a, **k):
    torch.cuda.synchronize()
    pr.enable()
    try:
        return orig(*a, **k)
    finally:
        torch.cuda.synchronize()
        pr.disable()
repair.make_irreducible_pass = wrapped
h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, sc)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
