import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_2506_08284_b200 import multigrid as mg
from paper_2506_08284_b200.assembly import make_device_config
for cfgname in ("C4", "C3"):
    s, rhs, cfg = make_device_config(cfgname, None)
    h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=1000))
    for li, lv in enumerate(h.levels[:-1]):
        e, a = lv.edge_sweeper.sell, lv.aux_sweeper.sell
        print(cfgname, li, lv.A_e.shape[0], "edge d16", e.d16 is not None, "aux d16", a.d16 is not None,
              "mid", None if lv.mid is None else (lv.mid.d16 is not None), "MB", e.padded * 12 / 1e6, a.padded * 12 / 1e6)
    del h
