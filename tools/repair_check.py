"""C4 hierarchy facts that pin the make_irreducible path: coarse edges
appended per level and the level sizes / iterations."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_08284_b200 import multigrid as mg
from paper_2506_08284_b200.assembly import make_device_config
if os.environ.get("OLD_REPAIR") == "1":      # the host main loop (previous commit)
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import _old_repair
    from paper_2506_08284_b200 import repair
    repair.make_irreducible_pass = _old_repair.make_irreducible_pass
s, rhs, cfg = make_device_config("C4")
b = torch.from_numpy(rhs).cuda()
h = mg.build_hierarchy(s.A_e, s.S, s.A_n, s.D, mg.SolverConfig(coarse_size=1000))
r = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
print("levels", [lv.A_e.shape[0] for lv in h.levels], "nnz", [lv.A_e.nnz for lv in h.levels])
print("n_augmented", [lv.n_augmented for lv in h.levels[:-1]], "its", r.iterations,
      "res", [float(f"{x:.6e}") for x in r.residual_history[-3:]])
print("comm", [lv.commutator_residual for lv in h.levels[:-1]])
