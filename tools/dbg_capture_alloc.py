import os, sys
sys.path.insert(0, "/root/repo")
import torch
import torch.cuda
from paper_2506_08284_b200 import multigrid as mg, device as dv
from paper_2506_08284_b200.inputs import make_config
s, rhs, cfg = make_config("C1")
A_e, S, A_n, D = (dv.DeviceCSR.from_scipy(M) for M in (s.A_e, s.S, s.A_n, s.D))
b = torch.from_numpy(rhs).cuda()
h = mg.build_hierarchy(A_e, S, A_n, D, mg.SolverConfig(coarse_size=1000))
torch.cuda.memory._record_memory_history(max_entries=100000)
res = mg.pcg_solve(h.levels[0].A_e, b, mg.v_cycle_preconditioner(h))
snap = torch.cuda.memory._snapshot()
for seg in snap["segments"]:
    if seg.get("segment_pool_id", (0, 0)) != (0, 0):
        print("private segment", seg["total_size"], seg.get("segment_pool_id"))
        for blk in seg["blocks"]:
            fr = blk.get("frames", [])
            print("  block", blk["size"], blk["state"], [f"{f['filename'].split('/')[-1]}:{f['line']}:{f['name']}" for f in fr[:12]])
