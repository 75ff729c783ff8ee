"""Probe (CPU): the oracle V-cycle's linearity defect in units of the fine
level's rounding, C4 recipe at small N (compare tools/probe_vlin3.py on GPU)."""
import sys
import numpy as np
from oracle import hcurl_oracle as O
from oracle.host_assembly import config_host

for N in [int(a) for a in sys.argv[1:]] or [16]:
    A_e, S, A_n, D, rhs, cfg = config_host("C4", N)
    h = O.build_hierarchy(A_e, S, A_n, D, coarse_size=1000 if N > 16 else 200, smoother="cheb")
    A = h.levels[0].A_e
    Aabs = abs(A)
    rng = np.random.default_rng(1)
    b1, b2 = rng.uniform(-1, 1, A.shape[0]), rng.uniform(-1, 1, A.shape[0])
    a, c = 0.37, -2.25
    b12 = a * b1 + c * b2
    V = lambda b: O.v_cycle(h, b)
    v1, v2, v12 = V(b1), V(b2), V(b12)
    d = v12 - (a * v1 + c * v2)
    unit = 2.0 ** -53 * np.linalg.norm(Aabs @ np.abs(v12))
    print("oracle N", N, "levels", [l.A_e.shape[0] for l in h.levels], "lin max rel", np.abs(d).max() / np.abs(v12).max(),
          "|A d|/unit", np.linalg.norm(A @ d) / unit, flush=True)
