import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, scipy.sparse as sp
from paper_2506_08284_b200 import device as dv
from paper_2506_08284_b200.inputs import discretize_hex
from oracle import hcurl_oracle as O
s = discretize_hex(4, 1.0, False)
memb, nagg = O.aggregate(O.strength_pattern(s.A_n))
P, _, _ = O.smoothed_prolongator(s.A_n, memb, nagg)
X = (s.A_n @ P).tocsr(); X.sort_indices()
PT = sp.csr_matrix(P.T); PT.sort_indices()
print("A_n", s.A_n.shape, s.A_n.nnz, "P", P.shape, P.nnz, "PT", PT.shape, "X", X.shape, X.nnz, flush=True)
for name, A, B in (("AP", s.A_n, P), ("PtX", PT, X)):
    for ordered in (False, True):
        try:
            C = dv.spgemm(dv.DeviceCSR.from_scipy(A), dv.DeviceCSR.from_scipy(B), ordered=ordered)
            torch.cuda.synchronize()
            print(name, ordered, "ok", C.nnz, flush=True)
        except Exception as e:
            print(name, ordered, "FAIL", str(e)[:200], flush=True)
            raise SystemExit
