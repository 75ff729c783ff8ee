import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, scipy.sparse as sp
from paper_2506_08284_b200 import device as dv
from paper_2506_08284_b200.inputs import discretize_hex
from oracle import hcurl_oracle as O
s = discretize_hex(4, 1.0, False)
h = O.build_hierarchy(s.A_e, s.S, s.A_n, s.D, coarse_size=40)
P = h.levels[0].P_e.tocsr(); P.sort_indices()
AP = (s.A_e @ P).tocsr(); AP.sort_indices()
R = sp.csr_matrix(P.T); R.sort_indices()
print("P rows max", np.diff(P.indptr).max(), "AP max", np.diff(AP.indptr).max(), "R max", np.diff(R.indptr).max(), flush=True)
for name, A, B in (("AP", s.A_e, P), ("RAP", R, AP)):
    for ordered in (False, True):
        try:
            C = dv.spgemm(dv.DeviceCSR.from_scipy(A), dv.DeviceCSR.from_scipy(B), ordered=ordered, drop=False)
            torch.cuda.synchronize()
            ref = (A @ B).tocsr()
            print(name, ordered, "ok", C.nnz, ref.nnz, flush=True)
        except Exception as e:
            print(name, ordered, "FAIL", str(e)[:300], flush=True)
            raise SystemExit
