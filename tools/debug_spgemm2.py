import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, scipy.sparse as sp
from paper_2506_08284_b200 import device as dv
from paper_2506_08284_b200.inputs import discretize_hex
s = discretize_hex(4, 1.0, False)
for name, A, B in (("SD", s.S, s.D), ("AD", s.A_e, s.D)):
    print(name, A.shape, A.nnz, B.shape, B.nnz, "maxrow", np.diff(A.indptr).max(), flush=True)
    for ordered in (False, True):
        try:
            C = dv.spgemm(dv.DeviceCSR.from_scipy(A), dv.DeviceCSR.from_scipy(B), ordered=ordered, drop=False)
            torch.cuda.synchronize()
            ref = A @ B
            print(name, ordered, "ok", C.nnz, ref.nnz, flush=True)
        except Exception as e:
            print(name, ordered, "FAIL", str(e)[:200], flush=True)
            raise SystemExit
