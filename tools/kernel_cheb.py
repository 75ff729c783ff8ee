"""Launch only the fused SELL Chebyshev step on a config's finest A_e (for
ncu captures): 5 launches, L2 flushed before each."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_08284_b200 import _lib, device as dv
from paper_2506_08284_b200.inputs import make_config
s, rhs, cfg = make_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
A = dv.DeviceCSR.from_scipy(s.A_e)
n = A.shape[0]
m = dv.sell(A)
dinv = dv.reciprocal(dv.diagonal(A))
b = torch.from_numpy(rhs).cuda()
x = torch.rand(n, dtype=torch.float64, device="cuda")
out, d = torch.empty_like(x), torch.zeros_like(x)
flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")
for i in range(5):
    flush.fill_(float(i))
    _lib.call("sphc_sell_cheb_step", n, m.slice_ptr, m.col, m.val, dinv, b, x, out, d, 0.3, 0.7, 0, m.padded)
torch.cuda.synchronize()
print("ok", n, A.nnz, m.padded)
