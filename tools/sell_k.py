"""Time the fused SELL Chebyshev step on a config's finest A_e (cold L2 and
warm); run once per SPHC_SELL_K setting."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_08284_b200 import _lib, device as dv
from paper_2506_08284_b200.inputs import make_config
s, rhs, cfg = make_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
A = dv.DeviceCSR.from_scipy(s.A_e)
n = A.shape[0]
m = dv.sell(A)
dinv = dv.reciprocal(dv.diagonal(A))
b = torch.from_numpy(rhs).cuda()
x = torch.rand(n, dtype=torch.float64, device="cuda")
out, d = torch.empty_like(x), torch.zeros_like(x)
flush = torch.empty(256 * 2**20 // 8, dtype=torch.float64, device="cuda")
k = lambda: _lib.call("sphc_sell_cheb_step", n, m.slice_ptr, m.col, m.val, dinv, b, x, out, d, 0.3, 0.7, 0, m.padded)
for _ in range(5):
    k()
E = lambda: torch.cuda.Event(enable_timing=True)
cold = []
for i in range(30):
    flush.fill_(float(i)); a, z = E(), E(); a.record(); k(); z.record(); torch.cuda.synchronize(); cold.append(a.elapsed_time(z))
a, z = E(), E(); a.record()
for _ in range(100):
    k()
z.record(); torch.cuda.synchronize()
cold.sort()
byts = 12 * A.nnz + 8 * (n + 1) + 48 * n
print(f"K={os.environ.get('SPHC_SELL_K','auto')} n={n} cold median {cold[15]*1e3:.1f} us ({byts/cold[15]/1e6:.0f} GB/s) warm {a.elapsed_time(z)*10:.1f} us")
