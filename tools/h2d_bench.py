"""Host->device upload options for the e2e leg (C2 inputs, ~84 MB)."""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2506_08284_b200 import device as dv
from paper_2506_08284_b200.inputs import make_config
s, rhs, cfg = make_config("C2")
mats = [s.A_e, s.S, s.A_n, s.D]
arrs = []
for M in mats:
    arrs += [M.indptr, M.indices, M.data]
tot = sum(a.nbytes for a in arrs)
print("bytes", tot, [a.dtype for a in arrs[:3]])
dev = torch.device("cuda")
def t(f, n=5):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts), 1e3 * sorted(ts)[n // 2]
print("has_canonical_format", t(lambda: [sp_can(M) for M in mats]) if False else "")
print("current dv.upload path", t(lambda: [dv.DeviceCSR.from_scipy(M) for M in mats]))
print("torch pageable .to(dev)", t(lambda: [torch.from_numpy(a).to(dev) for a in arrs]))
def reg():
    outs = []
    cr = torch.cuda.cudart()
    for a in arrs:
        cr.cudaHostRegister(a.ctypes.data, a.nbytes, 0)
    for a in arrs:
        outs.append(torch.from_numpy(a).to(dev, non_blocking=True))
    torch.cuda.synchronize()
    for a in arrs:
        cr.cudaHostUnregister(a.ctypes.data)
    return outs
print("cudaHostRegister + DMA", t(reg))
pin = torch.empty(tot + 4096 * len(arrs), dtype=torch.uint8, pin_memory=True)
def staged_threads(nthreads=8):
    offs = []
    o = 0
    for a in arrs:
        offs.append(o); o += (a.nbytes + 4095) // 4096 * 4096
    hostviews = [pin[offs[i]:offs[i] + a.nbytes].numpy().view(a.dtype) for i, a in enumerate(arrs)]
    # chunked parallel copies
    jobs = []
    for i, a in enumerate(arrs):
        fa = a.reshape(-1); fh = hostviews[i]
        step = max(1, fa.size // nthreads)
        for k in range(0, fa.size, step):
            jobs.append((fh[k:k + step], fa[k:k + step]))
    def work(js):
        for d, s_ in js:
            np.copyto(d, s_)
    th = [threading.Thread(target=work, args=(jobs[w::nthreads],)) for w in range(nthreads)]
    [x.start() for x in th]; [x.join() for x in th]
    return [pin[offs[i]:offs[i] + a.nbytes].to(dev, non_blocking=True) for i, a in enumerate(arrs)]
print("threaded staging x8 + DMA", t(staged_threads))
print("threaded staging x4 + DMA", t(lambda: staged_threads(4)))
def memcpy_only():
    o = 0
    for a in arrs:
        np.copyto(pin[o:o + a.nbytes].numpy().view(a.dtype), a); o += a.nbytes
print("single-thread memcpy to pinned", t(memcpy_only))
print("DMA from pinned only", t(lambda: pin[:tot].to(dev, non_blocking=True)))
