"""Time dense coarsest-inverse options on the GPU (diagnostic)."""
import time
import numpy as np
import torch

dev = torch.device("cuda")


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


for n in (36, 139, 200, 400):
    rng = np.random.default_rng(0)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.logspace(-13, 0, n)
    A = torch.tensor((Q * lam) @ Q.T, device=dev)
    A = 0.5 * (A + A.T)
    res = {}
    res["inv"] = t(lambda: torch.linalg.inv(A))
    res["eigh"] = t(lambda: torch.linalg.eigh(A))
    res["eigh_b"] = t(lambda: torch.linalg.eigh(A[None]))
    res["svd_j"] = t(lambda: torch.linalg.svd(A, driver="gesvdj"))
    res["chol+inv"] = t(lambda: torch.cholesky_inverse(torch.linalg.cholesky_ex(A)[0]))
    res["host_eigh"] = t(lambda: np.linalg.eigh(A.cpu().numpy()))
    print(n, {k: round(v, 3) for k, v in res.items()}, flush=True)
