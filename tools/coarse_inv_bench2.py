"""Coarsest SPD inverse variants at the C2 size (diagnostic): wall per call
(synchronised) and agreement with the float64 host inverse."""
import time
import numpy as np
import torch

dev = torch.device("cuda")


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


def chol_inv(A):
    L, info = torch.linalg.cholesky_ex(A)
    return torch.cholesky_inverse(L)


def chol_trsm(A):
    L, info = torch.linalg.cholesky_ex(A)
    Li = torch.linalg.solve_triangular(L, torch.eye(A.shape[0], dtype=A.dtype, device=A.device),
                                       upper=False)
    return Li.T @ Li


def host(A):
    a = A.cpu().numpy()
    L = np.linalg.cholesky(a)
    import scipy.linalg as sl
    Li = sl.solve_triangular(L, np.eye(a.shape[0]), lower=True)
    return torch.from_numpy(Li.T @ Li).to(A.device)


for n in (364, 1000):
    rng = np.random.default_rng(0)
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    lam = np.logspace(-10, 0, n)
    A = torch.tensor((Q * lam) @ Q.T, device=dev)
    A = 0.5 * (A + A.T)
    ref = chol_inv(A)
    for name, fn in (("chol+cholesky_inverse", chol_inv), ("chol+trsm+gemm", chol_trsm),
                     ("host chol+trsm", host)):
        for lib in ("default", "magma"):
            if lib == "magma" and name.startswith("host"):
                continue
            torch.backends.cuda.preferred_linalg_library(lib)
            ms = t(lambda: fn(A))
            err = float(((fn(A) - ref).abs().max() / ref.abs().max()))
            print(f"n={n} {name:24s} {lib:8s} {ms:7.3f} ms  rel diff {err:.2e}", flush=True)
    torch.backends.cuda.preferred_linalg_library("default")
