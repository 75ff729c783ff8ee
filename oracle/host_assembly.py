"""Host build of the device model-problem assembly -- TEST INFRASTRUCTURE.

``assemble_host`` runs the per-row arithmetic of csrc/assemble.cu on the CPU
(oracle/csrc/host_assemble.cpp compiles csrc/assemble_rows.cuh with explicit
IEEE rounding), so its (A_e, S, A_n, D) are bit-identical to
``paper_2506_08284_b200.assembly.assemble_hex`` on the B200. The golden
generator runs the unmodified reference on these host matrices for the
device-generated configs (C3, the C4 recipe); the GPU tests assemble the same
system on the device and check its sha256 against the golden's before
comparing hierarchies.
"""

import ctypes
import os
import subprocess

import numpy as np
import scipy.sparse as sp

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "_build", "libhostasm.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        lib = ctypes.CDLL(path)
        lib.host_hex_create.restype = ctypes.c_void_p
        lib.host_hex_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_double]
        lib.host_hex_sizes.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        lib.host_hex_fill.argtypes = [ctypes.c_void_p] + [ctypes.c_void_p] * 10
        lib.host_hex_destroy.argtypes = [ctypes.c_void_p]
        _LIB = lib
    return _LIB


def _ptr(a):
    return None if a is None else a.ctypes.data


def assemble_host(N, sigma=1.0, dirichlet=False, jitter=None):
    """(A_e, S, A_n, D) as canonical scipy CSR, bitwise equal to the device's."""
    N = int(N)
    jit = None if jitter is None else np.ascontiguousarray(jitter, dtype=np.float64).ravel()
    if jit is not None and jit.size != 3 * (N - 1) ** 3:
        raise ValueError("jitter must be ((N-1)^3, 3)")
    if np.ndim(sigma) == 0:
        sig, sig_c = None, float(sigma)
    else:
        sig, sig_c = np.ascontiguousarray(sigma, dtype=np.float64), 0.0
        if sig.size != N ** 3:
            raise ValueError("sigma must have one entry per hex")
    lib = _lib()
    h = lib.host_hex_create(N, int(bool(dirichlet)), _ptr(jit), _ptr(sig), sig_c)
    if not h:
        raise ValueError(f"need at least one cell per axis, got {N}")
    try:
        sz = np.zeros(5, dtype=np.int64)
        lib.host_hex_sizes(h, _ptr(sz))
        ne, nf, nnzE, nnzN, nnzD = (int(x) for x in sz)
        rpE = np.empty(ne + 1, np.int64)
        colE = np.empty(nnzE, np.int32)
        vA = np.empty(nnzE)
        vS = np.empty(nnzE)
        rpN = np.empty(nf + 1, np.int64)
        colN = np.empty(nnzN, np.int32)
        vN = np.empty(nnzN)
        rpD = np.empty(ne + 1, np.int64)
        colD = np.empty(nnzD, np.int32)
        vD = np.empty(nnzD)
        lib.host_hex_fill(h, *(_ptr(a) for a in (rpE, colE, vA, vS, rpN, colN, vN,
                                                 rpD, colD, vD)))
    finally:
        lib.host_hex_destroy(h)
    A_e = sp.csr_matrix((vA, colE, rpE), shape=(ne, ne))
    S = sp.csr_matrix((vS, colE.copy(), rpE.copy()), shape=(ne, ne))
    A_n = sp.csr_matrix((vN, colN, rpN), shape=(nf, nf))
    D = sp.csr_matrix((vD, colD, rpD), shape=(ne, nf))
    for M in (A_e, S, A_n, D):
        M.has_sorted_indices = True
    return A_e, S, A_n, D


def config_host(name, N=None):
    """(A_e, S, A_n, D, rhs, cfg) of a BASELINE config exactly as
    ``assembly.make_device_config`` builds it on the device (same draws from
    the same generator, same arithmetic)."""
    from paper_2506_08284_b200.assembly import config_draws
    cfg, sigma, jitter, rng = config_draws(name, N)
    A_e, S, A_n, D = assemble_host(cfg["N"], sigma, cfg["dirichlet"], jitter)
    rhs = rng.uniform(-1.0, 1.0, A_e.shape[0])
    return A_e, S, A_n, D, rhs, cfg
