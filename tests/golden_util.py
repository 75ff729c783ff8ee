"""Helpers to read the reference-generated golden fixtures (tests/golden)."""

import hashlib
import json
import os

import numpy as np
import scipy.sparse as sp

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def csr_hash(A):
    A = sp.csr_matrix(A)
    return sha(A.indptr.astype(np.int64), A.indices.astype(np.int64),
               A.data.astype(np.float64))


def load_case(name):
    with open(os.path.join(GOLDEN, f"hier_{name}.json")) as f:
        meta = json.load(f)
    arrays = dict(np.load(os.path.join(GOLDEN, f"hier_{name}.npz")))
    return meta, arrays


def golden_csr(arrays, key, shape):
    return sp.csr_matrix((arrays[key + "_data"], arrays[key + "_indices"],
                          arrays[key + "_indptr"]), shape=shape)


def inputs_table():
    with open(os.path.join(GOLDEN, "inputs.json")) as f:
        return json.load(f)


def rel_max_diff(A, B):
    """max |A - B| / max |B| over the union pattern (TOL metric)."""
    A = sp.csr_matrix(A)
    B = sp.csr_matrix(B)
    d = abs(A - B)
    scale = max(float(abs(B).max()) if B.nnz else 0.0, 1e-300)
    return (float(d.max()) if d.nnz else 0.0) / scale


CASES = ["N4n", "N6d", "N8d", "N10n", "C1", "N16n", "C2"]


RSAMG = ["R8d", "R12n", "R16d"]
RELAX = ["X8d", "X12n"]


def load_relax(name):
    with open(os.path.join(GOLDEN, f"relax_{name}.json")) as f:
        meta = json.load(f)
    return meta, dict(np.load(os.path.join(GOLDEN, f"relax_{name}.npz")))


def roundoff_pattern_diff(A, B, tol=1e-12):
    """Entries stored in exactly one of A, B: (count, max |value| / max |B|).
    rsamg's coarse patterns keep or drop entries by exact cancellation of
    values that carry the reference's QR round-off,
    so pattern parity there means: every entry in the symmetric difference
    is round-off, |a| <= tol max|B|."""
    A = sp.csr_matrix(A)
    B = sp.csr_matrix(B)
    pa = sp.csr_matrix((np.ones(A.nnz), A.indices, A.indptr), shape=A.shape)
    pb = sp.csr_matrix((np.ones(B.nnz), B.indices, B.indptr), shape=B.shape)
    only = abs(pa - pb)
    only.eliminate_zeros()
    if only.nnz == 0:
        return 0, 0.0
    mask = only.tocoo()
    va = np.asarray(A[mask.row, mask.col]).ravel()
    vb = np.asarray(B[mask.row, mask.col]).ravel()
    scale = max(float(abs(B).max()) if B.nnz else 0.0, 1e-300)
    return int(only.nnz), float(np.max(np.abs(np.concatenate([va, vb])))) / scale


def sampled_rows_vals(M, stride):
    """Values of rows 0, k, 2k, ... of a canonical scipy CSR, row-major."""
    rows = np.arange(0, M.shape[0], int(stride))
    ln = np.diff(M.indptr)[rows]
    idx = np.repeat(M.indptr[rows], ln) + (np.arange(int(ln.sum()))
                                           - np.repeat(np.cumsum(ln) - ln, ln))
    return M.data[idx]


def check_values(M, arrays, key, fro=None):
    """TOL on the stored values of ``key`` (pattern already proven equal)."""
    stride = int(arrays[key + "_stride"])
    ref = arrays[key + "_vals"]
    got = sampled_rows_vals(M, stride)
    assert got.shape == ref.shape, key
    scale = max(float(np.max(np.abs(M.data))) if M.nnz else 0.0, 1e-300)
    err = float(np.max(np.abs(got - ref))) if ref.size else 0.0
    assert err <= 1e-10 * scale, (key, err / scale)
    if fro is not None:
        assert abs(np.linalg.norm(M.data) - fro) <= 1e-10 * fro, key
    return stride


def pattern_sha(M):
    return sha(M.indptr.astype(np.int64), M.indices.astype(np.int64))


def embed_in_pattern(M, P):
    """M (pattern a subset of canonical CSR P's) on P's pattern with explicit
    zeros at the entries M lacks; returns (embedded CSR, number of entries
    added). Raises if M holds an entry outside P."""
    M = sp.csr_matrix(M)
    P = sp.csr_matrix(P)
    n = np.int64(P.shape[1])
    kp = np.repeat(np.arange(P.shape[0], dtype=np.int64), np.diff(P.indptr)) * n + P.indices
    km = np.repeat(np.arange(M.shape[0], dtype=np.int64), np.diff(M.indptr)) * n + M.indices
    pos = np.searchsorted(kp, km)
    if pos.size and (pos.max() >= kp.size or not np.array_equal(kp[pos], km)):
        raise AssertionError("pattern is not a subset")
    data = np.zeros(P.nnz)
    data[pos] = M.data
    return sp.csr_matrix((data, P.indices, P.indptr), shape=P.shape), int(P.nnz - M.nnz)


MESH = ["T9n", "T8d", "Q41d", "R33n"]
# a numerically singular coarsest operator (device parity only: the oracle's
# LU meets an exact zero pivot there, the reference's a round-off one)
MESH_SINGULAR = ["Q41s"]


def stored_inputs(arrays):
    """(A_e, S, A_n, D, rhs) of a golden that carries its own inputs (the
    reference's tet / quad / tri meshes: the repo's generators are hex only)."""
    out = []
    for k in ("A_e", "S", "A_n", "D"):
        out.append(sp.csr_matrix((arrays[f"in_{k}_data"], arrays[f"in_{k}_indices"],
                                  arrays[f"in_{k}_indptr"]),
                                 shape=tuple(int(x) for x in arrays[f"in_{k}_shape"])))
    return (*out, arrays["in_rhs"])


# non-default EminConfig / SolverConfig knobs (make_golden.py VARIANTS)
VARIANTS = ["V9a", "V9b", "V9e", "V11c", "V9d"]


def check_coarse_operator(M, L, arrays, li, key, A_struct=None):
    """A coarse A_e / S_e against its golden: pattern by sha256 and values to
    TOL. Both sides drop the EXACT zeros of P^T (X P) (compress,
    multigrid.py:150-151), and which round-off-sized entries cancel exactly
    depends on the summation order, so on a pattern mismatch the operator
    must equal the reference up to entries of magnitude <= 1e-12 max: checked
    on the stored pattern (small goldens) or, when the reference kept the
    whole structural pattern ``A_struct`` (large ones), on that pattern with
    zeros restored."""
    M = sp.csr_matrix(M)
    pre = f"L{li}_{key}"
    if pattern_sha(M) == L[f"{key}_pattern"]:
        check_values(M, arrays, pre, L[f"{key}_fro"])
        return
    if pre + "_indptr" in arrays:
        assert int(arrays[pre + "_stride"]) == 1
        ref = sp.csr_matrix((arrays[pre + "_vals"], arrays[pre + "_indices"],
                             arrays[pre + "_indptr"]), shape=M.shape)
        cnt, mag = roundoff_pattern_diff(M, ref)
        assert cnt <= max(8, ref.nnz // 100) and mag <= 1e-12, (li, key, cnt, mag)
        assert rel_max_diff(M, ref) <= 1e-10, (li, key)
        return
    assert A_struct is not None and L[f"{key}_nnz"] == A_struct.nnz, (li, key)
    E, missing = embed_in_pattern(M, A_struct)
    assert 0 < missing <= max(8, E.nnz // 1_000_000), (li, key, missing)
    assert pattern_sha(E) == L[f"{key}_pattern"], (li, key)
    check_values(E, arrays, pre, L[f"{key}_fro"])
