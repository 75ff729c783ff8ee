"""MatrixMarket ingestion of externally assembled systems (SPEC.md:594-620:
``read_matrix_market`` / ``write_matrix_market`` and the ``import`` workflow
that feeds ALEGRA-style exported (A_e, S, A_n, D) to the solver). The
reference specifies this path but does not ship it; it is host IO in front of
``build_hierarchy`` and the only way external matrices reach the B200 path.

Format: ``%%MatrixMarket matrix coordinate real general``,
1-based indices, values written with 17 significant digits so a write/read
round trip is bit-stable. Rejected with a ValueError: malformed banner or
size line, symmetric / skew / hermitian / pattern / array formats, indices
out of range (including 0), wrong entry counts.
"""

import os

import numpy as np
import scipy.sparse as sp

BANNER = "%%MatrixMarket matrix coordinate real general"


def _parse_entries(f, nnz, path):
    """(rows, cols, vals) of the remaining lines (pandas' C tokenizer with
    round-trip float parsing: large exports parse at disk speed)."""
    if nnz == 0:
        return (np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0))
    try:
        import pandas as pd
        df = pd.read_csv(f, sep=r"\s+", header=None, comment="%", engine="c",
                         dtype={0: np.int64, 1: np.int64, 2: np.float64}, na_filter=False,
                         float_precision="round_trip")
        if df.shape[1] != 3:
            raise ValueError(f"{path}: entry lines need 'row col value'")
        r, c, v = (df[k].to_numpy() for k in range(3))
    except (ValueError, TypeError) as e:
        if "entry lines" in str(e):
            raise
        raise ValueError(f"{path}: malformed entry line ({e})") from None
    return r, c, v


def read_matrix_market(path):
    """CSR matrix (canonical: sorted indices, duplicates summed) from a
    coordinate real general MatrixMarket file."""
    with open(path, "r") as f:
        head = f.readline()
        tok = head.strip().split()
        if len(tok) != 5 or tok[0] != "%%MatrixMarket" or tok[1].lower() != "matrix":
            raise ValueError(f"{path}: malformed MatrixMarket banner {head.strip()!r}")
        fmt, field, sym = (t.lower() for t in tok[2:])
        if sym != "general":
            raise ValueError(f"{path}: {sym}-format input is not supported "
                             "(write the full matrix as 'general')")
        if fmt != "coordinate" or field != "real":
            raise ValueError(f"{path}: only 'coordinate real general' is supported, "
                             f"got {fmt!r} {field!r}")
        line = f.readline()
        while line and line.lstrip().startswith("%"):
            line = f.readline()
        try:
            m, n, nnz = (int(x) for x in line.split())
        except ValueError:
            raise ValueError(f"{path}: malformed size line {line.strip()!r}") from None
        if m < 0 or n < 0 or nnz < 0:
            raise ValueError(f"{path}: negative size in {line.strip()!r}")
        r, c, v = _parse_entries(f, nnz, path)
    if r.size != nnz:
        raise ValueError(f"{path}: expected {nnz} entries, found {r.size}")
    if nnz and (r.min() < 1 or c.min() < 1 or r.max() > m or c.max() > n):
        bad = int(np.flatnonzero((r < 1) | (c < 1) | (r > m) | (c > n))[0])
        raise ValueError(f"{path}: entry {bad + 1} ({r[bad]} {c[bad]}) is out of range for a "
                         f"{m} x {n} matrix (indices are 1-based)")
    A = sp.csr_matrix((v, (r - 1, c - 1)), shape=(m, n))
    A.sum_duplicates()
    A.sort_indices()
    return A


def write_matrix_market(A, path):
    """Coordinate real general, 1-based, %.17g values (bit-stable round trip)."""
    A = sp.coo_matrix(A)
    with open(path, "w") as f:
        f.write(BANNER + "\n")
        f.write(f"{A.shape[0]} {A.shape[1]} {A.nnz}\n")
        if A.nnz:
            np.savetxt(f, np.column_stack([A.row + 1, A.col + 1, A.data]),
                       fmt=["%d", "%d", "%.17g"], delimiter=" ")


def load_system(Ae, S, An, D):
    """The import workflow's inputs: four MatrixMarket paths (or
    matrices) -> (A_e, S, A_n, D) as canonical CSR, dimensions checked. The
    fine-level null-space identity max|S D| <= 1e-10 max|S| is checked by
    build_hierarchy itself (multigrid.py:110-116), on the device."""
    mats = [read_matrix_market(x) if isinstance(x, (str, os.PathLike)) else sp.csr_matrix(x)
            for x in (Ae, S, An, D)]
    A_e, S_, A_n, D_ = mats
    n_e, n_n = D_.shape
    for name, M, shp in (("A_e", A_e, (n_e, n_e)), ("S", S_, (n_e, n_e)),
                         ("A_n", A_n, (n_n, n_n))):
        if M.shape != shp:
            raise ValueError(f"inconsistent import: {name} is {M.shape[0]} x {M.shape[1]}, "
                             f"D is {n_e} x {n_n} (expected {shp[0]} x {shp[1]})")
    return A_e, S_, A_n, D_
