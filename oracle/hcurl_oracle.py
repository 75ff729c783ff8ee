"""CPU restatement of the SpHcurlAMG hot path -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the B200 path. Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import it, and only as the thing compared against
or the CPU baseline, never as part of the product. The product package
(``paper_2506_08284_b200``) never imports it.

It restates the reference algorithm (``/root/reference/pkg/src/hcurlamg``),
function by function, with the reference's floating-point semantics where
they decide discrete outcomes (SURVEY.md Hazard 1):

* the Jacobi-smoothed nodal prolongator is built with the same accumulation
  orders as the reference's scipy calls (rows of ``diag(1/d) @ A`` are held in
  descending column order, sums are sequential, the power-method norms use
  a restatement of the OpenBLAS Haswell ``ddot`` kernel: ``oracle/csrc``);
* row sums follow ``np.add.reduceat`` (``a0 + pairwise(a1..)``);
* aggregation, piecewise-constant conversion and coarse-edge extraction are
  exact integer logic with the reference's tie rules.

The constrained energy minimisation uses the Gram-Cholesky form of the
reference's QR least-norm solve; that equivalence is
pinned (TOL 1e-10) by the golden fixtures.

Pinning: ``tests/golden/make_golden.py`` runs the reference itself under
``OPENBLAS_CORETYPE=Haswell OPENBLAS_NUM_THREADS=1`` and stores its outputs in
``tests/golden/*.npz``; ``tests/test_oracle.py`` checks this module against
every one of them (bit-exact for aggregates, nodal prolongators, coarse edges,
patterns and coarse counts; 1e-10 for edge prolongators and operators;
identical PCG iteration counts).

Extension beyond the reference (needed because the reference has no
parallel smoother, SURVEY.md Hazard 2): a Jacobi-preconditioned Chebyshev
sweeper (``ChebyshevSweeper``) that plugs into the reference's own sweeper
seam (``multigrid.py:79-80,167-172``). The B200 path implements the same
polynomial.
"""

import ctypes
import math
import os
import subprocess
from collections import Counter
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as la
import scipy.sparse as sp
from scipy.sparse.linalg import spsolve_triangular

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    """ctypes handle of oracle/_build/liboracle.so (built on first use)."""
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "_build", "liboracle.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-s", "-C", _HERE], check=True)
        lib = ctypes.CDLL(path)
        lib.oracle_hsw_ddot.restype = ctypes.c_double
        lib.oracle_hsw_ddot.argtypes = [ctypes.c_long, ctypes.c_void_p,
                                        ctypes.c_void_p]
        _LIB = lib
    return _LIB


# ---------------------------------------------------------------------------
# substrate (reference sparse_ops.py)


def canonical(A):
    """Sorted, duplicate-free CSR (reference sparse_ops.py:17-22)."""
    A = sp.csr_matrix(A)
    A.sum_duplicates()
    A.sort_indices()
    return A


def drop_zeros(A):
    """compress(A, 0.0) (reference sparse_ops.py:107-113)."""
    B = canonical(A).copy()
    B.eliminate_zeros()
    return B


def max_abs(A):
    A = sp.csr_matrix(A)
    return float(np.max(np.abs(A.data))) if A.nnz else 0.0


def row_ids(A):
    return np.repeat(np.arange(A.shape[0], dtype=np.int64), np.diff(A.indptr))


def hsw_dot(x, y):
    """OpenBLAS-Haswell ddot restatement (what numpy's dot runs under the
    survey's BLAS pin; reference nodal_amg.py:107,111)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    return _lib().oracle_hsw_ddot(x.size, x.ctypes.data, y.ctypes.data)


def hsw_norm(x):
    """np.linalg.norm(x) = sqrt(x . x) under the pinned BLAS."""
    return math.sqrt(hsw_dot(x, x))


def reduceat_rows(A, data=None):
    """Row sums as scipy's CSR ``sum(axis=1)`` computes them:
    ``np.add.reduceat`` = a0 + pairwise(a1, ...) per row (0 for empty rows)."""
    data = A.data if data is None else data
    out = np.zeros(A.shape[0])
    nz = np.flatnonzero(np.diff(A.indptr))
    if nz.size:
        out[nz] = np.add.reduceat(data, A.indptr[nz])
    return out


# ---------------------------------------------------------------------------
# nodal smoothed aggregation (reference nodal_amg.py)


def strength_pattern(A_n, drop_tol=0.0):
    """0/1 symmetric strength pattern incl. the diagonal (nodal_amg.py:33-56)."""
    A = canonical(A_n)
    d = A.diagonal()
    if np.any(d <= 0):
        raise ValueError(f"nonpositive diagonal entry in row "
                         f"{int(np.flatnonzero(d <= 0)[0])}")
    r = row_ids(A)
    c = A.indices.astype(np.int64)
    keep = np.abs(A.data) > drop_tol * np.sqrt(d[r] * d[c])
    n = A.shape[0]
    rr = np.concatenate([r[keep], np.arange(n)])
    cc = np.concatenate([c[keep], np.arange(n)])
    P = canonical(sp.coo_matrix((np.ones(rr.size), (rr, cc)), shape=A.shape))
    P = canonical(P + P.T)
    P.data[:] = 1.0
    return P


def aggregate(S):
    """Greedy two-phase root aggregation (nodal_amg.py:59-88).

    Phase 1: node i (index order) roots a new aggregate with its whole
    neighbourhood when none of it is aggregated yet. Phase 2: leftovers join
    the aggregate most frequent among their already-assigned neighbours,
    lowest aggregate id on ties (0 when no neighbour is assigned).
    """
    S = canonical(S)
    n = S.shape[0]
    ptr, idx = S.indptr, S.indices
    memb = np.full(n, -1, dtype=np.int64)
    n_agg = 0
    for i in range(n):
        if memb[i] >= 0:
            continue
        nb = idx[ptr[i]:ptr[i + 1]]
        if np.all(memb[nb] < 0):
            memb[nb] = n_agg
            memb[i] = n_agg
            n_agg += 1
    for i in range(n):
        if memb[i] >= 0:
            continue
        nb = idx[ptr[i]:ptr[i + 1]]
        own = memb[nb]
        own = own[(own >= 0) & (nb != i)]
        memb[i] = int(np.argmax(np.bincount(own, minlength=n_agg)))
    return memb, n_agg


def scaled_rows_desc(A):
    """diag(1/d) A with every row held in descending column order -- the
    storage scipy's ``diags(1/d) @ A`` produces (reverse first-touch)."""
    A = canonical(A)
    d = A.diagonal()
    if np.any(d == 0):
        raise ValueError("zero diagonal in nodal operator")
    inv = 1.0 / d
    r = row_ids(A)
    order = np.lexsort((-A.indices.astype(np.int64), r))
    vals = inv[r] * A.data
    return sp.csr_matrix((vals[order], A.indices[order], A.indptr.copy()),
                         shape=A.shape)


def power_rho(DA, iterations=10):
    """Ten-step power method on diag(1/d) A (nodal_amg.py:99-116)."""
    n = DA.shape[0]
    v = 1.0 + 0.01 * np.sin(np.arange(n, dtype=np.float64))
    v = v / hsw_norm(v)
    rho = 1.0
    for _ in range(iterations):
        w = DA @ v                       # csr_matvec: stored (descending) order
        nrm = hsw_norm(w)
        if nrm == 0.0:
            return 0.0
        rho = nrm
        v = w / nrm
    return float(rho)


def normalize_rows(P):
    """Unit row sums (nodal_amg.py:119-135)."""
    P = canonical(P)
    s = reduceat_rows(P)
    tol = 1e-13 * np.maximum(1.0, reduceat_rows(P, np.abs(P.data)))
    bad = np.flatnonzero(np.abs(s) <= tol)
    if bad.size:
        raise ValueError(f"zero row sum before scaling in row {bad[0]}")
    out = P.copy()
    out.data = (1.0 / s)[row_ids(P)] * P.data
    out.eliminate_zeros()          # diags(1/s) @ P drops exact-zero products
    return out


def smoothed_prolongator(A_n, memb, n_agg):
    """P = normalize((I - w D^-1 A) P_tent), w = 4/(3 rho)
    (nodal_amg.py:138-155). Returns (P, omega, rho)."""
    A = canonical(A_n)
    DA = scaled_rows_desc(A)
    rho = power_rho(DA)
    omega = 4.0 / (3.0 * rho)          # ZeroDivisionError for rho == 0, as reference
    n = A.shape[0]
    Pt = sp.csr_matrix((np.ones(n), memb.copy(), np.arange(n + 1)),
                       shape=(n, n_agg))
    X = canonical(DA @ Pt)              # sequential sums in descending k
    r = row_ids(X)
    y = np.where(X.indices == memb[r], 1.0, 0.0) - omega * X.data
    P = sp.csr_matrix((y, X.indices.copy(), X.indptr.copy()), shape=X.shape)
    P.eliminate_zeros()
    return normalize_rows(P), omega, rho


# ---------------------------------------------------------------------------
# coarse topology (reference coarse_gradient.py)


def piecewise_const(P, n_passes=2):
    """Algorithm 1: one unit entry per row (coarse_gradient.py:36-103).
    Returns the column assigned to each row."""
    P = canonical(P)
    m_h, m_H = P.shape
    Pc = canonical(P.T)
    col_nnz = np.diff(Pc.indptr)
    if np.any(col_nnz == 0):
        raise ValueError(f"empty column {int(np.flatnonzero(col_nnz == 0)[0])} "
                         "cannot be assigned any row")
    targets = np.maximum(1, np.rint(col_nnz / col_nnz.sum() * m_h).astype(np.int64))
    assign = np.full(m_h, -1, dtype=np.int64)

    def col(j):
        s = slice(Pc.indptr[j], Pc.indptr[j + 1])
        return Pc.indices[s].astype(np.int64), np.abs(Pc.data[s])

    for _ in range(n_passes):
        for j in range(m_H):
            rows, mags = col(j)
            free = assign[rows] < 0
            rows, mags = rows[free], mags[free]
            if rows.size == 0:
                continue
            take = -(-targets[j] // n_passes)
            sel = np.lexsort((rows, -mags))[:take]   # |P| desc, row asc
            assign[rows[sel]] = j
    counts = np.bincount(assign[assign >= 0], minlength=m_H)
    for i in np.flatnonzero(assign < 0):
        s = slice(P.indptr[i], P.indptr[i + 1])
        cols = P.indices[s].astype(np.int64)
        mags = np.abs(P.data[s])
        if cols.size == 0:
            raise ValueError(f"row {i} has no entries to assign")
        claimed = counts[cols] > 0
        if np.any(claimed):
            cols, mags = cols[claimed], mags[claimed]
        j = int(cols[np.lexsort((cols, -mags))[0]])
        assign[i] = j
        counts[j] += 1
    for j in np.flatnonzero(counts == 0):
        rows, mags = col(j)
        donor = counts[assign[rows]] > 1
        rows, mags = rows[donor], mags[donor]
        if rows.size == 0:
            raise ValueError(f"empty column {j} cannot be assigned any row")
        rr = int(rows[np.lexsort((rows, -mags))[0]])
        counts[assign[rr]] -= 1
        assign[rr] = j
        counts[j] += 1
    return assign


@dataclass
class CoarseEdges:
    """Coarse edge list: interior pairs (a < b) sorted, then single-node
    edges sorted by node (coarse_gradient.py:106-160), then the interior
    edges ``make_irreducible`` appended, in append order
    (coarse_gradient.py:163-171; duplicates of an existing pair allowed, as
    in the reference)."""

    pairs: np.ndarray           # (n_int, 2)
    singles: np.ndarray         # (n_single,)
    n_nodes: int
    augmented: np.ndarray = None  # (n_aug, 2), a < b

    def __post_init__(self):
        if self.augmented is None:
            self.augmented = np.zeros((0, 2), dtype=np.int64)

    @property
    def n_edges(self):
        return self.pairs.shape[0] + self.singles.size + self.augmented.shape[0]

    def endpoints(self):
        """Endpoint tuples by edge id (CoarseGradient.edge_endpoints)."""
        return ([(int(a), int(b)) for a, b in self.pairs]
                + [(int(c),) for c in self.singles]
                + [(int(a), int(b)) for a, b in self.augmented])

    def D_H(self):
        ni, ns = self.pairs.shape[0], self.singles.size
        na_ = self.augmented.shape[0]
        e = np.arange(ni)
        ea = ni + ns + np.arange(na_)
        rows = np.concatenate([e, e, ni + np.arange(ns), ea, ea])
        cols = np.concatenate([self.pairs[:, 0], self.pairs[:, 1], self.singles,
                               self.augmented[:, 0], self.augmented[:, 1]])
        vals = np.concatenate([-np.ones(ni), np.ones(ni), np.ones(ns),
                               -np.ones(na_), np.ones(na_)])
        return canonical(sp.coo_matrix((vals, (rows, cols)),
                                       shape=(self.n_edges, self.n_nodes)))


def coarse_edges(D_h, assign, n_agg):
    """Coarse edges = strictly-upper pattern of P^T|D|^T|D|P (one per pair of
    aggregates joined by a fine edge with two free ends), plus one single-node
    edge per aggregate owning the free end of a one-entry gradient row."""
    D = canonical(D_h)
    nnz = np.diff(D.indptr)
    two = np.flatnonzero(nnz == 2)
    a = assign[D.indices[D.indptr[two]]]
    b = assign[D.indices[D.indptr[two] + 1]]
    m = a != b
    lo, hi = np.minimum(a[m], b[m]), np.maximum(a[m], b[m])
    keys = np.unique(lo.astype(np.int64) * n_agg + hi)
    pairs = np.column_stack([keys // n_agg, keys % n_agg]).astype(np.int64)
    one = np.flatnonzero(nnz == 1)
    singles = np.unique(assign[D.indices[D.indptr[one]]]).astype(np.int64)
    return CoarseEdges(pairs=pairs, singles=singles, n_nodes=n_agg)


# ---------------------------------------------------------------------------
# constrained energy minimisation (reference emin_setup.py, edge_prolongator.py)


def _components(ends, I, J):
    """Union-find over the row's coarse nodes J; two-node coarse edges join
    their ends, one-node edges only mark incidence (emin_setup.py:150-171)."""
    pos = {int(c): x for x, c in enumerate(J)}
    parent = list(range(len(J)))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    inc = [False] * len(J)
    for e in I:
        ps = [pos[n] for n in ends[int(e)]]
        for p in ps:
            inc[p] = True
        if len(ps) == 2:
            x, y = find(ps[0]), find(ps[1])
            if x != y:
                parent[max(x, y)] = min(x, y)
    return [find(c) for c in range(len(J))], inc


def _irreducible(ends, I, J, cache=None):
    """check_irreducible (emin_setup.py:174-180); ``cache`` memoises it by
    the block's local structure (the reference's blocks repeat heavily)."""
    if len(J) == 0:
        return False
    if cache is not None:
        pos = {c: x for x, c in enumerate(J)}
        key = (len(J), tuple(tuple(pos[n] for n in ends[e]) for e in I))
        hit = cache.get(key)
        if hit is None:
            roots, inc = _components(ends, I, J)
            hit = cache[key] = all(inc) and len(set(roots)) == 1
        return hit
    roots, inc = _components(ends, I, J)
    return all(inc) and len(set(roots)) == 1


def _column_score(Rc, a, b):
    """|R_dp[:, a] . R_dp[:, b]| as the reference evaluates it
    (emin_setup.py:206): scipy csr_matmat of the transposed column a with
    column b, i.e. products summed sequentially from 0.0 in ascending fine
    edge, unfused; an exactly-zero sum scores 0."""
    sa = slice(Rc.indptr[a], Rc.indptr[a + 1])
    sb = slice(Rc.indptr[b], Rc.indptr[b + 1])
    ka, kb = Rc.indices[sa], Rc.indices[sb]
    _, ia, ib = np.intersect1d(ka, kb, assume_unique=True, return_indices=True)
    va, vb = Rc.data[sa][ia], Rc.data[sb][ib]
    s = 0.0
    for x, y in zip(va.tolist(), vb.tolist()):
        s += x * y
    return abs(s)


def make_irreducible(edge, I, J, ends, aug, Rc, score_cache):
    """Append coarse edges until the row's block is irreducible
    (emin_setup.py:183-217, coarse_gradient.py:163-171).

    Each step bridges two components with the pair (a, b), a < b in J order,
    of largest |R_dp[:, a] . R_dp[:, b]|; ties and zero scores go to the
    lexicographically smallest (a, b). The new edge takes the next id
    (``ends``/``aug`` grow; an existing pair may be appended again, as in
    the reference). Returns the grown edge list."""
    I = list(I)
    while not _irreducible(ends, I, J):
        roots, _ = _components(ends, I, J)
        if len(set(roots)) <= 1:
            raise ValueError(f"fine edge {edge}: cannot repair a single-node "
                             "constraint graph")
        best = None
        for ai in range(len(J)):
            for bi in range(ai + 1, len(J)):
                if roots[ai] == roots[bi]:
                    continue
                a, b = int(J[ai]), int(J[bi])
                sc = score_cache.get((a, b))
                if sc is None:
                    sc = score_cache[(a, b)] = _column_score(Rc, a, b)
                key = (-sc, a, b)
                if best is None or key < best:
                    best = key
        _, a, b = best
        ends.append((min(a, b), max(a, b)))
        aug.append((min(a, b), max(a, b)))
        I.append(len(ends) - 1)
    return I


def _rank_check(G, k, edge):
    """The reference's QR rank test (emin_setup.py:229-241)."""
    R = np.linalg.qr(G, mode="r")
    dg = np.abs(np.diag(R))
    scale = dg[0] if dg.size else 0.0
    if k < 1 or k > dg.size or scale == 0.0 or np.any(dg[:k] < 1e-10 * scale):
        raise ValueError(f"fine edge {edge}: numerical rank below the expected "
                         f"{k} (topology bug)")
    if dg.size > k and dg[k] >= 1e-10 * scale:
        raise ValueError(f"fine edge {edge}: constraint block rank exceeds the "
                         f"expected {k} (topology bug)")


def jacobi_diag(S):
    d = S.diagonal().copy()
    top = d.max() if d.size else 0.0
    if top <= 0.0:
        raise ValueError("curl-curl diagonal is entirely zero")
    d[d == 0.0] = 1e-12 * top
    return d


@dataclass
class EminResult:
    P_e: sp.csr_matrix
    energy_history: list
    commutator_residual: float
    subproblem_dims: Counter
    n_augmented: int = 0
    R_dp: sp.csr_matrix = None
    coarse: "CoarseEdges" = None


def emin_prolongator(D_h, P_n, ce, S, omega=0.5, iterations=1):
    """Pattern, irreducibility repair, feasible guess and projected Jacobi
    sweeps (emin_setup.py:62-336, edge_prolongator.py:104-228). The coarse
    edges make_irreducible appends come back in ``result.coarse``."""
    D = canonical(D_h)
    nnz = np.diff(D.indptr)
    badm = (nnz < 1) | (nnz > 2)
    if np.any(badm):
        b = int(np.flatnonzero(badm)[0])
        raise ValueError(f"malformed gradient: row {b} has {nnz[b]} nonzeros")
    P_n = canonical(P_n)
    R = canonical(D @ P_n)
    Rc = None
    rdp_scale = max(1.0, float(np.max(np.abs(R.data))) if R.nnz else 1.0)
    ni = ce.pairs.shape[0]
    adj = {(int(a), int(b)): e for e, (a, b) in enumerate(ce.pairs)}
    single = np.full(ce.n_nodes, -1, dtype=np.int64)
    single[ce.singles] = ni + np.arange(ce.singles.size)
    ends = ce.endpoints()
    n0 = len(ends)
    aug = [tuple(int(v) for v in e) for e in ce.augmented]
    n_aug_in = len(aug)
    score_cache, irr_cache = {}, {}

    n = D.shape[0]
    rows_I, rows_J, rows_N, rows_r = [None] * n, [None] * n, [None] * n, [None] * n

    # main loop (emin_setup.py:291-309)
    for i in range(n):
        ends_i = D.indices[D.indptr[i]:D.indptr[i + 1]]
        J = np.unique(np.concatenate([P_n.indices[P_n.indptr[e]:P_n.indptr[e + 1]]
                                      for e in ends_i])).astype(np.int64)
        Jl = J.tolist()
        I = [adj[(a, b)] for x, a in enumerate(Jl) for b in Jl[x + 1:]
             if (a, b) in adj]
        I += [int(single[c]) for c in Jl if single[c] >= 0]
        I.sort()
        s = slice(R.indptr[i], R.indptr[i + 1])
        r = np.zeros(J.size)
        r[np.searchsorted(J, R.indices[s])] = R.data[s]
        rows_J[i], rows_N[i], rows_r[i] = J, I, r
        if not I:
            if not np.any(np.abs(R.data[s]) > 1e-12 * rdp_scale):
                continue
            # _empty_shell (emin_setup.py:134-147)
            if J.size == 0:
                raise ValueError(f"fine edge {i} has an empty constraint "
                                 "pattern (isolated edge or pattern bug)")
            if J.size == 1:
                raise ValueError(
                    f"fine edge {i}: nonzero commutator row over a single "
                    "coarse node cannot be satisfied by interior coarse edges")
        if not _irreducible(ends, I, Jl, irr_cache):
            if Rc is None:
                Rc = R.tocsc()
                Rc.sort_indices()
            I = make_irreducible(i, I, Jl, ends, aug, Rc, score_cache)
        rows_I[i] = I

    # post pass (emin_setup.py:311-333): the main loop's new edges join
    # every row that sees both of their ends
    new_edges = list(range(n0, len(ends)))
    if new_edges:
        by_node = {}
        for e in new_edges:
            for c in ends[e]:
                by_node.setdefault(c, []).append(e)
        affected = []
        for i in range(n):
            Jset = set(rows_J[i].tolist())
            hit = False
            for c in Jset:
                for e in by_node.get(c, ()):
                    if all(x in Jset for x in ends[e]):
                        hit = True
                        break
                if hit:
                    break
            if hit:
                affected.append(i)
        for i in affected:
            if rows_I[i] is None:
                continue
            Jl = rows_J[i].tolist()
            Jset = set(Jl)
            add = [e for e in new_edges if all(x in Jset for x in ends[e])]
            I = sorted(set(rows_N[i]) | set(add))
            if not I:
                raise ValueError(f"fine edge {i} has an empty constraint "
                                 "pattern (isolated edge or pattern bug)")
            if len(I) == len(rows_I[i]):
                continue
            if not _irreducible(ends, I, Jl):
                I = make_irreducible(i, I, Jl, ends, aug, Rc, score_cache)
            rows_I[i] = I

    # factors (factor_subproblem, emin_setup.py:220-248; cached per block)
    n_single_end = ni + ce.singles.size
    factors, rows_p = [None] * n, [None] * n
    cache = {}
    dims = Counter()
    for i in range(n):
        I = rows_I[i]
        if I is None:
            continue
        J = rows_J[i]
        pos = {int(c): x for x, c in enumerate(J.tolist())}
        G = np.zeros((len(I), J.size))
        for x, e in enumerate(I):
            en = ends[e]
            if len(en) == 2:
                G[x, pos[en[0]]] = -1.0
                G[x, pos[en[1]]] = 1.0
            else:
                G[x, pos[en[0]]] = 1.0
        dirich = any(ni <= e < n_single_end for e in I)
        key = (G.shape, G.tobytes(), dirich)
        fac = cache.get(key)
        if fac is None:
            k = J.size - (0 if dirich else 1)
            _rank_check(G, k, i)
            Gk = G[:, :k]
            Minv = np.linalg.inv(Gk.T @ Gk)
            fac = (Gk, Minv, G.T @ np.ones(len(I)), k)
            cache[key] = fac
        Gk, Minv, gt1, k = fac
        c = rows_r[i] - gt1
        rows_p[i] = 1.0 + Gk @ (Minv @ c[:k])
        rows_I[i] = np.array(I, dtype=np.int64)
        factors[i] = fac
        dims[(len(I), J.size)] += 1
    ce = CoarseEdges(pairs=ce.pairs, singles=ce.singles, n_nodes=ce.n_nodes,
                     augmented=np.array(aug, dtype=np.int64).reshape(-1, 2))

    lengths = np.array([0 if x is None else x.size for x in rows_I], dtype=np.int64)
    indptr = np.concatenate([[0], np.cumsum(lengths)])
    used = [x for x in rows_I if x is not None]
    indices = np.concatenate(used) if used else np.zeros(0, dtype=np.int64)
    vals = np.concatenate([x for x in rows_p if x is not None]) if used else np.zeros(0)
    shape = (n, ce.n_edges)
    rows = np.repeat(np.arange(n, dtype=np.int64), lengths)
    keys = rows * shape[1] + indices

    def on_pattern(A):
        A = canonical(A)
        out = np.zeros(indices.size)
        ka = row_ids(A) * shape[1] + A.indices.astype(np.int64)
        p = np.clip(np.searchsorted(keys, ka), 0, max(keys.size - 1, 0))
        ok = (keys.size > 0) & (keys[p] == ka)
        out[p[ok]] = A.data[ok]
        return out

    def mat(v):
        return sp.csr_matrix((v.copy(), indices, indptr), shape=shape)

    def energy(v):
        return float(np.sum(v * on_pattern(S @ mat(v))))

    energy_hist = []
    if iterations:
        dinv = 1.0 / jacobi_diag(S)
        energy_hist.append(energy(vals))
        for _ in range(iterations):
            SP = canonical(S @ mat(vals))
            SP.data = dinv[row_ids(SP)] * SP.data
            dv = on_pattern(SP)
            for i in range(n):
                if factors[i] is None:
                    continue
                Gk, Minv, _, _ = factors[i]
                s = slice(indptr[i], indptr[i + 1])
                d = dv[s]
                dv[s] = d - Gk @ (Minv @ (Gk.T @ d))
            vals = vals - omega * dv
            energy_hist.append(energy(vals))
    P_e = mat(vals)
    res = max_abs(canonical(P_e @ ce.D_H() - R))
    return EminResult(P_e=P_e, energy_history=energy_hist,
                      commutator_residual=res, subproblem_dims=dims,
                      n_augmented=ce.augmented.shape[0] - n_aug_in, R_dp=R,
                      coarse=ce)


# ---------------------------------------------------------------------------
# smoothers


class GaussSeidelSweeper:
    """Symmetric Gauss-Seidel through triangular solves
    (reference multigrid.py:32-59)."""

    def __init__(self, A):
        A = canonical(A)
        d = A.diagonal()
        if np.any(d == 0.0):
            raise ValueError(f"zero diagonal entry in row "
                             f"{int(np.flatnonzero(d == 0.0)[0])}")
        self.A = A
        self.L = canonical(sp.tril(A, format="csr"))
        self.U = canonical(sp.triu(A, format="csr"))

    def symmetric(self, x, b, sweeps=1):
        for _ in range(sweeps):
            x = x + spsolve_triangular(self.L, b - self.A @ x, lower=True)
            x = x + spsolve_triangular(self.U, b - self.A @ x, lower=False)
        return x


def cheb_start_vector(n):
    """Deterministic start vector in [-1, 1): splitmix64 of the index."""
    z = np.arange(n, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    z = z ^ (z >> np.uint64(31))
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53) * 2.0 - 1.0


CHEB_POWER_ITERS = 15
CHEB_SAFETY = 1.1
CHEB_RATIO = 30.0


def lanczos_max(A, d, k):
    """Largest Ritz value of k Lanczos steps on D^-1 A in the D inner product
    (start vector cheb_start_vector; the B200 ChebyshevSweeper._bounds runs
    the same recurrence with device scalars)."""
    n = A.shape[0]
    if n == 0:
        return 1.0
    w = cheb_start_vector(n)
    v = w / np.sqrt(w @ (d * w))
    vprev = np.zeros(n)
    alpha, beta = [], [0.0]
    for j in range(k):
        u = A @ v
        a = float(u @ v)
        w = (1.0 / d) * u - a * v - beta[-1] * vprev
        b = float(np.sqrt(w @ (d * w)))
        alpha.append(a)
        beta.append(b)
        if not b > 0.0:
            break
        vprev, v = v, w / b
    m = len(alpha)
    T = np.diag(alpha) + np.diag(beta[1:m], 1) + np.diag(beta[1:m], -1)
    return float(np.linalg.eigvalsh(T)[-1])


class ChebyshevSweeper:
    """Jacobi-preconditioned Chebyshev polynomial smoother of degree ``degree``
    on [hi/30, hi], hi = 1.1 * (15-step Lanczos estimate of rho(D^-1 A)).
    ``symmetric(x, b)`` applies the polynomial once (a symmetric operator), in
    the reference sweeper seam. Same recurrence as the B200 kernel chain."""

    def __init__(self, A, degree=3):
        A = canonical(A)
        d = A.diagonal()
        if np.any(d == 0.0):
            raise ValueError(f"zero diagonal entry in row "
                             f"{int(np.flatnonzero(d == 0.0)[0])}")
        self.A = A
        self.dinv = 1.0 / d
        self.degree = degree
        self.hi = 0.0
        lam = lanczos_max(A, d, CHEB_POWER_ITERS)
        self.hi = CHEB_SAFETY * lam
        self.lo = self.hi / CHEB_RATIO

    def coefficients(self):
        """[(c_d, c_r)] per step: d <- c_d d + c_r D^-1 (b - A x); x += d."""
        theta = 0.5 * (self.hi + self.lo)
        delta = 0.5 * (self.hi - self.lo)
        sigma = theta / delta
        out = [(0.0, 1.0 / theta)]
        rho = 1.0 / sigma
        for _ in range(1, self.degree):
            rn = 1.0 / (2.0 * sigma - rho)
            out.append((rn * rho, 2.0 * rn / delta))
            rho = rn
        return out

    def symmetric(self, x, b, sweeps=1):
        x = np.array(x, dtype=np.float64)
        for _ in range(sweeps):
            d = np.zeros_like(x)
            for cd, cr in self.coefficients():
                d = cd * d + cr * (self.dinv * (b - self.A @ x))
                x = x + d
        return x


# ---------------------------------------------------------------------------
# hierarchy, V-cycle, PCG (reference multigrid.py)


@dataclass
class Level:
    A_e: sp.csr_matrix
    S_e: sp.csr_matrix
    D: sp.csr_matrix
    nodal_aux: sp.csr_matrix
    P_e: sp.csr_matrix = None
    P_n: sp.csr_matrix = None
    membership: np.ndarray = None
    assignment: np.ndarray = None
    coarse: CoarseEdges = None
    omega: float = 0.0
    rho: float = 0.0
    emin: EminResult = None
    edge_sweeper: object = None
    aux_sweeper: object = None


@dataclass
class Hierarchy:
    levels: list
    coarse_lu: tuple
    operator_complexity: float


def check_nullspace(S, D, where):
    defect = max_abs(canonical(S @ D))
    scale = max(max_abs(S), 1e-300)
    if defect > 1e-10 * scale:
        raise ValueError(f"curl null-space identity violated on {where}: "
                         f"max|S D| = {defect:.3e} vs max|S| = {scale:.3e}")


def make_sweeper(A, smoother, degree):
    if smoother == "gs":
        return GaussSeidelSweeper(A)
    return ChebyshevSweeper(A, degree)


def tentative_prolongator(memb, n_agg):
    """Piecewise-constant transfer, one unit entry per row (nodal_amg.py:91-96)."""
    n = memb.size
    return sp.csr_matrix((np.ones(n), memb.copy(), np.arange(n + 1)), shape=(n, n_agg))


def build_hierarchy(A_e, S_e, A_n, D, coarse_size=200, max_levels=10,
                    omega=0.5, iterations=1, n_passes=2, drop_tol=0.0,
                    smoother="gs", degree=3, mode="sphcurl"):
    """Galerkin hierarchy (multigrid.py:119-161) with the selected sweeper.
    mode="rsamg" (edge_prolongator.py:200-213): the nodal transfer is the
    tentative prolongator itself (omega = rho = 0) and no emin sweeps run."""
    A_e, S_e, A_n, D = (canonical(X) for X in (A_e, S_e, A_n, D))
    check_nullspace(S_e, D, "the fine level")
    levels = []

    def level(A, S, Dm, **kw):
        aux = canonical(Dm.T @ (A @ Dm))
        lv = Level(A_e=A, S_e=S, D=Dm, nodal_aux=aux, **kw)
        lv.edge_sweeper = make_sweeper(A, smoother, degree)
        lv.aux_sweeper = make_sweeper(aux, smoother, degree)
        return lv

    while A_e.shape[0] > coarse_size and len(levels) < max_levels - 1:
        memb, n_agg = aggregate(strength_pattern(A_n, drop_tol))
        if mode == "rsamg":
            P_n, w, rho = tentative_prolongator(memb, n_agg), 0.0, 0.0
        else:
            P_n, w, rho = smoothed_prolongator(A_n, memb, n_agg)
        assign = piecewise_const(P_n, n_passes)
        ce = coarse_edges(D, assign, n_agg)
        em = emin_prolongator(D, P_n, ce, S_e, omega,
                              0 if mode == "rsamg" else iterations)
        ce = em.coarse                  # with make_irreducible's new edges
        nH = ce.n_edges
        if nH == 0:
            break
        if nH >= 0.9 * A_e.shape[0]:
            raise ValueError(f"coarsening stagnated: {nH} coarse edges from "
                             f"{A_e.shape[0]} fine edges")
        P = em.P_e
        levels.append(level(A_e, S_e, D, P_e=P, P_n=P_n, membership=memb,
                            assignment=assign, coarse=ce, omega=w, rho=rho,
                            emin=em))
        A_e = drop_zeros(P.T @ (A_e @ P))
        S_e = drop_zeros(P.T @ (S_e @ P))
        A_n = drop_zeros(P_n.T @ (A_n @ P_n))
        D = ce.D_H()
        check_nullspace(S_e, D, f"level {len(levels)}")
    levels.append(level(A_e, S_e, D))
    lu = la.lu_factor(A_e.toarray())
    oc = sum(lv.A_e.nnz for lv in levels) / levels[0].A_e.nnz
    return Hierarchy(levels=levels, coarse_lu=lu, operator_complexity=oc)


def fine_level(A_e, S_e, D, smoother="gs", degree=3):
    """Single smoothing level without transfers (multigrid.py:204-207)."""
    A, S, Dm = canonical(A_e), canonical(S_e), canonical(D)
    aux = canonical(Dm.T @ (A @ Dm))
    lv = Level(A_e=A, S_e=S, D=Dm, nodal_aux=aux)
    lv.edge_sweeper = make_sweeper(A, smoother, degree)
    lv.aux_sweeper = make_sweeper(aux, smoother, degree)
    return lv


def relax_solve(lv, b, rtol=1e-8, maxit=500):
    """PCG preconditioned by one stand-alone Hiptmair sweep
    (hiptmair_preconditioner, multigrid.py:198-201)."""
    return pcg(lv.A_e, b, lambda r: hiptmair(lv, np.zeros(r.size), r), rtol, maxit)


def hiptmair(lv, x, b):
    x = lv.edge_sweeper.symmetric(x, b)
    r = b - lv.A_e @ x
    c = lv.aux_sweeper.symmetric(np.zeros(lv.nodal_aux.shape[0]), lv.D.T @ r)
    x = x + lv.D @ c
    return lv.edge_sweeper.symmetric(x, b)


def v_cycle(h, b, level=0):
    """V(b) from a zero initial guess (multigrid.py:176-195)."""
    lv = h.levels[level]
    if level == len(h.levels) - 1:
        return la.lu_solve(h.coarse_lu, b)
    x = hiptmair(lv, np.zeros(b.size), b)
    rc = lv.P_e.T @ (b - lv.A_e @ x)
    x = x + lv.P_e @ v_cycle(h, rc, level + 1)
    return hiptmair(lv, x, b)


@dataclass
class PcgResult:
    x: np.ndarray
    iterations: int
    residual_history: list
    precond_history: list
    status: str
    relative_residual: float


def pcg(A, b, precond, rtol=1e-8, maxit=500):
    """PCG from x = 0 (multigrid.py:220-274); same statuses and histories."""
    A = canonical(A)
    b = np.asarray(b, dtype=np.float64)
    nb = float(np.linalg.norm(b))
    x = np.zeros(b.size)
    if nb == 0.0:
        return PcgResult(x, 0, [0.0], [0.0], "converged", 0.0)
    r = b.copy()
    z = precond(r)
    p = z.copy()
    rz = float(r @ z)
    hist = [float(np.linalg.norm(r))]
    phist = [math.sqrt(max(rz, 0.0))]
    status, its = "maxit", 0
    for k in range(maxit):
        Ap = A @ p
        pAp = float(p @ Ap)
        if pAp <= 0.0:
            status = "indefinite"
            break
        a = rz / pAp
        xn = x + a * p
        if np.array_equal(xn, x):
            status, its = "stagnated", k + 1
            hist.append(float(np.linalg.norm(b - A @ xn)))
            phist.append(phist[-1])
            break
        x = xn
        r = r - a * Ap
        its = k + 1
        res = float(np.linalg.norm(r))
        hist.append(res)
        z = precond(r)
        rzn = float(r @ z)
        phist.append(math.sqrt(max(rzn, 0.0)))
        if res <= rtol * nb:
            status = "converged"
            break
        rz, p = rzn, z + (rzn / rz) * p
    return PcgResult(x, its, hist, phist, status, hist[-1] / nb)


def solve(h, b, rtol=1e-8, maxit=500):
    return pcg(h.levels[0].A_e, b, lambda r: v_cycle(h, r), rtol, maxit)
