"""Host pass for the rare constraint blocks that need new coarse edges.

Reference semantics (emin_setup.py:183-217, 256-336, coarse_gradient.py:163-171):

* main loop, fine edges in ascending order: a row whose pattern block G
  (original coarse edges N_i over its node set J_i) is reducible -- or whose
  pattern is empty while its commutator row is not ("empty shell") -- gets
  coarse edges appended until it is irreducible. Each step joins the pair
  (a, b) of nodes in different components with the largest
  |(D_h P_n)[:, a] . (D_h P_n)[:, b]| (ties / zeros: lexicographically
  smallest (a, b)); the new edge takes the next id and is appended to D_H.
* post pass over every row whose J contains both ends of an edge appended in
  the main loop (ascending, skipping rows left empty): its pattern becomes
  N_i plus those edges; if that grew it, the block is re-checked and, when
  reducible, repaired again (those further edges stay local to the row).

The device kernels flag the rows (sphc_emin_count rowflag), this module runs
the sequential decisions on the few rows involved, and the appended edges go
back to the device as per-row extras (xrp / xeid) plus new D_H rows. Column
dot products are summed in ascending fine-edge order, as scipy's csr_matmat
does for the reference's ``R_dp_csc[:, a].T @ R_dp_csc[:, b]``.
"""

import numpy as np
import torch

from . import device as dv
from .device import DeviceCSR


def _rows(M, rows):
    """[(cols, vals)] of the given rows of a DeviceCSR (one batched download)."""
    if len(rows) == 0:
        return []
    r = torch.as_tensor(np.asarray(rows, dtype=np.int64), device=M.rowptr.device)
    s, e = M.rowptr[r], M.rowptr[r + 1]
    ln = e - s
    idx = torch.repeat_interleave(s, ln) + (
        torch.arange(int(ln.sum().item()), device=M.rowptr.device)
        - torch.repeat_interleave(torch.cumsum(ln, 0) - ln, ln))
    cols = M.col[idx].cpu().numpy().astype(np.int64)
    vals = M.val[idx].cpu().numpy() if M.val is not None else None
    out, o = [], 0
    for k in ln.cpu().numpy():
        out.append((cols[o:o + k], None if vals is None else vals[o:o + k]))
        o += int(k)
    return out


def _isect_sorted(ka, kb):
    """Positions (ia, ib) of the common keys of two sorted unique arrays
    (a binary-search merge: no re-sort of the concatenation)."""
    if ka.size == 0 or kb.size == 0:
        z = np.zeros(0, dtype=np.int64)
        return z, z
    idx = np.searchsorted(kb, ka)
    ok = idx < kb.size
    ok[ok] = kb[idx[ok]] == ka[ok]
    ia = np.flatnonzero(ok)
    return ia, idx[ia]


class _Graph:
    """Components / incidence of one block (edges over node set J)."""

    @staticmethod
    def analyse(I, J, ends):
        pos = {int(c): x for x, c in enumerate(J)}
        parent = list(range(len(J)))

        def find(a):
            while parent[a] != a:
                parent[a] = parent[parent[a]]
                a = parent[a]
            return a

        inc = [False] * len(J)
        for e in I:
            en = ends[int(e)]
            ps = [pos[n] for n in en]
            for p in ps:
                inc[p] = True
            if len(ps) == 2:
                x, y = find(ps[0]), find(ps[1])
                if x != y:
                    parent[max(x, y)] = min(x, y)
        roots = [find(c) for c in range(len(J))]
        irreducible = len(J) > 0 and all(inc) and len(set(roots)) == 1
        return irreducible, roots


def make_irreducible_pass(need, flags, rowmax, rdp_scale, T, pattern, cg):
    """Run the reference's repair on the flagged rows. Returns
    (augmented CoarseGradient, xrp, xeid, n_augmented)."""
    dev = T.rowptr.device
    n_e = T.shape[0]
    need_rows = np.flatnonzero(need.cpu().numpy())
    flag_h = flags.cpu().numpy()
    ea = cg.ep_a.cpu().numpy().astype(np.int64)
    eb = cg.ep_b.cpu().numpy().astype(np.int64)
    ends = [((int(a), int(b)) if a >= 0 else (int(b),)) for a, b in zip(ea, eb)]
    n0 = len(ends)
    Tt = dv.transpose(T)                  # coarse node -> (fine edges, R_dp values)
    col_cache = {}

    def column(a):
        c = col_cache.get(a)
        if c is None:
            c = col_cache[a] = _rows(Tt, [a])[0]
        return c

    def score(a, b):
        ka, va = column(a)
        kb, vb = column(b)
        ia, ib = _isect_sorted(ka, kb)
        s = 0.0
        for x, y in zip(va[ia], vb[ib]):        # ascending fine edge, unfused
            s += float(x) * float(y)
        return abs(s)

    def approx_scores(J):
        """|J| x |J| column dot products via one dense product (BLAS order)
        and the structural overlap counts; the decision is then made with
        exact ascending-order scores on the near-best candidates only."""
        cols = [column(int(a)) for a in J]
        keys = np.concatenate([c[0] for c in cols]) if len(cols) else np.zeros(0, np.int64)
        keys.sort()
        if keys.size:
            keys = keys[np.concatenate([[True], keys[1:] != keys[:-1]])]
        X = np.zeros((keys.size, len(J)))
        for q, (k, v) in enumerate(cols):
            X[np.searchsorted(keys, k), q] = v
        Z = (X != 0).astype(np.float64)
        return np.abs(X.T @ X), Z.T @ Z

    def repair(i, I, J):
        I = list(I)
        S = O = None
        while True:
            ok, roots = _Graph.analyse(I, J, ends)
            if ok:
                return I
            if len(set(roots)) <= 1:
                raise ValueError(f"fine edge {i}: cannot repair a single-node "
                                 "constraint graph")
            if S is None:
                S, O = approx_scores(J)
            cand = [(x, y) for x in range(len(J)) for y in range(x + 1, len(J))
                    if roots[x] != roots[y]]
            top = max(S[x, y] for x, y in cand)
            # near-best window far wider than the BLAS-order rounding error;
            # structurally disjoint columns score exactly 0
            near = [(x, y) for x, y in cand if S[x, y] >= top * (1.0 - 1e-9)]
            best = None
            for x, y in near:
                a, b = int(J[x]), int(J[y])
                key = (-(score(a, b) if O[x, y] > 0 else 0.0), a, b)
                if best is None or key < best:
                    best = key
            _, a, b = best
            ends.append((min(a, b), max(a, b)))
            I.append(len(ends) - 1)

    data_T = dict(zip(need_rows.tolist(), _rows(T, need_rows)))
    data_I = dict(zip(need_rows.tolist(), _rows(pattern, need_rows)))
    # every candidate endpoint of a repair is a J node of a flagged row:
    # fetch all their R_dp columns in one batched download
    nodes = sorted({int(c) for i in need_rows.tolist() for c in data_T[i][0]})
    col_cache.update(zip(nodes, _rows(Tt, nodes)))
    final = {}
    for i in need_rows.tolist():
        J = data_T[i][0]
        I0 = data_I[i][0]
        if flag_h[i] & 2 and I0.size == 0:      # empty shell (emin_setup.py:134-147)
            if J.size == 0:
                raise ValueError(f"fine edge {i} has an empty constraint pattern "
                                 "(isolated edge or pattern bug)")
            if J.size == 1:
                raise ValueError(
                    f"fine edge {i}: nonzero commutator row over a single coarse node "
                    "cannot be satisfied by interior coarse edges")
    # the main loop's greedy joins, all flagged rows at once on the device
    # (csrc/emin.cu k_emin_repair); the new edges take ids in ascending row
    # order, as the reference appends them
    nr = len(need_rows)
    rows_d = torch.from_numpy(need_rows.astype(np.int64)).to(dev)
    ncnt = torch.empty(nr, dtype=torch.int32, device=dev)
    pairs = torch.empty(nr * 31 * 2, dtype=torch.int32, device=dev)
    st = dv.Status()
    dv.call("sphc_emin_repair", nr, rows_d, T.rowptr, T.col, pattern.rowptr, pattern.col,
            cg.ep_a, cg.ep_b, Tt.rowptr, Tt.col, Tt.val, ncnt, pairs, st.t)
    cnt_h, pairs_h = dv.readback(ncnt, pairs)
    pairs_h = pairs_h.reshape(nr, 31, 2)
    for r, i in enumerate(need_rows.tolist()):
        c = int(cnt_h[r])
        if c == -1:
            raise ValueError(f"fine edge {i}: cannot repair a single-node "
                             "constraint graph")
        if c < 0:
            raise RuntimeError(f"fine edge {i}: constraint block exceeds the device "
                               "make_irreducible kernel (|J| <= 32)")
        I = data_I[i][0].tolist()
        for j in range(c):
            a, b = int(pairs_h[r, j, 0]), int(pairs_h[r, j, 1])
            ends.append((min(a, b), max(a, b)))
            I.append(len(ends) - 1)
        final[i] = I
    # appended ids per repaired row (ascending); the rows' full patterns are
    # their original rows plus these
    extras = {i: [e for e in I if e >= n0] for i, I in final.items()}
    new_edges = list(range(n0, len(ends)))
    state = None
    if new_edges:
        # post pass (emin_setup.py:311-333), vectorised: a row sees appended
        # edge e iff its J holds both ends, i.e. iff it lies in both R_dp
        # columns -- the (row, edge) pairs come straight from the column
        # intersections, sorted by row then edge
        rr, ee = [], []
        for e in new_edges:
            a, b = ends[e]
            ka = column(a)[0]
            rows_e = ka[_isect_sorted(ka, column(b)[0])[0]]
            rr.append(rows_e)
            ee.append(np.full(rows_e.size, e, dtype=np.int64))
        rr, ee = np.concatenate(rr), np.concatenate(ee)
        order = np.lexsort((ee, rr))
        rr, ee = rr[order], ee[order]
        aff, start, cnt = np.unique(rr, return_index=True, return_counts=True)
        # original pattern lengths of the affected rows (one gather)
        aff_d = torch.from_numpy(aff).to(dev)
        len0 = (pattern.rowptr[aff_d + 1] - pattern.rowptr[aff_d]).cpu().numpy()
        emptyish = (flag_h[aff] & 2).astype(bool)
        repaired = np.isin(aff, need_rows)
        # rows the main loop left empty stay empty; every other row that was
        # not repaired grows by all the edges it sees
        grown = ~repaired & ~(emptyish & (len0 == 0))
        post = []
        for x in np.flatnonzero(grown):
            i = int(aff[x])
            extras[i] = ee[start[x]:start[x] + cnt[x]].tolist()
            post.append(i)
        for x in np.flatnonzero(repaired):       # few: the main loop's rows
            i = int(aff[x])
            merged = sorted(set(extras[i]) | set(ee[start[x]:start[x] + cnt[x]].tolist()))
            if len(merged) > len(extras[i]):
                extras[i] = merged
                post.append(i)
        # grown rows: the reference re-checks them in ascending order and
        # repairs the reducible ones. The check runs on the device (the
        # refill pass flags them, emin_setup.setup_constraints); only the
        # flagged rows come back here (finish_post_pass), in the same
        # order, so the appended edge ids are the reference's.
        state = _PostState(ends, extras, n0, set(post), repair, T, pattern)
    cg2, xrp, xeid = _extras(cg, ends, extras, n0, n_e, dev)
    return cg2, xrp, xeid, len(ends) - n0, state


class _PostState:
    """What finish_post_pass needs to repair the post-pass rows the device
    found reducible."""

    def __init__(self, ends, extras, n0, post, repair, T, pattern):
        self.ends, self.extras, self.n0, self.post = ends, extras, n0, post
        self.repair, self.T, self.pattern = repair, T, pattern


def finish_post_pass(state, rows, cg0, n_e):
    """Repair the post-pass rows the device flagged reducible, ascending
    (emin_setup.py:311-333: further edges stay local to the row). Returns the
    augmented coarse gradient and per-row extras like make_irreducible_pass."""
    rows = sorted(int(r) for r in rows)
    for i in rows:
        if i not in state.post:
            raise RuntimeError(f"fine edge {i}: reducible after the make_irreducible pass "
                               "(internal error)")
    Js = _rows(state.T, rows)
    I0s = _rows(state.pattern, rows)
    for i, (J, _), (I0, _) in zip(rows, Js, I0s):
        I = state.repair(i, I0.tolist() + list(state.extras[i]), J)
        state.extras[i] = [e for e in I if e >= state.n0]
    dev = cg0.ep_a.device
    cg2, xrp, xeid = _extras(cg0, state.ends, state.extras, state.n0, n_e, dev)
    return cg2, xrp, xeid, len(state.ends) - state.n0


def _extras(cg, ends, extras, n0, n_e, dev):
    """Per-row extras (appended ids of each repaired row, ascending) and
    the coarse gradient with the appended edges."""
    rows = sorted(i for i, ex in extras.items() if ex)
    counts = np.zeros(n_e, dtype=np.int64)
    if rows:
        counts[np.asarray(rows, dtype=np.int64)] = [len(extras[i]) for i in rows]
    items = [e for i in rows for e in extras[i]]
    xrp_h = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    xrp = torch.from_numpy(xrp_h).to(dev)
    xeid = torch.from_numpy(np.asarray(items, dtype=np.int32)).to(dev)
    return _augment(cg, ends[n0:], dev), xrp, xeid


def _augment(cg, new, dev):
    """Append interior coarse edges (a, b) to D_H and the endpoint tables
    (coarse_gradient.py:163-171 append_edge)."""
    if not new:
        return cg
    from .coarse_gradient import CoarseGradient
    k = len(new)
    a = torch.tensor([e[0] for e in new], dtype=torch.int32, device=dev)
    b = torch.tensor([e[1] for e in new], dtype=torch.int32, device=dev)
    D = cg.D_H
    last = D.rowptr[-1:]
    rp = torch.cat([D.rowptr, last + 2 * torch.arange(1, k + 1, device=dev)])
    ci = torch.cat([D.col, torch.stack([a, b], 1).reshape(-1)])
    v = torch.cat([D.val, torch.tensor([-1.0, 1.0] * k, dtype=torch.float64, device=dev)])
    n = D.shape[0] + k
    return CoarseGradient(D_H=DeviceCSR(rp, ci, v, (n, D.shape[1])),
                          n_interior=cg.n_interior, n_single=cg.n_single, adj=cg.adj,
                          ep_a=torch.cat([cg.ep_a, a]), ep_b=torch.cat([cg.ep_b, b]),
                          single_id=cg.single_id,
                          augmented_edges=list(cg.augmented_edges or []) + list(new))
