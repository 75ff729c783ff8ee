"""Independent numpy assembly of the model problem on curved (jittered,
isoparametric trilinear) hex meshes -- the checker for the device generator
(csrc/assemble.cu). Test infrastructure only.

It follows the reference's factorisation S = C^T W C (assembly.py:135-144,
231-290): C is the topological face-edge incidence with the reference's
cycle orientation (right-hand rule about +axis, assembly.py:22-27), W the
face-flux mass of the contravariant-Piola Raviart-Thomas basis. The device
kernels instead take the curl of the covariant-Piola edge basis directly, so
the two agree only if the de Rham relation curl phi_e = sum_f C_fe psi_f
holds with the reference's orientations. Edge mass: covariant Piola;
nodal: trilinear stiffness + sigma mass (assembly.py:373-386,404-434). All
element integrals use 3x3x3 Gauss. At zero jitter this must reproduce the
host generator (inputs.py, bit-faithful to the reference) to rounding.
"""

import numpy as np
import scipy.sparse as sp

from paper_2506_08284_b200.inputs import _LOCAL_EDGES, build_hex_mesh

_G = 0.5 * np.sqrt(3.0 / 5.0)
_QX = np.array([0.5 - _G, 0.5, 0.5 + _G])
_QW = np.array([5.0, 8.0, 5.0]) / 18.0


def _l(d, t):
    return t if d else 1.0 - t


def _quad():
    pts, wts = [], []
    for a in range(3):
        for b in range(3):
            for c in range(3):
                pts.append((_QX[a], _QX[b], _QX[c]))
                wts.append(_QW[a] * _QW[b] * _QW[c])
    return np.array(pts), np.array(wts)


def _local_C():
    """6 x 12 face-edge incidence of one hex, faces (axis, side)."""
    loc = {ce: k for k, ce in enumerate(_LOCAL_EDGES)}
    C = np.zeros((6, 12))
    for ax, (p, q) in enumerate(((1, 2), (2, 0), (0, 1))):
        for side in range(2):
            b = side << ax
            cyc = [b, b | (1 << p), b | (1 << p) | (1 << q), b | (1 << q)]
            for k in range(4):
                a, c = cyc[k], cyc[(k + 1) % 4]
                lo, hi = min(a, c), max(a, c)
                e_ax = (hi - lo).bit_length() - 1
                C[2 * ax + side, loc[(lo, e_ax)]] = 1.0 if a < c else -1.0
    return C


def coords(mesh, jitter=None):
    n = mesh.n
    v = np.arange(mesh.n_nodes)
    X = np.column_stack([v % n, (v // n) % n, v // (n * n)]).astype(np.float64) * (1.0 / mesh.N)
    if jitter is not None:
        t = np.column_stack([v % n, (v // n) % n, v // (n * n)])
        inner = np.all((t > 0) & (t < n - 1), axis=1)
        X[inner] += np.asarray(jitter).reshape(-1, 3)
    return X


def assemble(N, sigma=1.0, dirichlet=False, jitter=None):
    """(A_e, S, A_n, D) as scipy CSR."""
    from paper_2506_08284_b200.inputs import _element_edge_ids, discrete_gradient
    mesh = build_hex_mesh(N, dirichlet)
    X = coords(mesh, jitter)
    E = mesh.hexes.shape[0]
    xc = X[mesh.hexes]                                   # (E, 8, 3)
    sig = np.broadcast_to(np.asarray(sigma, dtype=np.float64), (E,))
    pts, wts = _quad()
    Q = len(wts)
    d = np.array([[(k >> a) & 1 for a in range(3)] for k in range(8)])   # corner bits
    # trilinear shape functions and reference gradients (Q, 8), (Q, 8, 3)
    Nq = np.ones((Q, 8))
    dN = np.ones((Q, 8, 3))
    for k in range(8):
        for a in range(3):
            la = _l(d[k, a], pts[:, a])
            Nq[:, k] *= la
            for q in range(3):
                dN[:, k, q] *= (1.0 if d[k, a] else -1.0) if q == a else la
    J = np.einsum("ekp,qkr->eqpr", xc, dN)               # (E, Q, 3, 3)  dx_p/dxi_r
    det = np.linalg.det(J)
    Ji = np.linalg.inv(J)
    w = wts[None, :] * det                               # (E, Q)
    G = np.einsum("eqij,eqkj->eqik", Ji, Ji) * w[..., None, None]   # det J^-1 J^-T
    H = np.einsum("eqji,eqjk->eqik", J, J) * (wts[None, :] / det)[..., None, None]

    # edge basis on the reference cube: phi_k = e_ax * s_k(xi)
    s = np.ones((Q, 12))
    axes = np.array([ax for _, ax in _LOCAL_EDGES])
    for k, (c, ax) in enumerate(_LOCAL_EDGES):
        for b in range(3):
            if b != ax:
                s[:, k] *= _l((c >> b) & 1, pts[:, b])
    Ga = G[:, :, axes][:, :, :, axes]                    # (E, Q, 12, 12)
    Me = np.einsum("eqij,qi,qj->eij", Ga, s, s) * sig[:, None, None]
    # face basis psi_f = e_ax l_side(xi_ax), f = 2 ax + side
    psi_ax = np.array([f // 2 for f in range(6)])
    ps = np.stack([_l(f % 2, pts[:, f // 2]) for f in range(6)], axis=1)   # (Q, 6)
    Ha = H[:, :, psi_ax][:, :, :, psi_ax]
    W = np.einsum("eqfg,qf,qg->efg", Ha, ps, ps)
    C = _local_C()
    Se = np.einsum("fi,efg,gj->eij", C, W, C)
    Kn = np.einsum("eqij,qai,qbj->eab", G, dN, dN)
    Mn = np.einsum("eq,qa,qb->eab", w, Nq, Nq) * sig[:, None, None]

    ee = _element_edge_ids(mesh)
    ne = mesh.n_edges
    r = np.repeat(ee, 12, axis=1).ravel()
    c_ = np.tile(ee, (1, 12)).ravel()
    ok = (r >= 0) & (c_ >= 0)

    def asm(vals, rr, cc, shape):
        A = sp.coo_matrix((vals.ravel()[ok], (rr[ok], cc[ok])), shape=shape).tocsr()
        A.sum_duplicates()
        A.sort_indices()
        return A

    S = asm(Se, r, c_, (ne, ne))
    M = asm(Me, r, c_, (ne, ne))
    A_e = (S + M).tocsr()
    A_e.sort_indices()
    hx = mesh.hexes
    rn = np.repeat(hx, 8, axis=1).ravel()
    cn = np.tile(hx, (1, 8)).ravel()
    An = sp.coo_matrix(((Kn + Mn).ravel(), (rn, cn)), shape=(mesh.n_nodes,) * 2).tocsr()
    free = np.flatnonzero(~mesh.boundary)
    An = An[np.ix_(free, free)].tocsr()
    An.sum_duplicates()
    An.sort_indices()
    return A_e, S, An, discrete_gradient(mesh)
