"""Model-problem inputs: uniform hex mesh of the unit cube, lowest-order
Nedelec edge operators and the auxiliary nodal problem.

This is the input generator for the benchmark configs, not part of the hot
path. For a constant sigma it reproduces, bit for bit, what the reference
produces with ``build_structured_mesh(3, 'hex', N + 1, dirichlet)`` followed
by ``discretize(mesh, sigma)`` (reference ``meshing.py:61-131``,
``assembly.py:47-54``): the same node / edge / face numbering, the same
factored curl-curl ``S = C^T W C`` (``assembly.py:135-144,231-290``), the same
edge mass (``assembly.py:297-306,346-366``), nodal operator
(``assembly.py:373-386,404-434``) and discrete gradient (``assembly.py:62-79``).
Bit equality is checked against hashes of reference-assembled matrices in
``tests/golden`` (``tests/test_inputs.py``).

Extension the reference does not have (SURVEY.md Hazard 3): ``sigma`` may be a
per-element array (config 3: coefficient jump). The element mass blocks are
then scaled before the scatter.

Numbering (reference conventions):
  * node ``v = x + n*y + n*n*z`` for nodal index (x, y, z), n = N + 1;
  * edges sorted by (tail, head); for a fixed tail the x-, y-, z-edge order;
  * faces sorted by (lowest corner node, normal axis);
  * hexes in C order over (x, y, z) cell indices (z fastest).
"""

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp


def _csr(A):
    """Canonical CSR (sorted, duplicates summed) of any scipy matrix."""
    A = sp.csr_matrix(A)
    A.sum_duplicates()
    A.sort_indices()
    return A


def _coo(rows, cols, vals, shape):
    rows = np.asarray(rows).ravel()
    cols = np.asarray(cols).ravel()
    vals = np.asarray(vals, dtype=np.float64).ravel()
    ok = (rows >= 0) & (cols >= 0)
    return _csr(sp.coo_matrix((vals[ok], (rows[ok], cols[ok])), shape=shape))


@dataclass
class HexMesh:
    N: int                    # cells per axis
    dirichlet: bool
    edges: np.ndarray         # (n_e, 2) tail < head, node ids
    edge_axis: np.ndarray     # (n_e,) 0/1/2
    edge_of: np.ndarray       # (n_nodes, 3) edge id of (tail node, axis), -1 if none
    hexes: np.ndarray         # (N^3, 8) corner node ids, corner = dx + 2 dy + 4 dz
    boundary: np.ndarray      # (n_nodes,) bool, Dirichlet flags
    h: float

    @property
    def n(self):
        return self.N + 1

    @property
    def n_nodes(self):
        return self.n ** 3

    @property
    def n_edges(self):
        return self.edges.shape[0]


def build_hex_mesh(N, dirichlet=False):
    """Uniform N^3-cell hex mesh of the unit cube with canonical numbering."""
    N = int(N)
    if N < 1:
        raise ValueError(f"need at least one cell per axis, got {N}")
    n = N + 1
    nn = n ** 3
    v = np.arange(nn, dtype=np.int64)
    ix, iy, iz = v % n, (v // n) % n, v // (n * n)
    step = np.array([1, n, n * n], dtype=np.int64)
    coord = (ix, iy, iz)
    # candidate edges keyed tail*3 + axis, which is (tail, head) order
    tails, axes = [], []
    for ax in range(3):
        ok = coord[ax] < n - 1
        tails.append(v[ok])
        axes.append(np.full(int(ok.sum()), ax, dtype=np.int64))
    tails = np.concatenate(tails)
    axes = np.concatenate(axes)
    order = np.argsort(tails * 3 + axes, kind="stable")
    tails, axes = tails[order], axes[order]
    heads = tails + step[axes]

    boundary = np.zeros(nn, dtype=bool)
    if dirichlet:
        for c in coord:
            boundary |= (c == 0) | (c == n - 1)
        keep = ~(boundary[tails] & boundary[heads])
        tails, heads, axes = tails[keep], heads[keep], axes[keep]

    edge_of = np.full((nn, 3), -1, dtype=np.int64)
    edge_of[tails, axes] = np.arange(tails.size)

    c = np.arange(N, dtype=np.int64)
    cx, cy, cz = np.meshgrid(c, c, c, indexing="ij")      # C order: z fastest
    base = (cx + n * cy + n * n * cz).reshape(-1)
    corner = np.array([dx + n * dy + n * n * dz
                       for dz in (0, 1) for dy in (0, 1) for dx in (0, 1)],
                      dtype=np.int64)
    hexes = base[:, None] + corner[None, :]
    return HexMesh(N=N, dirichlet=bool(dirichlet),
                   edges=np.column_stack([tails, heads]), edge_axis=axes,
                   edge_of=edge_of, hexes=hexes, boundary=boundary,
                   h=1.0 / N)


# local hex edges in the reference's local order: corner c ascending, then
# axis x, y, z for every axis whose bit in c is clear (meshing.py:183-189)
_LOCAL_EDGES = [(c, ax) for c in range(8) for ax in range(3)
                if not (c >> ax) & 1]


def _element_edge_ids(mesh):
    ids = np.empty((mesh.hexes.shape[0], 12), dtype=np.int64)
    for k, (c, ax) in enumerate(_LOCAL_EDGES):
        ids[:, k] = mesh.edge_of[mesh.hexes[:, c], ax]
    return ids


def _hat_mass(h):
    return (h / 6.0) * np.array([[2.0, 1.0], [1.0, 2.0]])


def _hat_stiff(h):
    return (1.0 / h) * np.array([[1.0, -1.0], [-1.0, 1.0]])


def discrete_gradient(mesh):
    """Edge-to-free-node incidence: -1 at the tail, +1 at the head."""
    free = np.flatnonzero(~mesh.boundary)
    col = np.full(mesh.n_nodes, -1, dtype=np.int64)
    col[free] = np.arange(free.size)
    t, hd = col[mesh.edges[:, 0]], col[mesh.edges[:, 1]]
    e = np.arange(mesh.n_edges)
    rows = np.concatenate([e, e])
    cols = np.concatenate([t, hd])
    vals = np.concatenate([-np.ones(e.size), np.ones(e.size)])
    return _coo(rows, cols, vals, (mesh.n_edges, free.size))


def _faces(mesh):
    """Face table keyed (lowest corner, normal axis) with 4-node cycles."""
    n = mesh.n
    nn = mesh.n_nodes
    v = np.arange(nn, dtype=np.int64)
    coord = (v % n, (v // n) % n, v // (n * n))
    s = (1, n, n * n)
    keys, cycles = [], []
    # cycles follow the right-hand rule about +axis (assembly.py:22-27)
    for ax, (p, q) in enumerate(((1, 2), (2, 0), (0, 1))):
        ok = (coord[p] < n - 1) & (coord[q] < n - 1)
        b = v[ok]
        keys.append(b * 3 + ax)
        cycles.append(np.column_stack([b, b + s[p], b + s[p] + s[q], b + s[q]]))
    keys = np.concatenate(keys)
    cycles = np.concatenate(cycles)
    order = np.argsort(keys, kind="stable")
    face_id = np.full((nn, 3), -1, dtype=np.int64)
    sk = keys[order]
    face_id[sk // 3, sk % 3] = np.arange(sk.size)
    return cycles[order], face_id


def curl_curl(mesh):
    """S = C^T W C with C the face-edge cycle incidence, W the face mass."""
    cycles, face_id = _faces(mesh)
    nf = cycles.shape[0]
    eo = mesh.edge_of
    rows, cols, vals = [], [], []
    f = np.arange(nf)
    for k in range(4):
        a, b = cycles[:, k], cycles[:, (k + 1) % 4]
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        d = hi - lo
        ax = np.where(d == 1, 0, np.where(d == mesh.n, 1, 2))
        rows.append(f)
        cols.append(eo[lo, ax])
        vals.append(np.where(a < b, 1.0, -1.0))
    C = _coo(np.concatenate(rows), np.concatenate(cols), np.concatenate(vals),
             (nf, mesh.n_edges))

    h = mesh.h
    n = mesh.n
    step = (1, n, n * n)
    m1 = _hat_mass(h) * (1.0 / (h * h))
    base = mesh.hexes[:, 0]
    rows, cols, vals = [], [], []
    for ax in range(3):
        f0 = face_id[base, ax]
        f1 = face_id[base + step[ax], ax]
        sides = (f0, f1)
        for i in range(2):
            for j in range(2):
                rows.append(sides[i])
                cols.append(sides[j])
                vals.append(np.full(base.size, m1[i, j]))
    W = _coo(np.concatenate(rows), np.concatenate(cols), np.concatenate(vals),
             (nf, nf))
    S = _csr(C.T @ (W @ C))
    return _csr((S + S.T) * 0.5)


def _edge_mass_block(h):
    """12 x 12 element edge mass of the unit-tangent Nedelec basis."""
    m1 = _hat_mass(h)
    loc = np.zeros((12, 12))
    offs = []
    for c, ax in _LOCAL_EDGES:
        bits = [(c >> k) & 1 for k in range(3)]
        offs.append(tuple(bits[k] for k in range(3) if k != ax))
    for i, (_, ai) in enumerate(_LOCAL_EDGES):
        for j, (_, aj) in enumerate(_LOCAL_EDGES):
            if ai != aj:
                continue
            val = 1.0 / h
            for t in range(2):
                val *= m1[offs[i][t], offs[j][t]]
            loc[i, j] = val
    return loc


def edge_mass(mesh, sigma):
    loc = _edge_mass_block(mesh.h)
    ee = _element_edge_ids(mesh)
    rows = np.repeat(ee, 12, axis=1)
    cols = np.tile(ee, (1, 12))
    if np.ndim(sigma) == 0:
        if sigma <= 0:
            raise ValueError(f"sigma must be positive, got {sigma}")
        vals = np.broadcast_to(loc.ravel(), (ee.shape[0], 144))
        M = _coo(rows, cols, vals, (mesh.n_edges,) * 2)
        M = _csr(M * sigma)
    else:
        sig = np.asarray(sigma, dtype=np.float64)
        if np.any(sig <= 0):
            raise ValueError("sigma must be positive")
        vals = sig[:, None] * loc.ravel()[None, :]
        M = _coo(rows, cols, vals, (mesh.n_edges,) * 2)
    return _csr((M + M.T) * 0.5)


def _nodal_blocks(h):
    ms, ss = _hat_mass(h), _hat_stiff(h)

    def tensor(kind):
        out = np.array([[1.0]])
        for ax in range(3):
            out = np.kron(ss if ax == kind else ms, out)
        return out

    stiff = sum(tensor(ax) for ax in range(3))
    return stiff, tensor(-1)


def nodal_operator(mesh, sigma):
    """-Laplace + sigma * mass on the free nodes (trilinear hexes)."""
    stiff, mass = _nodal_blocks(mesh.h)
    hx = mesh.hexes
    rows = np.repeat(hx, 8, axis=1)
    cols = np.tile(hx, (1, 8))
    shape = (mesh.n_nodes,) * 2
    K = _coo(rows, cols, np.broadcast_to(stiff.ravel(), (hx.shape[0], 64)), shape)
    if np.ndim(sigma) == 0:
        if sigma < 0:
            raise ValueError(f"sigma must be nonnegative, got {sigma}")
        Mn = _coo(rows, cols, np.broadcast_to(mass.ravel(), (hx.shape[0], 64)), shape)
        A = _csr(K + sigma * Mn)
    else:
        sig = np.asarray(sigma, dtype=np.float64)
        SM = _coo(rows, cols, sig[:, None] * mass.ravel()[None, :], shape)
        A = _csr(K + SM)
    A = _csr((A + A.T) * 0.5)
    free = np.flatnonzero(~mesh.boundary)
    if free.size != mesh.n_nodes:
        A = _csr(A[np.ix_(free, free)])
    return A


@dataclass
class EddyCurrentSystem:
    """Operators of one model problem (field names follow the reference's
    ``DiscretizedSystem``, assembly.py:35-44)."""

    S: sp.csr_matrix
    M: sp.csr_matrix
    A_e: sp.csr_matrix
    A_n: sp.csr_matrix
    D: sp.csr_matrix
    sigma: object
    mesh: HexMesh = None


def discretize_hex(N, sigma, dirichlet=False):
    mesh = build_hex_mesh(N, dirichlet)
    S = curl_curl(mesh)
    M = edge_mass(mesh, sigma)
    A_n = nodal_operator(mesh, sigma)
    D = discrete_gradient(mesh)
    return EddyCurrentSystem(S=S, M=M, A_e=_csr(S + M), A_n=A_n, D=D,
                             sigma=sigma, mesh=mesh)


def sigma_jump(N, inner=1e-6, outer=1.0):
    """Config 3 field: ``inner`` on cells whose centroid lies in the centred
    cube [0.25, 0.75]^3, ``outer`` elsewhere (per hex, hex order)."""
    c = (np.arange(N) + 0.5) / N
    cx, cy, cz = np.meshgrid(c, c, c, indexing="ij")
    ins = ((cx >= 0.25) & (cx <= 0.75) & (cy >= 0.25) & (cy <= 0.75)
           & (cz >= 0.25) & (cz <= 0.75)).reshape(-1)
    return np.where(ins, inner, outer)


# The five BASELINE.json configs. This host generator has
# uniform geometry only (make_config draws C4's jitter and leaves it
# unapplied); the device generator (assembly.make_device_config) and its
# bit-identical host build (oracle/host_assembly.py) apply C4's jittered
# isoparametric hexes. C5 coarsens to 10,000 edges.
CONFIGS = {
    "C1": dict(N=16, sigma=1.0, dirichlet=True, seed=0),
    "C2": dict(N=32, sigma=1e-2, dirichlet=True, seed=1),
    "C3": dict(N=64, sigma="jump", dirichlet=False, seed=2),
    # lognormal per-element sigma; jittered hexes on the device generator
    "C4": dict(N=128, sigma="lognormal", dirichlet=False, seed=3),
    "C5": dict(N=256, sigma=1e-4, dirichlet=False, seed=4, coarse_size=10000),
}


def make_config(name, N=None):
    """(system, rhs, meta) for a named config; ``N`` overrides the size.

    C4 draws from ONE generator default_rng(3) in the order fixed by
    SURVEY.md 8(d): the interior-node jitter (n_interior x 3, drawn and not
    applied here), then sigma (lognormal, mu = ln 1e-3, s = 2, one per hex in
    hex order), then the RHS U[-1, 1]."""
    cfg = dict(CONFIGS[name])
    if N is not None:
        cfg["N"] = int(N)
    sigma = cfg["sigma"]
    rng = np.random.default_rng(cfg["seed"])
    if sigma == "jump":
        sigma = sigma_jump(cfg["N"])
    elif sigma == "lognormal":
        n_int = (cfg["N"] - 1) ** 3
        h = 1.0 / cfg["N"]
        rng.uniform(-0.2 * h, 0.2 * h, (n_int, 3))        # jitter stream (unused)
        sigma = rng.lognormal(np.log(1e-3), 2.0, cfg["N"] ** 3)
        cfg["geometry"] = "uniform (jitter drawn, not applied)"
    sysm = discretize_hex(cfg["N"], sigma, cfg["dirichlet"])
    rhs = rng.uniform(-1.0, 1.0, sysm.A_e.shape[0])
    return sysm, rhs, cfg
