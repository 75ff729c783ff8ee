"""Multilevel hierarchy, hybrid smoothing, V-cycle and PCG on the B200.

Mirror of the reference's multigrid.py: ``SolverConfig``, ``Level``,
``Hierarchy``, ``PcgResult``, ``build_hierarchy``, ``hiptmair_smooth``,
``v_cycle``, ``v_cycle_preconditioner``, ``pcg_solve`` -- same arguments,
defaults, fields and ValueError texts. Inputs may be scipy CSR / numpy (they
are uploaded) or DeviceCSR / CUDA tensors. The whole hierarchy stays in HBM;
every numeric step is a libsphcurl kernel.

Smoother: the reference's symmetric Gauss-Seidel (multigrid.py:32-59) is a
sequential triangular solve. The B200 path plugs a Jacobi-preconditioned
Chebyshev polynomial of degree 3 (SpMV only, same pass count) into the same
hybrid Hiptmair structure (multigrid.py:164-173); the oracle applies the same
polynomial in the reference's own sweeper seam for parity.
"""

import math
import os
from dataclasses import dataclass, field
from types import SimpleNamespace

import numpy as np
import torch

from . import device as dv
from .device import checked, DeviceCSR, Status, as_device_csr, call, own_csr
from .edge_prolongator import EminConfig, build_edge_prolongator
from . import trace as _trace
from .trace import phase

_NULLSPACE_TOL = 1e-10
USE_SELL = os.environ.get("SPHC_SELL", "1") != "0"
USE_GRAPH = os.environ.get("SPHC_PCG_GRAPH", "1") != "0"
# fused Chebyshev steps (csrc/sell.cu k_sell_cheb_fused): operators with at
# least as many rows as the unfused kernel runs thread-per-row on (bitwise
# identical results), L2 window budget per pass. OFF by default: measured
# slower (C4 V-cycle 11.9 ms fused vs 9.2 ms unfused) -- the dependency lag
# is a whole z-plane of edges, so the rows in flight at full occupancy
# overflow L2 before the second step re-reads them, and capping the CTAs to
# fit starves the loads. SPHC_FUSE_MB=64 enables it.
FUSE_ROWS = 256
# Levels with at least this many edges (operators streamed from HBM) keep a
# SELL mirror of A_e D and take the Hiptmair mid step fused
# (sphc_sell_hipt_mid); -1 disables it.
HIPT_MID_MIN_ROWS = int(os.environ.get("SPHC_HIPT_MID_MIN_ROWS", str(148 * 48 * 32)))
# coarsest operators up to this size take the eigendecomposition (pseudo-
# inverse) when their Cholesky factorisation breaks down; larger ones the
# shifted factorisation first
COARSE_EIGH_MAX = int(os.environ.get("SPHC_COARSE_EIGH_MAX", "2048"))
FUSE_MIN_ROWS = int(os.environ.get("SPHC_FUSE_MIN_ROWS", str(148 * 48 * 32)))
FUSE_L2_BYTES = float(os.environ.get("SPHC_FUSE_MB", "0")) * 2**20

CHEB_POWER_ITERS = 15
CHEB_SAFETY = 1.1
CHEB_RATIO = 30.0


@dataclass
class SolverConfig:
    """Hierarchy construction knobs (multigrid.py:23-29) + the smoother."""

    coarse_size: int = 200
    max_levels: int = 10
    emin: EminConfig = field(default_factory=EminConfig)
    smoother: str = "chebyshev"      # or "gauss_seidel" (the reference's own smoother)
    cheb_degree: int = 3
    # coarsest solve: "cholesky" (default) = the Jacobi-equilibrated
    # Cholesky inverse with the shifted / eigendecomposition fallbacks for
    # numerically semidefinite operators; "lu" = the reference's
    # partial-pivoting LU (multigrid.py:156-157,180-181; applied as the
    # inverse its LU solves give). On the C4 recipe at 128^3 and C5's at
    # 64^3 the LU solve of the near-singular coarsest operator makes PCG
    # diverge (500 iterations, |r|/|b| 1e3 / 7) where the Cholesky inverse
    # converges in 81 / 40 (profiles/r02_probe_coarse.txt).
    coarse_solver: str = "cholesky"

    def __post_init__(self):
        if self.smoother not in SMOOTHERS:
            raise ValueError(f"unknown smoother {self.smoother!r}; "
                             f"expected one of {sorted(SMOOTHERS)}")
        if self.coarse_solver not in ("lu", "cholesky"):
            raise ValueError(f"unknown coarse_solver {self.coarse_solver!r}")


def lanczos_max(alpha, beta):
    """Largest eigenvalue of the Lanczos tridiagonal T (alpha_1..k on the
    diagonal, beta_1..k-1 off it; beta_0 = |v_0|), truncated at the first
    breakdown (beta_j == 0)."""
    k = len(alpha)
    for j in range(1, k):
        if not beta[j] > 0.0:
            k = j
            break
    T = np.diag(alpha[:k]) + np.diag(beta[1:k], 1) + np.diag(beta[1:k], -1)
    return float(np.linalg.eigvalsh(T)[-1]) if k else 0.0


def _zero_diag_check(rows):
    if "ZERO_DIAG" in rows:
        raise ValueError(f"zero diagonal entry in row {rows['ZERO_DIAG']}")


_UNFINISHED = []


def finalize_sweepers(*extra):
    """Read the Lanczos scalars of every sweeper built so far in one host
    readback (with the deferred status checks) and form their Chebyshev
    coefficients. ``extra`` device tensors ride on the same readback; their
    host copies are returned."""
    pend = list(_UNFINISHED)
    _UNFINISHED.clear()
    live = [sw for sw in pend if sw._sc is not None]
    bws = [sw for sw in pend if getattr(sw, "_bw", None) is not None]
    tens = [sw._sc for sw in live] + [sw._bw for sw in bws] + list(extra)
    hs = dv.readback(*tens) if tens else (dv.flush_checks() or [])
    it = iter(hs)
    for sw in pend:
        sw._finish(next(it) if sw._sc is not None else None)
    for sw in bws:
        sw._plan_fusion(int(next(it)[0]))
    return list(it)


class ChebyshevSweeper:
    """Degree-d Jacobi-Chebyshev on [hi/30, hi], hi = 1.1 x (15-step Lanczos
    estimate of rho(D^-1 A)); ``symmetric(x, b)`` applies it once. Each
    polynomial step is one fused libsphcurl launch."""

    def __init__(self, A, degree=3):
        self.A = A
        n = A.shape[0]
        st = Status()
        d = dv.diagonal(A, st)
        st.defer(_zero_diag_check)
        self.dinv = dv.reciprocal(d)
        self.diag = d
        self.degree = degree
        self.lanes = A.lanes()
        # solve-phase layout of A (csrc/sell.cu) unless SPHC_SELL=0
        self.sell = dv.sell(A) if USE_SELL else None
        self.d = dv.empty_f64(n)
        self.buf = [dv.empty_f64(n), dv.empty_f64(n)]
        # the Lanczos scalars are read back together with every other
        # sweeper's of the hierarchy (finalize_sweepers)
        self.hi = self.lo = self.coefs = None
        self._sc = self._lanczos()
        # fused multi-step launches for operators streamed from HBM
        # (sphc_sell_cheb_fused): needs the matrix bandwidth, read back
        # with the Lanczos scalars
        self.fuse, self._bw = 0, None
        if self.sell is not None and n >= FUSE_MIN_ROWS and degree >= 2:
            self._bw = torch.zeros(1, dtype=torch.int64, device=d.device)
            call("sphc_csr_bandwidth", n, A.rowptr, A.col, self._bw)
        _UNFINISHED.append(self)

    def _plan_fusion(self, bw):
        """Steps per pass: the most (<= 3) whose L2 window -- (steps - 1)
        dependency ranges of row blocks -- fits FUSE_L2_BYTES."""
        self._bw = None
        n = self.A.shape[0]
        nblk = (n + FUSE_ROWS - 1) // FUSE_ROWS
        self.fuse_L = -(-bw // FUSE_ROWS) + 1
        per_blk = 12.0 * self.sell.padded / nblk
        self.fuse = 0
        for ks in (3, 2):
            if ks <= self.degree and (ks - 1) * (self.fuse_L + 1) * per_blk <= FUSE_L2_BYTES:
                self.fuse = ks
                break
        if self.fuse:
            self.fuse_sync = torch.empty(1 + self.fuse * nblk, dtype=torch.int32,
                                         device=self.d.device)

    def _finish(self, sc):
        k = CHEB_POWER_ITERS
        lam = lanczos_max(*np.split(sc, [k])) if sc is not None else 1.0 / CHEB_SAFETY
        self.hi = CHEB_SAFETY * lam
        self.lo = self.hi / CHEB_RATIO
        self.coefs = self._coefficients()
        self._sc = None

    def _lanczos(self):
        """hi = 1.1 x the largest Ritz value of a 15-step Lanczos run on
        D^-1 A (self-adjoint in the D inner product). A power method of the
        same length underestimates rho(D^-1 A) by >10% on curved meshes with
        rough sigma (C4), which makes the polynomial amplify the top modes
        and the V-cycle indefinite; Lanczos converges to the extreme
        eigenvalue much faster. All scalars stay on the device; one host
        read per smoother."""
        n = self.A.shape[0]
        if n == 0:
            return None
        k = CHEB_POWER_ITERS
        d = self.diag
        v, vprev = self.buf
        sc = dv.empty_f64(2 * k + 1)            # [alpha_1..k | beta_0..k]
        m = self.sell
        if m is not None:
            # all k steps in one cooperative launch (csrc/sell.cu)
            u, w = dv.empty_f64(n), dv.empty_f64(n)
            call("sphc_lanczos_sell", n, m.slice_ptr, m.col, m.val, d, self.dinv, k, v, vprev,
                 w, u, sc)
            return sc
        u, w, dw = dv.empty_f64(n), dv.empty_f64(n), dv.empty_f64(n)
        alpha, beta = sc[:k], sc[k:]
        call("sphc_cheb_start", n, w)
        call("sphc_diag_scale", n, d, w, dw)
        sq = dv.empty_f64(1)
        dv.dot(w, dw, sq)
        call("sphc_scale_by_norm", n, w, sq, v, beta[0:1])
        for j in range(k):
            dv.spmv(self.A, v, u, lanes=self.lanes)
            dv.dot(u, v, alpha[j:j + 1])
            call("sphc_lanczos_update", n, u, self.dinv, d, v, vprev if j else None,
                 alpha[j:j + 1], beta[j:j + 1] if j else None, w, dw)
            dv.dot(w, dw, sq)
            vprev, v = v, vprev
            call("sphc_scale_by_norm", n, w, sq, v, beta[j + 1:j + 2])
        return sc

    def _coefficients(self):
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

    def symmetric(self, x, b, sweeps=1, x_zero=False):
        """Returns the smoothed iterate (a sweeper-owned buffer, never ``x``)."""
        if self.coefs is None:
            finalize_sweepers()
        A = self.A
        n = A.shape[0]
        cur = x
        if self.fuse:
            for _ in range(sweeps):
                cur = self._fused_sweep(cur, b, x_zero)
                x_zero = False
            return cur
        for _ in range(sweeps):
            for step, (cd, cr) in enumerate(self.coefs):
                out = self.buf[0] if cur is not self.buf[0] else self.buf[1]
                z = x_zero and step == 0
                m = self.sell
                if m is not None and m.d16 is not None and not z:
                    call("sphc_sell_cheb_step16", n, m.slice_ptr, m.d16, m.c0, m.val, self.dinv,
                         b, cur, out, self.d, cd, cr, m.nbase)
                elif m is not None:
                    call("sphc_sell_cheb_step", n, m.slice_ptr, m.col, m.val, self.dinv, b,
                         None if z else cur, out, self.d, cd, cr, int(z), m.padded)
                else:
                    call("sphc_cheb_step", n, A.rowptr, A.col, A.val, self.lanes, self.dinv,
                         b, None if z else cur, out, self.d, cd, cr, int(z))
                cur = out
            x_zero = False
        return cur


    def symmetric_mid(self, x, r, c, D, mid):
        """The sweep that follows the nodal correction of a Hiptmair step:
        x + D c smoothed once, with the first polynomial step taken from
        the residual r = b - A x the caller holds (sphc_sell_hipt_mid: one
        pass over the SELL mirror ``mid`` of A D instead of a D pass and an
        A pass); the remaining steps as in ``symmetric``. Returns
        (iterate, b-independent): the caller passes b for the later steps."""
        n = self.A.shape[0]
        out = self.buf[0] if x is not self.buf[0] else self.buf[1]
        _, cr = self.coefs[0]
        if mid.d16 is not None:
            call("sphc_sell_hipt_mid16", n, mid.slice_ptr, mid.d16, mid.c0, mid.val, D.rowptr,
                 D.col, D.val, self.dinv, r, c, x, out, self.d, cr, mid.nbase)
        else:
            call("sphc_sell_hipt_mid", n, mid.slice_ptr, mid.col, mid.val, D.rowptr, D.col,
                 D.val, self.dinv, r, c, x, out, self.d, cr, mid.padded)
        return out

    def _steps_from(self, cur, b, first):
        """Polynomial steps first.. of one sweep on the SELL mirror."""
        n, m = self.A.shape[0], self.sell
        for cd, cr in self.coefs[first:]:
            out = self.buf[0] if cur is not self.buf[0] else self.buf[1]
            if m.d16 is not None:
                call("sphc_sell_cheb_step16", n, m.slice_ptr, m.d16, m.c0, m.val, self.dinv, b,
                     cur, out, self.d, cd, cr, m.nbase)
            else:
                call("sphc_sell_cheb_step", n, m.slice_ptr, m.col, m.val, self.dinv, b, cur,
                     out, self.d, cd, cr, 0, m.padded)
            cur = out
        return cur

    def _fused_sweep(self, x, b, x_zero):
        """The polynomial's steps in passes of self.fuse steps (the same
        buffers and arithmetic as the step-by-step loop)."""
        m, n = self.sell, self.A.shape[0]
        seq, cur = [], x
        for cd, cr in self.coefs:
            out = self.buf[0] if cur is not self.buf[0] else self.buf[1]
            seq.append((cur, out, cd, cr))
            cur = out
        k = 0
        while k < len(seq):
            ks = min(self.fuse, len(seq) - k)
            z = int(x_zero and k == 0)
            if ks == 1:
                xin, xout, cd, cr = seq[k]
                call("sphc_sell_cheb_step", n, m.slice_ptr, m.col, m.val, self.dinv, b,
                     None if z else xin, xout, self.d, cd, cr, z, m.padded)
            else:
                st = seq[k:k + ks] + [(None, None, 0.0, 0.0)] * (3 - ks)
                args = []
                for j, (xin, xout, cd, cr) in enumerate(st):
                    args += [None if (z and j == 0) else xin, xout, cd, cr]
                call("sphc_sell_cheb_fused", n, m.slice_ptr, m.col, m.val, self.dinv, b,
                     self.d, ks, *args, z, self.fuse_L, self.fuse_sync)
            k += ks
        return cur


class GaussSeidelSweeper:
    """The reference's symmetric Gauss-Seidel (multigrid.py:32-66):
    x += tril(A)^-1 (b - A x), then x += triu(A)^-1 (b - A x), each half sweep
    one sync-free triangular-substitution launch (csrc/trsv.cu). Exact
    smoother of the reference; latency-bound (dependency depth ~16 N)."""

    def __init__(self, A, degree=None):
        self.A = A
        n = A.shape[0]
        st = Status()
        dv.diagonal(A, st)
        st.defer(_zero_diag_check)
        self.y = dv.empty_f64(n)
        self.ticket = torch.zeros(1, dtype=torch.int32, device=A.rowptr.device)
        self.status = Status()
        self.buf = [dv.empty_f64(n), dv.empty_f64(n)]

    def symmetric(self, x, b, sweeps=1, x_zero=False):
        """Returns the smoothed iterate (a sweeper-owned buffer, never ``x``)."""
        A = self.A
        cur = x
        for _ in range(sweeps):
            for lower in (1, 0):
                out = self.buf[0] if cur is not self.buf[0] else self.buf[1]
                call("sphc_gs_half_sweep", A.shape[0], A.rowptr, A.col, A.val, b,
                     None if x_zero else cur, out, self.y, self.ticket, lower, self.status.t)
                cur = out
                x_zero = False
        return cur

    def check(self):
        rows = self.status.rows()
        if "TRSV_STALL" in rows:
            raise RuntimeError(f"triangular sweep stalled at row {rows['TRSV_STALL']}")


SMOOTHERS = {"chebyshev": ChebyshevSweeper, "gauss_seidel": GaussSeidelSweeper,
             "gs": GaussSeidelSweeper}


@checked
def symmetric_gauss_seidel(A, x, b, sweeps=1):
    """Forward then backward Gauss-Seidel sweeps (multigrid.py:62-66), same
    signature: numpy x / b give a numpy result, device tensors a device
    tensor. Sync-free triangular substitution kernels (csrc/trsv.cu)."""
    A = as_device_csr(A)
    host = not isinstance(b, torch.Tensor)
    dev = A.rowptr.device
    xt = torch.as_tensor(np.asarray(x, dtype=np.float64) if host else x,
                         dtype=torch.float64, device=dev)
    bt = torch.as_tensor(np.asarray(b, dtype=np.float64) if host else b,
                         dtype=torch.float64, device=dev)
    sw = GaussSeidelSweeper(A)
    out = sw.symmetric(xt, bt, sweeps)
    sw.check()
    return out.cpu().numpy() if host else out.clone()


@dataclass
class Level:
    """One hierarchy level (multigrid.py:69-89) plus its device working set."""

    A_e: DeviceCSR
    S_e: DeviceCSR
    D: DeviceCSR
    nodal_aux: DeviceCSR
    P_e: DeviceCSR = None
    P_n: DeviceCSR = None
    edge_sweeper: ChebyshevSweeper = None
    aux_sweeper: ChebyshevSweeper = None
    emin_energy: list = field(default_factory=list)
    subproblem_dims: dict = field(default_factory=dict)
    commutator_residual: float = 0.0
    n_augmented: int = 0
    # B200 working set
    R_e: DeviceCSR = None            # explicit P_e^T (restriction, gather only)
    Dt: DeviceCSR = None             # explicit D^T
    r: torch.Tensor = None
    bn: torch.Tensor = None
    rc: torch.Tensor = None          # restricted residual (next level's rhs)
    mid: object = None               # SELL mirror of A_e D (fused Hiptmair mid step)
    membership: torch.Tensor = None
    assignment: torch.Tensor = None
    coarse_gradient: object = None
    omega: float = 0.0
    rho: float = 0.0

    @property
    def n_edges(self):
        return self.A_e.shape[0]


@dataclass
class Hierarchy:
    levels: list
    coarse_factorization: torch.Tensor   # explicit inverse of the coarsest A_e
    operator_complexity: float

    @property
    def n_levels(self):
        return len(self.levels)


def _make_level(A_e, S_e, D, cfg, AD=None, smooth=True, shard=None, **extra):
    Dt = dv.transpose(D)
    # D^T A D keeps exact cancellations as stored zeros (scipy drops them;
    # they change no value and no decision, and skipping the compaction
    # saves a host sync per level)
    if AD is None:
        AD = dv.spgemm(A_e, D, drop=False, shard=shard)
    nodal_aux = dv.spgemm(Dt, AD, drop=False, shard=shard)
    level = Level(A_e=A_e, S_e=S_e, D=D, nodal_aux=nodal_aux, Dt=Dt, **extra)
    if smooth:   # the coarsest level is solved directly, never smoothed
        sweeper = SMOOTHERS[cfg.smoother]
        level.edge_sweeper = sweeper(A_e, cfg.cheb_degree)
        level.aux_sweeper = sweeper(nodal_aux, cfg.cheb_degree)
        es = level.edge_sweeper
        if (HIPT_MID_MIN_ROWS >= 0 and A_e.shape[0] >= HIPT_MID_MIN_ROWS
                and isinstance(es, ChebyshevSweeper) and es.sell is not None
                and es.degree >= 1 and 12 * AD.nnz < 0.8 * 12 * A_e.nnz):
            # streaming levels: keep A D (SELL) for the fused mid step
            level.mid = dv.sell_rect(AD)
    level.r = dv.empty_f64(A_e.shape[0])
    level.bn = dv.empty_f64(D.shape[1])
    return level


def _check_nullspace(S, D, where, A=None, shard=None):
    """max|S D| <= 1e-10 max|S| (multigrid.py:110-116). With A (same pattern
    as S) the product A D is formed in the same pass and returned for the
    level's D^T A D."""
    AD = None
    if A is not None:
        A, S = _work_pair(A, S)
    if A is not None and dv.same_pattern(A, S):
        AD, SD = dv.spgemm_pair(A, S, D, D, drop=False, shard=shard)
        # (stored zeros of A D only feed D^T A D; see _make_level)
    else:
        SD = dv.spgemm(S, D, drop=False, shard=shard)
    m = dv.empty_f64(2)
    dv.maxabs(SD.val, m[0:1])
    dv.maxabs(S.val, m[1:2])
    defect, smax = (float(x) for x in dv.readback(m)[0])
    scale = max(smax, 1e-300)
    if defect > _NULLSPACE_TOL * scale:
        raise ValueError(
            f"curl null-space identity violated on {where}: "
            f"max|S D| = {defect:.3e} vs max|S| = {scale:.3e}")
    return AD


def _coarse_lu_inverse(Ad):
    """The reference's coarsest solve (multigrid.py:156-157,180-181):
    scipy ``lu_factor`` = LAPACK getrf with partial pivoting, then
    ``lu_solve``. Here getrf (cuSOLVER through torch) and the LU solves of
    the identity form the matrix those solves apply, A^-1 = U^-1 L^-1 P, so
    a V-cycle applies it as one GEMV. Nothing is symmetrised or regularised:
    on a numerically singular coarsest operator it behaves as the
    reference's LU does. Returns (inverse, info) -- info > 0 is getrf's
    exact-zero pivot (scipy only warns; the inverse then holds inf / nan)."""
    LU, piv, info = torch.linalg.lu_factor_ex(Ad)
    n = Ad.shape[0]
    inv = torch.linalg.lu_solve(LU, piv, torch.eye(n, dtype=Ad.dtype, device=Ad.device))
    return inv, info.reshape(1).to(torch.int64)


def _coarse_inverse_start(Ad, solver="cholesky"):
    if solver == "lu":
        inv, info = _coarse_lu_inverse(Ad)
        return inv, torch.zeros_like(info), None
    """Symmetric inverse of the coarsest operator (multigrid.py:157 factors it
    with LU). The coarsest A_e is SPD in exact arithmetic but badly scaled
    and ill-conditioned: the edge prolongators grow level by level (max|P_e|
    ~ 10 per level for every sigma, reference behaviour), so the diagonal of
    the coarsest operator spans 1e4..1e7 at N=32 and cond(A) reaches 1e16
    at N=128 with sigma = 1e-4 (C5's recipe), where a plain factorisation
    loses the small (gradient-like) modes. The inverse is therefore formed
    on the Jacobi-equilibrated matrix S A S, S = diag(A)^-1/2 (an exact
    identity: A^-1 = S (S A S)^-1 S), from its Cholesky factor (potrf,
    then L^-T L^-1: symmetric positive by construction; an explicit getri inverse is
    visibly non-symmetric at cond ~ 4e15 and made PCG diverge on C4). If the
    factorisation breaks down (numerically semidefinite: the Galerkin
    operator of a rank-deficient prolongator), S A S + n eps ||SAS|| I is
    factored instead (C5's 9,165-edge coarsest: 0.05 s against 0.9 s for
    the eigendecomposition); the symmetric eigendecomposition with
    eigenvalues <= n eps lambda_max treated as null space is the last
    resort."""
    # Queued without a host sync: the factorisation's status is read back
    # with the smoothers' Lanczos scalars (finalize_sweepers), and
    # _coarse_inverse_finish redoes the inverse on the rare breakdown.
    A = 0.5 * (Ad + Ad.T)
    d = torch.diagonal(A).clone()
    sc = torch.where(d > 0, d.rsqrt(), torch.ones_like(d))
    As = sc[:, None] * A * sc[None, :]
    As = 0.5 * (As + As.T)
    L, info = torch.linalg.cholesky_ex(As)
    # A factorisation that "succeeds" on a round-off pivot (an exactly
    # singular operator: min pivot^2 6e-19 on the 2-D quad case Q41s) is a
    # breakdown too: its inverse carries a 1e16 null-space mode and a
    # negative eigenvalue, and PCG stalls. Healthy coarsest operators sit
    # orders above the threshold (C3: 4.6e-12 against n eps = 3e-14).
    dl = torch.diagonal(L)
    n_ = As.shape[0]
    tiny = (dl.min() ** 2 < n_ * torch.finfo(torch.float64).eps * dl.max() ** 2)
    info = info.reshape(1).to(torch.int64) + tiny.reshape(1).to(torch.int64)
    # L^-T L^-1 from one triangular solve against I and a GEMM (0.37 ms
    # at n = 364 against 0.56 ms for cholesky_inverse's blocked potrs)
    Li = torch.linalg.solve_triangular(L, torch.eye(L.shape[0], dtype=L.dtype,
                                                    device=L.device), upper=False)
    inv = Li.T @ Li
    inv = sc[:, None] * inv * sc[None, :]
    return 0.5 * (inv + inv.T), info, (As, sc)


def _coarse_inverse_finish(inv, info, state):
    """The inverse from _coarse_inverse_start, or -- when its Cholesky broke
    down (info != 0) -- from the shifted / eigendecomposition fallbacks."""
    if int(info) == 0 or state is None:
        return inv
    As, sc = state
    # numerically singular: the Galerkin operator of a rank-deficient
    # prolongator (make_irreducible duplicates, deep levels of C5). A
    # shift of n eps ||SAS|| keeps the factor finite; the directions it
    # blows up are the null vectors of P (P A_c^-1 P^T never sees them),
    # and it perturbs the rest less than truncating them would.
    n = As.shape[0]
    info = 1
    if n > COARSE_EIGH_MAX:
        shift = n * torch.finfo(torch.float64).eps * As.abs().sum(1).max()
        L, info = torch.linalg.cholesky_ex(As + shift * torch.eye(n, dtype=As.dtype,
                                                                  device=As.device))
        if int(info) == 0:
            Li = torch.linalg.solve_triangular(L, torch.eye(n, dtype=L.dtype,
                                                            device=L.device), upper=False)
            inv = Li.T @ Li
    if int(info) != 0:
        # the pseudo-inverse: eigenvalues <= n eps lambda_max are the null
        # space of the prolongator (P A_c^+ P^T never sees them). Exact to
        # round-off on the range, where the shifted explicit inverse (entries
        # ~1 / shift) is only good to ~1e-3 -- enough for a preconditioner, so
        # it is kept for the big coarsest operators, whose eigendecomposition
        # costs ~1 s (C5's 9,165 edges)
        lam, V = torch.linalg.eigh(As)
        tiny = lam.abs().max() * As.shape[0] * torch.finfo(torch.float64).eps
        w = torch.where(lam > tiny, 1.0 / lam, torch.zeros_like(lam))
        inv = (V * w) @ V.T
    inv = sc[:, None] * inv * sc[None, :]
    return 0.5 * (inv + inv.T)


_SIDE = {}


def _side_stream():
    dev = torch.cuda.current_device()
    st = _SIDE.get(dev)
    if st is None:
        st = _SIDE[dev] = torch.cuda.Stream()
    return st


def _coarse_inverse(Ad, solver="cholesky"):
    """Synchronous form (the reuse path)."""
    inv, info, state = _coarse_inverse_start(Ad, solver)
    return _coarse_inverse_finish(inv, dv.readback(info)[0][0], state)


@checked
def build_hierarchy(A_e, S_e, A_n, D, cfg=None, shard=None):
    """Galerkin hierarchy driven by the constrained edge prolongator
    (multigrid.py:119-161). ``shard`` (sharding.Sharding, optional; not a
    reference argument) splits the row-parallel setup work over the ranks
    of a process group; the result is identical on every rank and bitwise
    equal to the unsharded hierarchy."""
    cfg = cfg or SolverConfig()
    first = None
    host_edge = (not isinstance(A_e, DeviceCSR) and not isinstance(S_e, DeviceCSR)
                 and os.environ.get("SPHC_ASYNC_UPLOAD", "1") != "0")
    if host_edge and A_e.shape[0] > cfg.coarse_size and cfg.max_levels > 1:
        # host inputs: A_e and S stream in behind the nodal chain (their
        # first use is the emin sweep); the fine-level null-space check runs
        # right after the first prolongator. A data error of the nodal chain
        # defers to that check's, so the reference's error order holds.
        # One background upload in order of first use: A_n and D (the
        # nodal chain starts as soon as they are queued), then S (the emin
        # sweep), then A_e.
        small = [M for M in (A_n, D) if not isinstance(M, DeviceCSR)]
        up = dv.AsyncUpload(small + [S_e, A_e])
        k = len(small)
        it = iter(range(k))
        A_n = own_csr(A_n) if isinstance(A_n, DeviceCSR) else up.get(next(it))
        D = own_csr(D) if isinstance(D, DeviceCSR) else up.get(next(it))
        try:
            first = build_edge_prolongator(A_n, dv.PendingCSR(up, k + 1),
                                           dv.PendingCSR(up, k), D, cfg.emin, shard=shard,
                                           final_energy=False)
        except ValueError:
            _check_nullspace(up.get(k), D, "the fine level", A=up.get(k + 1), shard=shard)
            raise
        A_e, S_e = up.get(k + 1), up.get(k)
    else:
        # solver-owned wrappers: the SELL mirrors and shared index arrays
        # the setup attaches never land on the caller's DeviceCSR objects
        A_e, S_e = own_csr(A_e), own_csr(S_e)
        A_n, D = own_csr(A_n), own_csr(D)
    AD = _check_nullspace(S_e, D, "the fine level", A=A_e, shard=shard)
    levels, traces = [], []
    while A_e.shape[0] > cfg.coarse_size and len(levels) < cfg.max_levels - 1:
        if first is not None:
            (prol, cg, nod), first = first, None
        else:
            prol, cg, nod = build_edge_prolongator(A_n, A_e, S_e, D, cfg.emin, shard=shard,
                                                   final_energy=False)
        P_e, P_n = prol.P_e, nod.P
        n_coarse = cg.n_edges
        if n_coarse == 0:
            break
        if n_coarse >= 0.9 * A_e.shape[0]:
            raise ValueError(
                f"coarsening stagnated: {n_coarse} coarse edges from "
                f"{A_e.shape[0]} fine edges")
        with phase("level.make_level"):
            lv = _make_level(A_e, S_e, D, cfg, AD=AD, shard=shard, P_e=P_e, P_n=P_n,
                             emin_energy=prol.energy_history,
                             subproblem_dims=dict(prol.subproblem_dims),
                             commutator_residual=prol.commutator_residual,
                             n_augmented=prol.n_augmented,
                             membership=prol.membership, assignment=prol.assignment,
                             coarse_gradient=cg, omega=nod.omega_used,
                             rho=nod.rho_estimate)
        with phase("level.transpose_Pe"):
            lv.R_e = dv.transpose(P_e)
        lv.rc = dv.empty_f64(n_coarse)
        levels.append(lv)
        with phase("level.galerkin_edge"):
            A_e, S_e = _galerkin_edge(A_e, S_e, P_e, lv.R_e, shard)
            if prol.energy_history:
                # the energy of the final iterate (edge_prolongator.py:154-156,
                # trace(P^T S P)) is the trace of the coarse curl-curl
                # operator just formed; read back with the sweepers' scalars
                tr = dv.zeros_f64(1)
                dv.vsum(dv.diagonal(S_e), tr)
                traces.append((lv, tr))
        with phase("level.galerkin_nodal"):
            A_n = dv.spgemm(dv.transpose(P_n), dv.spgemm(A_n, P_n, ordered=True, shard=shard),
                            ordered=True, shard=shard)
        D = cg.D_H
        with phase("level.nullspace_check"):
            AD = _check_nullspace(S_e, D, f"level {len(levels)}", A=A_e, shard=shard)
    with phase("coarsest"):
        # the dense inverse (cuSOLVER / cuBLAS) runs on a side stream while
        # this stream forms the coarsest level's D^T A D; its status comes
        # back with the Lanczos scalars
        main = torch.cuda.current_stream()
        side = _side_stream()
        Ad = dv.to_dense(A_e)
        Ad.record_stream(side)
        side.wait_stream(main)
        with torch.cuda.stream(side):
            inv, info, inv_state = _coarse_inverse_start(Ad, cfg.coarse_solver)
        last = _make_level(A_e, S_e, D, cfg, AD=AD, smooth=False, shard=shard)
        levels.append(last)
        main.wait_stream(side)
        for t in (inv, info, *(inv_state or ())):
            t.record_stream(main)
    last.r = dv.empty_f64(A_e.shape[0])
    nnz0 = levels[0].A_e.nnz
    oc = sum(lv.A_e.nnz for lv in levels) / nnz0
    info_h, *tr_h = finalize_sweepers(info, *(t for _, t in traces))
    for (lv, _), t in zip(traces, tr_h):
        lv.emin_energy = list(lv.emin_energy) + [float(t[0])]
    inv = _coarse_inverse_finish(inv, info_h[0], inv_state)
    return Hierarchy(levels=levels, coarse_factorization=inv, operator_complexity=oc)


def _work_pair(A, S):
    """The undropped, shared-pattern versions of a Galerkin pair (see
    _galerkin_edge), else the matrices themselves."""
    wa, ws = getattr(A, "_work", None), getattr(S, "_work", None)
    if wa is not None and ws is not None and wa.rowptr is ws.rowptr and wa.col is ws.col:
        return wa, ws
    return A, S


def _galerkin_edge(A_e, S_e, P_e, R_e, shard=None):
    """compress(P^T (A P)) for A_e and S_e (multigrid.py:150-151).

    The two products share one pattern and one pass. ``compress`` then drops
    each product's exact zeros, and a handful of round-off-sized entries of
    P^T (S P) do cancel exactly (2 of 25.9M at 128^3), which would split the
    patterns and send every later product of the pair through two separate
    passes. The returned (compressed) matrices therefore carry their
    undropped shared-pattern versions as ``_work``: the next level's pair
    products and null-space check run on those (stored zeros add nothing to
    any sum and cancel again in the products' own compress), and release
    them."""
    Aw, Sw = _work_pair(A_e, S_e)
    if dv.same_pattern(Aw, Sw):
        # one pass for both: P^T (A_e P) and P^T (S_e P) share patterns
        AP, SP = dv.spgemm_pair(Aw, Sw, P_e, P_e, drop=False, shard=shard)
        C1w, C2w = dv.spgemm_pair(R_e, R_e, AP, SP, drop=False, shard=shard)
        C1, C2 = dv.drop_zeros_many(C1w, C2w)
        if C1 is not C1w or C2 is not C2w:
            if C1 is C1w:          # keep the visible matrix free of the attribute cycle
                C1 = DeviceCSR(C1w.rowptr, C1w.col, C1w.val, C1w.shape)
            if C2 is C2w:
                C2 = DeviceCSR(C2w.rowptr, C2w.col, C2w.val, C2w.shape)
            C1._work, C2._work = C1w, C2w
    else:
        C1 = dv.spgemm(R_e, dv.spgemm(A_e, P_e, shard=shard), shard=shard)
        C2 = dv.spgemm(R_e, dv.spgemm(S_e, P_e, shard=shard), shard=shard)
    for M in (A_e, S_e):           # the inputs' work copies are spent
        if getattr(M, "_work", None) is not None:
            M._work = None
    return C1, C2


@checked
def reuse_hierarchy(h, A_e, S_e, cfg=None):
    """Setup reuse for a sequence of related systems (PAPER.md, closing
    remarks of the setup-cost discussion: "the interpolation operators can
    often be retained across a few linear solves (still re-projecting the
    discretization matrix for each solve)"; not part of the reference API).

    Keeps every level's transfers of ``h`` -- P_e, P_n, the coarse gradients
    and the explicit restrictions -- and re-projects the new fine operators
    (A_e, S_e: same edge numbering, e.g. a new sigma or time step) through
    them: Galerkin products, D^T A D, smoothers, coarsest inverse and the
    null-space checks of every level. Returns a new Hierarchy sharing the
    transfers with ``h`` (which stays usable)."""
    cfg = cfg or SolverConfig()
    A_e, S_e = own_csr(A_e), own_csr(S_e)
    old = h.levels
    if A_e.shape != old[0].A_e.shape or S_e.shape != old[0].S_e.shape:
        raise ValueError(f"operators {A_e.shape} / {S_e.shape} do not match the hierarchy's "
                         f"fine level {old[0].A_e.shape}")
    D = old[0].D
    AD = _check_nullspace(S_e, D, "the fine level", A=A_e)
    levels = []
    for li, lo in enumerate(old[:-1]):
        lv = _make_level(A_e, S_e, D, cfg, AD=AD, P_e=lo.P_e, P_n=lo.P_n,
                         emin_energy=lo.emin_energy, subproblem_dims=lo.subproblem_dims,
                         commutator_residual=lo.commutator_residual,
                         n_augmented=lo.n_augmented, membership=lo.membership,
                         assignment=lo.assignment, coarse_gradient=lo.coarse_gradient,
                         omega=lo.omega, rho=lo.rho)
        lv.R_e = lo.R_e
        lv.rc = dv.empty_f64(lo.P_e.shape[1])
        levels.append(lv)
        A_e, S_e = _galerkin_edge(A_e, S_e, lo.P_e, lo.R_e)
        D = old[li + 1].D
        AD = _check_nullspace(S_e, D, f"level {li + 1}", A=A_e)
    last = _make_level(A_e, S_e, D, cfg, AD=AD, smooth=False)
    last.r = dv.empty_f64(A_e.shape[0])
    levels.append(last)
    inv = _coarse_inverse(dv.to_dense(A_e), cfg.coarse_solver)
    oc = sum(lv.A_e.nnz for lv in levels) / levels[0].A_e.nnz
    finalize_sweepers()
    return Hierarchy(levels=levels, coarse_factorization=inv, operator_complexity=oc)


def hiptmair_smooth(level, x, b, x_zero=False):
    """Edge smoothing, nodal correction through the gradient, edge smoothing
    (multigrid.py:164-173). Returns the new iterate (may be a new buffer)."""
    x = level.edge_sweeper.symmetric(x, b, x_zero=x_zero)
    dv.spmv(level.A_e, x, level.r, alpha=-1.0, beta=1.0, z=b)        # r = b - A x
    dv.spmv(level.Dt, level.r, level.bn)                                # D^T r
    c = level.aux_sweeper.symmetric(None, level.bn, x_zero=True)
    if level.mid is not None:
        # x += D c and the next sweep's first step in one pass over A D
        es = level.edge_sweeper
        return es._steps_from(es.symmetric_mid(x, level.r, c, level.D, level.mid), b, 1)
    dv.spmv(level.D, c, x, alpha=1.0, beta=1.0, z=x)                   # x += D c
    return level.edge_sweeper.symmetric(x, b)


def v_cycle(h, x, b, level=0):
    """V-cycle with hybrid pre/post smoothing and the dense coarsest solve
    (multigrid.py:176-188). ``x`` None means a zero initial guess."""
    lv = h.levels[level]
    if level == h.n_levels - 1:
        n = lv.A_e.shape[0]
        call("sphc_dense_gemv", n, h.coarse_factorization, b, lv.r)
        return lv.r
    x = hiptmair_smooth(lv, x, b, x_zero=x is None)
    dv.spmv(lv.A_e, x, lv.r, alpha=-1.0, beta=1.0, z=b)
    dv.spmv(lv.R_e, lv.r, lv.rc)
    ec = v_cycle(h, None, lv.rc, level + 1)
    dv.spmv(lv.P_e, ec, x, alpha=1.0, beta=1.0, z=x)
    return hiptmair_smooth(lv, x, b)


def v_cycle_preconditioner(h):
    """The V-cycle as a fixed symmetric operator b -> V(b) (multigrid.py:191-195).

    It launches only fixed-address kernels with no host synchronisation, so
    pcg_solve may capture it in a CUDA graph (``graph_safe``)."""
    def apply(b):
        with phase("solve.vcycle"):
            return v_cycle(h, None, b)
    apply.graph_safe = not _trace.ENABLED     # tracing inserts host syncs
    apply.device_tensors = True
    apply.hierarchy = h
    return apply


def hiptmair_preconditioner(level):
    """One symmetric hybrid sweep from a zero guess as a stand-alone
    preconditioner (multigrid.py:198-201), graph-capturable like the V-cycle."""
    def apply(b):
        with phase("solve.hiptmair"):
            return hiptmair_smooth(level, None, b, x_zero=True)
    apply.graph_safe = not _trace.ENABLED
    apply.device_tensors = True
    # pcg_solve keeps its captured iteration on this holder and checks the
    # level's sweepers after the solve, as for a hierarchy
    holder = getattr(level, "_relax_holder", None)
    if holder is None:
        holder = level._relax_holder = SimpleNamespace(levels=[level])
    apply.hierarchy = holder
    return apply


@checked
def fine_level(A_e, S_e, D, cfg=None):
    """Single smoothing level without grid transfers, for the relaxation-only
    comparison (multigrid.py:204-207). ``cfg`` (not a reference argument)
    picks the smoother; the default is the Chebyshev-3 performance smoother."""
    cfg = cfg or SolverConfig()
    A_e, S_e, D = own_csr(A_e), own_csr(S_e), own_csr(D)
    lv = _make_level(A_e, S_e, D, cfg)
    finalize_sweepers()
    return lv


@dataclass
class PcgResult:
    x: object
    iterations: int
    residual_history: list
    precond_history: list
    status: str
    relative_residual: float


def _csr_key(A):
    return (A.rowptr.data_ptr(), A.col.data_ptr(), A.val.data_ptr(), A.shape)


class PcgGraph:
    """One PCG iteration captured from torch's current stream into a CUDA
    graph through libsphcurl's runtime capture (no torch graph pool: the
    iteration allocates nothing), replayed on the current stream."""

    def __init__(self, body):
        h = np.zeros(1, dtype=np.uint64)
        call("sphc_graph_begin")
        try:
            body()
        finally:
            call("sphc_graph_end", h)
        self.h = int(h[0])

    def replay(self):
        call("sphc_graph_launch", self.h)

    def __del__(self):
        if getattr(self, "h", 0):
            try:
                call("sphc_graph_destroy", self.h)
            except Exception:
                pass
            self.h = 0


def _true_residual(A, x, b, Ap, sc):
    dv.spmv(A, x, Ap, alpha=-1.0, beta=1.0, z=b)
    dv.dot(Ap, Ap, sc[0:1])
    return math.sqrt(float(dv.readback(sc[0:1])[0][0]))


class PcgLoop:
    """The whole PCG loop as one graph launch: a WHILE conditional node whose
    body is one captured iteration plus the device-side convergence / break-
    down test (sphc_pcg_check; include/sphcurl.h). Records |r| and sqrt(r.z)
    per iteration on the device."""

    def __init__(self, body, sc, ctl, hist):
        h = np.zeros(1, dtype=np.uint64)
        call("sphc_pcg_loop_begin", h)
        self.h = int(h[0])
        try:
            body()
            call("sphc_pcg_check", self.h, sc, ctl, hist)
        finally:
            call("sphc_pcg_loop_end", self.h)
        self.ctl = ctl

    def launch(self):
        k = np.zeros(1, dtype=np.int64)
        call("sphc_pcg_loop_launch", self.h, k)
        self.per_iter = int(k[0])

    def __del__(self):
        if getattr(self, "h", 0):
            try:
                call("sphc_pcg_loop_destroy", self.h)
            except Exception:
                pass
            self.h = 0


def _pcg_iteration(A, lanes, precond, x, r, p, Ap, sc, flag, stage, rotate=True):
    """One PCG iteration with device-resident scalars (sc slots as in
    include/sphcurl.h SPHC_PCG_*); ends with the scalars copied to ``stage``.
    ``rotate=False`` leaves r.z's rotation to sphc_pcg_check (graph loop)."""
    n = x.numel()
    dv.spmv(A, p, Ap, lanes=lanes)
    dv.dot(p, Ap, sc[0:1])
    call("sphc_pcg_update_rr", n, sc, p, Ap, x, r, flag)     # + sc[1] = r.r
    z = precond(r)
    dv.dot(r, z, sc[3:4])
    call("sphc_pcg_direction", n, sc, z, p)
    if stage is not None:
        call("sphc_copy_d2h", stage, sc, sc.numel() * 8)
    if rotate:
        call("sphc_pcg_rotate", sc)
    return z


def _device_precond(precond):
    """The reference's preconditioner contract is Callable[[ndarray],
    ndarray] (multigrid.py:220). Ours (``device_tensors``) map device
    tensors to device tensors; any other callable gets r as a host numpy
    array and may return numpy or torch. Such a callable runs in the host
    loop, never in the captured graph."""
    if getattr(precond, "device_tensors", False):
        return precond

    def apply(r):
        z = precond(r.cpu().numpy())
        if isinstance(z, torch.Tensor):
            return z.to(device=r.device, dtype=torch.float64)
        return torch.as_tensor(np.ascontiguousarray(z, dtype=np.float64), device=r.device)
    return apply


@checked
def pcg_solve(A, b, precond, rtol=1e-8, maxit=500):
    """Preconditioned CG from x = 0 (multigrid.py:220-274): same statuses
    (converged | maxit | stagnated | indefinite) and histories.

    The scalars alpha, beta live on the device. With a graph-safe
    preconditioner (ours) the whole loop is ONE CUDA graph launch: a WHILE
    conditional node around one captured iteration and a device-side test
    of the reference's conditions (PcgLoop), captured once per hierarchy;
    the histories come back in one readback after the loop."""
    A = as_device_csr(A)
    host = not isinstance(b, torch.Tensor)
    b = (dv.upload(np.asarray(b, dtype=np.float64), np.float64) if host
         else torch.as_tensor(b, dtype=torch.float64, device=dv.device()))
    n = b.numel()
    lanes = A.lanes()
    graph_ok = getattr(precond, "graph_safe", False) and maxit > 0 and USE_GRAPH
    hier = getattr(precond, "hierarchy", None)
    precond = _device_precond(precond)
    ws = getattr(hier, "_pcg_ws", None) if graph_ok else None
    if ws is not None and (ws["A"] is not A and ws["A_key"] != _csr_key(A) or ws["n"] != n):
        ws = None
    if ws is None:
        sc = torch.zeros(6, dtype=torch.float64, device=b.device)
        ws = dict(A=A, A_key=_csr_key(A), n=n, x=dv.empty_f64(n), r=dv.empty_f64(n),
                  p=dv.empty_f64(n), Ap=dv.empty_f64(n), sc=sc,
                  flag=sc.view(torch.int32)[8:9],           # overlaps sc[4]
                  stage=torch.zeros(6, dtype=torch.float64, pin_memory=True), graph=None)
    x, r, p, Ap, sc, flag, stage = (ws[k] for k in ("x", "r", "p", "Ap", "sc", "flag", "stage"))
    x.zero_()
    r.copy_(b)
    dv.dot(b, b, sc[1:2])
    # the first preconditioner application is queued before |b| is known (a
    # zero b gives z = 0 and returns below, as the reference does without
    # calling it), so the loop graph's capture and instantiation on the host
    # overlap it instead of following a sync
    z = precond(r)
    p.copy_(z)
    dv.dot(r, z, sc[2:3])
    if graph_ok:
        loop = ws.get("loop")
        if loop is None or ws["loop_maxit"] < maxit:
            ws["loop"] = loop = None
            ws["ctl"] = dv.zeros_f64(4)
            ws["hist"] = dv.zeros_f64(2 * (maxit + 1))
            ws["ctl_host"] = torch.zeros(4, dtype=torch.float64, pin_memory=True)
            # every buffer of the iteration exists already (precond(r) above
            # queued the V-cycle once); captured on a side stream
            cap = torch.cuda.Stream()
            cap.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cap):
                loop = PcgLoop(lambda: _pcg_iteration(A, lanes, precond, x, r, p, Ap, sc,
                                                      flag, None, rotate=False),
                               sc, ws["ctl"], ws["hist"])
            torch.cuda.current_stream().wait_stream(cap)
            ws["loop"], ws["loop_maxit"] = loop, maxit
            if hier is not None:
                hier._pcg_ws = ws
    bb, rz0 = (float(v) for v in dv.readback(sc[1:3])[0])
    nb = math.sqrt(bb)

    def out(v):
        return dv.to_host(v) if host else v.clone()

    if nb == 0.0:
        return PcgResult(out(x), 0, [0.0], [0.0], "converged", 0.0)
    history = [nb]
    precond_history = [math.sqrt(max(rz0, 0.0))]
    status, iters = "maxit", 0
    if graph_ok:
        # the whole loop on the device: one graph launch, one readback
        ctl, hist, ch = ws["ctl"], ws["hist"], ws["ctl_host"]
        ch.copy_(torch.tensor([rtol * nb, float(maxit), 0.0, 0.0], dtype=torch.float64))
        ctl.copy_(ch, non_blocking=True)
        sc[4] = 0.0
        loop.launch()
        cv, hv = dv.readback(ctl, hist)
        iters, code = int(cv[2]), int(cv[3])
        # launch accounting: every kernel of every executed loop body
        call("sphc_pcg_loop_add_launches", loop.per_iter * (iters + (code == 4)))
        history += [float(hv[2 * i]) for i in range(1, iters + 1)]
        precond_history += [float(hv[2 * i + 1]) for i in range(1, iters + 1)]
        status = {1: "converged", 2: "maxit", 3: "stagnated", 4: "indefinite"}[code]
        if code == 3:
            # the last entry is the true residual of the unchanged iterate
            history[-1] = _true_residual(A, x, b, Ap, sc)
            precond_history[-1] = precond_history[-2]
    else:
        for k in range(maxit):
            sc[4] = 0.0
            _pcg_iteration(A, lanes, precond, x, r, p, Ap, sc, flag, stage)
            torch.cuda.current_stream().synchronize()
            hv = stage.numpy()
            pAp = float(hv[0])
            if pAp <= 0.0:
                status = "indefinite"
                break
            iters = k + 1
            if hv.view(np.int32)[8] == 0:
                status = "stagnated"
                history.append(_true_residual(A, x, b, Ap, sc))
                precond_history.append(precond_history[-1])
                break
            res = math.sqrt(float(hv[1]))
            history.append(res)
            precond_history.append(math.sqrt(max(float(hv[3]), 0.0)))
            if res <= rtol * nb:
                status = "converged"
                break
    if hier is not None:
        for lv in hier.levels:
            for sw in (lv.edge_sweeper, lv.aux_sweeper):
                if hasattr(sw, "check"):
                    sw.check()
    return PcgResult(x=out(x), iterations=iters, residual_history=history,
                     precond_history=precond_history, status=status,
                     relative_residual=history[-1] / nb)
