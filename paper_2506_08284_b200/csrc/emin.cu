// Constrained energy minimisation of the edge prolongator, one warp per fine
// edge (reference emin_setup.py:62-336 and edge_prolongator.py:104-228;
// SURVEY.md Appendix C).
//
// For fine edge i with free endpoints t (and h):
//   J  = sorted union of the P_n rows of its free endpoints      (T row)
//   r  = (D_h P_n)_i on J                                          (R_dp row)
//   I  = coarse edges with both ends in J, then single-node edges of J nodes,
//        ascending ids (prolongator pattern row, N = [B == 2])
//   G  = D_H[I, J] (+-1), k = |J| - (no single-node edge in I)
//   M  = G_k^T G_k (graph Laplacian on the first k nodes), Cholesky in smem
// Feasible guess: p = 1 + G_k M^-1 (r - G^T 1)_k   (== Q R^-T c of the QR route)
// Jacobi step:    p' = p - omega (d - G_k M^-1 G_k^T d),  d = dinv_i (S P)|_I
#include "common.cuh"

#define EM_WARPS 4
#define JM SPHC_EMIN_JMAX
#define IM SPHC_EMIN_IMAX

// Per-warp working set of one constraint block. Two capacity classes: the
// on-chip default (|J| <= 16, |I| <= 128, 4 warps per CTA) that every mesh
// family of the reference fits, and a wide one (|J| <= 32 = one lane per
// coarse node, |I| <= 592, which |J| <= 32 bounds: 496 interior pairs + 32
// single-node edges + the appended ones; 1 warp per CTA) that the rows the
// default class cannot hold are re-run through. Same arithmetic, same order.
template <int JMAX_, int IMAX_, int HCAP_, typename HPOS>
struct EminRowT {
  static constexpr int JMAX = JMAX_, IMAX = IMAX_, HCAP = HCAP_;
  int J[JMAX_];
  double r[JMAX_];
  int Icol[IMAX_];
  signed char pa[IMAX_];  // position of tail node in J, -1 for single-node edges
  signed char pb[IMAX_];  // position of head (or the single) node in J
  double L[JMAX_ * (JMAX_ + 1) / 2];  // packed lower Cholesky factor, row p at p(p+1)/2
  double y[JMAX_];
  double g[IMAX_];
  double p[IMAX_];
  int sc[2][JMAX_];       // staged P_n rows of the two endpoints (em_build_J)
  double sv[2][JMAX_];
  unsigned adj[JMAX_];    // interior-edge adjacency bitmasks over J (em_factor)
  int hkey[HCAP_];        // coarse column -> position in Icol (masked S P lookups)
  HPOS hpos[HCAP_];
  unsigned incm;          // J nodes incident to some edge of I
  int nJ, nI, k, err, fc; // err: 1 = reported error, 2 = beyond this class's capacity
};
typedef EminRowT<JM, IM, 256, unsigned char> EminRow;
typedef EminRowT<SPHC_EMIN_JWIDE, SPHC_EMIN_IWIDE, 2048, unsigned short> EminRowWide;

__device__ __forceinline__ unsigned low_mask(int n) { return n >= 32 ? 0xffffffffu : (1u << n) - 1u; }

// all lanes: the P_n rows of the (<=2) free endpoints are staged in shared
// memory with one coalesced load each, then lane 0 merges them into J, r
// (scipy csr_matmat order). Serial global loads here used to dominate the
// pass: every merge step waited on an L2 round trip.
template <class Row>
__device__ void em_build_J(Row& R, i64 i, const i64* __restrict__ drp,
                           const int* __restrict__ dci, const double* __restrict__ dv,
                           const i64* __restrict__ prp, const int* __restrict__ pci,
                           const double* __restrict__ pv, i64* status, int lane) {
  i64 s = drp[i];
  int nd = (int)(drp[i + 1] - s);
  if (nd < 1 || nd > 2) {
    if (lane == 0) {
      report(status, SPHC_ST_MALFORMED_GRAD, i);
      R.err = 1;
      R.nJ = 0;
    }
    __syncwarp();
    return;
  }
  int ta = dci[s];
  double sa = dv[s];
  i64 a0 = prp[ta];
  int na = (int)(prp[ta + 1] - a0);
  int nb = 0;
  i64 b0 = 0;
  double sb = 0.0;
  if (nd == 2) {
    int hb = dci[s + 1];
    sb = dv[s + 1];
    b0 = prp[hb];
    nb = (int)(prp[hb + 1] - b0);
  }
  constexpr int JC = Row::JMAX;
  if (na > JC || nb > JC) {   // the merged row would exceed the class as well
    if (lane == 0) {
      R.err = 2;
      R.nJ = 0;
    }
    __syncwarp();
    return;
  }
  if (JC <= 16) {             // both rows in one round of loads
    if (lane < na) {
      R.sc[0][lane] = pci[a0 + lane];
      R.sv[0][lane] = pv[a0 + lane];
    } else if (lane >= 16 && lane - 16 < nb) {
      R.sc[1][lane - 16] = pci[b0 + lane - 16];
      R.sv[1][lane - 16] = pv[b0 + lane - 16];
    }
  } else {
    if (lane < na) {
      R.sc[0][lane] = pci[a0 + lane];
      R.sv[0][lane] = pv[a0 + lane];
    }
    if (lane < nb) {
      R.sc[1][lane] = pci[b0 + lane];
      R.sv[1][lane] = pv[b0 + lane];
    }
  }
  __syncwarp();
  if (lane == 0) {
    R.err = 0;
    int ia = 0, ib = 0, n = 0;
    while (ia < na || ib < nb) {
      int ca = ia < na ? R.sc[0][ia] : 0x7fffffff;
      int cb = ib < nb ? R.sc[1][ib] : 0x7fffffff;
      int c = ca < cb ? ca : cb;
      // scipy csr_matmat order: first D entry (lower column) then the second
      double acc = 0.0;
      if (ca == c) acc = __dadd_rn(acc, __dmul_rn(sa, R.sv[0][ia++]));
      if (cb == c) acc = __dadd_rn(acc, __dmul_rn(sb, R.sv[1][ib++]));
      if (n >= JC) {
        R.err = 2;
        n = 0;
        break;
      }
      R.J[n] = c;
      R.r[n] = acc;
      n++;
    }
    R.nJ = n;
    if (n == 0 && !R.err) {
      report(status, SPHC_ST_EMPTY_J, i);
      R.err = 1;
    }
  }
  __syncwarp();
}

// all lanes: I = interior coarse edges among J pairs (lexicographic = ascending
// ids) followed by single-node edges of J nodes (ascending ids).
template <class Row>
__device__ void em_build_I(Row& R, i64 i, const i64* __restrict__ adj_rp,
                           const int* __restrict__ adj_col, const int* __restrict__ single_id,
                           const i64* __restrict__ xrp, const int* __restrict__ xeid,
                           const int* __restrict__ ep_a, const int* __restrict__ ep_b,
                           i64* status, int lane) {
  constexpr int IC = Row::IMAX;
  int nJ = R.nJ;
  int npairs = nJ * (nJ - 1) / 2;
  int nI = 0;
  bool over = false;
  for (int base = 0; base < npairs; base += 32) {
    int t = base + lane;
    int e = -1, pa = 0, pb = 0;
    if (t < npairs) {
      int p = 0, rem = t;
      while (rem >= nJ - 1 - p) {
        rem -= nJ - 1 - p;
        p++;
      }
      int q = p + 1 + rem;
      int a = R.J[p], b = R.J[q];
      i64 lo = adj_rp[a], hi = adj_rp[a + 1];
      i64 pos = lower_bound_i32_g(adj_col, lo, hi, b);
      if (pos < hi && adj_col[pos] == b) {
        e = (int)pos;
        pa = p;
        pb = q;
      }
    }
    unsigned bal = __ballot_sync(FULL_MASK, e >= 0);
    if (e >= 0) {
      int o = nI + __popc(bal & ((1u << lane) - 1));
      if (o < IC) {
        R.Icol[o] = e;
        R.pa[o] = (signed char)pa;
        R.pb[o] = (signed char)pb;
      }
    }
    nI += __popc(bal);
  }
  for (int base = 0; base < nJ; base += 32) {
    int p = base + lane;
    int sid = p < nJ ? single_id[R.J[p]] : -1;
    unsigned bal = __ballot_sync(FULL_MASK, sid >= 0);
    if (sid >= 0) {
      int o = nI + __popc(bal & ((1u << lane) - 1));
      if (o < IC) {
        R.Icol[o] = sid;
        R.pa[o] = -1;
        R.pb[o] = (signed char)p;
      }
    }
    nI += __popc(bal);
  }
  // edges appended by make_irreducible for this row (ids above every
  // original edge, ascending): both endpoints lie in J by construction
  if (xrp) {
    i64 x0 = xrp[i], x1 = xrp[i + 1];
    for (i64 t = x0 + lane; t < x1; t += 32) {
      int o = nI + (int)(t - x0);
      int e = xeid[t];
      if (o < IC) {
        R.Icol[o] = e;
        R.pa[o] = (signed char)lower_bound_i32(R.J, nJ, ep_a[e]);
        R.pb[o] = (signed char)lower_bound_i32(R.J, nJ, ep_b[e]);
      }
    }
    nI += (int)(x1 - x0);
  }
  over = nI > IC;
  if (lane == 0) {
    R.nI = over ? 0 : nI;
    if (over) R.err = 2;
  }
  __syncwarp();
}

// packed lower-triangle index (m <= p)
__device__ __forceinline__ int tri(int p, int m) { return p * (p + 1) / 2 + m; }

// all lanes: irreducibility (bitmask BFS), k, the Gram matrix (exact
// integer atomics), then the left-looking Cholesky with the rows below the
// pivot spread over the lanes. Every factor entry is computed with the
// serial loop's operation order, so the factor is bitwise the serial one.
// Returns (warp-uniform) 0 ok, 1 reducible, 2 rank failure (reported).
template <class Row>
__device__ int em_factor(Row& R, i64 i, i64* status, int lane) {
  int nJ = R.nJ, nI = R.nI;
  // irreducibility (emin_setup.py check_irreducible): every J node incident
  // to an edge of I and J connected by the interior edges. Lanes take the
  // edges and build adjacency bitmasks; reachability from node 0 is a
  // warp-wide OR per BFS level (<= |J| levels).
  if (lane < Row::JMAX) R.adj[lane] = 0u;
  if (lane == 0) R.incm = 0u;
  __syncwarp();
  bool dir = false;
  for (int e = lane; e < nI; e += 32) {
    int a = R.pa[e], b = R.pb[e];
    if (a < 0) {
      dir = true;
      atomicOr(&R.incm, 1u << b);
    } else {
      atomicOr(&R.incm, (1u << a) | (1u << b));
      atomicOr(&R.adj[a], 1u << b);
      atomicOr(&R.adj[b], 1u << a);
    }
  }
  bool dirich = __any_sync(FULL_MASK, dir);
  __syncwarp();
  unsigned full = low_mask(nJ);
  unsigned myadj = lane < nJ ? R.adj[lane] : 0u;
  unsigned reach = nJ ? 1u : 0u;
  for (;;) {
    unsigned nr = reach | __reduce_or_sync(FULL_MASK, ((reach >> lane) & 1u) ? myadj : 0u);
    if (nr == reach) break;
    reach = nr;
  }
  if (!(R.incm == full && reach == full)) return 1;
  int k = nJ - (dirich ? 0 : 1);
  // expected rank must be in [1, min(|I|, |J|)]
  if (k < 1 || k > nI) {
    if (lane == 0) report(status, SPHC_ST_RANK_LOW, i);
    __syncwarp();
    return 2;
  }
  // Gram matrix G_k^T G_k: integer-valued, so the shared-memory atomic sums
  // are exact and order independent (bitwise the serial accumulation)
  double* Lg = R.L;
  for (int t = lane; t < k * (k + 1) / 2; t += 32) Lg[t] = 0.0;
  __syncwarp();
  for (int e = lane; e < nI; e += 32) {
    int a = R.pa[e], b = R.pb[e];
    if (b < k) atomicAdd(&Lg[tri(b, b)], 1.0);
    if (a >= 0 && a < k) {
      atomicAdd(&Lg[tri(a, a)], 1.0);
      if (b < k) atomicAdd(&Lg[a > b ? tri(a, b) : tri(b, a)], -1.0);
    }
  }
  if (lane == 0) R.k = k;
  __syncwarp();
  double* L = R.L;
  // in-place lower Cholesky; |R_jj| of the reference QR = L_jj
  for (int j = 0; j < k; j++) {
    const double* Lj = L + tri(j, 0);
    double d = Lj[j];
    for (int m = 0; m < j; m++) d -= Lj[m] * Lj[m];
    double ljj = d > 0.0 ? sqrt(d) : 0.0;
    if (!(ljj >= 1e-10 * (j ? L[0] : ljj)) || ljj == 0.0) {
      if (lane == 0) report(status, SPHC_ST_RANK_LOW, i);
      __syncwarp();
      return 2;
    }
    int p = j + 1 + lane;
    double x = 0.0;
    if (p < k) {
      const double* Lp = L + tri(p, 0);
      x = Lp[j];
      for (int m = 0; m < j; m++) x -= Lp[m] * Lj[m];
    }
    __syncwarp();   // every lane has read L[tri(j, j)] (via d) and its row
    if (p < k) L[tri(p, j)] = x / ljj;
    if (lane == 0) L[tri(j, j)] = ljj;
    __syncwarp();
  }
  return 0;
}

// lane 0: y <- M^-1 y (k entries) with the Cholesky factor
template <class Row>
__device__ void em_solve(const Row& R, double* y) {
  int k = R.k;
  const double* L = R.L;
  for (int j = 0; j < k; j++) {
    const double* Lj = L + tri(j, 0);
    double x = y[j];
    for (int m = 0; m < j; m++) x -= Lj[m] * y[m];
    y[j] = x / Lj[j];
  }
  for (int j = k - 1; j >= 0; j--) {
    double x = y[j];
    for (int m = j + 1; m < k; m++) x -= L[tri(m, j)] * y[m];
    y[j] = x / L[tri(j, j)];
  }
}

// One pass over the fine edges. WIDE = false: every row, the default class;
// rows beyond (jcap, icap) -- the class's capacity unless a test lowers it --
// are marked (count: icount = -1 and *over += 1) and left to the wide pass.
// WIDE = true: launched right behind on the same stream, returns at once
// unless *over != 0, then handles exactly the marked rows.
template <bool FILL, bool WIDE, class Row, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_emin_setup(i64 n_e, const i64* __restrict__ drp, const int* __restrict__ dci,
                 const double* __restrict__ dv, const i64* __restrict__ prp,
                 const int* __restrict__ pci, const double* __restrict__ pv,
                 const i64* __restrict__ adj_rp, const int* __restrict__ adj_col,
                 const int* __restrict__ single_id, const i64* __restrict__ xrp,
                 const int* __restrict__ xeid, const int* __restrict__ ep_a,
                 const int* __restrict__ ep_b, i64* icount, i64* jcount, double* rmax2,
                 i64* dims, unsigned char* rowflag, double* rowmax,
                 const i64* __restrict__ trp, int* __restrict__ tci,
                 double* __restrict__ tv, const i64* __restrict__ erp, int* __restrict__ eci,
                 double* __restrict__ ev, int jcap, int icap, i64* over, i64* status) {
  if (WIDE && *(volatile i64*)over == 0) return;
  __shared__ Row rows[WARPS];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  Row& R = rows[w];
  for (i64 i = (i64)blockIdx.x * WARPS + w; i < n_e; i += (i64)gridDim.x * WARPS) {
    if (FILL) {
      // the count pass sized the rows: the row's class follows from its sizes
      bool wide = trp[i + 1] - trp[i] > jcap || erp[i + 1] - erp[i] > icap;
      if (wide != WIDE) continue;
    } else if (WIDE && icount[i] != -1) {
      continue;
    }
    em_build_J(R, i, drp, dci, dv, prp, pci, pv, status, lane);
    if (!R.err && !WIDE && R.nJ > jcap) {
      __syncwarp();
      if (lane == 0) R.err = 2;
      __syncwarp();
    }
    if (!R.err) em_build_I(R, i, adj_rp, adj_col, single_id, xrp, xeid, ep_a, ep_b, status, lane);
    if (!R.err && !WIDE && R.nI > icap) {
      __syncwarp();
      if (lane == 0) R.err = 2;
      __syncwarp();
    }
    if (R.err) {
      if (lane == 0) {
        bool defer = R.err == 2 && !WIDE && !FILL;
        if (R.err == 2 && !defer) report(status, SPHC_ST_EMIN_CAPACITY, i);
        if (!FILL) {
          icount[i] = defer ? -1 : 0;
          jcount[i] = defer ? -1 : 0;
          if (defer) atomicAdd((unsigned long long*)over, 1ull);
        }
      }
      __syncwarp();
      continue;
    }
    int nJ = R.nJ, nI = R.nI;
    if (!FILL) {
      if (lane == 0) {
        double rm = 0.0;
        for (int q = 0; q < nJ; q++) rm = fmax(rm, fabs(R.r[q]));
        atomic_max_nonneg(&rmax2[0], rm);
        if (nI == 0) atomic_max_nonneg(&rmax2[1], rm);
        else if (nI < SPHC_DIMS_I && nJ < SPHC_DIMS_J)
          atomicAdd((unsigned long long*)&dims[nI * SPHC_DIMS_J + nJ], 1ull);
        icount[i] = nI;
        jcount[i] = nJ;
        if (rowflag) rowflag[i] = nI == 0 ? 2 : 0;
        if (rowmax) rowmax[i] = rm;
      }
    }
    if (FILL) {
      i64 to = trp[i];
      for (int q = lane; q < nJ; q += 32) {
        tci[to + q] = R.J[q];
        tv[to + q] = R.r[q];
      }
    }
    // the count pass only sizes the rows; irreducibility and rank are
    // established once, by the fill pass
    if (nI == 0 || !FILL) {
      __syncwarp();
      continue;
    }
    int fcw = em_factor(R, i, status, lane);
    if (lane == 0) {
      int fc = fcw;
      bool ok = fc == 0;
      // reducible blocks are flagged for the host make_irreducible pass
      // (rowflag != NULL) or are an error once the repair has been applied
      if (fc == 1) {
        if (rowflag) rowflag[i] |= 1;
        else report(status, SPHC_ST_REDUCIBLE, i);
      }
      if (ok && FILL) {
        // c = r - G^T 1 on the first k nodes, y = M^-1 c
        int k = R.k;
        for (int q = 0; q < k; q++) R.y[q] = R.r[q];
        for (int e = 0; e < nI; e++) {
          int a = R.pa[e], b = R.pb[e];
          if (b < k) R.y[b] -= 1.0;
          if (a >= 0 && a < k) R.y[a] += 1.0;
        }
        em_solve(R, R.y);
      }
      R.err = ok ? 0 : 1;
    }
    __syncwarp();
    if (FILL) {
      // the pattern is written even for a failed block (the host repair pass
      // reads the original rows); values only for factored blocks
      int k = R.k;
      bool okv = !R.err;
      i64 eo = erp[i];
      for (int e = lane; e < nI; e += 32) {
        eci[eo + e] = R.Icol[e];
        if (okv) {
          int a = R.pa[e], b = R.pb[e];
          double gy = (b < k ? R.y[b] : 0.0) - ((a >= 0 && a < k) ? R.y[a] : 0.0);
          ev[eo + e] = 1.0 + gy;
        }
      }
    }
    __syncwarp();
  }
}

static inline int em_cap(int cap, int top) { return cap <= 0 || cap > top ? top : cap; }

extern "C" int sphc_emin_count(int64_t n_e, const int64_t* drp, const int32_t* dci,
                               const double* dv, const int64_t* prp, const int32_t* pci,
                               const double* pv, const int64_t* adj_rp, const int32_t* adj_col,
                               int64_t n_int, const int32_t* single_id, const int64_t* xrp,
                               const int32_t* xeid, const int32_t* ep_a, const int32_t* ep_b,
                               int64_t* icount, int64_t* jcount, double* rmax2, int64_t* dims,
                               uint8_t* rowflag, double* rowmax, int32_t jcap, int32_t icap,
                               int64_t* over, int64_t* status, void* stream) {
  cudaStream_t s = as_stream(stream);
  jcap = em_cap(jcap, JM);
  icap = em_cap(icap, IM);
  k_emin_setup<false, false, EminRow, EM_WARPS>
      <<<grid_for(n_e, EM_WARPS, SPHC_NUM_SMS * 32), EM_WARPS * 32, 0, s>>>(
          n_e, drp, dci, dv, prp, pci, pv, adj_rp, adj_col, single_id, xrp, xeid, ep_a, ep_b,
          icount, jcount, rmax2, dims, rowflag, rowmax, nullptr, nullptr, nullptr, nullptr,
          nullptr, nullptr, jcap, icap, over, status);
  SPHC_LAUNCH_CHECK();
  k_emin_setup<false, true, EminRowWide, 1><<<grid_for(n_e, 1, SPHC_NUM_SMS * 32), 32, 0, s>>>(
      n_e, drp, dci, dv, prp, pci, pv, adj_rp, adj_col, single_id, xrp, xeid, ep_a, ep_b,
      icount, jcount, rmax2, dims, rowflag, rowmax, nullptr, nullptr, nullptr, nullptr,
      nullptr, nullptr, jcap, icap, over, status);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_emin_fill(int64_t n_e, const int64_t* drp, const int32_t* dci,
                              const double* dv, const int64_t* prp, const int32_t* pci,
                              const double* pv, const int64_t* adj_rp, const int32_t* adj_col,
                              int64_t n_int, const int32_t* single_id, const int64_t* xrp,
                              const int32_t* xeid, const int32_t* ep_a, const int32_t* ep_b,
                              const int64_t* trp, int32_t* tci, double* tv, const int64_t* erp,
                              int32_t* eci, double* ev, uint8_t* rowflag, int32_t jcap,
                              int32_t icap, int64_t* over, int64_t* status, void* stream) {
  cudaStream_t s = as_stream(stream);
  jcap = em_cap(jcap, JM);
  icap = em_cap(icap, IM);
  k_emin_setup<true, false, EminRow, EM_WARPS>
      <<<grid_for(n_e, EM_WARPS, SPHC_NUM_SMS * 32), EM_WARPS * 32, 0, s>>>(
          n_e, drp, dci, dv, prp, pci, pv, adj_rp, adj_col, single_id, xrp, xeid, ep_a, ep_b,
          nullptr, nullptr, nullptr, nullptr, rowflag, nullptr, trp, tci, tv, erp, eci, ev,
          jcap, icap, over, status);
  SPHC_LAUNCH_CHECK();
  k_emin_setup<true, true, EminRowWide, 1><<<grid_for(n_e, 1, SPHC_NUM_SMS * 32), 32, 0, s>>>(
      n_e, drp, dci, dv, prp, pci, pv, adj_rp, adj_col, single_id, xrp, xeid, ep_a, ep_b,
      nullptr, nullptr, nullptr, nullptr, rowflag, nullptr, trp, tci, tv, erp, eci, ev, jcap,
      icap, over, status);
  SPHC_LAUNCH_CHECK();
  return 0;
}

template <class Row>
__device__ __forceinline__ unsigned em_h(int col) {
  return ((unsigned)col * 2654435761u) & (Row::HCAP - 1);
}

// position of coarse column col in the row's I, -1 if absent
template <class Row>
__device__ __forceinline__ int em_lookup(const Row& R, int col) {
  unsigned h = em_h<Row>(col);
  for (;;) {
    int k = R.hkey[h];
    if (k == col) return R.hpos[h];
    if (k < 0) return -1;
    h = (h + 1) & (Row::HCAP - 1);
  }
}

template <bool WIDE, class Row, int WARPS>
__global__ void __launch_bounds__(WARPS * 32)
    k_emin_step(i64 row0, i64 row1, const i64* __restrict__ srp, const int* __restrict__ sci,
                const double* __restrict__ sv, const double* __restrict__ dinv,
                const i64* __restrict__ trp, const int* __restrict__ tci,
                const double* __restrict__ tv, const i64* __restrict__ erp,
                const int* __restrict__ eci, const double* __restrict__ p_in,
                double* __restrict__ p_out, const int* __restrict__ ep_a,
                const int* __restrict__ ep_b, double omega, int update,
                double* __restrict__ e_row, double* res_max, int jcap, int icap,
                const i64* over, i64* status) {
  if (WIDE && *(volatile const i64*)over == 0) return;
  __shared__ Row rows[WARPS];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  Row& R = rows[w];
  for (i64 i = row0 + (i64)blockIdx.x * WARPS + w; i < row1; i += (i64)gridDim.x * WARPS) {
    i64 t0 = trp[i], e0 = erp[i];
    int nJ = (int)(trp[i + 1] - t0), nI = (int)(erp[i + 1] - e0);
    if ((nJ > jcap || nI > icap) != WIDE) continue;      // the other class's row
    if (nI == 0 || nJ > Row::JMAX || nI > Row::IMAX) {
      if (lane == 0) e_row[i] = 0.0;
      continue;
    }
    for (int q = lane; q < nJ; q += 32) {
      R.J[q] = tci[t0 + q];
      R.r[q] = tv[t0 + q];
    }
    __syncwarp();
    for (int t = lane; t < Row::HCAP; t += 32) R.hkey[t] = -1;
    __syncwarp();
    for (int e = lane; e < nI; e += 32) {
      int col = eci[e0 + e];
      R.Icol[e] = col;
      R.p[e] = p_in[e0 + e];
      R.g[e] = 0.0;
      int a = ep_a[col], b = ep_b[col];
      R.pb[e] = (signed char)lower_bound_i32(R.J, nJ, b);
      R.pa[e] = (signed char)(a < 0 ? -1 : lower_bound_i32(R.J, nJ, a));
      unsigned h = em_h<Row>(col);     // columns of a row are distinct
      while (atomicCAS(&R.hkey[h], -1, col) != -1) h = (h + 1) & (Row::HCAP - 1);
      R.hpos[h] = e;
    }
    if (lane == 0) {
      R.nJ = nJ;
      R.nI = nI;
    }
    __syncwarp();
    // masked S P on the fixed pattern: ascending k, sequential per entry
    // (scipy's S @ P order, edge_prolongator.py:173); the next S entry's
    // P-row bounds are loaded while the current row is accumulated
    // S row entries staged 32 at a time (column, value, P-row bounds: one
    // coalesced round of loads), then the P rows walked in ascending k with
    // the next row's loads issued before the current row's accumulation.
    // Same sums in the same order as the entry-by-entry loop.
    i64 js = srp[i], se = srp[i + 1];
    for (i64 c0 = js; c0 < se; c0 += 32) {
      int nb = (int)min((i64)32, se - c0);
      double s_v = 0.0;
      i64 s_b = 0;
      int s_l = 0;
      if (lane < nb) {
        int k = sci[c0 + lane];
        s_v = sv[c0 + lane];
        s_b = erp[k];
        s_l = (int)(erp[k + 1] - s_b);
      }
      if (__any_sync(FULL_MASK, s_l > 32)) {
        // a P row longer than a warp (rare): entry by entry
        for (int t = 0; t < nb; t++) {
          double st = __shfl_sync(FULL_MASK, s_v, t);
          i64 b = __shfl_sync(FULL_MASK, s_b, t);
          int l = __shfl_sync(FULL_MASK, s_l, t);
          for (int q = lane; q < l; q += 32) {
            int slot = em_lookup(R, eci[b + q]);
            if (slot >= 0) R.g[slot] = __dadd_rn(R.g[slot], __dmul_rn(st, p_in[b + q]));
          }
          __syncwarp();
        }
        continue;
      }
      int coln = -1;
      double vn = 0.0;
      {
        i64 b = __shfl_sync(FULL_MASK, s_b, 0);
        int l = __shfl_sync(FULL_MASK, s_l, 0);
        if (lane < l) {
          coln = eci[b + lane];
          vn = p_in[b + lane];
        }
      }
      for (int t = 0; t < nb; t++) {
        int col = coln;
        double v = vn;
        double st = __shfl_sync(FULL_MASK, s_v, t);
        int tn = t + 1 < nb ? t + 1 : t;
        i64 b = __shfl_sync(FULL_MASK, s_b, tn);
        int l = __shfl_sync(FULL_MASK, s_l, tn);
        coln = -1;
        if (t + 1 < nb && lane < l) {
          coln = eci[b + lane];
          vn = p_in[b + lane];
        }
        if (col >= 0) {
          int slot = em_lookup(R, col);
          if (slot >= 0) R.g[slot] = __dadd_rn(R.g[slot], __dmul_rn(st, v));
        }
        __syncwarp();
      }
    }
    double en = 0.0;
    for (int e = lane; e < nI; e += 32) en += R.p[e] * R.g[e];
    en = warp_sum(en);
    if (lane == 0) e_row[i] = en;
    __syncwarp();
    if (update) {
      int fc = em_factor(R, i, status, lane);
      if (fc != 0) {                       // warp-uniform
        if (fc == 1 && lane == 0) report(status, SPHC_ST_REDUCIBLE, i);
        __syncwarp();
        continue;
      }
      int k = R.k;
      double di = dinv[i];
      for (int e = lane; e < nI; e += 32) R.g[e] = __dmul_rn(di, R.g[e]);  // delta
      __syncwarp();
      // y = G_k^T delta: lane q sums its J node's contributions in ascending
      // e, the serial loop's order for that entry (bitwise the same)
      if (lane < k) {
        double yq = 0.0;
        for (int e = 0; e < nI; e++) {
          if (R.pb[e] == lane) yq += R.g[e];
          else if (R.pa[e] == lane) yq -= R.g[e];
        }
        R.y[lane] = yq;
      }
      __syncwarp();
      if (lane == 0) em_solve(R, R.y);
      __syncwarp();
      for (int e = lane; e < nI; e += 32) {
        int a = R.pa[e], b = R.pb[e];
        double gz = (b < k ? R.y[b] : 0.0) - ((a >= 0 && a < k) ? R.y[a] : 0.0);
        double pn = R.p[e] - omega * (R.g[e] - gz);
        R.p[e] = pn;
        p_out[e0 + e] = pn;
      }
      __syncwarp();
    }
    // commutator residual max |G^T p - r| over all of J: lane q forms
    // (G^T p)_q in ascending e (the serial order), then a warp max
    double m = 0.0;
    if (lane < nJ) {
      double gq = 0.0;
      for (int e = 0; e < nI; e++) {
        if (R.pb[e] == lane) gq += R.p[e];
        else if (R.pa[e] == lane) gq -= R.p[e];
      }
      m = fabs(gq - R.r[lane]);
    }
    m = warp_max(m);
    if (lane == 0) atomic_max_nonneg(res_max, m);
    __syncwarp();
  }
}

extern "C" int sphc_emin_step(int64_t row0, int64_t row1, const int64_t* srp, const int32_t* sci,
                              const double* sv, const double* dinv, const int64_t* trp,
                              const int32_t* tci, const double* tv, const int64_t* erp,
                              const int32_t* eci, const double* p_in, double* p_out,
                              const int32_t* ep_a, const int32_t* ep_b, double omega, int update,
                              double* e_row, double* res_max, int32_t jcap, int32_t icap,
                              const int64_t* over, int64_t* status, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (row1 <= row0) return 0;
  jcap = em_cap(jcap, JM);
  icap = em_cap(icap, IM);
  k_emin_step<false, EminRow, EM_WARPS>
      <<<grid_for(row1 - row0, EM_WARPS, SPHC_NUM_SMS * 32), EM_WARPS * 32, 0, s>>>(
          row0, row1, srp, sci, sv, dinv, trp, tci, tv, erp, eci, p_in, p_out, ep_a, ep_b, omega,
          update, e_row, res_max, jcap, icap, over, status);
  SPHC_LAUNCH_CHECK();
  k_emin_step<true, EminRowWide, 1><<<grid_for(row1 - row0, 1, SPHC_NUM_SMS * 32), 32, 0, s>>>(
      row0, row1, srp, sci, sv, dinv, trp, tci, tv, erp, eci, p_in, p_out, ep_a, ep_b, omega,
      update, e_row, res_max, jcap, icap, over, status);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// make_irreducible's main loop (emin_setup.py:183-217, 283-301) for the rows
// the count/fill passes flagged: one warp per row. The row's constraint
// graph (coarse nodes J <= 32 from T, its original pattern edges I) is
// connected greedily: among node pairs in different components, join the
// one with the largest |(D_h P_n)[:, a] . (D_h P_n)[:, b]| (ties and zeros:
// lexicographically smallest (a, b)), until every node is incident to an
// edge and the graph is connected. The column dot products are summed in
// ascending fine edge with separate multiply and add, as scipy's
// csr_matmat does for the reference's R_dp_csc[:, a].T @ R_dp_csc[:, b], so
// the decisions are the reference's. Main-loop repairs do not see each
// other's new edges (the reference extracts every row from the original
// pattern), so rows are independent; the caller numbers the new edges in
// ascending row order. Output: ncnt[r] edges in pairs[r * 31 + j] (a, b);
// ncnt[r] = -1: single-node graph (the reference's ValueError), -2: the row
// exceeds the kernel's |J| <= 32.
#define RP_MAXNEW (SPHC_EMIN_JWIDE - 1)

__global__ void __launch_bounds__(128)
    k_emin_repair(i64 nrows, const i64* __restrict__ rows, const i64* __restrict__ trp,
                  const int* __restrict__ tci, const i64* __restrict__ prp,
                  const int* __restrict__ pci, const int* __restrict__ ep_a,
                  const int* __restrict__ ep_b, const i64* __restrict__ ttrp,
                  const int* __restrict__ ttci, const double* __restrict__ ttv,
                  int* __restrict__ ncnt, int2* __restrict__ pairs, i64* status) {
  __shared__ double prod[4][32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  i64 gw = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 r = gw; r < nrows; r += nw) {
    i64 i = rows[r];
    i64 t0 = trp[i];
    int nJ = (int)(trp[i + 1] - t0);
    if (nJ > SPHC_EMIN_JWIDE) {
      if (lane == 0) ncnt[r] = -2;
      continue;
    }
    int myJ = lane < nJ ? tci[t0 + lane] : 0x7fffffff;   // J sorted ascending
    // adjacency bitmasks over J from the original pattern edges
    unsigned adj = 0u, inc = 0u;
    i64 p0 = prp[i], p1 = prp[i + 1];
    for (i64 e = p0; e < p1; e++) {        // warp-uniform loop over the row's edges
      int col = pci[e];
      int a = ep_a[col], b = ep_b[col];
      unsigned ba = __ballot_sync(FULL_MASK, lane < nJ && myJ == b);
      unsigned aa = a >= 0 ? __ballot_sync(FULL_MASK, lane < nJ && myJ == a) : 0u;
      inc |= ba | aa;
      if (aa && ba) {
        int pa = __ffs(aa) - 1, pb = __ffs(ba) - 1;
        if (lane == pa) adj |= 1u << pb;
        if (lane == pb) adj |= 1u << pa;
      }
    }
    unsigned full = nJ >= 32 ? 0xffffffffu : ((1u << nJ) - 1u);
    int nnew = 0;
    for (;;) {
      // component label = lowest node index reachable (BFS by bitmask OR)
      unsigned reach = 1u << lane;
      if (lane >= nJ) reach = 0u;
      for (int it = 0; it < SPHC_EMIN_JWIDE; it++) {
        unsigned nr = reach;
        for (int q = 0; q < nJ; q++) {
          unsigned aq = __shfl_sync(FULL_MASK, adj, q);
          if ((reach >> q) & 1u) nr |= aq;
        }
        if (__all_sync(FULL_MASK, nr == reach)) break;
        reach = nr;
      }
      int comp = reach ? __ffs(reach) - 1 : 32;
      bool one = __all_sync(FULL_MASK, lane >= nJ || comp == 0);
      if (one && inc == full) break;
      if (one) {                 // a single node without edges: unrepairable
        nnew = -1;
        break;
      }
      if (nnew >= RP_MAXNEW) {   // cannot happen: each join merges two components
        nnew = -2;
        break;
      }
      // best bridging pair: exact scores in (x, y) order, strict > keeps the
      // lexicographically smallest pair among equal scores
      double best = -1.0;
      int bx = -1, by = -1;
      for (int x = 0; x < nJ; x++) {
        int cx = __shfl_sync(FULL_MASK, comp, x);
        int a = __shfl_sync(FULL_MASK, myJ, x);
        i64 a0 = ttrp[a], a1 = ttrp[a + 1];
        for (int y = x + 1; y < nJ; y++) {
          int cy = __shfl_sync(FULL_MASK, comp, y);
          if (cx == cy) continue;
          int b = __shfl_sync(FULL_MASK, myJ, y);
          i64 b0 = ttrp[b], b1 = ttrp[b + 1];
          double s = 0.0;
          for (i64 c0 = a0; c0 < a1; c0 += 32) {
            i64 e = c0 + lane;
            double pr = 0.0;
            bool hit = false;
            if (e < a1) {
              int k = ttci[e];
              i64 q = lower_bound_i32_g(ttci, b0, b1, k);
              if (q < b1 && ttci[q] == k) {
                hit = true;
                pr = __dmul_rn(ttv[e], ttv[q]);
              }
            }
            prod[w][lane] = pr;
            unsigned hm = __ballot_sync(FULL_MASK, hit);
            __syncwarp();
            if (lane == 0)
              for (int l = 0; l < 32; l++)
                if ((hm >> l) & 1u) s = __dadd_rn(s, prod[w][l]);
            __syncwarp();
          }
          s = __shfl_sync(FULL_MASK, fabs(s), 0);
          if (s > best) {
            best = s;
            bx = x;
            by = y;
          }
        }
      }
      // join (J[bx], J[by])
      {
        int vx = __shfl_sync(FULL_MASK, myJ, bx), vy = __shfl_sync(FULL_MASK, myJ, by);
        if (lane == 0) pairs[r * RP_MAXNEW + nnew] = make_int2(vx, vy);
      }
      if (lane == bx) adj |= 1u << by;
      if (lane == by) adj |= 1u << bx;
      inc |= (1u << bx) | (1u << by);
      nnew++;
    }
    if (lane == 0) ncnt[r] = nnew;
  }
}

extern "C" int sphc_emin_repair(int64_t nrows, const int64_t* rows, const int64_t* trp,
                                const int32_t* tci, const int64_t* prp, const int32_t* pci,
                                const int32_t* ep_a, const int32_t* ep_b, const int64_t* ttrp,
                                const int32_t* ttci, const double* ttv, int32_t* ncnt,
                                int32_t* pairs, int64_t* status, void* stream) {
  if (nrows <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  k_emin_repair<<<grid_for(nrows, 4), 128, 0, s>>>(nrows, rows, trp, tci, prp, pci, ep_a, ep_b,
                                                   ttrp, ttci, ttv, ncnt, (int2*)pairs, status);
  SPHC_LAUNCH_CHECK();
  return 0;
}
