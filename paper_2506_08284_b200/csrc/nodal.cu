// Nodal smoothed-aggregation chain, bit-faithful to the reference's scipy /
// numpy arithmetic (reference nodal_amg.py:33-155).
// Every product / sum here is an explicit round-to-nearest intrinsic: the
// values decide aggregates, the piecewise-constant map and the coarse edges.
#include "common.cuh"

// ------------------------------------------------------------------ strength
__global__ void k_strength(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                           const double* __restrict__ v, const double* __restrict__ d,
                           double drop_tol, i64* counts, const i64* __restrict__ frp,
                           int* __restrict__ fci, i64* status) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    double di = d[i];
    if (di <= 0.0) report(status, SPHC_ST_NONPOS_DIAG, i);
    i64 o = frp ? frp[i] : 0;
    i64 c = 0;
    bool diag_done = false;
    for (i64 j = rp[i]; j < rp[i + 1]; j++) {
      int col = ci[j];
      if (!diag_done && col >= (int)i) {
        if (fci) fci[o + c] = (int)i;
        c++;
        diag_done = true;
        if (col == (int)i) continue;
      }
      if (col == (int)i) continue;
      double th = __dmul_rn(drop_tol, __dsqrt_rn(__dmul_rn(di, d[col])));
      if (fabs(v[j]) > th) {
        if (fci) fci[o + c] = col;
        c++;
      }
    }
    if (!diag_done) {
      if (fci) fci[o + c] = (int)i;
      c++;
    }
    if (counts) counts[i] = c;
  }
}

extern "C" int sphc_strength_count(int64_t n, const int64_t* rp, const int32_t* ci,
                                   const double* v, const double* diag, double drop_tol,
                                   int64_t* counts, int64_t* status, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_strength<<<grid_for(n, 256), 256, 0, s>>>(n, rp, ci, v, diag, drop_tol, counts, nullptr,
                                              nullptr, status);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_strength_fill(int64_t n, const int64_t* rp, const int32_t* ci,
                                  const double* v, const double* diag, double drop_tol,
                                  const int64_t* frp, int32_t* fci, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_strength<<<grid_for(n, 256), 256, 0, s>>>(n, rp, ci, v, diag, drop_tol, nullptr, frp, fci,
                                              nullptr);
  SPHC_LAUNCH_CHECK();
  return 0;
}

__global__ void k_union(i64 n, const i64* __restrict__ arp, const int* __restrict__ aci,
                        const i64* __restrict__ brp, const int* __restrict__ bci, i64* counts,
                        const i64* __restrict__ crp, int* __restrict__ cci) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    i64 a = arp[i], ae = arp[i + 1], b = brp[i], be = brp[i + 1];
    i64 o = crp ? crp[i] : 0, c = 0;
    while (a < ae || b < be) {
      int x;
      if (b >= be || (a < ae && aci[a] < bci[b])) x = aci[a++];
      else if (a >= ae || bci[b] < aci[a]) x = bci[b++];
      else { x = aci[a++]; b++; }
      if (cci) cci[o + c] = x;
      c++;
    }
    if (counts) counts[i] = c;
  }
}

extern "C" int sphc_pattern_union_count(int64_t n, const int64_t* arp, const int32_t* aci,
                                        const int64_t* brp, const int32_t* bci,
                                        int64_t* counts, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_union<<<grid_for(n, 256), 256, 0, s>>>(n, arp, aci, brp, bci, counts, nullptr, nullptr);
  SPHC_LAUNCH_CHECK();
  return 0;
}
extern "C" int sphc_pattern_union_fill(int64_t n, const int64_t* arp, const int32_t* aci,
                                       const int64_t* brp, const int32_t* bci,
                                       const int64_t* crp, int32_t* cci, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_union<<<grid_for(n, 256), 256, 0, s>>>(n, arp, aci, brp, bci, nullptr, crp, cci);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// ------------------------------------------------------------------ power method
// w_i = sum over j DESCENDING of fl(fl(dinv_i a_ij) x_j), sequential from 0
// (DESC false: in storage order, scipy csr_matvec on any row order; dinv
// null: the stored values as they are)
// One thread per row keeps the sequential sum; the 32 rows of a warp are one
// contiguous CSR segment, staged in shared memory with coalesced loads first
// (a thread walking its own row straight from global memory reads 32 lines
// per step: 0.58 TB/s on the 57M-entry A_n of 128^3, ~10x under HBM speed, in
// the middle of the power method's serial chain). Segments beyond PMV_WCAP
// entries (irregular coarse rows) are read directly.
#define PMV_WCAP 1024
#define PMV_WARPS 4
template <bool DESC>
__global__ void __launch_bounds__(PMV_WARPS * 32)
    k_nodal_powmv(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                  const double* __restrict__ v, const double* __restrict__ dinv,
                  const double* __restrict__ x, double* __restrict__ y) {
  __shared__ int sc[PMV_WARPS][PMV_WCAP];
  __shared__ double sv[PMV_WARPS][PMV_WCAP];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (i64 row0 = ((i64)blockIdx.x * PMV_WARPS + w) * 32; row0 < n;
       row0 += (i64)gridDim.x * PMV_WARPS * 32) {
    i64 i = row0 + lane;
    bool act = i < n;
    i64 b = act ? rp[i] : 0, e = act ? rp[i + 1] : 0;
    i64 s0 = __shfl_sync(FULL_MASK, b, 0);
    i64 last = row0 + 32 < n ? row0 + 32 : n;
    i64 s1 = rp[last];
    int tot = (int)min(s1 - s0, (i64)PMV_WCAP + 1);
    bool staged = tot <= PMV_WCAP;
    if (staged) {
      for (int t = lane; t < tot; t += 32) {
        sc[w][t] = ci[s0 + t];
        sv[w][t] = v[s0 + t];
      }
    }
    __syncwarp();
    if (act) {
      double s = 0.0;
      int len = (int)(e - b);
      double inv = dinv ? dinv[i] : 0.0;
      if (staged) {
        const int* c = sc[w] + (b - s0);
        const double* a = sv[w] + (b - s0);
        for (int t = 0; t < len; t++) {
          int j = DESC ? len - 1 - t : t;
          double aj = dinv ? __dmul_rn(inv, a[j]) : a[j];
          s = __dadd_rn(s, __dmul_rn(aj, x[c[j]]));
        }
      } else {
        for (int t = 0; t < len; t++) {
          i64 j = DESC ? e - 1 - t : b + t;
          double aj = dinv ? __dmul_rn(inv, v[j]) : v[j];
          s = __dadd_rn(s, __dmul_rn(aj, x[ci[j]]));
        }
      }
      y[i] = s;
    }
    __syncwarp();
  }
}

extern "C" int sphc_nodal_powmv(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                                const double* dinv, const double* x, double* y, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_nodal_powmv<true><<<grid_for(n, PMV_WARPS * 32), PMV_WARPS * 32, 0, s>>>(n, rp, ci, v, dinv,
                                                                           x, y);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_spmv_stored_order(int64_t n, const int64_t* rp, const int32_t* ci,
                                      const double* v, const double* x, double* y,
                                      void* stream) {
  cudaStream_t s = as_stream(stream);
  k_nodal_powmv<false><<<grid_for(n, PMV_WARPS * 32), PMV_WARPS * 32, 0, s>>>(n, rp, ci, v,
                                                                            nullptr, x, y);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// ------------------------------------------------------------------ smoothing
// numpy's pairwise summation (DOUBLE_pairwise_sum), recursion unrolled with an
// explicit stack; np.add.reduceat of a row = a[0] + pairwise(a[1:])
__device__ double np_pairwise(const double* a, int n) {
  int st_off[32], st_n[32], sp = 0;
  double st_val[32];
  int st_state[32];
  // iterative post-order evaluation of the recursion tree
  st_off[0] = 0; st_n[0] = n; st_state[0] = 0; sp = 1;
  double ret = 0.0;
  while (sp) {
    int top = sp - 1;
    int off = st_off[top], m = st_n[top];
    if (m <= 128) {
      double res;
      if (m < 8) {
        res = 0.0;
        for (int i = 0; i < m; i++) res = __dadd_rn(res, a[off + i]);
      } else {
        double r[8];
        for (int j = 0; j < 8; j++) r[j] = a[off + j];
        int i = 8;
        for (; i < m - (m % 8); i += 8)
          for (int j = 0; j < 8; j++) r[j] = __dadd_rn(r[j], a[off + i + j]);
        res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                        __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
        for (; i < m; i++) res = __dadd_rn(res, a[off + i]);
      }
      sp--;
      // deliver to parent
      if (sp == 0) { ret = res; break; }
      int p = sp - 1;
      if (st_state[p] == 1) { st_val[p] = res; st_state[p] = 2; }
      else { st_val[p] = __dadd_rn(st_val[p], res); st_state[p] = 3; }
      continue;
    }
    int n2 = m / 2;
    n2 -= n2 % 8;
    if (st_state[top] == 0) {  // push left
      st_state[top] = 1;
      st_off[sp] = off; st_n[sp] = n2; st_state[sp] = 0; sp++;
    } else if (st_state[top] == 2) {  // push right
      st_off[sp] = off + n2; st_n[sp] = m - n2; st_state[sp] = 0; sp++;
    } else {  // state 3: both children done
      double res = st_val[top];
      sp--;
      if (sp == 0) { ret = res; break; }
      int p = sp - 1;
      if (st_state[p] == 1) { st_val[p] = res; st_state[p] = 2; }
      else { st_val[p] = __dadd_rn(st_val[p], res); st_state[p] = 3; }
    }
  }
  return ret;
}

#define SM_WARPS 4
#define SM_CAP 256  // max entries of an A_n row handled on chip

// One warp per row i of A_n:
//   s_c = sum over k DESCENDING, agg(k) = c, of fl(dinv_i a_ik)   (Dinv_A @ P_tent)
//   y_c = [c == agg(i)] - fl(omega s_c), exact zeros dropped      (P_tent - omega X)
//   p_c = fl(fl(1 / (y_0 + pairwise(y_1..))) y_c)                 (normalize_rows)
__global__ void __launch_bounds__(SM_WARPS * 32)
    k_nodal_smooth(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                   const double* __restrict__ v, const double* __restrict__ dinv,
                   const i64* __restrict__ memb, double omega, i64* counts,
                   const i64* __restrict__ prp, int* __restrict__ pci, double* __restrict__ pv,
                   i64* status) {
  __shared__ int keys[SM_WARPS][SM_CAP];
  __shared__ double xs[SM_WARPS][SM_CAP];
  __shared__ int uq[SM_WARPS][SM_CAP];
  __shared__ double ys[SM_WARPS][SM_CAP];
  __shared__ int yc[SM_WARPS][SM_CAP];
  __shared__ double ya[SM_WARPS][SM_CAP];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (i64 i = (i64)blockIdx.x * SM_WARPS + w; i < n; i += (i64)gridDim.x * SM_WARPS) {
    i64 s = rp[i];
    int len = (int)(rp[i + 1] - s);
    if (len > SM_CAP) {
      if (lane == 0) {
        report(status, SPHC_ST_SPGEMM_CAPACITY, i);
        if (counts) counts[i] = 0;
      }
      continue;
    }
    double inv = dinv[i];
    i64 aggi = memb[i];
    for (int t = lane; t < len; t += 32) {
      int k = (int)memb[ci[s + t]];
      keys[w][t] = k;
      uq[w][t] = k;
      xs[w][t] = __dmul_rn(inv, v[s + t]);
    }
    int m = 1;
    while (m < len) m <<= 1;
    for (int t = len + lane; t < m; t += 32) uq[w][t] = 0x7fffffff;
    __syncwarp();
    for (int size = 2; size <= m; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = lane; t < (m >> 1); t += 32) {
          int lo = ((t & ~(stride - 1)) << 1) | (t & (stride - 1)), hi = lo + stride;
          bool up = (lo & size) == 0;
          int a = uq[w][lo], b = uq[w][hi];
          if ((a > b) == up) { uq[w][lo] = b; uq[w][hi] = a; }
        }
        __syncwarp();
      }
    // compact unique aggregates (ascending) -> yc, with their y values
    int nu = 0;
    for (int base = 0; base < len; base += 32) {
      int t = base + lane;
      bool first = t < len && (t == 0 || uq[w][t] != uq[w][t - 1]);
      double y = 0.0;
      int c = 0;
      if (first) {
        c = uq[w][t];
        double acc = 0.0;
        for (int q = len - 1; q >= 0; q--)
          if (keys[w][q] == c) acc = __dadd_rn(acc, xs[w][q]);
        y = __dsub_rn(((i64)c == aggi) ? 1.0 : 0.0, __dmul_rn(omega, acc));
      }
      bool keep = first && y != 0.0;
      unsigned bal = __ballot_sync(FULL_MASK, keep);
      if (keep) {
        int pos = nu + __popc(bal & ((1u << lane) - 1));
        yc[w][pos] = c;
        ys[w][pos] = y;
        ya[w][pos] = fabs(y);
      }
      nu += __popc(bal);
    }
    __syncwarp();
    if (counts && lane == 0) counts[i] = nu;
    if (pci) {
      __shared__ double s_inv[SM_WARPS];
      if (lane == 0) {
        double sum = 0.0, asum = 0.0;
        if (nu > 0) {
          sum = __dadd_rn(ys[w][0], np_pairwise(&ys[w][1], nu - 1));
          asum = __dadd_rn(ya[w][0], np_pairwise(&ya[w][1], nu - 1));
        }
        double tol = __dmul_rn(1e-13, fmax(1.0, asum));
        if (fabs(sum) <= tol) report(status, SPHC_ST_ZERO_ROWSUM, i);
        s_inv[w] = __ddiv_rn(1.0, sum);
      }
      __syncwarp();
      double sinv = s_inv[w];
      i64 o = prp[i];
      for (int t = lane; t < nu; t += 32) {
        pci[o + t] = yc[w][t];
        pv[o + t] = __dmul_rn(sinv, ys[w][t]);
      }
    }
    __syncwarp();
  }
}

extern "C" int sphc_nodal_smooth_count(int64_t n, const int64_t* rp, const int32_t* ci,
                                       const double* v, const double* dinv, const int64_t* memb,
                                       double omega, int64_t* counts, int64_t* status,
                                       void* stream) {
  cudaStream_t s = as_stream(stream);
  k_nodal_smooth<<<grid_for(n, SM_WARPS, SPHC_NUM_SMS * 32), SM_WARPS * 32, 0, s>>>(
      n, rp, ci, v, dinv, memb, omega, counts, nullptr, nullptr, nullptr, status);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_nodal_smooth_fill(int64_t n, const int64_t* rp, const int32_t* ci,
                                      const double* v, const double* dinv, const int64_t* memb,
                                      double omega, const int64_t* prp, int32_t* pci, double* pv,
                                      int64_t* status, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_nodal_smooth<<<grid_for(n, SM_WARPS, SPHC_NUM_SMS * 32), SM_WARPS * 32, 0, s>>>(
      n, rp, ci, v, dinv, memb, omega, nullptr, prp, pci, pv, status);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// ------------------------------------------------------------------ normalize_rows
// normalize_rows (nodal_amg.py:119-135) of an arbitrary CSR: row sum as
// np.add.reduceat (a_0 + pairwise(a_1..)), |a| likewise for the zero-sum
// tolerance 1e-13 max(1, sum |a|), values fl(fl(1 / s) a) in place of the
// output (exact zeros are dropped afterwards by count_nonzero / compact,
// as the reference's diags(1 / s) @ P does). Thread per row; the pairwise
// sum reads the row straight from global memory.
__device__ double np_pairwise_abs(const double* a, int n, double* buf) {
  for (int t = 0; t < n; t++) buf[t] = fabs(a[t]);
  return np_pairwise(buf, n);
}

#define NR_CAP 256
__global__ void k_normalize_rows(i64 n, const i64* __restrict__ rp, const double* __restrict__ v,
                                 double* __restrict__ out, i64* status) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    i64 b = rp[i];
    int len = (int)(rp[i + 1] - b);
    double sum = 0.0, asum = 0.0;
    if (len > NR_CAP + 1) {
      report(status, SPHC_ST_SPGEMM_CAPACITY, i);
      continue;
    }
    if (len > 0) {
      double buf[NR_CAP];
      sum = __dadd_rn(v[b], np_pairwise(v + b + 1, len - 1));
      asum = __dadd_rn(fabs(v[b]), np_pairwise_abs(v + b + 1, len - 1, buf));
    }
    double tol = __dmul_rn(1e-13, fmax(1.0, asum));
    if (fabs(sum) <= tol) report(status, SPHC_ST_ZERO_ROWSUM, i);
    double inv = __ddiv_rn(1.0, sum);
    for (int t = 0; t < len; t++) out[b + t] = __dmul_rn(inv, v[b + t]);
  }
}

extern "C" int sphc_normalize_rows(int64_t n, const int64_t* rp, const double* v, double* out,
                                   int64_t* status, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_normalize_rows<<<grid_for(n, 128), 128, 0, s>>>(n, rp, v, out, status);
  SPHC_LAUNCH_CHECK();
  return 0;
}
