// Row-wise SpGEMM C = A B, one warp per row of A.
//
// Symbolic (count): lanes walk the row's flattened list of products (the B
//   rows reached from A's row, 32 A entries at a time) and insert the column
//   of each product into a per-warp open-addressing hash table in shared
//   memory, sized to the row (2 x its product count, power of two).
// Numeric (fill): the table is rebuilt at 2 x the known column count, the
//   columns are compacted and sorted into a dense slot list. Products are then
//   staged in shared memory in batches (all lanes loading in parallel: one
//   global latency per batch), as (slot, a_ik * b_kj) in k-major order, and
//   accumulated one B row per step from shared memory (a B row's entries have
//   distinct columns, so lanes never collide):
//   ORDERED:  B rows in ascending k with unfused sequential sums -- scipy
//             csr_matmat's order, bit-identical for the nodal Galerkin product
//             (SURVEY.md Appendix A);
//   !ORDERED: even / odd B rows go to two half-warps with their own
//             accumulator copy, summed at the end: deterministic, TOL class
//             (edge Galerkin products, D^T A D, S D).
#include "common.cuh"

#define SPG_WARPS 8
#define SPG_HCAP 512   // max hash slots per warp
#define SPG_CCAP 256   // max distinct columns per output row
#define SPG_FWARPS 4   // warps per block in the numeric pass (shared memory)

__device__ __forceinline__ int pow2_at_least(int n, int lo) {
  int m = lo;
  while (m < n) m <<= 1;
  return m;
}

// inserts col into a table of size ts (power of two); false on overflow
__device__ __forceinline__ bool spg_insert(int* table, int ts, int* ucount, int col) {
  unsigned h = ((unsigned)col * 2654435761u) & (ts - 1);
  for (int probe = 0; probe < ts; probe++) {
    int old = atomicCAS(&table[h], -1, col);
    if (old == -1) {
      atomicAdd(ucount, 1);
      return true;
    }
    if (old == col) return true;
    h = (h + 1) & (ts - 1);
  }
  return false;
}

struct SpgWarp {
  int off[32];  // inclusive prefix of B-row lengths of the current A batch
  i64 bs[32];   // B-row starts of the current A batch
  int ucount;
  int maxlen;
};

__device__ bool spg_symbolic(i64 row, const i64* __restrict__ arp, const int* __restrict__ aci,
                             const i64* __restrict__ brp, const int* __restrict__ bci,
                             int* table, int ts, SpgWarp& W, int lane) {
  for (int t = lane; t < ts; t += 32) table[t] = -1;
  if (lane == 0) W.ucount = 0;
  __syncwarp();
  bool ok = true;
  i64 as = arp[row], ae = arp[row + 1];
  int maxlen = 0;
  for (i64 c0 = as; c0 < ae; c0 += 32) {
    int len = 0;
    i64 bs = 0;
    if (c0 + lane < ae) {
      int k = aci[c0 + lane];
      bs = brp[k];
      len = (int)(brp[k + 1] - bs);
    }
    maxlen = max(maxlen, len);
    int incl = len;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(FULL_MASK, incl, o);
      if (lane >= o) incl += y;
    }
    W.off[lane] = incl;
    W.bs[lane] = bs;
    __syncwarp();
    int total = W.off[31];
    for (int f = lane; f < total; f += 32) {
      int lo = 0, hi = 31;
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (W.off[mid] > f) hi = mid; else lo = mid + 1;
      }
      int col = bci[W.bs[lo] + (f - (lo ? W.off[lo - 1] : 0))];
      ok &= spg_insert(table, ts, &W.ucount, col);
    }
    __syncwarp();
  }
  for (int o = 16; o > 0; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(FULL_MASK, maxlen, o));
  ok = __all_sync(FULL_MASK, ok);
  if (lane == 0) W.maxlen = maxlen;
  __syncwarp();
  return ok && W.ucount <= SPG_CCAP;
}

__device__ __forceinline__ int spg_row_products(i64 row, const i64* __restrict__ arp,
                                                const int* __restrict__ aci,
                                                const i64* __restrict__ brp, int lane) {
  int t = 0;
  for (i64 j = arp[row] + lane; j < arp[row + 1]; j += 32) {
    int k = aci[j];
    t += (int)(brp[k + 1] - brp[k]);
  }
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(FULL_MASK, t, o);
  return t;
}

__global__ void __launch_bounds__(SPG_WARPS * 32)
    k_spgemm_count(i64 n, const i64* __restrict__ arp, const int* __restrict__ aci,
                   const i64* __restrict__ brp, const int* __restrict__ bci,
                   i64* __restrict__ counts, i64* status) {
  __shared__ int table[SPG_WARPS][SPG_HCAP];
  __shared__ SpgWarp ws[SPG_WARPS];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (i64 row = (i64)blockIdx.x * SPG_WARPS + w; row < n; row += (i64)gridDim.x * SPG_WARPS) {
    int prods = spg_row_products(row, arp, aci, brp, lane);
    int ts = pow2_at_least(2 * prods, 32);
    if (ts > SPG_HCAP) ts = SPG_HCAP;
    bool ok = spg_symbolic(row, arp, aci, brp, bci, table[w], ts, ws[w], lane);
    if (lane == 0) {
      counts[row] = ok ? ws[w].ucount : 0;
      if (!ok) report(status, SPHC_ST_SPGEMM_CAPACITY, row);
    }
    __syncwarp();
  }
}

#define SPG_STG 512  // staged products per batch

struct SpgFill {
  int table[SPG_HCAP];
  double acc[2][SPG_CCAP];
  int sslot[SPG_STG];
  double sval[SPG_STG];
  int off[32];
  i64 bs[32];
  double a[32];
};

template <bool ORDERED>
__global__ void __launch_bounds__(SPG_FWARPS * 32)
    k_spgemm_fill(i64 n, const i64* __restrict__ arp, const int* __restrict__ aci,
                  const double* __restrict__ av, const i64* __restrict__ brp,
                  const int* __restrict__ bci, const double* __restrict__ bv,
                  const i64* __restrict__ crp, int* __restrict__ cci, double* __restrict__ cv,
                  i64* status) {
  extern __shared__ unsigned char spg_smem[];
  __shared__ SpgWarp ws[SPG_FWARPS];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  SpgFill& F = ((SpgFill*)spg_smem)[w];
  SpgWarp& W = ws[w];
  for (i64 row = (i64)blockIdx.x * SPG_FWARPS + w; row < n; row += (i64)gridDim.x * SPG_FWARPS) {
    int nu = (int)(crp[row + 1] - crp[row]);
    if (nu == 0) continue;
    int ts = pow2_at_least(2 * nu, 32);
    if (ts > SPG_HCAP) ts = SPG_HCAP;
    bool ok = spg_symbolic(row, arp, aci, brp, bci, F.table, ts, W, lane);
    if (!ok) continue;  // flagged by the count pass
    int* list = F.table;
    int cnt = 0;
    for (int b = 0; b < ts; b += 32) {
      int key = list[b + lane];
      unsigned bal = __ballot_sync(FULL_MASK, key >= 0);
      __syncwarp();
      if (key >= 0) list[cnt + __popc(bal & ((1u << lane) - 1))] = key;
      cnt += __popc(bal);
      __syncwarp();
    }
    int m = pow2_at_least(nu, 1);
    for (int t = nu + lane; t < m; t += 32) list[t] = 0x7fffffff;
    __syncwarp();
    for (int size = 2; size <= m; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = lane; t < (m >> 1); t += 32) {
          int lo = 2 * stride * (t / stride) + (t % stride), hi = lo + stride;
          bool up = (lo & size) == 0;
          int a = list[lo], b = list[hi];
          if ((a > b) == up) {
            list[lo] = b;
            list[hi] = a;
          }
        }
        __syncwarp();
      }
    for (int t = lane; t < nu; t += 32) {
      F.acc[0][t] = 0.0;
      F.acc[1][t] = 0.0;
    }
    __syncwarp();
    i64 as = arp[row], ae = arp[row + 1];
    const int G = ORDERED ? 1 : 2, LG = 32 / G;
    int g = lane / LG, l = lane % LG;
    double* my = F.acc[g];
    for (i64 c0 = as; c0 < ae;) {
      int len = 0;
      i64 bs = 0;
      double a = 0.0;
      if (c0 + lane < ae) {
        int k = aci[c0 + lane];
        a = av[c0 + lane];
        bs = brp[k];
        len = (int)(brp[k + 1] - bs);
      }
      int incl = len;
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(FULL_MASK, incl, o);
        if (lane >= o) incl += y;
      }
      // batch = the longest prefix of A entries whose products fit the stage
      unsigned fit = __ballot_sync(FULL_MASK, incl <= SPG_STG && c0 + lane < ae);
      int nb = __popc(fit);
      if (nb == 0) {  // a single B row longer than the stage
        if (lane == 0) report(status, SPHC_ST_SPGEMM_CAPACITY, row);
        break;
      }
      F.off[lane] = incl;
      F.bs[lane] = bs;
      F.a[lane] = a;
      __syncwarp();
      int total = F.off[nb - 1];
      for (int f = lane; f < total; f += 32) {
        int lo = 0, hi = nb - 1;
        while (lo < hi) {
          int mid = (lo + hi) >> 1;
          if (F.off[mid] > f) hi = mid; else lo = mid + 1;
        }
        i64 jb = F.bs[lo] + (f - (lo ? F.off[lo - 1] : 0));
        F.sslot[f] = lower_bound_i32(list, nu, bci[jb]);
        F.sval[f] = __dmul_rn(F.a[lo], bv[jb]);
      }
      __syncwarp();
      for (int t0 = 0; t0 < nb; t0 += G) {  // warp-uniform trip count
        int t = t0 + g;
        if (t < nb) {
          int p0 = t ? F.off[t - 1] : 0, p1 = F.off[t];
          for (int p = p0 + l; p < p1; p += LG) {
            int sl = F.sslot[p];
            my[sl] = ORDERED ? __dadd_rn(my[sl], F.sval[p]) : my[sl] + F.sval[p];
          }
        }
        __syncwarp();
      }
      __syncwarp();
      c0 += nb;
    }
    i64 o = crp[row];
    for (int t = lane; t < nu; t += 32) {
      cci[o + t] = list[t];
      cv[o + t] = ORDERED ? F.acc[0][t] : F.acc[0][t] + F.acc[1][t];
    }
    __syncwarp();
  }
}

extern "C" int sphc_spgemm_count(int64_t n, const int64_t* arp, const int32_t* aci,
                                 const int64_t* brp, const int32_t* bci, int64_t* counts,
                                 int64_t* status, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  k_spgemm_count<<<grid_for(n, SPG_WARPS, SPHC_NUM_SMS * 32), SPG_WARPS * 32, 0, s>>>(
      n, arp, aci, brp, bci, counts, status);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_spgemm_fill(int64_t n, const int64_t* arp, const int32_t* aci,
                                const double* av, const int64_t* brp, const int32_t* bci,
                                const double* bv, const int64_t* crp, int32_t* cci, double* cv,
                                int ordered, int64_t* status, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  size_t sm = SPG_FWARPS * sizeof(SpgFill);
  static bool attr = false;
  if (!attr) {
    SPHC_CUDA(cudaFuncSetAttribute(k_spgemm_fill<true>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    SPHC_CUDA(cudaFuncSetAttribute(k_spgemm_fill<false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    attr = true;
  }
  unsigned g = grid_for(n, SPG_FWARPS, SPHC_NUM_SMS * 32);
  if (ordered)
    k_spgemm_fill<true><<<g, SPG_FWARPS * 32, sm, s>>>(n, arp, aci, av, brp, bci, bv, crp,
                                                       cci, cv, status);
  else
    k_spgemm_fill<false><<<g, SPG_FWARPS * 32, sm, s>>>(n, arp, aci, av, brp, bci, bv, crp,
                                                        cci, cv, status);
  SPHC_LAUNCH_CHECK();
  return 0;
}
