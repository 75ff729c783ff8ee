// Row-wise SpGEMM C = A B, one warp per row of A.
//
// Symbolic: the columns of row i are inserted into a per-warp open-addressing
// hash table in shared memory (lanes over the flattened (k, j) products).
// Numeric: the unique columns are sorted (bitonic, shared memory) and every
// product a_ik b_kj is added into its column's accumulator in ascending k --
// lanes take the entries of B row k, which have distinct columns, so there are
// no write conflicts and every output entry is the sequential, unfused sum
// scipy's csr_matmat forms (bit-identical to the reference for the nodal
// Galerkin product; TOL-level for the edge Galerkin products).
#include "common.cuh"

#define SPG_WARPS 4
#define SPG_HCAP 1024  // hash slots per warp
#define SPG_CCAP 512   // max distinct columns per output row

__device__ __forceinline__ unsigned spg_hash(int c) {
  return ((unsigned)c * 2654435761u) & (SPG_HCAP - 1);
}

// inserts col; returns false on overflow
__device__ __forceinline__ bool spg_insert(int* table, int* ucount, int col) {
  unsigned h = spg_hash(col);
  for (int probe = 0; probe < SPG_HCAP; probe++) {
    int old = atomicCAS(&table[h], -1, col);
    if (old == -1) {
      atomicAdd(ucount, 1);
      return true;
    }
    if (old == col) return true;
    h = (h + 1) & (SPG_HCAP - 1);
  }
  return false;
}

// Insert all columns of row `row` of A B into the warp's table. Lanes walk the
// flattened list of B-row entries, 32 A-entries at a time.
__device__ bool spg_symbolic_row(i64 row, const i64* __restrict__ arp, const int* __restrict__ aci,
                                 const i64* __restrict__ brp, const int* __restrict__ bci,
                                 int* table, int* ucount, int* s_off, i64* s_bs, int lane) {
  for (int t = lane; t < SPG_HCAP; t += 32) table[t] = -1;
  if (lane == 0) *ucount = 0;
  __syncwarp();
  bool ok = true;
  i64 as = arp[row], ae = arp[row + 1];
  for (i64 c0 = as; c0 < ae; c0 += 32) {
    int len = 0;
    i64 bs = 0;
    if (c0 + lane < ae) {
      int k = aci[c0 + lane];
      bs = brp[k];
      len = (int)(brp[k + 1] - bs);
    }
    int incl = len;
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(FULL_MASK, incl, o);
      if (lane >= o) incl += y;
    }
    s_off[lane] = incl;  // inclusive prefix
    s_bs[lane] = bs;
    __syncwarp();
    int total = s_off[31];
    for (int f = lane; f < total; f += 32) {
      // find t with s_off[t-1] <= f < s_off[t]
      int lo = 0, hi = 31;
      while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (s_off[mid] > f) hi = mid; else lo = mid + 1;
      }
      int before = lo ? s_off[lo - 1] : 0;
      int col = bci[s_bs[lo] + (f - before)];
      ok &= spg_insert(table, ucount, col);
    }
    __syncwarp();
  }
  ok = __all_sync(FULL_MASK, ok);
  __syncwarp();
  return ok && (*ucount <= SPG_CCAP);
}

__global__ void __launch_bounds__(SPG_WARPS * 32)
    k_spgemm_count(i64 n, const i64* __restrict__ arp, const int* __restrict__ aci,
                   const i64* __restrict__ brp, const int* __restrict__ bci,
                   i64* __restrict__ counts, i64* status) {
  __shared__ int table[SPG_WARPS][SPG_HCAP];
  __shared__ int ucount[SPG_WARPS];
  __shared__ int s_off[SPG_WARPS][32];
  __shared__ i64 s_bs[SPG_WARPS][32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (i64 row = (i64)blockIdx.x * SPG_WARPS + w; row < n; row += (i64)gridDim.x * SPG_WARPS) {
    bool ok = spg_symbolic_row(row, arp, aci, brp, bci, table[w], &ucount[w], s_off[w], s_bs[w],
                               lane);
    if (lane == 0) {
      counts[row] = ok ? ucount[w] : 0;
      if (!ok) report(status, SPHC_ST_SPGEMM_CAPACITY, row);
    }
    __syncwarp();
  }
}

template <bool ORDERED>
__global__ void __launch_bounds__(SPG_WARPS * 32)
    k_spgemm_fill(i64 n, const i64* __restrict__ arp, const int* __restrict__ aci,
                  const double* __restrict__ av, const i64* __restrict__ brp,
                  const int* __restrict__ bci, const double* __restrict__ bv,
                  const i64* __restrict__ crp, int* __restrict__ cci, double* __restrict__ cv,
                  i64* status) {
  __shared__ int table[SPG_WARPS][SPG_HCAP];
  __shared__ int ucount[SPG_WARPS];
  __shared__ int s_off[SPG_WARPS][32];
  __shared__ i64 s_bs[SPG_WARPS][32];
  __shared__ int list[SPG_WARPS][SPG_CCAP];
  __shared__ double acc[SPG_WARPS][SPG_CCAP];
  __shared__ double s_a[SPG_WARPS][32];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (i64 row = (i64)blockIdx.x * SPG_WARPS + w; row < n; row += (i64)gridDim.x * SPG_WARPS) {
    bool ok = spg_symbolic_row(row, arp, aci, brp, bci, table[w], &ucount[w], s_off[w], s_bs[w],
                               lane);
    if (!ok) continue;  // flagged by the count pass
    int nu = ucount[w];
    // gather unique keys
    if (lane == 0) ucount[w] = 0;
    __syncwarp();
    for (int t = lane; t < SPG_HCAP; t += 32) {
      int key = table[w][t];
      if (key >= 0) list[w][atomicAdd(&ucount[w], 1)] = key;
    }
    __syncwarp();
    // bitonic sort of the (small) list
    int m = 1;
    while (m < nu) m <<= 1;
    for (int t = nu + lane; t < m; t += 32) list[w][t] = 0x7fffffff;
    __syncwarp();
    for (int size = 2; size <= m; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = lane; t < (m >> 1); t += 32) {
          int lo = 2 * stride * (t / stride) + (t % stride), hi = lo + stride;
          bool up = (lo & size) == 0;
          int a = list[w][lo], b = list[w][hi];
          if ((a > b) == up) {
            list[w][lo] = b;
            list[w][hi] = a;
          }
        }
        __syncwarp();
      }
    for (int t = lane; t < nu; t += 32) acc[w][t] = 0.0;
    __syncwarp();
    i64 as = arp[row], ae = arp[row + 1];
    if (ORDERED) {
      // ascending k, sequential unfused accumulation per column (scipy order)
      for (i64 ja = as; ja < ae; ja++) {
        int k = aci[ja];
        double a = av[ja];
        i64 be = brp[k + 1];
        for (i64 jb = brp[k] + lane; jb < be; jb += 32) {
          int slot = lower_bound_i32(list[w], nu, bci[jb]);
          acc[w][slot] = __dadd_rn(acc[w][slot], __dmul_rn(a, bv[jb]));
        }
        __syncwarp();
      }
    } else {
      // all lanes busy: chunks of 32 flattened products, sorted by column in
      // registers and reduced per column with a fixed shuffle tree, so the
      // result is deterministic (not scipy-bitwise; TOL class)
      for (i64 c0 = as; c0 < ae; c0 += 32) {
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
        s_off[w][lane] = incl;
        s_bs[w][lane] = bs;
        s_a[w][lane] = a;
        __syncwarp();
        int total = s_off[w][31];
        for (int f0 = 0; f0 < total; f0 += 32) {
          int f = f0 + lane;
          int key = 0x7fffffff;
          double val = 0.0;
          if (f < total) {
            int lo = 0, hi = 31;
            while (lo < hi) {
              int mid = (lo + hi) >> 1;
              if (s_off[w][mid] > f) hi = mid; else lo = mid + 1;
            }
            int before = lo ? s_off[w][lo - 1] : 0;
            i64 jb = s_bs[w][lo] + (f - before);
            key = lower_bound_i32(list[w], nu, bci[jb]);
            val = s_a[w][lo] * bv[jb];
          }
          // bitonic sort of (key, val) across the warp
          for (int kk = 2; kk <= 32; kk <<= 1)
            for (int j = kk >> 1; j > 0; j >>= 1) {
              int pk = __shfl_xor_sync(FULL_MASK, key, j);
              double pv = __shfl_xor_sync(FULL_MASK, val, j);
              bool up = (lane & kk) == 0;
              bool lower = (lane & j) == 0;
              bool sw = lower ? ((key > pk) == up) : ((key < pk) == up);
              if (key == pk) sw = false;
              if (sw) { key = pk; val = pv; }
            }
          // inclusive segmented scan; the last lane of each run owns the sum
          for (int o = 1; o < 32; o <<= 1) {
            double y = __shfl_up_sync(FULL_MASK, val, o);
            int yk = __shfl_up_sync(FULL_MASK, key, o);
            if (lane >= o && yk == key) val += y;
          }
          int nk = __shfl_down_sync(FULL_MASK, key, 1);
          bool last = (lane == 31) || (nk != key);
          if (last && key != 0x7fffffff) acc[w][key] += val;
          __syncwarp();
        }
        __syncwarp();
      }
    }
    i64 o = crp[row];
    for (int t = lane; t < nu; t += 32) {
      cci[o + t] = list[w][t];
      cv[o + t] = acc[w][t];
    }
    __syncwarp();
  }
}

extern "C" int sphc_spgemm_count(int64_t n, const int64_t* arp, const int32_t* aci,
                                 const int64_t* brp, const int32_t* bci, int64_t* counts,
                                 int64_t* status, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  k_spgemm_count<<<grid_for(n, SPG_WARPS, SPHC_NUM_SMS * 64), SPG_WARPS * 32, 0, s>>>(
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
  unsigned g = grid_for(n, SPG_WARPS, SPHC_NUM_SMS * 64);
  if (ordered)
    k_spgemm_fill<true><<<g, SPG_WARPS * 32, 0, s>>>(n, arp, aci, av, brp, bci, bv, crp, cci,
                                                     cv, status);
  else
    k_spgemm_fill<false><<<g, SPG_WARPS * 32, 0, s>>>(n, arp, aci, av, brp, bci, bv, crp, cci,
                                                      cv, status);
  SPHC_LAUNCH_CHECK();
  return 0;
}
