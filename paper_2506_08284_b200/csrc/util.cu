// Primitives: scan, deterministic reductions, the Haswell-order ddot, CSR
// utilities (diagonal, segmented row sort, transpose, zero compaction).
#include <stdarg.h>

#include "common.cuh"

static thread_local char g_err[1024] = "";

void sphc_set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

extern "C" const char* sphc_last_error(void) { return g_err; }
extern "C" int sphc_abi_version(void) { return 1; }

unsigned long long g_sphc_launches = 0;

int sphc_pool_init() {
  static int done = -1;
  int dev = 0;
  SPHC_CUDA(cudaGetDevice(&dev));
  if (done == dev) return 0;
  cudaMemPool_t pool;
  SPHC_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t thr = ~0ull;
  SPHC_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  done = dev;
  return 0;
}
extern "C" int64_t sphc_launch_count(void) { return (int64_t)g_sphc_launches; }

// ------------------------------------------------------------------ scan
#define SCAN_THREADS 512
#define SCAN_ITEMS 4
#define SCAN_TILE (SCAN_THREADS * SCAN_ITEMS)

__global__ void k_scan_tile(i64 n_items, i64 n_valid, const i64* __restrict__ in,
                            i64* __restrict__ out, i64* __restrict__ tile_sums) {
  __shared__ i64 warp_tot[SCAN_THREADS / 32];
  i64 base = (i64)blockIdx.x * SCAN_TILE + (i64)threadIdx.x * SCAN_ITEMS;
  i64 v[SCAN_ITEMS];
  i64 t = 0;
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; k++) {
    i64 idx = base + k;
    v[k] = (idx < n_valid) ? in[idx] : 0;
    t += v[k];
  }
  // inclusive warp scan of thread totals
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  i64 incl = t;
  for (int o = 1; o < 32; o <<= 1) {
    i64 y = __shfl_up_sync(FULL_MASK, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_tot[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    i64 w = (lane < SCAN_THREADS / 32) ? warp_tot[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      i64 y = __shfl_up_sync(FULL_MASK, w, o);
      if (lane >= o) w += y;
    }
    if (lane < SCAN_THREADS / 32) warp_tot[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  i64 excl = incl - t + (wid ? warp_tot[wid - 1] : 0);
#pragma unroll
  for (int k = 0; k < SCAN_ITEMS; k++) {
    i64 idx = base + k;
    if (idx < n_items) out[idx] = excl;
    excl += v[k];
  }
  if (threadIdx.x == SCAN_THREADS - 1) tile_sums[blockIdx.x] = warp_tot[SCAN_THREADS / 32 - 1];
}

__global__ void k_scan_add(i64 n_items, i64* __restrict__ out, const i64* __restrict__ offs) {
  i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n_items) out[i] += offs[i / SCAN_TILE];
}

// out[0..n] = exclusive scan of in[0..n-1], out[n] = total
int sphc_scan_impl(i64 n, const i64* in, i64* out, cudaStream_t s) {
  i64 items = n + 1;
  i64 tiles = (items + SCAN_TILE - 1) / SCAN_TILE;
  i64* sums = nullptr;
  if (scratch(&sums, tiles + 1, s)) return SPHC_ERR_CUDA;
  k_scan_tile<<<(unsigned)tiles, SCAN_THREADS, 0, s>>>(items, n, in, out, sums);
  SPHC_LAUNCH_CHECK();
  if (tiles > 1) {
    i64* offs = nullptr;
    if (scratch(&offs, tiles + 1, s)) return SPHC_ERR_CUDA;
    int rc = sphc_scan_impl(tiles, sums, offs, s);
    if (rc) return rc;
    k_scan_add<<<(unsigned)((items + 255) / 256), 256, 0, s>>>(items, out, offs);
    SPHC_LAUNCH_CHECK();
    scratch_free(offs, s);
  }
  scratch_free(sums, s);
  return 0;
}

extern "C" int sphc_scan_i64(int64_t n, const int64_t* counts, int64_t* offsets, void* stream) {
  if (n < 0) return SPHC_ERR_ARG;
  return sphc_scan_impl(n, counts, offsets, as_stream(stream));
}

// ------------------------------------------------------------------ reductions
__device__ __forceinline__ double block_max(double v, double* sh) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_max(v);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = (lane < (int)(blockDim.x >> 5)) ? sh[lane] : 0.0;
    t = warp_max(t);
  }
  __syncthreads();
  return t;
}

// One launch per reduction: every block writes its partial, and the last
// block to finish (ticket counter) combines all partials in index order with
// the same fixed tree, then re-arms the counter. The grid is fixed by n, so
// the result is deterministic.
template <int MODE>  // 0: dot, 1: maxabs, 2: sum
__global__ void k_reduce(i64 n, const double* __restrict__ x, const double* __restrict__ y,
                         double* part, unsigned* ticket, double* out) {
  pdl_begin();
  __shared__ double sh[32];
  __shared__ bool last;
  double acc = 0.0;
  i64 stride = (i64)gridDim.x * blockDim.x;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (MODE == 0) acc = fma(x[i], y[i], acc);
    else if (MODE == 2) acc += x[i];
    else acc = fmax(acc, fabs(x[i]));
  }
  double t = (MODE != 1) ? block_sum(acc, sh) : block_max(acc, sh);
  if (threadIdx.x == 0) {
    part[blockIdx.x] = t;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  acc = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) {
    double v = __ldcg(part + i);
    acc = (MODE != 1) ? acc + v : fmax(acc, v);
  }
  t = (MODE != 1) ? block_sum(acc, sh) : block_max(acc, sh);
  if (threadIdx.x == 0) {
    *out = t;
    *ticket = 0u;
  }
}

// persistent partials and ticket shared by every single-launch reduction:
// reductions are stream ordered, and fixed buffers keep them capturable in
// CUDA graphs (no allocation nodes)
int sphc_reduce_scratch(double** part, unsigned** ticket) {
  static double* p = nullptr;
  static unsigned* t = nullptr;
  if (!p) {
    SPHC_CUDA(cudaMalloc((void**)&p, RED_MAX_BLOCKS * sizeof(double)));
    SPHC_CUDA(cudaMalloc((void**)&t, sizeof(unsigned)));
    SPHC_CUDA(cudaMemset(t, 0, sizeof(unsigned)));
  }
  *part = p;
  *ticket = t;
  return 0;
}

template <int MODE>
static int reduce_launch(i64 n, const double* x, const double* y, double* out, cudaStream_t s) {
  double* part;
  unsigned* ticket;
  if (sphc_reduce_scratch(&part, &ticket)) return SPHC_ERR_CUDA;
  int nb = sphc_reduce_grid(n);
  launch_pdl(k_reduce<MODE>, nb, RED_THREADS, 0, s, n, x, y, part, ticket, out);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_dot(int64_t n, const double* x, const double* y, double* out, void* stream) {
  return reduce_launch<0>(n, x, y, out, as_stream(stream));
}
extern "C" int sphc_sum(int64_t n, const double* x, double* out, void* stream) {
  return reduce_launch<2>(n, x, nullptr, out, as_stream(stream));
}
extern "C" int sphc_maxabs(int64_t n, const double* x, double* out, void* stream) {
  return reduce_launch<1>(n, x, nullptr, out, as_stream(stream));
}

// OpenBLAS 0.3.30 Haswell ddot order: lane l (0..15) owns the FMA chain of
// elements i = 16 q + l; chains combine as (l, l+2) within each 4-lane ymm,
// then ymm0+ymm1, ymm2+ymm3, their sum, and a horizontal add; the n % 16 tail
// is added unfused in index order.
#define HSW_TILE 1024     // elements per shared-memory tile (x and y each)
#define HSW_STAGES 4      // tiles in flight (64 KB of bulk copies hide HBM latency)

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

// One warp. Lane 0 keeps HSW_STAGES bulk copies (cp.async.bulk, the TMA's
// 1-D path) of the next x / y tiles in flight, each completing on its
// stage's mbarrier; lanes 0..15 run the sixteen sequential FMA chains over
// the landed tile. The chains -- 1 dependent DFMA per 16 elements -- set the
// pace, not the loads, and the kernel holds one warp and 64 KB of one SM, so
// the setup's other kernels run beside it (nodal_amg.RhoEstimate).
// Requires 16-byte aligned x, y (any torch allocation); else the caller takes
// the plain-load variant.
template <bool BULK>
__global__ void __launch_bounds__(32)
    k_hsw_dot(i64 n, const double* __restrict__ x, const double* __restrict__ y, double* out) {
  extern __shared__ __align__(128) unsigned char hsw_raw[];
  double* tiles = (double*)hsw_raw;                           // [STAGES][2][TILE]
  unsigned long long* bars = (unsigned long long*)(tiles + (size_t)HSW_STAGES * 2 * HSW_TILE);
  int lane = threadIdx.x;
  i64 n1 = n & ~(i64)15;
  i64 ntiles = (n1 + HSW_TILE - 1) / HSW_TILE;
  double acc = 0.0;
  auto issue = [&](i64 t) {       // lane 0 (BULK) or the whole warp (!BULK)
    int st = (int)(t % HSW_STAGES);
    double* bx = tiles + (size_t)st * 2 * HSW_TILE;
    double* by = bx + HSW_TILE;
    i64 base = t * HSW_TILE;
    int m = (int)min((i64)HSW_TILE, n1 - base);
    if (BULK) {
      unsigned bytes = (unsigned)m * 8u, bar = smem_u32(&bars[st]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "r"(2u * bytes) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(smem_u32(bx)), "l"(x + base), "r"(bytes), "r"(bar) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
          ::"r"(smem_u32(by)), "l"(y + base), "r"(bytes), "r"(bar) : "memory");
    } else {
      for (int k = lane; k < m; k += 32) {
        bx[k] = x[base + k];
        by[k] = y[base + k];
      }
    }
  };
  if (BULK) {
    if (lane == 0) {
      for (int st = 0; st < HSW_STAGES; st++)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[st])));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (lane == 0)
      for (i64 t = 0; t < ntiles && t < HSW_STAGES; t++) issue(t);
  }
  for (i64 t = 0; t < ntiles; t++) {
    int st = (int)(t % HSW_STAGES);
    if (BULK) {
      unsigned bar = smem_u32(&bars[st]), parity = (unsigned)((t / HSW_STAGES) & 1), done = 0;
      while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
            "selp.u32 %0, 1, 0, p; }"
            : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    } else {
      issue(t);
      __syncwarp();
    }
    if (lane < 16) {
      const double* bx = tiles + (size_t)st * 2 * HSW_TILE;
      const double* by = bx + HSW_TILE;
      int m = (int)min((i64)HSW_TILE, n1 - t * HSW_TILE);
#pragma unroll 8
      for (int k = lane; k < m; k += 16) acc = __fma_rn(bx[k], by[k], acc);
    }
    __syncwarp();     // every chain is done with this stage before it is refilled
    if (BULK && lane == 0 && t + HSW_STAGES < ntiles) issue(t + HSW_STAGES);
  }
  double a[16];
#pragma unroll
  for (int l = 0; l < 16; l++) a[l] = __shfl_sync(FULL_MASK, acc, l);
  if (lane == 0) {
    double dot = 0.0;
    if (n1) {
      double h0[4], h1[4];
#pragma unroll
      for (int q = 0; q < 4; q++) {
        h0[q] = __dadd_rn(a[4 * q + 0], a[4 * q + 2]);
        h1[q] = __dadd_rn(a[4 * q + 1], a[4 * q + 3]);
      }
      double u0 = __dadd_rn(__dadd_rn(h0[0], h0[1]), __dadd_rn(h0[2], h0[3]));
      double u1 = __dadd_rn(__dadd_rn(h1[0], h1[1]), __dadd_rn(h1[2], h1[3]));
      dot = __dadd_rn(u0, u1);
    }
    for (i64 i = n1; i < n; i++) dot = __dadd_rn(dot, __dmul_rn(y[i], x[i]));
    *out = dot;
  }
}

extern "C" int sphc_hsw_dot(int64_t n, const double* x, const double* y, double* out,
                            void* stream) {
  cudaStream_t s = as_stream(stream);
  size_t sm = (size_t)HSW_STAGES * 2 * HSW_TILE * sizeof(double) + HSW_STAGES * 8;
  static bool attr = false;
  if (!attr) {
    SPHC_CUDA(cudaFuncSetAttribute(k_hsw_dot<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)sm));
    SPHC_CUDA(cudaFuncSetAttribute(k_hsw_dot<false>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    attr = true;
  }
  bool aligned = (((uintptr_t)x | (uintptr_t)y) & 15) == 0;
  if (aligned) k_hsw_dot<true><<<1, 32, sm, s>>>(n, x, y, out);
  else k_hsw_dot<false><<<1, 32, sm, s>>>(n, x, y, out);
  SPHC_LAUNCH_CHECK();
  return 0;
}

__global__ void k_scale_by_norm(i64 n, const double* __restrict__ w, const double* sq,
                                double* __restrict__ v, double* norm_out) {
  double nrm = __dsqrt_rn(*sq);
  i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i == 0 && norm_out) *norm_out = nrm;
  if (nrm == 0.0) return;  // the reference stops here (rho = 0)
  for (; i < n; i += (i64)gridDim.x * blockDim.x) v[i] = __ddiv_rn(w[i], nrm);
}

extern "C" int sphc_scale_by_norm(int64_t n, const double* w, const double* sq, double* v,
                                  double* norm_out, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_scale_by_norm<<<grid_for(n, 256), 256, 0, s>>>(n, w, sq, v, norm_out);
  SPHC_LAUNCH_CHECK();
  return 0;
}

__global__ void k_axpby(i64 n, double a, const double* __restrict__ x, double b,
                        double* __restrict__ y) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x)
    y[i] = a * x[i] + b * y[i];
}

extern "C" int sphc_axpby(int64_t n, double a, const double* x, double b, double* y,
                          void* stream) {
  cudaStream_t s = as_stream(stream);
  k_axpby<<<grid_for(n, 256), 256, 0, s>>>(n, a, x, b, y);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// ------------------------------------------------------------------ CSR utilities
__global__ void k_csr_diag(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                           const double* __restrict__ v, double* __restrict__ d, i64* status) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    i64 s = rp[i], e = rp[i + 1];
    i64 p = lower_bound_i32_g(ci, s, e, (int)i);
    double x = (p < e && ci[p] == (int)i) ? v[p] : 0.0;
    d[i] = x;
    if (x == 0.0) report(status, SPHC_ST_ZERO_DIAG, i);
  }
}

extern "C" int sphc_csr_diag(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                             double* d, int64_t* status, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_csr_diag<<<grid_for(n, 256), 256, 0, s>>>(n, rp, ci, v, d, status);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// Segmented sort: warp per row (<= WARP_SORT_CAP keys in shared memory), block
// per row for longer rows (<= BLOCK_SORT_CAP).
#define WARP_SORT_CAP 256
#define SORT_WARPS 4
#define BLOCK_SORT_CAP 4096

__device__ __forceinline__ int next_pow2(int n) {
  int m = 1;
  while (m < n) m <<= 1;
  return m;
}

template <bool BLOCK>
__device__ void bitonic(int* k, double* v, int n, int tid, int nthr) {
  int m = next_pow2(n);
  for (int i = n + tid; i < m; i += nthr) k[i] = 0x7fffffff;
  if (BLOCK) __syncthreads(); else __syncwarp();
  for (int size = 2; size <= m; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = tid; t < (m >> 1); t += nthr) {
        int lo = ((t & ~(stride - 1)) << 1) | (t & (stride - 1));
        int hi = lo + stride;
        bool up = (lo & size) == 0;
        int a = k[lo], b = k[hi];
        if ((a > b) == up) {
          k[lo] = b;
          k[hi] = a;
          if (v) {
            double tv = v[lo];
            v[lo] = v[hi];
            v[hi] = tv;
          }
        }
      }
      if (BLOCK) __syncthreads(); else __syncwarp();
    }
  }
}

// *any_long is set when some row is left to the block kernel, which returns
// at once otherwise (it would scan every row pointer for nothing)
__global__ void k_sort_rows_warp(i64 n, const i64* __restrict__ rp, int* ci, double* v,
                                 int* any_long, i64* status) {
  __shared__ int sk[SORT_WARPS][WARP_SORT_CAP];
  __shared__ double sv[SORT_WARPS][WARP_SORT_CAP];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  i64 row0 = (i64)blockIdx.x * SORT_WARPS + w;
  for (i64 row = row0; row < n; row += (i64)gridDim.x * SORT_WARPS) {
    i64 s = rp[row];
    int len = (int)(rp[row + 1] - s);
    if (len > WARP_SORT_CAP) {
      if (lane == 0 && !*(volatile int*)any_long) *any_long = 1;
      continue;
    }
    if (len <= 1) continue;
    // already sorted rows are left untouched
    bool sorted = true;
    for (int t = lane; t + 1 < len; t += 32) sorted &= ci[s + t] <= ci[s + t + 1];
    if (__all_sync(FULL_MASK, sorted)) continue;
    for (int t = lane; t < len; t += 32) {
      sk[w][t] = ci[s + t];
      if (v) sv[w][t] = v[s + t];
    }
    __syncwarp();
    bitonic<false>(sk[w], v ? sv[w] : nullptr, len, lane, 32);
    for (int t = lane; t < len; t += 32) {
      ci[s + t] = sk[w][t];
      if (v) v[s + t] = sv[w][t];
    }
    __syncwarp();
  }
}

__global__ void k_sort_rows_block(i64 n, const i64* __restrict__ rp, int* ci, double* v,
                                  const int* any_long, i64* status) {
  if (!*(volatile const int*)any_long) return;
  extern __shared__ unsigned char smem[];
  double* sv = (double*)smem;
  int* sk = (int*)(sv + BLOCK_SORT_CAP);
  for (i64 row = blockIdx.x; row < n; row += gridDim.x) {
    i64 s = rp[row];
    int len = (int)(rp[row + 1] - s);
    if (len <= WARP_SORT_CAP) continue;
    if (len > BLOCK_SORT_CAP) {
      if (threadIdx.x == 0) report(status, SPHC_ST_SORT_CAPACITY, row);
      continue;
    }
    for (int t = threadIdx.x; t < len; t += blockDim.x) {
      sk[t] = ci[s + t];
      if (v) sv[t] = v[s + t];
    }
    __syncthreads();
    bitonic<true>(sk, v ? sv : nullptr, len, threadIdx.x, blockDim.x);
    for (int t = threadIdx.x; t < len; t += blockDim.x) {
      ci[s + t] = sk[t];
      if (v) v[s + t] = sv[t];
    }
    __syncthreads();
  }
}

static int sort_rows(i64 n, const i64* rp, int* ci, double* v, i64* status, cudaStream_t s) {
  if (n <= 0) return 0;
  int* any_long = nullptr;
  if (scratch(&any_long, 1, s)) return SPHC_ERR_CUDA;
  SPHC_CUDA(cudaMemsetAsync(any_long, 0, sizeof(int), s));
  k_sort_rows_warp<<<grid_for(n, SORT_WARPS, 148 * 32), SORT_WARPS * 32, 0, s>>>(
      n, rp, ci, v, any_long, status);
  SPHC_LAUNCH_CHECK();
  size_t sm = BLOCK_SORT_CAP * (sizeof(double) + sizeof(int));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sort_rows_block, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    attr = true;
  }
  k_sort_rows_block<<<grid_for(n, 1, 148 * 4), 512, sm, s>>>(n, rp, ci, v, any_long, status);
  SPHC_LAUNCH_CHECK();
  return scratch_free(any_long, s);
}

extern "C" int sphc_csr_sort_rows(int64_t n, const int64_t* rp, int32_t* ci, double* v,
                                  int64_t* status, void* stream) {
  return sort_rows(n, rp, ci, v, status, as_stream(stream));
}

__global__ void k_col_count(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                            i64* __restrict__ cnt) {
  i64 nnz = rp[n];
  for (i64 j = (i64)blockIdx.x * blockDim.x + threadIdx.x; j < nnz;
       j += (i64)gridDim.x * blockDim.x)
    atomicAdd((unsigned long long*)&cnt[ci[j]], 1ull);
}

__global__ void k_transpose_scatter(i64 n, const i64* __restrict__ rp,
                                    const int* __restrict__ ci, const double* __restrict__ v,
                                    i64* __restrict__ cursor, int* __restrict__ tci,
                                    double* __restrict__ tv) {
  // one warp per row: rows visited in order per warp; final order fixed by sort
  int lane = threadIdx.x & 31;
  i64 w0 = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 row = w0; row < n; row += nw) {
    for (i64 j = rp[row] + lane; j < rp[row + 1]; j += 32) {
      int c = ci[j];
      i64 pos = (i64)atomicAdd((unsigned long long*)&cursor[c], 1ull);
      tci[pos] = (int)row;
      if (v) tv[pos] = v[j];
    }
  }
}

extern "C" int sphc_csr_transpose(int64_t n_rows, int64_t n_cols, int64_t nnz,
                                  const int64_t* rp, const int32_t* ci, const double* v,
                                  int64_t* trp, int32_t* tci, double* tv, int64_t* status,
                                  void* stream) {
  cudaStream_t s = as_stream(stream);
  i64* cnt = nullptr;
  if (scratch(&cnt, n_cols + 1, s)) return SPHC_ERR_CUDA;
  SPHC_CUDA(cudaMemsetAsync(cnt, 0, (n_cols + 1) * sizeof(i64), s));
  if (nnz) {
    k_col_count<<<grid_for(nnz, 256), 256, 0, s>>>(n_rows, rp, ci, cnt);
    SPHC_LAUNCH_CHECK();
  }
  int rc = sphc_scan_impl(n_cols, cnt, trp, s);
  if (rc) return rc;
  if (nnz) {
    SPHC_CUDA(cudaMemcpyAsync(cnt, trp, n_cols * sizeof(i64), cudaMemcpyDeviceToDevice, s));
    k_transpose_scatter<<<grid_for(n_rows * 32, 256), 256, 0, s>>>(n_rows, rp, ci, v, cnt, tci,
                                                                  tv);
    SPHC_LAUNCH_CHECK();
    rc = sort_rows(n_cols, trp, tci, tv, status, s);
    if (rc) return rc;
  }
  return scratch_free(cnt, s);
}

__global__ void k_count_nonzero(i64 n, const i64* __restrict__ rp, const double* __restrict__ v,
                                i64* __restrict__ cnt) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    i64 c = 0;
    for (i64 j = rp[i]; j < rp[i + 1]; j++) c += (v[j] != 0.0);
    cnt[i] = c;
  }
}

extern "C" int sphc_csr_count_nonzero(int64_t n, const int64_t* rp, const double* v,
                                      int64_t* counts, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_count_nonzero<<<grid_for(n, 256), 256, 0, s>>>(n, rp, v, counts);
  SPHC_LAUNCH_CHECK();
  return 0;
}

__global__ void k_compact(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                          const double* __restrict__ v, const i64* __restrict__ nrp,
                          int* __restrict__ nci, double* __restrict__ nv) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    i64 o = nrp[i];
    for (i64 j = rp[i]; j < rp[i + 1]; j++)
      if (v[j] != 0.0) {
        nci[o] = ci[j];
        nv[o] = v[j];
        o++;
      }
  }
}

extern "C" int sphc_csr_compact(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                                const int64_t* new_rp, int32_t* nci, double* nv, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_compact<<<grid_for(n, 256), 256, 0, s>>>(n, rp, ci, v, new_rp, nci, nv);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// unique count / fill on rows that are already sorted
__global__ void k_unique_count(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                               i64* __restrict__ cnt) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    i64 c = 0;
    for (i64 j = rp[i]; j < rp[i + 1]; j++) c += (j == rp[i] || ci[j] != ci[j - 1]);
    cnt[i] = c;
  }
}
__global__ void k_unique_fill(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                              const i64* __restrict__ urp, int* __restrict__ uci) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    i64 o = urp[i];
    for (i64 j = rp[i]; j < rp[i + 1]; j++)
      if (j == rp[i] || ci[j] != ci[j - 1]) uci[o++] = ci[j];
  }
}

extern "C" int sphc_unique_count(int64_t n, const int64_t* rp, const int32_t* ci,
                                 int64_t* counts, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_unique_count<<<grid_for(n, 256), 256, 0, s>>>(n, rp, ci, counts);
  SPHC_LAUNCH_CHECK();
  return 0;
}
extern "C" int sphc_unique_fill(int64_t n, const int64_t* rp, const int32_t* ci,
                                const int64_t* urp, int32_t* uci, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_unique_fill<<<grid_for(n, 256), 256, 0, s>>>(n, rp, ci, urp, uci);
  SPHC_LAUNCH_CHECK();
  return 0;
}

__global__ void k_csr_to_dense(i64 n, i64 n_cols, const i64* __restrict__ rp,
                               const int* __restrict__ ci, const double* __restrict__ v,
                               double* __restrict__ out) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x)
    for (i64 j = rp[i]; j < rp[i + 1]; j++) out[i * n_cols + ci[j]] = v[j];
}

extern "C" int sphc_csr_to_dense(int64_t n_rows, int64_t n_cols, const int64_t* rp,
                                 const int32_t* ci, const double* v, double* out, void* stream) {
  cudaStream_t s = as_stream(stream);
  SPHC_CUDA(cudaMemsetAsync(out, 0, (size_t)n_rows * n_cols * sizeof(double), s));
  k_csr_to_dense<<<grid_for(n_rows, 128), 128, 0, s>>>(n_rows, n_cols, rp, ci, v, out);
  SPHC_LAUNCH_CHECK();
  return 0;
}

__global__ void k_reciprocal(i64 n, const double* __restrict__ x, const double* zero_sub,
                             double* __restrict__ y) {
  double zs = zero_sub ? *zero_sub : 0.0;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    double v = x[i];
    y[i] = __ddiv_rn(1.0, (v == 0.0 && zero_sub) ? zs : v);
  }
}

extern "C" int sphc_reciprocal(int64_t n, const double* x, const double* zero_sub, double* y,
                               void* stream) {
  cudaStream_t s = as_stream(stream);
  k_reciprocal<<<grid_for(n, 256), 256, 0, s>>>(n, x, zero_sub, y);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// ------------------------------------------------------------------ host memory
// Page-lock a caller's host array in place so uploads DMA straight from it
// (no staging copy); registered once per array by the Python side.
extern "C" int sphc_host_register(void* p, int64_t bytes) {
  cudaError_t e = cudaHostRegister(p, (size_t)bytes, cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    cudaGetLastError();   // not sticky: the caller falls back to staging
    sphc_set_error("cudaHostRegister: %s", cudaGetErrorString(e));
    return SPHC_ERR_CUDA;
  }
  return 0;
}

extern "C" int sphc_host_unregister(void* p) {
  cudaError_t e = cudaHostUnregister(p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return SPHC_ERR_CUDA;
  }
  return 0;
}

// dst (device) <- src (host, page-locked), asynchronous on stream
extern "C" int sphc_copy_h2d(void* dst, const void* src, int64_t bytes, void* stream) {
  SPHC_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, as_stream(stream)));
  return 0;
}


// ------------------------------------------------------------------ C = alpha A + beta B
// union pattern of two canonical CSR matrices (scipy csr_binop_csr): an
// entry present in one operand only takes fl(alpha a) or fl(beta b); count
// pass (cc) then fill (crp, cci, cv). Thread per row, sorted merge.
__global__ void k_csr_add(i64 n, const i64* __restrict__ arp, const int* __restrict__ aci,
                          const double* __restrict__ av, const i64* __restrict__ brp,
                          const int* __restrict__ bci, const double* __restrict__ bv,
                          double alpha, double beta, i64* cc, const i64* __restrict__ crp,
                          int* __restrict__ cci, double* __restrict__ cv) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    i64 a = arp[i], ae = arp[i + 1], b = brp[i], be = brp[i + 1];
    i64 o = crp ? crp[i] : 0, c = 0;
    while (a < ae || b < be) {
      int col;
      double x;
      if (b >= be || (a < ae && aci[a] < bci[b])) {
        col = aci[a];
        x = cv ? __dmul_rn(alpha, av[a]) : 0.0;
        a++;
      } else if (a >= ae || bci[b] < aci[a]) {
        col = bci[b];
        x = cv ? __dmul_rn(beta, bv[b]) : 0.0;
        b++;
      } else {
        col = aci[a];
        x = cv ? __dadd_rn(__dmul_rn(alpha, av[a]), __dmul_rn(beta, bv[b])) : 0.0;
        a++;
        b++;
      }
      if (cci) {
        cci[o + c] = col;
        cv[o + c] = x;
      }
      c++;
    }
    if (cc) cc[i] = c;
  }
}

extern "C" int sphc_csr_add_count(int64_t n, const int64_t* arp, const int32_t* aci,
                                  const int64_t* brp, const int32_t* bci, int64_t* counts,
                                  void* stream) {
  cudaStream_t s = as_stream(stream);
  k_csr_add<<<grid_for(n, 128), 128, 0, s>>>(n, arp, aci, nullptr, brp, bci, nullptr, 0.0, 0.0,
                                             counts, nullptr, nullptr, nullptr);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_csr_add_fill(int64_t n, const int64_t* arp, const int32_t* aci,
                                 const double* av, const int64_t* brp, const int32_t* bci,
                                 const double* bv, double alpha, double beta, const int64_t* crp,
                                 int32_t* cci, double* cv, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_csr_add<<<grid_for(n, 128), 128, 0, s>>>(n, arp, aci, av, brp, bci, bv, alpha, beta, nullptr,
                                             crp, cci, cv);
  SPHC_LAUNCH_CHECK();
  return 0;
}
