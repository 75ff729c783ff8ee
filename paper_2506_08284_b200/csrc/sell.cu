// SELL-32 mirror of the square smoother operators (A_e, D^T A_e D on every
// level): slices of 32 consecutive rows stored column-major and padded to the
// slice's longest row, so one warp = one slice and one thread = one row. Every
// load of the j-loop is a coalesced 256 B (values) / 128 B (columns) line and
// a thread's loads are independent, which keeps many requests in flight per
// SM -- the HBM-bound V-cycle kernels run on this layout.
// Padding entries carry value 0 and the row's own column.
#include "common.cuh"
#include <stdlib.h>

#define SELL_C 32
#define SELL_PER_BLOCK 256   // threads per block of the SpMV-type kernels

__global__ void k_sell_widths(i64 n, const i64* __restrict__ rp, i64* __restrict__ width) {
  i64 ns = (n + SELL_C - 1) / SELL_C;
  int lane = threadIdx.x & 31;
  i64 w0 = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 s = w0; s < ns; s += nw) {
    i64 row = s * SELL_C + lane;
    int len = row < n ? (int)(rp[row + 1] - rp[row]) : 0;
    for (int o = 16; o > 0; o >>= 1) len = max(len, __shfl_xor_sync(FULL_MASK, len, o));
    if (lane == 0) width[s] = (i64)len * SELL_C;   // entries of the slice
  }
}

extern "C" int sphc_sell_sizes(int64_t n, const int64_t* rp, int64_t* slice_entries,
                               void* stream) {
  cudaStream_t s = as_stream(stream);
  k_sell_widths<<<grid_for(n, 256), 256, 0, s>>>(n, rp, slice_entries);
  SPHC_LAUNCH_CHECK();
  return 0;
}

template <bool RECT>
__global__ void k_sell_fill(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                            const double* __restrict__ v, const i64* __restrict__ sp,
                            int* __restrict__ sci, double* __restrict__ sv) {
  for (i64 row = (i64)blockIdx.x * blockDim.x + threadIdx.x; row < ((n + 31) & ~(i64)31);
       row += (i64)gridDim.x * blockDim.x) {
    i64 s = row / SELL_C;
    int r = (int)(row % SELL_C);
    int w = (int)((sp[s + 1] - sp[s]) / SELL_C);
    i64 base = sp[s] + r;
    int len = 0;
    i64 j0 = 0;
    if (row < n) {
      j0 = rp[row];
      len = (int)(rp[row + 1] - j0);
    }
    int self = RECT ? (len ? ci[j0] : 0) : (row < n ? (int)row : 0);
    for (int j = 0; j < w; j++) {
      bool real = j < len;
      sci[base + (i64)j * SELL_C] = real ? ci[j0 + j] : self;
      sv[base + (i64)j * SELL_C] = real ? v[j0 + j] : 0.0;
    }
  }
}

extern "C" int sphc_sell_fill(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                              const int64_t* slice_ptr, int32_t* sci, double* sv,
                              void* stream) {
  cudaStream_t s = as_stream(stream);
  k_sell_fill<false><<<grid_for(n, 256), 256, 0, s>>>(n, rp, ci, v, slice_ptr, sci, sv);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// Rectangular operators (A_e D: n_e x n_n): a padding entry repeats the
// row's first column (0 for an empty row) instead of the row index, which
// need not be a valid column.
extern "C" int sphc_sell_fill_rect(int64_t n, const int64_t* rp, const int32_t* ci,
                                   const double* v, const int64_t* slice_ptr, int32_t* sci,
                                   double* sv, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_sell_fill<true><<<grid_for(n, 256), 256, 0, s>>>(n, rp, ci, v, slice_ptr, sci, sv);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// Operators whose SELL arrays exceed this stay out of L2 (streaming,
// evict-first loads keep the x gathers resident); smaller ones (coarse
// levels, the C2 finest level) are re-read by every Chebyshev step and are
// loaded with the default policy so they stay L2-resident across the V-cycle.
#define SELL_STREAM_BYTES (48ll << 20)

// One thread's share of a row: entries j = q, q + K, ... of its SELL row,
// summed in ascending j with fma (the same order for every K = 1 launch).
// Entries are processed in groups of SELL_U: the group's column / value
// loads are all issued before any dependent x gather, so a cold row costs
// ~2 memory round trips per group instead of per entry pair.
// Groups of 8 for the L2-sized operators (latency bound: few warps per SM);
// 4 for the streaming ones (bandwidth bound: 32 registers keep 64 warps
// resident per SM).
template <bool STREAM, int K, int SELL_U = STREAM ? 4 : 8>
__device__ __forceinline__ double sell_row(i64 base, int w, int q, const int* __restrict__ sci,
                                           const double* __restrict__ sv,
                                           const double* __restrict__ x) {
  double acc = 0.0;
  for (int j0 = q; j0 < w; j0 += SELL_U * K) {
    int c[SELL_U];
    double v[SELL_U];
#pragma unroll
    for (int u = 0; u < SELL_U; u++) {
      int j = j0 + u * K;
      if (j < w) {
        i64 o = base + (i64)j * SELL_C;
        v[u] = STREAM ? __ldcs(sv + o) : __ldg(sv + o);
        c[u] = STREAM ? __ldcs(sci + o) : __ldg(sci + o);
      }
    }
#pragma unroll
    for (int u = 0; u < SELL_U; u++)
      if (j0 + u * K < w) acc = fma(v[u], __ldg(x + c[u]), acc);
  }
  return acc;
}

// Row sums of A x over the slice owned by this warp. K > 1 splits every
// slice's columns over K warps of the block (interleaved j = q, q + K, ...;
// each load stays a coalesced 256 B line) and combines the partial sums in
// shared memory in a fixed order: small operators (C2's finest level has
// 2,883 slices, ~19 warps per SM at K = 1) get K times the loads in flight.
// Returns true on the lane that owns the epilogue of `row`.
template <bool STREAM, int K>
__device__ __forceinline__ bool sell_rowsum(i64 n, const i64* __restrict__ sp,
                                            const int* __restrict__ sci,
                                            const double* __restrict__ sv,
                                            const double* __restrict__ x, bool skip, i64& row,
                                            double& acc) {
  __shared__ double part[SELL_PER_BLOCK / 32][32];
  int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int q = warp % K;
  i64 s = (i64)blockIdx.x * (SELL_PER_BLOCK / 32 / K) + warp / K;
  i64 ns = (n + SELL_C - 1) / SELL_C;
  row = s * SELL_C + lane;
  acc = 0.0;
  if (s < ns && !skip) {
    i64 b0 = sp[s];
    int w = (int)((sp[s + 1] - b0) / SELL_C);
    acc = sell_row<STREAM, K>(b0 + lane, w, q, sci, sv, x);
  }
  if (K > 1) {
    part[warp][lane] = acc;
    __syncthreads();
    if (q != 0) return false;
    acc = part[warp][lane];
    for (int t = 1; t < K; t++) acc += part[warp + t][lane];
  }
  return s < ns && row < n;
}

// y = alpha A x + beta z
template <bool STREAM, int K>
__global__ void __launch_bounds__(SELL_PER_BLOCK, (STREAM && K == 1) ? 8 : 5)
    k_sell_spmv(i64 n, const i64* __restrict__ sp, const int* __restrict__ sci,
                const double* __restrict__ sv, const double* __restrict__ x, double alpha,
                double beta, const double* z, double* y) {
  pdl_begin();
  i64 row;
  double acc;
  if (!sell_rowsum<STREAM, K>(n, sp, sci, sv, x, false, row, acc)) return;
  double r = alpha * acc;
  if (z) r = fma(beta, z[row], r);
  y[row] = r;
}

// d <- cd d + cr dinv (b - A x_in); x_out = x_in + d
template <bool STREAM, int K>
__global__ void __launch_bounds__(SELL_PER_BLOCK, (STREAM && K == 1) ? 8 : 5)
    k_sell_cheb(i64 n, const i64* __restrict__ sp, const int* __restrict__ sci,
                const double* __restrict__ sv, const double* __restrict__ dinv,
                const double* __restrict__ b, const double* __restrict__ x_in,
                double* __restrict__ x_out, double* __restrict__ d, double cd, double cr,
                int x_zero) {
  pdl_begin();
  i64 row;
  double ax;
  if (!sell_rowsum<STREAM, K>(n, sp, sci, sv, x_in, x_zero != 0, row, ax)) return;
  double r = b[row] - ax;
  double dn = cr * dinv[row] * r;
  if (cd != 0.0) dn = fma(cd, d[row], dn);
  d[row] = dn;
  x_out[row] = (x_zero ? 0.0 : x_in[row]) + dn;
}

// warps per slice: K = 1 once the slices alone fill ~48 warps per SM;
// K = 8 for tiny operators (below); otherwise the largest K in {2, 4} whose
// grid still fits one wave
// (8 blocks of 256 threads per SM) -- a second partial wave costs more than
// the extra loads in flight gain. SPHC_SELL_K overrides (tuning).
static inline int sell_split(i64 n) {
  static int forced = -1, sell_k8 = -1;
  if (sell_k8 < 0) {
    const char* e = getenv("SPHC_SELL_K8");
    sell_k8 = (e && e[0] == '0') ? 0 : 1;
  }
  if (forced < 0) {
    const char* e = getenv("SPHC_SELL_K");
    forced = e ? atoi(e) : 0;
  }
  if (forced == 1 || forced == 2 || forced == 4 || forced == 8) return forced;
  i64 ns = (n + SELL_C - 1) / SELL_C;
  if (ns >= (i64)SPHC_NUM_SMS * 48) return 1;
  const i64 wave = (i64)SPHC_NUM_SMS * 8;
  // 1 slice per block for the smallest operators (C2 level 1: 219 slices,
  // ~44 entries per row -> one load group per thread; 4.96 -> 4.88 ms per
  // C2 solve). Measured slower at C2's 931-slice level-0 nodal operator.
  if (sell_k8 && ns * 4 <= wave) return 8;
  if ((ns + 1) / 2 <= wave) return 4;    // 2 slices per block
  if ((ns + 3) / 4 <= wave) return 2;    // 4 slices per block
  return 1;
}

static inline unsigned sell_grid(i64 n, int K) {
  i64 ns = (n + SELL_C - 1) / SELL_C;
  i64 per = SELL_PER_BLOCK / 32 / K;
  return (unsigned)((ns + per - 1) / per);
}

#define SELL_DISPATCH(KERNEL, STREAMING, ...)                                     \
  do {                                                                           \
    int K_ = sell_split(n);                                                      \
    unsigned g_ = sell_grid(n, K_);                                              \
    if (STREAMING) {                                                             \
      if (K_ == 1) launch_pdl(KERNEL<true, 1>, g_, SELL_PER_BLOCK, 0, s, __VA_ARGS__);   \
      else if (K_ == 2) launch_pdl(KERNEL<true, 2>, g_, SELL_PER_BLOCK, 0, s, __VA_ARGS__); \
      else if (K_ == 4) launch_pdl(KERNEL<true, 4>, g_, SELL_PER_BLOCK, 0, s, __VA_ARGS__); \
      else launch_pdl(KERNEL<true, 8>, g_, SELL_PER_BLOCK, 0, s, __VA_ARGS__);           \
    } else {                                                                     \
      if (K_ == 1) launch_pdl(KERNEL<false, 1>, g_, SELL_PER_BLOCK, 0, s, __VA_ARGS__);  \
      else if (K_ == 2) launch_pdl(KERNEL<false, 2>, g_, SELL_PER_BLOCK, 0, s, __VA_ARGS__); \
      else if (K_ == 4) launch_pdl(KERNEL<false, 4>, g_, SELL_PER_BLOCK, 0, s, __VA_ARGS__); \
      else launch_pdl(KERNEL<false, 8>, g_, SELL_PER_BLOCK, 0, s, __VA_ARGS__);          \
    }                                                                            \
  } while (0)

extern "C" int sphc_sell_spmv(int64_t n, const int64_t* slice_ptr, const int32_t* sci,
                              const double* sv, const double* x, double alpha, double beta,
                              const double* z, double* y, int64_t padded, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  SELL_DISPATCH(k_sell_spmv, padded * 12 > SELL_STREAM_BYTES, n, slice_ptr, sci, sv, x, alpha,
                beta, z, y);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_sell_cheb_step(int64_t n, const int64_t* slice_ptr, const int32_t* sci,
                                   const double* sv, const double* dinv, const double* b,
                                   const double* x_in, double* x_out, double* d, double cd,
                                   double cr, int x_zero, int64_t padded, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  SELL_DISPATCH(k_sell_cheb, padded * 12 > SELL_STREAM_BYTES, n, slice_ptr, sci, sv, dinv, b,
                x_in, x_out, d, cd, cr, x_zero);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// Delta-coded columns for the streamed operators. A row's sorted columns are
// stored as 16-bit differences to the previous one (the first column of every
// row in a 32-bit array; padding repeats the last column: delta 0, value 0),
// so a pass moves 10 instead of 12 bytes per stored entry -- the V-cycle's
// A_e passes run at the HBM roofline, so fewer bytes is the only lever left.
// Same entries, same order, same fma chain: bitwise the 32-bit kernels.
// Eligible when every difference fits 16 bits (sphc_sell_fill16 reports it):
// true for the 128^3 mesh numbering (largest jump ~3 N^2 = 49.9k).
#define SELL16_ESC 0xFFFF   // difference code: restart from the row's next base
#define SELL16_NBASE 4      // bases per row of the escaped variant

__global__ void k_sell_fill16(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                              const i64* __restrict__ sp, unsigned short* __restrict__ d16,
                              int* __restrict__ c0, int* too_big, int rect, int nbase) {
  bool big = false;
  for (i64 row = (i64)blockIdx.x * blockDim.x + threadIdx.x; row < ((n + 31) & ~(i64)31);
       row += (i64)gridDim.x * blockDim.x) {
    i64 s = row / SELL_C;
    int r = (int)(row % SELL_C);
    int w = (int)((sp[s + 1] - sp[s]) / SELL_C);
    i64 base = sp[s] + r;
    int len = 0;
    i64 j0 = 0;
    if (row < n) {
      j0 = rp[row];
      len = (int)(rp[row + 1] - j0);
    }
    int prev = len ? ci[j0] : ((row < n && !rect) ? (int)row : 0);
    int g = 0;
    if (row < n) {
      c0[row * nbase] = prev;
      for (int q = 1; q < nbase; q++) c0[row * nbase + q] = prev;
    }
    for (int j = 0; j < w; j++) {
      int c = j < len ? ci[j0 + j] : prev;
      int d = c - prev;
      if (d < 0 || d >= SELL16_ESC) {
        // a jump beyond 16 bits (the next mesh plane at 256^3): restart from
        // the row's next 32-bit base, if it has one left
        if (g + 1 < nbase && row < n) {
          c0[row * nbase + (++g)] = c;
          d = SELL16_ESC;
        } else {
          big = true;
          d = 0;
        }
      }
      d16[base + (i64)j * SELL_C] = (unsigned short)d;
      prev = c;
    }
  }
  if (big) *too_big = 1;
}

extern "C" int sphc_sell_fill16(int64_t n, const int64_t* rp, const int32_t* ci,
                                const int64_t* slice_ptr, uint16_t* d16, int32_t* c0,
                                int32_t* too_big, int rect, int nbase, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (nbase != 1 && nbase != SELL16_NBASE) return SPHC_ERR_ARG;
  SPHC_CUDA(cudaMemsetAsync(too_big, 0, sizeof(int32_t), s));
  k_sell_fill16<<<grid_for(n, 256), 256, 0, s>>>(n, rp, ci, slice_ptr, d16, c0, too_big, rect,
                                                 nbase);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// entries per load group: 6 keeps ~50% more bytes in flight than the 32-bit
// kernels' 4 at the same 32 registers (C4: 0.4065 -> 0.3865 ms per pass; 8
// measures the same; packing two differences per word measured slower)
#ifndef SELL16_U
#define SELL16_U 6
#endif
// one thread's row: the column runs along with the 16-bit differences
template <int NB>
__device__ __forceinline__ double sell_row16(i64 base, int w, const int* __restrict__ bases,
                                             const unsigned short* __restrict__ d16,
                                             const double* __restrict__ sv,
                                             const double* __restrict__ x) {
  constexpr int U = SELL16_U;
  double acc = 0.0;
  int c = bases[0];
  int nb[NB > 1 ? NB - 1 : 1];
  if (NB > 1) {
#pragma unroll
    for (int q = 1; q < NB; q++) nb[q - 1] = bases[q];
  }
  int g = 0;
  for (int j0 = 0; j0 < w; j0 += U) {
    unsigned short d[U];
    double v[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      int j = j0 + u;
      d[u] = 0;
      v[u] = 0.0;
      if (j < w) {
        i64 o = base + (i64)j * SELL_C;
        v[u] = __ldcs(sv + o);
        d[u] = __ldcs(d16 + o);
      }
    }
#pragma unroll
    for (int u = 0; u < U; u++)
      if (j0 + u < w) {
        if (NB > 1 && d[u] == SELL16_ESC) {
          // (NB - 1 = 3 further bases: a select chain, no local memory)
          c = g == 0 ? nb[0] : (g == 1 ? nb[NB > 2 ? 1 : 0] : nb[NB > 3 ? 2 : 0]);
          g++;
        } else {
          c += d[u];
        }
        acc = fma(v[u], __ldg(x + c), acc);
      }
  }
  return acc;
}

// y = alpha A x + beta z (streamed operators, one warp per slice)
template <int NB>
__global__ void __launch_bounds__(SELL_PER_BLOCK, NB > 1 ? 6 : 8)
    k_sell_spmv16(i64 n, const i64* __restrict__ sp, const unsigned short* __restrict__ d16,
                  const int* __restrict__ c0, const double* __restrict__ sv,
                  const double* __restrict__ x, double alpha, double beta, const double* z,
                  double* y) {
  pdl_begin();
  i64 row = (i64)blockIdx.x * SELL_PER_BLOCK + threadIdx.x;
  if (row >= n) return;
  i64 s = row >> 5;
  i64 b0 = sp[s];
  int w = (int)((sp[s + 1] - b0) / SELL_C);
  double acc = sell_row16<NB>(b0 + (threadIdx.x & 31), w, c0 + row * NB, d16, sv, x);
  double r = alpha * acc;
  if (z) r = fma(beta, z[row], r);
  y[row] = r;
}

// d <- cd d + cr dinv (b - A x_in); x_out = x_in + d
template <int NB>
__global__ void __launch_bounds__(SELL_PER_BLOCK, NB > 1 ? 6 : 8)
    k_sell_cheb16(i64 n, const i64* __restrict__ sp, const unsigned short* __restrict__ d16,
                  const int* __restrict__ c0, const double* __restrict__ sv,
                  const double* __restrict__ dinv, const double* __restrict__ b,
                  const double* __restrict__ x_in, double* __restrict__ x_out,
                  double* __restrict__ d, double cd, double cr) {
  pdl_begin();
  i64 row = (i64)blockIdx.x * SELL_PER_BLOCK + threadIdx.x;
  if (row >= n) return;
  i64 s = row >> 5;
  i64 b0 = sp[s];
  int w = (int)((sp[s + 1] - b0) / SELL_C);
  double ax = sell_row16<NB>(b0 + (threadIdx.x & 31), w, c0 + row * NB, d16, sv, x_in);
  double r = b[row] - ax;
  double dn = cr * dinv[row] * r;
  if (cd != 0.0) dn = fma(cd, d[row], dn);
  d[row] = dn;
  x_out[row] = x_in[row] + dn;
}

extern "C" int sphc_sell_spmv16(int64_t n, const int64_t* slice_ptr, const uint16_t* d16,
                                const int32_t* c0, const double* sv, const double* x,
                                double alpha, double beta, const double* z, double* y,
                                int nbase, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  unsigned g = (unsigned)((n + SELL_PER_BLOCK - 1) / SELL_PER_BLOCK);
  if (nbase == 1)
    launch_pdl(k_sell_spmv16<1>, g, SELL_PER_BLOCK, 0, s, n, slice_ptr, d16, c0, sv, x, alpha,
               beta, z, y);
  else
    launch_pdl(k_sell_spmv16<SELL16_NBASE>, g, SELL_PER_BLOCK, 0, s, n, slice_ptr, d16, c0, sv,
               x, alpha, beta, z, y);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_sell_cheb_step16(int64_t n, const int64_t* slice_ptr, const uint16_t* d16,
                                     const int32_t* c0, const double* sv, const double* dinv,
                                     const double* b, const double* x_in, double* x_out,
                                     double* d, double cd, double cr, int nbase,
                                     void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  unsigned g = (unsigned)((n + SELL_PER_BLOCK - 1) / SELL_PER_BLOCK);
  if (nbase == 1)
    launch_pdl(k_sell_cheb16<1>, g, SELL_PER_BLOCK, 0, s, n, slice_ptr, d16, c0, sv, dinv, b,
               x_in, x_out, d, cd, cr);
  else
    launch_pdl(k_sell_cheb16<SELL16_NBASE>, g, SELL_PER_BLOCK, 0, s, n, slice_ptr, d16, c0, sv,
               dinv, b, x_in, x_out, d, cd, cr);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// Hiptmair mid step (multigrid.py:164-173, between the nodal correction and
// the second edge sweep): x1 = x + D c, then the first Chebyshev step of the
// next edge sweep taken from the residual r = b - A x the caller already
// holds, since b - A (x + D c) = r - (A D) c:
//   d = cr dinv (r - (A D) c);   x_out = (x + D c) + d
// One pass over the SELL mirror of A D (~18 entries per row against ~33 for
// A_e) replaces the D pass and one A_e pass of the V-cycle. D from its CSR
// (<= 2 entries per row on these gradients; any length is handled).
template <bool STREAM, int K>
__global__ void __launch_bounds__(SELL_PER_BLOCK, (STREAM && K == 1) ? 8 : 5)
    k_sell_hipt_mid(i64 n, const i64* __restrict__ sp, const int* __restrict__ sci,
                    const double* __restrict__ sv, const i64* __restrict__ drp,
                    const int* __restrict__ dci, const double* __restrict__ dvv,
                    const double* __restrict__ dinv, const double* __restrict__ r,
                    const double* __restrict__ c, const double* __restrict__ x_in,
                    double* __restrict__ x_out, double* __restrict__ d, double cr) {
  pdl_begin();
  i64 row;
  double adc;
  if (!sell_rowsum<STREAM, K>(n, sp, sci, sv, c, false, row, adc)) return;
  i64 j0 = drp[row], j1 = drp[row + 1];
  double u = 0.0;
  for (i64 j = j0; j < j1; j++) u = fma(dvv[j], __ldg(c + dci[j]), u);
  double dn = cr * dinv[row] * (r[row] - adc);
  d[row] = dn;
  x_out[row] = (x_in[row] + u) + dn;
}

// the same step on delta-coded columns of A D (one warp per slice)
template <int NB>
__global__ void __launch_bounds__(SELL_PER_BLOCK, NB > 1 ? 6 : 8)
    k_sell_hipt_mid16(i64 n, const i64* __restrict__ sp, const unsigned short* __restrict__ d16,
                      const int* __restrict__ c0, const double* __restrict__ sv,
                      const i64* __restrict__ drp, const int* __restrict__ dci,
                      const double* __restrict__ dvv, const double* __restrict__ dinv,
                      const double* __restrict__ r, const double* __restrict__ c,
                      const double* __restrict__ x_in, double* __restrict__ x_out,
                      double* __restrict__ d, double cr) {
  pdl_begin();
  i64 row = (i64)blockIdx.x * SELL_PER_BLOCK + threadIdx.x;
  if (row >= n) return;
  i64 s = row >> 5;
  i64 b0 = sp[s];
  int w = (int)((sp[s + 1] - b0) / SELL_C);
  double adc = sell_row16<NB>(b0 + (threadIdx.x & 31), w, c0 + row * NB, d16, sv, c);
  i64 j0 = drp[row], j1 = drp[row + 1];
  double u = 0.0;
  for (i64 j = j0; j < j1; j++) u = fma(dvv[j], __ldg(c + dci[j]), u);
  double dn = cr * dinv[row] * (r[row] - adc);
  d[row] = dn;
  x_out[row] = (x_in[row] + u) + dn;
}

extern "C" int sphc_sell_hipt_mid16(int64_t n, const int64_t* slice_ptr, const uint16_t* d16,
                                    const int32_t* c0, const double* sv, const int64_t* drp,
                                    const int32_t* dci, const double* dv, const double* dinv,
                                    const double* r, const double* c, const double* x_in,
                                    double* x_out, double* d, double cr, int nbase,
                                    void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  unsigned g = (unsigned)((n + SELL_PER_BLOCK - 1) / SELL_PER_BLOCK);
  if (nbase == 1)
    launch_pdl(k_sell_hipt_mid16<1>, g, SELL_PER_BLOCK, 0, s, n, slice_ptr, d16, c0, sv, drp, dci,
               dv, dinv, r, c, x_in, x_out, d, cr);
  else
    launch_pdl(k_sell_hipt_mid16<SELL16_NBASE>, g, SELL_PER_BLOCK, 0, s, n, slice_ptr, d16, c0, sv,
               drp, dci, dv, dinv, r, c, x_in, x_out, d, cr);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_sell_hipt_mid(int64_t n, const int64_t* slice_ptr, const int32_t* sci,
                                  const double* sv, const int64_t* drp, const int32_t* dci,
                                  const double* dv, const double* dinv, const double* r,
                                  const double* c, const double* x_in, double* x_out,
                                  double* d, double cr, int64_t padded, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  SELL_DISPATCH(k_sell_hipt_mid, padded * 12 > SELL_STREAM_BYTES, n, slice_ptr, sci, sv, drp,
                dci, dv, dinv, r, c, x_in, x_out, d, cr);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// ---------------------------------------------------------------------------
// The whole k-step Lanczos bound estimate of a Chebyshev smoother (D^-1 A in
// the D inner product, ChebyshevSweeper._lanczos) in ONE cooperative launch:
// grid-wide barriers replace the ~7 launches per step of the step-by-step
// version. Per step: (A) v = w / |w|_D and u = A v on this thread's rows,
// partial u.v; (B) w = D^-1 u - alpha v - beta v_prev, partial w.Dw. Dot
// products are block trees written to per-block partials and summed by every
// block in the same fixed order (deterministic, identical in every block).
#include <cooperative_groups.h>
namespace cgrp = cooperative_groups;

#define LZ_THREADS 256
#define LZ_MAX_BLOCKS 2048

__device__ __forceinline__ double lz_block_sum(double v, double* sh) {
  v = warp_sum(v);
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = lane < (int)(blockDim.x >> 5) ? sh[lane] : 0.0;
    t = warp_sum(t);
  }
  return t;   // valid in warp 0
}

// grid-wide deterministic sum; `part` alternates halves between calls
__device__ __forceinline__ double lz_grid_sum(double v, double* part, int& half,
                                              cgrp::grid_group& grid, double* sh) {
  double b = lz_block_sum(v, sh);
  double* P = part + half * LZ_MAX_BLOCKS;
  half ^= 1;
  if (threadIdx.x == 0) P[blockIdx.x] = b;
  grid.sync();
  double t = 0.0;
  if (threadIdx.x < 32) {
    for (int i = threadIdx.x; i < (int)gridDim.x; i += 32) t += P[i];
    t = warp_sum(t);
    if (threadIdx.x == 0) sh[32] = t;
  }
  __syncthreads();
  return sh[32];
}

__device__ __forceinline__ double lz_start(i64 i) {
  unsigned long long z = (unsigned long long)i + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z = z ^ (z >> 31);
  return (double)(z >> 11) * 0x1p-53 * 2.0 - 1.0;
}

__global__ void __launch_bounds__(LZ_THREADS)
    k_lanczos_coop(i64 n, const i64* __restrict__ sp, const int* __restrict__ sci,
                   const double* __restrict__ sv, const double* __restrict__ d,
                   const double* __restrict__ dinv, double* v, double* vprev, double* w,
                   double* u, int k, double* sc, double* part, int K) {
  cgrp::grid_group grid = cgrp::this_grid();
  __shared__ double sh[33];
  int half = 0;
  const i64 nt = (i64)gridDim.x * blockDim.x;
  const i64 t0 = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  for (i64 i = t0; i < n; i += nt) {
    double x = lz_start(i);
    w[i] = x;
    acc += x * (d[i] * x);
  }
  double nrm = sqrt(lz_grid_sum(acc, part, half, grid, sh));
  if (t0 == 0) sc[k] = nrm;                         // beta_0
  for (int j = 0; j < k; j++) {
    acc = 0.0;
    double inv = 1.0 / nrm;
    // (A): K consecutive lanes share a row (K > 1 when the rows alone cannot
    // fill the SMs), each taking every K-th SELL column; lane-group trees
    const i64 nrt = ((n + 31) & ~(i64)31) * K;     // warp-uniform trip count
    for (i64 g = t0; g < nrt; g += nt) {
      i64 i = g / K;
      int part = (int)(g % K);
      double t = 0.0;
      if (i < n) {
        i64 s = i / SELL_C;
        int r = (int)(i % SELL_C);
        i64 base = sp[s] + r;
        int width = (int)((sp[s + 1] - sp[s]) / SELL_C);
#pragma unroll 4
        for (int q = part; q < width; q += K) {
          i64 e = base + (i64)q * SELL_C;
          t = fma(sv[e], w[sci[e]], t);
        }
      }
      for (int o = K >> 1; o > 0; o >>= 1) t += __shfl_xor_sync(FULL_MASK, t, o);
      if (i < n && part == 0) {
        double vi = w[i] * inv, ui = t * inv;
        v[i] = vi;
        u[i] = ui;
        acc += ui * vi;
      }
    }
    double alpha = lz_grid_sum(acc, part, half, grid, sh);
    if (t0 == 0) sc[j] = alpha;
    acc = 0.0;
    for (i64 i = t0; i < n; i += nt) {               // (B)
      double t = dinv[i] * u[i] - alpha * v[i];
      if (j) t -= nrm * vprev[i];
      w[i] = t;
      acc += t * (d[i] * t);
    }
    nrm = sqrt(lz_grid_sum(acc, part, half, grid, sh));
    if (t0 == 0) sc[k + j + 1] = nrm;               // beta_{j+1}
    double* tmp = v;
    v = vprev;
    vprev = tmp;
  }
}

extern "C" int sphc_lanczos_sell(int64_t n, const int64_t* slice_ptr, const int32_t* sci,
                                 const double* sv, const double* d, const double* dinv, int k,
                                 double* v, double* vprev, double* w, double* u, double* sc,
                                 void* stream) {
  if (n <= 0) return 0;
  static double* part = nullptr;
  static int max_blocks = 0;
  if (!part) {
    SPHC_CUDA(cudaMalloc((void**)&part, 2 * LZ_MAX_BLOCKS * sizeof(double)));
    int per_sm = 0;
    SPHC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lanczos_coop,
                                                            LZ_THREADS, 0));
    max_blocks = per_sm * SPHC_NUM_SMS;
    if (max_blocks > LZ_MAX_BLOCKS) max_blocks = LZ_MAX_BLOCKS;
  }
  // lanes per row: enough rows x lanes for ~2 blocks per SM
  int K = 1;
  while (K < 32 && n * K < (i64)2 * SPHC_NUM_SMS * LZ_THREADS) K <<= 1;
  i64 want = (((n + 31) & ~(i64)31) * K + LZ_THREADS - 1) / LZ_THREADS;
  int g = (int)(want < max_blocks ? want : max_blocks);
  i64 nn = n;
  void* args[] = {&nn, (void*)&slice_ptr, (void*)&sci, (void*)&sv, (void*)&d, (void*)&dinv,
                  &v, &vprev, &w, &u, &k, &sc, &part, &K};
  SPHC_CUDA(cudaLaunchCooperativeKernel((void*)k_lanczos_coop, dim3(g), dim3(LZ_THREADS), args,
                                        0, as_stream(stream)));
  g_sphc_launches++;
  return 0;
}

// ---------------------------------------------------------------------------
// KS consecutive Chebyshev steps (KS = 2 or 3) in ONE pass over the matrix:
// the rows are cut into blocks of FZ_ROWS; CTAs claim time slots t in
// ascending order and, at slot t, run step p on block t - (p-1)(L+1) for
// p = 1..KS. Step p of block b waits until step p-1 is done on every block
// within the matrix bandwidth (blocks b-L..b+L), so it reads complete
// values, and it reads block b's SELL rows while step p-1 left them in L2
// (the window of (KS-1)(L+1) blocks is sized to fit L2 by the caller).
// Every row's arithmetic is the unfused kernel's (k_sell_cheb<true,1>): same
// loads, same fma order, same epilogue -- the result is bitwise identical.
// Buffers written by one CTA and read by another go through L2 (ld.cg /
// release-acquire flags): L1 is not coherent across SMs.
#define FZ_ROWS 256

struct FzStep {
  const double* xin;
  double* xout;
  double cd, cr;
};
struct FzArgs {
  FzStep st[3];
};

__device__ __forceinline__ int fz_ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int KS>
__global__ void __launch_bounds__(FZ_ROWS)
    k_sell_cheb_fused(i64 n, const i64* __restrict__ sp, const int* __restrict__ sci,
                      const double* __restrict__ sv, const double* __restrict__ dinv,
                      const double* __restrict__ b, double* d, FzArgs a, int x_zero, int L,
                      int nblk, int* ticket, int* done) {
  __shared__ int slot;
  const int nslots = nblk + (KS - 1) * (L + 1);
  for (;;) {
    if (threadIdx.x == 0) slot = atomicAdd(ticket, 1);
    __syncthreads();
    int t = slot;
    __syncthreads();
    if (t >= nslots) return;
#pragma unroll
    for (int p = 0; p < KS; p++) {
      int blk = t - p * (L + 1);
      if (blk < 0 || blk >= nblk) continue;
      if (p > 0) {   // step p-1 done on blocks [blk - L, blk + L]
        const int* prev = done + (size_t)(p - 1) * nblk;
        int lo = max(0, blk - L), hi = min(nblk - 1, blk + L);
        for (;;) {
          bool ok = true;
          for (int c = lo + threadIdx.x; c <= hi; c += FZ_ROWS) ok &= fz_ld_acquire(prev + c) != 0;
          if (__syncthreads_and(ok)) break;
        }
      }
      const FzStep st = a.st[p];
      const bool zero = x_zero && p == 0;
      i64 row = (i64)blk * FZ_ROWS + threadIdx.x;
      if (row < n) {
        i64 s = row / SELL_C;
        int r = (int)(row % SELL_C);
        i64 b0 = sp[s];
        int w = (int)((sp[s + 1] - b0) / SELL_C);
        double acc = 0.0;
        if (!zero) {
          i64 base = b0 + r;
          for (int j0 = 0; j0 < w; j0 += 4) {
            int c[4];
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
              int j = j0 + u;
              if (j < w) {
                i64 o = base + (i64)j * SELL_C;
                // the last step streams the matrix out of L2; earlier ones
                // leave it for the next step
                v[u] = (p == KS - 1) ? __ldcs(sv + o) : __ldg(sv + o);
                c[u] = (p == KS - 1) ? __ldcs(sci + o) : __ldg(sci + o);
              }
            }
#pragma unroll
            for (int u = 0; u < 4; u++)
              if (j0 + u < w) acc = fma(v[u], __ldcg(st.xin + c[u]), acc);
          }
        }
        double res = b[row] - acc;
        double dn = st.cr * dinv[row] * res;
        if (st.cd != 0.0) dn = fma(st.cd, __ldcg(d + row), dn);
        __stcg(d + row, dn);
        __stcg(st.xout + row, (zero ? 0.0 : __ldcg(st.xin + row)) + dn);
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(done + (size_t)p * nblk + blk),
                     "r"(1)
                     : "memory");
      }
    }
  }
}

// maximum |col - row| of a CSR matrix (the fused steps' dependency range)
__global__ void k_csr_bandwidth(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                                unsigned long long* out) {
  unsigned long long m = 0;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    i64 s = rp[i], e = rp[i + 1];
    if (e > s) {
      i64 a = (i64)ci[s] - i, z = (i64)ci[e - 1] - i;   // sorted columns
      unsigned long long v = (unsigned long long)max(a < 0 ? -a : a, z < 0 ? -z : z);
      m = max(m, v);
    }
  }
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(FULL_MASK, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

extern "C" int sphc_csr_bandwidth(int64_t n, const int64_t* rp, const int32_t* ci,
                                  int64_t* out, void* stream) {
  cudaStream_t s = as_stream(stream);
  SPHC_CUDA(cudaMemsetAsync(out, 0, sizeof(int64_t), s));
  if (n <= 0) return 0;
  k_csr_bandwidth<<<grid_for(n, 256), 256, 0, s>>>(n, rp, ci, (unsigned long long*)out);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_sell_cheb_fused(int64_t n, const int64_t* slice_ptr, const int32_t* sci,
                                    const double* sv, const double* dinv, const double* b,
                                    double* d, int nsteps, const double* xin0, double* xout0,
                                    double cd0, double cr0, const double* xin1, double* xout1,
                                    double cd1, double cr1, const double* xin2, double* xout2,
                                    double cd2, double cr2, int x_zero, int L, int32_t* sync,
                                    void* stream) {
  if (n <= 0) return 0;
  if (nsteps < 2 || nsteps > 3 || L < 0) {
    sphc_set_error("sphc_sell_cheb_fused: nsteps must be 2 or 3");
    return SPHC_ERR_ARG;
  }
  cudaStream_t s = as_stream(stream);
  int nblk = (int)((n + FZ_ROWS - 1) / FZ_ROWS);
  // sync = [ticket | done flags: nsteps x nblk]
  SPHC_CUDA(cudaMemsetAsync(sync, 0, (size_t)(1 + nsteps * nblk) * sizeof(int32_t), s));
  FzArgs a;
  a.st[0] = {xin0, xout0, cd0, cr0};
  a.st[1] = {xin1, xout1, cd1, cr1};
  a.st[2] = {xin2, xout2, cd2, cr2};
  static int per_sm[4] = {0, 0, 0, 0};
  if (!per_sm[nsteps]) {
    if (nsteps == 2)
      SPHC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[2], k_sell_cheb_fused<2>,
                                                              FZ_ROWS, 0));
    else
      SPHC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[3], k_sell_cheb_fused<3>,
                                                              FZ_ROWS, 0));
  }
  // persistent CTAs, all resident (a CTA may wait on slots claimed earlier)
  int g = per_sm[nsteps] * SPHC_NUM_SMS;
  static int cap = -1;
  if (cap < 0) {
    const char* e = getenv("SPHC_FUSE_CTAS");
    cap = e ? atoi(e) : 0;
  }
  if (cap > 0 && g > cap) g = cap;
  int nslots = nblk + (nsteps - 1) * (L + 1);
  if (g > nslots) g = nslots;
  if (nsteps == 2)
    k_sell_cheb_fused<2><<<g, FZ_ROWS, 0, s>>>(n, slice_ptr, sci, sv, dinv, b, d, a, x_zero, L,
                                               nblk, sync, sync + 1);
  else
    k_sell_cheb_fused<3><<<g, FZ_ROWS, 0, s>>>(n, slice_ptr, sci, sv, dinv, b, d, a, x_zero, L,
                                               nblk, sync, sync + 1);
  SPHC_LAUNCH_CHECK();
  return 0;
}
