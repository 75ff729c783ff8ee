// Gauss-Seidel half sweeps for the reference's exact smoother
// (multigrid.py:32-66: x += tril(A)^-1 (b - A x), then x += triu(A)^-1 (b - A x)).
//
// Sync-free triangular substitution, one warp per row: rows are claimed from
// an atomic ticket in dependency order (ascending for tril, descending for
// triu), so every row a warp waits on is already owned by a running warp and
// the kernel cannot deadlock. The solution vector itself is the ready flag:
// y is reset to a NaN sentinel and a lane spins on y[j] until it changes (a
// single aligned 64-bit location, so no separate flag / fence pairing). The
// residual part (b - A x_in)_i has no dependencies and is summed before the
// wait. The dependency depth of the natural edge ordering is ~16 N levels on
// an N^3 hex mesh, so the sweep is latency-bound (~1 us per level).
#include "common.cuh"

#define GS_WARPS 4
#define GS_SENT 0xFFFFFFFFFFFFFFFFull  // NaN pattern never produced by arithmetic
#define GS_SPIN_LIMIT (1ll << 26)

__device__ __forceinline__ double ld_relaxed(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return __longlong_as_double((long long)v);
}
__device__ __forceinline__ void st_relaxed(double* p, double x) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(x))
               : "memory");
}

template <bool LOWER, bool XZERO>
__global__ void __launch_bounds__(GS_WARPS * 32)
    k_gs_half(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
              const double* __restrict__ v, const double* __restrict__ b,
              const double* __restrict__ x_in, double* __restrict__ x_out, double* y,
              int* ticket, i64* status) {
  int lane = threadIdx.x & 31;
  while (true) {
    int t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1);
    t = __shfl_sync(FULL_MASK, t, 0);
    if (t >= n) return;
    i64 i = LOWER ? (i64)t : n - 1 - (i64)t;
    i64 s = rp[i], e = rp[i + 1];
    double ax = 0.0, ty = 0.0, dg = 0.0;
    bool stall = false;
    for (i64 k = s + lane; k < e; k += 32) {
      int j = ci[k];
      double a = v[k];
      if (!XZERO) ax += a * x_in[j];
      if (j == i) dg = a;
      bool dep = LOWER ? (j < i) : (j > i);
      if (dep) {
        double yj;
        i64 spins = 0;
        do {
          yj = ld_relaxed(y + j);
        } while (__double_as_longlong(yj) == (long long)GS_SENT && ++spins < GS_SPIN_LIMIT);
        if (spins >= GS_SPIN_LIMIT) stall = true;
        ty += a * yj;
      }
    }
    ax = warp_sum(ax);
    ty = warp_sum(ty);
    dg = warp_sum(dg);
    unsigned st = __ballot_sync(FULL_MASK, stall);
    if (lane == 0) {
      if (st) report(status, SPHC_ST_TRSV_STALL, i);
      if (dg == 0.0) report(status, SPHC_ST_ZERO_DIAG, i);
      double r = b[i] - ax;
      double yi = (r - ty) / dg;
      if ((unsigned long long)__double_as_longlong(yi) == GS_SENT)
        yi = __longlong_as_double(0x7FF8000000000000ll);
      x_out[i] = XZERO ? yi : x_in[i] + yi;
      st_relaxed(y + i, yi);
    }
  }
}

extern "C" int sphc_gs_half_sweep(int64_t n, const int64_t* rp, const int32_t* ci,
                                  const double* v, const double* b, const double* x_in,
                                  double* x_out, double* y, int32_t* ticket, int lower,
                                  int64_t* status, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) return 0;
  SPHC_CUDA(cudaMemsetAsync(y, 0xFF, (size_t)n * sizeof(double), s));
  SPHC_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int32_t), s));
  unsigned grid = grid_for(n, GS_WARPS, SPHC_NUM_SMS * 16);
  dim3 blk(GS_WARPS * 32);
  bool xz = x_in == nullptr;
  if (lower) {
    if (xz) k_gs_half<true, true><<<grid, blk, 0, s>>>(n, rp, ci, v, b, x_in, x_out, y, ticket, status);
    else k_gs_half<true, false><<<grid, blk, 0, s>>>(n, rp, ci, v, b, x_in, x_out, y, ticket, status);
  } else {
    if (xz) k_gs_half<false, true><<<grid, blk, 0, s>>>(n, rp, ci, v, b, x_in, x_out, y, ticket, status);
    else k_gs_half<false, false><<<grid, blk, 0, s>>>(n, rp, ci, v, b, x_in, x_out, y, ticket, status);
  }
  SPHC_LAUNCH_CHECK();
  return 0;
}
