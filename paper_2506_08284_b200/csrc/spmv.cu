// Solve-phase kernels: row-grouped CSR SpMV (L lanes per row, shuffle
// segmented reduction), the fused Chebyshev step, fused PCG vector updates
// and the coarsest-level dense GEMV. All fp64 and HBM-bound.
#include "common.cuh"

#define SPMV_THREADS 256

template <int L>
__device__ __forceinline__ double row_dot(i64 row, i64 n, const i64* __restrict__ rp,
                                          const int* __restrict__ ci,
                                          const double* __restrict__ v,
                                          const double* __restrict__ x, int lane) {
  double acc = 0.0;
  if (row < n) {
    i64 e = rp[row + 1];
    for (i64 j = rp[row] + lane; j < e; j += L) acc = fma(v[j], __ldg(x + ci[j]), acc);
  }
#pragma unroll
  for (int o = L / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL_MASK, acc, o);
  return acc;
}

// y = alpha * A x + beta * z
template <int L>
__global__ void __launch_bounds__(SPMV_THREADS)
    k_spmv(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
           const double* __restrict__ v, const double* __restrict__ x, double alpha,
           double beta, const double* z, double* y) {
  pdl_begin();
  const int RPW = 32 / L;
  int lane = threadIdx.x & (L - 1);
  int sub = (threadIdx.x & 31) / L;
  i64 warp = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 base = warp * RPW; base < n; base += nw * RPW) {
    i64 row = base + sub;
    double acc = row_dot<L>(row, n, rp, ci, v, x, lane);
    if (row < n && lane == 0) {
      double r = alpha * acc;
      if (z) r = fma(beta, z[row], r);
      y[row] = r;
    }
  }
}

// d <- cd d + cr dinv (b - A x_in); x_out = x_in + d
template <int L>
__global__ void __launch_bounds__(SPMV_THREADS)
    k_cheb(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
           const double* __restrict__ v, const double* __restrict__ dinv,
           const double* __restrict__ b, const double* __restrict__ x_in,
           double* __restrict__ x_out, double* __restrict__ d, double cd, double cr,
           int x_zero) {
  pdl_begin();
  const int RPW = 32 / L;
  int lane = threadIdx.x & (L - 1);
  int sub = (threadIdx.x & 31) / L;
  i64 warp = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 base = warp * RPW; base < n; base += nw * RPW) {
    i64 row = base + sub;
    double ax = x_zero ? 0.0 : row_dot<L>(row, n, rp, ci, v, x_in, lane);
    if (row < n && lane == 0) {
      double r = b[row] - ax;
      double dn = cr * dinv[row] * r;
      if (cd != 0.0) dn = fma(cd, d[row], dn);
      d[row] = dn;
      x_out[row] = (x_zero ? 0.0 : x_in[row]) + dn;
    }
  }
}

static unsigned spmv_grid(i64 n, int L) {
  i64 rows_per_block = (SPMV_THREADS / 32) * (32 / L);
  return grid_for(n, (int)rows_per_block, SPHC_NUM_SMS * 16);
}

#define DISPATCH_L(L, CALL)                \
  switch (L) {                             \
    case 1: { const int LL = 1; CALL; } break;  \
    case 2: { const int LL = 2; CALL; } break;  \
    case 4: { const int LL = 4; CALL; } break;  \
    case 8: { const int LL = 8; CALL; } break;  \
    case 16: { const int LL = 16; CALL; } break; \
    case 32: { const int LL = 32; CALL; } break; \
    default: sphc_set_error("lanes must be 1,2,4,8,16,32"); return SPHC_ERR_ARG; \
  }

// y = alpha A x + beta z with one CTA per row (rows of hundreds of entries,
// too few rows to fill the SMs warp per row): strided fma per thread, then
// the fixed-order block tree (deterministic)
__global__ void __launch_bounds__(256)
    k_spmv_cta(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
               const double* __restrict__ v, const double* __restrict__ x, double alpha,
               double beta, const double* z, double* y) {
  pdl_begin();
  __shared__ double sh[32];
  for (i64 row = blockIdx.x; row < n; row += gridDim.x) {
    double acc = 0.0;
    for (i64 j = rp[row] + threadIdx.x; j < rp[row + 1]; j += blockDim.x)
      acc = fma(v[j], x[ci[j]], acc);
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) {
      double r = alpha * acc;
      if (z) r = fma(beta, z[row], r);
      y[row] = r;
    }
  }
}

extern "C" int sphc_spmv(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                         int lanes, const double* x, double alpha, double beta,
                         const double* z, double* y, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  if (lanes == 256) {
    launch_pdl(k_spmv_cta, grid_for(n, 1, SPHC_NUM_SMS * 8), 256, 0, s, n, rp, ci, v, x, alpha,
               beta, z, y);
    SPHC_LAUNCH_CHECK();
    return 0;
  }
  DISPATCH_L(lanes, (launch_pdl(k_spmv<LL>, spmv_grid(n, LL), SPMV_THREADS, 0, s,
                                    n, rp, ci, v, x, alpha, beta, z, y)));
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_cheb_step(int64_t n, const int64_t* rp, const int32_t* ci, const double* v,
                              int lanes, const double* dinv, const double* b,
                              const double* x_in, double* x_out, double* d, double cd,
                              double cr, int x_zero, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  DISPATCH_L(lanes, (launch_pdl(k_cheb<LL>, spmv_grid(n, LL), SPMV_THREADS, 0, s,
                                    n, rp, ci, v, dinv, b, x_in, x_out, d, cd, cr, x_zero)));
  SPHC_LAUNCH_CHECK();
  return 0;
}

// PCG scalars live on the device (slots SPHC_PCG_*), so a whole iteration
// can be replayed as one CUDA graph with a single small readback.
__global__ void k_pcg_update(i64 n, const double* __restrict__ sc, const double* __restrict__ p,
                             const double* __restrict__ Ap, double* __restrict__ x,
                             double* __restrict__ r, int* changed) {
  pdl_begin();
  double pAp = sc[SPHC_PCG_PAP];
  if (!(pAp > 0.0)) return;  // "indefinite": the reference stops before updating
  double alpha = sc[SPHC_PCG_RZ] / pAp;
  int ch = 0;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    double xo = x[i];
    double xn = xo + alpha * p[i];
    ch |= (xn != xo);
    x[i] = xn;
    r[i] = r[i] - alpha * Ap[i];
  }
  ch = __syncthreads_or(ch);
  if (ch && threadIdx.x == 0) atomicOr(changed, 1);
}

extern "C" int sphc_pcg_update(int64_t n, const double* sc, const double* p, const double* Ap,
                               double* x, double* r, int32_t* changed, void* stream) {
  cudaStream_t s = as_stream(stream);
  launch_pdl(k_pcg_update, grid_for(n, 256), 256, 0, s, n, sc, p, Ap, x, r, changed);
  SPHC_LAUNCH_CHECK();
  return 0;
}

__global__ void k_pcg_dir(i64 n, const double* __restrict__ sc, const double* __restrict__ z,
                          double* __restrict__ p) {
  pdl_begin();
  double beta = sc[SPHC_PCG_RZN] / sc[SPHC_PCG_RZ];
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}

// sphc_pcg_update plus r.r of the new residual (the grid and summation
// order of sphc_dot(n, r, r), so bitwise the same value) in one launch
__global__ void k_pcg_update_rr(i64 n, double* __restrict__ sc, const double* __restrict__ p,
                                const double* __restrict__ Ap, double* __restrict__ x,
                                double* __restrict__ r, int* changed, double* part,
                                unsigned* ticket) {
  pdl_begin();
  __shared__ double sh[32];
  double pAp = sc[SPHC_PCG_PAP];
  if (!(pAp > 0.0)) return;
  double alpha = sc[SPHC_PCG_RZ] / pAp;
  int ch = 0;
  double acc = 0.0;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    double xo = x[i];
    double xn = xo + alpha * p[i];
    ch |= (xn != xo);
    x[i] = xn;
    double rn = r[i] - alpha * Ap[i];
    r[i] = rn;
    acc = fma(rn, rn, acc);
  }
  ch = __syncthreads_or(ch);
  if (ch && threadIdx.x == 0) atomicOr(changed, 1);
  double t = block_sum(acc, sh);
  double total;
  if (last_block_sum(t, part, ticket, sh, &total) && threadIdx.x == 0)
    sc[SPHC_PCG_RR] = total;
}

extern "C" int sphc_pcg_update_rr(int64_t n, double* sc, const double* p, const double* Ap,
                                  double* x, double* r, int32_t* changed, void* stream) {
  cudaStream_t s = as_stream(stream);
  double* part;
  unsigned* ticket;
  if (sphc_reduce_scratch(&part, &ticket)) return SPHC_ERR_CUDA;
  launch_pdl(k_pcg_update_rr, sphc_reduce_grid(n), RED_THREADS, 0, s, n, sc, p, Ap, x, r,
             changed, part, ticket);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_pcg_direction(int64_t n, const double* sc, const double* z, double* p,
                                  void* stream) {
  cudaStream_t s = as_stream(stream);
  launch_pdl(k_pcg_dir, grid_for(n, 256), 256, 0, s, n, sc, z, p);
  SPHC_LAUNCH_CHECK();
  return 0;
}

__global__ void k_pcg_rotate(double* sc) {
  pdl_begin();
  sc[SPHC_PCG_RZ] = sc[SPHC_PCG_RZN];
}

extern "C" int sphc_pcg_rotate(double* sc, void* stream) {
  cudaStream_t s = as_stream(stream);
  launch_pdl(k_pcg_rotate, 1, 1, 0, s, sc);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// A captured graph and the number of libsphcurl kernels in it (a replay
// counts them all in sphc_launch_count).
struct SphcGraph {
  cudaGraphExec_t exec;
  unsigned long long kernels;
};
static thread_local unsigned long long g_capture_start = 0;

extern "C" int sphc_graph_begin(void* stream) {
  SPHC_CUDA(cudaStreamBeginCapture(as_stream(stream), cudaStreamCaptureModeThreadLocal));
  g_capture_start = g_sphc_launches;
  return 0;
}

extern "C" int sphc_graph_end(void** exec, void* stream) {
  cudaGraph_t g = nullptr;
  unsigned long long k = g_sphc_launches - g_capture_start;
  g_sphc_launches = g_capture_start;  // captured, not launched
  SPHC_CUDA(cudaStreamEndCapture(as_stream(stream), &g));
  cudaGraphExec_t e = nullptr;
  cudaError_t err = cudaGraphInstantiate(&e, g, 0);
  cudaGraphDestroy(g);
  if (err != cudaSuccess) {
    sphc_set_error("cudaGraphInstantiate: %s", cudaGetErrorString(err));
    return SPHC_ERR_CUDA;
  }
  exec[0] = (void*)new SphcGraph{e, k};
  return 0;
}

extern "C" int sphc_graph_launch(void* exec, void* stream) {
  SphcGraph* G = (SphcGraph*)exec;
  SPHC_CUDA(cudaGraphLaunch(G->exec, as_stream(stream)));
  g_sphc_launches += G->kernels;
  return 0;
}

extern "C" int sphc_graph_destroy(void* exec) {
  SphcGraph* G = (SphcGraph*)exec;
  if (!G) return 0;
  cudaError_t err = cudaGraphExecDestroy(G->exec);
  delete G;
  if (err != cudaSuccess) {
    sphc_set_error("cudaGraphExecDestroy: %s", cudaGetErrorString(err));
    return SPHC_ERR_CUDA;
  }
  return 0;
}

// ---------------------------------------------------------------------------
// The whole PCG loop as ONE graph launch: a WHILE conditional node whose body
// is one captured iteration followed by k_pcg_check, which records the
// iteration's residual / preconditioned norms on the device, evaluates the
// reference's tests (multigrid.py:244-266) and sets the loop condition. No
// host round trip per iteration.
//   ctl[0] = rtol * |b| (set before each launch), ctl[1] = maxit,
//   ctl[2] = iterations done, ctl[3] = status (0 running, 1 converged,
//   2 maxit, 3 stagnated, 4 indefinite); hist[2 it] = |r|, hist[2 it + 1] =
//   sqrt(max(r.z, 0)) for it = 1..iterations.
struct SphcLoop {
  cudaGraph_t graph;
  cudaGraphExec_t exec;
  cudaGraphConditionalHandle handle;
  cudaGraph_t body;
  unsigned long long start, kernels;
};

__global__ void k_pcg_check(double* sc, double* ctl, double* hist,
                            cudaGraphConditionalHandle handle) {
  double pAp = sc[SPHC_PCG_PAP];
  sc[SPHC_PCG_RZ] = sc[SPHC_PCG_RZN];   // the rotate of sphc_pcg_rotate, folded in
  int st = 0;
  int32_t* flag = reinterpret_cast<int32_t*>(sc + 4);
  if (pAp <= 0.0) {
    st = 4;
  } else {
    double it = ctl[2] + 1.0;
    ctl[2] = it;
    if (*flag == 0) {
      st = 3;
    } else {
      double res = sqrt(sc[SPHC_PCG_RR]);
      long i = (long)it;
      hist[2 * i] = res;
      hist[2 * i + 1] = sqrt(fmax(sc[SPHC_PCG_RZN], 0.0));
      if (res <= ctl[0]) st = 1;
      else if (it >= ctl[1]) st = 2;
    }
  }
  ctl[3] = (double)st;
  sc[4] = 0.0;   // the next iteration's change flag
  cudaGraphSetConditional(handle, st == 0 ? 1u : 0u);
}

extern "C" int sphc_pcg_loop_begin(void** state, void* stream) {
  SphcLoop* L = new SphcLoop();
  cudaError_t e = cudaGraphCreate(&L->graph, 0);
  if (e == cudaSuccess)
    e = cudaGraphConditionalHandleCreate(&L->handle, L->graph, 1, cudaGraphCondAssignDefault);
  cudaGraphNode_t node;
  cudaGraphNodeParams prm = {};
  if (e == cudaSuccess) {
    prm.type = cudaGraphNodeTypeConditional;
    prm.conditional.handle = L->handle;
    prm.conditional.type = cudaGraphCondTypeWhile;
    prm.conditional.size = 1;
    e = cudaGraphAddNode(&node, L->graph, nullptr, 0, &prm);
  }
  if (e == cudaSuccess) {
    L->body = prm.conditional.phGraph_out[0];
    e = cudaStreamBeginCaptureToGraph(as_stream(stream), L->body, nullptr, nullptr, 0,
                                      cudaStreamCaptureModeThreadLocal);
  }
  if (e != cudaSuccess) {
    if (L->graph) cudaGraphDestroy(L->graph);
    delete L;
    sphc_set_error("sphc_pcg_loop_begin: %s", cudaGetErrorString(e));
    return SPHC_ERR_CUDA;
  }
  L->start = g_sphc_launches;
  state[0] = L;
  return 0;
}

extern "C" int sphc_pcg_check(void* state, double* sc, double* ctl, double* hist, void* stream) {
  SphcLoop* L = (SphcLoop*)state;
  k_pcg_check<<<1, 1, 0, as_stream(stream)>>>(sc, ctl, hist, L->handle);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_pcg_loop_end(void* state, void* stream) {
  SphcLoop* L = (SphcLoop*)state;
  L->kernels = g_sphc_launches - L->start;   // per iteration
  g_sphc_launches = L->start;
  cudaGraph_t g = nullptr;
  SPHC_CUDA(cudaStreamEndCapture(as_stream(stream), &g));
  cudaError_t e = cudaGraphInstantiate(&L->exec, L->graph, 0);
  if (e != cudaSuccess) {
    sphc_set_error("cudaGraphInstantiate (PCG loop): %s", cudaGetErrorString(e));
    return SPHC_ERR_CUDA;
  }
  return 0;
}

// runs the loop; *kernels_per_iteration lets the caller count launches
extern "C" int sphc_pcg_loop_launch(void* state, int64_t* kernels_per_iteration, void* stream) {
  SphcLoop* L = (SphcLoop*)state;
  SPHC_CUDA(cudaGraphLaunch(L->exec, as_stream(stream)));
  if (kernels_per_iteration) *kernels_per_iteration = (int64_t)L->kernels;
  return 0;
}

extern "C" int sphc_pcg_loop_add_launches(int64_t n) {
  g_sphc_launches += (unsigned long long)n;
  return 0;
}

extern "C" int sphc_pcg_loop_destroy(void* state) {
  SphcLoop* L = (SphcLoop*)state;
  if (!L) return 0;
  if (L->exec) cudaGraphExecDestroy(L->exec);
  if (L->graph) cudaGraphDestroy(L->graph);
  delete L;
  return 0;
}

extern "C" int sphc_copy_d2h(void* dst, const void* src, int64_t bytes, void* stream) {
  SPHC_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, as_stream(stream)));
  return 0;
}

#define RB_MAX 16
struct RbParts {
  const uint32_t* src[RB_MAX];
  int64_t words[RB_MAX];
  int64_t off[RB_MAX];
  int count;
};

// one CTA per range: 4-byte words from device memory to mapped host memory
__global__ void k_readback_gather(RbParts P, uint32_t* dst) {
  pdl_begin();
  int r = blockIdx.x;
  if (r >= P.count) return;
  const uint32_t* s = P.src[r];
  uint32_t* d = dst + P.off[r] / 4;
  for (int64_t i = threadIdx.x; i < P.words[r]; i += blockDim.x) d[i] = s[i];
}

extern "C" int sphc_readback_gather(int32_t count, const int64_t* desc, void* dst,
                                    void* stream) {
  if (count <= 0) return 0;
  if (count > RB_MAX) {
    sphc_set_error("sphc_readback_gather: %d ranges (max %d)", count, RB_MAX);
    return SPHC_ERR_ARG;
  }
  RbParts P = {};
  P.count = count;
  for (int i = 0; i < count; i++) {
    const int64_t* r = desc + 3 * i;
    if ((r[1] | r[2]) & 3) {
      sphc_set_error("sphc_readback_gather: range %d not 4-byte aligned", i);
      return SPHC_ERR_ARG;
    }
    P.src[i] = (const uint32_t*)r[0];
    P.words[i] = r[1] / 4;
    P.off[i] = r[2];
  }
  // the staging buffer's device alias (the same address under unified
  // addressing for mapped page-locked memory); a buffer that is not mapped
  // falls back to one copy-engine transfer per range
  static void* last_host = nullptr;
  static void* last_dev = nullptr;
  if (dst != last_host) {
    void* dp = nullptr;
    if (cudaHostGetDevicePointer(&dp, dst, 0) != cudaSuccess) {
      (void)cudaGetLastError();
      for (int i = 0; i < count; i++)
        SPHC_CUDA(cudaMemcpyAsync((char*)dst + P.off[i], P.src[i], (size_t)P.words[i] * 4,
                                  cudaMemcpyDeviceToHost, as_stream(stream)));
      return 0;
    }
    last_host = dst;
    last_dev = dp;
  }
  launch_pdl(k_readback_gather, count, 256, 0, as_stream(stream), P, (uint32_t*)last_dev);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_stream_sync(void* stream) {
  SPHC_CUDA(cudaStreamSynchronize(as_stream(stream)));
  return 0;
}

// y = A x, A dense row-major n x n: one warp per row, fixed-order reduction
__global__ void k_dense_gemv(i64 n, const double* __restrict__ A, const double* __restrict__ x,
                             double* __restrict__ y) {
  pdl_begin();
  int lane = threadIdx.x & 31;
  i64 w = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 row = w; row < n; row += nw) {
    const double* a = A + row * n;
    double acc = 0.0;
    for (i64 j = lane; j < n; j += 32) acc = fma(a[j], x[j], acc);
    acc = warp_sum(acc);
    if (lane == 0) y[row] = acc;
  }
}

extern "C" int sphc_dense_gemv(int64_t n, const double* A, const double* x, double* y,
                               void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  launch_pdl(k_dense_gemv, grid_for(n * 32, 256), 256, 0, s, n, A, x, y);
  SPHC_LAUNCH_CHECK();
  return 0;
}

__global__ void k_gather(i64 n, const i64* __restrict__ idx, const double* __restrict__ x,
                         double* __restrict__ out) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x)
    out[i] = x[idx[i]];
}

extern "C" int sphc_gather(int64_t n, const int64_t* idx, const double* x, double* out,
                           void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  k_gather<<<grid_for(n, 256), 256, 0, s>>>(n, idx, x, out);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// y_i = d_i x_i
__global__ void k_diag_scale(i64 n, const double* __restrict__ d, const double* __restrict__ x,
                             double* __restrict__ y) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x)
    y[i] = d[i] * x[i];
}

extern "C" int sphc_diag_scale(int64_t n, const double* d, const double* x, double* y,
                               void* stream) {
  cudaStream_t s = as_stream(stream);
  k_diag_scale<<<grid_for(n, 256), 256, 0, s>>>(n, d, x, y);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// One Lanczos step for D^-1 A in the D inner product (the Chebyshev bound
// estimate): w = D^-1 u - alpha v - beta_prev v_prev with u = A v, and
// dw = D w for the next norm. alpha / beta_prev are device scalars.
__global__ void k_lanczos_update(i64 n, const double* __restrict__ u, const double* __restrict__ dinv,
                                 const double* __restrict__ d, const double* __restrict__ v,
                                 const double* __restrict__ vprev, const double* alpha,
                                 const double* beta_prev, double* __restrict__ w,
                                 double* __restrict__ dw) {
  double a = *alpha, b = beta_prev ? *beta_prev : 0.0;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    double t = dinv[i] * u[i] - a * v[i];
    if (beta_prev) t -= b * vprev[i];
    w[i] = t;
    dw[i] = d[i] * t;
  }
}

extern "C" int sphc_lanczos_update(int64_t n, const double* u, const double* dinv, const double* d,
                                   const double* v, const double* vprev, const double* alpha,
                                   const double* beta_prev, double* w, double* dw, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  k_lanczos_update<<<grid_for(n, 256), 256, 0, s>>>(n, u, dinv, d, v, vprev, alpha, beta_prev, w,
                                                    dw);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// deterministic start vector in [-1, 1): splitmix64 of the index (same
// integer arithmetic as oracle.cheb_start_vector)
__global__ void k_cheb_start(i64 n, double* __restrict__ x) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x) {
    unsigned long long z = (unsigned long long)i + 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    x[i] = (double)(z >> 11) * 0x1p-53 * 2.0 - 1.0;
  }
}

extern "C" int sphc_cheb_start(int64_t n, double* x, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_cheb_start<<<grid_for(n, 256), 256, 0, s>>>(n, x);
  SPHC_LAUNCH_CHECK();
  return 0;
}
