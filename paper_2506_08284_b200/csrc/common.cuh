// Shared device helpers for libsphcurl (sm_100a, fp64, HBM-bound sparse work).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/sphcurl.h"

typedef int64_t i64;

#define SPHC_WARP 32
#define FULL_MASK 0xffffffffu

// Number of resident CTAs we size persistent / grid-stride grids for: 148 SMs
// (2 dies x 74) times a small multiple.
#define SPHC_NUM_SMS 148

// thread-local last error message (sphc_last_error)
void sphc_set_error(const char* fmt, ...);

#define SPHC_CUDA(call)                                                      \
  do {                                                                       \
    cudaError_t _e = (call);                                                 \
    if (_e != cudaSuccess) {                                                 \
      sphc_set_error("%s:%d %s: %s", __FILE__, __LINE__, #call,              \
                     cudaGetErrorString(_e));                                \
      return SPHC_ERR_CUDA;                                                  \
    }                                                                        \
  } while (0)

extern unsigned long long g_sphc_launches;

#define SPHC_LAUNCH_CHECK()                                                  \
  do {                                                                       \
    g_sphc_launches++;                                                       \
    cudaError_t _e = cudaGetLastError();                                     \
    if (_e != cudaSuccess) {                                                 \
      sphc_set_error("%s:%d launch: %s", __FILE__, __LINE__,                 \
                     cudaGetErrorString(_e));                                \
      return SPHC_ERR_CUDA;                                                  \
    }                                                                        \
  } while (0)

static inline cudaStream_t as_stream(void* s) { return (cudaStream_t)s; }

// Programmatic dependent launch (PDL) for the solve's chains of short
// dependent kernels (V-cycle, PCG vector ops, reductions): the next grid is
// launched as the previous one's CTAs exit (the implicit trigger) instead of
// after its completion is signalled, hiding most of the launch gap. Every
// kernel launched through launch_pdl starts with pdl_begin():
// griddepcontrol.wait returns once all prerequisite grids have completed and
// their writes are visible, so the kernel body sees exactly what a plain
// stream-ordered launch would (and, each kernel waiting on its predecessor,
// the ordering is transitive). Without the launch attribute it is a no-op.
// An explicit early griddepcontrol.launch_dependents was measured slower
// (C2 solve 5.2 -> 5.6 ms: waiting CTAs of the next grid skew its placement);
// wait-only gives 5.2 -> 4.9 ms. SPHC_PDL=0 disables the attribute.
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

static inline bool sphc_pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SPHC_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

template <typename... KArgs, typename... Args>
static inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = sphc_pdl_enabled() ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

static inline unsigned grid_for(i64 work, int block, int max_blocks = 148 * 16) {
  i64 g = (work + block - 1) / block;
  if (g < 1) g = 1;
  if (g > max_blocks) g = max_blocks;
  return (unsigned)g;
}

// record the first (lowest) failing row for an error code
__device__ __forceinline__ void report(i64* status, int code, i64 row) {
  if (status) atomicMin((unsigned long long*)&status[code], (unsigned long long)row);
}

// exact IEEE helpers (no contraction): used wherever the reference's scipy /
// numpy accumulation order defines discrete outcomes
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL_MASK, v, o));
  return v;
}
__device__ __forceinline__ i64 warp_sum_i64(i64 v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}

// atomic max for non-negative doubles through their ordered bit pattern
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax((unsigned long long*)addr, (unsigned long long)__double_as_longlong(v));
}

// stream-ordered scratch from the device's default pool; the pool keeps its
// memory across synchronisations (release threshold = max) so repeated
// setup passes do not re-map pages
int sphc_pool_init();
template <typename T>
static inline int scratch(T** p, size_t n, cudaStream_t s) {
  if (sphc_pool_init()) return SPHC_ERR_CUDA;
  SPHC_CUDA(cudaMallocAsync((void**)p, (n ? n : 1) * sizeof(T), s));
  return 0;
}
static inline int scratch_free(void* p, cudaStream_t s) {
  SPHC_CUDA(cudaFreeAsync(p, s));
  return 0;
}

// lower_bound in a sorted int array (shared or global)
__device__ __forceinline__ int lower_bound_i32(const int* a, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ i64 lower_bound_i32_g(const int* a, i64 lo, i64 hi, int key) {
  while (lo < hi) {
    i64 mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// single-launch reductions (util.cu): grid of a length-n reduction, the
// shared partials / ticket, and the in-kernel combine of the last block
#define RED_THREADS 256
#define RED_MAX_BLOCKS (SPHC_NUM_SMS * 8)
static inline int sphc_reduce_grid(i64 n) { return (int)grid_for(n, RED_THREADS, RED_MAX_BLOCKS); }
int sphc_reduce_scratch(double** part, unsigned** ticket);

__device__ __forceinline__ double block_sum(double v, double* sh) {
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  v = warp_sum(v);
  if (lane == 0) sh[wid] = v;
  __syncthreads();
  double t = 0.0;
  if (wid == 0) {
    t = (lane < (int)(blockDim.x >> 5)) ? sh[lane] : 0.0;
    t = warp_sum(t);
  }
  __syncthreads();
  return t;
}

// block partial t -> part[blockIdx.x]; the last block to arrive returns true
// with the fixed-order sum of all partials in *total (thread 0) and re-arms
// the ticket. Every thread of the block must call it.
__device__ __forceinline__ bool last_block_sum(double t, double* part, unsigned* ticket,
                                               double* sh, double* total) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = t;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double acc = 0.0;
  for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) acc += __ldcg(part + i);
  acc = block_sum(acc, sh);
  if (threadIdx.x == 0) {
    *total = acc;
    *ticket = 0u;
  }
  return true;
}

// internal host-side helpers shared across translation units
int sphc_scan_impl(i64 n, const i64* in, i64* out, cudaStream_t s);
