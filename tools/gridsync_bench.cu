// Grid barrier cost on B200 (diagnostic): cooperative_groups grid.sync()
// against a sense-reversing barrier (one atomicAdd per CTA, acquire spin).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, double* sink) {
  cg::grid_group g = cg::this_grid();
  double a = 0;
  for (int i = 0; i < iters; i++) { a += i; g.sync(); }
  if (threadIdx.x == 0 && a < 0) sink[blockIdx.x] = a;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void bar(unsigned* count, unsigned* gen, unsigned& my_gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned target = my_gen + 1;
    __threadfence();
    unsigned arrived = atomicAdd(count, 1u);
    if (arrived == gridDim.x - 1) {
      *count = 0;
      __threadfence();
      atomicExch(gen, target);
    } else {
      while (ld_acquire(gen) != target) { }
    }
    my_gen = target;
  }
  __syncthreads();
}

__global__ void k_custom(int iters, unsigned* count, unsigned* gen, double* sink) {
  __shared__ unsigned sg;
  if (threadIdx.x == 0) sg = ld_acquire(gen);
  __syncthreads();
  unsigned my_gen = sg;
  double a = 0;
  for (int i = 0; i < iters; i++) { a += i; bar(count, gen, my_gen); }
  if (threadIdx.x == 0 && a < 0) sink[blockIdx.x] = a;
}

int main() {
  double* sink; unsigned *cnt, *gen;
  cudaMalloc(&sink, 1 << 20); cudaMalloc(&cnt, 4); cudaMalloc(&gen, 4);
  cudaMemset(cnt, 0, 4); cudaMemset(gen, 0, 4);
  int iters = 2000;
  for (int blocks : {84, 148, 296, 361, 592, 1184}) {
    for (int v = 0; v < 2; v++) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      void* args0[] = {&iters, &sink};
      void* args1[] = {&iters, &cnt, &gen, &sink};
      for (int rep = 0; rep < 2; rep++) {
        cudaEventRecord(a);
        cudaError_t e = v == 0 ? cudaLaunchCooperativeKernel((void*)k_cg, blocks, 256, args0)
                               : cudaLaunchCooperativeKernel((void*)k_custom, blocks, 256, args1);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); break; }
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep) printf("blocks %4d %-10s %.3f us per barrier\n", blocks, v ? "custom" : "cg::grid", ms * 1e3 / iters);
      }
    }
  }
  return 0;
}
