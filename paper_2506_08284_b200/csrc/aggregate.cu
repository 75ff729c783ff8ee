// Greedy root aggregation (reference nodal_amg.py:59-88) on the device,
// bit-identical to the sequential loops.
//
// Phase 1 (index order: i roots an aggregate iff none of N[i] is aggregated
// yet) is the lexicographically-first maximal independent set of G^2: i is a
// root iff no root r < i lies within distance 2. It runs sync-free: warps take
// nodes in ascending order from an atomic ticket; node i scans N[j] for every
// j in N[i] and waits only on the lower nodes it finds there (their state is
// final before i's in the sequential order too), stopping at the first root.
// Aggregate ids follow root order (exclusive scan of the root flags), and
// every phase-1 member has exactly one root in its neighbourhood (roots are
// >= 3 apart), so membership is a parallel scatter from the roots.
//
// Phase 2 (leftovers in index order join the aggregate most frequent among
// their assigned neighbours, lowest id on ties, 0 if none) is sync-free too:
// a leftover waits for its lower leftover neighbours (a higher one waits for
// it in turn, so it still reads -1 there, as the sequential loop does).
#include "common.cuh"

extern "C" int sphc_scan_i64(int64_t n, const int64_t* counts, int64_t* offsets, void* stream);

#define AGG_WARPS 4
#define AGG_CAP 256  // neighbour owners buffered per leftover node (beyond: global reads)

__device__ __forceinline__ int agg_ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void agg_st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ i64 agg_ld_acquire64(const i64* p) {
  i64 v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void agg_st_release64(i64* p, i64 v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// state: 0 undecided, 1 root, 2 not a root.
// Node i gathers the lower nodes of its distance-2 neighbourhood into shared
// memory once, then rescans their states until it can decide: a root among
// them decides "not a root" at once (whatever is still pending), all of them
// decided without a root decides "root". Deciding as early as the data
// allows keeps the dependency depth at the wavefront depth (~2N on an N^3
// mesh) instead of a chain through every lower node.
#define AGG_LCAP 256   // distinct lower distance-2 nodes held per warp
#define AGG_HCAP 512   // open-addressing slots of the de-duplication set
__global__ void __launch_bounds__(AGG_WARPS * 32)
    k_agg_roots(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci, int* state,
                int* ticket) {
  __shared__ int lst[AGG_WARPS][AGG_LCAP];
  __shared__ int hset[AGG_WARPS][AGG_HCAP];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  volatile int* vs = state;
  while (true) {
    int t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1);
    t = __shfl_sync(FULL_MASK, t, 0);
    if (t >= n) return;
    i64 i = t;
    // distinct lower distance-2 nodes; lanes over j in N[i]. A 27-point
    // stencil lists each distance-2 node up to 8 times: a shared-memory
    // hash set keeps first occurrences only (the wait below is order
    // independent; a sort + unique pass here cost ~4x the rest of the kernel)
    int* L = lst[w];
    int* H = hset[w];
    for (int a = lane; a < AGG_HCAP; a += 32) H[a] = -1;
    __syncwarp();
    int cnt = 0;
    bool over = false;
    i64 js = rp[i], je = rp[i + 1];
    for (i64 b = js; b < je; b += 32) {
      i64 jj = b + lane;
      int j = jj < je ? ci[jj] : 0;
      i64 k0 = jj < je ? rp[j] : 0, k1 = jj < je ? rp[j + 1] : 0;
      // walk all the lanes' N[j] lists in lockstep
      int len = (int)(k1 - k0);
      int mx = len;
      for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL_MASK, mx, o));
      for (int u = 0; u < mx; u++) {
        int k = u < len ? ci[k0 + u] : 0x7fffffff;
        bool fresh = false;
        if (k < i) {
          unsigned h = ((unsigned)k * 2654435761u) >> 23;     // 9 bits: AGG_HCAP slots
          int probe = 0;
          for (; probe < AGG_HCAP; probe++) {
            int cur = ((volatile int*)H)[h];
            if (cur == k) break;
            if (cur == -1) {
              int old = atomicCAS(&H[h], -1, k);
              if (old == -1) {
                fresh = true;
                break;
              }
              if (old == k) break;
            }
            h = (h + 1) & (AGG_HCAP - 1);
          }
          if (probe == AGG_HCAP) over = true;
        }
        unsigned bal = __ballot_sync(FULL_MASK, fresh);
        int o = cnt + __popc(bal & ((1u << lane) - 1));
        if (fresh) {
          if (o < AGG_LCAP) L[o] = k;
          else over = true;
        }
        cnt += __popc(bal);
      }
    }
    over = __any_sync(FULL_MASK, over);
    __syncwarp();
    bool covered = false;
    if (!over) {
      // wait: drop decided non-roots each rescan, stop at the first root
      while (true) {
        bool root = false;
        int keep = 0;
        for (int a0 = 0; a0 < cnt; a0 += 32) {
          int a = a0 + lane;
          int key = a < cnt ? L[a] : 0;
          int sk = a < cnt ? vs[key] : 2;
          root |= sk == 1;
          bool pend = sk == 0;
          unsigned bal = __ballot_sync(FULL_MASK, pend);
          __syncwarp();
          if (pend) L[keep + __popc(bal & ((1u << lane) - 1))] = key;
          keep += __popc(bal);
          __syncwarp();
        }
        if (__any_sync(FULL_MASK, root)) {
          covered = true;
          break;
        }
        if (keep == 0) break;
        cnt = keep;
      }
    } else {
      // very long neighbourhoods: rescan through global memory
      while (true) {
        bool pend = false, root = false;
        for (i64 jj = js + lane; jj < je; jj += 32) {
          int j = ci[jj];
          for (i64 kk = rp[j]; kk < rp[j + 1]; kk++) {
            int k = ci[kk];
            if (k >= i) continue;
            int sk = vs[k];
            pend |= sk == 0;
            root |= sk == 1;
          }
        }
        if (__any_sync(FULL_MASK, root)) {
          covered = true;
          break;
        }
        if (!__any_sync(FULL_MASK, pend)) break;
      }
    }
    if (lane == 0) agg_st_release(state + i, covered ? 2 : 1);
    __syncwarp();
  }
}

__global__ void k_agg_root_flags(i64 n, const int* __restrict__ state, i64* __restrict__ flags) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x)
    flags[i] = state[i] == 1;
}

__global__ void k_agg_members(i64 n, const i64* __restrict__ rp, const int* __restrict__ ci,
                              const int* __restrict__ state, const i64* __restrict__ rootpos,
                              i64* __restrict__ memb) {
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < n;
       r += (i64)gridDim.x * blockDim.x) {
    if (state[r] != 1) continue;
    i64 id = rootpos[r];
    for (i64 q = rp[r]; q < rp[r + 1]; q++) memb[ci[q]] = id;
    memb[r] = id;
  }
}

__global__ void k_agg_left_flags(i64 n, const i64* __restrict__ memb, i64* __restrict__ flags) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x)
    flags[i] = memb[i] < 0;
}

__global__ void k_agg_list(i64 n, const i64* __restrict__ flags, const i64* __restrict__ pos,
                           i64* __restrict__ list) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x)
    if (flags[i]) list[pos[i]] = i;
}

__global__ void __launch_bounds__(AGG_WARPS * 32)
    k_agg_leftovers(const i64* __restrict__ nlist, const i64* __restrict__ list,
                    const i64* __restrict__ rp, const int* __restrict__ ci, i64* memb,
                    int* ticket, i64* status) {
  __shared__ i64 own[AGG_WARPS][AGG_CAP];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  i64 nl = *nlist;
  while (true) {
    int t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1);
    t = __shfl_sync(FULL_MASK, t, 0);
    if (t >= nl) return;
    i64 i = list[t];
    i64 s = rp[i], e = rp[i + 1];
    int d = 0;
    bool over = false;
    for (i64 b = s; b < e; b += 32) {
      i64 q = b + lane;
      i64 v = -1;
      if (q < e) {
        int j = ci[q];
        if (j != i) {
          if (j < i)
            while ((v = agg_ld_acquire64(memb + j)) < 0) {
            }
          else
            v = agg_ld_acquire64(memb + j);
        }
      }
      unsigned bal = __ballot_sync(FULL_MASK, v >= 0);
      int o = d + __popc(bal & ((1u << lane) - 1));
      if (v >= 0) {
        if (o < AGG_CAP) own[w][o] = v;
        else over = true;
      }
      d += __popc(bal);
    }
    over = __any_sync(FULL_MASK, over);
    __syncwarp();
    // most frequent owner, lowest id on ties; 0 when no neighbour is assigned
    int bc = 0;
    i64 bv = -1;
    if (!over) {
      for (int a = lane; a < d; a += 32) {
        i64 v = own[w][a];
        int c = 0;
        for (int b2 = 0; b2 < d; b2++) c += own[w][b2] == v;
        if (c > bc || (c == bc && (bv < 0 || v < bv))) {
          bc = c;
          bv = v;
        }
      }
    } else {
      // more assigned neighbours than the buffer holds: the same counts
      // straight from global memory (O(d^2) reads; rare high-degree nodes).
      // Lower neighbours were acquired above; a higher LEFTOVER neighbour is
      // still unassigned (it waits for this node), exactly the reference's
      // "currently assigned" set.
      for (i64 qa = s + lane; qa < e; qa += 32) {
        int ja = ci[qa];
        i64 v = ja == (int)i ? -1 : agg_ld_acquire64(memb + ja);
        if (v < 0) continue;
        int c = 0;
        for (i64 qb = s; qb < e; qb++) {
          int jb = ci[qb];
          if (jb != (int)i && agg_ld_acquire64(memb + jb) == v) c++;
        }
        if (c > bc || (c == bc && (bv < 0 || v < bv))) {
          bc = c;
          bv = v;
        }
      }
      over = false;
    }
    for (int o = 16; o > 0; o >>= 1) {
      int c2 = __shfl_xor_sync(FULL_MASK, bc, o);
      i64 v2 = __shfl_xor_sync(FULL_MASK, bv, o);
      if (v2 >= 0 && (c2 > bc || (c2 == bc && (bv < 0 || v2 < bv)))) {
        bc = c2;
        bv = v2;
      }
    }
    if (lane == 0) {
      if (over) report(status, SPHC_ST_AGG_CAPACITY, i);
      agg_st_release64(memb + i, bv < 0 ? 0 : bv);
    }
    __syncwarp();
  }
}

extern "C" int sphc_aggregate(int64_t n, const int64_t* rp, const int32_t* ci, int32_t* state,
                              int32_t* ticket, int64_t* flags, int64_t* pos, int64_t* list,
                              int64_t* memb, int64_t* status, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) return 0;
  const int TB = 256;
  SPHC_CUDA(cudaMemsetAsync(state, 0, (size_t)n * sizeof(int32_t), s));
  SPHC_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int32_t), s));
  k_agg_roots<<<grid_for(n, AGG_WARPS, SPHC_NUM_SMS * 16), AGG_WARPS * 32, 0, s>>>(n, rp, ci,
                                                                                   state, ticket);
  SPHC_LAUNCH_CHECK();
  SPHC_CUDA(cudaMemsetAsync(flags + n, 0, sizeof(int64_t), s));
  k_agg_root_flags<<<grid_for(n, TB), TB, 0, s>>>(n, state, flags);
  SPHC_LAUNCH_CHECK();
  int rc = sphc_scan_i64(n + 1, flags, pos, stream);  // pos[n] = n_agg
  if (rc) return rc;
  SPHC_CUDA(cudaMemsetAsync(memb, 0xFF, (size_t)n * sizeof(int64_t), s));
  k_agg_members<<<grid_for(n, TB), TB, 0, s>>>(n, rp, ci, state, pos, memb);
  SPHC_LAUNCH_CHECK();
  // list[n] <- n_agg before pos is reused for the leftover offsets
  SPHC_CUDA(cudaMemcpyAsync(list + n, pos + n, sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  k_agg_left_flags<<<grid_for(n, TB), TB, 0, s>>>(n, memb, flags);
  SPHC_LAUNCH_CHECK();
  rc = sphc_scan_i64(n + 1, flags, pos, stream);  // pos[n] = number of leftovers
  if (rc) return rc;
  k_agg_list<<<grid_for(n, TB), TB, 0, s>>>(n, flags, pos, list);
  SPHC_LAUNCH_CHECK();
  SPHC_CUDA(cudaMemsetAsync(ticket, 0, sizeof(int32_t), s));
  k_agg_leftovers<<<grid_for(n, AGG_WARPS, SPHC_NUM_SMS * 16), AGG_WARPS * 32, 0, s>>>(
      pos + n, list, rp, ci, memb, ticket, status);
  SPHC_LAUNCH_CHECK();
  return 0;
}
