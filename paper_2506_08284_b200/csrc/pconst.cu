// Algorithm 1 of the paper (reference coarse_gradient.py:36-103,
// gen_piecewise_const) on the device, bit-identical to the sequential loop.
//
//   targets   t_j = max(1, rint(nnz_j / total * m_h))              (thread/col)
//   passes    for pass, for j ascending: column j claims its ceil(t_j/passes)
//             largest-|P| unassigned rows (ties -> lower row)
//   leftovers rows still unassigned, ascending: the largest-|P| column among
//             those with count > 0 (all columns if none), ties -> lower column
//   safeguard columns with count 0, ascending: take the best donor row whose
//             column keeps >= 1 row
//
// Each pass is solved as a fixed point instead of a sweep: every column's
// candidates are pre-sorted once by (|P| desc, row asc); given the current
// claims, column j takes the first ceil(t_j/passes) rows of its list that
// are free at the start of the pass and not claimed by a LOWER column, and a
// row's owner is the lowest column claiming it. Column 0 is exact after one
// iteration, and by induction a column is exact once every lower column it
// shares a row with is, so the iteration reaches the sequential loop's
// result in at most (dependency depth + 1) steps -- in practice a handful,
// whereas waiting column by column serialises on chains of adjacent
// aggregates. Leftover rows whose every column already has count > 0 cannot be
// influenced by other leftovers (a count > 0 predicate never flips back), so
// they are decided in parallel; rows touching a zero-count column, and the
// safeguard, run in order on one warp (both are rare).
#include "common.cuh"

extern "C" int sphc_scan_i64(int64_t n, const int64_t* counts, int64_t* offsets, void* stream);

#define PC_WARPS 4

// (mag, idx) ordering of the reference's lexsort((idx, -mag)): larger
// magnitude first, then the lower index
__device__ __forceinline__ bool pc_better(double m1, i64 i1, double m2, i64 i2) {
  return m1 > m2 || (m1 == m2 && i1 < i2);
}

__device__ __forceinline__ void pc_warp_argmax(double& m, i64& idx) {
  for (int o = 16; o > 0; o >>= 1) {
    double m2 = __shfl_xor_sync(FULL_MASK, m, o);
    i64 i2 = __shfl_xor_sync(FULL_MASK, idx, o);
    if (i2 >= 0 && (idx < 0 || pc_better(m2, i2, m, idx))) {
      m = m2;
      idx = i2;
    }
  }
}

__global__ void k_pc_targets(i64 m_H, i64 m_h, const i64* __restrict__ crp,
                             i64* __restrict__ target, i64* status) {
  i64 total = crp[m_H];
  for (i64 c = (i64)blockIdx.x * blockDim.x + threadIdx.x; c < m_H;
       c += (i64)gridDim.x * blockDim.x) {
    i64 nz = crp[c + 1] - crp[c];
    if (nz == 0) report(status, SPHC_ST_PC_EMPTY_COLUMN, c);
    double t = __dmul_rn(__ddiv_rn((double)nz, (double)total), (double)m_h);
    i64 ti = (i64)rint(t);
    target[c] = ti < 1 ? 1 : ti;
  }
}

// candidates of every column sorted by (|P| desc, row asc): rank sort, warp
// per column (ranks are unique: the order is total)
__global__ void __launch_bounds__(PC_WARPS * 32)
    k_pc_sort(i64 m_H, const i64* __restrict__ crp, const int* __restrict__ crow,
              const double* __restrict__ cval, int* __restrict__ srow) {
  int lane = threadIdx.x & 31;
  i64 gw = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 j = gw; j < m_H; j += nw) {
    i64 c0 = crp[j], c1 = crp[j + 1];
    for (i64 e = c0 + lane; e < c1; e += 32) {
      double m = fabs(cval[e]);
      int r = crow[e];
      i64 rank = 0;
      for (i64 f = c0; f < c1; f++) rank += pc_better(fabs(cval[f]), crow[f], m, r);
      srow[c0 + rank] = r;
    }
  }
}

#define PC_FREE 0x7F7F7F7F  // byte-wise memset value, above any column id

// one fixed-point step of a claiming pass (see the top of the file)
__global__ void __launch_bounds__(PC_WARPS * 32)
    k_pc_choose(i64 m_H, const i64* __restrict__ crp, const int* __restrict__ srow,
                const i64* __restrict__ target, int n_passes, const i64* __restrict__ assign,
                const int* __restrict__ owner_prev, int* owner_cur) {
  int lane = threadIdx.x & 31;
  i64 gw = ((i64)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  i64 nw = ((i64)gridDim.x * blockDim.x) >> 5;
  for (i64 j = gw; j < m_H; j += nw) {
    i64 c0 = crp[j], c1 = crp[j + 1];
    i64 take = (target[j] + n_passes - 1) / n_passes;
    i64 got = 0;
    for (i64 b = c0; b < c1 && got < take; b += 32) {
      i64 e = b + lane;
      bool ok = false;
      int r = 0;
      if (e < c1) {
        r = srow[e];
        ok = assign[r] < 0 && owner_prev[r] >= (int)j;
      }
      unsigned bal = __ballot_sync(FULL_MASK, ok);
      i64 rank = got + __popc(bal & ((1u << lane) - 1));
      if (ok && rank < take) atomicMin(owner_cur + r, (int)j);
      got += __popc(bal);
    }
  }
}

__global__ void k_pc_diff(i64 m_h, const int* __restrict__ a, const int* __restrict__ b,
                          int* changed) {
  bool d = false;
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < m_h;
       r += (i64)gridDim.x * blockDim.x)
    d |= a[r] != b[r];
  if (__syncthreads_or(d) && threadIdx.x == 0) *changed = 1;
}

// One claiming pass's whole fixed-point iteration in a single cooperative
// launch (formerly one choose + diff launch pair and a host round trip per
// iteration): grid-wide barriers separate the owner reset, the claims and
// the change test; changed[2] alternates so a reset never races a read.
#include <cooperative_groups.h>
namespace pcg_ = cooperative_groups;

__global__ void __launch_bounds__(PC_WARPS * 32)
    k_pc_fixpoint(i64 m_h, i64 m_H, const i64* __restrict__ crp, const int* __restrict__ srow,
                  const i64* __restrict__ target, int n_passes, const i64* __restrict__ assign,
                  int* own0, int* own1, int* changed, i64* status) {
  pcg_::grid_group grid = pcg_::this_grid();
  const i64 nt = (i64)gridDim.x * blockDim.x;
  const i64 t0 = (i64)blockIdx.x * blockDim.x + threadIdx.x;
  int lane = threadIdx.x & 31;
  i64 gw = t0 >> 5, nw = nt >> 5;
  for (i64 r = t0; r < m_h; r += nt) own0[r] = PC_FREE;
  if (t0 == 0) changed[0] = changed[1] = 0;
  int cur = 0;
  bool done = false;
  for (i64 it = 0; it <= m_H + 1 && !done; it++) {
    int* oprev = cur ? own1 : own0;
    cur ^= 1;
    int* ocur = cur ? own1 : own0;
    int f = (int)(it & 1);
    for (i64 r = t0; r < m_h; r += nt) ocur[r] = PC_FREE;
    if (t0 == 0) changed[f] = 0;
    grid.sync();
    for (i64 j = gw; j < m_H; j += nw) {           // claims (k_pc_choose)
      i64 c0 = crp[j], c1 = crp[j + 1];
      i64 take = (target[j] + n_passes - 1) / n_passes;
      i64 got = 0;
      for (i64 b = c0; b < c1 && got < take; b += 32) {
        i64 e = b + lane;
        bool ok = false;
        int r = 0;
        if (e < c1) {
          r = srow[e];
          ok = assign[r] < 0 && oprev[r] >= (int)j;
        }
        unsigned bal = __ballot_sync(FULL_MASK, ok);
        i64 rank = got + __popc(bal & ((1u << lane) - 1));
        if (ok && rank < take) atomicMin(ocur + r, (int)j);
        got += __popc(bal);
      }
    }
    grid.sync();
    bool d = false;
    for (i64 r = t0; r < m_h; r += nt) d |= oprev[r] != ocur[r];
    if (__syncthreads_or(d) && threadIdx.x == 0) atomicOr(changed + f, 1);
    grid.sync();
    done = ((volatile int*)changed)[f] == 0;
  }
  // the owners of the fixed point are in own[cur]; leave them in own0
  if (cur == 1)
    for (i64 r = t0; r < m_h; r += nt) own0[r] = own1[r];
  if (!done && t0 == 0) report(status, SPHC_ST_PC_NO_FIXPOINT, 0);
}

__global__ void k_pc_commit(i64 m_h, const int* __restrict__ owner, i64* assign) {
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < m_h;
       r += (i64)gridDim.x * blockDim.x)
    if (assign[r] < 0 && owner[r] != PC_FREE) assign[r] = owner[r];
}

__global__ void k_pc_counts(i64 m_h, const i64* __restrict__ assign, i64* counts) {
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < m_h;
       r += (i64)gridDim.x * blockDim.x) {
    i64 a = assign[r];
    if (a >= 0) atomicAdd((unsigned long long*)&counts[a], 1ull);
  }
}

// leftover rows: decided here when none of their columns has count 0
// (flags[r] = 1 marks the rows left for the ordered pass)
__global__ void k_pc_left(i64 m_h, const i64* __restrict__ prp, const int* __restrict__ pci,
                          const double* __restrict__ pv, i64* assign, i64* counts,
                          i64* __restrict__ flags, i64* status) {
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < m_h;
       r += (i64)gridDim.x * blockDim.x) {
    flags[r] = 0;
    if (assign[r] >= 0) continue;
    i64 s = prp[r], e = prp[r + 1];
    if (s == e) {
      report(status, SPHC_ST_PC_EMPTY_ROW, r);
      continue;
    }
    bool dep = false;
    for (i64 q = s; q < e; q++) dep |= __ldcg(counts + pci[q]) == 0;
    if (dep) {
      flags[r] = 1;
      continue;
    }
    double bm = -1.0;
    i64 bc = -1;
    for (i64 q = s; q < e; q++) {
      double m = fabs(pv[q]);
      if (bc < 0 || pc_better(m, pci[q], bm, bc)) {
        bm = m;
        bc = pci[q];
      }
    }
    assign[r] = bc;
    atomicAdd((unsigned long long*)&counts[bc], 1ull);
  }
}

__global__ void k_pc_list(i64 n, const i64* __restrict__ flags, const i64* __restrict__ pos,
                          i64* __restrict__ list) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (i64)gridDim.x * blockDim.x)
    if (flags[i]) list[pos[i]] = i;
}

// ordered leftover rows (one warp): the reference's loop over the remaining rows
__global__ void k_pc_left_ordered(const i64* __restrict__ nlist, const i64* __restrict__ list,
                                  const i64* __restrict__ prp, const int* __restrict__ pci,
                                  const double* __restrict__ pv, i64* assign, i64* counts) {
  int lane = threadIdx.x;
  i64 n = *nlist;
  for (i64 t = 0; t < n; t++) {
    i64 r = list[t];
    i64 s = prp[r], e = prp[r + 1];
    bool claimed = false;
    for (i64 q = s + lane; q < e; q += 32) claimed |= ((volatile i64*)counts)[pci[q]] > 0;
    claimed = __any_sync(FULL_MASK, claimed);
    double bm = -1.0;
    i64 bc = -1;
    for (i64 q = s + lane; q < e; q += 32) {
      if (claimed && ((volatile i64*)counts)[pci[q]] == 0) continue;
      double m = fabs(pv[q]);
      if (bc < 0 || pc_better(m, pci[q], bm, bc)) {
        bm = m;
        bc = pci[q];
      }
    }
    pc_warp_argmax(bm, bc);
    if (lane == 0) {
      assign[r] = bc;
      ((volatile i64*)counts)[bc] += 1;
    }
    __syncwarp();
  }
}

__global__ void k_pc_zero_cols(i64 m_H, const i64* __restrict__ counts, i64* __restrict__ flags) {
  for (i64 c = (i64)blockIdx.x * blockDim.x + threadIdx.x; c < m_H;
       c += (i64)gridDim.x * blockDim.x)
    flags[c] = counts[c] == 0;
}

// safeguard (one warp): every column keeps at least one row
__global__ void k_pc_safeguard(const i64* __restrict__ nlist, const i64* __restrict__ list,
                               const i64* __restrict__ crp, const int* __restrict__ crow,
                               const double* __restrict__ cval, i64* assign, i64* counts,
                               i64* status) {
  int lane = threadIdx.x;
  i64 n = *nlist;
  volatile i64* vc = counts;
  volatile i64* va = assign;
  for (i64 t = 0; t < n; t++) {
    i64 c = list[t];
    double bm = -1.0;
    i64 br = -1;
    for (i64 e = crp[c] + lane; e < crp[c + 1]; e += 32) {
      int r = crow[e];
      if (vc[va[r]] <= 1) continue;
      double m = fabs(cval[e]);
      if (br < 0 || pc_better(m, r, bm, br)) {
        bm = m;
        br = r;
      }
    }
    pc_warp_argmax(bm, br);
    if (br < 0) {
      if (lane == 0) report(status, SPHC_ST_PC_NO_DONOR, c);
      return;
    }
    if (lane == 0) {
      vc[va[br]] -= 1;
      va[br] = c;
      vc[c] += 1;
    }
    __syncwarp();
  }
}

extern "C" int sphc_piecewise_const(int64_t m_h, int64_t m_H, const int64_t* prp,
                                    const int32_t* pci, const double* pv, const int64_t* crp,
                                    const int32_t* crow, const double* cval, int n_passes,
                                    int64_t* target, int64_t* counts, int32_t* srow,
                                    int32_t* owner, int32_t* changed, int64_t* flags,
                                    int64_t* pos, int64_t* list, int64_t* assign,
                                    int64_t* status, void* stream) {
  cudaStream_t s = as_stream(stream);
  if (m_h <= 0 || m_H <= 0) return 0;
  const int TB = 256;
  unsigned gw = grid_for(m_H, PC_WARPS, SPHC_NUM_SMS * 16);
  k_pc_targets<<<grid_for(m_H, TB), TB, 0, s>>>(m_H, m_h, crp, target, status);
  SPHC_LAUNCH_CHECK();
  k_pc_sort<<<gw, PC_WARPS * 32, 0, s>>>(m_H, crp, crow, cval, srow);
  SPHC_LAUNCH_CHECK();
  SPHC_CUDA(cudaMemsetAsync(assign, 0xFF, (size_t)m_h * sizeof(int64_t), s));  // -1
  int* own[2] = {owner, owner + m_h};
  static int max_blocks = 0;
  if (!max_blocks) {
    int per_sm = 0;
    SPHC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pc_fixpoint,
                                                            PC_WARPS * 32, 0));
    max_blocks = per_sm * SPHC_NUM_SMS;
  }
  // few blocks: the pass is a chain of grid barriers, whose cost grows with
  // the block count; 2 per SM keep every SM busy on the claims
  i64 want = (m_H > m_h ? m_H : m_h) * 32 / (PC_WARPS * 32) + 1;
  int cap = max_blocks < 2 * SPHC_NUM_SMS ? max_blocks : 2 * SPHC_NUM_SMS;
  int gfp = (int)(want < cap ? want : cap);
  i64 mh = m_h, mH = m_H;
  int* own0 = own[0];
  int* own1 = own[1];
  // changed: 2 ints (the device array holds at least one int64 slot's worth)
  for (int pass = 0; pass < n_passes; pass++) {
    void* args[] = {&mh, &mH, (void*)&crp, (void*)&srow, (void*)&target, &n_passes,
                    (void*)&assign, &own0, &own1, &changed, &status};
    SPHC_CUDA(cudaLaunchCooperativeKernel((void*)k_pc_fixpoint, dim3(gfp), dim3(PC_WARPS * 32),
                                          args, 0, s));
    g_sphc_launches++;
    k_pc_commit<<<grid_for(m_h, TB), TB, 0, s>>>(m_h, own0, assign);
    SPHC_LAUNCH_CHECK();
  }
  int rc = 0;
  SPHC_CUDA(cudaMemsetAsync(counts, 0, (size_t)m_H * sizeof(int64_t), s));
  k_pc_counts<<<grid_for(m_h, TB), TB, 0, s>>>(m_h, assign, counts);
  SPHC_LAUNCH_CHECK();
  // parallel leftovers; flags marks the rows that must go in order
  SPHC_CUDA(cudaMemsetAsync(flags + m_h, 0, sizeof(int64_t), s));
  k_pc_left<<<grid_for(m_h, TB), TB, 0, s>>>(m_h, prp, pci, pv, assign, counts, flags, status);
  SPHC_LAUNCH_CHECK();
  rc = sphc_scan_i64(m_h + 1, flags, pos, stream);
  if (rc) return rc;
  k_pc_list<<<grid_for(m_h, TB), TB, 0, s>>>(m_h, flags, pos, list);
  SPHC_LAUNCH_CHECK();
  k_pc_left_ordered<<<1, 32, 0, s>>>(pos + m_h, list, prp, pci, pv, assign, counts);
  SPHC_LAUNCH_CHECK();
  // safeguard over the columns left empty
  SPHC_CUDA(cudaMemsetAsync(flags + m_H, 0, sizeof(int64_t), s));
  k_pc_zero_cols<<<grid_for(m_H, TB), TB, 0, s>>>(m_H, counts, flags);
  SPHC_LAUNCH_CHECK();
  rc = sphc_scan_i64(m_H + 1, flags, pos, stream);
  if (rc) return rc;
  k_pc_list<<<grid_for(m_H, TB), TB, 0, s>>>(m_H, flags, pos, list);
  SPHC_LAUNCH_CHECK();
  k_pc_safeguard<<<1, 32, 0, s>>>(pos + m_H, list, crp, crow, cval, assign, counts, status);
  SPHC_LAUNCH_CHECK();
  return 0;
}
