// Row-wise SpGEMM C = A B, one warp per row of A.
//
// A row's products (a_ik b_kj for the B rows reached from A's row) are walked
// in batches: the longest prefix of A entries whose products fit a staging
// window of SPG_STG. Each batch records, per product, the A entry that owns it
// (owner[], written by the owning lane), so any lane can address any product
// in O(1).
//
// Symbolic (count): product columns go into a per-warp open-addressing hash
//   table in shared memory, sized to the row (2 x its product count).
// Numeric (fill): the table is rebuilt at 2 x the known column count, the
//   keys are sorted into the output column list and each hash slot records
//   its column's sorted position, so a product finds its accumulator with one
//   or two hash probes. Products are staged as (slot, a_ik * b_kj) in k-major
//   order, then accumulated one B row per step from shared memory (a B row's
//   entries have distinct columns, so lanes never collide):
//   ORDERED:  B rows in ascending k with unfused sequential sums -- scipy
//             csr_matmat's order, bit-identical for the nodal Galerkin product
//             (SURVEY.md Appendix A);
//   !ORDERED: even / odd B rows go to two half-warps with their own
//             accumulator copy, summed at the end: deterministic, TOL class
//             (edge Galerkin products, D^T A D, S D).
#include "common.cuh"

#define SPG_WARPS 8    // symbolic pass
#define SPG_HCAP 512   // max hash slots per warp
#define SPG_CCAP 256   // max distinct columns per output row
#define SPG_STG 256    // products per batch
#define SPG_PER_LANE (SPG_STG / 32)

// Numeric-pass capacities. Big: any row up to SPG_CCAP columns, 4 warps per
// block (shared-memory bound, 12 warps per SM). Small: rows of <= 64
// columns (A_e D, S_e D, A_e P_e: every product of the hierarchy but R (A P))
// in a quarter of the shared memory, 8 warps per block and 64 registers, so
// ~3x the warps per SM hide the row's dependent load chains.
template <int STG_, int HCAP_, int CCAP_, int FW_, int MINB_>
struct SpgCfg {
  static constexpr int STG = STG_, HCAP = HCAP_, CCAP = CCAP_, FW = FW_, MINB = MINB_;
  static constexpr int PER_LANE = STG_ / 32;
};
using SpgBig = SpgCfg<256, 512, 256, 4, 1>;
using SpgSmall = SpgCfg<128, 128, 64, 8, 4>;

__device__ __forceinline__ int pow2_at_least(int n, int lo) {
  int m = lo;
  while (m < n) m <<= 1;
  return m;
}

template <int STG>
struct SpgBatchT {
  int off[32];     // inclusive prefix of B-row lengths
  int start[32];   // exclusive prefix
  i64 bs[32];      // B-row starts
  double a[32];    // A values
  unsigned char owner[STG];
};
using SpgBatch = SpgBatchT<SPG_STG>;

// Load the next batch of A row entries [c0, ae). Returns the number of A
// entries in the batch (0 if a single B row exceeds the window) and the
// batch's product count in *total.
template <int STG>
__device__ __forceinline__ int spg_batch(SpgBatchT<STG>& B, i64 c0, i64 ae,
                                         const int* __restrict__ aci,
                                         const double* __restrict__ av,
                                         const i64* __restrict__ brp, int lane, int* total) {
  int len = 0;
  i64 bs = 0;
  double a = 0.0;
  bool valid = c0 + lane < ae;
  if (valid) {
    int k = aci[c0 + lane];
    if (av) a = av[c0 + lane];
    bs = brp[k];
    len = (int)(brp[k + 1] - bs);
  }
  int incl = len;
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(FULL_MASK, incl, o);
    if (lane >= o) incl += y;
  }
  unsigned fit = __ballot_sync(FULL_MASK, valid && incl <= STG);
  int nb = __popc(fit);
  B.off[lane] = incl;
  B.start[lane] = incl - len;
  B.bs[lane] = bs;
  B.a[lane] = a;
  if (lane < nb)
    for (int p = incl - len; p < incl; p++) B.owner[p] = (unsigned char)lane;
  __syncwarp();
  *total = nb ? B.off[nb - 1] : 0;
  return nb;
}

template <class BT>
__device__ __forceinline__ i64 spg_product(const BT& B, int f, int* t_out) {
  int t = B.owner[f];
  *t_out = t;
  return B.bs[t] + (f - B.start[t]);
}

__device__ __forceinline__ unsigned spg_h(int col, int ts) {
  return ((unsigned)col * 2654435761u) & (ts - 1);
}

// inserts col; false on overflow
__device__ __forceinline__ bool spg_insert(int* keys, int ts, int* ucount, int col) {
  unsigned h = spg_h(col, ts);
  for (int probe = 0; probe < ts; probe++) {
    // plain read first: most products hit an already-present column, and a
    // CAS on it would serialise the warp on a handful of addresses
    int cur = ((volatile int*)keys)[h];
    if (cur == col) return true;
    if (cur != -1) {
      h = (h + 1) & (ts - 1);
      continue;
    }
    int old = atomicCAS(&keys[h], -1, col);
    if (old == -1) {
      atomicAdd(ucount, 1);
      return true;
    }
    if (old == col) return true;
    h = (h + 1) & (ts - 1);
  }
  return false;
}

__device__ __forceinline__ int spg_find(const int* keys, int ts, int col) {
  unsigned h = spg_h(col, ts);
  while (keys[h] != col) h = (h + 1) & (ts - 1);
  return (int)h;
}

// Insert the distinct columns of row `row` into keys (size ts).
template <int STG, int CCAP>
__device__ bool spg_symbolic(i64 row, const i64* __restrict__ arp, const int* __restrict__ aci,
                             const i64* __restrict__ brp, const int* __restrict__ bci,
                             int* keys, int ts, int* ucount, SpgBatchT<STG>& B, int lane) {
  constexpr int PER_LANE = STG / 32;
  for (int t = lane; t < ts; t += 32) keys[t] = -1;
  if (lane == 0) *ucount = 0;
  __syncwarp();
  bool ok = true;
  i64 as = arp[row], ae = arp[row + 1];
  for (i64 c0 = as; c0 < ae && ok;) {
    int total;
    int nb = spg_batch(B, c0, ae, aci, nullptr, brp, lane, &total);
    if (nb == 0) {
      ok = false;
      break;
    }
    // all column loads of the batch first (one L2 round trip per batch, not
    // per product: the shared-memory CAS would otherwise serialise them)
    int col[PER_LANE];
#pragma unroll
    for (int u = 0; u < PER_LANE; u++) {
      int f = lane + 32 * u, t;
      col[u] = f < total ? bci[spg_product(B, f, &t)] : -1;
    }
#pragma unroll
    for (int u = 0; u < PER_LANE; u++)
      if (col[u] >= 0) ok &= spg_insert(keys, ts, ucount, col[u]);
    ok = __all_sync(FULL_MASK, ok);
    c0 += nb;
  }
  __syncwarp();
  return ok && *ucount <= CCAP;
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

struct SpgCount {
  int keys[SPG_HCAP];
  SpgBatch B;
  int ucount;
};

__global__ void __launch_bounds__(SPG_WARPS * 32)
    k_spgemm_count(i64 n, const i64* __restrict__ arp, const int* __restrict__ aci,
                   const i64* __restrict__ brp, const int* __restrict__ bci,
                   i64* __restrict__ counts, i64* status) {
  __shared__ SpgCount sc[SPG_WARPS];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  SpgCount& S = sc[w];
  for (i64 row = (i64)blockIdx.x * SPG_WARPS + w; row < n; row += (i64)gridDim.x * SPG_WARPS) {
    int prods = spg_row_products(row, arp, aci, brp, lane);
    int ts = pow2_at_least(2 * prods, 32);
    if (ts > SPG_HCAP) ts = SPG_HCAP;
    bool ok = spg_symbolic<SPG_STG, SPG_CCAP>(row, arp, aci, brp, bci, S.keys, ts, &S.ucount,
                                              S.B, lane);
    if (lane == 0) {
      // -1: beyond the on-chip capacity; the global-memory path
      // (sphc_spgemm_global) counts and fills this row
      counts[row] = ok ? S.ucount : -1;
      if (!ok) report(status, SPHC_ST_SPGEMM_CAPACITY, row);
    }
    __syncwarp();
  }
}

template <class C>
struct SpgFill {
  int keys[C::HCAP];
  short slot[C::HCAP];      // sorted position of the column in keys[h]
  int list[C::CCAP];        // sorted output columns
  double acc[2][C::CCAP];
  short sslot[C::STG];      // staged product slots
  double sval[C::STG];      // staged product values
  SpgBatchT<C::STG> B;
  int ucount;
};

template <class C>
struct SpgFillPair {         // two products on one pattern
  SpgFill<C> f;
  double a2[32];             // second A's values of the batch
  double sval2[C::STG];
  double acc2[2][C::CCAP];   // second product's accumulators (one per group)
};

// ORDERED / unordered as described at the top. PAIR: C1 = A1 B1 and C2 = A2 B2
// with A1, A2 (and B1, B2) sharing one pattern -- the A_e and S_e Galerkin
// products of a level -- computed in one pass (one symbolic phase, indices
// read once); single lane group, accumulators acc[0] / acc[1].
template <bool ORDERED, bool PAIR, class C>
__global__ void __launch_bounds__(C::FW * 32, C::MINB)
    k_spgemm_fill(i64 n, const i64* __restrict__ arp, const int* __restrict__ aci,
                  const double* __restrict__ av, const double* __restrict__ av2,
                  const i64* __restrict__ brp, const int* __restrict__ bci,
                  const double* __restrict__ bv, const double* __restrict__ bv2,
                  const i64* __restrict__ crp, int* __restrict__ cci, double* __restrict__ cv,
                  double* __restrict__ cv2, i64* status, int skip_le) {
  extern __shared__ unsigned char spg_smem[];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  typedef SpgFill<C> Fill;
  typedef SpgFillPair<C> FillPair;
  Fill& F = PAIR ? ((FillPair*)spg_smem)[w].f : ((Fill*)spg_smem)[w];
  double* a2 = PAIR ? ((FillPair*)spg_smem)[w].a2 : nullptr;
  double* sval2 = PAIR ? ((FillPair*)spg_smem)[w].sval2 : nullptr;
  double* acc2 = PAIR ? &((FillPair*)spg_smem)[w].acc2[0][0] : nullptr;
  constexpr int PER_LANE = C::PER_LANE;
  for (i64 row = (i64)blockIdx.x * C::FW + w; row < n; row += (i64)gridDim.x * C::FW) {
    int nu = (int)(crp[row + 1] - crp[row]);
    // rows of another variant's size class: (skip_le, C::CCAP] are ours
    if (nu <= skip_le || nu > C::CCAP) continue;
    int ts = pow2_at_least(2 * nu, 32);
    if (ts > C::HCAP) ts = C::HCAP;
    bool ok = spg_symbolic<C::STG, C::CCAP>(row, arp, aci, brp, bci, F.keys, ts, &F.ucount,
                                             F.B, lane);
    if (!ok) continue;  // flagged by the count pass
    // sorted column list
    int cnt = 0;
    for (int b = 0; b < ts; b += 32) {
      int key = F.keys[b + lane];
      unsigned bal = __ballot_sync(FULL_MASK, key >= 0);
      if (key >= 0) F.list[cnt + __popc(bal & ((1u << lane) - 1))] = key;
      cnt += __popc(bal);
    }
    int m = pow2_at_least(nu, 1);
    for (int t = nu + lane; t < m; t += 32) F.list[t] = 0x7fffffff;
    __syncwarp();
    for (int size = 2; size <= m; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = lane; t < (m >> 1); t += 32) {
          int lo = ((t & ~(stride - 1)) << 1) | (t & (stride - 1)), hi = lo + stride;
          bool up = (lo & size) == 0;
          int a = F.list[lo], b = F.list[hi];
          if ((a > b) == up) {
            F.list[lo] = b;
            F.list[hi] = a;
          }
        }
        __syncwarp();
      }
    for (int t = lane; t < nu; t += 32) {
      F.slot[spg_find(F.keys, ts, F.list[t])] = (short)t;
      F.acc[0][t] = 0.0;
      F.acc[1][t] = 0.0;
      if (PAIR) {
        acc2[t] = 0.0;
        acc2[C::CCAP + t] = 0.0;
      }
    }
    __syncwarp();
    i64 as = arp[row], ae = arp[row + 1];
    const int G = ORDERED ? 1 : 2, LG = 32 / G;
    int g = lane / LG, l = lane % LG;
    double* my = F.acc[g];
    double* my2 = PAIR ? acc2 + g * C::CCAP : nullptr;
    for (i64 c0 = as; c0 < ae;) {
      int total;
      int nb = spg_batch(F.B, c0, ae, aci, av, brp, lane, &total);
      if (nb == 0) {
        if (lane == 0) report(status, SPHC_ST_SPGEMM_CAPACITY, row);
        break;
      }
      if (PAIR) {
        a2[lane] = (c0 + lane < ae) ? av2[c0 + lane] : 0.0;
        __syncwarp();
      }
      {
        // loads of the whole batch first, then the hash lookups
        int col[PER_LANE], own[PER_LANE];
        double v1[PER_LANE], v2[PER_LANE];
#pragma unroll
        for (int u = 0; u < PER_LANE; u++) {
          int f = lane + 32 * u;
          col[u] = -1;
          if (f < total) {
            i64 jb = spg_product(F.B, f, &own[u]);
            col[u] = bci[jb];
            v1[u] = bv[jb];
            if (PAIR) v2[u] = bv2[jb];
          }
        }
#pragma unroll
        for (int u = 0; u < PER_LANE; u++) {
          int f = lane + 32 * u;
          if (col[u] >= 0) {
            F.sslot[f] = F.slot[spg_find(F.keys, ts, col[u])];
            F.sval[f] = __dmul_rn(F.B.a[own[u]], v1[u]);
            if (PAIR) sval2[f] = a2[own[u]] * v2[u];
          }
        }
      }
      __syncwarp();
      for (int t0 = 0; t0 < nb; t0 += G) {  // warp-uniform trip count
        int t = t0 + g;
        if (t < nb) {
          int p1 = F.B.off[t];
          for (int p = F.B.start[t] + l; p < p1; p += LG) {
            int sl = F.sslot[p];
            if (ORDERED) my[sl] = __dadd_rn(my[sl], F.sval[p]);
            else my[sl] += F.sval[p];
            if (PAIR) my2[sl] += sval2[p];
          }
        }
        __syncwarp();
      }
      c0 += nb;
    }
    i64 o = crp[row];
    for (int t = lane; t < nu; t += 32) {
      cci[o + t] = F.list[t];
      if (PAIR) {
        cv[o + t] = F.acc[0][t] + F.acc[1][t];
        cv2[o + t] = acc2[t] + acc2[C::CCAP + t];
      } else {
        cv[o + t] = ORDERED ? F.acc[0][t] : F.acc[0][t] + F.acc[1][t];
      }
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

template <bool ORDERED, bool PAIR, class C>
static int fill_launch_c(i64 n, const i64* arp, const int* aci, const double* av,
                         const double* av2, const i64* brp, const int* bci, const double* bv,
                         const double* bv2, const i64* crp, int* cci, double* cv, double* cv2,
                         i64* status, cudaStream_t s, int skip_le) {
  size_t sm = C::FW * (PAIR ? sizeof(SpgFillPair<C>) : sizeof(SpgFill<C>));
  static bool attr = false;
  if (!attr) {
    SPHC_CUDA(cudaFuncSetAttribute(k_spgemm_fill<ORDERED, PAIR, C>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    attr = true;
  }
  unsigned g = grid_for(n, C::FW, SPHC_NUM_SMS * 32);
  k_spgemm_fill<ORDERED, PAIR, C><<<g, C::FW * 32, sm, s>>>(
      n, arp, aci, av, av2, brp, bci, bv, bv2, crp, cci, cv, cv2, status, skip_le);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// max_cols: the longest output row (from the count pass). Rows of <= 64
// columns go to the small-footprint variant; if longer rows exist, the big
// variant runs after it on those rows only (each skips the other's rows).
template <bool ORDERED, bool PAIR>
static int fill_launch(i64 n, const i64* arp, const int* aci, const double* av,
                       const double* av2, const i64* brp, const int* bci, const double* bv,
                       const double* bv2, const i64* crp, int* cci, double* cv, double* cv2,
                       i64* status, cudaStream_t s, i64 max_cols, int skip0 = 0) {
  int rc = fill_launch_c<ORDERED, PAIR, SpgSmall>(n, arp, aci, av, av2, brp, bci, bv, bv2, crp,
                                                  cci, cv, cv2, status, s, skip0);
  if (rc || (max_cols >= 0 && max_cols <= SpgSmall::CCAP)) return rc;
  return fill_launch_c<ORDERED, PAIR, SpgBig>(n, arp, aci, av, av2, brp, bci, bv, bv2, crp, cci,
                                              cv, cv2, status, s, SpgSmall::CCAP);
}

extern "C" int sphc_spgemm_fill(int64_t n, const int64_t* arp, const int32_t* aci,
                                const double* av, const int64_t* brp, const int32_t* bci,
                                const double* bv, const int64_t* crp, int32_t* cci, double* cv,
                                int ordered, int64_t max_cols, int64_t* status, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  if (ordered)
    return fill_launch<true, false>(n, arp, aci, av, nullptr, brp, bci, bv, nullptr, crp, cci,
                                    cv, nullptr, status, s, max_cols);
  return fill_launch<false, false>(n, arp, aci, av, nullptr, brp, bci, bv, nullptr, crp, cci,
                                   cv, nullptr, status, s, max_cols);
}

extern "C" int sphc_spgemm_fill_pair(int64_t n, const int64_t* arp, const int32_t* aci,
                                     const double* av1, const double* av2, const int64_t* brp,
                                     const int32_t* bci, const double* bv1, const double* bv2,
                                     const int64_t* crp, int32_t* cci, double* cv1,
                                     double* cv2, int64_t max_cols, int64_t* status,
                                     void* stream) {
  if (n <= 0) return 0;
  return fill_launch<false, true>(n, arp, aci, av1, av2, brp, bci, bv1, bv2, crp, cci, cv1,
                                  cv2, status, as_stream(stream), max_cols);
}

// ---------------------------------------------------------------------------
// Thin rows: one THREAD per output row, for products whose rows have few
// products and <= THIN_CAP distinct columns (A_e D, S_e D: 66 products and
// ~18 columns per row; D^T (A D): ~108 and ~27). A warp per row left most
// lanes idle on these and spent ~2,600 warp instructions per row on batch
// bookkeeping; here a thread walks its row's products in scipy's order
// (A entries ascending, each B row ascending, separate multiply and add --
// bitwise csr_matmat, so ORDERED for free) into a private THIN_CAP-slot hash
// table that lives in shared memory, transposed ([slot][thread]) so a warp's
// accesses are conflict free whatever the slots. Rows with more distinct
// columns are counted -1 and left to the warp kernels (the fill skips them
// by their count).
#define THIN_CAP 32
#define THIN_TPB 128

__device__ __forceinline__ unsigned thin_h(int col) {
  return ((unsigned)col * 2654435761u) >> 27;    // 5 bits: THIN_CAP slots
}

// slot of col in the thread's table (inserting it), -1 if the table is full
__device__ __forceinline__ int thin_slot(int (*keys)[THIN_TPB], int tid, int col, int& used) {
  unsigned h = thin_h(col);
  for (int p = 0; p < THIN_CAP; p++) {
    int cur = keys[h][tid];
    if (cur == col) return (int)h;
    if (cur < 0) {
      keys[h][tid] = col;
      used++;
      return (int)h;
    }
    h = (h + 1) & (THIN_CAP - 1);
  }
  return -1;
}

// only_missing: count only the rows another pass left at -1 (never here:
// the thin pass runs first); counts[row] = -1 for rows beyond THIN_CAP.
__global__ void __launch_bounds__(THIN_TPB)
    k_spgemm_thin_count(i64 n, const i64* __restrict__ arp, const int* __restrict__ aci,
                        const i64* __restrict__ brp, const int* __restrict__ bci,
                        i64* __restrict__ counts, int* any_over) {
  __shared__ int keys[THIN_CAP][THIN_TPB];
  int tid = threadIdx.x;
  for (i64 row = (i64)blockIdx.x * THIN_TPB + tid; row < n; row += (i64)gridDim.x * THIN_TPB) {
#pragma unroll
    for (int q = 0; q < THIN_CAP; q++) keys[q][tid] = -1;
    int used = 0;
    bool ok = true;
    i64 ae = arp[row + 1];
    for (i64 j = arp[row]; j < ae && ok; j++) {
      int k = aci[j];
      i64 be = brp[k + 1];
      for (i64 q = brp[k]; q < be; q++)
        if (thin_slot(keys, tid, bci[q], used) < 0) {
          ok = false;
          break;
        }
    }
    counts[row] = ok ? used : -1;
    if (!ok) *any_over = 1;
  }
}

template <bool PAIR>
__global__ void __launch_bounds__(THIN_TPB)
    k_spgemm_thin_fill(i64 n, const i64* __restrict__ arp, const int* __restrict__ aci,
                       const double* __restrict__ av, const double* __restrict__ av2,
                       const i64* __restrict__ brp, const int* __restrict__ bci,
                       const double* __restrict__ bv, const double* __restrict__ bv2,
                       const i64* __restrict__ crp, int* __restrict__ cci,
                       double* __restrict__ cv, double* __restrict__ cv2) {
  extern __shared__ unsigned char thin_smem[];
  int (*keys)[THIN_TPB] = (int (*)[THIN_TPB])thin_smem;
  double (*acc)[THIN_TPB] = (double (*)[THIN_TPB])(thin_smem + sizeof(int) * THIN_CAP * THIN_TPB);
  double (*acc2)[THIN_TPB] = PAIR ? acc + THIN_CAP : nullptr;
  int tid = threadIdx.x;
  for (i64 row = (i64)blockIdx.x * THIN_TPB + tid; row < n; row += (i64)gridDim.x * THIN_TPB) {
    int nu = (int)(crp[row + 1] - crp[row]);
    if (nu > THIN_CAP) continue;            // a warp-kernel row (> THIN_CAP columns)
#pragma unroll
    for (int q = 0; q < THIN_CAP; q++) keys[q][tid] = -1;
    int used = 0;
    i64 aj = arp[row], ae = arp[row + 1];
    // the next A entry and its B-row bounds are loaded while the current B
    // row is accumulated (the chain A col -> B bounds -> B entries is
    // otherwise exposed once per A entry: only ~8 warps per SM run here)
    int kn = 0;
    double an = 0.0, an2 = 0.0;
    i64 bsn = 0, ben = 0;
    if (aj < ae) {
      kn = aci[aj];
      an = av[aj];
      if (PAIR) an2 = av2[aj];
      bsn = brp[kn];
      ben = brp[kn + 1];
    }
    for (i64 j = aj; j < ae; j++) {
      double a = an, a2 = an2;
      i64 bs = bsn, be = ben;
      if (j + 1 < ae) {
        kn = aci[j + 1];
        an = av[j + 1];
        if (PAIR) an2 = av2[j + 1];
        bsn = brp[kn];
        ben = brp[kn + 1];
      }
      for (i64 q = bs; q < be; q++) {
        int before = used;
        int sl = thin_slot(keys, tid, bci[q], used);
        double p1 = __dmul_rn(a, bv[q]);
        double p2 = PAIR ? __dmul_rn(a2, bv2[q]) : 0.0;
        if (used != before) {               // first term of this column: 0 + p
          acc[sl][tid] = __dadd_rn(0.0, p1);
          if (PAIR) acc2[sl][tid] = __dadd_rn(0.0, p2);
        } else {
          acc[sl][tid] = __dadd_rn(acc[sl][tid], p1);
          if (PAIR) acc2[sl][tid] = __dadd_rn(acc2[sl][tid], p2);
        }
      }
    }
    // ascending columns: repeated minimum over the table
    i64 o = crp[row];
    int last = -1;
    for (int t = 0; t < nu; t++) {
      int best = 0x7fffffff, bs = 0;
#pragma unroll
      for (int q = 0; q < THIN_CAP; q++) {
        int kq = keys[q][tid];
        if (kq > last && kq < best) {
          best = kq;
          bs = q;
        }
      }
      cci[o + t] = best;
      cv[o + t] = acc[bs][tid];
      if (PAIR) cv2[o + t] = acc2[bs][tid];
      last = best;
    }
  }
}

// the warp kernel on the rows the thin pass left at -1 (none, usually)
__global__ void __launch_bounds__(SPG_WARPS * 32)
    k_spgemm_count_missing(i64 n, const i64* __restrict__ arp, const int* __restrict__ aci,
                           const i64* __restrict__ brp, const int* __restrict__ bci,
                           i64* __restrict__ counts, const int* any_over, i64* status) {
  if (!*any_over) return;
  __shared__ SpgCount sc[SPG_WARPS];
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  SpgCount& S = sc[w];
  for (i64 row = (i64)blockIdx.x * SPG_WARPS + w; row < n; row += (i64)gridDim.x * SPG_WARPS) {
    if (counts[row] >= 0) continue;
    int prods = spg_row_products(row, arp, aci, brp, lane);
    int ts = pow2_at_least(2 * prods, 32);
    if (ts > SPG_HCAP) ts = SPG_HCAP;
    bool ok = spg_symbolic<SPG_STG, SPG_CCAP>(row, arp, aci, brp, bci, S.keys, ts, &S.ucount,
                                              S.B, lane);
    if (lane == 0) {
      counts[row] = ok ? S.ucount : -1;
      if (!ok) report(status, SPHC_ST_SPGEMM_CAPACITY, row);
    }
    __syncwarp();
  }
}

extern "C" int sphc_spgemm_count_thin(int64_t n, const int64_t* arp, const int32_t* aci,
                                      const int64_t* brp, const int32_t* bci, int64_t* counts,
                                      int32_t* any_over, int64_t* status, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  SPHC_CUDA(cudaMemsetAsync(any_over, 0, sizeof(int32_t), s));
  k_spgemm_thin_count<<<grid_for(n, THIN_TPB, SPHC_NUM_SMS * 16), THIN_TPB, 0, s>>>(
      n, arp, aci, brp, bci, counts, any_over);
  SPHC_LAUNCH_CHECK();
  k_spgemm_count_missing<<<grid_for(n, SPG_WARPS, SPHC_NUM_SMS * 32), SPG_WARPS * 32, 0, s>>>(
      n, arp, aci, brp, bci, counts, any_over, status);
  SPHC_LAUNCH_CHECK();
  return 0;
}

template <bool PAIR>
static int thin_fill_launch(i64 n, const i64* arp, const int* aci, const double* av,
                            const double* av2, const i64* brp, const int* bci, const double* bv,
                            const double* bv2, const i64* crp, int* cci, double* cv, double* cv2,
                            cudaStream_t s) {
  size_t sm = (size_t)THIN_CAP * THIN_TPB * (sizeof(int) + (PAIR ? 2 : 1) * sizeof(double));
  static bool attr = false;
  if (!attr) {
    SPHC_CUDA(cudaFuncSetAttribute(k_spgemm_thin_fill<PAIR>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    attr = true;
  }
  k_spgemm_thin_fill<PAIR><<<grid_for(n, THIN_TPB, SPHC_NUM_SMS * 16), THIN_TPB, sm, s>>>(
      n, arp, aci, av, av2, brp, bci, bv, bv2, crp, cci, cv, cv2);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// Thin rows by the thread-per-row kernel, the rest (max_cols > THIN_CAP; a
// negative max_cols = unknown) by the warp kernels, which skip the thin rows.
extern "C" int sphc_spgemm_fill_thin(int64_t n, const int64_t* arp, const int32_t* aci,
                                     const double* av1, const double* av2, const int64_t* brp,
                                     const int32_t* bci, const double* bv1, const double* bv2,
                                     const int64_t* crp, int32_t* cci, double* cv1,
                                     double* cv2, int ordered, int64_t max_cols,
                                     int64_t* status, void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  int rc = av2 ? thin_fill_launch<true>(n, arp, aci, av1, av2, brp, bci, bv1, bv2, crp, cci, cv1,
                                        cv2, s)
               : thin_fill_launch<false>(n, arp, aci, av1, nullptr, brp, bci, bv1, nullptr, crp,
                                         cci, cv1, nullptr, s);
  if (rc || (max_cols >= 0 && max_cols <= THIN_CAP)) return rc;
  if (av2)
    return fill_launch<false, true>(n, arp, aci, av1, av2, brp, bci, bv1, bv2, crp, cci, cv1,
                                    cv2, status, s, max_cols, THIN_CAP);
  if (ordered)
    return fill_launch<true, false>(n, arp, aci, av1, nullptr, brp, bci, bv1, nullptr, crp, cci,
                                    cv1, nullptr, status, s, max_cols, THIN_CAP);
  return fill_launch<false, false>(n, arp, aci, av1, nullptr, brp, bci, bv1, nullptr, crp, cci,
                                   cv1, nullptr, status, s, max_cols, THIN_CAP);
}

// ---------------------------------------------------------------------------
// Long rows: one CTA of SPC_W warps per output row (C = R (A P) Galerkin
// products, whose rows have 150-2000 A entries and 4k-60k products but only
// ~40-100 distinct columns). The row's A entries are cut into chunks of
// SPC_CH; chunk c belongs to warp c % SPC_W, which walks its B rows in order
// and accumulates into its own copy of the row's accumulators (a B row's
// columns are distinct, so its lanes never collide). The copies are summed
// in warp order: deterministic, TOL class like the unordered warp kernel.
#define SPC_W 8
#define SPC_CH 16
#define SPC_HCAP 1024
#define SPC_CCAP 256
#define SPC_U 4     // B rows loaded per step (independent loads in flight)

struct SpcHead {
  int keys[SPC_HCAP];
  short slot[SPC_HCAP];
  int list[SPC_CCAP];
  int ucount;
  int bad;
};

// Every warp inserts the columns of its chunks' B rows into the CTA's table.
__device__ __forceinline__ void spc_symbolic(i64 as, i64 ae, const int* __restrict__ aci,
                                             const i64* __restrict__ brp,
                                             const int* __restrict__ bci, SpcHead& H, int ts,
                                             int w, int lane) {
  bool ok = true;
  for (i64 c0 = as + (i64)w * SPC_CH; c0 < ae; c0 += (i64)SPC_W * SPC_CH) {
    int nb = (int)min((i64)SPC_CH, ae - c0);
    i64 bs = 0;
    int len = 0;
    if (lane < nb) {
      int k = aci[c0 + lane];
      bs = brp[k];
      len = (int)(brp[k + 1] - bs);
    }
    for (int t0 = 0; t0 < nb; t0 += SPC_U) {
      int col[SPC_U];
#pragma unroll
      for (int u = 0; u < SPC_U; u++) {
        int t = t0 + u;
        i64 b = __shfl_sync(FULL_MASK, bs, t & 31);
        int l = __shfl_sync(FULL_MASK, len, t & 31);
        col[u] = (t < nb && lane < l) ? bci[b + lane] : -1;
      }
#pragma unroll
      for (int u = 0; u < SPC_U; u++)
        if (col[u] >= 0) ok &= spg_insert(H.keys, ts, &H.ucount, col[u]);
      // B rows longer than a warp (rare)
      for (int u = 0; u < SPC_U; u++) {
        int t = t0 + u;
        i64 b = __shfl_sync(FULL_MASK, bs, t & 31);
        int l = __shfl_sync(FULL_MASK, len, t & 31);
        if (t < nb)
          for (int q = 32 + lane; q < l; q += 32) ok &= spg_insert(H.keys, ts, &H.ucount, bci[b + q]);
      }
    }
  }
  if (!ok) H.bad = 1;
}

__device__ __forceinline__ void spc_clear(SpcHead& H, int ts) {
  for (int t = threadIdx.x; t < ts; t += blockDim.x) H.keys[t] = -1;
  if (threadIdx.x == 0) {
    H.ucount = 0;
    H.bad = 0;
  }
}

__global__ void __launch_bounds__(SPC_W * 32)
    k_spgemm_count_cta(i64 n, const i64* __restrict__ arp, const int* __restrict__ aci,
                       const i64* __restrict__ brp, const int* __restrict__ bci,
                       i64* __restrict__ counts, i64* status) {
  __shared__ SpcHead H;
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (i64 row = blockIdx.x; row < n; row += gridDim.x) {
    spc_clear(H, SPC_HCAP);
    __syncthreads();
    spc_symbolic(arp[row], arp[row + 1], aci, brp, bci, H, SPC_HCAP, w, lane);
    __syncthreads();
    if (threadIdx.x == 0) {
      bool ok = !H.bad && H.ucount <= SPC_CCAP;
      counts[row] = ok ? H.ucount : -1;   // -1: global-memory path
      if (!ok) report(status, SPHC_ST_SPGEMM_CAPACITY, row);
    }
    __syncthreads();
  }
}

template <bool PAIR>
__global__ void __launch_bounds__(SPC_W * 32)
    k_spgemm_fill_cta(i64 n, const i64* __restrict__ arp, const int* __restrict__ aci,
                      const double* __restrict__ av, const double* __restrict__ av2,
                      const i64* __restrict__ brp, const int* __restrict__ bci,
                      const double* __restrict__ bv, const double* __restrict__ bv2,
                      const i64* __restrict__ crp, int* __restrict__ cci, double* __restrict__ cv,
                      double* __restrict__ cv2) {
  __shared__ SpcHead H;
  extern __shared__ double spc_acc[];   // [PAIR + 1][SPC_W][SPC_CCAP]
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* my = spc_acc + w * SPC_CCAP;
  double* my2 = PAIR ? spc_acc + (SPC_W + w) * SPC_CCAP : nullptr;
  for (i64 row = blockIdx.x; row < n; row += gridDim.x) {
    int nu = (int)(crp[row + 1] - crp[row]);
    // empty, or beyond the on-chip capacity (the global-memory path's row)
    if (nu == 0 || nu > SPC_CCAP) continue;
    int ts = pow2_at_least(2 * nu, 64);
    if (ts > SPC_HCAP) ts = SPC_HCAP;
    i64 as = arp[row], ae = arp[row + 1];
    spc_clear(H, ts);
    for (int t = threadIdx.x; t < SPC_W * SPC_CCAP; t += blockDim.x) {
      spc_acc[t] = 0.0;
      if (PAIR) spc_acc[SPC_W * SPC_CCAP + t] = 0.0;
    }
    __syncthreads();
    spc_symbolic(as, ae, aci, brp, bci, H, ts, w, lane);
    __syncthreads();
    // rank sort: each occupied slot learns its column's sorted position
    for (int h = threadIdx.x; h < ts; h += blockDim.x) {
      int key = H.keys[h];
      if (key < 0) continue;
      int r = 0;
      for (int g = 0; g < ts; g++) {
        int o = H.keys[g];
        r += (o >= 0) & (o < key);
      }
      H.slot[h] = (short)r;
      H.list[r] = key;
    }
    __syncthreads();
    // numeric: each warp over its chunks, one B row per lane-group step
    for (i64 c0 = as + (i64)w * SPC_CH; c0 < ae; c0 += (i64)SPC_W * SPC_CH) {
      int nb = (int)min((i64)SPC_CH, ae - c0);
      i64 bs = 0;
      int len = 0;
      double a = 0.0, a2 = 0.0;
      if (lane < nb) {
        int k = aci[c0 + lane];
        bs = brp[k];
        len = (int)(brp[k + 1] - bs);
        a = av[c0 + lane];
        if (PAIR) a2 = av2[c0 + lane];
      }
      for (int t0 = 0; t0 < nb; t0 += SPC_U) {
        int col[SPC_U];
        double v[SPC_U], v2[SPC_U];
#pragma unroll
        for (int u = 0; u < SPC_U; u++) {
          int t = t0 + u;
          i64 b = __shfl_sync(FULL_MASK, bs, t & 31);
          int l = __shfl_sync(FULL_MASK, len, t & 31);
          col[u] = -1;
          if (t < nb && lane < l) {
            col[u] = bci[b + lane];
            v[u] = bv[b + lane];
            if (PAIR) v2[u] = bv2[b + lane];
          }
        }
#pragma unroll
        for (int u = 0; u < SPC_U; u++) {
          int t = t0 + u;
          double at = __shfl_sync(FULL_MASK, a, t & 31);
          double at2 = PAIR ? __shfl_sync(FULL_MASK, a2, t & 31) : 0.0;
          if (col[u] >= 0) {
            int sl = H.slot[spg_find(H.keys, ts, col[u])];
            my[sl] += at * v[u];
            if (PAIR) my2[sl] += at2 * v2[u];
          }
          __syncwarp();
        }
        for (int u = 0; u < SPC_U; u++) {   // B rows longer than a warp (rare)
          int t = t0 + u;
          i64 b = __shfl_sync(FULL_MASK, bs, t & 31);
          int l = __shfl_sync(FULL_MASK, len, t & 31);
          double at = __shfl_sync(FULL_MASK, a, t & 31);
          double at2 = PAIR ? __shfl_sync(FULL_MASK, a2, t & 31) : 0.0;
          if (t < nb)
            for (int q = 32 + lane; q < l; q += 32) {
              int sl = H.slot[spg_find(H.keys, ts, bci[b + q])];
              my[sl] += at * bv[b + q];
              if (PAIR) my2[sl] += at2 * bv2[b + q];
            }
          __syncwarp();
        }
      }
    }
    __syncthreads();
    i64 o = crp[row];
    for (int t = threadIdx.x; t < nu; t += blockDim.x) {
      double s = 0.0, s2 = 0.0;
#pragma unroll
      for (int g = 0; g < SPC_W; g++) {
        s += spc_acc[g * SPC_CCAP + t];
        if (PAIR) s2 += spc_acc[(SPC_W + g) * SPC_CCAP + t];
      }
      cci[o + t] = H.list[t];
      cv[o + t] = s;
      if (PAIR) cv2[o + t] = s2;
    }
    __syncthreads();
  }
}

static unsigned cta_grid(i64 n) {
  // 4 resident CTAs per SM (pair accumulators: 32 KB + 7 KB of table per CTA)
  i64 g = n < (i64)SPHC_NUM_SMS * 16 ? n : (i64)SPHC_NUM_SMS * 16;
  return (unsigned)(g > 0 ? g : 1);
}

extern "C" int sphc_spgemm_count_long(int64_t n, const int64_t* arp, const int32_t* aci,
                                      const int64_t* brp, const int32_t* bci, int64_t* counts,
                                      int64_t* status, void* stream) {
  if (n <= 0) return 0;
  k_spgemm_count_cta<<<cta_grid(n), SPC_W * 32, 0, as_stream(stream)>>>(n, arp, aci, brp, bci,
                                                                         counts, status);
  SPHC_LAUNCH_CHECK();
  return 0;
}

template <bool PAIR>
static int fill_cta_launch(i64 n, const i64* arp, const int* aci, const double* av,
                           const double* av2, const i64* brp, const int* bci, const double* bv,
                           const double* bv2, const i64* crp, int* cci, double* cv, double* cv2,
                           cudaStream_t s) {
  size_t sm = (PAIR ? 2 : 1) * SPC_W * SPC_CCAP * sizeof(double);
  static bool attr = false;
  if (!attr) {
    SPHC_CUDA(cudaFuncSetAttribute(k_spgemm_fill_cta<PAIR>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
    attr = true;
  }
  k_spgemm_fill_cta<PAIR><<<cta_grid(n), SPC_W * 32, sm, s>>>(n, arp, aci, av, av2, brp, bci, bv,
                                                              bv2, crp, cci, cv, cv2);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_spgemm_fill_long(int64_t n, const int64_t* arp, const int32_t* aci,
                                     const double* av, const double* av2, const int64_t* brp,
                                     const int32_t* bci, const double* bv, const double* bv2,
                                     const int64_t* crp, int32_t* cci, double* cv1, double* cv2,
                                     void* stream) {
  if (n <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  if (av2)
    return fill_cta_launch<true>(n, arp, aci, av, av2, brp, bci, bv, bv2, crp, cci, cv1, cv2, s);
  return fill_cta_launch<false>(n, arp, aci, av, nullptr, brp, bci, bv, nullptr, crp, cci, cv1,
                                nullptr, s);
}

// ---------------------------------------------------------------------------
// Global-memory path for the rows the on-chip kernels cannot hold (more
// than 256 distinct columns, a B row longer than a staging window, or a
// hash table overflow; the count kernels mark them with -1). One CTA per
// such row, the row's hash table in global scratch (hoff: per-row offsets,
// power-of-two sizes >= 2 x the row's products):
//   COUNT: insert every product column, count the distinct ones;
//   FILL:  insert again, collect the columns, sort them in shared memory
//          (bitonic, <= SPG_GCAP columns), record each column's sorted slot,
//          then accumulate A entry by A entry in ascending k (a B row's
//          columns are distinct, so the threads never collide) with
//          unfused sums: scipy's csr_matmat order, bitwise ORDERED.
#define SPG_GT 256
#define SPG_GCAP 8192

__global__ void k_spgemm_global_products(i64 nrows, const i64* __restrict__ rows,
                                         const i64* __restrict__ arp, const int* __restrict__ aci,
                                         const i64* __restrict__ brp, i64* __restrict__ prods) {
  for (i64 r = blockIdx.x; r < nrows; r += gridDim.x) {
    i64 row = rows[r];
    i64 t = 0;
    for (i64 j = arp[row] + threadIdx.x; j < arp[row + 1]; j += blockDim.x) {
      int k = aci[j];
      t += brp[k + 1] - brp[k];
    }
    __shared__ i64 red[SPG_GT];
    red[threadIdx.x] = t;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) prods[r] = red[0];
    __syncthreads();
  }
}

__device__ __forceinline__ i64 spg_gh(int col, i64 ts) {
  return (i64)(((unsigned long long)(unsigned)col * 11400714819323198485ull) >> 20) & (ts - 1);
}

__device__ int spg_ginsert(int* keys, i64 ts, int col) {   // 1 if newly inserted
  i64 h = spg_gh(col, ts);
  for (;;) {
    int cur = ((volatile int*)keys)[h];
    if (cur == col) return 0;
    if (cur == -1) {
      int old = atomicCAS(&keys[h], -1, col);
      if (old == -1) return 1;
      if (old == col) return 0;
    }
    h = (h + 1) & (ts - 1);
  }
}

__device__ __forceinline__ i64 spg_gfind(const int* keys, i64 ts, int col) {
  i64 h = spg_gh(col, ts);
  while (keys[h] != col) h = (h + 1) & (ts - 1);
  return h;
}

template <bool FILL, bool PAIR>
__global__ void __launch_bounds__(SPG_GT)
    k_spgemm_global(i64 nrows, const i64* __restrict__ rows, const i64* __restrict__ hoff,
                    int* __restrict__ hkeys, int* __restrict__ hslot,
                    const i64* __restrict__ arp, const int* __restrict__ aci,
                    const double* __restrict__ av, const double* __restrict__ av2,
                    const i64* __restrict__ brp, const int* __restrict__ bci,
                    const double* __restrict__ bv, const double* __restrict__ bv2,
                    i64* __restrict__ counts, const i64* __restrict__ crp,
                    int* __restrict__ cci, double* __restrict__ cv, double* __restrict__ cv2,
                    i64* status) {
  extern __shared__ int glist[];          // FILL: sorted columns (<= SPG_GCAP)
  __shared__ int ucount;
  for (i64 r = blockIdx.x; r < nrows; r += gridDim.x) {
    i64 row = rows[r];
    i64 ts = hoff[r + 1] - hoff[r];
    int* keys = hkeys + hoff[r];
    int* slot = hslot + hoff[r];
    for (i64 h = threadIdx.x; h < ts; h += blockDim.x) keys[h] = -1;
    if (threadIdx.x == 0) ucount = 0;
    __syncthreads();
    i64 as = arp[row], ae = arp[row + 1];
    int mine = 0;
    // products: A entries in chunks, every thread walks one B row at a time
    for (i64 j = as; j < ae; j++) {
      int k = aci[j];
      for (i64 q = brp[k] + threadIdx.x; q < brp[k + 1]; q += blockDim.x)
        mine += spg_ginsert(keys, ts, bci[q]);
    }
    atomicAdd(&ucount, mine);
    __syncthreads();
    int nu = ucount;
    // every thread holds nu before thread 0 reuses the counter below (a
    // late reader saw 0 or a partial collect count: its sort loops then ran
    // a different number of barriers -- an intermittent hang)
    __syncthreads();
    if (!FILL) {
      if (threadIdx.x == 0) counts[row] = nu;
      __syncthreads();
      continue;
    }
    if (nu > SPG_GCAP) {
      if (threadIdx.x == 0) report(status, SPHC_ST_SPGEMM_CAPACITY, row);
      __syncthreads();
      continue;
    }
    // collect, then bitonic sort in shared memory
    if (threadIdx.x == 0) ucount = 0;
    __syncthreads();
    for (i64 h = threadIdx.x; h < ts; h += blockDim.x) {
      int key = keys[h];
      if (key >= 0) glist[atomicAdd(&ucount, 1)] = key;
    }
    int m = 1;
    while (m < nu) m <<= 1;
    __syncthreads();
    for (int t = nu + threadIdx.x; t < m; t += blockDim.x) glist[t] = 0x7fffffff;
    __syncthreads();
    for (int size = 2; size <= m; size <<= 1)
      for (int stride = size >> 1; stride > 0; stride >>= 1) {
        for (int t = threadIdx.x; t < (m >> 1); t += blockDim.x) {
          int lo = ((t & ~(stride - 1)) << 1) | (t & (stride - 1)), hi = lo + stride;
          bool up = (lo & size) == 0;
          int a = glist[lo], b = glist[hi];
          if ((a > b) == up) {
            glist[lo] = b;
            glist[hi] = a;
          }
        }
        __syncthreads();
      }
    i64 o = crp[row];
    for (int t = threadIdx.x; t < nu; t += blockDim.x) {
      slot[spg_gfind(keys, ts, glist[t])] = t;
      cci[o + t] = glist[t];
      cv[o + t] = 0.0;
      if (PAIR) cv2[o + t] = 0.0;
    }
    __syncthreads();
    for (i64 j = as; j < ae; j++) {
      int k = aci[j];
      double a = av[j], a2 = PAIR ? av2[j] : 0.0;
      for (i64 q = brp[k] + threadIdx.x; q < brp[k + 1]; q += blockDim.x) {
        int sl = slot[spg_gfind(keys, ts, bci[q])];
        cv[o + sl] = __dadd_rn(cv[o + sl], __dmul_rn(a, bv[q]));
        if (PAIR) cv2[o + sl] = __dadd_rn(cv2[o + sl], __dmul_rn(a2, bv2[q]));
      }
      __syncthreads();
    }
  }
}

extern "C" int sphc_spgemm_global_products(int64_t nrows, const int64_t* rows,
                                           const int64_t* arp, const int32_t* aci,
                                           const int64_t* brp, int64_t* prods, void* stream) {
  if (nrows <= 0) return 0;
  k_spgemm_global_products<<<grid_for(nrows, 1, SPHC_NUM_SMS * 8), SPG_GT, 0,
                             as_stream(stream)>>>(nrows, rows, arp, aci, brp, prods);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_spgemm_global(int64_t nrows, const int64_t* rows, const int64_t* hoff,
                                  int32_t* hkeys, int32_t* hslot, const int64_t* arp,
                                  const int32_t* aci, const double* av, const double* av2,
                                  const int64_t* brp, const int32_t* bci, const double* bv,
                                  const double* bv2, int64_t* counts, const int64_t* crp,
                                  int32_t* cci, double* cv, double* cv2, int64_t* status,
                                  void* stream) {
  if (nrows <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  unsigned g = grid_for(nrows, 1, SPHC_NUM_SMS * 8);
  size_t sm = SPG_GCAP * sizeof(int);
  if (!crp) {
    k_spgemm_global<false, false><<<g, SPG_GT, 0, s>>>(nrows, rows, hoff, hkeys, hslot, arp,
                                                        aci, av, av2, brp, bci, bv, bv2, counts,
                                                        crp, cci, cv, cv2, status);
  } else if (av2) {
    static bool attr = false;
    if (!attr) {
      SPHC_CUDA(cudaFuncSetAttribute(k_spgemm_global<true, true>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      attr = true;
    }
    k_spgemm_global<true, true><<<g, SPG_GT, sm, s>>>(nrows, rows, hoff, hkeys, hslot, arp, aci,
                                                       av, av2, brp, bci, bv, bv2, counts, crp,
                                                       cci, cv, cv2, status);
  } else {
    static bool attr = false;
    if (!attr) {
      SPHC_CUDA(cudaFuncSetAttribute(k_spgemm_global<true, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      attr = true;
    }
    k_spgemm_global<true, false><<<g, SPG_GT, sm, s>>>(nrows, rows, hoff, hkeys, hslot, arp,
                                                        aci, av, av2, brp, bci, bv, bv2, counts,
                                                        crp, cci, cv, cv2, status);
  }
  SPHC_LAUNCH_CHECK();
  return 0;
}
