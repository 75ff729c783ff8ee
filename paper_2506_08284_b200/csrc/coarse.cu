// Coarse topology on device (reference coarse_gradient.py:106-160).
// Coarse edges = sorted unique (min, max)(agg(t), agg(h)) over fine gradient
// rows with two free ends in different aggregates,
// bucketed by the lower aggregate; single-node edges for aggregates owning the
// free end of a one-entry gradient row, appended in aggregate order.
#include "common.cuh"

__global__ void k_pairs(i64 n_e, const i64* __restrict__ drp, const int* __restrict__ dci,
                        const i64* __restrict__ assign, i64* counts, const i64* __restrict__ brp,
                        i64* cursor, int* __restrict__ bcol) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n_e;
       i += (i64)gridDim.x * blockDim.x) {
    i64 s = drp[i];
    if (drp[i + 1] - s != 2) continue;
    i64 a = assign[dci[s]], b = assign[dci[s + 1]];
    if (a == b) continue;
    i64 lo = a < b ? a : b, hi = a < b ? b : a;
    if (counts) {
      atomicAdd((unsigned long long*)&counts[lo], 1ull);
    } else {
      i64 pos = brp[lo] + (i64)atomicAdd((unsigned long long*)&cursor[lo], 1ull);
      bcol[pos] = (int)hi;
    }
  }
}

extern "C" int sphc_coarse_pairs_count(int64_t n_e, const int64_t* drp, const int32_t* dci,
                                       const int64_t* assign, int64_t* counts, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_pairs<<<grid_for(n_e, 256), 256, 0, s>>>(n_e, drp, dci, assign, counts, nullptr, nullptr,
                                             nullptr);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_coarse_pairs_fill(int64_t n_e, const int64_t* drp, const int32_t* dci,
                                      const int64_t* assign, const int64_t* brp, int64_t* cursor,
                                      int32_t* bcol, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_pairs<<<grid_for(n_e, 256), 256, 0, s>>>(n_e, drp, dci, assign, nullptr, brp, cursor, bcol);
  SPHC_LAUNCH_CHECK();
  return 0;
}

__global__ void k_single_flags(i64 n_e, const i64* __restrict__ drp, const int* __restrict__ dci,
                               const i64* __restrict__ assign, i64* flags) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n_e;
       i += (i64)gridDim.x * blockDim.x) {
    i64 s = drp[i];
    if (drp[i + 1] - s == 1) flags[assign[dci[s]]] = 1;
  }
}

extern "C" int sphc_single_flags(int64_t n_e, const int64_t* drp, const int32_t* dci,
                                 const int64_t* assign, int64_t* flags, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_single_flags<<<grid_for(n_e, 256), 256, 0, s>>>(n_e, drp, dci, assign, flags);
  SPHC_LAUNCH_CHECK();
  return 0;
}

// thread per coarse node a: its interior edges (a, b) are adj positions
// adj_rp[a]..adj_rp[a+1] (edge id = position); its single-node edge, if any,
// is n_int + single_off[a].
__global__ void k_build_dh(i64 n_agg, i64 n_int, const i64* __restrict__ adj_rp,
                           const int* __restrict__ adj_col, const i64* __restrict__ single_off,
                           i64* __restrict__ dh_rp, int* __restrict__ dh_ci,
                           double* __restrict__ dh_v, int* __restrict__ ep_a,
                           int* __restrict__ ep_b, int* __restrict__ single_id, i64 n_single) {
  for (i64 a = (i64)blockIdx.x * blockDim.x + threadIdx.x; a < n_agg;
       a += (i64)gridDim.x * blockDim.x) {
    for (i64 e = adj_rp[a]; e < adj_rp[a + 1]; e++) {
      dh_rp[e] = 2 * e;
      dh_ci[2 * e] = (int)a;
      dh_ci[2 * e + 1] = adj_col[e];
      dh_v[2 * e] = -1.0;
      dh_v[2 * e + 1] = 1.0;
      ep_a[e] = (int)a;
      ep_b[e] = adj_col[e];
    }
    bool has = single_off[a + 1] > single_off[a];
    if (has) {
      i64 r = single_off[a];
      i64 e = n_int + r;
      dh_rp[e] = 2 * n_int + r;
      dh_ci[2 * n_int + r] = (int)a;
      dh_v[2 * n_int + r] = 1.0;
      ep_a[e] = -1;
      ep_b[e] = (int)a;
      single_id[a] = (int)e;
    } else {
      single_id[a] = -1;
    }
    if (a == 0) dh_rp[n_int + n_single] = 2 * n_int + n_single;
  }
}

extern "C" int sphc_build_coarse_gradient(int64_t n_agg, int64_t n_int, const int64_t* adj_rp,
                                          const int32_t* adj_col, const int64_t* single_off,
                                          int64_t n_single, int64_t* dh_rp, int32_t* dh_ci,
                                          double* dh_v, int32_t* ep_a, int32_t* ep_b,
                                          int32_t* single_id, void* stream) {
  cudaStream_t s = as_stream(stream);
  k_build_dh<<<grid_for(n_agg, 128), 128, 0, s>>>(n_agg, n_int, adj_rp, adj_col, single_off,
                                                  dh_rp, dh_ci, dh_v, ep_a, ep_b, single_id,
                                                  n_single);
  SPHC_LAUNCH_CHECK();
  return 0;
}
