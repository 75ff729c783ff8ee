// Model-problem operators assembled on the device:
// the hex mesh of the unit cube, lowest-order Nedelec edge operators and the
// auxiliary nodal problem, generated straight into HBM as CSR.
//
// The host generator (paper_2506_08284_b200/inputs.py) reproduces the
// reference's `build_structured_mesh` + `discretize` (meshing.py:61-131,
// assembly.py:47-54) bit for bit, but it takes minutes and >100 GB of host
// RAM at 256^3 and has no curved geometry. Here every output row is computed
// by one thread from the mesh topology alone (the numbering is the
// reference's: node v = x + n y + n^2 z, edges sorted by (tail, axis), hexes
// in C order over (cx, cy, cz)), so there is no COO scatter, no sort and no
// atomics: a row enumerates its <=4 (edge) or <=8 (node) hexes in ascending
// hex order, evaluates the element-matrix row it needs by 3x3x3 Gauss
// quadrature on the trilinear (isoparametric) map, and walks its candidate
// columns in ascending id order, summing the hexes' contributions in hex
// order. Outputs:
//   A_e = S + M  and  S   (one shared pattern: edges sharing a hex)
//   A_n = K + sigma M_n   (free nodes sharing a hex)
//   D                     (edge -> free node incidence, -1 tail / +1 head)
// with S = curl-curl (curl of the covariant-Piola edge basis, contravariant
// metric J^T J / det J; equal to the reference's C^T W C), M = sigma-weighted
// edge mass (covariant Piola, metric det J J^-1 J^-T), K / M_n the trilinear
// nodal stiffness / mass. Every element entry is formed with (lo, hi) roles
// fixed by local index and explicitly rounded operations, so the assembled
// matrices are exactly symmetric. Uniform meshes (no coordinates given) use
// J = h I exactly.
//
// The per-row arithmetic lives in assemble_rows.cuh so that the host build of
// the same rows (oracle/csrc/host_assemble.cpp, golden-input generation) is
// bit-identical.
#include "common.cuh"
#include "assemble_rows.cuh"

using namespace sphc_asm;

// ---------------------------------------------------------------- topology

__global__ void k_hex_node_counts(int N, int dirichlet, i64* __restrict__ ecnt,
                                  i64* __restrict__ fcnt) {
  i64 nn = (i64)(N + 1) * (N + 1) * (N + 1);
  for (i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x; v < nn;
       v += (i64)gridDim.x * blockDim.x)
    node_counts(N, dirichlet, v, ecnt, fcnt);
}

__global__ void k_hex_tables(int N, int dirichlet, const i64* __restrict__ eoff,
                             const i64* __restrict__ foff, int* __restrict__ edge_of,
                             i64* __restrict__ ecode, int* __restrict__ fid,
                             int* __restrict__ flist) {
  i64 nn = (i64)(N + 1) * (N + 1) * (N + 1);
  for (i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x; v < nn;
       v += (i64)gridDim.x * blockDim.x)
    node_tables(N, dirichlet, v, eoff, foff, edge_of, ecode, fid, flist);
}

__global__ void k_hex_coords(int N, const double* __restrict__ jitter, double* __restrict__ X) {
  i64 nn = (i64)(N + 1) * (N + 1) * (N + 1);
  for (i64 v = (i64)blockIdx.x * blockDim.x + threadIdx.x; v < nn;
       v += (i64)gridDim.x * blockDim.x)
    node_coords(N, v, jitter, X);
}

// ---------------------------------------------------------------- rows

template <bool FILL>
__global__ void __launch_bounds__(128)
    k_hex_edge_rows(int N, i64 ne, const i64* __restrict__ ecode, const int* __restrict__ edge_of,
                    const double* __restrict__ X, const double* __restrict__ sig, double sig_c,
                    const i64* __restrict__ rp, i64* __restrict__ cnt, int* __restrict__ col,
                    double* __restrict__ vA, double* __restrict__ vS) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < ne;
       i += (i64)gridDim.x * blockDim.x)
    edge_row<FILL>(N, i, ecode, edge_of, X, sig, sig_c, rp, cnt, col, vA, vS);
}

template <bool FILL>
__global__ void __launch_bounds__(128)
    k_hex_node_rows(int N, i64 nf, const int* __restrict__ flist, const int* __restrict__ fid,
                    const double* __restrict__ X, const double* __restrict__ sig, double sig_c,
                    const i64* __restrict__ rp, i64* __restrict__ cnt, int* __restrict__ col,
                    double* __restrict__ val) {
  for (i64 r = (i64)blockIdx.x * blockDim.x + threadIdx.x; r < nf;
       r += (i64)gridDim.x * blockDim.x)
    node_row<FILL>(N, r, flist, fid, X, sig, sig_c, rp, cnt, col, val);
}

template <bool FILL>
__global__ void k_hex_grad_rows(int N, i64 ne, const i64* __restrict__ ecode,
                                const int* __restrict__ fid, const i64* __restrict__ rp,
                                i64* __restrict__ cnt, int* __restrict__ col,
                                double* __restrict__ val) {
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < ne;
       i += (i64)gridDim.x * blockDim.x)
    grad_row<FILL>(N, i, ecode, fid, rp, cnt, col, val);
}

// ---------------------------------------------------------------- C ABI

extern "C" int sphc_hex_node_counts(int N, int dirichlet, int64_t* ecnt, int64_t* fcnt,
                                    void* stream) {
  if (N < 1) return SPHC_ERR_ARG;
  i64 nn = (i64)(N + 1) * (N + 1) * (N + 1);
  k_hex_node_counts<<<grid_for(nn, 256), 256, 0, as_stream(stream)>>>(N, dirichlet, ecnt, fcnt);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_hex_tables(int N, int dirichlet, const int64_t* eoff, const int64_t* foff,
                               int32_t* edge_of, int64_t* ecode, int32_t* fid, int32_t* flist,
                               void* stream) {
  if (N < 1) return SPHC_ERR_ARG;
  i64 nn = (i64)(N + 1) * (N + 1) * (N + 1);
  k_hex_tables<<<grid_for(nn, 256), 256, 0, as_stream(stream)>>>(N, dirichlet, eoff, foff,
                                                                   edge_of, ecode, fid, flist);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_hex_coords(int N, const double* jitter, double* X, void* stream) {
  if (N < 1) return SPHC_ERR_ARG;
  i64 nn = (i64)(N + 1) * (N + 1) * (N + 1);
  k_hex_coords<<<grid_for(nn, 256), 256, 0, as_stream(stream)>>>(N, jitter, X);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_hex_edge_rows(int N, int64_t ne, const int64_t* ecode, const int32_t* edge_of,
                                  const double* X, const double* sigma, double sigma_const,
                                  const int64_t* rp, int64_t* counts, int32_t* col, double* vA,
                                  double* vS, void* stream) {
  if (ne <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  unsigned g = grid_for(ne, 128, 148 * 64);
  if (rp)
    k_hex_edge_rows<true><<<g, 128, 0, s>>>(N, ne, ecode, edge_of, X, sigma, sigma_const, rp,
                                             counts, col, vA, vS);
  else
    k_hex_edge_rows<false><<<g, 128, 0, s>>>(N, ne, ecode, edge_of, X, sigma, sigma_const, rp,
                                              counts, col, vA, vS);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_hex_node_rows(int N, int64_t nf, const int32_t* flist, const int32_t* fid,
                                  const double* X, const double* sigma, double sigma_const,
                                  const int64_t* rp, int64_t* counts, int32_t* col, double* val,
                                  void* stream) {
  if (nf <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  unsigned g = grid_for(nf, 128, 148 * 64);
  if (rp)
    k_hex_node_rows<true><<<g, 128, 0, s>>>(N, nf, flist, fid, X, sigma, sigma_const, rp, counts,
                                             col, val);
  else
    k_hex_node_rows<false><<<g, 128, 0, s>>>(N, nf, flist, fid, X, sigma, sigma_const, rp,
                                              counts, col, val);
  SPHC_LAUNCH_CHECK();
  return 0;
}

extern "C" int sphc_hex_grad_rows(int N, int64_t ne, const int64_t* ecode, const int32_t* fid,
                                  const int64_t* rp, int64_t* counts, int32_t* col, double* val,
                                  void* stream) {
  if (ne <= 0) return 0;
  cudaStream_t s = as_stream(stream);
  unsigned g = grid_for(ne, 256);
  if (rp)
    k_hex_grad_rows<true><<<g, 256, 0, s>>>(N, ne, ecode, fid, rp, counts, col, val);
  else
    k_hex_grad_rows<false><<<g, 256, 0, s>>>(N, ne, ecode, fid, rp, counts, col, val);
  SPHC_LAUNCH_CHECK();
  return 0;
}
