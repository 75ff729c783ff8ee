// Host build of the device model-problem assembly (csrc/assemble.cu) --
// TEST INFRASTRUCTURE ONLY. It compiles the very same per-row arithmetic
// (paper_2506_08284_b200/csrc/assemble_rows.cuh) for the CPU, with
// -ffp-contract=off, so (A_e, S, A_n, D) come out bit-identical to the device
// generator. tests/golden/make_golden.py uses it to build the C3 / C4-recipe
// inputs the unmodified reference is run on; the GPU tests then assemble the
// same system on the device, check its sha256 against the golden's and
// compare the device hierarchy with the reference's.
#include <stdint.h>
#include <stdlib.h>
#include <thread>
#include <vector>

#include "assemble_rows.cuh"

using namespace sphc_asm;

namespace {

struct Ctx {
  int N, dirichlet;
  i64 nn, ne, nf;
  std::vector<i64> ecode, rpE, rpN, rpD, cnt;
  std::vector<int> edge_of, fid, flist;
  std::vector<double> X, sig;
  double sig_c;
};

// rows are independent: split [0, n) into contiguous chunks over the host
// threads (each row's arithmetic is fixed, so the split does not matter)
template <class F>
void parallel_rows(i64 n, F f) {
  unsigned nt = std::thread::hardware_concurrency();
  if (nt < 1) nt = 1;
  if (n < 4096) nt = 1;
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; t++)
    th.emplace_back([=] {
      i64 lo = n * t / nt, hi = n * (t + 1) / nt;
      for (i64 i = lo; i < hi; i++) f(i);
    });
  for (auto& x : th) x.join();
}

void scan(std::vector<i64>& c, std::vector<i64>& rp) {
  rp.assign(c.size() + 1, 0);
  for (size_t i = 0; i < c.size(); i++) rp[i + 1] = rp[i] + c[i];
}

}  // namespace

extern "C" void* host_hex_create(int N, int dirichlet, const double* jitter, const double* sigma,
                                 double sigma_c) {
  if (N < 1) return nullptr;
  Ctx* c = new Ctx();
  c->N = N;
  c->dirichlet = dirichlet;
  int n = N + 1;
  c->nn = (i64)n * n * n;
  std::vector<i64> ecnt(c->nn), fcnt(c->nn), eoff, foff;
  for (i64 v = 0; v < c->nn; v++) node_counts(N, dirichlet, v, ecnt.data(), fcnt.data());
  scan(ecnt, eoff);
  scan(fcnt, foff);
  c->ne = eoff[c->nn];
  c->nf = foff[c->nn];
  c->edge_of.resize(3 * c->nn);
  c->ecode.resize(c->ne);
  c->fid.resize(c->nn);
  c->flist.resize(c->nf > 0 ? c->nf : 1);
  for (i64 v = 0; v < c->nn; v++)
    node_tables(N, dirichlet, v, eoff.data(), foff.data(), c->edge_of.data(), c->ecode.data(),
                c->fid.data(), c->flist.data());
  if (jitter) {
    c->X.resize(3 * c->nn);
    for (i64 v = 0; v < c->nn; v++) node_coords(N, v, jitter, c->X.data());
  }
  if (sigma) c->sig.assign(sigma, sigma + (i64)N * N * N);
  c->sig_c = sigma_c;
  const double* X = c->X.empty() ? nullptr : c->X.data();
  const double* sg = c->sig.empty() ? nullptr : c->sig.data();
  c->cnt.assign(c->ne, 0);
  parallel_rows(c->ne, [&](i64 i) {
    edge_row<false>(N, i, c->ecode.data(), c->edge_of.data(), X, sg, sigma_c, nullptr,
                    c->cnt.data(), nullptr, nullptr, nullptr);
  });
  scan(c->cnt, c->rpE);
  std::vector<i64> cn(c->nf, 0);
  parallel_rows(c->nf, [&](i64 r) {
    node_row<false>(N, r, c->flist.data(), c->fid.data(), X, sg, sigma_c, nullptr, cn.data(),
                    nullptr, nullptr);
  });
  scan(cn, c->rpN);
  std::vector<i64> cd(c->ne, 0);
  for (i64 i = 0; i < c->ne; i++)
    grad_row<false>(N, i, c->ecode.data(), c->fid.data(), nullptr, cd.data(), nullptr, nullptr);
  scan(cd, c->rpD);
  return c;
}

// sizes: ne, nf, nnz(A_e) = nnz(S), nnz(A_n), nnz(D)
extern "C" void host_hex_sizes(void* h, int64_t* out) {
  Ctx* c = (Ctx*)h;
  out[0] = c->ne;
  out[1] = c->nf;
  out[2] = c->rpE[c->ne];
  out[3] = c->rpN[c->nf];
  out[4] = c->rpD[c->ne];
}

extern "C" void host_hex_fill(void* h, int64_t* rpE, int32_t* colE, double* vA, double* vS,
                              int64_t* rpN, int32_t* colN, double* vN, int64_t* rpD,
                              int32_t* colD, double* vD) {
  Ctx* c = (Ctx*)h;
  int N = c->N;
  const double* X = c->X.empty() ? nullptr : c->X.data();
  const double* sg = c->sig.empty() ? nullptr : c->sig.data();
  for (i64 i = 0; i <= c->ne; i++) rpE[i] = c->rpE[i];
  for (i64 i = 0; i <= c->nf; i++) rpN[i] = c->rpN[i];
  for (i64 i = 0; i <= c->ne; i++) rpD[i] = c->rpD[i];
  parallel_rows(c->ne, [&](i64 i) {
    edge_row<true>(N, i, c->ecode.data(), c->edge_of.data(), X, sg, c->sig_c, rpE, nullptr, colE,
                   vA, vS);
  });
  parallel_rows(c->nf, [&](i64 r) {
    node_row<true>(N, r, c->flist.data(), c->fid.data(), X, sg, c->sig_c, rpN, nullptr, colN,
                   vN);
  });
  for (i64 i = 0; i < c->ne; i++)
    grad_row<true>(N, i, c->ecode.data(), c->fid.data(), rpD, nullptr, colD, vD);
}

extern "C" void host_hex_destroy(void* h) { delete (Ctx*)h; }
