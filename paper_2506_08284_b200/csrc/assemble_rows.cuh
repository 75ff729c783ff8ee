// Per-row arithmetic of the model-problem assembly (assemble.cu), shared by
// the device kernels and the host build of the same rows
// (oracle/csrc/host_assemble.cpp, test infrastructure: it generates the
// inputs the reference is run on for the golden fixtures). Every rounding
// step is explicit (M_/A_/S_ are __dmul_rn/__dadd_rn/__dsub_rn on the device,
// plain IEEE operations on the host compiled with -ffp-contract=off) and the
// rest are single correctly rounded IEEE operations (/, 1 - t), so both
// builds produce the same bits.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define SPHC_HD __host__ __device__ inline
#define SPHC_HDI __host__ __device__ __forceinline__
#define SPHC_ASM_TABLE __constant__
#else
#define SPHC_HD static inline
#define SPHC_HDI static inline
#define SPHC_ASM_TABLE static const
#endif

namespace sphc_asm {

typedef int64_t i64;


// local hex edges in the reference's order (corner c ascending, then axis),
// inputs.py _LOCAL_EDGES / meshing.py:183-189: LOC[c][axis] -> local index
SPHC_ASM_TABLE signed char LOC[8][3] = {{0, 1, 2},  {-1, 3, 4}, {5, -1, 6}, {-1, -1, 7},
                                      {8, 9, -1}, {-1, 10, -1}, {11, -1, -1}, {-1, -1, -1}};
SPHC_ASM_TABLE unsigned char LCORNER[12] = {0, 0, 0, 1, 1, 2, 2, 3, 4, 4, 5, 6};
SPHC_ASM_TABLE unsigned char LAXIS[12] = {0, 1, 2, 1, 2, 0, 2, 2, 0, 1, 1, 0};

#ifdef __CUDA_ARCH__
SPHC_HDI double M_(double a, double b) { return __dmul_rn(a, b); }
SPHC_HDI double A_(double a, double b) { return __dadd_rn(a, b); }
SPHC_HDI double S_(double a, double b) { return __dsub_rn(a, b); }
#else
// host build (g++ -ffp-contract=off): plain IEEE operations round the same way
SPHC_HDI double M_(double a, double b) { return a * b; }
SPHC_HDI double A_(double a, double b) { return a + b; }
SPHC_HDI double S_(double a, double b) { return a - b; }
#endif

// 3-point Gauss on [0, 1]
SPHC_HDI void gauss3(int q, double& t, double& w) {
  const double r = 0.38729833462074170;   // sqrt(3/5) / 2
  t = q == 0 ? 0.5 - r : (q == 1 ? 0.5 : 0.5 + r);
  w = q == 1 ? 8.0 / 18.0 : 5.0 / 18.0;
}

SPHC_HDI double hat(int d, double t) { return d ? t : 1.0 - t; }
SPHC_HDI double dhat(int d) { return d ? 1.0 : -1.0; }

struct Geo {
  // metrics at one quadrature point, scaled by the weight:
  //   G = w det(J) J^-1 J^-T  (covariant: edge mass, nodal stiffness)
  //   H = w J^T J / det(J)    (contravariant: curl-curl)
  //   wdet = w det(J)         (nodal mass)
  double G[6], H[6], wdet;   // symmetric 3x3 packed xx yy zz xy xz yz
};

SPHC_HDI double sym(const double* P, int a, int b) {
  if (a == b) return P[a];
  int s = a + b;   // (0,1) -> 3, (0,2) -> 4, (1,2) -> 5
  return P[s == 1 ? 3 : (s == 2 ? 4 : 5)];
}

// corner coordinates of hex c (8 x 3) from X (n^3 x 3)
SPHC_HDI void load_corners(const double* __restrict__ X, int n, const int c[3],
                                             double xc[8][3]) {
  for (int k = 0; k < 8; k++) {
    i64 v = (i64)(c[0] + (k & 1)) + (i64)n * ((c[1] + ((k >> 1) & 1)) +
                                              (i64)n * (c[2] + ((k >> 2) & 1)));
    xc[k][0] = X[3 * v];
    xc[k][1] = X[3 * v + 1];
    xc[k][2] = X[3 * v + 2];
  }
}

SPHC_HD void geometry(const double xc[8][3], bool uniform, double h, const double xi[3],
                         double w, Geo& g) {
  if (uniform) {
    // J = h I: G = w h I, H = w I / h, wdet = w h^3
    double gd = M_(w, h), hd = w / h;
    g.G[0] = g.G[1] = g.G[2] = gd;
    g.H[0] = g.H[1] = g.H[2] = hd;
    g.G[3] = g.G[4] = g.G[5] = 0.0;
    g.H[3] = g.H[4] = g.H[5] = 0.0;
    g.wdet = M_(w, M_(M_(h, h), h));
    return;
  }
  double J[3][3];
  for (int p = 0; p < 3; p++)
    for (int q = 0; q < 3; q++) J[p][q] = 0.0;
  for (int k = 0; k < 8; k++) {
    int d[3] = {k & 1, (k >> 1) & 1, (k >> 2) & 1};
    double dN[3];
    for (int q = 0; q < 3; q++) {
      double v = dhat(d[q]);
      for (int r = 0; r < 3; r++)
        if (r != q) v = M_(v, hat(d[r], xi[r]));
      dN[q] = v;
    }
    for (int p = 0; p < 3; p++)
      for (int q = 0; q < 3; q++) J[p][q] = A_(J[p][q], M_(xc[k][p], dN[q]));
  }
  // adjugate: J^-1 = adj / det
  double C[3][3];
  C[0][0] = S_(M_(J[1][1], J[2][2]), M_(J[1][2], J[2][1]));
  C[0][1] = S_(M_(J[0][2], J[2][1]), M_(J[0][1], J[2][2]));
  C[0][2] = S_(M_(J[0][1], J[1][2]), M_(J[0][2], J[1][1]));
  C[1][0] = S_(M_(J[1][2], J[2][0]), M_(J[1][0], J[2][2]));
  C[1][1] = S_(M_(J[0][0], J[2][2]), M_(J[0][2], J[2][0]));
  C[1][2] = S_(M_(J[0][2], J[1][0]), M_(J[0][0], J[1][2]));
  C[2][0] = S_(M_(J[1][0], J[2][1]), M_(J[1][1], J[2][0]));
  C[2][1] = S_(M_(J[0][1], J[2][0]), M_(J[0][0], J[2][1]));
  C[2][2] = S_(M_(J[0][0], J[1][1]), M_(J[0][1], J[1][0]));
  double det = A_(A_(M_(J[0][0], C[0][0]), M_(J[0][1], C[1][0])), M_(J[0][2], C[2][0]));
  // G = w det J^-1 J^-T = w adj adj^T / det ; H = w J^T J / det
  const int PA[6] = {0, 1, 2, 0, 0, 1}, PB[6] = {0, 1, 2, 1, 2, 2};
  double wd = w / det;
  for (int s = 0; s < 6; s++) {
    int a = PA[s], b = PB[s];
    double ga = A_(A_(M_(C[a][0], C[b][0]), M_(C[a][1], C[b][1])), M_(C[a][2], C[b][2]));
    double ha = A_(A_(M_(J[0][a], J[0][b]), M_(J[1][a], J[1][b])), M_(J[2][a], J[2][b]));
    g.G[s] = M_(wd, ga);
    g.H[s] = M_(wd, ha);
  }
  g.wdet = M_(w, det);
}

// reference-cube curl of the edge function of local edge k at xi:
// phi_k = e_ax prod_{b != ax} l_{d_b}(xi_b), curl = grad f x e_ax
SPHC_HDI void ref_curl(int k, const double xi[3], double cu[3]) {
  int c = LCORNER[k], ax = LAXIS[k];
  int d[3] = {c & 1, (c >> 1) & 1, (c >> 2) & 1};
  double g[3] = {0.0, 0.0, 0.0};
  for (int b = 0; b < 3; b++) {
    if (b == ax) continue;
    int o = 3 - ax - b;
    g[b] = M_(dhat(d[b]), hat(d[o], xi[o]));
  }
  if (ax == 0) { cu[0] = 0.0; cu[1] = g[2]; cu[2] = -g[1]; }
  else if (ax == 1) { cu[0] = -g[2]; cu[1] = 0.0; cu[2] = g[0]; }
  else { cu[0] = g[1]; cu[1] = -g[0]; cu[2] = 0.0; }
}

SPHC_HDI double ref_shape2(int k, const double xi[3]) {
  int c = LCORNER[k], ax = LAXIS[k];
  double v = 1.0;
  for (int b = 0; b < 3; b++)
    if (b != ax) v = M_(v, hat((c >> b) & 1, xi[b]));
  return v;
}

// u^T P v for symmetric packed P, fixed operation order
SPHC_HDI double form(const double* P, const double u[3], const double v[3]) {
  double r = 0.0;
  for (int p = 0; p < 3; p++) {
    double t = A_(A_(M_(sym(P, p, 0), v[0]), M_(sym(P, p, 1), v[1])), M_(sym(P, p, 2), v[2]));
    r = A_(r, M_(u[p], t));
  }
  return r;
}

// row li of the 12 x 12 curl-curl and (unit-sigma) mass blocks of one hex
SPHC_HD void edge_elem_row(const double* __restrict__ X, int n, int N, const int c[3], int li,
                              double rowS[12], double rowM[12]) {
  bool uniform = X == nullptr;
  double h = 1.0 / (double)N;
  double xc[8][3];
  if (!uniform) load_corners(X, n, c, xc);
  for (int j = 0; j < 12; j++) rowS[j] = rowM[j] = 0.0;
  int ai = LAXIS[li];
  for (int q0 = 0; q0 < 3; q0++)
    for (int q1 = 0; q1 < 3; q1++)
      for (int q2 = 0; q2 < 3; q2++) {
        double xi[3], w0, w1, w2;
        gauss3(q0, xi[0], w0);
        gauss3(q1, xi[1], w1);
        gauss3(q2, xi[2], w2);
        Geo g;
        geometry(xc, uniform, h, xi, M_(M_(w0, w1), w2), g);
        double ci[3], si = ref_shape2(li, xi);
        ref_curl(li, xi, ci);
        for (int j = 0; j < 12; j++) {
          double cj[3];
          ref_curl(j, xi, cj);
          double sj = ref_shape2(j, xi);
          int aj = LAXIS[j];
          // (lo, hi) roles by local index -> bitwise symmetric blocks
          double sv = j < li ? form(g.H, cj, ci) : form(g.H, ci, cj);
          double mv = j < li ? M_(sym(g.G, aj, ai), M_(sj, si)) : M_(sym(g.G, ai, aj), M_(si, sj));
          rowS[j] = A_(rowS[j], sv);
          rowM[j] = A_(rowM[j], mv);
        }
      }
}

// row a of the 8 x 8 trilinear stiffness and mass blocks of one hex
SPHC_HD void node_elem_row(const double* __restrict__ X, int n, int N, const int c[3], int a,
                              double rowK[8], double rowM[8]) {
  bool uniform = X == nullptr;
  double h = 1.0 / (double)N;
  double xc[8][3];
  if (!uniform) load_corners(X, n, c, xc);
  for (int b = 0; b < 8; b++) rowK[b] = rowM[b] = 0.0;
  for (int q0 = 0; q0 < 3; q0++)
    for (int q1 = 0; q1 < 3; q1++)
      for (int q2 = 0; q2 < 3; q2++) {
        double xi[3], w0, w1, w2;
        gauss3(q0, xi[0], w0);
        gauss3(q1, xi[1], w1);
        gauss3(q2, xi[2], w2);
        Geo g;
        geometry(xc, uniform, h, xi, M_(M_(w0, w1), w2), g);
        double Nv[8], dN[8][3];
        for (int k = 0; k < 8; k++) {
          int d[3] = {k & 1, (k >> 1) & 1, (k >> 2) & 1};
          double v = 1.0;
          for (int r = 0; r < 3; r++) v = M_(v, hat(d[r], xi[r]));
          Nv[k] = v;
          for (int q = 0; q < 3; q++) {
            double t = dhat(d[q]);
            for (int r = 0; r < 3; r++)
              if (r != q) t = M_(t, hat(d[r], xi[r]));
            dN[k][q] = t;
          }
        }
        for (int b = 0; b < 8; b++) {
          double kv = b < a ? form(g.G, dN[b], dN[a]) : form(g.G, dN[a], dN[b]);
          double mv = M_(g.wdet, b < a ? M_(Nv[b], Nv[a]) : M_(Nv[a], Nv[b]));
          rowK[b] = A_(rowK[b], kv);
          rowM[b] = A_(rowM[b], mv);
        }
      }
}

SPHC_HDI void node_xyz(i64 v, int n, int t[3]) {
  t[0] = (int)(v % n);
  t[1] = (int)((v / n) % n);
  t[2] = (int)(v / ((i64)n * n));
}

SPHC_HDI bool on_boundary(const int t[3], int n) {
  return t[0] == 0 || t[1] == 0 || t[2] == 0 || t[0] == n - 1 || t[1] == n - 1 ||
         t[2] == n - 1;
}


// ---------------------------------------------------------------- topology

// edges leaving node v (by axis) and whether v is a free node
SPHC_HDI void node_counts(int N, int dirichlet, i64 v, i64* ecnt, i64* fcnt) {
  int n = N + 1;
  int t[3];
  node_xyz(v, n, t);
  bool bt = dirichlet && on_boundary(t, n);
  int c = 0;
  for (int a = 0; a < 3; a++) {
    if (t[a] >= N) continue;
    if (bt) {
      int hd[3] = {t[0], t[1], t[2]};
      hd[a]++;
      if (on_boundary(hd, n)) continue;
    }
    c++;
  }
  ecnt[v] = c;
  fcnt[v] = bt ? 0 : 1;
}

SPHC_HDI void node_tables(int N, int dirichlet, i64 v, const i64* eoff, const i64* foff,
                          int* edge_of, i64* ecode, int* fid, int* flist) {
  int n = N + 1;
  int t[3];
  node_xyz(v, n, t);
  i64 e = eoff[v];
  int k = 0;
  bool bt = dirichlet && on_boundary(t, n);
  for (int a = 0; a < 3; a++) {
    bool ok = t[a] < N;
    if (ok && bt) {
      int hd[3] = {t[0], t[1], t[2]};
      hd[a]++;
      ok = !on_boundary(hd, n);
    }
    if (ok) {
      edge_of[3 * v + a] = (int)(e + k);
      ecode[e + k] = 3 * v + a;
      k++;
    } else {
      edge_of[3 * v + a] = -1;
    }
  }
  bool fr = foff[v + 1] > foff[v];
  fid[v] = fr ? (int)foff[v] : -1;
  if (fr) flist[foff[v]] = (int)v;
}

SPHC_HDI void node_coords(int N, i64 v, const double* jitter, double* X) {
  int n = N + 1;
  double h = 1.0 / (double)N;
  int t[3];
  node_xyz(v, n, t);
  bool interior = !on_boundary(t, n);
  i64 ii = interior ? (i64)(t[0] - 1) + (i64)(N - 1) * ((t[1] - 1) + (i64)(N - 1) * (t[2] - 1))
                    : -1;
  for (int a = 0; a < 3; a++) {
    double x = M_((double)t[a], h);
    if (interior && jitter) x = A_(x, jitter[3 * ii + a]);
    X[3 * v + a] = x;
  }
}

// ---------------------------------------------------------------- edge rows

// row i of A_e = S + sigma M and S: count pass (FILL false: cnt[i]) or fill
template <bool FILL>
SPHC_HD void edge_row(int N, i64 i, const i64* ecode, const int* edge_of, const double* X,
                      const double* sig, double sig_c, const i64* rp, i64* cnt, int* col,
                      double* vA, double* vS) {
  int n = N + 1;
  i64 code = ecode[i];
  i64 tv = code / 3;
  int a = (int)(code % 3);
  int t[3];
  node_xyz(tv, n, t);
  int b1 = a == 0 ? 1 : 0, b2 = a == 2 ? 1 : 2;
  int hc[4][3], nh = 0;
  for (int o1 = -1; o1 <= 0; o1++)
    for (int o2 = -1; o2 <= 0; o2++) {
      int c[3] = {t[0], t[1], t[2]};
      c[b1] += o1;
      c[b2] += o2;
      if (c[b1] < 0 || c[b1] >= N || c[b2] < 0 || c[b2] >= N) continue;
      hc[nh][0] = c[0];
      hc[nh][1] = c[1];
      hc[nh][2] = c[2];
      nh++;
    }
  double rS[4][12], rM[4][12], sg[4];
  if (FILL) {
    for (int k = 0; k < nh; k++) {
      int d = (t[0] - hc[k][0]) + 2 * (t[1] - hc[k][1]) + 4 * (t[2] - hc[k][2]);
      edge_elem_row(X, n, N, hc[k], LOC[d][a], rS[k], rM[k]);
      i64 hid = ((i64)hc[k][0] * N + hc[k][1]) * N + hc[k][2];
      sg[k] = sig ? sig[hid] : sig_c;
    }
  }
  i64 pos = FILL ? rp[i] : 0;
  int count = 0;
  for (int oz = -1; oz <= 1; oz++)
    for (int oy = -1; oy <= 1; oy++)
      for (int ox = -1; ox <= 1; ox++) {
        int u[3] = {t[0] + ox, t[1] + oy, t[2] + oz};
        if (u[0] < 0 || u[1] < 0 || u[2] < 0 || u[0] >= n || u[1] >= n || u[2] >= n) continue;
        i64 uv = (i64)u[0] + (i64)n * (u[1] + (i64)n * u[2]);
        for (int b = 0; b < 3; b++) {
          int e = edge_of[3 * uv + b];
          if (e < 0) continue;
          bool hit = false;
          double sS = 0.0, sM = 0.0;
          for (int k = 0; k < nh; k++) {
            int d0 = u[0] - hc[k][0], d1 = u[1] - hc[k][1], d2 = u[2] - hc[k][2];
            if ((unsigned)d0 > 1u || (unsigned)d1 > 1u || (unsigned)d2 > 1u) continue;
            int lk = LOC[d0 + 2 * d1 + 4 * d2][b];
            if (lk < 0) continue;
            hit = true;
            if (FILL) {
              sS = A_(sS, rS[k][lk]);
              sM = A_(sM, M_(sg[k], rM[k][lk]));
            }
          }
          if (!hit) continue;
          if (FILL) {
            col[pos + count] = e;
            vS[pos + count] = sS;
            vA[pos + count] = A_(sS, sM);
          }
          count++;
        }
      }
  if (!FILL) cnt[i] = count;
}

// ---------------------------------------------------------------- node rows

// row r of A_n = K + sigma M_n over the free nodes
template <bool FILL>
SPHC_HD void node_row(int N, i64 r, const int* flist, const int* fid, const double* X,
                      const double* sig, double sig_c, const i64* rp, i64* cnt, int* col,
                      double* val) {
  int n = N + 1;
  i64 v = flist[r];
  int t[3];
  node_xyz(v, n, t);
  int hc[8][3], nh = 0;
  for (int ox = -1; ox <= 0; ox++)
    for (int oy = -1; oy <= 0; oy++)
      for (int oz = -1; oz <= 0; oz++) {
        int c[3] = {t[0] + ox, t[1] + oy, t[2] + oz};
        if (c[0] < 0 || c[1] < 0 || c[2] < 0 || c[0] >= N || c[1] >= N || c[2] >= N) continue;
        hc[nh][0] = c[0];
        hc[nh][1] = c[1];
        hc[nh][2] = c[2];
        nh++;
      }
  double rK[8][8], rM[8][8], sg[8];
  if (FILL) {
    for (int k = 0; k < nh; k++) {
      int d = (t[0] - hc[k][0]) + 2 * (t[1] - hc[k][1]) + 4 * (t[2] - hc[k][2]);
      node_elem_row(X, n, N, hc[k], d, rK[k], rM[k]);
      i64 hid = ((i64)hc[k][0] * N + hc[k][1]) * N + hc[k][2];
      sg[k] = sig ? sig[hid] : sig_c;
    }
  }
  i64 pos = FILL ? rp[r] : 0;
  int count = 0;
  for (int oz = -1; oz <= 1; oz++)
    for (int oy = -1; oy <= 1; oy++)
      for (int ox = -1; ox <= 1; ox++) {
        int u[3] = {t[0] + ox, t[1] + oy, t[2] + oz};
        if (u[0] < 0 || u[1] < 0 || u[2] < 0 || u[0] >= n || u[1] >= n || u[2] >= n) continue;
        i64 uv = (i64)u[0] + (i64)n * (u[1] + (i64)n * u[2]);
        int fu = fid[uv];
        if (fu < 0) continue;
        if (FILL) {
          double sK = 0.0, sM = 0.0;
          for (int k = 0; k < nh; k++) {
            int d0 = u[0] - hc[k][0], d1 = u[1] - hc[k][1], d2 = u[2] - hc[k][2];
            if ((unsigned)d0 > 1u || (unsigned)d1 > 1u || (unsigned)d2 > 1u) continue;
            int bb = d0 + 2 * d1 + 4 * d2;
            sK = A_(sK, rK[k][bb]);
            sM = A_(sM, M_(sg[k], rM[k][bb]));
          }
          col[pos + count] = fu;
          val[pos + count] = A_(sK, sM);
        }
        count++;
      }
  if (!FILL) cnt[r] = count;
}

// ---------------------------------------------------------------- gradient

template <bool FILL>
SPHC_HDI void grad_row(int N, i64 i, const i64* ecode, const int* fid, const i64* rp, i64* cnt,
                       int* col, double* val) {
  int n = N + 1;
  const i64 step[3] = {1, n, (i64)n * n};
  i64 code = ecode[i];
  i64 tv = code / 3, hv = tv + step[code % 3];
  int ft = fid[tv], fh = fid[hv];
  if (!FILL) {
    cnt[i] = (ft >= 0) + (fh >= 0);
    return;
  }
  i64 p = rp[i];
  if (ft >= 0) { col[p] = ft; val[p] = -1.0; p++; }
  if (fh >= 0) { col[p] = fh; val[p] = 1.0; }
}

}  // namespace sphc_asm
