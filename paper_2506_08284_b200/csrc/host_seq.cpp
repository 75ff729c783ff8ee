// Host C++ for the two inherently sequential, integer-only steps of the nodal
// chain: greedy aggregation and Algorithm 1. Both are order-
// dependent greedy passes whose outcome is defined by index order and tie
// rules; they run on the host on downloaded patterns / values and their
// results are uploaded. O(nnz) each.
#include <math.h>
#include <stdint.h>

#include <algorithm>
#include <vector>

#include "../../include/sphcurl.h"

typedef int64_t i64;

// nodal_amg.py:59-88. Phase 1 roots an aggregate at every node whose whole
// neighbourhood (pattern row, diagonal included) is unaggregated; phase 2
// gives each leftover the most frequent aggregate among its assigned
// neighbours (lowest id on ties; 0 when it has none).
extern "C" int sphc_host_aggregate(int64_t n, const int64_t* rp, const int32_t* ci,
                                   int64_t* memb, int64_t* n_agg_out) {
  for (i64 i = 0; i < n; i++) memb[i] = -1;
  i64 n_agg = 0;
  for (i64 i = 0; i < n; i++) {
    if (memb[i] >= 0) continue;
    bool free_nbhd = true;
    for (i64 j = rp[i]; j < rp[i + 1] && free_nbhd; j++) free_nbhd = memb[ci[j]] < 0;
    if (!free_nbhd) continue;
    for (i64 j = rp[i]; j < rp[i + 1]; j++) memb[ci[j]] = n_agg;
    memb[i] = n_agg;
    n_agg++;
  }
  std::vector<i64> own;
  for (i64 i = 0; i < n; i++) {
    if (memb[i] >= 0) continue;
    own.clear();
    for (i64 j = rp[i]; j < rp[i + 1]; j++) {
      i64 c = ci[j];
      if (c != i && memb[c] >= 0) own.push_back(memb[c]);
    }
    std::sort(own.begin(), own.end());
    i64 best = 0, best_cnt = 0;
    for (size_t a = 0; a < own.size();) {
      size_t b = a;
      while (b < own.size() && own[b] == own[a]) b++;
      i64 cnt = (i64)(b - a);
      if (cnt > best_cnt) {  // strictly greater keeps the lowest id on ties
        best_cnt = cnt;
        best = own[a];
      }
      a = b;
    }
    memb[i] = best;
  }
  *n_agg_out = n_agg;
  return SPHC_OK;
}

// coarse_gradient.py:36-103 (Algorithm 1). Ordering keys are the reference's
// lexsort keys: |P| descending, then the lower row (or column) index.
extern "C" int sphc_host_piecewise_const(int64_t m_h, int64_t m_H, const int64_t* rp,
                                         const int32_t* ci, const double* v, int n_passes,
                                         int64_t* assign, int64_t* err) {
  err[0] = 0;
  err[1] = 0;
  // column view (rows ascending within a column)
  std::vector<i64> cp(m_H + 1, 0);
  for (i64 j = 0; j < rp[m_h]; j++) cp[ci[j] + 1]++;
  for (i64 c = 0; c < m_H; c++) cp[c + 1] += cp[c];
  std::vector<i64> cur(cp.begin(), cp.end() - 1);
  struct Ent {
    double mag;
    i64 row;
  };
  std::vector<Ent> col(rp[m_h]);
  for (i64 r = 0; r < m_h; r++)
    for (i64 j = rp[r]; j < rp[r + 1]; j++) col[cur[ci[j]]++] = Ent{fabs(v[j]), r};
  i64 total = 0;
  for (i64 c = 0; c < m_H; c++) {
    i64 nz = cp[c + 1] - cp[c];
    if (nz == 0) {
      err[0] = 1;
      err[1] = c;
      return SPHC_ERR_HOST;
    }
    total += nz;
  }
  std::vector<i64> target(m_H);
  for (i64 c = 0; c < m_H; c++) {
    double t = (double)(cp[c + 1] - cp[c]) / (double)total * (double)m_h;
    i64 ti = (i64)nearbyint(t);
    target[c] = ti < 1 ? 1 : ti;
  }
  for (i64 r = 0; r < m_h; r++) assign[r] = -1;
  std::vector<Ent> cand;
  for (int pass = 0; pass < n_passes; pass++) {
    for (i64 c = 0; c < m_H; c++) {
      cand.clear();
      for (i64 j = cp[c]; j < cp[c + 1]; j++)
        if (assign[col[j].row] < 0) cand.push_back(col[j]);
      if (cand.empty()) continue;
      i64 take = (target[c] + n_passes - 1) / n_passes;
      if (take > (i64)cand.size()) take = (i64)cand.size();
      // (|P| desc, row asc) is a total order, so the first `take` of a
      // partial sort are exactly the reference's lexsort prefix
      std::partial_sort(cand.begin(), cand.begin() + take, cand.end(),
                        [](const Ent& a, const Ent& b) {
                          if (a.mag != b.mag) return a.mag > b.mag;
                          return a.row < b.row;
                        });
      for (i64 t = 0; t < take; t++) assign[cand[t].row] = c;
    }
  }
  std::vector<i64> counts(m_H, 0);
  for (i64 r = 0; r < m_h; r++)
    if (assign[r] >= 0) counts[assign[r]]++;
  std::vector<i64> left;
  for (i64 r = 0; r < m_h; r++)
    if (assign[r] < 0) left.push_back(r);
  for (i64 r : left) {
    if (rp[r + 1] == rp[r]) {
      err[0] = 2;
      err[1] = r;
      return SPHC_ERR_HOST;
    }
    bool any_claimed = false;
    for (i64 j = rp[r]; j < rp[r + 1]; j++) any_claimed |= counts[ci[j]] > 0;
    i64 best = -1;
    double bm = 0.0;
    for (i64 j = rp[r]; j < rp[r + 1]; j++) {
      if (any_claimed && counts[ci[j]] == 0) continue;
      double m = fabs(v[j]);
      if (best < 0 || m > bm || (m == bm && ci[j] < best)) {
        best = ci[j];
        bm = m;
      }
    }
    assign[r] = best;
    counts[best]++;
  }
  std::vector<i64> empty;
  for (i64 c = 0; c < m_H; c++)
    if (counts[c] == 0) empty.push_back(c);
  for (i64 c : empty) {
    i64 best = -1;
    double bm = 0.0;
    for (i64 j = cp[c]; j < cp[c + 1]; j++) {
      i64 r = col[j].row;
      if (counts[assign[r]] <= 1) continue;
      if (best < 0 || col[j].mag > bm || (col[j].mag == bm && r < best)) {
        best = r;
        bm = col[j].mag;
      }
    }
    if (best < 0) {
      err[0] = 3;
      err[1] = c;
      return SPHC_ERR_HOST;
    }
    counts[assign[best]]--;
    assign[best] = c;
    counts[c]++;
  }
  return SPHC_OK;
}
