// flow_plan.cpp -- see flow_plan.h.
#include "flow_plan.h"
#include "host_par.h"

#include <algorithm>
#include <climits>

namespace igb {

bool build_flow_plan(int n, const int* ptr, const int* col, const double* val, const int* dpos, bool upper,
                     int G, int crit_lag, int late_max, FlowPlanHost& out) {
  out = FlowPlanHost{};
  out.n = n;
  std::vector<int> lv(n, 0);
  long long ent = 0;
  int maxl = -1;
  auto lo = [&](int i) { return upper ? dpos[i] + 1 : ptr[i]; };
  auto hi = [&](int i) { return upper ? ptr[i + 1] : dpos[i]; };
  for (int t = 0; t < n; ++t) {
    const int i = upper ? n - 1 - t : t;
    int l = 0;
    for (int k = lo(i); k < hi(i); ++k) l = std::max(l, lv[col[k]] + 1);
    lv[i] = l;
    maxl = std::max(maxl, l);
    ent += hi(i) - lo(i);
  }
  if (ent > INT_MAX) return false;
  if (G <= 0) {
    const double mean = n ? double(ent) / n : 0.0;
    G = mean <= 24.0 ? 8 : mean <= 56.0 ? 16 : 32;
  }
  const int rpw = 32 / G;
  out.G = G;
  out.nlev = maxl + 1;
  std::vector<int> cnt(out.nlev + 1, 0);
  for (int i = 0; i < n; ++i) cnt[lv[i] + 1]++;
  std::vector<long long> start(out.nlev + 1, 0);  // padded slot offsets per level
  for (int l = 0; l < out.nlev; ++l) start[l + 1] = start[l] + (cnt[l + 1] + rpw - 1) / rpw * rpw;
  if (start[out.nlev] > INT_MAX - 1) return false;
  out.nq = (int)start[out.nlev];
  out.row.assign(out.nq, -1);
  std::vector<long long> pos(start.begin(), start.end() - 1);
  for (int i = 0; i < n; ++i) out.row[pos[lv[i]]++] = i;  // ascending rows within a level
  out.qlev.resize(out.nq);
  for (int l = 0; l < out.nlev; ++l)
    for (long long q = start[l]; q < start[l + 1]; ++q) out.qlev[q] = l;
  out.eptr.assign(out.nq + 1, 0);
  out.idiag.assign(out.nq, 0.0);
  out.crit.assign(out.nq, -1);
  out.ecol.resize(ent);
  out.eval.resize(ent);
  for (int q = 0; q < out.nq; ++q) {
    const int i = out.row[q];
    out.eptr[q + 1] = out.eptr[q] + (i >= 0 ? hi(i) - lo(i) : 0);
  }
  out.elate.assign(out.nq, 0);
  parallel_for(out.nq, [&](long long qa, long long qb) {
    for (long long q = qa; q < qb; ++q) {
      const int i = out.row[q];
      if (i < 0) {
        out.elate[q] = out.eptr[q];
        continue;
      }
      int best = -1, nlate = 0;
      for (int k = lo(i); k < hi(i); ++k) nlate += lv[col[k]] > lv[i] - crit_lag;
      if (nlate > late_max) nlate = 0;  // too many newest values: one batch as before
      // early entries first (row order), then the late ones (row order)
      long long e = out.eptr[q], el = out.eptr[q + 1] - nlate;
      out.elate[q] = (int)el;
      for (int k = lo(i); k < hi(i); ++k) {
        const int c = col[k];
        const bool late = nlate > 0 && lv[c] > lv[i] - crit_lag;
        const long long at = late ? el++ : e++;
        out.ecol[at] = c;
        out.eval[at] = val[k];
        // latest-finishing dependency at least crit_lag levels back: highest level, then latest
        // in the list (upper: lowest row)
        if (lv[c] > lv[i] - crit_lag) continue;
        if (best < 0 || lv[c] > lv[best] || (lv[c] == lv[best] && (upper ? c < best : c > best))) best = c;
      }
      out.crit[q] = best;
      out.idiag[q] = 1.0 / val[dpos[i]];
    }
  });
  out.entries = ent;
  return true;
}

}  // namespace igb
