// panel_plan.cpp -- see panel_plan.h.
#include "panel_plan.h"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <cmath>
#include <thread>

namespace igb {

namespace {

int round_up_variant(int k, std::initializer_list<int> variants) {
  for (int v : variants)
    if (k <= v) return v;
  return -1;
}

// Panels of ranges that start at positions rs[0] = 0 < rs[1] < ... < rs[K] = n: B rows
// each from the range start, the last one of a range possibly shorter.
std::vector<int> panel_starts(const std::vector<int>& rs, int B) {
  std::vector<int> ps;
  for (size_t c = 0; c + 1 < rs.size(); ++c)
    for (int p = rs[c]; p < rs[c + 1]; p += B) ps.push_back(p);
  ps.push_back(rs.back());
  return ps;
}

// Completion time (in panel-times) of the ranges rs: a panel starts after its predecessor in
// the range and after the latest panel of every earlier range it reads (+ lag: such values
// are fetched one panel ahead and polled from L2).  maxref(r, lo, hi) = largest position in
// [lo, hi) row r reads, or -1.
template <class MaxRef>
double simulate_ranges(int n, int B, const std::vector<int>& rs, MaxRef maxref) {
  const double lag = 1.5;
  const std::vector<int> ps = panel_starts(rs, B);
  const int npan = (int)ps.size() - 1;
  std::vector<double> F(npan, 0.0);
  auto panel_of = [&](int q) { return (int)(std::upper_bound(ps.begin(), ps.end(), q) - ps.begin()) - 1; };
  double make = 0;
  int k = 0;
  for (size_t c = 0; c + 1 < rs.size(); ++c) {
    for (bool first = true; k < npan && ps[k] < rs[c + 1]; ++k, first = false) {
      double st = first ? 0.0 : F[k - 1];
      for (size_t e = 0; e < c; ++e) {
        int m = -1;
        for (int r = ps[k]; r < ps[k + 1]; r += 4) m = std::max(m, maxref(r, rs[e], rs[e + 1]));
        if (m >= 0) st = std::max(st, F[panel_of(m)] + lag);
      }
      F[k] = st + 1.0;
      make = std::max(make, F[k]);
    }
  }
  (void)n;
  return make;
}

}  // namespace

bool build_panel_plan(int n, const int* ptr, const int* col, const double* val, const int* dpos,
                      bool upper, int G, int W, int R, int max_clusters, PanelPlanHost& out, bool allow_kf10) {
  if (W != 16 && W != 8) return false;
  const int B = 2 * G * W;
  if (n <= 0 || (R & (R - 1)) || R < B) return false;
  out = PanelPlanHost{};
  out.n = n;
  out.B = B;
  out.G = G;
  out.W = W;
  out.R = R;
  out.KBC = B / 32 + 1;
  auto row_of = [&](int p) { return upper ? n - 1 - p : p; };
  // strict-triangle entries of position p as (position, value)
  auto for_entries = [&](int p, auto&& fn) {
    const int r = row_of(p);
    if (upper) {
      for (int j = dpos[r] + 1; j < ptr[r + 1]; ++j) fn(n - 1 - col[j], val[j]);
    } else {
      for (int j = ptr[r]; j < dpos[r]; ++j) fn(col[j], val[j]);
    }
  };

  // ranges: candidates are rows whose nearest earlier dependency is >= 2B back (patch starts
  // in patch-wise numberings); greedily add the range start that shortens the simulated
  // completion time most, up to max_clusters ranges, while it buys > 3%
  std::vector<int> rs{0, n};
  {
    std::vector<std::pair<int, int>> cand;  // (lookback, position)
    for (int p = B; p + B <= n; ++p) {
      int mx = -1;
      for_entries(p, [&](int q, double) { mx = std::max(mx, q); });
      const int lb = p - mx;
      if (mx >= 0 && lb >= 2 * B) cand.push_back({lb, p});
    }
    std::sort(cand.begin(), cand.end(), [](auto& x, auto& y) { return x.first > y.first; });
    if (cand.size() > 12) cand.resize(12);
    auto maxref = [&](int r, int lo, int hi) {
      int m = -1;
      for_entries(r, [&](int q, double) {
        if (q >= lo && q < hi) m = std::max(m, q);
      });
      return m;
    };
    double best = simulate_ranges(n, B, rs, maxref);
    const int kmax = std::max(1, std::min(max_clusters, 8));
    while ((int)rs.size() - 1 < kmax) {
      double cbest = best;
      int pick = -1;
      for (auto& c : cand) {
        if (std::find(rs.begin(), rs.end(), c.second) != rs.end()) continue;
        std::vector<int> t = rs;
        t.insert(std::upper_bound(t.begin(), t.end(), c.second), c.second);
        const double m = simulate_ranges(n, B, t, maxref);
        if (m < cbest) {
          cbest = m;
          pick = c.second;
        }
      }
      if (pick < 0 || cbest > best * 0.97) break;
      rs.insert(std::upper_bound(rs.begin(), rs.end(), pick), pick);
      best = cbest;
    }
    out.makespan = best;
  }
  out.nclu = (int)rs.size() - 1;
  out.rstart = rs;
  const std::vector<int> ps = panel_starts(rs, B);
  out.npan = (int)ps.size() - 1;
  const int npan = out.npan;
  out.split.assign(out.nclu + 1, 0);
  std::vector<int> range_of_panel(npan), panel_of(n);
  for (int k = 0, c = 0; k < npan; ++k) {
    while (ps[k] >= rs[c + 1]) ++c;
    range_of_panel[k] = c;
    for (int p = ps[k]; p < ps[k + 1]; ++p) panel_of[p] = k;
  }
  for (int c = 0; c < out.nclu; ++c)
    out.split[c] = (int)(std::lower_bound(ps.begin(), ps.end(), rs[c]) - ps.begin());
  out.split[out.nclu] = npan;
  // a ref q of a row in panel k is read from the ring iff it is in k's range and within R
  auto is_near = [&](int q, int k) { return q >= ps[k] - R && q >= rs[range_of_panel[k]]; };

  // pass 1: off-panel counts -> KA, KF
  int max_near = 0, max_far = 0;
  for (int p = 0; p < n; ++p) {
    const int k = panel_of[p], k0 = ps[k];
    int nn = 0, nf = 0;
    for_entries(p, [&](int q, double) {
      if (q >= k0) return;
      if (is_near(q, k)) ++nn; else ++nf;
    });
    max_near = std::max(max_near, nn);
    max_far = std::max(max_far, nf);
    out.near_entries += nn;
    out.far_entries += nf;
  }
  out.KA = W == 16 ? round_up_variant((max_near + 15) / 16, {2, 4, 8, 12, 14})
                   : round_up_variant((max_near + 15) / 16, {4, 8, 12, 14, 18});
  out.KF = W == 16 ? round_up_variant((max_far + 15) / 16, {0, 1, 4, 5})
                   : (allow_kf10 ? round_up_variant((max_far + 15) / 16, {0, 4, 8, 10})
                                 : round_up_variant((max_far + 15) / 16, {0, 4, 8}));
  if (W == 8 && out.KF == 10) {
    if (out.KA > 12) out.KF = -1;  // KF 10 exists with KA 12 only
    else out.KA = 12;
  }
  if (W == 16 && out.KA == 14 && out.KF != 0) out.KA = -1;  // B = 512: the KA 14 variant exists without far slots only
  // B = 256 long-row variants (interface rows of small 3-D levels: up to 279 near entries backward):
  // KA 14 with KF 0 / 4, KA 18 with KF 0
  if (W == 8 && out.KA == 14 && out.KF > 4) out.KA = -1;
  if (W == 8 && out.KA == 14 && out.KF > 0) out.KF = 4;
  if (W == 8 && out.KA == 18 && out.KF != 0) out.KA = -1;
  if (out.KF == 5 && out.KA > 8) out.KF = -1;     // KF 5 exists with KA <= 8 only
  if (out.KF == 5) out.KA = 8;
  if (out.KA < 0 || out.KF < 0) {
    if (std::getenv("IGB_VERBOSE"))
      std::fprintf(stderr, "[igb] panel plan (%s, W %d, %d ranges): max near %d, max far %d entries per row -- "
                   "beyond the kernel variants\n", upper ? "upper" : "lower", W, out.nclu, max_near, max_far);
    // cross-range references overflowed the kernel variants: one range (if that fits)
    if (out.nclu > 1) return build_panel_plan(n, ptr, col, val, dpos, upper, G, W, R, 1, out, allow_kf10);
    return false;
  }
  const int KA = out.KA, KF = out.KF, KBC = out.KBC;

  const size_t per_cta_lin = (size_t)W * KBC * 32, per_cta_ent = (size_t)W * KA * 32,
               per_cta_far = (size_t)W * KF * 32;
  out.lin.assign((size_t)npan * G * per_cta_lin, 0.0);
  out.ev.assign((size_t)npan * G * per_cta_ent, 0.0);
  out.ec.assign(out.ev.size(), 0);
  out.fv.assign((size_t)(npan + 1) * G * per_cta_far, 0.0);  // + zero panel read past the end
  out.fc.assign(out.fv.size(), -1);  // -1: padding (the kernel neither loads nor polls it)

  // pass 2 (threaded over panels): dense inverse of the diagonal block + layouts
  std::atomic<int> next{0};
  std::atomic<bool> bad{false};
  std::vector<double> ratios(npan, 0.0);
  auto worker = [&]() {
    std::vector<double> inv((size_t)B * B);
    std::vector<double> tmp(B);
    for (int k; (k = next.fetch_add(1)) < npan;) {
      const int k0 = ps[k], b = ps[k + 1] - k0;
      double tmax = 0, imax = 0;
      // row recurrence: inv[i][:] = (e_i - sum_{m<i} T_im inv[m][:]) / T_ii
      for (int i = 0; i < b; ++i) {
        std::fill(tmp.begin(), tmp.begin() + i + 1, 0.0);
        tmp[i] = 1.0;
        for_entries(k0 + i, [&](int q, double v) {
          if (q < k0) return;
          const int m = q - k0;
          const double* im = &inv[(size_t)m * B];
          for (int c = 0; c <= m; ++c) tmp[c] -= v * im[c];
          tmax = std::max(tmax, std::fabs(v));
        });
        const double d = val[dpos[row_of(k0 + i)]];
        if (!(d != 0.0)) {
          bad = true;
          return;
        }
        tmax = std::max(tmax, std::fabs(d));
        double* ii = &inv[(size_t)i * B];
        for (int c = 0; c <= i; ++c) {
          ii[c] = tmp[c] / d;
          imax = std::max(imax, std::fabs(ii[c]));
        }
      }
      ratios[k] = imax * tmax;
      for (int pq = 0; pq < B / 2; ++pq) {
        const int cta = pq % G, w = pq / G;
        const int r1 = pq, r2 = b - 1 - pq;
        const bool v1 = pq < (b + 1) / 2, v2 = pq < b / 2;
        const int len1 = v1 ? r1 + 1 : 0, len2 = v2 ? r2 + 1 : 0;
        // row r1's chunks (column j = 32c + lane), then row r2's, each zero padded to whole chunks
        double* L = &out.lin[(((size_t)k * G + cta) * W + w) * KBC * 32];
        const int nc1 = (len1 + 31) / 32;
        for (int e = 0; e < len1; ++e) L[e] = inv[(size_t)r1 * B + e];
        for (int e = 0; e < len2; ++e) L[32 * nc1 + e] = inv[(size_t)r2 * B + e];
      }
      for (int i = 0; i < b; ++i) {  // phase-A rows: contiguous chunk per CTA
        const int cta = i / (B / G), w = (i % (B / G)) / 2, h = i % 2;
        {
          const int p = k0 + i;
          int jn = 0, jf = 0;
          const size_t eb = (((size_t)k * G + cta) * W + w) * KA * 32;
          const size_t fb = (((size_t)k * G + cta) * W + w) * KF * 32;
          for_entries(p, [&](int q, double v) {
            if (q >= k0) return;
            if (is_near(q, k)) {
              const size_t at = eb + (size_t)(jn / 16) * 32 + h * 16 + jn % 16;
              out.ev[at] = v;
              out.ec[at] = q & (R - 1);
              ++jn;
            } else {
              const size_t at = fb + (size_t)(jf / 16) * 32 + h * 16 + jf % 16;
              out.fv[at] = v;
              out.fc[at] = q;
              ++jf;
            }
          });
        }
      }
    }
  };
  const int nth = std::max(1, std::min<int>(npan, (int)std::thread::hardware_concurrency()));
  std::vector<std::thread> pool;
  for (int t = 1; t < nth; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  if (bad) return false;
  for (double r : ratios) out.max_inv_ratio = std::max(out.max_inv_ratio, r);
  // destinations of every solution value: the CTAs whose phase-A rows read it from the ring
  out.xmask.assign((size_t)npan * B, 0);
  out.xcnt.assign((size_t)(npan + 1) * G, 0);
  const int chunk = B / G;
  for (int p = 0; p < n; ++p) {
    const int k = panel_of[p], k0 = ps[k];
    const unsigned short bit = (unsigned short)(1u << ((p - k0) / chunk));
    for_entries(p, [&](int q, double) {
      if (q < k0 && is_near(q, k)) out.xmask[q] |= bit;
    });
  }
  // every CTA receives at least one value of every panel: the kernel's ordering
  // argument (panel.cu) needs "sending r(t+2) implies having received x(t+1)"
  for (int k = 0; k < npan; ++k) {
    unsigned short any = 0;
    const int k0 = ps[k], b = ps[k + 1] - k0;
    for (int i = 0; i < b; ++i) any |= out.xmask[k0 + i];
    out.xmask[k0 + b - 1] |= (unsigned short)(~any & ((1u << G) - 1));
  }
  for (int q = 0; q < n; ++q)
    for (int d = 0; d < G; ++d)
      if (out.xmask[q] >> d & 1) {
        ++out.xcnt[(size_t)panel_of[q] * G + d];
        ++out.x_messages;
      }
  // bits 16..: far slots (of 16 lanes) the CTA's rows of panel k+2 use -- read by the
  // kernel when it loads panel k+2's far entries, from the count it already holds (0 when
  // panel k+2 belongs to the next range: this cluster never processes it)
  if (KF > 0) {
    std::vector<int> slots((size_t)(npan + 2) * G, 0);
    for (int p = 0; p < n; ++p) {
      const int k = panel_of[p], k0 = ps[k], cta = (p - k0) / chunk;
      int nf = 0;
      for_entries(p, [&](int q, double) { nf += (q < k0 && !is_near(q, k)); });
      int& sl = slots[(size_t)k * G + cta];
      sl = std::max(sl, (nf + 15) / 16);
    }
    for (int k = 0; k < npan; ++k)
      if (k + 2 < npan && range_of_panel[k + 2] == range_of_panel[k])
        for (int d = 0; d < G; ++d) out.xcnt[(size_t)k * G + d] |= slots[(size_t)(k + 2) * G + d] << 16;
  }
  return true;
}

}  // namespace igb
