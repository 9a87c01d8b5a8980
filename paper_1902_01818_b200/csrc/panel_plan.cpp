// panel_plan.cpp -- see panel_plan.h.
#include "panel_plan.h"

#include <algorithm>
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

}  // namespace

bool build_panel_plan(int n, const int* ptr, const int* col, const double* val, const int* dpos,
                      bool upper, int G, int R, PanelPlanHost& out) {
  const int W = 16;
  const int B = 2 * G * W;
  if (n <= 0 || (R & (R - 1)) || R < B) return false;
  out = PanelPlanHost{};
  out.n = n;
  out.B = B;
  out.G = G;
  out.W = W;
  out.R = R;
  out.KBC = B / 32 + 1;
  out.npan = (n + B - 1) / B;
  const int npan = out.npan;
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

  // pass 1: off-panel counts -> KA, KF
  int max_near = 0, max_far = 0;
  for (int p = 0; p < n; ++p) {
    const int k0 = (p / B) * B;
    int nn = 0, nf = 0;
    for_entries(p, [&](int q, double) {
      if (q >= k0) return;
      if (q >= k0 - R) ++nn; else ++nf;
    });
    max_near = std::max(max_near, nn);
    max_far = std::max(max_far, nf);
    out.near_entries += nn;
    out.far_entries += nf;
  }
  out.KA = round_up_variant((max_near + 15) / 16, {2, 4, 8, 12});
  out.KF = round_up_variant((max_far + 15) / 16, {0, 1, 4});
  if (out.KA < 0 || out.KF < 0) return false;
  const int KA = out.KA, KF = out.KF, KBC = out.KBC;

  const size_t per_cta_lin = (size_t)W * KBC * 32, per_cta_ent = (size_t)W * KA * 32,
               per_cta_far = (size_t)W * KF * 32;
  out.lin.assign((size_t)npan * G * per_cta_lin, 0.0);
  out.ev.assign((size_t)npan * G * per_cta_ent, 0.0);
  out.ec.assign(out.ev.size(), 0);
  out.fv.assign((size_t)(npan + 1) * G * per_cta_far, 0.0);  // + zero panel read past the end
  out.fc.assign(out.fv.size(), 0);

  // pass 2 (threaded over panels): dense inverse of the diagonal block + layouts
  std::atomic<int> next{0};
  std::atomic<bool> bad{false};
  std::vector<double> ratios(npan, 0.0);
  auto worker = [&]() {
    std::vector<double> inv((size_t)B * B);
    std::vector<double> tmp(B);
    for (int k; (k = next.fetch_add(1)) < npan;) {
      const int k0 = k * B, b = std::min(B, n - k0);
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
            if (q >= k0 - R) {
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
    const int k0 = (p / B) * B;
    const unsigned short bit = (unsigned short)(1u << ((p - k0) / chunk));
    for_entries(p, [&](int q, double) {
      if (q < k0 && q >= k0 - R) out.xmask[q] |= bit;
    });
  }
  // every CTA receives at least one value of every panel: the kernel's ordering
  // argument (panel.cu) needs "sending r(t+2) implies having received x(t+1)"
  for (int k = 0; k < npan; ++k) {
    unsigned short any = 0;
    const int k0 = k * B, b = std::min(B, n - k0);
    for (int i = 0; i < b; ++i) any |= out.xmask[k0 + i];
    out.xmask[k0 + b - 1] |= (unsigned short)(~any & ((1u << G) - 1));
  }
  for (int q = 0; q < n; ++q)
    for (int d = 0; d < G; ++d)
      if (out.xmask[q] >> d & 1) {
        ++out.xcnt[(size_t)(q / B) * G + d];
        ++out.x_messages;
      }
  // bits 16..: far slots (of 16 lanes) the CTA's rows of panel k+2 use -- read by the
  // kernel when it loads panel k+2's far entries, from the count it already holds
  if (KF > 0) {
    std::vector<int> slots((size_t)(npan + 2) * G, 0);
    for (int p = 0; p < n; ++p) {
      const int k = p / B, k0 = k * B, cta = (p - k0) / chunk;
      int nf = 0;
      for_entries(p, [&](int q, double) { nf += (q < k0 - R); });
      int& sl = slots[(size_t)k * G + cta];
      sl = std::max(sl, (nf + 15) / 16);
    }
    for (int k = 0; k < npan; ++k)
      for (int d = 0; d < G; ++d) out.xcnt[(size_t)k * G + d] |= slots[(size_t)(k + 2) * G + d] << 16;
  }
  return true;
}

}  // namespace igb
