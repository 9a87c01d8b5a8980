// wave_plan.cpp -- see wave_plan.h.
#include "wave_plan.h"

#include <algorithm>
#include <climits>

#include "host_par.h"

namespace igb {

bool build_wave_plan(int n, const int* ptr, const int* col, const double* val, const int* dpos, bool upper,
                     int rb_min, int rb_cap, int crit_lag, int late_max, int groups, WavePlanHost& out) {
  out = WavePlanHost{};
  out.n = n;
  if (n <= 0 || rb_cap > 65000) return false;
  constexpr int GI = WAVE_GI, KI = WAVE_KI, SP = WAVE_SP, CAPI = GI * KI;
  auto row_of = [&](int p) { return upper ? n - 1 - p : p; };
  // strict-triangle entries of position p as positions q < p
  auto for_entries = [&](int p, auto&& f) {
    const int r = row_of(p);
    if (!upper) {
      for (int k = ptr[r]; k < dpos[r]; ++k) f(col[k], val[k]);
    } else {
      for (int k = ptr[r + 1] - 1; k > dpos[r]; --k) f(n - 1 - col[k], val[k]);
    }
  };
  auto last_entry = [&](int p) {  // largest q of position p, -1 if none
    const int r = row_of(p);
    if (!upper) return dpos[r] > ptr[r] ? col[dpos[r] - 1] : -1;
    return ptr[r + 1] - 1 > dpos[r] ? n - 1 - col[dpos[r] + 1] : -1;
  };
  // lines: a new line where the row does not read its predecessor
  std::vector<int> lstart{0};
  for (int p = 1; p < n; ++p)
    if (!(last_entry(p) == p - 1 && p - lstart.back() < rb_cap)) lstart.push_back(p);
  lstart.push_back(n);
  const int nl = (int)lstart.size() - 1;
  // detached lines: no row reads the previous line
  std::vector<char> detached(nl, 1);
  parallel_for(nl, [&](long long la, long long lb) {
    for (long long l = std::max(1LL, la); l < lb; ++l) {
      const int s0 = lstart[l - 1], s1 = lstart[l];
      bool reads = false;
      for (int p = lstart[l]; p < lstart[l + 1] && !reads; ++p)
        for_entries(p, [&](int q, double) { reads |= (q >= s0 && q < s1); });
      detached[l] = reads ? 0 : 1;
    }
  }, 64);
  // bundles
  std::vector<int> bstart{0};
  {
    int rows = 0;
    for (int l = 0; l < nl; ++l) {
      const int len = lstart[l + 1] - lstart[l];
      if (len > rb_cap) return false;
      if (rows > 0 && (rows + len > rb_cap || (detached[l] && rows >= rb_min))) {
        bstart.push_back(lstart[l]);
        rows = 0;
      }
      rows += len;
    }
    bstart.push_back(n);
  }
  const int nb = out.nb = (int)bstart.size() - 1;
  std::vector<int> bundle_of(n);
  for (int b = 0; b < nb; ++b) {
    for (int p = bstart[b]; p < bstart[b + 1]; ++p) bundle_of[p] = b;
    out.rb_max = std::max(out.rb_max, bstart[b + 1] - bstart[b]);
  }
  // dependency levels: global (all entries) and inside the bundle (entries of the own bundle)
  std::vector<int> lv(n, 0), ilv(n, 0);
  int maxl = 0;
  for (int p = 0; p < n; ++p) {
    int l = 0, il = 0;
    const int bs = bstart[bundle_of[p]];
    for_entries(p, [&](int q, double) {
      l = std::max(l, lv[q] + 1);
      if (q >= bs) il = std::max(il, ilv[q] + 1);
    });
    lv[p] = l;
    ilv[p] = il;
    maxl = std::max(maxl, l);
  }
  out.nlev = maxl + 1;
  // occupancy: bundles are handed out in position order; bundle b can only start once all but
  // groups - 1 of the earlier bundles are finished, and an earlier bundle b' is certainly finished
  // before b is needed only if its last level lies below b's first
  {
    std::vector<int> mn(nb, INT_MAX), mx(nb, -1);
    for (int p = 0; p < n; ++p) {
      mn[bundle_of[p]] = std::min(mn[bundle_of[p]], lv[p]);
      mx[bundle_of[p]] = std::max(mx[bundle_of[p]], lv[p]);
    }
    // sliding check: earlier bundles sorted by position; count those with mx >= mn[b]
    for (int b = 0; b < nb; ++b) {
      int held = 1;
      for (int c = b - 1; c >= 0 && b - c <= 4 * groups + 64; --c) held += mx[c] >= mn[b];
      out.occupancy = std::max(out.occupancy, held);
    }
    if (out.occupancy > groups) return false;
  }
  // frames: per bundle, rows sorted by (in-bundle level, position), levels cut into frames of SP
  std::vector<int> slot_of(n);       // global slot of each position
  out.b_frame.assign(nb + 1, 0);
  out.b_rows.assign(nb, 0);
  {
    std::vector<int> nframes_b(nb, 0);
    parallel_for(nb, [&](long long ba, long long bb) {
      std::vector<int> cnt;
      for (long long b = ba; b < bb; ++b) {
        int ml = 0;
        for (int p = bstart[b]; p < bstart[b + 1]; ++p) ml = std::max(ml, ilv[p]);
        cnt.assign(ml + 1, 0);
        for (int p = bstart[b]; p < bstart[b + 1]; ++p) cnt[ilv[p]]++;
        int f = 0;
        for (int l = 0; l <= ml; ++l) f += (cnt[l] + SP - 1) / SP;
        nframes_b[b] = f;
      }
    }, 8);
    long long tot = 0;
    for (int b = 0; b < nb; ++b) {
      out.b_frame[b] = (int)tot;
      tot += nframes_b[b];
      out.b_rows[b] = bstart[b + 1] - bstart[b];
    }
    if (tot * SP * GI >= INT_MAX / 2) return false;
    out.b_frame[nb] = (int)tot;
    out.nframes = (int)tot;
  }
  out.slot.assign((size_t)out.nframes * SP, WaveSlot{-1, 0, 0, 0.0});
  out.recA.assign((size_t)out.nframes * SP * GI, WaveRecA{0.0, 0.0});
  out.recB.resize((size_t)out.nframes * SP * GI);
  std::vector<int> wid(nb, 0);
  parallel_for(nb, [&](long long ba, long long bb) {
    std::vector<int> cnt, start, fill;
    for (long long b = ba; b < bb; ++b) {
      const int bs = bstart[b], be = bstart[b + 1];
      int ml = 0;
      for (int p = bs; p < be; ++p) ml = std::max(ml, ilv[p]);
      cnt.assign(ml + 1, 0);
      for (int p = bs; p < be; ++p) cnt[ilv[p]]++;
      start.assign(ml + 1, 0);   // first frame of each level
      int f = out.b_frame[b];
      for (int l = 0; l <= ml; ++l) {
        start[l] = f;
        f += (cnt[l] + SP - 1) / SP;
        wid[b] = std::max(wid[b], cnt[l]);
      }
      fill.assign(ml + 1, 0);
      for (int p = bs; p < be; ++p) {  // ascending position within a level
        const int l = ilv[p], k = fill[l]++;
        slot_of[p] = (start[l] + k / SP) * SP + k % SP;
      }
      // unused lane records of the bundle read its zero slot
      const WaveRecB zb{0.0, (unsigned short)(be - bs), (unsigned short)(be - bs), (unsigned short)(be - bs), 0};
      for (size_t i = (size_t)out.b_frame[b] * SP * GI; i < (size_t)out.b_frame[b + 1] * SP * GI; ++i)
        out.recB[i] = zb;
    }
  }, 8);
  for (int b = 0; b < nb; ++b) out.max_level_rows = std::max(out.max_level_rows, wid[b]);
  // per position: internal entries (at most CAPI, the newest in-bundle levels first), the rest external
  std::vector<int> next(n, 0);  // external entry count per position
  std::vector<long long> cnt_int(1, 0), cnt_dem(1, 0);
  struct Cand { int q; double v; };
  auto split = [&](int p, std::vector<Cand>& in, auto&& ext) {
    const int bs = bstart[bundle_of[p]];
    in.clear();
    for_entries(p, [&](int q, double v) {
      if (q >= bs) in.push_back(Cand{q, v});
      else ext(q, v, false);
    });
    if ((int)in.size() > CAPI) {  // demote the oldest (lowest in-bundle level, then lowest position)
      std::sort(in.begin(), in.end(), [&](const Cand& a, const Cand& b) {
        return ilv[a.q] != ilv[b.q] ? ilv[a.q] > ilv[b.q] : a.q > b.q;
      });
      for (size_t k = CAPI; k < in.size(); ++k) ext(in[k].q, in[k].v, true);
      in.resize(CAPI);
    }
    std::sort(in.begin(), in.end(), [](const Cand& a, const Cand& b) { return a.q < b.q; });
  };
  {
    std::vector<long long> ci(64, 0), cd(64, 0);
    std::atomic<int> tix{0};
    parallel_for(n, [&](long long pa, long long pb) {
      const int me = tix++ % 64;
      std::vector<Cand> in;
      long long li = 0, ld = 0;
      for (long long p = pa; p < pb; ++p) {
        int ne = 0;
        split((int)p, in, [&](int, double, bool dem) { ++ne; ld += dem; });
        next[p] = ne;
        li += (long long)in.size();
        const int s = slot_of[p], bs = bstart[bundle_of[p]];
        WaveSlot& S = out.slot[s];
        S.row = row_of((int)p);
        S.loc = (unsigned short)(p - bs);
        S.flags = ne > 0 ? 1 : 0;
        S.idiag = 1.0 / val[dpos[row_of((int)p)]];
        for (size_t e = 0; e < in.size(); ++e) {  // entry e: lane e % GI, k = e / GI
          const size_t at = (size_t)s * GI + e % GI;
          const int k = (int)(e / GI);
          const unsigned short li16 = (unsigned short)(in[e].q - bs);
          if (k == 0) { out.recA[at].c0 = in[e].v; out.recB[at].i0 = li16; }
          else if (k == 1) { out.recA[at].c1 = in[e].v; out.recB[at].i1 = li16; }
          else { out.recB[at].c2 = in[e].v; out.recB[at].i2 = li16; }
        }
      }
      ci[me] += li;  // distinct chunks get distinct counters only by chance: totals are diagnostics
      cd[me] += ld;
    });
    for (int i = 0; i < 64; ++i) { out.internal += ci[i]; out.demoted += cd[i]; }
  }
  // external list: positions with external entries in (level, position) order
  {
    std::vector<int> cntl(out.nlev + 1, 0);
    for (int p = 0; p < n; ++p)
      if (next[p] > 0) cntl[lv[p] + 1]++;
    for (int l = 0; l < out.nlev; ++l) cntl[l + 1] += cntl[l];
    out.nq = cntl[out.nlev];
    std::vector<int> qpos(out.nq);
    {
      std::vector<int> at(cntl.begin(), cntl.end() - 1);
      for (int p = 0; p < n; ++p)
        if (next[p] > 0) qpos[at[lv[p]]++] = p;
    }
    out.e_row.resize(out.nq);
    out.eptr.assign(out.nq + 1, 0);
    long long tot = 0;
    for (int q = 0; q < out.nq; ++q) {
      out.eptr[q] = (int)tot;
      tot += next[qpos[q]];
      if (tot >= INT_MAX) return false;
    }
    out.eptr[out.nq] = (int)tot;
    out.external = tot;
    out.ecol.resize(tot);
    out.eval.resize(tot);
    out.crit.assign(out.nq, -1);
    out.elate.assign(out.nq, 0);
    parallel_for(out.nq, [&](long long qa, long long qb) {
      std::vector<Cand> in, ex;
      for (long long q = qa; q < qb; ++q) {
        const int p = qpos[q];
        out.e_row[q] = row_of(p);
        ex.clear();
        split(p, in, [&](int c, double v, bool) { ex.push_back(Cand{c, v}); });
        std::sort(ex.begin(), ex.end(), [](const Cand& a, const Cand& b) { return a.q < b.q; });
        int nlate = 0;
        for (auto& e : ex) nlate += lv[e.q] > lv[p] - crit_lag;
        if (nlate > late_max) nlate = 0;
        long long e0 = out.eptr[q], el = out.eptr[q + 1] - nlate;
        out.elate[q] = (int)el;
        int best = -1;
        for (auto& e : ex) {
          const bool late = nlate > 0 && lv[e.q] > lv[p] - crit_lag;
          const long long at = late ? el++ : e0++;
          out.ecol[at] = row_of(e.q);
          out.eval[at] = e.v;
          if (lv[e.q] > lv[p] - crit_lag) continue;
          if (best < 0 || lv[e.q] > lv[best] || (lv[e.q] == lv[best] && e.q > best)) best = e.q;
        }
        out.crit[q] = best >= 0 ? row_of(best) : -1;
      }
    });
  }
  return true;
}

}  // namespace igb
