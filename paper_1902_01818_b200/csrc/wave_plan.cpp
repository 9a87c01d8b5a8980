// wave_plan.cpp -- see wave_plan.h.
#include "wave_plan.h"

#include <algorithm>
#include <atomic>
#include <climits>

#include "host_par.h"

namespace igb {

bool build_wave_plan(int n, const int* ptr, const int* col, const double* val, const int* dpos, bool upper,
                     int rb_min, int rb_cap, int late_lag, int crit_lag, int late_max, int groups,
                     WavePlanHost& out) {
  out = WavePlanHost{};
  out.n = n;
  if (n <= 0 || rb_cap > 65000) return false;
  constexpr int GI = WAVE_GI, KI = WAVE_KI, SP = WAVE_SP, CAPI = GI * KI, LN = WAVE_LN;
  static_assert(KI == 3, "lane record layout holds three entries");
  auto row_of = [&](int p) { return upper ? n - 1 - p : p; };
  // strict-triangle entries of position p as positions q < p, ascending
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
  out.b_start = bstart;
  std::vector<int> bundle_of(n);
  for (int b = 0; b < nb; ++b) {
    for (int p = bstart[b]; p < bstart[b + 1]; ++p) bundle_of[p] = b;
    out.rb_max = std::max(out.rb_max, bstart[b + 1] - bstart[b]);
  }
  // levels inside the bundle (entries of the own bundle)
  std::vector<int> ilv(n, 0);
  parallel_for(nb, [&](long long ba, long long bb) {
    for (long long b = ba; b < bb; ++b) {
      const int bs = bstart[b];
      for (int p = bs; p < bstart[b + 1]; ++p) {
        int il = 0;
        for_entries(p, [&](int q, double) {
          if (q >= bs) il = std::max(il, ilv[q] + 1);
        });
        ilv[p] = il;
      }
    }
  }, 8);
  // frames: per bundle, rows sorted by (in-bundle level, position), levels cut into frames of SP;
  // sweep order u: bundle by bundle, frame by frame, slot by slot
  std::vector<int> frame_of(n), slot_of(n), u_of(n);
  out.b_frame.assign(nb + 1, 0);
  {
    std::vector<int> nframes_b(nb, 0), wid(nb, 0);
    parallel_for(nb, [&](long long ba, long long bb) {
      std::vector<int> cnt;
      for (long long b = ba; b < bb; ++b) {
        int ml = 0;
        for (int p = bstart[b]; p < bstart[b + 1]; ++p) ml = std::max(ml, ilv[p]);
        cnt.assign(ml + 1, 0);
        for (int p = bstart[b]; p < bstart[b + 1]; ++p) cnt[ilv[p]]++;
        int f = 0;
        for (int l = 0; l <= ml; ++l) {
          f += (cnt[l] + SP - 1) / SP;
          wid[b] = std::max(wid[b], cnt[l]);
        }
        nframes_b[b] = f;
      }
    }, 8);
    long long tot = 0;
    for (int b = 0; b < nb; ++b) {
      out.b_frame[b] = (int)tot;
      tot += nframes_b[b];
      out.max_level_rows = std::max(out.max_level_rows, wid[b]);
    }
    if (tot * SP * GI >= INT_MAX / 2) return false;
    out.b_frame[nb] = (int)tot;
    out.nframes = (int)tot;
    parallel_for(nb, [&](long long ba, long long bb) {
      std::vector<int> cnt, start, ustart, fill;
      for (long long b = ba; b < bb; ++b) {
        const int bs = bstart[b], be = bstart[b + 1];
        int ml = 0;
        for (int p = bs; p < be; ++p) ml = std::max(ml, ilv[p]);
        cnt.assign(ml + 1, 0);
        for (int p = bs; p < be; ++p) cnt[ilv[p]]++;
        start.assign(ml + 1, 0);   // first frame of each level
        ustart.assign(ml + 1, 0);  // first sweep index of each level
        int f = out.b_frame[b], u = bs;
        for (int l = 0; l <= ml; ++l) {
          start[l] = f;
          ustart[l] = u;
          f += (cnt[l] + SP - 1) / SP;
          u += cnt[l];
        }
        fill.assign(ml + 1, 0);
        for (int p = bs; p < be; ++p) {  // ascending position within a level
          const int l = ilv[p], k = fill[l]++;
          frame_of[p] = start[l] + k / SP;
          slot_of[p] = k % SP;
          u_of[p] = ustart[l] + k;
        }
      }
    }, 8);
  }
  // schedule levels: frames of a bundle run in order; key(f) = 1 + the highest key f reads or follows
  std::vector<int> alv(n, 0);
  out.f_key.assign(out.nframes, 0);
  out.f_end.assign(out.nframes, 0);
  {
    std::vector<int> by_u(n);  // position of sweep index u
    for (int p = 0; p < n; ++p) by_u[u_of[p]] = p;
    int maxk = 0;
    for (int b = 0; b < nb; ++b) {
      int u = bstart[b];
      for (int f = out.b_frame[b]; f < out.b_frame[b + 1]; ++f) {
        int key = f > out.b_frame[b] ? out.f_key[f - 1] + 1 : 0;
        const int u0 = u;
        while (u < bstart[b + 1] && frame_of[by_u[u]] == f) {
          for_entries(by_u[u], [&](int q, double) { key = std::max(key, alv[q] + 1); });
          ++u;
        }
        out.f_key[f] = key;
        out.f_end[f] = u - bstart[b];
        for (int v = u0; v < u; ++v) alv[by_u[v]] = key;
        maxk = std::max(maxk, key);
      }
    }
    out.nlev = maxk + 1;
  }
  // occupancy: bundles are handed out in position order; when bundle b must start (key of its first
  // frame) every earlier bundle whose last frame has a key >= that may still be held by a group
  {
    std::vector<int> fen(out.nlev + 2, 0);
    auto add = [&](int l) { for (int i = l + 1; i <= out.nlev + 1; i += i & -i) fen[i]++; };
    auto below = [&](int l) { int sum = 0; for (int i = l; i > 0; i -= i & -i) sum += fen[i]; return sum; };  // mx < l
    for (int b = 0; b < nb; ++b) {
      const int mn = out.f_key[out.b_frame[b]], mx = out.f_key[out.b_frame[b + 1] - 1];
      out.occupancy = std::max(out.occupancy, 1 + b - below(mn));
      add(mx);
    }
    if (out.occupancy > groups) return false;
  }
  // classification of a position's entries: internal (own bundle, at most CAPI, the newest
  // in-bundle levels first), late (other entries produced fewer than late_lag levels ago, at most
  // LN, the newest first), external (the rest)
  struct Cand { int q; double v; };
  struct Split { std::vector<Cand> in, late, ext, tmp; };
  auto split = [&](int p, Split& S) {
    const int bs = bstart[bundle_of[p]];
    S.in.clear(); S.late.clear(); S.ext.clear(); S.tmp.clear();
    int demoted = 0;
    for_entries(p, [&](int q, double v) { (q >= bs ? S.in : S.tmp).push_back(Cand{q, v}); });
    if ((int)S.in.size() > CAPI) {  // demote the oldest (lowest in-bundle level, then lowest position)
      std::sort(S.in.begin(), S.in.end(), [&](const Cand& a, const Cand& b) {
        return ilv[a.q] != ilv[b.q] ? ilv[a.q] > ilv[b.q] : a.q > b.q;
      });
      demoted = (int)S.in.size() - CAPI;
      S.tmp.insert(S.tmp.end(), S.in.begin() + CAPI, S.in.end());
      S.in.resize(CAPI);
    }
    std::sort(S.in.begin(), S.in.end(), [](const Cand& a, const Cand& b) { return a.q < b.q; });
    // newest first
    std::sort(S.tmp.begin(), S.tmp.end(), [&](const Cand& a, const Cand& b) {
      return alv[a.q] != alv[b.q] ? alv[a.q] > alv[b.q] : a.q > b.q;
    });
    for (auto& c : S.tmp) {
      if ((int)S.late.size() < LN && alv[c.q] > alv[p] - late_lag) S.late.push_back(c);
      else S.ext.push_back(c);
    }
    std::sort(S.late.begin(), S.late.end(), [](const Cand& a, const Cand& b) { return a.q < b.q; });
    std::sort(S.ext.begin(), S.ext.end(), [](const Cand& a, const Cand& b) { return a.q < b.q; });
    return demoted;
  };
  out.hdr.assign(n, WaveHdr{-1, 0, 0, 0.0});
  out.lcol.assign((size_t)n * LN, -1);
  out.lval.assign((size_t)n * LN, 0.0);
  out.recA.assign((size_t)out.nframes * SP * GI, WaveRecA{0.0, 0.0});
  out.recB.resize((size_t)out.nframes * SP * GI);
  parallel_for(nb, [&](long long ba, long long bb) {  // unused lane records read the bundle's zero slot
    for (long long b = ba; b < bb; ++b) {
      const unsigned short z = (unsigned short)(bstart[b + 1] - bstart[b]);
      const WaveRecB zb{0.0, z, z, z, 0};
      for (size_t i = (size_t)out.b_frame[b] * SP * GI; i < (size_t)out.b_frame[b + 1] * SP * GI; ++i)
        out.recB[i] = zb;
    }
  }, 8);
  std::vector<int> next(n, 0);  // external entry count per position
  {
    std::vector<long long> ci(64, 0), cd(64, 0), cl(64, 0);
    std::atomic<int> tix{0};
    parallel_for(n, [&](long long pa, long long pb) {
      const int me = tix++ % 64;
      Split S;
      for (long long p = pa; p < pb; ++p) {
        cd[me] += split((int)p, S);
        ci[me] += (long long)S.in.size();
        cl[me] += (long long)S.late.size();
        next[p] = (int)S.ext.size();
        const int bs = bstart[bundle_of[p]], u = u_of[p];
        WaveHdr& H = out.hdr[u];
        H.row = row_of((int)p);
        H.loc = (unsigned short)(p - bs);
        H.flags = S.ext.empty() ? 0 : 1;
        H.idiag = 1.0 / val[dpos[row_of((int)p)]];
        for (size_t e = 0; e < S.late.size(); ++e) {
          out.lcol[(size_t)u * LN + e] = row_of(S.late[e].q);
          out.lval[(size_t)u * LN + e] = S.late[e].v;
        }
        const size_t s = (size_t)frame_of[p] * SP + slot_of[p];
        const unsigned short ord = (unsigned short)(1 + (u - bs) % WAVE_RQ);
        for (int gl = 0; gl < GI; ++gl) out.recB[s * GI + gl].ord = ord;
        for (size_t e = 0; e < S.in.size(); ++e) {  // entry e: lane e % GI, k = e / GI
          const size_t at = s * GI + e % GI;
          const int k = (int)(e / GI);
          const unsigned short li16 = (unsigned short)(S.in[e].q - bs);
          if (k == 0) { out.recA[at].c0 = S.in[e].v; out.recB[at].i0 = li16; }
          else if (k == 1) { out.recA[at].c1 = S.in[e].v; out.recB[at].i1 = li16; }
          else { out.recB[at].c2 = S.in[e].v; out.recB[at].i2 = li16; }
        }
      }
    });
    for (int i = 0; i < 64; ++i) { out.internal += ci[i]; out.demoted += cd[i]; out.late += cl[i]; }
  }
  // external list: positions with external entries in (schedule level, position) order
  {
    std::vector<int> cntl(out.nlev + 1, 0);
    for (int p = 0; p < n; ++p)
      if (next[p] > 0) cntl[alv[p] + 1]++;
    for (int l = 0; l < out.nlev; ++l) cntl[l + 1] += cntl[l];
    out.nq = cntl[out.nlev];
    std::vector<int> qpos(out.nq);
    {
      std::vector<int> at(cntl.begin(), cntl.end() - 1);
      for (int p = 0; p < n; ++p)
        if (next[p] > 0) qpos[at[alv[p]]++] = p;
    }
    out.e_row.resize(out.nq);
    out.e_key.resize(out.nq);
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
      Split S;
      for (long long q = qa; q < qb; ++q) {
        const int p = qpos[q];
        out.e_row[q] = row_of(p);
        out.e_key[q] = alv[p];
        split(p, S);
        int nlate = 0;
        for (auto& e : S.ext) nlate += alv[e.q] > alv[p] - crit_lag;
        if (nlate > late_max) nlate = 0;
        long long e0 = out.eptr[q], el = out.eptr[q + 1] - nlate;
        out.elate[q] = (int)el;
        int best = -1;
        for (auto& e : S.ext) {
          const bool late = nlate > 0 && alv[e.q] > alv[p] - crit_lag;
          const long long at = late ? el++ : e0++;
          out.ecol[at] = row_of(e.q);
          out.eval[at] = e.v;
          if (alv[e.q] > alv[p] - crit_lag) continue;
          if (best < 0 || alv[e.q] > alv[best] || (alv[e.q] == alv[best] && e.q > best)) best = e.q;
        }
        out.crit[q] = best >= 0 ? row_of(best) : -1;
      }
    });
  }
  return true;
}

}  // namespace igb
