// line_plan.cpp -- see line_plan.h.
#include "line_plan.h"

#include <algorithm>
#include <atomic>
#include <climits>

#include "host_par.h"

namespace igb {

bool build_line_plan(int n, const int* ptr, const int* col, const double* val, const int* dpos, bool upper,
                     int rb_min, int rb_cap, int cmax, LinePlanHost& out) {
  out = LinePlanHost{};
  out.n = n;
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
  out.lstart.push_back(0);
  for (int p = 1; p < n; ++p) {
    const bool attached = last_entry(p) == p - 1 && p - out.lstart.back() < rb_cap;
    if (!attached) out.lstart.push_back(p);
  }
  out.lstart.push_back(n);
  out.nl = (int)out.lstart.size() - 1;
  std::vector<int> line_of(n);
  for (int l = 0; l < out.nl; ++l) {
    for (int p = out.lstart[l]; p < out.lstart[l + 1]; ++p) line_of[p] = l;
    out.max_line = std::max(out.max_line, out.lstart[l + 1] - out.lstart[l]);
  }
  if (out.max_line > rb_cap) return false;
  // detached lines: no row reads the previous line
  std::vector<char> detached(out.nl, 1);
  parallel_for(out.nl, [&](long long la, long long lb) {
    for (long long l = std::max(1LL, la); l < lb; ++l) {
      const int s0 = out.lstart[l - 1], s1 = out.lstart[l];
      bool reads = false;
      for (int p = out.lstart[l]; p < out.lstart[l + 1] && !reads; ++p)
        for_entries(p, [&](int q, double) { reads |= (q >= s0 && q < s1); });
      detached[l] = reads ? 0 : 1;
    }
  }, 64);
  // bundles
  out.bstart.push_back(0);
  out.bline.push_back(0);
  int rows = 0;
  for (int l = 0; l < out.nl; ++l) {
    const int len = out.lstart[l + 1] - out.lstart[l];
    if (rows > 0 && (rows + len > rb_cap || (detached[l] && rows >= rb_min))) {
      out.bstart.push_back(out.lstart[l]);
      out.bline.push_back(l);
      rows = 0;
    }
    rows += len;
  }
  out.bstart.push_back(n);
  out.bline.push_back(out.nl);
  out.nb = (int)out.bstart.size() - 1;
  std::vector<int> bundle_of_line(out.nl);
  for (int b = 0; b < out.nb; ++b) {
    for (int l = out.bline[b]; l < out.bline[b + 1]; ++l) bundle_of_line[l] = b;
    out.rb_max = std::max(out.rb_max, out.bstart[b + 1] - out.bstart[b]);
  }
  // dependency levels (positions)
  std::vector<int> lv(n, 0);
  for (int p = 0; p < n; ++p) {
    int l = 0;
    for_entries(p, [&](int q, double) { l = std::max(l, lv[q] + 1); });
    lv[p] = l;
  }
  // late entries: not own-recent, produced in the last LINE_LATE_LAG dependency levels; at most
  // LINE_LATE (the newest levels, then the highest positions), ordered oldest first
  auto is_own = [&](long long p, int q, int ls) { return q >= ls && p - q <= 3; };
  auto pick_late = [&](long long p, int ls, int* late) {
    int nl = 0;
    for (int j = 0; j < LINE_LATE; ++j) late[j] = -1;
    auto newer = [&](int a, int b) { return lv[a] != lv[b] ? lv[a] > lv[b] : a > b; };
    for_entries((int)p, [&](int q, double) {
      if (is_own(p, q, ls) || lv[q] < lv[p] - LINE_LATE_LAG) return;
      if (nl < LINE_LATE) {
        late[nl++] = q;
      } else {  // replace the oldest kept one if q is newer
        int m = 0;
        for (int j = 1; j < LINE_LATE; ++j)
          if (newer(late[m], late[j])) m = j;
        if (newer(q, late[m])) late[m] = q;
      }
    });
    std::sort(late, late + nl, [&](int a, int b) { return newer(b, a); });  // oldest first
    return nl;
  };
  // pass 1: chunks per position
  std::vector<int> nch(n, 0);
  std::atomic<long long> ent{0};
  parallel_for(n, [&](long long pa, long long pb) {
    long long e_loc = 0;
    for (long long p = pa; p < pb; ++p) {
      const int ls = out.lstart[line_of[p]];
      int late[LINE_LATE];
      const int nl = pick_late(p, ls, late);
      int e = 0;
      for_entries((int)p, [&](int q, double) {
        ++e_loc;
        if (!is_own(p, q, ls)) ++e;
      });
      nch[p] = (e - nl + 31) / 32;
    }
    ent += e_loc;
  });
  out.entries = ent;
  for (int p = 0; p < n; ++p) out.cmax = std::max(out.cmax, nch[p]);
  out.C = out.cmax <= 2 ? 2 : out.cmax <= 4 ? 4 : 6;
  if (cmax > 0 && out.C > cmax) out.C = cmax;
  const int C = out.C;
  std::vector<long long> optr(n + 1, 0);
  for (int p = 0; p < n; ++p) {
    optr[p + 1] = optr[p] + std::max(0, nch[p] - C);
    out.chunks += nch[p];
    out.ovf_rows += nch[p] > C;
  }
  if (optr[n] * 32 >= INT_MAX) return false;
  const size_t rb = line_rec_bytes(C);
  out.rec.assign(n * rb / 8, 0.0);
  out.ocol.assign(optr[n] * 32, -1 - out.rb_max);
  out.oval.assign(optr[n] * 32, 0.0);
  // pass 2: records
  parallel_for(n, [&](long long pa, long long pb) {
    for (long long p = pa; p < pb; ++p) {
      char* r = reinterpret_cast<char*>(out.rec.data()) + p * rb;
      int* cc = reinterpret_cast<int*>(r);
      double* cv = reinterpret_cast<double*>(r + line_off_cv(C));
      int* meta = reinterpret_cast<int*>(r + line_off_meta(C));
      double* lvv = reinterpret_cast<double*>(r + line_off_lv(C));
      double* own = reinterpret_cast<double*>(r + line_off_own(C));
      for (int i = 0; i < 32 * C; ++i) cc[i] = -1 - out.rb_max;
      for (int j = 0; j < LINE_LATE; ++j) meta[j] = -1 - out.rb_max;
      meta[LINE_LATE] = (int)optr[p];
      meta[LINE_LATE + 1] = (int)(optr[p + 1] - optr[p]);
      const int l = line_of[p], ls = out.lstart[l];
      const int bs = out.bstart[bundle_of_line[l]];
      int late[LINE_LATE];
      pick_late(p, ls, late);
      int e = 0;
      for_entries((int)p, [&](int q, double v) {
        if (is_own(p, q, ls)) {
          own[p - q - 1] = v;
          return;
        }
        const int code = q >= bs ? -1 - (q - bs) : q;
        for (int j = 0; j < LINE_LATE; ++j)
          if (late[j] == q) {
            meta[j] = code;
            lvv[j] = v;
            return;
          }
        if (e < 32 * C) {
          cc[e] = code;
          cv[e] = v;
        } else {
          const long long at = optr[p] * 32 + (e - 32 * C);
          out.ocol[at] = code;
          out.oval[at] = v;
        }
        ++e;
      });
      own[3] = 1.0 / val[dpos[row_of((int)p)]];
    }
  });
  return true;
}

}  // namespace igb
