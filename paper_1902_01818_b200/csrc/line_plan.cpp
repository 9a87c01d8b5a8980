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
  // pass 1: chunks per position
  out.cptr.assign(n + 1, 0);
  out.own.assign((size_t)3 * n, 0.0);
  out.idiag.assign(n, 0.0);
  std::atomic<int> too_long{0};
  std::atomic<long long> ent{0};
  parallel_for(n, [&](long long pa, long long pb) {
    long long e_loc = 0;
    for (long long p = pa; p < pb; ++p) {
      const int ls = out.lstart[line_of[p]];
      int e = 0;
      for_entries((int)p, [&](int q, double v) {
        ++e_loc;
        if (q >= ls && p - q <= 3) out.own[3 * p + (p - q - 1)] = v;
        else ++e;
      });
      const int c = (e + 31) / 32;
      if (c > cmax) too_long = 1;
      out.cptr[p + 1] = c;
      out.idiag[p] = 1.0 / val[dpos[row_of((int)p)]];
    }
    ent += e_loc;
  });
  if (too_long) return false;
  for (int p = 0; p < n; ++p) out.cptr[p + 1] += out.cptr[p];
  out.entries = ent;
  out.slots = (long long)out.cptr[n] * 32;
  if (out.slots >= INT_MAX) return false;
  for (int p = 0; p < n; ++p) out.C = std::max(out.C, out.cptr[p + 1] - out.cptr[p]);
  out.ccol.assign(out.slots, -1 - out.rb_max);  // padding: the always-zero shared slot
  out.cval.assign(out.slots, 0.0);
  // pass 2: fill
  parallel_for(n, [&](long long pa, long long pb) {
    for (long long p = pa; p < pb; ++p) {
      const int l = line_of[p], ls = out.lstart[l];
      const int bs = out.bstart[bundle_of_line[l]];
      long long at = (long long)out.cptr[p] * 32;
      for_entries((int)p, [&](int q, double v) {
        if (q >= ls && p - q <= 3) return;
        out.ccol[at] = q >= bs ? -1 - (q - bs) : q;
        out.cval[at] = v;
        ++at;
      });
    }
  });
  return true;
}

}  // namespace igb
