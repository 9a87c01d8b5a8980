// level_plan.cpp -- see level_plan.h.
#include "level_plan.h"

#include <algorithm>

namespace igb {

namespace {
inline int round_up(int v, int m) { return (v + m - 1) / m * m; }
}  // namespace

bool build_level_plan(int n, const int* ptr, const int* col, const double* val, const int* dpos,
                      bool upper, int NT, int R, int kmax, LevelPlanHost& out) {
  out = LevelPlanHost();
  out.n = n;
  out.NT = NT;
  out.R = R;
  if (n <= 0) return false;
  auto dep_begin = [&](int r) { return upper ? dpos[r] + 1 : ptr[r]; };
  auto dep_end = [&](int r) { return upper ? ptr[r + 1] : dpos[r]; };

  // ---- dependency levels (sweep order: ascending rows forward, descending backward)
  std::vector<int> lv(n, 0);
  int nlev = 0, maxdeps = 0;
  for (int k = 0; k < n; ++k) {
    const int r = upper ? n - 1 - k : k;
    int l = 0;
    for (int j = dep_begin(r); j < dep_end(r); ++j) l = std::max(l, lv[col[j]] + 1);
    lv[r] = l;
    nlev = std::max(nlev, l + 1);
    maxdeps = std::max(maxdeps, dep_end(r) - dep_begin(r));
  }
  out.nlevels = nlev;
  int TPR = 1;
  while (TPR < 32 && (maxdeps + TPR - 1) / TPR > kmax) TPR *= 2;
  if ((maxdeps + TPR - 1) / TPR > kmax) return false;
  out.TPR = TPR;
  const int RPR = NT / TPR;

  // ---- level order (rows ascending inside a level) and positions
  std::vector<int> cnt(nlev + 1, 0), pos(n);
  out.rows.assign(n, 0);
  for (int r = 0; r < n; ++r) cnt[lv[r] + 1]++;
  for (int l = 0; l < nlev; ++l) cnt[l + 1] += cnt[l];
  {
    std::vector<int> fill(cnt.begin(), cnt.end() - 1);
    for (int r = 0; r < n; ++r) out.rows[fill[lv[r]]++] = r;
  }
  for (int p = 0; p < n; ++p) pos[out.rows[p]] = p;

  // ---- steps: chunks of <= RPR rows of one level
  // block: [double invd[rpra]] [double2 val[kt/2][nthr]] [int2 src[kt/2][nthr]]
  // kt = entries per thread (multiple of 2); thread i*TPR + j holds entries j, j+TPR, ...
  long long total = 0;
  for (int l = 0; l < nlev; ++l)
    for (int s = cnt[l]; s < cnt[l + 1]; s += RPR) {
      LevelMeta m{};
      m.start = s;
      m.nrows = std::min(RPR, cnt[l + 1] - s);
      int krow = 0;
      for (int i = 0; i < m.nrows; ++i) {
        const int r = out.rows[s + i];
        krow = std::max(krow, dep_end(r) - dep_begin(r));
      }
      const int kt = kmax;  // fixed-length per-thread entry lists (zero padded)
      (void)krow;
      m.K = kt;
      if (total / 16 >= (1LL << 31)) return false;
      m.off16 = (int)(total / 16);
      const long long nthr = (long long)m.nrows * TPR;
      total += 8LL * round_up(m.nrows, 2) + 8LL * kt * nthr + 4LL * kt * nthr;
      total = (total + 15) / 16 * 16;
      out.meta.push_back(m);
    }
  out.nsteps = (int)out.meta.size();
  out.stream.assign((size_t)total, 0);

  // ---- emit
  for (LevelMeta& m : out.meta) {
    unsigned char* blk = out.stream.data() + 16LL * m.off16;
    const int kt = m.K;
    const int rpra = round_up(m.nrows, 2);
    const long long nthr = (long long)m.nrows * TPR;
    double* invd = reinterpret_cast<double*>(blk);
    double* vals = reinterpret_cast<double*>(blk + 8LL * rpra);
    int* srcs = reinterpret_cast<int*>(blk + 8LL * rpra + 8LL * kt * nthr);
    const int end_pos = m.start + m.nrows;
    bool has_old = false;
    for (int i = 0; i < m.nrows; ++i) {
      const int r = out.rows[m.start + i];
      invd[i] = 1.0 / val[dpos[r]];
      int k = 0;
      for (int j = dep_begin(r); j < dep_end(r); ++j, ++k) {
        const long long th = (long long)i * TPR + (k % TPR);
        const int slot = k / TPR;
        const int pc = pos[col[j]];
        int code;
        if (pc >= end_pos - R) {
          code = pc & (R - 1);
        } else {
          code = -(pc + 1);
          ++out.global_refs;
          has_old = true;
        }
        // interleaved for coalesced 128-bit loads: double2 [slot/2][thread], int4 [slot/4][thread]
        vals[((long long)(slot / 2) * nthr + th) * 2 + (slot & 1)] = val[j];
        srcs[((long long)(slot / 2) * nthr + th) * 2 + (slot & 1)] = code;
        ++out.entries;
      }
    }
    if (has_old) out.has_old = true;
    // padding entries stay (0.0, ring slot 0): ring slot 0 always holds a finite value
  }
  return true;
}

}  // namespace igb
