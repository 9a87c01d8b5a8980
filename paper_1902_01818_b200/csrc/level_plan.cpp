// level_plan.cpp -- see level_plan.h.
#include "level_plan.h"

#include <algorithm>
#include <cstring>

namespace igb {

namespace {
inline int round_up(int v, int m) { return (v + m - 1) / m * m; }
}  // namespace

bool build_level_plan(int n, const int* ptr, const int* col, const double* val, const int* dpos,
                      bool upper, int NT, int R, int D, int G, int chunk_target, LevelPlanHost& out) {
  out = LevelPlanHost();
  out.n = n;
  out.NT = NT;
  out.R = R;
  out.D = D;
  out.G = G;
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
  while (TPR < 16 && (maxdeps + TPR - 1) / TPR > 16) TPR *= 2;
  out.TPR = TPR;
  const int RPR = NT / TPR;

  // ---- level order (rows ascending inside a level) and positions
  std::vector<int> cnt(nlev + 1, 0), order(n), pos(n);
  for (int r = 0; r < n; ++r) cnt[lv[r] + 1]++;
  for (int l = 0; l < nlev; ++l) cnt[l + 1] += cnt[l];
  {
    std::vector<int> fill(cnt.begin(), cnt.end() - 1);
    for (int r = 0; r < n; ++r) order[fill[lv[r]]++] = r;
  }
  for (int p = 0; p < n; ++p) pos[order[p]] = p;

  // ---- steps: chunks of <= RPR rows of one level
  struct Step {
    int start, nrows, K, ng, nta, bytes;
    long long off;
  };
  std::vector<Step> steps;
  for (int l = 0; l < nlev; ++l)
    for (int s = cnt[l]; s < cnt[l + 1]; s += RPR) {
      Step st{};
      st.start = s;
      st.nrows = std::min(RPR, cnt[l + 1] - s);
      steps.push_back(st);
    }
  const int T = (int)steps.size();
  out.nsteps = T;
  std::vector<int> step_of_pos(n);
  for (int t = 0; t < T; ++t)
    for (int i = 0; i < steps[t].nrows; ++i) step_of_pos[steps[t].start + i] = t;

  // ---- sizes; validate that every gathered value is at least G+1 steps old
  long long total = 0;
  for (int t = 0; t < T; ++t) {
    Step& st = steps[t];
    const int end_pos = st.start + st.nrows;
    int K = 0, ng = 0;
    for (int i = 0; i < st.nrows; ++i) {
      const int r = order[st.start + i];
      const int d = dep_end(r) - dep_begin(r);
      K = std::max(K, ((d + TPR - 1) / TPR + 3) & ~3);  // padded to a multiple of 4
      for (int j = dep_begin(r); j < dep_end(r); ++j) {
        const int pc = pos[col[j]];
        if (pc >= end_pos - R) continue;  // ring
        if (step_of_pos[pc] > t - G - 1) return false;
        ++ng;
      }
    }
    st.K = K;
    st.ng = ng;
    st.nta = round_up(st.nrows * TPR, 32);
    const int rpra = round_up(st.nrows, 4);
    const int nga = round_up(ng, 4);
    st.bytes = 32 + 12 * rpra + 12 * K * st.nta + 4 * nga;
    if (K > 16) return false;  // kernel unrolls at most 16 entries per thread
    st.off = total;
    total += st.bytes;
    out.max_bytes = std::max(out.max_bytes, st.bytes);
    out.max_ng = std::max(out.max_ng, nga);
    out.max_rows = std::max(out.max_rows, rpra);
  }
  out.max_ng = std::max(out.max_ng, 4);
  out.max_rows = std::max(out.max_rows, 4);
  // chunks of consecutive blocks, one TMA bulk copy each
  std::vector<int> chunk_of(T);
  {
    long long cur = 0;
    int c = 0;
    out.chunk_off.push_back(0);
    for (int t = 0; t < T; ++t) {
      if (cur > 0 && cur + steps[t].bytes > chunk_target) {
        out.chunk_off.push_back(steps[t].off);
        out.chunk_bytes = std::max(out.chunk_bytes, (int)cur);
        cur = 0;
        ++c;
      }
      chunk_of[t] = c;
      cur += steps[t].bytes;
    }
    out.chunk_bytes = std::max(out.chunk_bytes, (int)cur);
    out.chunk_off.push_back(total);
    out.nchunks = c + 1;
  }
  out.stream.assign((size_t)total, 0);
  const int GS = G + 2;
  const long long slot_stride = 2LL * out.max_ng + 2LL * out.max_rows;  // doubles per gather slot

  // ---- emit
  for (int t = 0; t < T; ++t) {
    const Step& st = steps[t];
    unsigned char* blk = out.stream.data() + st.off;
    const int rpra = round_up(st.nrows, 4);
    int* hdr = reinterpret_cast<int*>(blk);
    hdr[0] = st.K;
    hdr[1] = st.nrows;
    hdr[2] = st.ng;
    hdr[3] = st.start;
    hdr[4] = st.bytes;
    hdr[5] = st.nta;
    hdr[6] = (t + 1 == T || chunk_of[t + 1] != chunk_of[t]) ? 1 : 0;
    hdr[7] = 0;
    int* rows = reinterpret_cast<int*>(blk + 32);
    double* invd = reinterpret_cast<double*>(blk + 32 + 4 * rpra);
    double* vals = reinterpret_cast<double*>(blk + 32 + 12 * rpra);
    int* srcs = reinterpret_cast<int*>(blk + 32 + 12 * rpra + 8 * st.K * st.nta);
    int* gsrc = reinterpret_cast<int*>(blk + 32 + 12 * rpra + 12 * st.K * st.nta);
    const int end_pos = st.start + st.nrows;
    const long long gbase = (long long)R + (long long)(t % GS) * slot_stride;
    for (int i = 0; i < st.K * st.nta; ++i) {
      vals[i] = 0.0;
      srcs[i] = 0;   // padding: coefficient 0 against ring slot 0 (always finite)
    }
    int ng = 0;
    for (int i = 0; i < st.nrows; ++i) {
      const int r = order[st.start + i];
      rows[i] = r;
      invd[i] = 1.0 / val[dpos[r]];
      int k = 0;
      for (int j = dep_begin(r); j < dep_end(r); ++j, ++k) {
        const int tid = i * TPR + (k % TPR);
        const int slot = k / TPR;
        const int pc = pos[col[j]];
        long long code;
        if (pc >= end_pos - R) {
          code = pc & (R - 1);
        } else {
          gsrc[ng] = col[j];
          code = gbase + 2LL * ng + (col[j] & 1);
          ++ng;
        }
        vals[slot * st.nta + tid] = val[j];
        srcs[slot * st.nta + tid] = (int)code;
        ++out.entries;
      }
    }
    for (int i = st.nrows; i < rpra; ++i) {
      rows[i] = 0;
      invd[i] = 0.0;
    }
  }
  return true;
}

}  // namespace igb
