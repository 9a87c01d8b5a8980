// Host emulation of the wave sweep (wave.cu) on a plan from build_wave_plan, with the kernel's
// resources: `groups` compute groups taking bundles by ticket and sweeping them frame by frame,
// `ewarps` external warps walking their round-robin share of the external list in order.  Every
// actor advances only when what it reads has been produced; the emulation fails if nobody can
// advance (a deadlock of the schedule) and otherwise must reproduce the substitution.
// Built by tests/test_wave_plan.py with g++ (no CUDA).
#include <cmath>
#include <cstdio>
#include <vector>

#include "wave_plan.h"

using namespace igb;

extern "C" int wave_plan_emulate(int n, const int* ptr, const int* col, const double* val, const int* dpos, int upper,
                                 int rb_min, int rb_cap, int late_lag, int groups, int ewarps, const double* rhs,
                                 double* x, int* stats) {
  WavePlanHost P;
  if (!build_wave_plan(n, ptr, col, val, dpos, upper != 0, rb_min, rb_cap, late_lag, 4, 32, groups, P)) {
    stats[0] = P.nb;
    stats[1] = P.occupancy;
    return 1;
  }
  constexpr int SP = WAVE_SP, GI = WAVE_GI, LN = WAVE_LN;
  std::vector<char> done(n, 0), edone(n, 0);
  std::vector<double> ext(n, 0.0);
  // per group: bundle, frame, shared vector
  struct Group { int b = -1, f = 0, u = 0; std::vector<double> xs; bool finished = false; };
  std::vector<Group> G(groups);
  int ticket = 0;
  std::vector<long long> epos(ewarps);
  for (int w = 0; w < ewarps; ++w) epos[w] = w;
  long long remaining = n, used = 0;
  // frame keys must increase inside a bundle and the external list must be sorted by key
  for (int b = 0; b < P.nb; ++b)
    for (int f = P.b_frame[b] + 1; f < P.b_frame[b + 1]; ++f)
      if (P.f_key[f] <= P.f_key[f - 1]) return 8;
  for (int q = 1; q < P.nq; ++q)
    if (P.e_key[q] < P.e_key[q - 1]) return 9;
  while (remaining > 0) {
    bool progress = false;
    for (int w = 0; w < ewarps; ++w) {   // external warps
      while (epos[w] < P.nq) {
        const long long q = epos[w];
        bool ready = true;
        for (int k = P.eptr[q]; k < P.eptr[q + 1] && ready; ++k) ready = done[P.ecol[k]];
        if (P.crit[q] >= 0 && !done[P.crit[q]]) ready = false;
        if (!ready) break;
        double acc = 0.0;
        for (int k = P.eptr[q]; k < P.eptr[q + 1]; ++k) acc = std::fma(P.eval[k], x[P.ecol[k]], acc);
        ext[P.e_row[q]] = acc;
        edone[P.e_row[q]] = 1;
        epos[w] += ewarps;
        progress = true;
      }
    }
    for (auto& g : G) {   // compute groups + their pollers
      if (g.finished) continue;
      if (g.b < 0) {
        if (ticket >= P.nb) { g.finished = true; continue; }
        g.b = ticket++;
        g.f = P.b_frame[g.b];
        g.u = P.b_start[g.b];
        g.xs.assign(P.b_start[g.b + 1] - P.b_start[g.b] + 1, NAN);
        g.xs.back() = 0.0;
        progress = true;
      }
      while (g.f < P.b_frame[g.b + 1]) {
        // rows of this frame: the lane records with ord != 0, in slot order = sweep order
        int cnt = 0;
        for (int r = 0; r < SP; ++r) cnt += P.recB[((size_t)g.f * SP + r) * GI].ord != 0;
        bool ready = true;
        for (int i = 0; i < cnt && ready; ++i) {
          const int u = g.u + i;
          const WaveHdr& H = P.hdr[u];
          if ((H.flags & 1) && !edone[H.row]) ready = false;
          for (int k = 0; k < LN && ready; ++k)
            if (P.lcol[(size_t)u * LN + k] >= 0 && !done[P.lcol[(size_t)u * LN + k]]) ready = false;
        }
        if (!ready) break;
        std::vector<std::pair<int, double>> produced;
        int i = 0;
        for (int r = 0; r < SP; ++r) {
          const size_t s = (size_t)g.f * SP + r;
          if (P.recB[s * GI].ord == 0) continue;
          const int u = g.u + i++;
          const WaveHdr& H = P.hdr[u];
          if (P.recB[s * GI].ord != 1 + (u - P.b_start[g.b]) % WAVE_RQ) return 10;
          double lane[GI];
          for (int gl = 0; gl < GI; ++gl) {
            const WaveRecA& A = P.recA[s * GI + gl];
            const WaveRecB& B = P.recB[s * GI + gl];
            for (unsigned short ix : {B.i0, B.i1, B.i2})
              if (ix >= g.xs.size() || std::isnan(g.xs[ix])) return 2;  // read before produced
            double a = A.c0 * g.xs[B.i0];
            a = std::fma(A.c1, g.xs[B.i1], a);
            a = std::fma(B.c2, g.xs[B.i2], a);
            lane[gl] = a;
          }
          for (int o = GI / 2; o > 0; o >>= 1)
            for (int gl = 0; gl < o; ++gl) lane[gl] += lane[gl + o];
          double late = 0.0;  // poller quad: lane ql sums its LK entries, then the quad is reduced
          {
            double part[WAVE_PQ];
            for (int ql = 0; ql < WAVE_PQ; ++ql) {
              double a = 0.0;
              for (int k = 0; k < WAVE_LK; ++k) {
                const size_t at = (size_t)u * LN + ql * WAVE_LK + k;
                if (P.lcol[at] >= 0) a = std::fma(P.lval[at], x[P.lcol[at]], a);
              }
              part[ql] = a;
            }
            late = (part[0] + part[1]) + (part[2] + part[3]);
          }
          const double e = ((H.flags & 1) ? ext[H.row] : 0.0) + late;
          const double xv = (rhs[H.row] - (e + lane[0])) * H.idiag;
          produced.push_back({H.loc, xv});
          x[H.row] = xv;
          ++used;
        }
        for (auto& pr : produced) g.xs[pr.first] = pr.second;
        for (int k = 0; k < cnt; ++k) done[P.hdr[g.u + k].row] = 1;
        remaining -= cnt;
        g.u += cnt;
        ++g.f;
        progress = true;
      }
      if (g.f == P.b_frame[g.b + 1]) g.b = -1;
    }
    if (!progress) return 4;  // deadlock
  }
  stats[0] = P.nb;
  stats[1] = P.occupancy;
  stats[2] = P.nframes;
  stats[3] = P.rb_max;
  stats[4] = (int)P.internal;
  stats[5] = (int)P.demoted;
  stats[6] = (int)P.external;
  stats[7] = P.nlev;
  stats[8] = (int)used;
  stats[9] = P.max_level_rows;
  stats[10] = (int)P.late;
  return 0;
}
