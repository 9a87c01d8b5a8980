// level_plan.h -- host planner for the level-set triangular sweep (one CTA).
//
// A Gauss-Seidel sweep in the reference's natural order (smoothers.py:178-190)
// is a sparse triangular solve; its rows are grouped into dependency levels
// (every row of level l depends only on rows of levels < l).  One CTA runs the
// whole sweep, one level (or a chunk of <= NT/TPR rows of it) per step, with a
// single __syncthreads between steps.  Vectors are handled in *level order*
// (position p = index of the row in the level-ordered row list `rows`): a
// gather kernel builds the level-ordered right-hand side, the sweep writes the
// level-ordered solution, a scatter kernel adds it into u.  So every per-step
// access is contiguous and addressable from the step metadata alone.
//
// Layout (read-only on the device):
//   meta[t] = {int off16, int K, int nrows, int start}   (block offset in 16-byte units;
//             K = kt = entries per thread = kmax, zero padded)
//   block t: [double invd[rpra]] [double2 val[kt/2][nthr]] [int2 src[kt/2][nthr]]
//     (interleaved so a warp's 128-bit loads are contiguous; nthr = nrows * TPR):
//     thread i*TPR + j owns row slot i and the row's entries j, j+TPR, ...;
//     padded with zero coefficients against ring slot 0;
//     src >= 0: ring slot (position & (R-1)) of a value produced recently;
//     src < 0: position -src-1 of an older value in the level-ordered solution.
#pragma once
#include <vector>

namespace igb {

struct LevelMeta {
  int off16, K, nrows, start;
};

struct LevelPlanHost {
  int n = 0;
  int nsteps = 0;
  int nlevels = 0;
  int NT = 256;        // threads of the CTA
  int TPR = 1;         // threads per row
  int R = 4096;        // ring slots (power of two)
  long long entries = 0;
  long long global_refs = 0;
  bool has_old = false;        // some entries lie outside the ring
  std::vector<LevelMeta> meta;
  std::vector<int> rows;       // level order -> row
  std::vector<unsigned char> stream;
};

// Dependencies of row r: entries [ptr[r], dpos[r]) (lower / forward sweep) or
// (dpos[r], ptr[r+1]) (upper / backward sweep).  Returns false if no TPR <= 32
// brings the per-thread entry count down to kmax.
bool build_level_plan(int n, const int* ptr, const int* col, const double* val, const int* dpos,
                      bool upper, int NT, int R, int kmax, LevelPlanHost& out);

}  // namespace igb
