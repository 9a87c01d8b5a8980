// level_plan.h -- host planner for the streamed level-set triangular sweep.
//
// A Gauss-Seidel sweep in the reference's natural order (smoothers.py:178-190)
// is a sparse triangular solve; its rows are grouped into dependency levels
// (every row of level l depends only on rows of levels < l).  One CTA runs the
// whole sweep, one level (or a chunk of a large level) per step with a single
// __syncthreads between steps.  Everything a step touches is in shared memory
// before the step starts:
//   * the step's block (rows, 1/diag, coefficients, where each x comes from)
//     is streamed by a TMA bulk copy D steps ahead;
//   * x values produced more than G steps earlier ("old") and the rows' rhs
//     and u values are gathered with cp.async G steps ahead;
//   * x values produced recently live in a shared ring indexed by level-order
//     position (slot = pos & (R-1)).
// Block layout (every section 16-byte aligned), nta = active threads (mult. of 32):
//   [int K, int nrows, int ng, int start_pos] [int bytes, int nta, int chunk_end, int pad]
//   [int rows[rpra]] [double invd[rpra]] [double val[K][nta]] [int src[K][nta]] [int gsrc[nga]]
//   src: index into the kernel's shared double array [ring (R) | gather slots],
//   already resolved for this step's gather slot (t % (G+2)) and the 16-byte
//   parity of the gathered row, so the inner loop is one dependent LDS.
// Consecutive blocks are packed into chunks (<= chunk_bytes); one TMA bulk copy
// fetches a chunk.  chunk_end = 1 on the last block of a chunk.
#pragma once
#include <vector>

namespace igb {

struct LevelPlanHost {
  int n = 0;
  int nsteps = 0;
  int nlevels = 0;
  int NT = 128;        // threads of the CTA
  int TPR = 1;         // threads per row
  int R = 4096;        // ring slots (power of two)
  int D = 4;           // bulk-copy lookahead (steps)
  int G = 2;           // gather lookahead (steps)
  int max_bytes = 0;   // largest block
  int max_ng = 0;      // most gathered x values in one step (multiple of 4)
  int max_rows = 0;    // most rows in one step (multiple of 4)
  long long entries = 0;
  int chunk_bytes = 0;              // stage size (largest chunk)
  int nchunks = 0;
  std::vector<long long> chunk_off;   // chunk c = stream[chunk_off[c], chunk_off[c+1])
  std::vector<unsigned char> stream;
};

// Dependencies of row r: entries [ptr[r], dpos[r]) (lower / forward sweep) or
// (dpos[r], ptr[r+1]) (upper / backward sweep).  Returns false when the ring is
// too small for the dependency distances (caller keeps the plain level kernel).
bool build_level_plan(int n, const int* ptr, const int* col, const double* val, const int* dpos,
                      bool upper, int NT, int R, int D, int G, int chunk_target, LevelPlanHost& out);

}  // namespace igb
