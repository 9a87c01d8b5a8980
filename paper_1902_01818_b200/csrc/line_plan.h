// line_plan.h -- host planner for the line sweep (line.cu): Gauss-Seidel in the reference's
// natural order (smoothers.py:178-190) as a triangular solve T c = r, T = tril(A) / triu(A),
// scheduled along *lines*.
//
// In position space (p = i forward, p = n-1-i backward) T is lower triangular.  A line is a
// maximal run of consecutive positions in which every row reads its predecessor (a grid line
// along the fastest tensor axis of a patch: 65 rows on cfg5's finest level); a bundle is a run of
// consecutive lines whose solution values fit one CTA's shared memory (a plane of a 3-D patch,
// a band of grid lines in 2-D).  One warp walks a line row by row: the row's three newest
// same-line values stay in registers, values of the bundle's other lines come from shared memory
// (written by the CTA's other warps a few rows earlier), values of other bundles from the global
// solution copy (L2).  The critical path of the sweep is then mostly register and shared-memory
// hand-offs; the L2 round trip is paid where the path crosses bundles (once per plane step in 3-D)
// instead of at every dependency level as in the flow sweep (flow.cu).
//
// Per position p the planner emits one fixed-size record (line_rec_bytes(C) bytes, so the
// kernel computes its address and bulk-prefetches it into L2 rows ahead without indirection):
//   int    cc[C][32]   codes of the row's "early" entries, 32 per chunk (entry e at chunk e / 32,
//                      lane e % 32, ascending position): code >= 0 the global position q; code < 0
//                      shared-memory slot -1 - code (q minus the bundle's start); padding reads the
//                      always-zero slot rb_max;
//   double cv[C][32]   their coefficients;
//   int    lc[LINE_LATE], ovf_start, ovf_chunks
//                      late entries: up to LINE_LATE entries produced in the last LINE_LATE_LAG
//                      dependency levels before p (the neighbour line's and the previous plane's
//                      newest values), oldest first, gathered one row ahead and added after the
//                      row's reduction; chunks beyond C (long interface rows) in the overflow
//                      arrays at [ovf_start, ovf_start + ovf_chunks);
//   double lv[LINE_LATE]  late coefficients;
//   double own[3], idiag  coefficients of x(p-1), x(p-2), x(p-3) when in p's line (else 0), 1/a_pp.
#pragma once
#include <vector>

namespace igb {

constexpr int LINE_LATE = 6;   // late entries per row (3-D p = 3: the neighbour line's and the
                                // previous plane's values of the last three dependency levels)
constexpr int LINE_LATE_LAG = 3;

#ifdef __CUDACC__
#define LINE_HD __host__ __device__
#else
#define LINE_HD
#endif
// record layout (bytes) for C register chunks
LINE_HD constexpr int line_off_cv(int C) { return 128 * C; }
LINE_HD constexpr int line_off_meta(int C) { return 384 * C; }
LINE_HD constexpr int line_off_lv(int C) { return 384 * C + 4 * (LINE_LATE + 2); }
LINE_HD constexpr int line_off_own(int C) { return line_off_lv(C) + 8 * LINE_LATE; }
LINE_HD constexpr int line_rec_bytes(int C) { return line_off_own(C) + 32; }
static_assert(line_rec_bytes(6) % 16 == 0 && line_off_lv(6) % 8 == 0, "record alignment");

struct LinePlanHost {
  int n = 0, nb = 0, nl = 0;
  int C = 0;        // register chunks per record (2, 4, 6); longer rows spill into the overflow
  int cmax = 0;     // chunks of the longest row
  int rb_max = 0;   // rows of the largest bundle (shared-memory slots)
  long long entries = 0, chunks = 0, ovf_rows = 0;
  int max_line = 0;
  std::vector<int> bstart;   // [nb + 1] positions
  std::vector<int> bline;    // [nb + 1] first line of each bundle
  std::vector<int> lstart;   // [nl + 1] positions
  std::vector<double> rec;   // [n * line_rec_bytes(C) / 8]
  std::vector<int> ocol;     // overflow chunks [32 * k]
  std::vector<double> oval;
};

// Dependencies of row r: entries [ptr[r], dpos[r]) (lower) or (dpos[r], ptr[r+1]) (upper).
// A new bundle starts at a line that reads nothing of the previous line once the bundle holds
// >= rb_min rows, or wherever the next line would exceed rb_cap rows.  Rows may have any number
// of chunks (C reports the largest); returns false when a line exceeds rb_cap rows.
bool build_line_plan(int n, const int* ptr, const int* col, const double* val, const int* dpos, bool upper,
                     int rb_min, int rb_cap, int cmax, LinePlanHost& out);

}  // namespace igb
