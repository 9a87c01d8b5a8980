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
// Per position p the planner emits
//   own[3p + d - 1]  coefficient of x(p - d), d = 1..3, when p - d is in p's line (else 0);
//   chunks           the other strict-triangle entries, 32 per chunk (entry e at chunk e / 32,
//                    lane e % 32, ascending position), as (code, value): code >= 0 the global
//                    position q; code < 0 shared-memory slot -1 - code (q minus the bundle's start);
//                    padding reads the always-zero slot rb_max;
//   cptr[p]          first chunk of p (chunks of a row are contiguous, rows in position order);
//   idiag[p]         1 / a_pp.
#pragma once
#include <vector>

namespace igb {

struct LinePlanHost {
  int n = 0, nb = 0, nl = 0;
  int C = 0;        // max chunks of one row
  int rb_max = 0;   // rows of the largest bundle (shared-memory slots)
  long long entries = 0, slots = 0;
  int max_line = 0;
  std::vector<int> bstart;   // [nb + 1] positions
  std::vector<int> bline;    // [nb + 1] first line of each bundle
  std::vector<int> lstart;   // [nl + 1] positions
  std::vector<int> cptr;     // [n + 1] chunk offsets
  std::vector<int> ccol;     // [slots]
  std::vector<double> cval;  // [slots]
  std::vector<double> own;   // [3 n]
  std::vector<double> idiag; // [n]
};

// Dependencies of row r: entries [ptr[r], dpos[r]) (lower) or (dpos[r], ptr[r+1]) (upper).
// A new bundle starts at a line that reads nothing of the previous line once the bundle holds
// >= rb_min rows, or wherever the next line would exceed rb_cap rows.  Returns false when a row
// has more than cmax chunks of entries or a line exceeds rb_cap rows.
bool build_line_plan(int n, const int* ptr, const int* col, const double* val, const int* dpos, bool upper,
                     int rb_min, int rb_cap, int cmax, LinePlanHost& out);

}  // namespace igb
