// flow_plan.h -- host planner for the dependency-driven triangular sweep (flow.cu).
//
// A Gauss-Seidel sweep in the reference's natural order (smoothers.py:178-190) is a sparse
// triangular solve on tril(A) (forward) or triu(A) (backward).  The plan lists the rows in
// dependency-level order (every row of level l reads only rows of levels < l; rows of one
// level ascending), pads every level to a multiple of the rows one warp takes at once
// (32 / G), and stores each row's strict-triangle entries contiguously in list order, so a
// warp's entry loads are coalesced and its rows come in increasing level order.
#pragma once
#include <vector>

namespace igb {

struct FlowPlanHost {
  int n = 0, nq = 0, nlev = 0, G = 32;
  long long entries = 0;
  std::vector<int> row;      // [nq], -1 = padding
  std::vector<int> eptr;     // [nq + 1]
  std::vector<int> ecol;     // [entries]
  std::vector<double> eval;  // [entries]
  std::vector<double> idiag; // [nq]
  std::vector<int> crit;     // [nq] see build_flow_plan (-1: none)
  std::vector<int> elate;    // [nq] first "late" entry of the slot's row (eptr[q] <= elate[q] <= eptr[q+1])
  std::vector<int> qlev;     // [nq] dependency level of each slot (host diagnostics)
};

// Dependencies of row r: entries [ptr[r], dpos[r]) (lower) or (dpos[r], ptr[r+1]) (upper).
// G = lanes per row (8, 16 or 32); 0 picks it from the mean entries per row.  crit[q] = the
// latest dependency at least crit_lag levels below the row (polled alone before the row's
// values are loaded).  Entries of dependencies fewer than crit_lag levels below the row ("late":
// the newest values, at most late_max, else they stay early) are stored after the others: the
// kernel reduces the early ones as soon as crit is ready and adds the late ones, polled by every
// lane, in a short serial tail.  late_max = 0 keeps the single-batch layout.  Returns false if the
// entry count does not fit 32-bit offsets.
bool build_flow_plan(int n, const int* ptr, const int* col, const double* val, const int* dpos, bool upper,
                     int G, int crit_lag, int late_max, FlowPlanHost& out);

}  // namespace igb
