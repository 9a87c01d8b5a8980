// panel_plan.h -- host planner for the row-panel triangular sweep (one thread-block cluster).
//
// A Gauss-Seidel sweep in the reference's natural order (smoothers.py:178-190) is
// the triangular solve T c = r with T = tril(A) (forward) or triu(A) (backward).
// In *position* space (p = i forward, p = n-1-i backward) T is lower triangular.
// The positions are cut into panels of B consecutive rows; for panel k
//
//     c_k = T_kk^{-1} (r_k - T_{k,<k} c_{<k})
//
// which is the same solve reassociated: the dependency chain is n/B panels long
// instead of the DAG depth (1303 levels on the cfg2 finest level, 171 panels of
// 393 rows or 132 of 512).  T_kk^{-1} is dense lower triangular and computed here
// once per setup (fp64 row recurrence; |T_kk^{-1}| |T_kk| stays O(1) for these
// matrices, tests/test_gpu_parity.py holds the sweep to 1e-12 of SuperLU).
//
// Device work split (G CTAs of W = B/(2G) warps): panel rows are paired
// (q, b-1-q) so every pair owns b+1 inverse entries; pair q belongs to CTA q % G,
// warp q / G.  Per panel and CTA the planner emits
//   lin [W][KBC][32]    inverse rows of the warp's pair: row q's entries at chunks
//                       0..nc1-1 (column 32c + lane), then row b-1-q's at chunks
//                       nc1.. (column 32(c - nc1) + lane), zero padded; nc1 + nc2 <= KBC;
//   ev/ec [W][KA][32]   off-panel coefficients with ring slots (position & (R-1)) of
//                       the CTA's phase-A rows: CTA s owns the contiguous rows
//                       [s*B/G, (s+1)*B/G), warp w half h row s*B/G + 2w + h; entry j
//                       at slot j/16, lane h*16 + j%16;
//   fv/fc [W][KF][32]   off-panel coefficients outside the ring: older than kB-R, or in an
//                       earlier range (another cluster) -- read from the global
//                       position-ordered solution, polled until it holds this sweep's value;
//   xmask [npan*B]      CTAs whose phase-A rows read position p from the ring (bit d =
//                       CTA d): c_p is sent only there;
//   xcnt [npan][G]      values of panel k each CTA receives (its mbarrier byte count / 8).
//
// Ranges: the panels are split into nclu contiguous ranges, one thread-block cluster each,
// running concurrently.  A range depends on earlier ranges only through global values, so
// e.g. the second of two side-by-side patches lags the first by a few grid lines instead of
// waiting for it.  Range starts are rows whose nearest earlier dependency lies >= 2B back
// (patch starts in patch-wise numberings), added greedily while a simulation of panel
// completion times improves (panel_plan.cpp).
#pragma once
#include <vector>

namespace igb {

struct PanelPlanHost {
  int n = 0;
  int B = 512, G = 16, W = 16, R = 8192;
  int KBC = 17, KA = 0, KF = 0;
  int npan = 0;
  int nclu = 1;                      // clusters (ranges)
  std::vector<int> split;            // nclu + 1 panel indices, split[0] = 0, split[nclu] = npan
  std::vector<int> rstart;           // nclu + 1 positions: range c = [rstart[c], rstart[c+1]); its
                                     // panels start at rstart[c] + j B
  double makespan = 0;               // simulated panel-times of the chosen ranges (nclu = 1: npan)
  long long near_entries = 0, far_entries = 0;
  double max_inv_ratio = 0;  // max_k |T_kk^-1|_max * |T_kk|_max (growth diagnostic)
  std::vector<double> lin;   // [npan][G][W][KBC][32]
  std::vector<double> ev;    // [npan][G][W][KA][32]
  std::vector<int> ec;
  std::vector<double> fv;    // [npan + 1][G][W][KF][32] (last panel: zero pad)
  std::vector<int> fc;
  std::vector<unsigned short> xmask;  // [npan * B]
  std::vector<int> xcnt;              // [npan + 1][G]
  long long x_messages = 0;           // sum of popcount(xmask)
};

// Dependencies of row r: entries [ptr[r], dpos[r]) (lower) or (dpos[r], ptr[r+1])
// (upper), diagonal val[dpos[r]].  Returns false when a row has more off-panel
// entries than the kernel variants cover (KA > 14, KA 14 with far entries, or KF > 4).
// W = 16 (B = 32 G, KA in {2,4,8,12}, KF in {0,1,4}; KA 14 with KF 0; KA 8 with KF 5) or W = 8 (B = 16 G, KA in {4,8,12},
// KF in {0,4,8}: entry-heavy 3-D rows).
bool build_panel_plan(int n, const int* ptr, const int* col, const double* val, const int* dpos,
                      bool upper, int G, int W, int R, int max_clusters, PanelPlanHost& out,
                      bool allow_kf10 = false);

}  // namespace igb
