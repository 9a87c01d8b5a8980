// wave_plan.h -- host planner for the wave sweep (wave.cu): Gauss-Seidel in the reference's
// natural order (smoothers.py:178-190) as the triangular solve T c = r, T = tril(A) / triu(A),
// with the dependency chain kept inside one CTA wherever the grid structure allows it.
//
// In position space (p = i forward, p = n-1-i backward) T is lower triangular.  The positions are
// cut into *bundles*: runs of consecutive grid lines (a line = maximal run of positions in which
// every row reads its predecessor) that end where the next line reads nothing of the previous one
// -- a plane of a lexicographically numbered 3-D patch, a band of lines in 2-D.  Every entry of a
// row is either
//   internal: its column lies in the row's own bundle (3-D, p = 3: the 24 in-plane neighbours) --
//             at most GI * KI per row, the newest first; or
//   external: everything else (the three previous planes, interface rows, demoted internals).
// One CTA group sweeps a bundle level by level (levels of the bundle's own dependency graph): the
// bundle's solution values live in shared memory, so a dependency level costs a shared-memory
// gather, a short reduction and one named barrier instead of an L2 round trip.  The external
// sums are computed off that chain by the rest of the GPU in the flow sweep's manner (rows in
// global dependency-level order, values polled from a global copy) and handed over per row.
//
// Frames: a bundle level is stored as ceil(rows / SP) frames of SP row slots (SP = compute lanes /
// GI); slot s of frame f is global slot f * SP + s.  Per slot a 16-byte header (row, in-bundle
// index, flags, 1 / a_ii) and GI lane records of KI coefficients + KI in-bundle indices, split
// into two 16-byte planes (recA: c0, c1; recB: c2, idx0..2) so a lane's copy is two aligned
// 16-byte cp.async.
#pragma once
#include <cstdint>
#include <vector>

namespace igb {

constexpr int WAVE_GI = 8;    // lanes per row in the compute group
constexpr int WAVE_KI = 3;    // internal entries per lane
constexpr int WAVE_NI = 5;    // compute warps per CTA
constexpr int WAVE_SP = WAVE_NI * 32 / WAVE_GI;   // row slots per frame (20)

struct WaveSlot {   // 16 bytes
  int row;                // matrix row (-1: unused slot)
  unsigned short loc;     // index of the row's value in the bundle's shared-memory vector
  unsigned short flags;   // bit 0: the row has an external sum
  double idiag;           // 1 / a_ii
};
struct WaveRecA { double c0, c1; };
struct WaveRecB { double c2; unsigned short i0, i1, i2, pad; };

struct WavePlanHost {
  int n = 0, nb = 0, nframes = 0, nlev = 0;
  int rb_max = 0;          // rows of the largest bundle
  int occupancy = 0;       // most bundles that must be held at once (deadlock bound, see wave_plan.cpp)
  long long internal = 0, demoted = 0, external = 0;
  int max_level_rows = 0;  // widest bundle level
  std::vector<int> b_frame;   // [nb + 1] first frame of each bundle
  std::vector<int> b_rows;    // [nb] rows of the bundle (= index of its always-zero slot)
  std::vector<WaveSlot> slot; // [nframes * SP]
  std::vector<WaveRecA> recA; // [nframes * SP * GI]
  std::vector<WaveRecB> recB;
  // external sums, flow-sweep layout (flow_plan.h): rows with external entries in global
  // dependency-level order, entries contiguous per row as [early | late]
  int nq = 0;
  std::vector<int> e_row;     // [nq]
  std::vector<int> eptr;      // [nq + 1]
  std::vector<int> ecol;      // [external] rows
  std::vector<double> eval;
  std::vector<int> crit;      // [nq] latest dependency at least crit_lag levels back (-1 none)
  std::vector<int> elate;     // [nq] first late entry
};

// Dependencies of row r: entries [ptr[r], dpos[r]) (lower) or (dpos[r], ptr[r+1]) (upper).
// rb_min / rb_cap: a bundle ends at a detached line once it holds rb_min rows, and before it
// would exceed rb_cap rows.  groups: CTAs that will sweep bundles (occupancy bound).  Returns
// false when the structure does not fit (a line longer than rb_cap, 32-bit offsets, occupancy).
bool build_wave_plan(int n, const int* ptr, const int* col, const double* val, const int* dpos, bool upper,
                     int rb_min, int rb_cap, int crit_lag, int late_max, int groups, WavePlanHost& out);

}  // namespace igb
