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
// GI).  Per slot GI lane records of KI coefficients + KI in-bundle indices, split into two 16-byte
// planes (recA: c0, c1; recB: c2, idx0..2, ord) so a lane's copy is two aligned 16-byte cp.async.
//
// Schedule levels: the frames of a bundle run one after the other, which adds edges to the
// dependency graph (a row waits for the frame before its own even if it reads nothing of it).
// The level of a frame is 1 + the highest level it reads or follows; the external rows are
// listed by the level of their row's frame, so a warp that walks its share of the list in order
// never waits for a value that (through the frame order) waits for a later entry of its own.
#pragma once
#include <cstdint>
#include <vector>

namespace igb {

constexpr int WAVE_GI = 8;    // lanes per row in the compute group
constexpr int WAVE_KI = 3;    // internal entries per lane
constexpr int WAVE_NI = 5;    // compute warps per CTA
constexpr int WAVE_SP = WAVE_NI * 32 / WAVE_GI;   // row slots per frame (20)
constexpr int WAVE_PQ = 4;    // poller lanes per row
constexpr int WAVE_LK = 3;    // late external entries per poller lane
constexpr int WAVE_LN = WAVE_PQ * WAVE_LK;        // late external entries per row (12)
constexpr int WAVE_RQ = 512;  // queue slots between pollers and compute lanes

// Per row, in sweep order (bundle by bundle, frame by frame, slot by slot): the u-th row of the
// sweep has header hdr[u] and late entries lcol / lval [u * LN, (u + 1) * LN).
struct WaveHdr {   // 16 bytes
  int row;                // matrix row
  unsigned short loc;     // index of the row's value in the bundle's shared-memory vector
  unsigned short flags;   // bit 0: the row has an external sum from the external warps
  double idiag;           // 1 / a_ii
};
struct WaveRecA { double c0, c1; };
struct WaveRecB { double c2; unsigned short i0, i1, i2, ord; };  // ord: 1 + (row's number in its bundle mod RQ), 0 = unused slot

struct WavePlanHost {
  int n = 0, nb = 0, nframes = 0, nlev = 0;
  int rb_max = 0;          // rows of the largest bundle
  int occupancy = 0;       // most bundles that must be held at once (deadlock bound, see wave_plan.cpp)
  long long internal = 0, demoted = 0, late = 0, external = 0;
  int max_level_rows = 0;  // widest bundle level
  std::vector<int> b_frame;   // [nb + 1] first frame of each bundle
  std::vector<int> b_start;   // [nb + 1] first row (sweep order) of each bundle; rows of bundle b = b_start[b+1] - b_start[b]
  std::vector<WaveHdr> hdr;   // [n] sweep order
  std::vector<int> lcol;      // [n * LN] rows (-1: none)
  std::vector<double> lval;   // [n * LN]
  std::vector<WaveRecA> recA; // [nframes * SP * GI]
  std::vector<WaveRecB> recB;
  // external sums, flow-sweep layout (flow_plan.h): rows with external entries in schedule-level
  // order, entries contiguous per row as [early | late]
  int nq = 0;
  std::vector<int> e_row;     // [nq]
  std::vector<int> eptr;      // [nq + 1]
  std::vector<int> ecol;      // [external] rows
  std::vector<double> eval;
  std::vector<int> crit;      // [nq] latest dependency at least crit_lag levels back (-1 none)
  std::vector<int> elate;     // [nq] first late entry
  std::vector<int> e_key;     // [nq] schedule level of the row (host diagnostics / emulation)
  std::vector<int> f_key;     // [nframes] schedule level of each frame
  std::vector<int> f_end;     // [nframes] rows of the frame's bundle in frames up to and including it
};

// Dependencies of row r: entries [ptr[r], dpos[r]) (lower) or (dpos[r], ptr[r+1]) (upper).
// rb_min / rb_cap: a bundle ends at a detached line once it holds rb_min rows, and before it
// would exceed rb_cap rows.  late_lag: external entries produced fewer than late_lag schedule
// levels before the row are "late" (at most LN, the newest first): the bundle's own pollers add
// them, so the hand-over between planes is one global round trip.  groups: CTAs that will sweep
// bundles (occupancy bound).  Returns false when the structure does not fit (a line longer than
// rb_cap, 32-bit offsets, occupancy).
bool build_wave_plan(int n, const int* ptr, const int* col, const double* val, const int* dpos, bool upper,
                     int rb_min, int rb_cap, int late_lag, int crit_lag, int late_max, int groups,
                     WavePlanHost& out);

}  // namespace igb
