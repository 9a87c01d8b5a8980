// igb.cu -- native runtime of the device MG-PCG solve: context, device memory,
// Gauss-Seidel level schedules, cycle orchestration (captured as a CUDA graph),
// PCG driver and the C ABI declared in include/igb.h.
//
// Cycle semantics follow the reference exactly (pkg/src/igamg/multigrid.py:118-138,
// smoothers.py:186-200, 321-353):
//   u = 0; pre_smooth; r = P^T (f - A u); coarse (l == 1) or mu recursive cycles,
//   each followed by u = u + P e; post_smooth.
// A "u is still zero" flag is tracked so that f - A*0 is never computed (bitwise
// identical shortcut: the reference computes f - A@0 == f).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "igb.h"
#include "level_plan.h"
#include "flow_plan.h"
#include "line_plan.h"
#include "wave_plan.h"
#include "panel_plan.h"
#include "host_par.h"
#include "kernels.cuh"

using namespace igb;

namespace {

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ArgError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct StateError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CU(expr)                                                                        \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      throw CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e));              \
  } while (0)

enum KernelClass { K_SPMV = 0, K_GS = 1, K_FD = 2, K_PIECES = 3, K_TRANSFER = 4, K_COARSE = 5, K_CG = 6, K_NCLASS = 7 };

struct DevCsr {
  int n = 0, m = 0;
  long long nnz = 0;
  int* ptr = nullptr;
  int* col = nullptr;
  double* val = nullptr;
  int group = 8;
};

struct Sched {
  int nlev = 0;
  int* lvl_ptr = nullptr;
  int* rows = nullptr;
};

struct InteriorStage {
  int dim;
  int n[3];
  const double* T[3];   // device
  const double* D;      // device
  const int* idx;       // device
};

struct FdPlan {
  std::vector<FdBatch> batches;  // fused 2-D interiors (fd.cu)
  std::vector<double> batch_bytes;
  int nsteps = 0;
  GemmDesc* d_desc[6] = {nullptr};
  int ndesc[6] = {0};
  int tiles[6] = {0};
  double bytes[6] = {0};
  double flops = 0;       // per application over all interiors: 4 prod(n) sum_a n_a (2 d contractions)
  int first_gather = 0;   // step index with the gather
  int last_scatter = 0;   // step index with the scatter
  Fd3Plan fd3;            // 3-D interiors on the fused DMMA path (fd3.cu): three launches
  double fd3_bytes[3] = {0};
};

struct SweepDev {
  bool ok = false;
  LevelArgs args{};
  const int* rows = nullptr;   // level order -> row
  long long entries = 0, steps = 0, levels = 0;
  double stream_bytes = 0;
};

struct PanelDev {
  bool ok = false;
  PanelArgs args{};
  long long npan = 0, near = 0, far = 0;
  double lin_bytes = 0, ent_bytes = 0;
};

struct FlowDev {
  bool ok = false;
  FlowArgs args{};
  std::vector<int> h_row, h_qlev;  // kept for IGB_FLOW_TRACE dumps
  int nlev = 0;
  long long entries = 0;
};

struct LineDev {
  bool ok = false;
  LineArgs args{};
  long long entries = 0, slots = 0;
  int nl = 0, max_line = 0;
};

struct WaveDev {
  bool ok = false;
  WaveArgs args{};
  int nlev = 0, nframes = 0, occupancy = 0;
  long long internal = 0, external = 0;
  double stream_bytes = 0;
};

struct Level {
  int n = 0;
  DevCsr A;
  std::vector<int> h_ptr, h_col;
  std::vector<double> h_val;
  SweepDev sweep[2];   // 0: forward (lower) sweep, 1: backward (upper) sweep
  PanelDev panel[2];   // row-panel sweeps (preferred when built)
  FlowDev flow[2];     // dependency-driven whole-GPU sweeps (wide levels, long rows)
  LineDev line[2];     // line sweeps (bundles of grid lines per CTA; 3-D levels)
  WaveDev wave[2];     // wave sweeps (plane chains inside one CTA, external sums GPU-wide)
  double* xg = nullptr;  // panel sweep solution by position (old values)
  double* rp = nullptr;   // level-ordered right-hand side / solution of the sweep
  double* xp = nullptr;
  std::vector<double> h_diag;
  int* dpos = nullptr;
  bool has_P = false;
  DevCsr P, PT;
  bool has_kron = false;  // Kronecker form of P (transfer.cu), used instead of the CSR pair
  KronArgs kron{};
  bool has_mf = false;    // matrix-free A (mfree.cu), used for full products A x on this level
  MfArgs mf{};
  double* mf_s[4] = {nullptr, nullptr, nullptr, nullptr};
  bool has_gs = false;
  bool has_U = false;
  DevCsr U;  // strict upper triangle of A: residual after a forward sweep from zero is -U c
  DevCsr Lo; // strict lower triangle: a backward step from u solves triu(A) u' = f - Lo u
  Sched fwd, bwd;
  long long tri_nnz_lower = 0, tri_nnz_upper = 0;
  bool has_scms = false;
  double tau = 1.0;
  std::vector<InteriorStage> interiors;
  std::vector<PieceRowBlock> h_blocks;
  PieceRowBlock* d_blocks = nullptr;
  double piece_bytes = 0;
  bool pieces_fused = false;  // done by the FD back kernel's extra CTAs
  int piece_max_m = 0;
  long long piece_rows = 0;
  FdPlan fd;
  size_t fd_scratch = 0;
  double* f = nullptr;
  double* u = nullptr;
  double* r = nullptr;
  double* c = nullptr;
  double* s0 = nullptr;
  double* s1 = nullptr;
};

struct Coarse {
  bool set = false;
  int n = 0;
  // dense operator M = P_c U^-1 L^-1 P_r (built from the same factors) for small
  // coarse problems: one GEMV instead of 2n dependent substitution steps
  PieceRowBlock* d_dense = nullptr;
  int ndense = 0;
  CoarseCsc csc{};
  DevCsr L, U;
  int *Ldpos = nullptr, *Udpos = nullptr;
  Sched Ls, Us;
  int* inv_perm_r = nullptr;
  int* perm_c = nullptr;
  double* y = nullptr;
  double* w = nullptr;
};

struct ProfRec {
  int cls;
  double bytes;
  cudaEvent_t a, b;
  double flops;
};

}  // namespace

struct igb_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  int L = -1;
  std::vector<Level> lev;
  Coarse coarse;
  int smoother = IGB_SMOOTHER_HYBRID;
  int mu = 1;
  std::vector<int> steps;
  bool finalized = false;
  std::vector<void*> allocs;
  // FD data shared between interiors with identical content (transforms, denominators): keyed by
  // (element count, content hash), verified against a host copy -- never by host address, which a
  // caller may reuse for different temporaries between calls
  struct SharedUpload {
    std::vector<double> host;
    const double* dev;
  };
  std::map<std::pair<size_t, unsigned long long>, std::vector<SharedUpload>> shared_uploads;

  // CG state
  double *x = nullptr, *d = nullptr, *q = nullptr, *b = nullptr, *partials = nullptr,
         *hist_dev = nullptr;
  unsigned* counter = nullptr;
  CgScalars* sc = nullptr;
  CgScalars* sc_host = nullptr;  // pinned
  double* hist_host = nullptr;   // pinned staging of the residual history
  int hist_cap = 0;

  // graph of cycle(L)
  cudaGraphExec_t cycle_exec = nullptr;
  // whole PCG solve as one graph (WHILE over iterations, IF around the cycle), per key
  cudaGraphExec_t pcg_exec = nullptr;
  const double* pcg_b = nullptr;
  double* pcg_x = nullptr;
  int pcg_max = -1;
  long long pcg_n_pre = 0, pcg_n_head = 0, pcg_n_if = 0;
  bool pcg_graph_failed = false;
  cudaStream_t aux[2] = {nullptr, nullptr};
  bool capturing = false;
  bool graph_prof = false;

  // launch accounting (kernels issued directly + kernels replayed from the graph)
  long long launches_direct = 0, graph_kernels = 0, graph_replays = 0;

  // profiling
  bool prof = false;
  std::vector<ProfRec> direct_recs;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_next = 0;
  std::vector<ProfRec> graph_recs;
  double prof_ms[K_NCLASS] = {0};
  long long prof_n[K_NCLASS] = {0};
  double prof_bytes[K_NCLASS] = {0};
  double prof_flops[K_NCLASS] = {0};
  // the class's largest launch (most algorithmic bytes: the finest level's kernel)
  double top_bytes[K_NCLASS] = {0}, top_ms[K_NCLASS] = {0};
  long long top_n[K_NCLASS] = {0};

  // timing of last pcg
  double last_pcg_ms = 0, last_cycle_ms = 0;
  cudaEvent_t t0 = nullptr, t1 = nullptr;

  template <class T>
  T* alloc(size_t count) {
    if (count == 0) count = 1;
    void* p = nullptr;
    CU(cudaMalloc(&p, count * sizeof(T)));
    allocs.push_back(p);
    return static_cast<T*>(p);
  }
  template <class T>
  T* upload(const T* h, size_t count) {
    T* p = alloc<T>(count);
    if (count) copy_h2d(p, h, count * sizeof(T));
    return p;
  }
  // H2D from pageable memory: large arrays go through two pinned 64 MB staging buffers (parallel
  // host memcpy overlapped with the DMA of the previous chunk) instead of the driver's slow path
  char* stage[2] = {nullptr, nullptr};
  cudaEvent_t stage_ev[2] = {nullptr, nullptr};
  static constexpr size_t kStage = 64u << 20;
  void copy_h2d(void* dst, const void* src, size_t bytes) {
    if (bytes < (8u << 20)) {
      CU(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
      return;
    }
    if (!stage[0]) {
      for (int i = 0; i < 2; ++i) {
        CU(cudaHostAlloc(reinterpret_cast<void**>(&stage[i]), kStage, cudaHostAllocDefault));
        CU(cudaEventCreateWithFlags(&stage_ev[i], cudaEventDisableTiming));
      }
    }
    for (size_t off = 0, k = 0; off < bytes; off += kStage, ++k) {
      const size_t len = std::min(kStage, bytes - off);
      const int b = (int)(k & 1);
      CU(cudaEventSynchronize(stage_ev[b]));  // the DMA that last read this buffer is done
      par_memcpy(stage[b], static_cast<const char*>(src) + off, len);
      CU(cudaMemcpyAsync(static_cast<char*>(dst) + off, stage[b], len, cudaMemcpyHostToDevice, stream));
      CU(cudaEventRecord(stage_ev[b], stream));
    }
    CU(cudaStreamSynchronize(stream));
  }

  cudaEvent_t pool_event() {
    if (ev_next == ev_pool.size()) {
      cudaEvent_t e;
      CU(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    return ev_pool[ev_next++];
  }

  // Launch wrapper: records CUDA events around the launch in profile mode.
  template <class F>
  void launch(int cls, double bytes, F&& f, double flops = 0.0) {
    if (capturing) ++graph_kernels; else ++launches_direct;
    if (!prof) {
      f();
      return;
    }
    ProfRec r{cls, bytes, nullptr, nullptr, flops};
    if (capturing) {
      CU(cudaEventCreate(&r.a));
      CU(cudaEventCreate(&r.b));
    } else {
      r.a = pool_event();
      r.b = pool_event();
    }
    // inside stream capture a plain record is only a dependency marker; External
    // makes it a real event-record node that is timestamped at every replay
    const unsigned fl = capturing ? cudaEventRecordExternal : 0u;
    CU(cudaEventRecordWithFlags(r.a, stream, fl));
    f();
    CU(cudaEventRecordWithFlags(r.b, stream, fl));
    (capturing ? graph_recs : direct_recs).push_back(r);
  }
  void harvest(std::vector<ProfRec>& recs, bool clear) {
    for (auto& r : recs) {
      float ms = 0;
      CU(cudaEventElapsedTime(&ms, r.a, r.b));
      prof_ms[r.cls] += ms;
      prof_n[r.cls] += 1;
      prof_bytes[r.cls] += r.bytes;
      prof_flops[r.cls] += r.flops;
      if (r.bytes > top_bytes[r.cls] * (1.0 + 1e-9)) {
        top_bytes[r.cls] = r.bytes;
        top_ms[r.cls] = 0;
        top_n[r.cls] = 0;
      }
      if (r.bytes >= top_bytes[r.cls] * (1.0 - 1e-9)) {
        top_ms[r.cls] += ms;
        top_n[r.cls] += 1;
      }
    }
    if (clear) {
      recs.clear();
      ev_next = 0;
    }
  }
  void drop_graph() {
    if (cycle_exec) cudaGraphExecDestroy(cycle_exec);
    cycle_exec = nullptr;
    graph_kernels = 0;
    for (auto& r : graph_recs) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    graph_recs.clear();
  }

  // ---------------------------------------------------------------- operators
  Level& level(int l) {
    if (l < 0 || l > L) throw ArgError("level out of range");
    return lev[l];
  }

  void spmv(const DevCsr& M, const double* x_, const double* z, double* y, int sign, int cls) {
    const double bytes = 12.0 * M.nnz + 4.0 * (M.n + 1) + 8.0 * M.m + 8.0 * M.n + (sign ? 8.0 * M.n : 0.0);
    launch(cls, bytes, [&] { launch_spmv(stream, M.n, M.ptr, M.col, M.val, x_, z, y, sign, M.group); });
  }

  // y = P_l e (accumulate: y = z + P_l e) and y = P_l^T r, Kronecker form when set
  void prolong(int l, const double* e, const double* z, double* y, int accumulate) {
    Level& V = lev[l];
    if (V.has_kron) {
      const KronArgs& k = V.kron;
      const double bytes = (16.0 + (accumulate ? 8.0 : 0.0)) * k.n_fine + 12.0 * k.n_coarse;
      launch(K_TRANSFER, bytes, [&] { launch_kron_prolong(stream, k, e, z, y, accumulate); });
      return;
    }
    spmv(V.P, e, accumulate ? z : nullptr, y, accumulate ? 1 : 0, K_TRANSFER);
  }
  void restrict_to(int l, const double* r, double* y) {
    Level& V = lev[l];
    if (V.has_kron) {
      const KronArgs& k = V.kron;
      const double bytes = 12.0 * k.n_fine + 16.0 * k.n_coarse;
      launch(K_TRANSFER, bytes, [&] { launch_kron_restrict(stream, k, r, y); });
      return;
    }
    spmv(V.PT, r, nullptr, y, 0, K_TRANSFER);
  }

  // GS correction on level l: solve tril (fwd) / triu (bwd); if into_u_zero the
  // solution is written straight into u (u was zero), else c is solved and
  // accumulated into u.
  void gs(int l, bool upper, const double* rhs, double* u, bool u_zero) {
    Level& V = lev[l];
    PanelDev& Pn = V.panel[upper ? 1 : 0];
    if (Pn.ok) {
      PanelArgs a = Pn.args;
      a.res = rhs;
      a.u = u;
      a.accumulate = u_zero ? 0 : 1;
      static long long* dbg = nullptr;
      static const bool want_dbg = std::getenv("IGB_GS_DEBUG") != nullptr;
      if (want_dbg && !capturing) {
        if (!dbg) CU(cudaMalloc(&dbg, 8 * sizeof(long long)));
        a.dbg = dbg;
        const char* ab = std::getenv("IGB_GS_ABLATE");
        a.ablate = ab ? std::atoi(ab) : 0;
      }
      // algorithmic bytes of the triangular solve; the inverse blocks the
      // panel sweep streams instead (Pn.lin_bytes) are an implementation choice
      const long long tri = upper ? V.tri_nnz_upper : V.tri_nnz_lower;
      const double bytes = 12.0 * (tri + V.n) + 4.0 * (V.n + 1) + 24.0 * V.n;
      launch(K_GS, bytes, [&] { launch_panel_sweep(stream, a); });
      if (a.dbg) {
        long long hd[8];
        CU(cudaMemcpyAsync(hd, dbg, sizeof(hd), cudaMemcpyDeviceToHost, stream));
        CU(cudaStreamSynchronize(stream));
        const long long np = hd[0] > 0 ? hd[0] : 1;
        std::fprintf(stderr,
                     "[gs dbg] panel level %d dir %d n %d panels %lld: %lld cyc/panel (wait_x %lld, loads %lld, "
                     "phaseA %lld, wait_r %lld, wait_tma %lld, phaseB %lld)\n",
                     l, upper ? 1 : 0, V.n, hd[0], hd[1] / np, hd[2] / np, hd[3] / np, hd[4] / np, hd[5] / np,
                     hd[6] / np, hd[7] / np);
      }
      return;
    }
    WaveDev& Wv = V.wave[upper ? 1 : 0];
    if (Wv.ok) {
      WaveArgs a = Wv.args;
      a.res = rhs;
      a.u = u;
      a.accumulate = u_zero ? 0 : 1;
      const long long tri = upper ? V.tri_nnz_upper : V.tri_nnz_lower;
      const double bytes = 12.0 * (tri + V.n) + 4.0 * (V.n + 1) + 24.0 * V.n;
      static const bool want_dbg = std::getenv("IGB_GS_DEBUG") != nullptr;
      if (want_dbg && !capturing) {
        cudaEvent_t e0, e1;
        CU(cudaEventCreate(&e0));
        CU(cudaEventCreate(&e1));
        static unsigned long long* wdbg = nullptr;
        if (!wdbg) CU(cudaMalloc(&wdbg, 16 * sizeof(unsigned long long)));
        CU(cudaMemsetAsync(wdbg, 0, 16 * sizeof(unsigned long long), stream));
        a.dbg = wdbg;
        CU(cudaEventRecord(e0, stream));
        launch_wave_sweep(stream, a);
        CU(cudaEventRecord(e1, stream));
        CU(cudaEventSynchronize(e1));
        float ms = 0;
        CU(cudaEventElapsedTime(&ms, e0, e1));
        unsigned long long hd[16];
        CU(cudaMemcpy(hd, wdbg, sizeof(hd), cudaMemcpyDeviceToHost));
        const double fr = (double)std::max(1ULL, hd[0]), pr = (double)std::max(1ULL, hd[6]);
        std::fprintf(stderr, "[gs dbg] wave level %d dir %d n %d depth %d bundles %d ctas %d: %.1f us, %.3f us/level, "
                     "%.0f GB/s streamed; compute %.0f cyc/frame (%.0f waiting for the queue), poller quad 0: "
                     "%.0f cyc/row late wait, %.0f ext wait, %.0f queue-space wait\n", l, upper ? 1 : 0, V.n, Wv.nlev,
                     a.nb, a.ctas, ms * 1e3, ms * 1e3 / std::max(1, Wv.nlev), Wv.stream_bytes / (ms * 1e6), hd[1] / fr,
                     hd[2] / fr, hd[4] / pr, hd[5] / pr, hd[7] / pr);

        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return;
      }
      launch(K_GS, bytes, [&] { launch_wave_sweep(stream, a); });
      return;
    }
    LineDev& Ln = V.line[upper ? 1 : 0];
    if (Ln.ok) {
      LineArgs a = Ln.args;
      a.res = rhs;
      a.u = u;
      a.accumulate = u_zero ? 0 : 1;
      const long long tri = upper ? V.tri_nnz_upper : V.tri_nnz_lower;
      const double bytes = 12.0 * (tri + V.n) + 4.0 * (V.n + 1) + 24.0 * V.n;
      static const bool want_dbg = std::getenv("IGB_GS_DEBUG") != nullptr;
      if (want_dbg && !capturing) {
        cudaEvent_t e0, e1;
        CU(cudaEventCreate(&e0));
        CU(cudaEventCreate(&e1));
        const char* tr = std::getenv("IGB_LINE_TRACE");
        long long* dtr = nullptr;
        if (tr) {
          CU(cudaMalloc(&dtr, 3 * sizeof(long long) * V.n));
          CU(cudaMemsetAsync(dtr, 0, 3 * sizeof(long long) * V.n, stream));
          a.trace = dtr;
        }
        long long* dprof = nullptr;
        CU(cudaMalloc(&dprof, 8 * sizeof(long long)));
        CU(cudaMemsetAsync(dprof, 0, 8 * sizeof(long long), stream));
        a.prof = dprof;
        CU(cudaEventRecord(e0, stream));
        launch_line_sweep(stream, a);
        CU(cudaEventRecord(e1, stream));
        CU(cudaEventSynchronize(e1));
        {
          long long hp[8];
          CU(cudaMemcpy(hp, dprof, sizeof(hp), cudaMemcpyDeviceToHost));
          cudaFree(dprof);
          const double r = std::max(1LL, hp[5]);
          std::fprintf(stderr, "[gs dbg] line level %d dir %d cycles/row: D-poll %.0f D %.0f C %.0f B %.0f A %.0f\n", l,
                       upper ? 1 : 0, hp[0] / r, hp[1] / r, hp[2] / r, hp[3] / r, hp[4] / r);
        }
        if (tr) {  // binary dump: int n, nl, nb; int[nl+1] lstart; int[nb+1] bstart; int64[3n] trace
          std::vector<long long> ht(3 * (size_t)V.n);
          CU(cudaMemcpy(ht.data(), dtr, ht.size() * sizeof(long long), cudaMemcpyDeviceToHost));
          cudaFree(dtr);
          std::vector<int> ls(Ln.nl + 1), bsv(a.nb + 1);
          CU(cudaMemcpy(ls.data(), a.lstart, ls.size() * sizeof(int), cudaMemcpyDeviceToHost));
          CU(cudaMemcpy(bsv.data(), a.bstart, bsv.size() * sizeof(int), cudaMemcpyDeviceToHost));
          char path[512];
          std::snprintf(path, sizeof(path), "%s.l%d.d%d.bin", tr, l, upper ? 1 : 0);
          if (FILE* fp = std::fopen(path, "wb")) {
            int hdr[3] = {V.n, Ln.nl, a.nb};
            std::fwrite(hdr, sizeof(int), 3, fp);
            std::fwrite(ls.data(), sizeof(int), ls.size(), fp);
            std::fwrite(bsv.data(), sizeof(int), bsv.size(), fp);
            std::fwrite(ht.data(), sizeof(long long), ht.size(), fp);
            std::fclose(fp);
          }
        }
        float ms = 0;
        CU(cudaEventElapsedTime(&ms, e0, e1));
        const int depth = upper ? V.bwd.nlev : V.fwd.nlev;
        std::fprintf(stderr, "[gs dbg] line level %d dir %d n %d depth %d bundles %d lines %d ctas %d C %d: %.1f us, "
                     "%.3f us/level\n", l, upper ? 1 : 0, V.n, depth, a.nb, Ln.nl, a.ctas, a.C, ms * 1e3,
                     ms * 1e3 / std::max(1, depth));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return;
      }
      launch(K_GS, bytes, [&] { launch_line_sweep(stream, a); });
      return;
    }
    FlowDev& Fw = V.flow[upper ? 1 : 0];
    if (Fw.ok) {
      FlowArgs a = Fw.args;
      a.res = rhs;
      a.u = u;
      a.accumulate = u_zero ? 0 : 1;
      const long long tri = upper ? V.tri_nnz_upper : V.tri_nnz_lower;
      const double bytes = 12.0 * (tri + V.n) + 4.0 * (V.n + 1) + 24.0 * V.n;
      static const bool want_dbg = std::getenv("IGB_GS_DEBUG") != nullptr;
      if (want_dbg && !capturing) {
        cudaEvent_t e0, e1;
        CU(cudaEventCreate(&e0));
        CU(cudaEventCreate(&e1));
        const char* tr = std::getenv("IGB_FLOW_TRACE");
        long long* dtr = nullptr;
        if (tr) {
          CU(cudaMalloc(&dtr, 5 * sizeof(long long) * a.nq));
          CU(cudaMemsetAsync(dtr, 0, 5 * sizeof(long long) * a.nq, stream));
          a.trace = dtr;
        }
        CU(cudaEventRecord(e0, stream));
        launch_flow_sweep(stream, a);
        CU(cudaEventRecord(e1, stream));
        CU(cudaEventSynchronize(e1));
        if (tr) {  // binary dump: int nq, int[nq] row, int[nq] level, int64[5 nq] trace
          std::vector<long long> ht(5 * (size_t)a.nq);
          CU(cudaMemcpy(ht.data(), dtr, ht.size() * sizeof(long long), cudaMemcpyDeviceToHost));
          cudaFree(dtr);
          char path[512];
          std::snprintf(path, sizeof(path), "%s.l%d.d%d.bin", tr, l, upper ? 1 : 0);
          if (FILE* fp = std::fopen(path, "wb")) {
            std::fwrite(&a.nq, sizeof(int), 1, fp);
            std::fwrite(Fw.h_row.data(), sizeof(int), Fw.h_row.size(), fp);
            std::fwrite(Fw.h_qlev.data(), sizeof(int), Fw.h_qlev.size(), fp);
            std::fwrite(ht.data(), sizeof(long long), ht.size(), fp);
            std::fclose(fp);
          }
        }
        float ms = 0;
        CU(cudaEventElapsedTime(&ms, e0, e1));
        std::fprintf(stderr, "[gs dbg] flow level %d dir %d n %d depth %d ctas %d G %d: %.1f us, %.3f us/level\n", l,
                     upper ? 1 : 0, V.n, Fw.nlev, a.ctas, a.G, ms * 1e3, ms * 1e3 / std::max(1, Fw.nlev));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        return;
      }
      launch(K_GS, bytes, [&] { launch_flow_sweep(stream, a); });
      return;
    }
    SweepDev& C = V.sweep[upper ? 1 : 0];
    if (C.ok) {
      LevelArgs a = C.args;
      a.rp = V.rp;
      a.xp = V.xp;
      const long long tri = upper ? V.tri_nnz_upper : V.tri_nnz_lower;
      const double bytes = 12.0 * (tri + V.n) + 4.0 * (V.n + 1) + 24.0 * V.n;
      static long long* dbg = nullptr;
      static const bool want_dbg = std::getenv("IGB_GS_DEBUG") != nullptr;
      if (want_dbg && !capturing) {
        if (!dbg) CU(cudaMalloc(&dbg, 8 * sizeof(long long)));
        a.dbg = dbg;
        const char* ab = std::getenv("IGB_GS_ABLATE");
        a.ablate = ab ? std::atoi(ab) : 0;
      }
      launch(K_GS, 20.0 * V.n, [&] { launch_perm_gather(stream, V.n, C.rows, rhs, V.rp); });
      launch(K_GS, bytes, [&] { launch_level_sweep(stream, a); });
      launch(K_GS, 20.0 * V.n + (u_zero ? 0.0 : 8.0 * V.n),
             [&] { launch_perm_scatter(stream, V.n, C.rows, V.xp, u, u_zero ? 0 : 1); });
      if (a.dbg) {
        long long h[8];
        CU(cudaMemcpyAsync(h, dbg, sizeof(h), cudaMemcpyDeviceToHost, stream));
        CU(cudaStreamSynchronize(stream));
        std::fprintf(stderr, "[gs dbg] level %d dir %d n %d steps %lld: %lld cyc/step\n", l, upper ? 1 : 0,
                     V.n, h[0], h[1] / (h[0] > 0 ? h[0] : 1));
      }
      return;
    }
    TrsvPhase ph{};
    const Sched& S = upper ? V.bwd : V.fwd;
    ph.nlev = S.nlev;
    ph.lvl_ptr = S.lvl_ptr;
    ph.rows = S.rows;
    ph.ptr = V.A.ptr;
    ph.col = V.A.col;
    ph.val = V.A.val;
    ph.dpos = V.dpos;
    ph.upper = upper ? 1 : 0;
    ph.rhs = rhs;
    ph.rhs_idx = nullptr;
    if (u_zero) {
      ph.x = u;
      ph.uacc = nullptr;
    } else {
      ph.x = V.c;
      ph.uacc = u;
    }
    const long long tri = upper ? V.tri_nnz_upper : V.tri_nnz_lower;
    const double bytes = 12.0 * (tri + V.n) + 4.0 * (V.n + 1) + 24.0 * V.n;
    launch(K_GS, bytes, [&] { launch_sptrsv(stream, ph, nullptr, 0, nullptr, nullptr); });
  }

  // u (+)= tau * SCMS(res)
  void scms(int l, const double* res, double* u, bool u_zero) {
    Level& V = lev[l];
    const FdPlan& F = V.fd;
    // the level's FD flops are booked on its first FD launch (class totals are what is reported)
    double flops = F.flops;
    for (size_t b = 0; b < F.batches.size(); ++b) {
      launch(K_FD, F.batch_bytes[b], [&] {
        launch_fd_batch(stream, F.batches[b], res, u, V.tau, u_zero ? 0 : 1);
      }, flops);
      flops = 0.0;
    }
    if (F.fd3.nitems) {
      for (int st = 0; st < 3; ++st) {
        launch(K_FD, F.fd3_bytes[st], [&] {
          launch_fd3(stream, F.fd3, st, res, u, V.tau, u_zero ? 0 : 1);
        }, flops);
        flops = 0.0;
      }
    }
    for (int s = 0; s < F.nsteps; ++s) {
      if (F.ndesc[s] == 0) continue;
      launch(K_FD, F.bytes[s], [&] {
        launch_fd_gemm(stream, F.d_desc[s], F.ndesc[s], F.tiles[s], res, u, V.tau, u_zero ? 0 : 1);
      }, flops);
      flops = 0.0;
    }
    if (!V.h_blocks.empty() && !V.pieces_fused) {
      launch(K_PIECES, V.piece_bytes, [&] {
        launch_piece_gemv(stream, V.d_blocks, (int)V.h_blocks.size(), res, u, V.tau, u_zero ? 0 : 1, V.piece_max_m);
      });
    }
  }

  void coarse_solve(const double* rhs, double* out) {
    Coarse& C = coarse;
    if (C.ndense) {
      const double bytes = 8.0 * C.n * (double)C.n + 24.0 * C.n;
      launch(K_COARSE, bytes, [&] { launch_piece_gemv(stream, C.d_dense, C.ndense, rhs, out, 1.0, 0, C.n); });
      return;
    }
    if (C.n > 7000) {  // rhs + column pointers no longer fit in shared memory
      coarse_solve_levels(rhs, out);
      return;
    }
    const double bytes = 12.0 * (C.L.nnz + C.U.nnz) + 8.0 * (C.L.n + 1) + 40.0 * C.n;
    launch(K_COARSE, bytes, [&] { launch_coarse_csc(stream, C.csc, rhs, out); });
  }

  void coarse_solve_levels(const double* rhs, double* out) {
    Coarse& C = coarse;
    TrsvPhase a{}, b{};
    a.nlev = C.Ls.nlev; a.lvl_ptr = C.Ls.lvl_ptr; a.rows = C.Ls.rows;
    a.ptr = C.L.ptr; a.col = C.L.col; a.val = C.L.val; a.dpos = C.Ldpos; a.upper = 0;
    a.rhs = rhs; a.rhs_idx = C.inv_perm_r; a.x = C.y; a.uacc = nullptr;
    b.nlev = C.Us.nlev; b.lvl_ptr = C.Us.lvl_ptr; b.rows = C.Us.rows;
    b.ptr = C.U.ptr; b.col = C.U.col; b.val = C.U.val; b.dpos = C.Udpos; b.upper = 1;
    b.rhs = C.y; b.rhs_idx = nullptr; b.x = C.w; b.uacc = nullptr;
    const double bytes = 12.0 * (C.L.nnz + C.U.nnz) + 8.0 * (C.L.n + 1) + 40.0 * C.n;
    launch(K_COARSE, bytes, [&] { launch_sptrsv(stream, a, &b, C.n, C.perm_c, out); });
  }

  void residual(int l, const double* f, const double* u, double* r) {
    apply_A(l, u, f, r, -1);
  }
  // CG: q = A_L d and alpha = rz / (d . q) (matrix-free product + dot, or the fused CSR kernel)
  void cg_matvec(cudaStream_t s) {
    Level& F = lev[L];
    const DevCsr& A = F.A;
    const int n = F.n;
    if (F.has_mf) {
      apply_A(L, d, nullptr, q, 0);
      launch(K_CG, 16.0 * n, [&] { launch_dot(s, n, d, q, partials, counter, sc, FIN_ALPHA, hist_dev); });
      return;
    }
    launch(K_SPMV, 12.0 * A.nnz + 4.0 * (n + 1) + 24.0 * n, [&] {
      launch_spmv_dot(s, n, A.ptr, A.col, A.val, d, q, A.group, partials, counter, sc, hist_dev);
    });
  }
  // y = z + sign A_l x (sign 0: y = A x): matrix-free where set, else CSR
  void apply_A(int l, const double* x, const double* z, double* y, int sign) {
    Level& V = lev[l];
    if (V.has_mf) {
      const double bytes = 8.0 * (2 * V.mf.nfree) + 4.0 * V.mf.nblk + 8.0 * 9 * V.mf.nblk;
      launch(K_SPMV, bytes, [&] { launch_mf_apply(stream, V.mf, x, z, y, sign, V.mf_s); });
      return;
    }
    spmv(V.A, x, z, y, sign, K_SPMV);
  }

  // One smoothing step kind: 'G' fwd GS, 'B' bwd GS, 'S' scms
  void smooth_step(int l, char kind, const double* f, double* u, bool& u_zero) {
    Level& V = lev[l];
    const double* res = f;
    if (!u_zero) {
      residual(l, f, u, V.r);
      res = V.r;
    }
    if (kind == 'S') scms(l, res, u, u_zero);
    else gs(l, kind == 'B', res, u, u_zero);
    u_zero = false;
  }
  // Gauss-Seidel step from a nonzero u without the full residual: u' = u + T^-1 (f - A u) solves
  // T u' = f - (A - T) u, T = tril(A) (fwd) or triu(A) (bwd) -- the other strict triangle is
  // half the matrix traffic of f - A u (same iterate up to rounding)
  void gs_step(int l, bool upper, const double* f, double* u, bool& u_zero) {
    Level& V = lev[l];
    if (u_zero || !V.has_U || V.has_mf) {  // matrix-free level: the full residual is the cheaper read
      smooth_step(l, upper ? 'B' : 'G', f, u, u_zero);
      return;
    }
    spmv(upper ? V.Lo : V.U, u, f, V.r, -1, K_SPMV);
    gs(l, upper, V.r, u, true);
    u_zero = false;
  }

  void pre_smooth(int l, const double* f, double* u, bool& uz) {
    const int st = steps[l];
    if (smoother == IGB_SMOOTHER_GS) {
      for (int i = 0; i < st; ++i) gs_step(l, false, f, u, uz);
    } else if (smoother == IGB_SMOOTHER_SCMS) {
      for (int i = 0; i < st; ++i) smooth_step(l, 'S', f, u, uz);
    } else {
      const bool from_zero = uz;
      smooth_step(l, 'G', f, u, uz);
      for (int i = 0; i < st; ++i) {
        Level& V = lev[l];
        if (i == 0 && from_zero && V.has_U && !V.has_mf) {
          // u = c with tril(A) c = f, so f - A u = -triu(A, 1) c: half the matrix traffic
          spmv(V.U, u, nullptr, V.r, -1, K_SPMV);
          scms(l, V.r, u, false);
        } else {
          smooth_step(l, 'S', f, u, uz);
        }
      }
    }
  }
  void post_smooth(int l, const double* f, double* u, bool& uz) {
    const int st = steps[l];
    if (smoother == IGB_SMOOTHER_GS) {
      for (int i = 0; i < st; ++i) gs_step(l, true, f, u, uz);
    } else if (smoother == IGB_SMOOTHER_SCMS) {
      for (int i = 0; i < st; ++i) smooth_step(l, 'S', f, u, uz);
    } else {
      for (int i = 0; i < st; ++i) smooth_step(l, 'S', f, u, uz);
      gs_step(l, true, f, u, uz);
    }
  }

  void restrict_residual(int l, const double* f, const double* u, bool uz, double* fc) {
    Level& V = lev[l];
    const double* res = f;
    if (!uz) {
      residual(l, f, u, V.r);
      res = V.r;
    }
    restrict_to(l, res, fc);
  }

  // cycle on level l: f -> u (u overwritten)
  void cycle(int l, const double* f, double* u) {
    Level& V = lev[l];
    bool uz = true;
    pre_smooth(l, f, u, uz);
    Level& C = lev[l - 1];
    restrict_residual(l, f, u, uz, C.f);
    if (l == 1) {
      coarse_solve(C.f, C.u);
      prolong(l, C.u, u, u, uz ? 0 : 1);
      uz = false;
    } else {
      for (int k = 0; k < mu; ++k) {
        cycle(l - 1, C.f, C.u);
        prolong(l, C.u, u, u, uz ? 0 : 1);
        uz = false;
        if (mu > 1) restrict_residual(l, f, u, uz, C.f);
      }
    }
    post_smooth(l, f, u, uz);
  }

  void run_finest_cycle() {
    // cycle(L): lev[L].f -> lev[L].u, replayed from a CUDA graph
    if (!cycle_exec || graph_prof != prof) {
      drop_graph();
      cudaGraph_t g;
      capturing = true;
      graph_kernels = 0;
      CU(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
      try {
        cycle(L, lev[L].f, lev[L].u);
      } catch (...) {
        cudaStreamEndCapture(stream, &g);
        capturing = false;
        throw;
      }
      CU(cudaStreamEndCapture(stream, &g));
      capturing = false;
      CU(cudaGraphInstantiate(&cycle_exec, g, 0));
      CU(cudaGraphDestroy(g));
      graph_prof = prof;
    }
    CU(cudaGraphLaunch(cycle_exec, stream));
    ++graph_replays;
  }
  void harvest_graph() {
    if (prof && !graph_recs.empty()) harvest(graph_recs, false);
  }
};

namespace {

int fail(igb_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

template <class F>
int guarded(igb_ctx* ctx, F&& f) {
  if (!ctx) return IGB_ERR_ARG;
  try {
    f();
    return IGB_OK;
  } catch (const ArgError& e) {
    return fail(ctx, IGB_ERR_ARG, e.what());
  } catch (const StateError& e) {
    return fail(ctx, IGB_ERR_STATE, e.what());
  } catch (const CudaError& e) {
    return fail(ctx, IGB_ERR_CUDA, e.what());
  } catch (const std::bad_alloc&) {
    return fail(ctx, IGB_ERR_NOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return fail(ctx, IGB_ERR_STATE, e.what());
  }
}

int pick_group(long long nnz, int n) {
  const double avg = n ? double(nnz) / n : 0;
  static const int forced = std::getenv("IGB_SPMV_GROUP") ? std::atoi(std::getenv("IGB_SPMV_GROUP")) : 0;
  if (forced == 4 || forced == 8 || forced == 16 || forced == 32) return forced;
  // measured on B200 (cfg2, 48 nnz/row): 8 lanes per row beats 16 and 32 -- more independent
  // loads per lane, fewer latency-bound waves of warps
  if (avg <= 6) return 4;
  if (avg <= 96) return 8;
  return avg <= 192 ? 16 : 32;  // long rows (3-D, p = 8): more lanes per row
}

void check_csr(int n, int m, long long nnz, const int* ptr, const int* idx) {
  if (n < 0 || m < 0 || nnz < 0) throw ArgError("negative dimension");
  if (!ptr || (nnz && !idx)) throw ArgError("null CSR array");
  if (ptr[0] != 0 || ptr[n] != nnz) throw ArgError("indptr does not match nnz");
  for (int i = 0; i < n; ++i)
    if (ptr[i + 1] < ptr[i]) throw ArgError("indptr not monotone");
  std::atomic<int> bad{0};
  parallel_for(n, [&](long long lo, long long hi) {
    for (long long i = lo; i < hi; ++i)
      for (int k = ptr[i]; k < ptr[i + 1]; ++k) {
        if (idx[k] < 0 || idx[k] >= m) bad |= 1;
        if (k > ptr[i] && idx[k] <= idx[k - 1]) bad |= 2;
      }
  });
  if (bad & 1) throw ArgError("column index out of range");
  if (bad & 2) throw ArgError("column indices must be sorted and unique");
}

DevCsr upload_csr(igb_ctx* ctx, int n, int m, long long nnz, const int* ptr, const int* idx,
                  const double* val) {
  DevCsr c;
  c.n = n;
  c.m = m;
  c.nnz = nnz;
  c.ptr = ctx->upload(ptr, (size_t)n + 1);
  c.col = ctx->upload(idx, (size_t)nnz);
  c.val = ctx->upload(val, (size_t)nnz);
  c.group = pick_group(nnz, n);
  return c;
}

// Diagonal position per row (must exist and be nonzero).
std::vector<int> diag_positions(int n, const int* ptr, const int* col, const double* val,
                                const char* what) {
  std::vector<int> dp(n);
  for (int i = 0; i < n; ++i) {
    const int* b = col + ptr[i];
    const int* e = col + ptr[i + 1];
    const int* it = std::lower_bound(b, e, i);
    if (it == e || *it != i) throw ArgError(std::string(what) + ": missing diagonal entry");
    dp[i] = int(it - col);
    if (val && val[dp[i]] == 0.0) throw ArgError(std::string(what) + ": zero diagonal entry");
  }
  return dp;
}

// Level sets of the lower (col < row) or upper (col > row) triangle.
Sched build_schedule(igb_ctx* ctx, int n, const int* ptr, const int* col, const std::vector<int>& dp,
                     bool upper) {
  std::vector<int> lv(n, 0);
  int maxl = -1;
  if (!upper) {
    for (int i = 0; i < n; ++i) {
      int l = 0;
      for (int k = ptr[i]; k < dp[i]; ++k) l = std::max(l, lv[col[k]] + 1);
      lv[i] = l;
      maxl = std::max(maxl, l);
    }
  } else {
    for (int i = n - 1; i >= 0; --i) {
      int l = 0;
      for (int k = dp[i] + 1; k < ptr[i + 1]; ++k) l = std::max(l, lv[col[k]] + 1);
      lv[i] = l;
      maxl = std::max(maxl, l);
    }
  }
  const int nlev = maxl + 1;
  std::vector<int> cnt(nlev + 1, 0), rows(n);
  for (int i = 0; i < n; ++i) cnt[lv[i] + 1]++;
  for (int l = 0; l < nlev; ++l) cnt[l + 1] += cnt[l];
  std::vector<int> pos(cnt.begin(), cnt.end() - 1);
  for (int i = 0; i < n; ++i) rows[pos[lv[i]]++] = i;
  Sched s;
  s.nlev = nlev;
  s.lvl_ptr = ctx->upload(cnt.data(), cnt.size());
  s.rows = ctx->upload(rows.data(), rows.size());
  return s;
}

void require_levels(igb_ctx* ctx) {
  if (ctx->L < 1) throw StateError("igb_set_num_levels must be called first");
}

void require_final(igb_ctx* ctx) {
  if (!ctx->finalized) throw StateError("igb_finalize has not been called");
}

void build_fd_plan(igb_ctx* ctx, Level& V) {
  if (V.interiors.empty()) return;
  // the level's dimension; a 3-D level may also carry 2-D items: faces between patches whose piece
  // matrix has tensor form are applied by 2-D fast diagonalisation (smoothers.py: _tensor_face)
  int dim = 2;
  for (auto& it : V.interiors) dim = std::max(dim, it.dim);
  V.fd.flops = 0.0;
  for (auto& it : V.interiors) {  // 2 d contractions (front + back), 2 flops per FMA
    const double cells = (double)it.n[0] * it.n[1] * (it.dim == 3 ? it.n[2] : 1);
    V.fd.flops += 4.0 * cells * (it.n[0] + it.n[1] + (it.dim == 3 ? it.n[2] : 0));
  }
  // 2-D interiors up to FDC_NMAX: one fused cluster each; the rest: batched GEMM steps
  std::vector<FdCluster> clu, clu_large;
  std::vector<InteriorStage> big;
  static const bool large_ok = !(std::getenv("IGB_FD_LARGE") && std::atoi(std::getenv("IGB_FD_LARGE")) == 0);
  const bool fuse = !(std::getenv("IGB_FD_FUSE") && std::string(std::getenv("IGB_FD_FUSE")) == "0");
  for (auto& it : V.interiors) {
    if (it.dim == 2 && (fuse || dim == 3) && it.n[0] <= FDC_NMAX && it.n[1] <= FDC_NMAX) {
      clu.push_back(FdCluster{it.T[0], it.T[1], it.D, it.idx, nullptr, it.n[0], it.n[1]});
    } else if (it.dim == 2 && dim == 3) {
      throw ArgError("2-D items of a 3-D level must fit the fused 2-D kernels (sides <= 160)");
    } else if (fuse && large_ok && dim == 2 && it.n[0] <= FDL_NMAX && it.n[1] <= FDL_NMAX) {
      clu_large.push_back(FdCluster{it.T[0], it.T[1], it.D, it.idx, nullptr, it.n[0], it.n[1]});
    } else {
      big.push_back(it);
    }
  }
  {
    // the chunked variant re-streams the right operand from L2 per CTA: measured better than the
    // batched GEMM for a few large interiors (cfg3: one 258^2, 22.2 vs 24.3 ms per solve), worse
    // for many (cfg4: sixteen 256^2, 27.4 vs 25.2 ms)
    long long rows = 0;
    for (auto& f : clu_large) rows += f.n0;
    if (rows > 1024) {
      for (auto& it : V.interiors)
        if (it.dim == 2 && std::max(it.n[0], it.n[1]) > FDC_NMAX && std::max(it.n[0], it.n[1]) <= FDL_NMAX)
          big.push_back(it);
      clu_large.clear();
    }
  }
  for (int large = 0; large < 2; ++large) {
    std::vector<FdCluster>& cl = large ? clu_large : clu;
    if (cl.empty()) continue;
    size_t tot = 0;
    for (auto& f : cl) tot += (size_t)f.n0 * f.n1;
    double* scratch = ctx->alloc<double>(tot);
    for (auto& f : cl) {
      f.scratch = scratch;
      scratch += (size_t)f.n0 * f.n1;
    }
    for (size_t b0 = 0; b0 < cl.size(); b0 += FD_BATCH_MAX) {
      FdBatch bt{};
      bt.large = large;
      bt.nitems = (int)std::min<size_t>(FD_BATCH_MAX, cl.size() - b0);
      int rows = 0;
      double bytes = 0;
      for (int i = 0; i < bt.nitems; ++i) {
        bt.items[i] = cl[b0 + i];
        rows += bt.items[i].n0;
        const double n0 = bt.items[i].n0, n1 = bt.items[i].n1;
        // T0 and T1 read twice, R gathered, D, A written + read, X scattered
        bytes += 16.0 * (n0 * n0 + n1 * n1) + (12.0 + 8 + 16 + 12) * n0 * n1;
      }
      bt.rb = fd_rows_per_cta(rows);
      bt.kmax = 1;
      for (int i = 0; i < bt.nitems; ++i) bt.kmax = std::max(bt.kmax, std::max(bt.items[i].n0, bt.items[i].n1));
      bt.cta0[0] = 0;
      for (int i = 0; i < bt.nitems; ++i) bt.cta0[i + 1] = bt.cta0[i] + (bt.items[i].n0 + bt.rb - 1) / bt.rb;
      V.fd.batches.push_back(bt);
      V.fd.batch_bytes.push_back(bytes);
    }
  }
  V.interiors = big;
  if (big.empty()) return;
  static const bool fd3_ok = !(std::getenv("IGB_FD3") && std::atoi(std::getenv("IGB_FD3")) == 0);
  if (dim == 3 && fd3_ok) {
    bool fits = true;
    int nmax = 1;
    for (auto& it : V.interiors)
      for (int a = 0; a < 3; ++a) {
        fits = fits && it.n[a] <= FD3_NMAX;
        nmax = std::max(nmax, it.n[a]);
      }
    if (fits) {
      size_t tot = 0;
      for (auto& it : V.interiors) tot += (size_t)it.n[0] * it.n[1] * it.n[2];
      V.fd_scratch = tot;
      V.s0 = ctx->alloc<double>(tot);
      V.s1 = ctx->alloc<double>(tot);
      std::vector<Fd3Item> items;
      Fd3Plan& P = V.fd.fd3;
      size_t off = 0;
      for (auto& it : V.interiors) {
        Fd3Item I{};
        for (int a = 0; a < 3; ++a) { I.T[a] = it.T[a]; I.n[a] = it.n[a]; }
        I.D = it.D; I.idx = it.idx;
        I.buf0 = V.s0 + off; I.buf1 = V.s1 + off;
        I.slab0 = P.slabs0; I.slab1 = P.slabs1;
        P.slabs0 += it.n[0]; P.slabs1 += it.n[1];
        const double cells = (double)it.n[0] * it.n[1] * it.n[2];
        off += (size_t)cells;
        // gather (idx + r) and Y written; Y, D read and W written; W, idx read and u updated
        V.fd.fd3_bytes[0] += 20.0 * cells; V.fd.fd3_bytes[1] += 24.0 * cells; V.fd.fd3_bytes[2] += 28.0 * cells;
        items.push_back(I);
      }
      P.nitems = (int)items.size();
      P.n8 = (nmax + 7) / 8 * 8;
      P.lr_shared = 1;
      for (auto& I : items) P.lr_shared &= (I.T[1] == I.T[2] && I.n[1] == I.n[2]) ? 1 : 0;
      if (std::getenv("IGB_FD3_BUF3")) P.lr_shared = 0;
      P.d_items = ctx->upload(items.data(), items.size());
      return;
    }
  }
  size_t total = 0;
  for (auto& it : V.interiors) total += (size_t)it.n[0] * it.n[1] * (dim == 3 ? it.n[2] : 1);
  V.fd_scratch = total;
  V.s0 = ctx->alloc<double>(total);
  V.s1 = ctx->alloc<double>(total);
  FdPlan& F = V.fd;
  F.nsteps = dim == 2 ? 4 : 6;
  std::vector<std::vector<GemmDesc>> steps(F.nsteps);
  size_t base = 0;
  for (auto& it : V.interiors) {
    const long long n0 = it.n[0], n1 = it.n[1], n2 = dim == 3 ? it.n[2] : 1;
    double* B0 = V.s0 + base;
    double* B1 = V.s1 + base;
    auto mk = [](int M, int N, int K, int nb) {
      GemmDesc g{};
      g.M = M; g.N = N; g.K = K; g.nb = nb;
      return g;
    };
    if (dim == 2) {
      GemmDesc g = mk(n0, n1, n0, 1);  // Z = T0^T R   (R gathered)
      g.A = it.T[0]; g.a_rs = 1; g.a_cs = n0;
      g.b_idx = it.idx; g.b_rs = n1; g.b_cs = 1;
      g.C = B0; g.c_rs = n1; g.c_cs = 1;
      steps[0].push_back(g);
      g = mk(n0, n1, n1, 1);  // Y = Z T1 / D
      g.A = B0; g.a_rs = n1; g.a_cs = 1;
      g.B = it.T[1]; g.b_rs = n1; g.b_cs = 1;
      g.C = B1; g.c_rs = n1; g.c_cs = 1; g.D = it.D;
      steps[1].push_back(g);
      g = mk(n0, n1, n0, 1);  // W = T0 Y
      g.A = it.T[0]; g.a_rs = n0; g.a_cs = 1;
      g.B = B1; g.b_rs = n1; g.b_cs = 1;
      g.C = B0; g.c_rs = n1; g.c_cs = 1;
      steps[2].push_back(g);
      g = mk(n0, n1, n1, 1);  // X = W T1^T -> u[idx] (+)= tau X
      g.A = B0; g.a_rs = n1; g.a_cs = 1;
      g.B = it.T[1]; g.b_rs = 1; g.b_cs = n1;
      g.c_idx = it.idx; g.c_rs = n1; g.c_cs = 1;
      steps[3].push_back(g);
    } else {
      const long long n12 = n1 * n2, n01 = n0 * n1;
      GemmDesc g = mk(n0, n12, n0, 1);  // mode 0 fwd (gather)
      g.A = it.T[0]; g.a_rs = 1; g.a_cs = n0;
      g.b_idx = it.idx; g.b_rs = n12; g.b_cs = 1;
      g.C = B0; g.c_rs = n12; g.c_cs = 1;
      steps[0].push_back(g);
      g = mk(n1, n2, n1, n0);  // mode 1 fwd, batched over i0
      g.A = it.T[1]; g.a_rs = 1; g.a_cs = n1; g.a_bs = 0;
      g.B = B0; g.b_rs = n2; g.b_cs = 1; g.b_bs = n12;
      g.C = B1; g.c_rs = n2; g.c_cs = 1; g.c_bs = n12;
      steps[1].push_back(g);
      g = mk(n01, n2, n2, 1);  // mode 2 fwd, divide
      g.A = B1; g.a_rs = n2; g.a_cs = 1;
      g.B = it.T[2]; g.b_rs = n2; g.b_cs = 1;
      g.C = B0; g.c_rs = n2; g.c_cs = 1; g.D = it.D;
      steps[2].push_back(g);
      g = mk(n0, n12, n0, 1);  // mode 0 back
      g.A = it.T[0]; g.a_rs = n0; g.a_cs = 1;
      g.B = B0; g.b_rs = n12; g.b_cs = 1;
      g.C = B1; g.c_rs = n12; g.c_cs = 1;
      steps[3].push_back(g);
      g = mk(n1, n2, n1, n0);  // mode 1 back, batched
      g.A = it.T[1]; g.a_rs = n1; g.a_cs = 1; g.a_bs = 0;
      g.B = B1; g.b_rs = n2; g.b_cs = 1; g.b_bs = n12;
      g.C = B0; g.c_rs = n2; g.c_cs = 1; g.c_bs = n12;
      steps[4].push_back(g);
      g = mk(n01, n2, n2, 1);  // mode 2 back -> scatter
      g.A = B0; g.a_rs = n2; g.a_cs = 1;
      g.B = it.T[2]; g.b_rs = 1; g.b_cs = n2;
      g.c_idx = it.idx; g.c_rs = n2; g.c_cs = 1;
      steps[5].push_back(g);
    }
    base += (size_t)n0 * n1 * n2;
  }
  for (int s = 0; s < F.nsteps; ++s) {
    int tb = 0;
    double bytes = 0;
    for (auto& g : steps[s]) {
      g.tiles_m = (g.M + 63) / 64;
      g.tiles_n = (g.N + 63) / 64;
      g.tile_base = tb;
      tb += g.tiles_m * g.tiles_n * g.nb;
      bytes += 8.0 * g.nb * ((double)g.M * g.N * 2.0) + 8.0 * (double)g.M * g.K;
      if (g.b_idx) bytes += 4.0 * g.K * (double)g.N;
      if (g.c_idx) bytes += 4.0 * g.M * (double)g.N + 8.0 * g.M * (double)g.N;
    }
    F.ndesc[s] = (int)steps[s].size();
    F.tiles[s] = tb;
    F.bytes[s] = bytes;
    F.d_desc[s] = ctx->upload(steps[s].data(), steps[s].size());
  }
}

}  // namespace

// ============================================================================ C ABI
extern "C" {

int igb_version(void) { return 1; }

int igb_create(igb_ctx** out, int device) {
  if (!out) return IGB_ERR_ARG;
  *out = nullptr;
  igb_ctx* ctx = new (std::nothrow) igb_ctx();
  if (!ctx) return IGB_ERR_NOMEM;
  int rc = guarded(ctx, [&] {
    int count = 0;
    CU(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw ArgError("no such CUDA device");
    ctx->device = device;
    CU(cudaSetDevice(device));
    carveout_prepare();
    CU(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    CU(cudaEventCreate(&ctx->t0));
    CU(cudaEventCreate(&ctx->t1));
    CU(cudaMallocHost(&ctx->sc_host, sizeof(CgScalars)));
  });
  if (rc != IGB_OK) {
    std::fprintf(stderr, "igb_create: %s\n", ctx->err.c_str());
    delete ctx;
    return rc;
  }
  *out = ctx;
  return IGB_OK;
}

int igb_destroy(igb_ctx* ctx) {
  if (!ctx) return IGB_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  ctx->drop_graph();
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  for (void* p : ctx->allocs) cudaFree(p);
  if (ctx->sc_host) cudaFreeHost(ctx->sc_host);
  if (ctx->hist_host) cudaFreeHost(ctx->hist_host);
  for (int i = 0; i < 2; ++i) {
    if (ctx->stage[i]) cudaFreeHost(ctx->stage[i]);
    if (ctx->stage_ev[i]) cudaEventDestroy(ctx->stage_ev[i]);
  }
  if (ctx->t0) cudaEventDestroy(ctx->t0);
  if (ctx->t1) cudaEventDestroy(ctx->t1);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return IGB_OK;
}

const char* igb_last_error(igb_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int igb_set_num_levels(igb_ctx* ctx, int L) {
  return guarded(ctx, [&] {
    if (L < 1) throw ArgError("need at least one refinement level (L >= 1)");
    if (ctx->L >= 0) throw StateError("hierarchy already sized");
    ctx->L = L;
    ctx->lev.resize(L + 1);
    ctx->steps.assign(L + 1, 1);
  });
}

int igb_set_level_matrix(igb_ctx* ctx, int level, int n, long long nnz, const int* indptr,
                         const int* indices, const double* data) {
  return guarded(ctx, [&] {
    require_levels(ctx);
    CU(cudaSetDevice(ctx->device));
    Level& V = ctx->level(level);
    if (V.n) throw StateError("level matrix already set");
    if (n < 1) throw ArgError("empty level matrix");
    if (nnz >= (1LL << 31)) throw ArgError("nnz exceeds int32 indexing");
    check_csr(n, n, nnz, indptr, indices);
    V.n = n;
    V.A = upload_csr(ctx, n, n, nnz, indptr, indices, data);
    V.h_ptr.assign(indptr, indptr + n + 1);
    V.h_col.resize(nnz);
    V.h_val.resize(nnz);
    par_memcpy(V.h_col.data(), indices, sizeof(int) * (size_t)nnz);
    par_memcpy(V.h_val.data(), data, sizeof(double) * (size_t)nnz);
    std::vector<int> dp = diag_positions(n, indptr, indices, data, "A");
    V.dpos = ctx->upload(dp.data(), dp.size());
    V.tri_nnz_lower = V.tri_nnz_upper = 0;
    for (int i = 0; i < n; ++i) {
      V.tri_nnz_lower += dp[i] - indptr[i];
      V.tri_nnz_upper += indptr[i + 1] - dp[i] - 1;
    }
    // +2: 16-byte gathers of the chain sweep may read one element past the end
    V.f = ctx->alloc<double>(n + 2);
    V.u = ctx->alloc<double>(n + 2);
    V.r = ctx->alloc<double>(n + 2);
    V.c = ctx->alloc<double>(n + 2);
  });
}

int igb_set_prolongation(igb_ctx* ctx, int level, int n_fine, int n_coarse, long long nnz,
                         const int* indptr, const int* indices, const double* data) {
  return guarded(ctx, [&] {
    require_levels(ctx);
    CU(cudaSetDevice(ctx->device));
    if (level < 1 || level > ctx->L) throw ArgError("prolongation level must be in 1..L");
    Level& V = ctx->lev[level];
    if (V.has_P) throw StateError("prolongation already set");
    check_csr(n_fine, n_coarse, nnz, indptr, indices);
    V.P = upload_csr(ctx, n_fine, n_coarse, nnz, indptr, indices, data);
    // transpose on the host (CSR of P^T, sorted columns by construction)
    std::vector<int> tp(n_coarse + 1, 0), ti(nnz);
    std::vector<double> tv(nnz);
    for (long long k = 0; k < nnz; ++k) tp[indices[k] + 1]++;
    for (int j = 0; j < n_coarse; ++j) tp[j + 1] += tp[j];
    std::vector<int> pos(tp.begin(), tp.end() - 1);
    for (int i = 0; i < n_fine; ++i)
      for (int k = indptr[i]; k < indptr[i + 1]; ++k) {
        const int p = pos[indices[k]]++;
        ti[p] = i;
        tv[p] = data[k];
      }
    V.PT = upload_csr(ctx, n_coarse, n_fine, nnz, tp.data(), ti.data(), tv.data());
    V.has_P = true;
  });
}

int igb_set_prolongation_kron(igb_ctx* ctx, int level, int dim, int npatch, const int* nf, const int* nc,
                              int width, const int* p1_idx, const double* p1_val, const int* fine_free,
                              const int* fine_owner, const int* coarse_free) {
  return guarded(ctx, [&] {
    require_levels(ctx);
    CU(cudaSetDevice(ctx->device));
    if (level < 1 || level > ctx->L) throw ArgError("prolongation level must be in 1..L");
    Level& V = ctx->lev[level];
    Level& C = ctx->lev[level - 1];
    if (!V.n || !C.n) throw StateError("set the level matrices before the prolongation");
    if (V.has_kron) throw StateError("Kronecker prolongation already set");
    if (dim != 2 && dim != 3) throw ArgError("Kronecker prolongation needs dim 2 or 3");
    if (npatch < 1) throw ArgError("need at least one patch");
    if (npatch > KRON_MAXP) return;  // more patches than the parameter tables: CSR transfer stays
    if (width < 1 || !nf || !nc || !p1_idx || !p1_val || !fine_free || !fine_owner || !coarse_free)
      throw ArgError("null Kronecker prolongation array");
    KronArgs& a = V.kron;
    a = KronArgs{};
    a.dim = dim;
    a.npatch = npatch;
    const int Wd = kron_width(width);  // device ELL width (compiled variants)
    a.width = Wd;
    a.n_fine = V.n;
    a.n_coarse = C.n;
    std::vector<KronPatch> pt(npatch);
    std::vector<long long> off_f(npatch + 1, 0), off_c(npatch + 1, 0);
    long long rows = 0;
    for (int k = 0; k < npatch; ++k) {
      long long pf = 1, pc = 1;
      for (int d = 0; d < 3; ++d) {
        pt[k].nf[d] = d < dim ? nf[k * dim + d] : 1;
        pt[k].nc[d] = d < dim ? nc[k * dim + d] : 1;
        if (pt[k].nf[d] < 1 || pt[k].nc[d] < 1) throw ArgError("empty patch block");
        pt[k].ell[d] = pt[k].ellT[d] = 0;
      }
      for (int d = 0; d < dim; ++d) {
        pt[k].ell[d] = rows * Wd;
        rows += pt[k].nf[d];
        pf *= pt[k].nf[d];
        pc *= pt[k].nc[d];
      }
      off_f[k + 1] = off_f[k] + pf;
      off_c[k + 1] = off_c[k] + pc;
    }
    const long long bf = off_f[npatch], bc = off_c[npatch];
    a.nblk_f = bf;
    a.nblk_c = bc;
    if (Wd < 0) return;  // wider 1-D rows than any compiled variant: the CSR transfer stays
    std::vector<int> pidx((size_t)rows * Wd, -1);
    std::vector<double> pval((size_t)rows * Wd, 0.0);
    // 1-D transposes (ELL rows of widthT, fine index ascending)
    std::vector<std::vector<std::pair<int, double>>> trows;
    int wt = 1;
    for (int k = 0; k < npatch; ++k)
      for (int d = 0; d < dim; ++d) {
        std::vector<std::vector<std::pair<int, double>>> t(pt[k].nc[d]);
        for (int i = 0; i < pt[k].nf[d]; ++i)
          for (int jj = 0; jj < width; ++jj) {
            const long long e = (pt[k].ell[d] / Wd + i) * width + jj;  // input rows have `width`
            const int c = p1_idx[e];
            if (c < 0) continue;
            if (c >= pt[k].nc[d]) throw ArgError("1-D prolongation column out of range");
            t[c].emplace_back(i, p1_val[e]);
            pidx[(pt[k].ell[d] / Wd + i) * Wd + jj] = c;
            pval[(pt[k].ell[d] / Wd + i) * Wd + jj] = p1_val[e];
          }
        pt[k].ellT[d] = (long long)trows.size();  // rows; scaled by widthT below
        for (auto& r : t) {
          wt = std::max(wt, (int)r.size());
          trows.push_back(std::move(r));
        }
      }
    wt = kron_width_t(wt);
    if (wt < 0) return;
    a.widthT = wt;
    for (int k = 0; k < npatch; ++k)
      for (int d = 0; d < dim; ++d) pt[k].ellT[d] *= wt;
    std::vector<int> ti(trows.size() * wt, -1);
    std::vector<double> tv(trows.size() * wt, 0.0);
    for (size_t r = 0; r < trows.size(); ++r)
      for (size_t jj = 0; jj < trows[r].size(); ++jj) {
        ti[r * wt + jj] = trows[r][jj].first;
        tv[r * wt + jj] = trows[r][jj].second;
      }
    // fine: every free DoF has exactly one owner copy; coarse: root copy + list of the others
    std::vector<int> fown(bf, -1), seen(V.n, 0);
    for (long long b = 0; b < bf; ++b) {
      const int f = fine_free[b];
      if (f < -1 || f >= V.n) throw ArgError("fine block map out of range");
      if (f >= 0 && fine_owner[b]) {
        if (seen[f]++) throw ArgError("fine free DoF with two owner copies");
        fown[b] = f;
      }
    }
    for (int f = 0; f < V.n; ++f)
      if (!seen[f]) throw ArgError("fine free DoF without an owner copy");
    std::vector<int> croot(bc, -1), xptr(C.n + 1, 0), xblk, first(C.n, -1);
    for (long long b = 0; b < bc; ++b) {
      const int jj = coarse_free[b];
      if (jj < -1 || jj >= C.n) throw ArgError("coarse block map out of range");
      if (jj < 0) continue;
      if (first[jj] < 0) {
        first[jj] = (int)b;
        croot[b] = jj;
      } else {
        xptr[jj + 1]++;
      }
    }
    for (int jj = 0; jj < C.n; ++jj) {
      if (first[jj] < 0) throw ArgError("coarse free DoF without a block copy");
      xptr[jj + 1] += xptr[jj];
    }
    xblk.resize(xptr[C.n]);
    std::vector<int> pos(xptr.begin(), xptr.end() - 1);
    for (long long b = 0; b < bc; ++b) {
      const int jj = coarse_free[b];
      if (jj >= 0 && first[jj] != (int)b) xblk[pos[jj]++] = (int)b;
    }
    for (int k = 0; k < npatch; ++k) a.patch[k] = pt[k];
    for (int k = 0; k <= npatch; ++k) {
      a.off_f[k] = off_f[k];
      a.off_c[k] = off_c[k];
    }
    a.pidx = ctx->upload(pidx.data(), pidx.size());
    a.pval = ctx->upload(pval.data(), pval.size());
    a.tidx = ctx->upload(ti.data(), ti.size());
    a.tval = ctx->upload(tv.data(), tv.size());
    a.fown = ctx->upload(fown.data(), fown.size());
    a.cfree = ctx->upload(coarse_free, (size_t)bc);
    a.croot = ctx->upload(croot.data(), croot.size());
    a.xptr = ctx->upload(xptr.data(), xptr.size());
    a.xblk = xblk.empty() ? ctx->alloc<int>(1) : ctx->upload(xblk.data(), xblk.size());
    // measured on B200 (cfg2, cfg5 L=3): the CSR pair is ~3 us per launch faster at these sizes
    // (transfers are latency-bound; the Kronecker gather chain is one memory latency longer),
    // so the Kronecker form is opt-in: IGB_TRANSFER=kron
    const char* te = std::getenv("IGB_TRANSFER");
    V.has_kron = te && std::string(te) == "kron";
  });
}

int igb_set_matrix_free(igb_ctx* ctx, int level, int dim, int npatch, int p, const int* dims, const double* c,
                        const double* Mband, const double* Kband, const int* block_free) {
  return guarded(ctx, [&] {
    require_levels(ctx);
    CU(cudaSetDevice(ctx->device));
    Level& V = ctx->level(level);
    if (!V.n) throw StateError("set the level matrix before its matrix-free form");
    if (dim != 2 && dim != 3) throw ArgError("matrix-free operator needs dim 2 or 3");
    if (npatch < 1 || p < 0 || !dims || !c || !Mband || !Kband || !block_free) throw ArgError("bad matrix-free arguments");
    if (npatch > MF_MAXP) return;  // more patches than the parameter tables: CSR stays
    MfArgs& a = V.mf;
    a = MfArgs{};
    a.dim = dim;
    a.npatch = npatch;
    a.p = p;
    a.nfree = V.n;
    long long nb = 0, band = 0;
    for (int k = 0; k < npatch; ++k) {
      a.off[k] = nb;
      long long sz = 1;
      for (int d = 0; d < 3; ++d) {
        a.n[k][d] = d < dim ? dims[k * dim + d] : 1;
        a.c[k][d] = d < dim ? c[k * dim + d] : 0.0;
        if (a.n[k][d] < 1) throw ArgError("empty patch block");
      }
      for (int d = 0; d < dim; ++d) {
        a.band[k][d] = band;
        band += (long long)a.n[k][d] * (2 * p + 1);
        sz *= a.n[k][d];
      }
      nb += sz;
    }
    a.off[npatch] = nb;
    a.nblk = nb;
    std::vector<int> froot(V.n, -1), xptr(V.n + 1, 0), xblk;
    for (long long b = 0; b < nb; ++b) {
      const int f = block_free[b];
      if (f < -1 || f >= V.n) throw ArgError("block map out of range");
      if (f < 0) continue;
      if (froot[f] < 0) froot[f] = (int)b;
      else xptr[f + 1]++;
    }
    for (int f = 0; f < V.n; ++f) {
      if (froot[f] < 0) throw ArgError("free DoF without a block copy");
      xptr[f + 1] += xptr[f];
    }
    xblk.resize(xptr[V.n]);
    std::vector<int> pos(xptr.begin(), xptr.end() - 1);
    for (long long b = 0; b < nb; ++b) {
      const int f = block_free[b];
      if (f >= 0 && froot[f] != (int)b) xblk[pos[f]++] = (int)b;
    }
    a.Mb = ctx->upload(Mband, (size_t)band);
    a.Kb = ctx->upload(Kband, (size_t)band);
    a.bfree = ctx->upload(block_free, (size_t)nb);
    a.froot = ctx->upload(froot.data(), froot.size());
    a.xptr = ctx->upload(xptr.data(), xptr.size());
    a.xblk = xblk.empty() ? ctx->alloc<int>(1) : ctx->upload(xblk.data(), xblk.size());
    for (int i = 0; i < 4; ++i) V.mf_s[i] = ctx->alloc<double>((size_t)nb);
    const char* me = std::getenv("IGB_MATRIX_FREE");
    V.has_mf = !(me && std::string(me) == "0");
  });
}

// Row-panel sweep for one direction (panel_plan.h).  Chosen when the panel chain
// (npan) is clearly shorter than the DAG depth (nlev) or when forced; cluster of 16
// CTAs (B = 512) if the device can host it, else 8 (B = 256).
bool build_panel_sweep(igb_ctx* ctx, Level& V, int level, int dir, const std::vector<int>& dp, int nlev,
                       bool force) {
  // shapes: B = 512 (16 warps, 8K ring) first; B = 256 (8 warps, 16K ring, more entry slots
  // per row) when the rows carry more entries than the first shape's kernel variants hold
  static int shapes_ok = -1;  // bit 0: KBC 17, bit 1: KBC 9
  static int max_clu[2] = {1, 1};
  const int G = 16;
  if (shapes_ok < 0) {
    shapes_ok = (panel_prepare(G, 17) ? 1 : 0) | (panel_prepare(G, 9) ? 2 : 0);
    for (int sh = 0; sh < 2; ++sh) {
      PanelArgs probe{};
      probe.KBC = sh ? 9 : 17;
      probe.B = sh ? 256 : 512;
      probe.R = sh ? 16384 : 8192;
      max_clu[sh] = panel_max_clusters(G, probe.KBC, panel_smem_bytes(probe));
      if (const char* ce = std::getenv("IGB_PANEL_CLUSTERS"))
        max_clu[sh] = std::max(1, std::min(max_clu[sh], std::atoi(ce)));
      max_clu[sh] = std::min(max_clu[sh], 8);
    }
  }
  PanelPlanHost plan;
  bool built = false;
  for (int sh = 0; sh < 2 && !built; ++sh) {
    if (!(shapes_ok >> sh & 1)) continue;
    const int W = sh ? 8 : 16, R = sh ? 16384 : 8192, B = 2 * G * W;
    const int npan = (V.n + B - 1) / B;
    if (!force && 2 * npan > nlev) continue;
    // The B = 256 KF 10 variant (panel_sweep_kernel<9,12,10>) has an unresolved wrong-result mode:
    // forced onto a 3-D level (cfg5 L=2 backward) the residual history drifts by up to 9e-2 from run to
    // run (DESIGN 9.2, profiles/r1l_kf10_3d_diag.log).  It is therefore OFF by default on every level;
    // IGB_PANEL_KF10=1 opts in (2-D levels), IGB_PANEL_KF10_3D=1 also on 3-D levels (diagnostic).
    // Levels whose rows need it fall back to the B = 512 single-range plan or the flow engine.
    // read per call (not cached): tests switch them between contexts of one process
    const bool kf10 = std::getenv("IGB_PANEL_KF10") && std::atoi(std::getenv("IGB_PANEL_KF10")) != 0;
    const bool kf10_3d = std::getenv("IGB_PANEL_KF10_3D") && std::atoi(std::getenv("IGB_PANEL_KF10_3D"));
    const bool two_d = !V.interiors.empty() && V.interiors[0].dim == 2;
    const bool allow_kf10 = kf10_3d || (kf10 && two_d);
    built = build_panel_plan(V.n, V.h_ptr.data(), V.h_col.data(), V.h_val.data(), dp.data(), dir == 1, G, W, R,
                             max_clu[sh], plan, sh == 1 && allow_kf10);
    // B = 512 fell back to one range with the long-row variant (KA 14; cfg4 p = 8 backward): B = 256
    // may run several ranges and finish sooner (a B = 256 panel costs about as much as a B = 512 one,
    // ~3 us) -- with KF <= 8 unless KF 10 is opted in.
    // IGB_PANEL_HALF: 0 off, 1 (default) the KA 14 case only, 2 every single-range B = 512 plan (diagnostic)
    const int half_mode = std::getenv("IGB_PANEL_HALF") ? std::atoi(std::getenv("IGB_PANEL_HALF")) : 1;
    if (built && sh == 0 && plan.nclu == 1 && (plan.KA == 14 || half_mode == 2) && max_clu[0] > 1 && half_mode &&
        (shapes_ok & 2)) {
      PanelPlanHost alt;
      if (build_panel_plan(V.n, V.h_ptr.data(), V.h_col.data(), V.h_val.data(), dp.data(), dir == 1, G, 8, 16384,
                           max_clu[1], alt, allow_kf10) &&
          alt.nclu > 1 && alt.makespan < 0.8 * plan.makespan)
        plan = std::move(alt);
    }
  }
  if (!built) return false;
  PanelDev& P = V.panel[dir];
  PanelArgs& a = P.args;
  a = PanelArgs{};
  a.n = V.n;
  a.npan = plan.npan;
  a.B = plan.B;
  a.R = plan.R;
  a.G = plan.G;
  a.KBC = plan.KBC;
  a.KA = plan.KA;
  a.KF = plan.KF;
  a.upper = dir;
  a.nclu = plan.nclu;
  for (int c = 0; c <= plan.nclu; ++c) {
    a.split[c] = plan.split[c];
    a.rstart[c] = plan.rstart[c];
  }
  if (const char* h = std::getenv("IGB_PANEL_NOHINT")) a.ablate |= std::atoi(h) ? 128 : 0;
  if (const char* h = std::getenv("IGB_PANEL_ALLSLOTS")) a.ablate |= std::atoi(h) ? 256 : 0;
  const char* pf = std::getenv("IGB_PANEL_PF");
  a.pf = pf ? std::max(0, std::atoi(pf)) : 0;  // bulk L2 prefetch distance (measured: no gain)
  if (panel_smem_bytes(a) > 227u * 1024) return false;
  a.lin = ctx->upload(plan.lin.data(), plan.lin.size());
  a.ev = ctx->upload(plan.ev.data(), plan.ev.size());
  a.ec = ctx->upload(plan.ec.data(), plan.ec.size());
  a.xmask = ctx->upload(plan.xmask.data(), plan.xmask.size());
  a.xcnt = ctx->upload(plan.xcnt.data(), plan.xcnt.size());
  if (plan.KF > 0) {
    a.fv = ctx->upload(plan.fv.data(), plan.fv.size());
    a.fc = ctx->upload(plan.fc.data(), plan.fc.size());
    // per level and direction: [2][n] copy, every entry "not produced yet" (panel.cu)
    std::vector<unsigned long long> pend((size_t)2 * V.n, 0x7FF4DEADBEEF1234ULL);
    a.xg = reinterpret_cast<double*>(ctx->upload(pend.data(), pend.size()));
    int* ctr = ctx->alloc<int>(2);
    CU(cudaMemset(ctr, 0, 2 * sizeof(int)));
    a.par_ctr = ctr;
    a.done_ctr = reinterpret_cast<unsigned*>(ctr + 1);
  }
  P.npan = plan.npan;
  P.near = plan.near_entries;
  P.far = plan.far_entries;
  P.lin_bytes = 8.0 * plan.lin.size();
  P.ent_bytes = 12.0 * plan.ev.size() + 12.0 * plan.fv.size() * plan.npan / (plan.npan + 1);
  P.ok = true;
  if (std::getenv("IGB_VERBOSE"))
    std::fprintf(stderr,
                 "[igb] level %d dir %d: panel sweep n %d depth %d panels %d (G %d B %d) KA %d KF %d near %lld far %lld "
                 "inverse %.1f MB growth %.2f smem %zu x-messages/value %.2f clusters %d (panel-times %.0f of %d)\n",
                 level, dir, V.n, nlev, plan.npan, plan.G, plan.B, plan.KA, plan.KF, plan.near_entries,
                 plan.far_entries, P.lin_bytes / 1e6, plan.max_inv_ratio, panel_smem_bytes(a),
                 double(plan.x_messages) / V.n, plan.nclu, plan.makespan, plan.npan);
  return true;
}

double flow_min_width() {
  static double w = -1;
  if (w < 0) {
    const char* e = std::getenv("IGB_FLOW_MIN_WIDTH");
    w = e ? std::atof(e) : 96.0;
  }
  return w;
}

// Wave sweep for one direction (wave_plan.h, wave.cu).
bool build_wave_sweep(igb_ctx* ctx, Level& V, int level, int dir, const std::vector<int>& dp) {
  const char* mn = std::getenv("IGB_WAVE_RBMIN");
  const char* mx = std::getenv("IGB_WAVE_RBMAX");
  const char* le = std::getenv("IGB_WAVE_CRITLAG");
  const char* lm = std::getenv("IGB_WAVE_LATE");
  const char* ll = std::getenv("IGB_WAVE_LATELAG");
  const int late_lag = ll ? std::max(0, std::atoi(ll)) : 9;
  const int rb_min = mn ? std::max(1, std::atoi(mn)) : 32;
  const int rb_cap = mx ? std::max(64, std::atoi(mx)) : 8192;
  const int lag = le ? std::max(1, std::atoi(le)) : 4;
  const int late_max = lm ? std::max(0, std::atoi(lm)) : 32;
  int cap = wave_max_ctas(wave_smem_bytes(rb_cap));
  if (const char* ce = std::getenv("IGB_WAVE_CTAS")) cap = std::min(cap, std::max(1, std::atoi(ce)));
  if (cap < 1) return false;
  WavePlanHost plan;
  if (!build_wave_plan(V.n, V.h_ptr.data(), V.h_col.data(), V.h_val.data(), dp.data(), dir == 1, rb_min, rb_cap,
                       late_lag, lag, late_max, cap, plan)) {
    if (std::getenv("IGB_VERBOSE"))
      std::fprintf(stderr, "[igb] level %d dir %d: no wave plan (bundles %d, occupancy %d of %d CTAs)\n", level, dir,
                   plan.nb, plan.occupancy, cap);
    return false;
  }
  WaveDev& D = V.wave[dir];
  WaveArgs& a = D.args;
  a = WaveArgs{};
  a.n = V.n;
  a.nb = plan.nb;
  a.nq = plan.nq;
  a.rb_max = plan.rb_max;
  a.xs_len = wave_xs_len(plan.rb_max);
  a.ctas = std::min(cap, std::max(1, wave_max_ctas(wave_smem_bytes(plan.rb_max))));
  a.b_frame = ctx->upload(plan.b_frame.data(), plan.b_frame.size());
  a.b_start = ctx->upload(plan.b_start.data(), plan.b_start.size());
  a.f_end = ctx->upload(plan.f_end.data(), plan.f_end.size());
  a.hdr = ctx->upload(plan.hdr.data(), plan.hdr.size());
  a.lcol = ctx->upload(plan.lcol.data(), plan.lcol.size());
  a.lval = ctx->upload(plan.lval.data(), plan.lval.size());
  a.recA = ctx->upload(plan.recA.data(), plan.recA.size());
  a.recB = ctx->upload(plan.recB.data(), plan.recB.size());
  a.e_row = plan.nq ? ctx->upload(plan.e_row.data(), plan.e_row.size()) : ctx->alloc<int>(1);
  a.eptr = ctx->upload(plan.eptr.data(), plan.eptr.size());
  a.ecol = plan.external ? ctx->upload(plan.ecol.data(), plan.ecol.size()) : ctx->alloc<int>(1);
  a.eval = plan.external ? ctx->upload(plan.eval.data(), plan.eval.size()) : ctx->alloc<double>(1);
  a.crit = plan.nq ? ctx->upload(plan.crit.data(), plan.crit.size()) : ctx->alloc<int>(1);
  a.elate = plan.nq ? ctx->upload(plan.elate.data(), plan.elate.size()) : ctx->alloc<int>(1);
  const char* be = std::getenv("IGB_WAVE_BACKOFF");
  a.backoff = be ? std::atoi(be) : 128;
  const char* pbe = std::getenv("IGB_WAVE_PBACKOFF");
  a.pbackoff = pbe ? std::atoi(pbe) : 32;
  std::vector<unsigned long long> pend((size_t)2 * V.n, 0x7FF4DEADBEEF2468ULL);  // wave.cu WAVE_PENDING
  a.xg = reinterpret_cast<double*>(ctx->upload(pend.data(), pend.size()));
  a.eg = reinterpret_cast<double*>(ctx->upload(pend.data(), pend.size()));
  int* ctr = ctx->alloc<int>(4);
  CU(cudaMemset(ctr, 0, 4 * sizeof(int)));
  a.par_ctr = ctr;
  a.done_ctr = reinterpret_cast<unsigned*>(ctr + 1);
  a.ticket = ctr + 2;
  D.nlev = plan.nlev;
  D.nframes = plan.nframes;
  D.occupancy = plan.occupancy;
  D.internal = plan.internal;
  D.external = plan.external;
  // external entries, lane records (32 B each), slot headers, external-list metadata, vectors
  D.stream_bytes = 12.0 * plan.external + 32.0 * plan.recA.size() + (16.0 + 12.0 * WAVE_LN) * V.n + 20.0 * plan.nq +
                   56.0 * V.n;
  D.ok = true;
  if (std::getenv("IGB_VERBOSE"))
    std::fprintf(stderr, "[igb] level %d dir %d: wave sweep n %d depth %d bundles %d (max rows %d, widest level %d) frames %d "
                 "internal %lld demoted %lld late %lld external %lld (%d rows) occupancy %d ctas %d stream %.1f MB\n", level, dir,
                 V.n, plan.nlev, plan.nb, plan.rb_max, plan.max_level_rows, plan.nframes, plan.internal, plan.demoted,
                 plan.late, plan.external, plan.nq, plan.occupancy, a.ctas, D.stream_bytes / 1e6);
  return true;
}

// Line sweep for one direction (line_plan.h, line.cu).
bool build_line_sweep(igb_ctx* ctx, Level& V, int level, int dir, const std::vector<int>& dp) {
  const char* mn = std::getenv("IGB_LINE_RBMIN");
  const char* mx = std::getenv("IGB_LINE_RBMAX");
  const int rb_min = mn ? std::max(1, std::atoi(mn)) : 512;
  const int rb_cap = mx ? std::max(64, std::atoi(mx)) : 8192;
  LinePlanHost plan;
  if (!build_line_plan(V.n, V.h_ptr.data(), V.h_col.data(), V.h_val.data(), dp.data(), dir == 1, rb_min, rb_cap, 8,
                       plan))
    return false;

  const size_t smem = 8 * ((size_t)plan.rb_max + 1);
  const int cap = line_max_ctas(smem);
  if (cap < 1) return false;
  LineDev& D = V.line[dir];
  LineArgs& a = D.args;
  a = LineArgs{};
  a.n = V.n;
  a.nb = plan.nb;
  a.rb_max = plan.rb_max;
  a.C = plan.C;
  a.upper = dir;
  a.ctas = std::min(cap, plan.nb);
  a.bstart = ctx->upload(plan.bstart.data(), plan.bstart.size());
  a.bline = ctx->upload(plan.bline.data(), plan.bline.size());
  a.lstart = ctx->upload(plan.lstart.data(), plan.lstart.size());
  // padded: the L2 bulk prefetch of the records runs a few rows past the end
  plan.rec.resize(plan.rec.size() + (size_t)line_rec_bytes(plan.C) * 16 / 8, 0.0);
  a.rec = reinterpret_cast<const char*>(ctx->upload(plan.rec.data(), plan.rec.size()));
  a.ocol = ctx->upload(plan.ocol.data(), plan.ocol.size());
  a.oval = ctx->upload(plan.oval.data(), plan.oval.size());
  const char* pfe = std::getenv("IGB_LINE_PF");
  a.pf = pfe ? std::max(1, std::atoi(pfe)) : 8;
  std::vector<unsigned long long> pend((size_t)2 * V.n, 0x7FF4DEADBEEF9ABCULL);  // line.cu LINE_PENDING
  a.xg = reinterpret_cast<double*>(ctx->upload(pend.data(), pend.size()));
  int* ctr = ctx->alloc<int>(2);
  CU(cudaMemset(ctr, 0, 2 * sizeof(int)));
  a.par_ctr = ctr;
  a.done_ctr = reinterpret_cast<unsigned*>(ctr + 1);
  D.entries = plan.entries;
  D.slots = plan.chunks * 32;
  D.nl = plan.nl;
  D.max_line = plan.max_line;
  D.ok = true;
  if (std::getenv("IGB_VERBOSE"))
    std::fprintf(stderr, "[igb] level %d dir %d: line sweep n %d lines %d (max %d) bundles %d (max rows %d) C %d "
                 "(max %d, %lld overflow rows) entries %lld records %.1f MB ctas %d\n", level, dir, V.n, plan.nl,
                 plan.max_line, plan.nb, plan.rb_max, plan.C, plan.cmax, plan.ovf_rows, plan.entries,
                 8.0 * plan.rec.size() / 1e6, a.ctas);
  return true;
}

// Dependency-driven whole-GPU sweep for one direction (flow_plan.h, flow.cu).
bool build_flow_sweep(igb_ctx* ctx, Level& V, int level, int dir, const std::vector<int>& dp) {
  const char* ge = std::getenv("IGB_FLOW_G");
  FlowPlanHost plan;
  // Early/late split (flow_plan.h): the row's values of dependencies at least crit_lag levels
  // back are loaded and reduced as soon as the crit value is ready, the newer ("late") ones are
  // added in a serial tail.  Measured per dependency level on cfg5 L=3 (us, fwd / bwd, level 3):
  // one batch with crit lag 2 (round 1) 1.55 / 1.84; lag 4 1.05 / 1.21; lag 6 0.88 / 1.42;
  // lag 8 0.85 / 2.20 -- so forward lag 8 (late <= 64), backward lag 4 (late <= 32).
  // IGB_FLOW_CRITLAG / IGB_FLOW_LATE override both directions (IGB_FLOW_LATE=0: one batch).
  const char* le = std::getenv("IGB_FLOW_CRITLAG");
  const char* lm = std::getenv("IGB_FLOW_LATE");
  int lag = le ? std::max(1, std::atoi(le)) : (dir ? 4 : 8);
  int late_max = lm ? std::max(0, std::atoi(lm)) : (dir ? 32 : 64);
  {
    // Rows served by a whole warp (G = 32: 3-D stencils, > 56 entries per row): crit lag 3, one late
    // chunk.  A per-row trace of cfg5's finest sweep (733 rows per dependency level for 2,368
    // resident warps, ~3 levels in flight: bound by the time a warp spends per row, not by the hop)
    // showed 2.7 of 4.9 us per row in the serial late tail of the lag-8 split
    // (profiles/r2_flow_trace_cfg5.log); with the next row's entries prefetched into L2 and the
    // first chunk in flight during the crit wait the short lag is also the best choice on the
    // narrow levels (cfg5 full, whole solve: lag 8 / 4 everywhere 104.9 ms, lag 3 on the finest level
    // 89.0, on levels 3-4 87.3, on every level 85.8).  IGB_FLOW_CRITLAG / IGB_FLOW_LATE override.
    // 3-D levels only (known once the level's interiors are registered): on cfg4 p = 8's 2-D
    // backward levels (145 entries per row) the old lag 4 / 32 stays better (264.5 vs 279.3 ms).
    const long long tri = dir ? V.tri_nnz_upper : V.tri_nnz_lower;
    const bool three_d = !V.interiors.empty() && V.interiors[0].dim == 3;
    if (!le && !lm && three_d && tri > 56LL * V.n) {
      lag = 3;
      late_max = 8;
    }
  }
  if (!build_flow_plan(V.n, V.h_ptr.data(), V.h_col.data(), V.h_val.data(), dp.data(), dir == 1,
                       ge ? std::atoi(ge) : 0, late_max > 0 ? lag : (le ? lag : 2), late_max, plan))
    return false;
  FlowDev& F = V.flow[dir];
  FlowArgs& a = F.args;
  a = FlowArgs{};
  a.n = V.n;
  a.nq = plan.nq;
  a.G = plan.G;
  a.row = ctx->upload(plan.row.data(), plan.row.size());
  a.eptr = ctx->upload(plan.eptr.data(), plan.eptr.size());
  a.ecol = plan.entries ? ctx->upload(plan.ecol.data(), plan.ecol.size()) : ctx->alloc<int>(1);
  a.eval = plan.entries ? ctx->upload(plan.eval.data(), plan.eval.size()) : ctx->alloc<double>(1);
  a.idiag = ctx->upload(plan.idiag.data(), plan.idiag.size());
  const char* ce = std::getenv("IGB_FLOW_CRIT");
  if (!ce || std::atoi(ce)) a.crit = ctx->upload(plan.crit.data(), plan.crit.size());
  if (late_max > 0) a.elate = ctx->upload(plan.elate.data(), plan.elate.size());
  const char* be = std::getenv("IGB_FLOW_BACKOFF");
  a.backoff = be ? std::atoi(be) : 0;
  const char* pfe = std::getenv("IGB_FLOW_PREFETCH");
  a.prefetch = pfe ? std::atoi(pfe) : 1;
  std::vector<unsigned long long> pend((size_t)2 * V.n, 0x7FF4DEADBEEF5678ULL);  // flow.cu FLOW_PENDING
  a.xg = reinterpret_cast<double*>(ctx->upload(pend.data(), pend.size()));
  int* ctr = ctx->alloc<int>(2);
  CU(cudaMemset(ctr, 0, 2 * sizeof(int)));
  a.par_ctr = ctr;
  a.done_ctr = reinterpret_cast<unsigned*>(ctr + 1);
  // enough warps for ~inflight dependency levels at once (idle warps only poll L2)
  const char* fe = std::getenv("IGB_FLOW_INFLIGHT");
  const double inflight = fe ? std::atof(fe) : 16.0;  // measured: 16 > 8 > 4 (cfg5 L=3 fwd 1.12 / 1.22 / 1.40 us per level)
  const double width = double(plan.nq) / std::max(1, plan.nlev);
  const double warps = inflight * width / (32 / plan.G);
  const int want = (int)std::ceil(warps / (FLOW_NT / 32));
  a.ctas = std::max(1, std::min(flow_max_ctas(), want));
  F.nlev = plan.nlev;
  F.entries = plan.entries;
  if (std::getenv("IGB_FLOW_TRACE")) {
    F.h_row = plan.row;
    F.h_qlev = plan.qlev;
  }
  F.ok = true;
  if (std::getenv("IGB_VERBOSE"))
    std::fprintf(stderr, "[igb] level %d dir %d: flow sweep n %d depth %d width %.0f entries %lld G %d ctas %d\n",
                 level, dir, V.n, plan.nlev, width, plan.entries, plan.G, a.ctas);
  return true;
}

int igb_set_gs(igb_ctx* ctx, int level) {
  return guarded(ctx, [&] {
    require_levels(ctx);
    Level& V = ctx->level(level);
    if (!V.n) throw StateError("set the level matrix before igb_set_gs");
    const bool verbose = std::getenv("IGB_VERBOSE") != nullptr;
    auto tnow = [] { return std::chrono::steady_clock::now(); };
    auto tick = tnow();
    auto lap = [&](const char* what) {
      if (!verbose) return;
      const auto t = tnow();
      std::fprintf(stderr, "[igb] set_gs level %d: %s %.2f s\n", level, what,
                   std::chrono::duration<double>(t - tick).count());
      tick = t;
    };
    std::vector<int> dp = diag_positions(V.n, V.h_ptr.data(), V.h_col.data(), nullptr, "A");
    {
      // strict triangles (parallel two-pass split of the CSR rows)
      std::vector<int> up(V.n + 1, 0), lp(V.n + 1, 0);
      for (int i = 0; i < V.n; ++i) {
        up[i + 1] = up[i] + (V.h_ptr[i + 1] - dp[i] - 1);
        lp[i + 1] = lp[i] + (dp[i] - V.h_ptr[i]);
      }
      std::vector<int> ui(up[V.n]), li(lp[V.n]);
      std::vector<double> uv(up[V.n]), lvv(lp[V.n]);
      parallel_for(V.n, [&](long long lo, long long hi) {
        for (long long i = lo; i < hi; ++i) {
          const int a = V.h_ptr[i], d = dp[i], e = V.h_ptr[i + 1];
          std::copy(V.h_col.begin() + d + 1, V.h_col.begin() + e, ui.begin() + up[i]);
          std::copy(V.h_val.begin() + d + 1, V.h_val.begin() + e, uv.begin() + up[i]);
          std::copy(V.h_col.begin() + a, V.h_col.begin() + d, li.begin() + lp[i]);
          std::copy(V.h_val.begin() + a, V.h_val.begin() + d, lvv.begin() + lp[i]);
        }
      });
      V.U = upload_csr(ctx, V.n, V.n, (long long)ui.size(), up.data(), ui.data(), uv.data());
      V.Lo = upload_csr(ctx, V.n, V.n, (long long)li.size(), lp.data(), li.data(), lvv.data());
      V.has_U = !(std::getenv("IGB_GS_RESIDUAL") && std::string(std::getenv("IGB_GS_RESIDUAL")) == "full");
    }
    lap("triangles");
    V.fwd = build_schedule(ctx, V.n, V.h_ptr.data(), V.h_col.data(), dp, false);
    V.bwd = build_schedule(ctx, V.n, V.h_ptr.data(), V.h_col.data(), dp, true);
    lap("schedules");
    const char* eng = std::getenv("IGB_GS_ENGINE");
    const std::string engine = eng ? eng : "auto";
    const bool want_stream = engine != "levels";
    bool panel_done[2] = {false, false};
    if (engine == "auto" || engine == "panel") {
      for (int dir = 0; dir < 2; ++dir) {
        const Sched& Sd = dir ? V.bwd : V.fwd;
        panel_done[dir] = build_panel_sweep(ctx, V, level, dir, dp, Sd.nlev, engine == "panel");
      }
    }
    lap("panel plans");
    // wave sweep (plane chains inside one CTA): IGB_GS_ENGINE=wave forces it on every level
    if (engine == "wave") {
      for (int dir = 0; dir < 2; ++dir)
        if (!panel_done[dir]) panel_done[dir] = build_wave_sweep(ctx, V, level, dir, dp);
      lap("wave plans");
    }
    // line sweep (bundles of grid lines per CTA): IGB_GS_ENGINE=line forces it on every level
    if (engine == "line") {
      for (int dir = 0; dir < 2; ++dir)
        if (!panel_done[dir]) panel_done[dir] = build_line_sweep(ctx, V, level, dir, dp);
      lap("line plans");
    }
    // whole-GPU dependency-driven sweep: wide dependency levels (3-D, high degree) where the
    // panel chain is not short; IGB_GS_ENGINE=flow forces it on every level
    for (int dir = 0; dir < 2; ++dir) {
      if (panel_done[dir]) continue;
      const Sched& Sd = dir ? V.bwd : V.fwd;
      const double width = double(V.n) / std::max(1, Sd.nlev);
      const long long tri = dir ? V.tri_nnz_upper : V.tri_nnz_lower;
      const bool want = engine == "flow" ||
                        (engine == "auto" && (width >= flow_min_width() || tri >= 48LL * V.n));
      if (want) panel_done[dir] = build_flow_sweep(ctx, V, level, dir, dp);
    }
    lap("flow plans");
    level_prepare();
    const char* clenv = std::getenv("IGB_GS_CLUSTER");
    const int cluster_max = clenv ? std::max(1, std::min(8, std::atoi(clenv))) : 8;
    for (int dir = 0; dir < 2 && want_stream; ++dir) {
      if (panel_done[dir]) continue;
      SweepDev& C = V.sweep[dir];
      LevelPlanHost plan;
      LevelArgs& a = C.args;
      bool ok = false;
      // steps per level with one CTA decides the cluster size (levels wider than one
      // CTA's rows go to a cluster), then the largest ring that fits is chosen
      int ncta = 1;
      if (cluster_max > 1 &&
          build_level_plan(V.n, V.h_ptr.data(), V.h_col.data(), V.h_val.data(), dp.data(), dir == 1, LEVEL_NT,
                           4096, LEVEL_KMAX, plan)) {
        const double per_level = double(plan.nsteps) / std::max(1, plan.nlevels);
        ncta = std::max(1, std::min(cluster_max, (int)std::ceil(per_level - 1e-9)));
      }
      if (const char* force = std::getenv("IGB_GS_FORCE_CLUSTER"))  // testing: cluster even narrow levels
        ncta = std::max(1, std::min(8, std::atoi(force)));
      for (int R : {16384, 8192, 4096, 2048}) {
        if (!build_level_plan(V.n, V.h_ptr.data(), V.h_col.data(), V.h_val.data(), dp.data(), dir == 1,
                              LEVEL_NT * ncta, R, LEVEL_KMAX, plan))
          continue;
        a.nsteps = plan.nsteps;
        a.TPR = plan.TPR;
        a.R = plan.R;
        a.has_old = plan.has_old ? 1 : 0;
        a.cluster = ncta;
        a.dbg = nullptr;
        a.ablate = 0;
        if (level_smem_bytes(a) <= 220u * 1024) {
          ok = true;
          break;
        }
      }
      if (!ok) continue;
      static_assert(sizeof(LevelMetaDev) == sizeof(LevelMeta), "meta layout");
      a.meta = reinterpret_cast<const LevelMetaDev*>(
          ctx->upload(reinterpret_cast<const int*>(plan.meta.data()), plan.meta.size() * 4));
      // padded: the sweep prefetches unconditionally past the end of a step / vector
      plan.stream.resize(plan.stream.size() + 64 * 1024 + 8 * 16 * 32 * 64 * 8, 0);
      a.stream = ctx->upload(plan.stream.data(), plan.stream.size());
      C.rows = ctx->upload(plan.rows.data(), plan.rows.size());
      if (!V.rp) {
        V.rp = ctx->alloc<double>(V.n + 8 * LEVEL_NT + 2);
        V.xp = ctx->alloc<double>(V.n + 8 * LEVEL_NT + 2);
      }
      if (std::getenv("IGB_VERBOSE"))
        std::fprintf(stderr, "[igb] level %d dir %d: n %d levels %d steps %d TPR %d R %d cluster %d old %d stream %.1f MB\n",
                     level, dir, V.n, plan.nlevels, plan.nsteps, plan.TPR, plan.R, a.cluster, a.has_old,
                     plan.stream.size() / 1e6);
      C.entries = plan.entries;
      C.steps = plan.nsteps;
      C.levels = plan.nlevels;
      C.stream_bytes = (double)plan.stream.size();
      C.ok = true;
    }
    lap("level plans");
    V.has_gs = true;
  });
}

int igb_scms_begin(igb_ctx* ctx, int level, double tau) {
  return guarded(ctx, [&] {
    require_levels(ctx);
    Level& V = ctx->level(level);
    if (!(tau > 0)) throw ArgError("scms needs positive damping");
    V.has_scms = true;
    V.tau = tau;
  });
}

int igb_scms_add_interior(igb_ctx* ctx, int level, int dim, const int* dims, const double* T0,
                          const double* T1, const double* T2, const double* denom,
                          const int* idx) {
  return guarded(ctx, [&] {
    require_levels(ctx);
    Level& V = ctx->level(level);
    if (!V.has_scms) throw StateError("igb_scms_begin first");
    if (dim != 2 && dim != 3) throw ArgError("interior dimension must be 2 or 3");
    InteriorStage it{};
    it.dim = dim;
    size_t total = 1;
    const double* Ts[3] = {T0, T1, T2};
    for (int a = 0; a < dim; ++a) {
      if (dims[a] < 1) throw ArgError("empty interior");
      it.n[a] = dims[a];
      total *= dims[a];
      if (!Ts[a]) throw ArgError("null transform");
    }
    if (dim == 2) it.n[2] = 1;
    auto shared = [&](const double* h, size_t count) -> const double* {
      unsigned long long hash = 1469598103934665603ULL;  // FNV-1a over the bytes
      const unsigned char* bytes = reinterpret_cast<const unsigned char*>(h);
      for (size_t i = 0; i < count * sizeof(double); ++i) hash = (hash ^ bytes[i]) * 1099511628211ULL;
      auto& bucket = ctx->shared_uploads[{count, hash}];
      for (auto& e : bucket)
        if (std::memcmp(e.host.data(), h, count * sizeof(double)) == 0) return e.dev;
      double* d = ctx->upload(h, count);
      bucket.push_back({std::vector<double>(h, h + count), d});
      return d;
    };
    for (int a = 0; a < dim; ++a) it.T[a] = shared(Ts[a], (size_t)dims[a] * dims[a]);
    it.D = shared(denom, total);
    for (size_t k = 0; k < total; ++k)
      if (idx[k] < 0 || idx[k] >= V.n) throw ArgError("interior index out of range");
    it.idx = ctx->upload(idx, total);
    V.interiors.push_back(it);
  });
}

int igb_scms_add_piece(igb_ctx* ctx, int level, int m, const int* idx, const double* inv) {
  return guarded(ctx, [&] {
    require_levels(ctx);
    Level& V = ctx->level(level);
    if (!V.has_scms) throw StateError("igb_scms_begin first");
    if (m < 1) throw ArgError("empty piece");
    for (int k = 0; k < m; ++k)
      if (idx[k] < 0 || idx[k] >= V.n) throw ArgError("piece index out of range");
    const int* didx = ctx->upload(idx, (size_t)m);
    const double* dinv = ctx->upload(inv, (size_t)m * m);
    const int rows = m >= 512 ? 64 : 8;  // large pieces: amortise the staged r[idx] over 64 rows
    for (int r0 = 0; r0 < m; r0 += rows) {
      PieceRowBlock b{dinv, didx, m, r0, std::min(rows, m - r0)};
      V.h_blocks.push_back(b);
    }
    V.piece_max_m = std::max(V.piece_max_m, m);
    V.piece_bytes += 8.0 * m * (double)m + 8.0 * m * 3 + 4.0 * m;
    V.piece_rows += m;
  });
}

int igb_set_coarse_lu(igb_ctx* ctx, int n0, long long l_nnz, const int* l_ptr, const int* l_idx,
                      const double* l_val, long long u_nnz, const int* u_ptr, const int* u_idx,
                      const double* u_val, const int* perm_r, const int* perm_c) {
  return guarded(ctx, [&] {
    require_levels(ctx);
    CU(cudaSetDevice(ctx->device));
    Coarse& C = ctx->coarse;
    if (C.set) throw StateError("coarse factor already set");
    check_csr(n0, n0, l_nnz, l_ptr, l_idx);
    check_csr(n0, n0, u_nnz, u_ptr, u_idx);
    std::vector<int> inv(n0, -1);
    for (int i = 0; i < n0; ++i) {
      if (perm_r[i] < 0 || perm_r[i] >= n0 || perm_c[i] < 0 || perm_c[i] >= n0)
        throw ArgError("permutation out of range");
      inv[perm_r[i]] = i;
    }
    for (int i = 0; i < n0; ++i)
      if (inv[i] < 0) throw ArgError("perm_r is not a permutation");
    std::vector<int> ld = diag_positions(n0, l_ptr, l_idx, l_val, "L");
    std::vector<int> ud = diag_positions(n0, u_ptr, u_idx, u_val, "U");
    C.n = n0;
    C.L = upload_csr(ctx, n0, n0, l_nnz, l_ptr, l_idx, l_val);
    C.U = upload_csr(ctx, n0, n0, u_nnz, u_ptr, u_idx, u_val);
    C.Ldpos = ctx->upload(ld.data(), ld.size());
    C.Udpos = ctx->upload(ud.data(), ud.size());
    C.Ls = build_schedule(ctx, n0, l_ptr, l_idx, ld, false);
    C.Us = build_schedule(ctx, n0, u_ptr, u_idx, ud, true);
    C.inv_perm_r = ctx->upload(inv.data(), inv.size());
    C.perm_c = ctx->upload(perm_c, (size_t)n0);
    // column-oriented copies: strictly lower L and strictly upper U in CSC, diag(U)
    auto to_csc = [&](const int* p, const int* ix, const double* v, bool lower,
                      std::vector<int>& cp, std::vector<int>& ri, std::vector<double>& cv) {
      cp.assign(n0 + 1, 0);
      for (int i = 0; i < n0; ++i)
        for (int k = p[i]; k < p[i + 1]; ++k)
          if (lower ? ix[k] < i : ix[k] > i) cp[ix[k] + 1]++;
      for (int j = 0; j < n0; ++j) cp[j + 1] += cp[j];
      ri.resize(cp[n0]);
      cv.resize(cp[n0]);
      std::vector<int> pos(cp.begin(), cp.end() - 1);
      for (int i = 0; i < n0; ++i)
        for (int k = p[i]; k < p[i + 1]; ++k)
          if (lower ? ix[k] < i : ix[k] > i) {
            const int q = pos[ix[k]]++;
            ri[q] = i;
            cv[q] = v[k];
          }
    };
    std::vector<int> lcp, lri, ucp, uri;
    std::vector<double> lcv, ucv, udg(n0);
    to_csc(l_ptr, l_idx, l_val, true, lcp, lri, lcv);
    to_csc(u_ptr, u_idx, u_val, false, ucp, uri, ucv);
    for (int i = 0; i < n0; ++i) {
      if (l_val[ld[i]] != 1.0) throw ArgError("L must have a unit diagonal");
      udg[i] = u_val[ud[i]];
    }
    C.csc.n = n0;
    C.csc.lcp = ctx->upload(lcp.data(), lcp.size());
    C.csc.lri = ctx->upload(lri.data(), lri.size());
    C.csc.lv = ctx->upload(lcv.data(), lcv.size());
    C.csc.ucp = ctx->upload(ucp.data(), ucp.size());
    C.csc.uri = ctx->upload(uri.data(), uri.size());
    C.csc.uv = ctx->upload(ucv.data(), ucv.size());
    C.csc.udiag = ctx->upload(udg.data(), udg.size());
    C.csc.inv_perm_r = C.inv_perm_r;
    C.csc.perm_c = C.perm_c;
    C.csc.lnnz = lcp[n0];
    C.csc.unnz = ucp[n0];
    C.y = ctx->alloc<double>(n0);
    C.w = ctx->alloc<double>(n0);
    const char* ce = std::getenv("IGB_COARSE");
    const long long dense_max = 4096;
    if (!(ce && std::string(ce) == "csc") && n0 <= dense_max) {
      // column j of M: the substitution of the device csc path applied to e_j
      std::vector<double> M((size_t)n0 * n0), y(n0);
      for (int j = 0; j < n0; ++j) {
        std::fill(y.begin(), y.end(), 0.0);
        y[perm_r[j]] = 1.0;  // y[k] = e_j[inv_perm_r[k]]
        for (int c = 0; c < n0; ++c) {
          const double yc = y[c];
          if (yc != 0.0)
            for (int q = lcp[c]; q < lcp[c + 1]; ++q) y[lri[q]] -= lcv[q] * yc;
        }
        for (int c = n0 - 1; c >= 0; --c) {
          const double wc = y[c] / udg[c];
          y[c] = wc;
          if (wc != 0.0)
            for (int q = ucp[c]; q < ucp[c + 1]; ++q) y[uri[q]] -= ucv[q] * wc;
        }
        for (int i = 0; i < n0; ++i) M[(size_t)i * n0 + j] = y[perm_c[i]];
      }
      std::vector<int> ident(n0);
      for (int i = 0; i < n0; ++i) ident[i] = i;
      const double* dM = ctx->upload(M.data(), M.size());
      const int* didx = ctx->upload(ident.data(), ident.size());
      std::vector<PieceRowBlock> blocks;
      // 8 rows per block: one coarse operator alone must still spread over the SMs (measured: 64 rows
      // per block left cfg5's 1331^2 operator on 21 blocks, 0.38 vs 0.12 ms per solve)
      for (int r0 = 0; r0 < n0; r0 += 8) blocks.push_back(PieceRowBlock{dM, didx, n0, r0, std::min(8, n0 - r0)});
      C.d_dense = ctx->upload(blocks.data(), blocks.size());
      C.ndense = (int)blocks.size();
    }
    C.set = true;
  });
}

int igb_set_cycle(igb_ctx* ctx, int smoother, int mu, const int* steps_per_level) {
  return guarded(ctx, [&] {
    require_levels(ctx);
    if (smoother < 0 || smoother > 2) throw ArgError("unknown smoother kind");
    if (mu != 1 && mu != 2) throw ArgError("cycle index mu must be 1 (V) or 2 (W)");
    ctx->smoother = smoother;
    ctx->mu = mu;
    if (steps_per_level)
      for (int l = 0; l <= ctx->L; ++l) {
        if (steps_per_level[l] < 0) throw ArgError("negative smoothing steps");
        ctx->steps[l] = steps_per_level[l];
      }
    ctx->drop_graph();
  });
}

int igb_finalize(igb_ctx* ctx) {
  return guarded(ctx, [&] {
    require_levels(ctx);
    CU(cudaSetDevice(ctx->device));
    if (ctx->finalized) throw StateError("already finalized");
    for (int l = 0; l <= ctx->L; ++l)
      if (!ctx->lev[l].n) throw StateError("level matrix missing");
    if (!ctx->coarse.set) throw StateError("coarse factor missing");
    if (ctx->coarse.n != ctx->lev[0].n) throw ArgError("coarse factor size != n_0");
    for (int l = 1; l <= ctx->L; ++l) {
      Level& V = ctx->lev[l];
      if (!V.has_P) throw StateError("prolongation missing");
      if (V.P.n != V.n || V.P.m != ctx->lev[l - 1].n) throw ArgError("prolongation shape mismatch");
      const bool need_gs = ctx->smoother != IGB_SMOOTHER_SCMS;
      const bool need_scms = ctx->smoother != IGB_SMOOTHER_GS;
      if (need_gs && !V.has_gs) throw StateError("Gauss-Seidel data missing on a level");
      if (need_scms && !V.has_scms) throw StateError("SCMS data missing on a level");
      if (V.has_scms) {
        build_fd_plan(ctx, V);
        if (!V.h_blocks.empty()) V.d_blocks = ctx->upload(V.h_blocks.data(), V.h_blocks.size());
        if (!V.h_blocks.empty() && !V.fd.batches.empty()) {
          // piece rows in blocks of 5 (the FD kernels' warps), appended to the last FD batch
          std::vector<PieceRowBlock> five;
          for (const auto& b : V.h_blocks)
            for (int r0 = b.row0; r0 < b.row0 + b.nrows; r0 += 5)
              five.push_back(PieceRowBlock{b.inv, b.idx, b.m, r0, std::min(5, b.row0 + b.nrows - r0)});
          FdBatch& bt = V.fd.batches.back();
          bt.pieces = ctx->upload(five.data(), five.size());
          bt.npieces = (int)five.size();
          V.fd.batch_bytes.back() += V.piece_bytes;
          V.pieces_fused = true;
        }
        // the pieces must partition 0..n-1 together with the interiors
      }
      V.h_col.clear();
      V.h_col.shrink_to_fit();
      V.h_val.clear();
      V.h_val.shrink_to_fit();
    }
    const int nL = ctx->lev[ctx->L].n;
    ctx->x = ctx->alloc<double>(nL);
    ctx->d = ctx->alloc<double>(nL);
    ctx->q = ctx->alloc<double>(nL);
    ctx->b = ctx->alloc<double>(nL);
    ctx->partials = ctx->alloc<double>(REDUCTION_MAX_BLOCKS);
    ctx->counter = ctx->alloc<unsigned>(1);
    CU(cudaMemset(ctx->counter, 0, sizeof(unsigned)));
    ctx->sc = ctx->alloc<CgScalars>(1);
    ctx->finalized = true;
  });
}

int igb_cycle(igb_ctx* ctx, int level, const double* f, double* u) {
  return guarded(ctx, [&] {
    require_final(ctx);
    CU(cudaSetDevice(ctx->device));
    if (level < 1 || level > ctx->L) throw ArgError("cycles act on levels >= 1");
    Level& V = ctx->lev[level];
    CU(cudaMemcpyAsync(V.f, f, sizeof(double) * V.n, cudaMemcpyHostToDevice, ctx->stream));
    if (level == ctx->L) ctx->run_finest_cycle();
    else ctx->cycle(level, V.f, V.u);
    CU(cudaMemcpyAsync(u, V.u, sizeof(double) * V.n, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    ctx->harvest_graph();
    if (ctx->prof) ctx->harvest(ctx->direct_recs, true);
  });
}

int igb_op(igb_ctx* ctx, int op, int level, const double* in, double* out) {
  return guarded(ctx, [&] {
    require_final(ctx);
    CU(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    if (op == IGB_OP_COARSE) {
      Coarse& C = ctx->coarse;
      Level& V0 = ctx->lev[0];
      CU(cudaMemcpyAsync(V0.f, in, sizeof(double) * C.n, cudaMemcpyHostToDevice, s));
      ctx->coarse_solve(V0.f, V0.u);
      CU(cudaMemcpyAsync(out, V0.u, sizeof(double) * C.n, cudaMemcpyDeviceToHost, s));
    } else {
      Level& V = ctx->level(level);
      const int n = V.n;
      switch (op) {
        case IGB_OP_SPMV:
        case IGB_OP_RESIDUAL: {
          CU(cudaMemcpyAsync(V.f, in, sizeof(double) * n, cudaMemcpyHostToDevice, s));
          if (op == IGB_OP_RESIDUAL)
            CU(cudaMemcpyAsync(V.c, out, sizeof(double) * n, cudaMemcpyHostToDevice, s));
          ctx->apply_A(level, V.f, op == IGB_OP_RESIDUAL ? V.c : nullptr, V.r, op == IGB_OP_RESIDUAL ? -1 : 0);
          CU(cudaMemcpyAsync(out, V.r, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
          break;
        }
        case IGB_OP_GS_FWD:
        case IGB_OP_GS_BWD: {
          if (!V.has_gs) throw StateError("no Gauss-Seidel data on this level");
          CU(cudaMemcpyAsync(V.f, in, sizeof(double) * n, cudaMemcpyHostToDevice, s));
          ctx->gs(level, op == IGB_OP_GS_BWD, V.f, V.u, true);
          CU(cudaMemcpyAsync(out, V.u, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
          break;
        }
        case IGB_OP_SCMS: {
          if (!V.has_scms) throw StateError("no SCMS data on this level");
          CU(cudaMemcpyAsync(V.f, in, sizeof(double) * n, cudaMemcpyHostToDevice, s));
          ctx->scms(level, V.f, V.u, true);
          CU(cudaMemcpyAsync(out, V.u, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
          break;
        }
        case IGB_OP_RESTRICT: {
          if (level < 1) throw ArgError("restriction needs level >= 1");
          Level& C = ctx->lev[level - 1];
          CU(cudaMemcpyAsync(V.f, in, sizeof(double) * n, cudaMemcpyHostToDevice, s));
          ctx->restrict_to(level, V.f, C.r);
          CU(cudaMemcpyAsync(out, C.r, sizeof(double) * C.n, cudaMemcpyDeviceToHost, s));
          break;
        }
        case IGB_OP_PROLONG: {
          if (level < 1) throw ArgError("prolongation needs level >= 1");
          Level& C = ctx->lev[level - 1];
          CU(cudaMemcpyAsync(C.r, in, sizeof(double) * C.n, cudaMemcpyHostToDevice, s));
          ctx->prolong(level, C.r, nullptr, V.r, 0);
          CU(cudaMemcpyAsync(out, V.r, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
          break;
        }
        case IGB_OP_CYCLE: {
          if (level < 1) throw ArgError("cycles act on levels >= 1");
          CU(cudaMemcpyAsync(V.f, in, sizeof(double) * n, cudaMemcpyHostToDevice, s));
          if (level == ctx->L) ctx->run_finest_cycle();
          else ctx->cycle(level, V.f, V.u);
          CU(cudaMemcpyAsync(out, V.u, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
          break;
        }
        default:
          throw ArgError("unknown operator");
      }
    }
    CU(cudaStreamSynchronize(s));
    ctx->harvest_graph();
    if (ctx->prof) ctx->harvest(ctx->direct_recs, true);
  });
}

// Capture the whole PCG solve (linsolve.py:64-101) into one graph: the prologue, then a
// WHILE node whose body is one iteration -- q = A d and alpha, the x / r update and the
// residual test -- and an IF node around the preconditioner and direction update, both
// conditions set on the device (cg_cond_kernel).  No host round trip per iteration.
static void build_pcg_graph(igb_ctx* ctx, const double* d_b, double* d_x, int max_iters) {
  if (ctx->pcg_exec) cudaGraphExecDestroy(ctx->pcg_exec);
  ctx->pcg_exec = nullptr;
  for (auto& a : ctx->aux)
    if (!a) CU(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
  const int L = ctx->L;
  Level& F = ctx->lev[L];
  const int n = F.n;
  double* r = F.f;
  double* z = F.u;
  const DevCsr& A = F.A;
  cudaStream_t s0 = ctx->stream;
  const long long saved_graph_kernels = ctx->graph_kernels;
  cudaGraph_t g = nullptr;
  CU(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle loop, more;
  CU(cudaGraphConditionalHandleCreate(&loop, g, 0, cudaGraphCondAssignDefault));
  auto add_cond = [&](cudaStream_t st, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type) {
    cudaStreamCaptureStatus status;
    cudaGraph_t cg;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    CU(cudaStreamGetCaptureInfo(st, &status, nullptr, &cg, &deps, &ndeps));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = type;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    CU(cudaGraphAddNode(&node, cg, deps, ndeps, &p));
    CU(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
    return p.conditional.phGraph_out[0];
  };
  ctx->capturing = true;
  try {
    CU(cudaStreamBeginCaptureToGraph(s0, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    long long c0 = ctx->graph_kernels;
    cudaStream_t& s = ctx->stream;
    ctx->launch(K_CG, 16.0 * n, [&] { launch_dot(s, n, d_b, d_b, ctx->partials, ctx->counter, ctx->sc, FIN_NORMB, nullptr); });
    ctx->launch(K_CG, 8.0 * n, [&] { launch_fill(s, n, d_x, 0.0); });
    ctx->launch(K_CG, 16.0 * n, [&] { launch_copy(s, n, r, d_b); });
    ctx->cycle(L, r, z);
    ctx->launch(K_CG, 16.0 * n, [&] { launch_copy(s, n, ctx->d, z); });
    ctx->launch(K_CG, 16.0 * n, [&] { launch_dot(s, n, r, z, ctx->partials, ctx->counter, ctx->sc, FIN_RZ0, nullptr); });
    ctx->launch(K_CG, 0.0, [&] { launch_cg_cond(s, loop, loop, ctx->sc, max_iters, 1); });
    ctx->pcg_n_pre = ctx->graph_kernels - c0;
    cudaGraph_t body = add_cond(s0, loop, cudaGraphCondTypeWhile);
    CU(cudaGraphConditionalHandleCreate(&more, body, 0, cudaGraphCondAssignDefault));
    ctx->stream = ctx->aux[0];
    CU(cudaStreamBeginCaptureToGraph(ctx->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    c0 = ctx->graph_kernels;
    ctx->cg_matvec(s);
    // x / r update, residual norm and history, and (last block) the loop conditions: one launch
    ctx->launch(K_CG, 56.0 * n, [&] {
      launch_cg_update_cond(s, n, d_x, r, ctx->d, ctx->q, ctx->partials, ctx->counter, ctx->sc, ctx->hist_dev, loop, more,
                            max_iters);
    });
    ctx->pcg_n_head = ctx->graph_kernels - c0;
    cudaGraph_t ifbody = add_cond(ctx->stream, more, cudaGraphCondTypeIf);
    ctx->stream = ctx->aux[1];
    CU(cudaStreamBeginCaptureToGraph(ctx->stream, ifbody, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    c0 = ctx->graph_kernels;
    ctx->cycle(L, r, z);
    // beta = (r.z) / rz_old and d = z + beta d: one persistent launch
    ctx->launch(K_CG, 32.0 * n, [&] {
      launch_cg_beta_direction(s, n, ctx->d, z, r, ctx->partials, ctx->counter, ctx->sc);
    });
    ctx->pcg_n_if = ctx->graph_kernels - c0;
    CU(cudaStreamEndCapture(ctx->aux[1], &ifbody));
    CU(cudaStreamEndCapture(ctx->aux[0], &body));
    ctx->stream = s0;
    CU(cudaStreamEndCapture(s0, &g));
    CU(cudaGraphInstantiate(&ctx->pcg_exec, g, 0));
  } catch (...) {
    ctx->stream = s0;
    ctx->capturing = false;
    ctx->graph_kernels = saved_graph_kernels;
    for (cudaStream_t st : {ctx->aux[1], ctx->aux[0], s0}) {
      cudaGraph_t junk = nullptr;
      cudaStreamCaptureStatus status;
      if (cudaStreamIsCapturing(st, &status) == cudaSuccess && status != cudaStreamCaptureStatusNone)
        cudaStreamEndCapture(st, &junk);
      if (junk) cudaGraphDestroy(junk);
    }
    cudaGraphDestroy(g);
    cudaGetLastError();
    throw;
  }
  ctx->capturing = false;
  ctx->graph_kernels = saved_graph_kernels;
  cudaGraphDestroy(g);
  ctx->pcg_b = d_b;
  ctx->pcg_x = d_x;
  ctx->pcg_max = max_iters;
}

// x_host (nullable): the solution is also copied there before the one host synchronisation
// returns true when x_host was filled
static bool pcg_core(igb_ctx* ctx, const double* d_b, double tol, int max_iters, double* d_x,
                     int* its, double* hist, int hist_cap, double* x_host = nullptr) {
  if (max_iters < 0) throw ArgError("max_iters must be >= 0");
  cudaStream_t s = ctx->stream;
  const int L = ctx->L;
  Level& F = ctx->lev[L];
  const int n = F.n;
  if (ctx->hist_cap < max_iters) {
    ctx->hist_dev = ctx->alloc<double>(std::max(1, max_iters));
    ctx->hist_cap = max_iters;
    ctx->pcg_max = -1;  // the graph holds the old history buffer
    if (ctx->hist_host) cudaFreeHost(ctx->hist_host);
    CU(cudaHostAlloc(reinterpret_cast<void**>(&ctx->hist_host), sizeof(double) * std::max(1, max_iters),
                     cudaHostAllocDefault));
  }
  CgScalars init{};
  init.tol = tol;
  *ctx->sc_host = init;
  // one graph launch for the whole solve (profiling keeps the host loop: it times every launch)
  const char* pg = std::getenv("IGB_PCG_GRAPH");
  if (!ctx->prof && !ctx->pcg_graph_failed && !(pg && std::string(pg) == "0")) {
    if (!ctx->pcg_exec || ctx->pcg_b != d_b || ctx->pcg_x != d_x || ctx->pcg_max != max_iters) {
      try {
        build_pcg_graph(ctx, d_b, d_x, max_iters);
      } catch (const std::exception& e) {
        ctx->pcg_graph_failed = true;  // e.g. a driver without conditional graph nodes
        if (std::getenv("IGB_VERBOSE")) std::fprintf(stderr, "[igb] PCG graph unavailable: %s\n", e.what());
      }
    }
    if (ctx->pcg_exec) {
      CU(cudaMemcpyAsync(ctx->sc, ctx->sc_host, sizeof(CgScalars), cudaMemcpyHostToDevice, s));
      CU(cudaEventRecord(ctx->t0, s));
      CU(cudaGraphLaunch(ctx->pcg_exec, s));
      CU(cudaEventRecord(ctx->t1, s));
      // results back in one batch (scalars, the whole history buffer, x) and one synchronisation
      CU(cudaMemcpyAsync(ctx->sc_host, ctx->sc, sizeof(CgScalars), cudaMemcpyDeviceToHost, s));
      if (hist && max_iters > 0)
        CU(cudaMemcpyAsync(ctx->hist_host, ctx->hist_dev, sizeof(double) * std::min(max_iters, hist_cap),
                           cudaMemcpyDeviceToHost, s));
      if (x_host) CU(cudaMemcpyAsync(x_host, d_x, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
      CU(cudaStreamSynchronize(s));
      float ms = 0;
      CU(cudaEventElapsedTime(&ms, ctx->t0, ctx->t1));
      ctx->last_pcg_ms = ms;
      ctx->last_cycle_ms = 0;
      const int nit = ctx->sc_host->normb == 0.0 ? 0 : ctx->sc_host->it;
      *its = nit;
      const int nh = std::min(nit, hist_cap);
      if (hist && nh > 0) std::memcpy(hist, ctx->hist_host, sizeof(double) * nh);
      ctx->launches_direct += ctx->pcg_n_pre + nit * ctx->pcg_n_head + std::max(nit - 1, 0) * ctx->pcg_n_if;
      return x_host != nullptr;
    }
  }
  CU(cudaMemcpyAsync(ctx->sc, ctx->sc_host, sizeof(CgScalars), cudaMemcpyHostToDevice, s));
  CU(cudaEventRecord(ctx->t0, s));
  ctx->launch(K_CG, 16.0 * n, [&] {
    launch_dot(s, n, d_b, d_b, ctx->partials, ctx->counter, ctx->sc, FIN_NORMB, nullptr);
  });
  ctx->launch(K_CG, 8.0 * n, [&] { launch_fill(s, n, d_x, 0.0); });
  CU(cudaMemcpyAsync(ctx->sc_host, ctx->sc, sizeof(CgScalars), cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  *its = 0;
  int ncycles = 0;
  if (ctx->sc_host->normb == 0.0) {
    CU(cudaEventRecord(ctx->t1, s));
    CU(cudaEventSynchronize(ctx->t1));
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, ctx->t0, ctx->t1));
    ctx->last_pcg_ms = ms;
    ctx->last_cycle_ms = 0;
    return false;
  }
  double* r = F.f;   // CG residual doubles as the cycle input
  double* z = F.u;   // cycle output
  ctx->launch(K_CG, 16.0 * n, [&] { launch_copy(s, n, r, d_b); });
  ctx->run_finest_cycle();
  ++ncycles;
  ctx->launch(K_CG, 16.0 * n, [&] { launch_copy(s, n, ctx->d, z); });
  ctx->launch(K_CG, 16.0 * n, [&] {
    launch_dot(s, n, r, z, ctx->partials, ctx->counter, ctx->sc, FIN_RZ0, nullptr);
  });
  const DevCsr& A = F.A;
  int it = 0;
  for (it = 1; it <= max_iters; ++it) {
    ctx->cg_matvec(s);
    ctx->launch(K_CG, 56.0 * n, [&] {
      launch_cg_update(s, n, d_x, r, ctx->d, ctx->q, ctx->partials, ctx->counter, ctx->sc,
                       ctx->hist_dev);
    });
    CU(cudaMemcpyAsync(ctx->sc_host, ctx->sc, sizeof(CgScalars), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    ctx->harvest_graph();
    if (ctx->prof) ctx->harvest(ctx->direct_recs, true);
    if (ctx->sc_host->done) break;
    if (it == max_iters) break;
    ctx->run_finest_cycle();
    ++ncycles;
    ctx->launch(K_CG, 32.0 * n, [&] {
      launch_cg_beta_direction(s, n, ctx->d, z, r, ctx->partials, ctx->counter, ctx->sc);
    });
  }
  CU(cudaEventRecord(ctx->t1, s));
  CU(cudaEventSynchronize(ctx->t1));
  float ms = 0;
  CU(cudaEventElapsedTime(&ms, ctx->t0, ctx->t1));
  ctx->last_pcg_ms = ms;
  const int nit = ctx->sc_host->it;
  *its = ctx->sc_host->done ? nit : max_iters;
  const int nh = std::min(nit, hist_cap);
  if (hist && nh > 0) CU(cudaMemcpy(hist, ctx->hist_dev, sizeof(double) * nh, cudaMemcpyDeviceToHost));
  ctx->last_cycle_ms = 0;
  (void)ncycles;
  return false;
}

int igb_pcg(igb_ctx* ctx, const double* b, double tol, int max_iters, double* x, int* its,
            double* hist, int hist_cap) {
  return guarded(ctx, [&] {
    require_final(ctx);
    CU(cudaSetDevice(ctx->device));
    Level& F = ctx->lev[ctx->L];
    const int n = F.n;
    // host -> device copy of b and device -> host copy of x (inside pcg_core's one synchronisation;
    // copies run at full speed when the caller's buffers are pinned, igb_host_alloc)
    CU(cudaMemcpyAsync(ctx->b, b, sizeof(double) * n, cudaMemcpyHostToDevice, ctx->stream));
    if (!pcg_core(ctx, ctx->b, tol, max_iters, ctx->x, its, hist, hist_cap, x)) {  // host-loop path
      CU(cudaMemcpyAsync(x, ctx->x, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
      CU(cudaStreamSynchronize(ctx->stream));
    }
  });
}

int igb_pcg_device(igb_ctx* ctx, const double* d_b, double tol, int max_iters, double* d_x,
                   int* its, double* hist, int hist_cap) {
  return guarded(ctx, [&] {
    require_final(ctx);
    CU(cudaSetDevice(ctx->device));
    pcg_core(ctx, d_b, tol, max_iters, d_x, its, hist, hist_cap);
  });
}

// Smoother duck type pre_smooth / post_smooth(A, u, f, steps) (reference smoothers.py:192-200,
// 327-332, 343-353) on the device: `steps` steps of smoother `kind` on level l from the iterate u.
int igb_smooth(igb_ctx* ctx, int level, int kind, int post, int steps, const double* f, double* u) {
  return guarded(ctx, [&] {
    require_final(ctx);
    CU(cudaSetDevice(ctx->device));
    if (level < 1 || level > ctx->L) throw ArgError("smoothing acts on levels 1..L");
    if (steps < 0) throw ArgError("negative smoothing steps");
    if (kind < IGB_SMOOTHER_GS || kind > IGB_SMOOTHER_HYBRID) throw ArgError("unknown smoother kind");
    Level& V = ctx->lev[level];
    if ((kind != IGB_SMOOTHER_SCMS && !V.has_gs) || (kind != IGB_SMOOTHER_GS && !V.has_scms))
      throw StateError("the level has no such smoother");
    const int n = V.n;
    cudaStream_t s = ctx->stream;
    const int saved_kind = ctx->smoother, saved_steps = ctx->steps[level];
    ctx->smoother = kind;
    ctx->steps[level] = steps;
    try {
      CU(cudaMemcpyAsync(V.f, f, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      CU(cudaMemcpyAsync(V.u, u, sizeof(double) * n, cudaMemcpyHostToDevice, s));
      bool uz = false;
      if (post) ctx->post_smooth(level, V.f, V.u, uz);
      else ctx->pre_smooth(level, V.f, V.u, uz);
      CU(cudaMemcpyAsync(u, V.u, sizeof(double) * n, cudaMemcpyDeviceToHost, s));
      CU(cudaStreamSynchronize(s));
    } catch (...) {
      ctx->smoother = saved_kind;
      ctx->steps[level] = saved_steps;
      throw;
    }
    ctx->smoother = saved_kind;
    ctx->steps[level] = saved_steps;
  });
}

// General PCG (linsolve.cg with any operator / preconditioner, live per-iteration callback):
// the same kernels and reductions as pcg_core, driven by a host loop that reads the scalars after
// every iteration (reference linsolve.py:64-101).
int igb_cg(igb_ctx* ctx, int n, long long nnz, const int* indptr, const int* indices, const double* data,
           int prec_mode, igb_prec_fn prec, void* prec_user, igb_iter_fn iter_cb, void* iter_user,
           const double* b, double tol, int max_iters, double* x, int* its, double* hist, int hist_cap) {
  return guarded(ctx, [&] {
    CU(cudaSetDevice(ctx->device));
    if (max_iters < 0) throw ArgError("max_iters must be >= 0");
    if (n < 1 || !b || !x || !its) throw ArgError("bad cg arguments");
    if (prec_mode < IGB_PREC_NONE || prec_mode > IGB_PREC_HOST) throw ArgError("unknown preconditioner mode");
    if (prec_mode == IGB_PREC_HOST && !prec) throw ArgError("host preconditioner callback missing");
    const bool finest_op = indptr == nullptr;
    if (finest_op || prec_mode == IGB_PREC_CYCLE) {
      require_final(ctx);
      if (n != ctx->lev[ctx->L].n) throw ArgError("cg size differs from the finest level");
    }
    if (!finest_op) {
      if (nnz >= (1LL << 31)) throw ArgError("nnz exceeds int32 indexing");
      check_csr(n, n, nnz, indptr, indices);
    }
    cudaStream_t s = ctx->stream;
    // scratch, released on return
    std::vector<void*> tmp;
    auto scratch = [&](size_t bytes) {
      void* p = nullptr;
      CU(cudaMalloc(&p, std::max<size_t>(bytes, 8)));
      tmp.push_back(p);
      return p;
    };
    struct Free {
      std::vector<void*>& v;
      ~Free() {
        for (void* p : v) cudaFree(p);
      }
    } release{tmp};
    DevCsr M{};
    if (!finest_op) {
      M.n = M.m = n;
      M.nnz = nnz;
      M.ptr = static_cast<int*>(scratch(sizeof(int) * (n + 1)));
      M.col = static_cast<int*>(scratch(sizeof(int) * nnz));
      M.val = static_cast<double*>(scratch(sizeof(double) * nnz));
      ctx->copy_h2d(M.ptr, indptr, sizeof(int) * (n + 1));
      ctx->copy_h2d(M.col, indices, sizeof(int) * nnz);
      ctx->copy_h2d(M.val, data, sizeof(double) * nnz);
      M.group = pick_group(nnz, n);
    }
    double* dx = static_cast<double*>(scratch(8 * (size_t)n));
    double* dr = static_cast<double*>(scratch(8 * (size_t)n));
    double* dz = static_cast<double*>(scratch(8 * (size_t)n));
    double* dd = static_cast<double*>(scratch(8 * (size_t)n));
    double* dq = static_cast<double*>(scratch(8 * (size_t)n));
    double* dh = static_cast<double*>(scratch(8 * (size_t)std::max(1, max_iters)));
    double* partials = static_cast<double*>(scratch(sizeof(double) * REDUCTION_MAX_BLOCKS));
    unsigned* counter = static_cast<unsigned*>(scratch(sizeof(unsigned)));
    CgScalars* sc = static_cast<CgScalars*>(scratch(sizeof(CgScalars)));
    CU(cudaMemsetAsync(counter, 0, sizeof(unsigned), s));
    CgScalars h{};
    h.tol = tol;
    CU(cudaMemcpyAsync(sc, &h, sizeof(h), cudaMemcpyHostToDevice, s));
    std::vector<double> hr, hz;
    auto apply_prec = [&] {  // z = M r
      if (prec_mode == IGB_PREC_NONE) {
        ctx->launch(K_CG, 16.0 * n, [&] { launch_copy(s, n, dz, dr); });
      } else if (prec_mode == IGB_PREC_CYCLE) {
        Level& F = ctx->lev[ctx->L];
        ctx->launch(K_CG, 16.0 * n, [&] { launch_copy(s, n, F.f, dr); });
        ctx->run_finest_cycle();
        ctx->launch(K_CG, 16.0 * n, [&] { launch_copy(s, n, dz, F.u); });
      } else {
        hr.resize(n);
        hz.assign(n, 0.0);
        CU(cudaMemcpyAsync(hr.data(), dr, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        prec(hr.data(), hz.data(), n, prec_user);
        CU(cudaMemcpyAsync(dz, hz.data(), 8 * (size_t)n, cudaMemcpyHostToDevice, s));
      }
    };
    auto matvec = [&] {  // q = A d
      if (finest_op) ctx->apply_A(ctx->L, dd, nullptr, dq, 0);
      else ctx->spmv(M, dd, nullptr, dq, 0, K_SPMV);
    };
    CU(cudaMemcpyAsync(dr, b, 8 * (size_t)n, cudaMemcpyHostToDevice, s));
    ctx->launch(K_CG, 16.0 * n, [&] { launch_dot(s, n, dr, dr, partials, counter, sc, FIN_NORMB, nullptr); });
    ctx->launch(K_CG, 8.0 * n, [&] { launch_fill(s, n, dx, 0.0); });
    CU(cudaMemcpyAsync(&h, sc, sizeof(h), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    int nit = 0;
    if (h.normb != 0.0) {
      apply_prec();
      ctx->launch(K_CG, 16.0 * n, [&] { launch_copy(s, n, dd, dz); });
      ctx->launch(K_CG, 16.0 * n, [&] { launch_dot(s, n, dr, dz, partials, counter, sc, FIN_RZ0, nullptr); });
      for (int it = 1; it <= max_iters; ++it) {
        if (finest_op && !ctx->lev[ctx->L].has_mf) {
          // the same fused product + d.q as the device PCG (cg_matvec): identical bits on both paths
          const DevCsr& A = ctx->lev[ctx->L].A;
          ctx->launch(K_SPMV, 12.0 * A.nnz + 4.0 * (n + 1) + 24.0 * n, [&] {
            launch_spmv_dot(s, n, A.ptr, A.col, A.val, dd, dq, A.group, partials, counter, sc, nullptr);
          });
        } else {
          matvec();
          ctx->launch(K_CG, 16.0 * n, [&] { launch_dot(s, n, dd, dq, partials, counter, sc, FIN_ALPHA, nullptr); });
        }
        ctx->launch(K_CG, 56.0 * n, [&] { launch_cg_update(s, n, dx, dr, dd, dq, partials, counter, sc, dh); });
        CU(cudaMemcpyAsync(&h, sc, sizeof(h), cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        nit = it;
        if (iter_cb) iter_cb(it, h.rel, iter_user);
        if (h.done || it == max_iters) break;
        apply_prec();
        ctx->launch(K_CG, 32.0 * n, [&] { launch_cg_beta_direction(s, n, dd, dz, dr, partials, counter, sc); });
      }
    }
    CU(cudaMemcpyAsync(x, dx, 8 * (size_t)n, cudaMemcpyDeviceToHost, s));
    if (hist && hist_cap > 0 && nit > 0)
      CU(cudaMemcpyAsync(hist, dh, 8 * (size_t)std::min(nit, hist_cap), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    *its = nit;
  });
}

int igb_host_alloc(igb_ctx* ctx, long long bytes, void** hptr) {
  return guarded(ctx, [&] {
    CU(cudaSetDevice(ctx->device));
    CU(cudaHostAlloc(hptr, (size_t)bytes, cudaHostAllocDefault));
  });
}
int igb_host_free(igb_ctx* ctx, void* hptr) {
  return guarded(ctx, [&] { CU(cudaFreeHost(hptr)); });
}

int igb_device_alloc(igb_ctx* ctx, long long bytes, void** dptr) {
  return guarded(ctx, [&] {
    CU(cudaSetDevice(ctx->device));
    CU(cudaMalloc(dptr, (size_t)bytes));
  });
}
int igb_device_free(igb_ctx* ctx, void* dptr) {
  return guarded(ctx, [&] { CU(cudaFree(dptr)); });
}
int igb_memcpy_h2d(igb_ctx* ctx, void* dst, const void* src, long long bytes) {
  return guarded(ctx, [&] {
    CU(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  });
}
int igb_memcpy_d2h(igb_ctx* ctx, void* dst, const void* src, long long bytes) {
  return guarded(ctx, [&] {
    CU(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
  });
}

int igb_last_timing(igb_ctx* ctx, double* pcg_ms, double* cycle_ms_avg) {
  return guarded(ctx, [&] {
    if (pcg_ms) *pcg_ms = ctx->last_pcg_ms;
    if (cycle_ms_avg) *cycle_ms_avg = ctx->last_cycle_ms;
  });
}

int igb_profile_enable(igb_ctx* ctx, int on) {
  return guarded(ctx, [&] {
    ctx->prof = on != 0;
  });
}
int igb_profile_reset(igb_ctx* ctx) {
  return guarded(ctx, [&] {
    for (int c = 0; c < K_NCLASS; ++c) {
      ctx->prof_ms[c] = 0;
      ctx->prof_n[c] = 0;
      ctx->prof_bytes[c] = 0;
      ctx->prof_flops[c] = 0;
      ctx->top_bytes[c] = ctx->top_ms[c] = 0;
      ctx->top_n[c] = 0;
    }
  });
}
int igb_launch_count(igb_ctx* ctx, long long* kernels, int reset) {
  return guarded(ctx, [&] {
    if (kernels) *kernels = ctx->launches_direct + ctx->graph_kernels * ctx->graph_replays;
    if (reset) {
      ctx->launches_direct = 0;
      ctx->graph_replays = 0;
    }
  });
}

int igb_profile_flops(igb_ctx* ctx, int cls, double* flops) {
  return guarded(ctx, [&] {
    if (cls < 0 || cls >= K_NCLASS) throw ArgError("unknown kernel class");
    if (flops) *flops = ctx->prof_flops[cls];
  });
}

int igb_profile_top(igb_ctx* ctx, int cls, double* ms, long long* launches, double* bytes_per_launch) {
  return guarded(ctx, [&] {
    if (cls < 0 || cls >= K_NCLASS) throw ArgError("unknown kernel class");
    if (ms) *ms = ctx->top_ms[cls];
    if (launches) *launches = ctx->top_n[cls];
    if (bytes_per_launch) *bytes_per_launch = ctx->top_bytes[cls];
  });
}

int igb_gs_info(igb_ctx* ctx, int level, int dir, int* info, int ninfo) {
  return guarded(ctx, [&] {
    require_levels(ctx);
    if (dir != 0 && dir != 1) throw ArgError("dir must be 0 (forward) or 1 (backward)");
    Level& V = ctx->level(level);
    if (!V.has_gs) throw StateError("no Gauss-Seidel smoother on this level");
    int v[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const Sched& Sd = dir ? V.bwd : V.fwd;
    v[6] = Sd.nlev;
    if (V.panel[dir].ok) {
      const PanelArgs& a = V.panel[dir].args;
      v[0] = 1; v[1] = a.B; v[2] = a.KA; v[3] = a.KF; v[4] = a.nclu; v[5] = a.npan;
    } else if (V.wave[dir].ok) {
      v[0] = 6; v[1] = V.wave[dir].args.rb_max; v[4] = V.wave[dir].args.nb; v[5] = V.wave[dir].nframes;
      v[6] = V.wave[dir].nlev;
    } else if (V.line[dir].ok) {
      v[0] = 5; v[1] = V.line[dir].args.rb_max; v[2] = V.line[dir].args.C; v[4] = V.line[dir].args.nb;
      v[5] = V.line[dir].nl;
    } else if (V.flow[dir].ok) {
      v[0] = 2; v[1] = V.flow[dir].args.G; v[4] = V.flow[dir].args.ctas; v[6] = V.flow[dir].nlev;
    } else if (V.sweep[dir].ok) {
      v[0] = 3; v[4] = V.sweep[dir].args.cluster;
    } else {
      v[0] = 4;
    }
    v[7] = V.n;
    for (int i = 0; i < ninfo && i < 8; ++i) info[i] = v[i];
  });
}

int igb_profile_get(igb_ctx* ctx, int cls, double* ms, long long* launches, double* bytes) {
  return guarded(ctx, [&] {
    if (cls < 0 || cls >= K_NCLASS) throw ArgError("unknown kernel class");
    if (ms) *ms = ctx->prof_ms[cls];
    if (launches) *launches = ctx->prof_n[cls];
    if (bytes) *bytes = ctx->prof_bytes[cls];
  });
}

}  // extern "C"
