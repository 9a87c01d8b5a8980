// kernels.cuh -- device kernels of the MG-PCG solve phase (sm_100a, fp64).
//
// Every kernel here replaces one third-party native routine that the
// reference's solve phase calls:
//   spmv_*          scipy csr_matvec / csc_matvec        (A@x, f-A@u, P@e, P.T@r)
//   sptrsv_levels   SuperLU dgstrs on tril(A) / coarse LU (GS sweeps, coarse solve)
//   fd_gemm         OpenBLAS dgemm under np.tensordot    (SCMS fast diagonalisation)
//   piece_gemv      SuperLU dgstrs on interface pieces   (SCMS edge/face/vertex)
//   cg_*            numpy BLAS-1 in linsolve.cg          (dots, norm, axpy)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <utility>

namespace igb {

// Programmatic dependent launch: every kernel of the solve is launched with the
// programmatic-serialization attribute and begins with pdl_begin() (griddepcontrol.wait:
// the predecessor grid has completed and its writes are visible; then allow the next
// kernel to be scheduled).  The successor's launch and ramp-up overlap this kernel's tail
// instead of a full drain between dependent kernels.  IGB_PDL=0 disables the attribute.
inline bool pdl_enabled() {
  static const bool on = !(std::getenv("IGB_PDL") && std::atoi(std::getenv("IGB_PDL")) == 0);
  return on;
}
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
#endif
template <class... KArgs, class... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Same preferred shared-memory carveout for every kernel (kernels.cu).
void carveout_prepare();
void set_carveout_panel_fd(int pct);   // panel.cu / fd.cu kernels

// ---- CSR SpMV: y = z + sign * A x  (sign 0: y = A x; sign < 0 and z null: y = -A x) ------
void launch_spmv(cudaStream_t s, int n, const int* ptr, const int* col, const double* val,
                 const double* x, const double* z, double* y, int sign, int group);

// ---- level-scheduled triangular solve, one CTA ---------------------------------
// Solves rows in level order.  For row i (taken from `rows`):
//   lower (fwd):  uses entries [ptr[i], dpos[i])      x_i = (b_i - s) / val[dpos[i]]
//   upper (bwd):  uses entries (dpos[i], ptr[i+1])    x_i = (b_i - s) / val[dpos[i]]
// b_i = rhs[rhs_idx ? rhs_idx[i] : i].  If uacc: uacc[i] += x_i.
struct TrsvPhase {
  int nlev;
  const int* lvl_ptr;   // nlev+1
  const int* rows;      // n
  const int* ptr;       // CSR
  const int* col;
  const double* val;
  const int* dpos;      // diagonal position per row
  int upper;            // 0 fwd / 1 bwd
  const double* rhs;
  const int* rhs_idx;   // nullable gather
  double* x;            // solution (also read for dependencies)
  double* uacc;         // nullable: uacc[i] += x_i
};
// One or two phases run back to back in one launch (coarse: L then U), then an
// optional output gather out[i] = x_last[out_idx[i]] for i < n_out.
void launch_sptrsv(cudaStream_t s, const TrsvPhase& a, const TrsvPhase* b,
                   int n_out, const int* out_idx, double* out);

// ---- level-set triangular sweep (Gauss-Seidel in natural order), one CTA ----
// See level_plan.h: vectors in level order, step metadata staged in shared memory.
struct LevelMetaDev {
  int off16, K, nrows, start;
};
struct LevelArgs {
  const LevelMetaDev* meta;
  int nsteps;
  const unsigned char* stream;
  const double* rp;   // right-hand side in level order
  double* xp;         // solution in level order
  int TPR, R;
  int has_old;        // some entries read values outside the shared ring
  int cluster;        // CTAs per sweep (thread-block cluster when > 1)
  long long* dbg;     // nullable: clock64 totals of thread 0 (debug)
  int ablate;         // debug: bit0 skip loads, bit1 skip dot, bit2 skip reduce+store
};
constexpr int LEVEL_NT = 384;
constexpr int LEVEL_KMAX = 8;
size_t level_smem_bytes(const LevelArgs& a);
void level_prepare();
void launch_level_sweep(cudaStream_t s, const LevelArgs& a);
// out[i] = in[rows[i]]  /  u[rows[i]] (+)= xp[i]
void launch_perm_gather(cudaStream_t s, int n, const int* rows, const double* in, double* out);
void launch_perm_scatter(cudaStream_t s, int n, const int* rows, const double* xp, double* u, int accumulate);

// ---- row-panel triangular sweep (Gauss-Seidel in natural order), one cluster ----
// See panel_plan.h: G CTAs x W warps (16 or 8), panels of B = 2 G W rows, inverse blocks
// streamed by TMA, recent solution values in a DSMEM-broadcast ring of R slots.
constexpr int PANEL_W = 16;
constexpr int PANEL_STAGES = 2;   // TMA stages of the inverse slices (power of two)
struct PanelArgs {
  const double* lin;  // [npan][G][W][KBC][32]
  const double* ev;   // [npan][G][W][KA][32]
  const int* ec;
  const double* fv;   // [npan][G][W][KF][32]
  const int* fc;
  const unsigned short* xmask;  // [npan*B] destination CTAs of each solution value
  const int* xcnt;              // [npan+1][G] values each CTA receives per panel
  const double* res;  // right-hand side by row
  double* u;          // u (+)= c by row
  double* xg;         // [2][n] c by position, halves by sweep parity (only when KF > 0)
  int* par_ctr;       // sweep parity of this level and direction (device)
  unsigned* done_ctr; // CTAs finished (device), reset by the last one
  int n, npan, B, R, G, KBC, KA, KF;
  int nclu;           // clusters, one per panel range
  int split[9];       // panel ranges: cluster c sweeps panels [split[c], split[c+1]) ...
  int rstart[9];      // ... = positions [rstart[c], rstart[c+1]), panels of B rows from rstart[c]
  int upper, accumulate, pf;
  long long* dbg;     // nullable: clock64 totals of CTA 0 thread 0 (debug)
  int ablate;         // debug: bit0 no TMA, bit1 no cluster barriers, bit2 no inverse product,
                      // bit3 local stores only, bit4 no phase-A gathers,
                      // bit5 no u / xg traffic, bit7 no L2 evict-first hint on the inverse stream
};
size_t panel_smem_bytes(const PanelArgs& a);
bool panel_prepare(int G, int KBC);   // false: no cluster of G CTAs fits this device
int panel_max_clusters(int G, int KBC, size_t smem);  // clusters of G CTAs co-resident
void launch_panel_sweep(cudaStream_t s, const PanelArgs& a);

// ---- dependency-driven triangular sweep over the whole GPU (flow.cu, flow_plan.h) ----
// Rows in dependency-level order (list slot q -> row[q], -1 = padding), strict-triangle
// entries of slot q at [eptr[q], eptr[q+1]) (ecol: row index, eval), idiag[q] = 1 / a_qq.
// Solution values published in xg[par][row] (sentinel until produced; see flow.cu).
constexpr int FLOW_NT = 256;
struct FlowArgs {
  const int* row;      // [nq]
  const int* eptr;     // [nq + 1]
  const int* ecol;
  const double* eval;
  const double* idiag; // [nq]
  const double* res;   // right-hand side by row
  double* u;           // u (+)= c by row
  double* xg;          // [2][n]
  int* par_ctr;        // sweep parity of this level and direction (device)
  unsigned* done_ctr;  // CTAs finished (device), reset by the last one
  int n, nq, G, ctas, accumulate;
  const int* crit;     // nullable: [nq] the dependency of the highest level (polled first)
  const int* elate;    // [nq] first late entry of the row (flow_plan.h): early entries are reduced
                       // first, the late ones (newest dependencies) added serially by every lane
  int backoff;         // ns slept between polls of crit (0: spin)
  int prefetch;        // L2-prefetch the next row's entries while the current row is processed
  long long* trace;    // debug (nullable): per slot globaltimer at start / deps ready / stored
};
int flow_max_ctas();  // co-resident CTAs of FLOW_NT threads (all variants)
void flow_set_carveout(int pct);
void launch_flow_sweep(cudaStream_t s, const FlowArgs& a);

// ---- wave sweep: GS with the dependency chain inside one CTA per grid plane (wave.cu, wave_plan.h)
constexpr int WAVE_NT = 1024;  // 32 warps per CTA, one CTA per SM
struct WaveHdr;
struct WaveRecA;
struct WaveRecB;
struct WaveArgs {
  const int* b_frame;  // [nb + 1] first frame of each bundle
  const int* b_start;  // [nb + 1] first row (sweep order) of each bundle
  const int* f_end;    // [nframes] rows of the frame's bundle in frames up to and including it
  const WaveHdr* hdr;  // [n] sweep order
  const int* lcol;     // [n * LN] late entries (rows, -1 none)
  const double* lval;
  const WaveRecA* recA;
  const WaveRecB* recB;
  const int* e_row;    // external list (flow layout)
  const int* eptr;
  const int* ecol;
  const double* eval;
  const int* crit;
  const int* elate;
  const double* res;   // right-hand side by row
  double* u;           // u (+)= c by row
  double* xg;          // [2][n] solution by row, pending until produced
  double* eg;          // [2][n] external sums by row, pending until produced
  int* par_ctr;        // sweep parity of this level and direction (device)
  unsigned* done_ctr;  // CTAs finished (device), reset by the last one
  int* ticket;         // next bundle to hand out (device), rewound by the last CTA
  int n, nb, nq, ctas, accumulate, backoff, pbackoff;   // backoff: ns slept between polls (external warps / pollers)
  int rb_max, xs_len;
  unsigned long long* dbg;   // nullable: 8 counters (wave.cu)
};
size_t wave_smem_bytes(int rb_max);
int wave_xs_len(int rb_max);
int wave_max_ctas(size_t smem);
void wave_set_carveout(int pct);
void launch_wave_sweep(cudaStream_t s, const WaveArgs& a);

// ---- line sweep: GS along grid lines, bundles of lines per CTA (line.cu, line_plan.h) -------
constexpr int LINE_NT = 512;  // 16 warps per CTA
struct LineArgs {
  const int* bstart;   // [nb + 1] positions
  const int* bline;    // [nb + 1] first line per bundle
  const int* lstart;   // [nl + 1] positions
  const char* rec;     // [n] fixed-size records (line_plan.h), line_rec_bytes(C) each
  const int* ocol;     // overflow chunks of long rows (codes / values)
  const double* oval;
  const double* res;   // right-hand side by row
  double* u;           // u (+)= c by row
  double* xg;          // [2][n] by position
  int* par_ctr;
  unsigned* done_ctr;
  int n, nb, rb_max, C, upper, accumulate, ctas, pf;
  long long* trace;    // debug (nullable): per position [publish globaltimer, D poll cycles, C poll cycles]
  long long* prof;     // debug (nullable): [5] cycles summed over warps in D-poll, D, C, B, A + [5] rows
};
int line_chunk_variant(int C);           // kernel variant for C chunks per row (-1: none)
int line_max_ctas(size_t smem_bytes);    // co-resident CTAs of LINE_NT threads
void launch_line_sweep(cudaStream_t s, const LineArgs& a);

// ---- intergrid transfers as per-patch Kronecker products (transfer.cu) --------------
struct KronPatch {
  int nf[3], nc[3];            // block sizes per axis (1 past dim)
  long long ell[3], ellT[3];   // row-0 offsets of P_{k,a} / P_{k,a}^T in the ELL pools
};
constexpr int KRON_MAXP = 16;  // patches per level in the kernel-parameter tables (size: launch cost)
struct KronArgs {
  int dim, npatch, width, widthT, n_fine, n_coarse;
  long long nblk_f, nblk_c;
  KronPatch patch[KRON_MAXP];                     // per-patch sizes and ELL row offsets
  long long off_f[KRON_MAXP + 1], off_c[KRON_MAXP + 1];  // block offsets
  const int* pidx; const double* pval;    // ELL rows (width) of the 1-D matrices, col -1 = pad
  const int* tidx; const double* tval;    // ELL rows (widthT) of their transposes
  const int* fown;   // fine block -> free if the copy is the owner (class root), else -1
  const int* cfree;  // coarse block -> free (-1: Dirichlet)
  const int* croot;  // coarse block -> free if the copy is the class root, else -1
  const int* xptr; const int* xblk;  // coarse free DoF -> its non-root block copies
};
void kron_set_carveout(int pct);
int kron_width(int w);    // compiled ELL widths: smallest >= w, -1 if none
int kron_width_t(int w);
void launch_kron_prolong(cudaStream_t s, const KronArgs& a, const double* e, const double* z, double* y,
                         int accumulate);
void launch_kron_restrict(cudaStream_t s, const KronArgs& a, const double* r, double* y);

// ---- matrix-free finest-level operator on affine conforming patches (mfree.cu) ----------
constexpr int MF_MAXP = 16;
struct MfArgs {
  int dim, npatch, p, nfree;
  long long nblk;
  long long off[MF_MAXP + 1];      // block offsets per patch
  int n[MF_MAXP][3];               // block sizes per axis
  long long band[MF_MAXP][3];      // offsets of the (n x (2p+1)) band arrays in Mb / Kb
  double c[MF_MAXP][3];            // det / s_a^2 per stiffness term
  const double* Mb; const double* Kb;
  const int* bfree;                // block -> free (-1 Dirichlet)
  const int* froot; const int* xptr; const int* xblk;  // free -> root block, other copies
};
void mf_set_carveout(int pct);
void launch_mf_apply(cudaStream_t s, const MfArgs& a, const double* x, const double* z, double* y, int sign,
                     double* const scratch[4]);

// ---- coarse solve: column-oriented sparse LU substitution, one CTA, rhs in smem
// y[k] = rhs[inv_perm_r[k]];  L y = y (unit lower, CSC);  U w = y (CSC, diag at udiag[j]);
// out[i] = w[perm_c[i]].  Column j updates run in parallel; one barrier per column.
struct CoarseCsc {
  int n;
  const int* lcp; const int* lri; const double* lv;   // strictly lower part of L, CSC
  const int* ucp; const int* uri; const double* uv;   // strictly upper part of U, CSC
  const double* udiag;                                 // diag of U
  const int* inv_perm_r; const int* perm_c;
  long long lnnz, unnz;                                // host copies of lcp[n], ucp[n]
};
void launch_coarse_csc(cudaStream_t s, const CoarseCsc& c, const double* rhs, double* out);

// ---- batched fp64 GEMM for fast diagonalisation ------------------------------
struct GemmDesc {
  int M, N, K, nb;           // nb batches with batch strides
  long long a_rs, a_cs, a_bs;
  long long b_rs, b_cs, b_bs;
  long long c_rs, c_cs, c_bs;
  const double* A;
  const double* B;
  const int* b_idx;          // gather: B(k,j) = gsrc[b_idx[off]] (B unused)
  double* C;
  const int* c_idx;          // scatter: sdst[c_idx[off]] (+)= alpha * acc
  const double* D;           // divide: acc / D[off_c]
  int tiles_m, tiles_n;
  int tile_base;             // prefix over descriptors
};
// gsrc: gather source for descriptors with b_idx; sdst: scatter target for
// descriptors with c_idx (u[idx] = (accumulate ? u[idx] : 0) + alpha * acc).
void launch_fd_gemm(cudaStream_t s, const GemmDesc* d_descs, int ndesc, int total_tiles,
                    const double* gsrc, double* sdst, double alpha, int accumulate);

// ---- fused 3-factor fast diagonalisation on fp64 tensor cores (fd3.cu) --------
constexpr int FD3_NMAX = 72;       // largest interior side (multiple of 8)
constexpr int FD3_MAXWARPS = 9;
struct Fd3Item {
  const double* T[3];   // n_a x n_a, row-major
  const double* D;      // prod n_a
  const int* idx;       // prod n_a
  double* buf0;         // Y  (modes 1, 2 transformed)
  double* buf1;         // W  (mode 0 transformed, divided, mode 0 back)
  int n[3];
  int slab0, slab1;     // first CTA of this interior in the i0-slab / i1-slab launches
};
struct Fd3Plan {
  Fd3Item* d_items = nullptr;
  int nitems = 0, n8 = 0, slabs0 = 0, slabs1 = 0;
  int lr_shared = 0;    // every interior has T[1] == T[2]: two shared-memory buffers per CTA
};
void launch_fd3(cudaStream_t s, const Fd3Plan& P, int stage, const double* r, double* u, double alpha, int accumulate);
void fd3_set_carveout(int pct);

// ---- fused fast diagonalisation of small 2-D interiors (one CTA per interior) --
// X = T0 ((T0^T R T1) ./ D) T1^T with R = r[idx] and u[idx] (+)= alpha X, all in smem.

// ---- interface-piece dense solves (precomputed inverses) ---------------------
struct PieceRowBlock {
  const double* inv;   // m x m
  const int* idx;      // m
  int m;
  int row0;            // first row handled by this block
  int nrows;           // rows in this block (piece_gemv: any; fused FD back kernel: <= its warps)
};

// ---- fused 2-D fast diagonalisation (fd.cu): two launches per application, RB rows of
// one interior per CTA, all interiors of a level (up to FD_BATCH_MAX per batch) in one grid.
// n0, n1 <= FDC_NMAX; scratch: n0 * n1 doubles per interior (the middle intermediate).
constexpr int FDC_NMAX = 160;
constexpr int FDC_NT = 160;
constexpr int FDL_NMAX = 264;  // large variant: right operands streamed in chunks
constexpr int FDL_NT = 264;   // one column per thread (8.25 warps)
constexpr int FD_BATCH_MAX = 16;
struct FdCluster {
  const double* T0;
  const double* T1;
  const double* D;
  const int* idx;
  double* scratch;
  int n0, n1;
};
struct FdBatch {
  FdCluster items[FD_BATCH_MAX];
  int cta0[FD_BATCH_MAX + 1];  // first CTA of each item; cta0[nitems] = grid size
  int nitems;
  int rb;                      // rows per CTA: 2, 4 or 8
  int kmax;                    // largest n0 / n1 of the batch (shared-memory buffer rows)
  int large;                   // 1: the FDL_NMAX variant (chunked right operands)
  const PieceRowBlock* pieces; // interface-piece rows (<= 5 per block) done by extra CTAs of
  int npieces;                 // the back kernel (disjoint u entries), or none
};
int fd_rows_per_cta(int total_rows);
void launch_fd_batch(cudaStream_t s, const FdBatch& bt, const double* r, double* u, double alpha, int accumulate);

// max_m: the largest piece order among the blocks (shared-memory staging of r[idx]; 0 = none)
void launch_piece_gemv(cudaStream_t s, const PieceRowBlock* d_blocks, int nblocks,
                       const double* r, double* u, double tau, int accumulate, int max_m);

// ---- CG vector kernels with deterministic reductions -------------------------
struct CgScalars {
  double normb, rz, alpha, beta, rel, tol;
  int it, done;
  double pAp, rr;
  int beta_epoch, pad;   // iteration whose beta is published (cg_beta_direction's in-kernel hand-over)
};
enum FinalizeKind { FIN_NORMB = 0, FIN_RZ0 = 1, FIN_ALPHA = 2, FIN_REL = 3, FIN_BETA = 4 };

constexpr int REDUCTION_MAX_BLOCKS = 16384;  // size of the partials buffer (grid-stride beyond)
int reduction_grid(int n);
// q = A d ; then partial d.q -> alpha = rz / (d.q)
void launch_spmv_dot(cudaStream_t s, int n, const int* ptr, const int* col, const double* val,
                     const double* d, double* q, int group, double* partials,
                     unsigned* counter, CgScalars* sc, double* hist);
// dot(a, b) with finalize
void launch_dot(cudaStream_t s, int n, const double* a, const double* b, double* partials,
                unsigned* counter, CgScalars* sc, int kind, double* hist);
// x += alpha d ; r -= alpha q ; rr = r.r -> rel
void launch_cg_update(cudaStream_t s, int n, double* x, double* r, const double* d,
                      const double* q, double* partials, unsigned* counter, CgScalars* sc,
                      double* hist);
// d = z + beta d
void launch_cg_direction(cudaStream_t s, int n, double* d, const double* z, const CgScalars* sc);
// the same two steps in one persistent launch: beta = (r.z) / rz_old by the last block to arrive,
// every block waits for it and updates its part of d = z + beta d (linsolve.py:97-100)
void launch_cg_beta_direction(cudaStream_t s, int n, double* d, const double* z, const double* r, double* partials,
                              unsigned* counter, CgScalars* sc);
// cg_update whose last block also sets the device-side loop conditions (replaces launch_cg_cond
// after the update inside the captured PCG graph)
void launch_cg_update_cond(cudaStream_t s, int n, double* x, double* r, const double* d, const double* q,
                           double* partials, unsigned* counter, CgScalars* sc, double* hist,
                           cudaGraphConditionalHandle loop, cudaGraphConditionalHandle more, int max_iters);
// sets the WHILE (loop) and IF (more) conditions of the device-resident PCG graph
void launch_cg_cond(cudaStream_t s, cudaGraphConditionalHandle loop, cudaGraphConditionalHandle more,
                    const CgScalars* sc, int max_iters, int start);
void launch_copy(cudaStream_t s, int n, double* dst, const double* src);
void launch_fill(cudaStream_t s, int n, double* dst, double v);

}  // namespace igb
