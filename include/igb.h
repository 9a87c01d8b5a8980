/*
 * igb.h -- C ABI of the B200-native MG-PCG solve phase (libigb.so).
 *
 * The reference (igamg, pure Python/SciPy) has no native interface; each
 * entry point below replaces the Python call that the reference's solve
 * phase makes, so a host binding (ctypes / cffi / a C++ driver) can swap the
 * CPU path for the device path one call at a time:
 *
 *   igb_set_level_matrix   <- MultigridSolver.__init__ storing A_l
 *                             (reference pkg/src/igamg/multigrid.py:92-99)
 *   igb_set_prolongation   <- assembly.prolongation / self.P[l]
 *                             (assembly.py:672-702, multigrid.py:96)
 *   igb_set_prolongation_kron <- the same P in per-patch Kronecker form
 *                             (assembly.py:672-702, bspline.py:233-246)
 *   igb_set_gs             <- smoothers.GaussSeidel.__init__ (smoothers.py:174-184)
 *   igb_scms_add_interior  <- smoothers.ScmsInteriorSolver.__init__ (smoothers.py:232-281)
 *   igb_scms_add_piece     <- SubspaceCorrectedMass piece factorizations (smoothers.py:316-319)
 *   igb_set_coarse_lu      <- linsolve.factorize(A_0) (multigrid.py:100, linsolve.py:33-46)
 *   igb_set_cycle          <- CycleConfig (multigrid.py:23-50) + build_smoother kind
 *   igb_cycle              <- MultigridSolver.cycle (multigrid.py:118-138)
 *   igb_pcg / igb_pcg_device <- linsolve.cg(A_L, b, preconditioner=cycle) (linsolve.py:64-101)
 *   igb_op                 <- single hot-path operators for parity tests:
 *                             A@x, f-A@u (scipy csr_matvec), GaussSeidel.apply_forward /
 *                             apply_backward (smoothers.py:186-190),
 *                             SubspaceCorrectedMass.apply (smoothers.py:321-325),
 *                             P.T@r, P@e (multigrid.py:127,130,134),
 *                             coarse_solver(r) (linsolve.py:48-53)
 *
 * Conventions: every function returns 0 on success and a negative code on
 * failure (igb_last_error(ctx) gives a message).  Host pointers are borrowed
 * for the duration of the call (data is copied).  All matrices are CSR with
 * int32 indices and float64 values, rows with sorted column indices.  Level 0
 * is the coarsest level; cycles act on levels >= 1 (multigrid.py:120-121).
 * A context owns one CUDA stream and all device memory; it is not thread-safe.
 */
#ifndef IGB_H
#define IGB_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct igb_ctx igb_ctx;

enum {
  IGB_OK = 0,
  IGB_ERR_ARG = -1,
  IGB_ERR_CUDA = -2,
  IGB_ERR_STATE = -3,
  IGB_ERR_SINGULAR = -4,
  IGB_ERR_NOMEM = -5
};

/* smoother kinds (smoothers.py:356-367) */
enum { IGB_SMOOTHER_GS = 0, IGB_SMOOTHER_SCMS = 1, IGB_SMOOTHER_HYBRID = 2 };

/* operators for igb_op */
enum {
  IGB_OP_SPMV = 0,      /* out = A_l in                                   */
  IGB_OP_RESIDUAL = 1,  /* out = out - A_l in  (out holds f on entry)      */
  IGB_OP_GS_FWD = 2,    /* out = tril(A_l)^{-1} in                          */
  IGB_OP_GS_BWD = 3,    /* out = tril(A_l)^{-T} in                          */
  IGB_OP_SCMS = 4,      /* out = tau * sum_T P_T L_T^{-1} P_T^T in          */
  IGB_OP_RESTRICT = 5,  /* out = P_l^T in   (in: n_l, out: n_{l-1})         */
  IGB_OP_PROLONG = 6,   /* out = P_l in     (in: n_{l-1}, out: n_l)         */
  IGB_OP_COARSE = 7,    /* out = A_0^{-1} in (level ignored)                */
  IGB_OP_CYCLE = 8      /* out = cycle(l, in) from u = 0                    */
};

int igb_create(igb_ctx** ctx, int device);
int igb_destroy(igb_ctx* ctx);
const char* igb_last_error(igb_ctx* ctx);
int igb_version(void);

/* Hierarchy with levels 0..L (L >= 1). Must be called first. */
int igb_set_num_levels(igb_ctx* ctx, int L);

/* A_l (l = 0..L): n x n CSR. */
int igb_set_level_matrix(igb_ctx* ctx, int level, int n, long long nnz,
                         const int* indptr, const int* indices, const double* data);

/* P_l (l = 1..L): n_l x n_{l-1} CSR; the transpose for restriction is built here. */
int igb_set_prolongation(igb_ctx* ctx, int level, int n_fine, int n_coarse, long long nnz,
                         const int* indptr, const int* indices, const double* data);

/* Kronecker form of P_l (replaces assembly.prolongation's assembled matrix on the device,
 * assembly.py:672-702: per patch the kron of bspline.two_scale_refine 1-D matrices,
 * bspline.py:233-246, mapped to free DoFs with shared rows assigned once).  With
 * IGB_TRANSFER=kron in the environment restriction and prolongation on level l use it; by
 * default the CSR pair of igb_set_prolongation runs (measured faster on B200 at the BASELINE
 * sizes).  Needs both level matrices set.
 *   nf, nc      [npatch * dim] per-patch block sizes per axis, fine / coarse level
 *   p1_idx/val  the 1-D matrices P_{k,a} (patch-major, then axis), each n_f,a rows of
 *               `width` ELL entries, columns ascending, -1 = padding
 *   fine_free   [sum_k prod nf] block index -> free id (-1 Dirichlet); coarse_free likewise
 *   fine_owner  [sum_k prod nf] 1 where the block copy is its DoF class root, else 0 */
int igb_set_prolongation_kron(igb_ctx* ctx, int level, int dim, int npatch, const int* nf, const int* nc,
                              int width, const int* p1_idx, const double* p1_val, const int* fine_free,
                              const int* fine_owner, const int* coarse_free);

/* Matrix-free form of A_l for conforming spaces on affine patches (assembly.py:333-344: per patch
 * sum_a c_a (x)_i (K_i if i == a else M_i) reduced to free DoFs, shared copies summed).  Full products
 * A_l x (residuals, the CG product) then run by sum factorisation instead of reading A_l
 * (IGB_MATRIX_FREE=0 keeps the CSR).  The CSR of igb_set_level_matrix stays required (Gauss-Seidel).
 *   dims   [npatch * dim] block sizes;  c [npatch * dim] coefficient of stiffness term a
 *   Mband, Kband  1-D mass / stiffness per (patch, axis) as n x (2p+1) bands (entry j - i + p)
 *   block_free    [sum prod dims] block index -> free id (-1 Dirichlet) */
int igb_set_matrix_free(igb_ctx* ctx, int level, int dim, int npatch, int p, const int* dims, const double* c,
                        const double* Mband, const double* Kband, const int* block_free);

/* Gauss-Seidel on A_l in natural order (level schedules are built here).  Call it after the
 * level's igb_scms_add_interior calls when the smoother is hybrid: the sweep planner tunes the flow
 * sweep's early / late split by the level's dimension (results do not depend on it, only speed). */
int igb_set_gs(igb_ctx* ctx, int level);

/* SCMS smoother of level l: damping tau; then interiors and interface pieces. */
int igb_scms_begin(igb_ctx* ctx, int level, double tau);
/* One patch interior: dim in {2,3}; dims[a] = n_a; T_a is n_a x n_a row-major
 * (columns = eigenvectors of the split subspaces, [W_L V_L | W_C V_C]);
 * denom has prod(n_a) entries (C order); idx maps the C-order tensor to free ids.
 * T2 is ignored when dim == 2. Interiors whose T / denom have identical content share one device
 * copy (content-hashed and compared; buffers are copied during the call and may be reused).
 * Any index set whose piece operator has this tensor form may be passed: a 3-D level also takes
 * dim == 2 items (sides <= 160) -- the faces between conforming affine patches, whose SuperLU solve
 * (reference smoothers.py:316-319) equals X = V1 ((V1^T R V2) ./ denom) V2^T with the generalized
 * eigenvectors of the tangential 1-D stiffness / mass pairs. */
int igb_scms_add_interior(igb_ctx* ctx, int level, int dim, const int* dims,
                          const double* T0, const double* T1, const double* T2,
                          const double* denom, const int* idx);
/* One interface piece (edge/face/vertex): m free ids and the dense inverse
 * (m x m row-major) of A_l[idx][:, idx]. */
int igb_scms_add_piece(igb_ctx* ctx, int level, int m, const int* idx, const double* inv);

/* Coarse solver from SciPy SuperLU factors of A_0: Pr A Pc = L U with
 * Pr[perm_r[i], i] = 1, Pc[i, perm_c[i]] = 1. L, U given as CSR (n0 x n0). */
int igb_set_coarse_lu(igb_ctx* ctx, int n0,
                      long long l_nnz, const int* l_ptr, const int* l_idx, const double* l_val,
                      long long u_nnz, const int* u_ptr, const int* u_idx, const double* u_val,
                      const int* perm_r, const int* perm_c);

/* Cycle shape: smoother kind, mu (1 = V, 2 = W), steps per level (L+1 entries, index = level). */
int igb_set_cycle(igb_ctx* ctx, int smoother, int mu, const int* steps_per_level);

/* Upload done: validates the hierarchy and captures the cycle as a CUDA graph. */
int igb_finalize(igb_ctx* ctx);

/* One cycle on level l from u = 0 (host buffers of length n_l). */
int igb_cycle(igb_ctx* ctx, int level, const double* f, double* u);

/* Single operator (host buffers). */
int igb_op(igb_ctx* ctx, int op, int level, const double* in, double* out);

/* Preconditioned CG on A_L with one cycle as preconditioner, x0 = 0
 * (linsolve.py:64-101 semantics). Host buffers: b, x (length n_L), hist
 * (capacity hist_cap; hist[i] = ||r_{i+1}|| / ||b||). *its receives the
 * iteration count (max_iters if not converged). */
int igb_pcg(igb_ctx* ctx, const double* b, double tol, int max_iters,
            double* x, int* its, double* hist, int hist_cap);

/* Smoother duck type (smoothers.py:192-200 GaussSeidel, 327-332 SubspaceCorrectedMass,
 * 343-353 HybridSmoother): u <- pre_smooth / post_smooth(A_l, u, f, steps) with smoother kind
 * IGB_SMOOTHER_* on level l (post != 0: post-smoothing), host buffers (u in/out). */
int igb_smooth(igb_ctx* ctx, int level, int kind, int post, int steps, const double* f, double* u);

/* General PCG: linsolve.cg(A, b, preconditioner, tol, max_iters, callback) (linsolve.py:64-101)
 * for any operator and preconditioner, with a live per-iteration callback.
 *   A: n x n CSR (copied for the call), or indptr == NULL for the context's finest operator;
 *   prec_mode: IGB_PREC_NONE (z = r), IGB_PREC_CYCLE (one cycle of the context's hierarchy from
 *   u = 0, as MultigridSolver.preconditioner()), IGB_PREC_HOST (prec(r, z, n, prec_user) on host
 *   buffers: the reference's arbitrary callable);
 *   iter_cb(it, rel, iter_user) after every iteration (nullable).
 * Same stopping rule, history and non-convergence semantics as igb_pcg (which runs the whole
 * solve as one CUDA graph and is the fast path for the cycle preconditioner without callback). */
enum { IGB_PREC_NONE = 0, IGB_PREC_CYCLE = 1, IGB_PREC_HOST = 2 };
typedef void (*igb_prec_fn)(const double* r, double* z, int n, void* user);
typedef void (*igb_iter_fn)(int it, double rel, void* user);
int igb_cg(igb_ctx* ctx, int n, long long nnz, const int* indptr, const int* indices, const double* data,
           int prec_mode, igb_prec_fn prec, void* prec_user, igb_iter_fn iter_cb, void* iter_user,
           const double* b, double tol, int max_iters, double* x, int* its, double* hist, int hist_cap);

/* Same with device-resident b and x (device pointers); hist stays a host buffer. */
int igb_pcg_device(igb_ctx* ctx, const double* d_b, double tol, int max_iters,
                   double* d_x, int* its, double* hist, int hist_cap);

/* Device scratch helpers for device-resident benchmarking. */
/* Pinned (page-locked) host buffers for the host-buffer entry points (igb_pcg's b and x): the
 * copies then run at full link speed inside the solve's single synchronisation. */
int igb_host_alloc(igb_ctx* ctx, long long bytes, void** hptr);
int igb_host_free(igb_ctx* ctx, void* hptr);

int igb_device_alloc(igb_ctx* ctx, long long bytes, void** dptr);
int igb_device_free(igb_ctx* ctx, void* dptr);
int igb_memcpy_h2d(igb_ctx* ctx, void* dst, const void* src, long long bytes);
int igb_memcpy_d2h(igb_ctx* ctx, void* dst, const void* src, long long bytes);

/* Device milliseconds (CUDA events) of the last igb_pcg / igb_pcg_device CG loop,
 * and the average device time of one cycle in it. */
int igb_last_timing(igb_ctx* ctx, double* pcg_ms, double* cycle_ms_avg);

/* Kernels launched by the library since the last reset (direct launches plus
 * kernels replayed from the captured cycle graph); reset != 0 clears the count. */
int igb_launch_count(igb_ctx* ctx, long long* kernels, int reset);

/* Per-kernel-class accumulated device time (ms) and launch counts since
 * igb_profile_reset; classes: 0 spmv, 1 gs, 2 fd, 3 pieces, 4 transfer,
 * 5 coarse, 6 cg-vector. Enabled by igb_profile_enable(ctx, 1). */
int igb_profile_enable(igb_ctx* ctx, int on);
int igb_profile_reset(igb_ctx* ctx);
int igb_profile_get(igb_ctx* ctx, int cls, double* ms, long long* launches, double* bytes);
/* Algorithmic flops of a class since igb_profile_reset (the fast-diagonalisation class 2:
 * 4 prod(n) sum_a n_a per interior and application, i.e. 8 n^3 in 2-D, 12 n^4 in 3-D). */
int igb_profile_flops(igb_ctx* ctx, int cls, double* flops);
/* The class's largest launch since igb_profile_reset (most algorithmic bytes per launch: the
 * finest level's kernel): accumulated time, count and the bytes of one such launch -- the launch
 * an ncu capture of the class's dominant kernel shows, so roofline and traffic refer to the same
 * thing (bench.py; no reference counterpart: measurement only). */
int igb_profile_top(igb_ctx* ctx, int cls, double* ms, long long* launches, double* bytes_per_launch);

/* Which Gauss-Seidel engine igb_set_gs planned for (level, dir) (dir 0 forward, 1 backward);
 * info[0..ninfo) receives: engine (1 panel sweep, 2 flow sweep, 3 level-set sweep, 4 level
 * schedule, 5 line sweep), panel rows B (flow: lanes per row; line: largest bundle), KA near
 * slots (line: chunks per row), KF far slots, clusters / ranges (flow: CTAs; line: bundles),
 * panels (line: lines), dependency levels, n.  Diagnostic; no reference counterpart.
 * Note: the opt-in B = 256 / KF 10 panel variant (IGB_PANEL_KF10=1) reads the level's dimension
 * from its interiors, so with it igb_set_gs must follow igb_scms_add_interior; by default the
 * plan does not depend on call order. */
int igb_gs_info(igb_ctx* ctx, int level, int dir, int* info, int ninfo);

#ifdef __cplusplus
}
#endif
#endif /* IGB_H */
