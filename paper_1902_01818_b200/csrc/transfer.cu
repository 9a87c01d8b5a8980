// transfer.cu -- intergrid transfers as per-patch Kronecker products of 1-D two-scale
// matrices (the reference's P, assembly.py:672-702: per patch kron of bspline.two_scale_refine
// matrices, bspline.py:233-246, mapped to free DoFs with shared rows assigned once).
//
//   prolongation  y (=|+=) P e     multigrid.py:130, 134 (u + P e)
//   restriction   y = P^T r        multigrid.py:127 (P^T (f - A u))
//
// Nothing of P is stored but the 1-D matrices (ELL rows, a few KB) and the block <-> free maps,
// so a transfer moves ~16-28 bytes per fine DoF instead of 12 bytes per entry of P ((p+2)^d/2^d
// entries per fine row: 6.25 at p = 3 in 2-D, 15.6 in 3-D) -- HBM-bound, one thread per output.
//
// Prolongation: thread per fine block index; the owner copy (class root) of a free DoF f in
// patch k at multi-index i writes y_f = sum_{a,b(,c)} P_k0[i0,a] P_k1[i1,b] (P_k2[i2,c]) e[free(k;
// a,b,c)] (weights multiplied in the order scipy's kron chain forms the entries of P).
// Restriction: thread per coarse block index; the root copy of coarse free DoF j sums, over its
// block and then the class's other copies (patches sharing j), sum_i P_k0[i0,a] P_k1[i1,b] ...
// r[owner-free(k; i)] -- a fine value is read only through its owner copy, so each fine row of P
// counts once, exactly as in P^T.  Fixed summation order: the result is deterministic.
#include "kernels.cuh"

namespace igb {
namespace {

// patch tables live in the kernel parameters (constant bank): no memory latency on the chain
__device__ __forceinline__ int patch_of(const long long* off, int npatch, long long b) {
  int k = 0;
  while (k + 1 < npatch && off[k + 1] <= b) ++k;
  return k;
}

// All loops have compile-time trip counts (ELL width W / WT, padding index -1 = predicated off),
// so every gather of a thread is issued before the first one is consumed: a transfer costs a few
// dependent memory latencies, not one per entry.

// Prolongation: thread per fine block index b (multi-index by arithmetic); only owner copies
// write (every fine free DoF has exactly one).
template <int DIM, int W>
__global__ void __launch_bounds__(256) kron_prolong_kernel(const __grid_constant__ KronArgs a, const double* __restrict__ e,
                                                           const double* z, double* y, int accumulate) {
  pdl_begin();
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.nblk_f) return;
  const int f = __ldg(a.fown + b);
  if (f < 0) return;
  const int k = patch_of(a.off_f, a.npatch, b);
  const KronPatch& P = a.patch[k];
  int loc = (int)(b - a.off_f[k]);  // 32-bit index arithmetic (blocks < 2^31)
  int i[3] = {0, 0, 0};
#pragma unroll
  for (int d = DIM - 1; d >= 0; --d) {
    const int n = P.nf[d];
    i[d] = (int)(loc % n);
    loc /= n;
  }
  const long long oc = a.off_c[k];
  const int nc1 = P.nc[1], nc2 = DIM == 3 ? P.nc[2] : 1;
  int c[DIM][W];
  double w[DIM][W];
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    const long long r0 = P.ell[d] + (long long)i[d] * W;
#pragma unroll
    for (int t = 0; t < W; ++t) {
      c[d][t] = __ldg(a.pidx + r0 + t);
      w[d][t] = __ldg(a.pval + r0 + t);
    }
  }
  double s = 0.0;
  const int n0 = DIM == 3 ? W : 1;
  for (int t0 = 0; t0 < n0; ++t0) {  // outer axis of 3-D (one pass in 2-D)
    int c0 = c[0][0];
    double w0 = w[0][0];
#pragma unroll
    for (int q = 1; q < W; ++q)  // select without dynamic register-array indexing
      if (q == t0) {
        c0 = c[0][q];
        w0 = w[0][q];
      }
    if (DIM == 3 && c0 < 0) break;
    int cf[W * W];
    double ev[W * W];
#pragma unroll
    for (int ta = 0; ta < W; ++ta)
#pragma unroll
      for (int tb = 0; tb < W; ++tb) {
        const int A = DIM == 3 ? c[1][ta] : c[0][ta], B = DIM == 3 ? c[2][tb] : c[1][tb];
        long long blk = DIM == 3 ? ((long long)c0 * nc1 + A) * nc2 + B : (long long)A * nc1 + B;
        cf[ta * W + tb] = (A >= 0 && B >= 0) ? __ldg(a.cfree + oc + blk) : -1;
      }
#pragma unroll
    for (int q = 0; q < W * W; ++q) ev[q] = cf[q] >= 0 ? __ldg(e + cf[q]) : 0.0;
#pragma unroll
    for (int ta = 0; ta < W; ++ta)
#pragma unroll
      for (int tb = 0; tb < W; ++tb) {
        const int q = ta * W + tb;
        if (cf[q] < 0) continue;
        const double wab = DIM == 3 ? w0 * w[1][ta] * w[2][tb] : w[0][ta] * w[1][tb];
        s = fma(wab, ev[q], s);
      }
  }
  y[f] = accumulate ? __dadd_rn(z[f], s) : s;
}

// contribution of coarse block b (patch k) to (P^T r)
template <int DIM, int WT>
__device__ __forceinline__ double restrict_block(const KronArgs& a, long long b, const double* __restrict__ r,
                                                 double s) {
  const int k = patch_of(a.off_c, a.npatch, b);
  const KronPatch& P = a.patch[k];
  int loc = (int)(b - a.off_c[k]);
  int cc[3] = {0, 0, 0};
#pragma unroll
  for (int d = DIM - 1; d >= 0; --d) {
    const int n = P.nc[d];
    cc[d] = (int)(loc % n);
    loc /= n;
  }
  const long long of = a.off_f[k];
  const int nf1 = P.nf[1], nf2 = DIM == 3 ? P.nf[2] : 1;
  int c[DIM][WT];
  double w[DIM][WT];
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    const long long r0 = P.ellT[d] + (long long)cc[d] * WT;
#pragma unroll
    for (int t = 0; t < WT; ++t) {
      c[d][t] = __ldg(a.tidx + r0 + t);
      w[d][t] = __ldg(a.tval + r0 + t);
    }
  }
  const int n0 = DIM == 3 ? WT : 1;
  for (int t0 = 0; t0 < n0; ++t0) {
    int c0 = c[0][0];
    double w0 = w[0][0];
#pragma unroll
    for (int q = 1; q < WT; ++q)  // select without dynamic register-array indexing
      if (q == t0) {
        c0 = c[0][q];
        w0 = w[0][q];
      }
    if (DIM == 3 && c0 < 0) break;
    int fi[WT * WT];
    double rv[WT * WT];
#pragma unroll
    for (int ta = 0; ta < WT; ++ta)
#pragma unroll
      for (int tb = 0; tb < WT; ++tb) {
        const int A = DIM == 3 ? c[1][ta] : c[0][ta], B = DIM == 3 ? c[2][tb] : c[1][tb];
        long long blk = DIM == 3 ? ((long long)c0 * nf1 + A) * nf2 + B : (long long)A * nf1 + B;
        fi[ta * WT + tb] = (A >= 0 && B >= 0) ? __ldg(a.fown + of + blk) : -1;
      }
#pragma unroll
    for (int q = 0; q < WT * WT; ++q) rv[q] = fi[q] >= 0 ? __ldg(r + fi[q]) : 0.0;
#pragma unroll
    for (int ta = 0; ta < WT; ++ta)
#pragma unroll
      for (int tb = 0; tb < WT; ++tb) {
        const int q = ta * WT + tb;
        if (fi[q] < 0) continue;
        const double wab = DIM == 3 ? w0 * w[1][ta] * w[2][tb] : w[0][ta] * w[1][tb];
        s = fma(wab, rv[q], s);
      }
  }
  return s;
}

// Restriction: thread per coarse block index b; the root copy of each free class sums its own
// block and then the class's other copies (shared interface DoFs; fixed order).
template <int DIM, int WT>
__global__ void __launch_bounds__(256) kron_restrict_kernel(const __grid_constant__ KronArgs a, const double* __restrict__ r, double* y) {
  pdl_begin();
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.nblk_c) return;
  const int j = __ldg(a.croot + b);
  if (j < 0) return;
  const int x0 = __ldg(a.xptr + j), x1 = __ldg(a.xptr + j + 1);
  double s = restrict_block<DIM, WT>(a, b, r, 0.0);
  for (int t = x0; t < x1; ++t) s = restrict_block<DIM, WT>(a, __ldg(a.xblk + t), r, s);
  y[j] = s;
}

#define KRON_PROLONG_W(X) X(2, 2) X(2, 3) X(2, 4) X(2, 6) X(3, 2) X(3, 3) X(3, 4) X(3, 6)
#define KRON_RESTRICT_W(X) X(2, 4) X(2, 5) X(2, 6) X(2, 8) X(2, 10) X(3, 4) X(3, 5) X(3, 6) X(3, 8) X(3, 10)

}  // namespace

int kron_width(int w) { return w <= 2 ? 2 : w <= 3 ? 3 : w <= 4 ? 4 : w <= 6 ? 6 : -1; }
int kron_width_t(int w) { return w <= 4 ? 4 : w <= 5 ? 5 : w <= 6 ? 6 : w <= 8 ? 8 : w <= 10 ? 10 : -1; }

void kron_set_carveout(int pct) {
#define SETP(D, W) cudaFuncSetAttribute(kron_prolong_kernel<D, W>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
#define SETR(D, W) cudaFuncSetAttribute(kron_restrict_kernel<D, W>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  KRON_PROLONG_W(SETP)
  KRON_RESTRICT_W(SETR)
#undef SETP
#undef SETR
  cudaGetLastError();
}

void launch_kron_prolong(cudaStream_t s, const KronArgs& a, const double* e, const double* z, double* y,
                         int accumulate) {
  const dim3 grid((unsigned)((a.nblk_f + 255) / 256)), block(256);
#define LP(D, W) \
  if (a.dim == D && a.width == W) { launch_k(kron_prolong_kernel<D, W>, grid, block, 0, s, a, e, z, y, accumulate); return; }
  KRON_PROLONG_W(LP)
#undef LP
}

void launch_kron_restrict(cudaStream_t s, const KronArgs& a, const double* r, double* y) {
  const dim3 grid((unsigned)((a.nblk_c + 255) / 256)), block(256);
#define LR(D, W) \
  if (a.dim == D && a.widthT == W) { launch_k(kron_restrict_kernel<D, W>, grid, block, 0, s, a, r, y); return; }
  KRON_RESTRICT_W(LR)
#undef LR
}

}  // namespace igb
