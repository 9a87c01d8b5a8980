// fd3.cu -- fused 3-factor fast diagonalisation on fp64 tensor cores (DMMA m8n8k4), sm_100a.
//
// Replaces the six np.tensordot contractions of ScmsInteriorSolver.solve (reference
// smoothers.py:283-294) for 3-D interiors with sides <= FD3_NMAX:
//     X = (T0 x T1 x T2) [ ((T0 x T1 x T2)^T R) ./ D ]
// in three launches over slabs (a slab = one 2-D slice of one interior, whole in shared memory):
//   stage 0, slab i0:  Y[i0]      = T1^T R[i0] T2          (R gathered through idx)
//   stage 1, slab i1:  W[:,i1,:]  = T0 ((T0^T Y[:,i1,:]) ./ D[:,i1,:])
//   stage 2, slab i0:  u[idx[i0]] (+)= alpha * T1 W[i0] T2^T
// Every stage is two chained slab GEMMs.  A warp owns WM x WN output tiles of 8 x 8 and issues
// mma.sync.m8n8k4.f64 with A / B fragments read straight from shared memory; the row pitch
// ld = n8 + 4 (n8 = side rounded up to 8) makes all four fragment patterns (A or B, plain or
// transposed) bank-conflict free: a half-warp touches 4 rows x 4 columns, and 4 * ld = 16 mod 32
// four-byte banks.  Padding rows / columns are zero, so K runs to the next multiple of 4.
#include "kernels.cuh"

namespace igb {
namespace {

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// C(M x N) = op(A)(M x K) op(B)(K x N), all operands in shared memory with pitch ld.
// AT: A is stored transposed (A(m,k) = As[k*ld + m]); BT: B(k,n) = Bs[n*ld + k].
// tm, tn: number of 8-row / 8-column tiles; ksteps: K / 4 (padding is zero).
// epi(row, col, v0, v1): called once per lane with its two adjacent outputs (col even).
template <int WM, int WN, bool AT, bool BT, class Epi>
__device__ __forceinline__ void slab_gemm(const double* __restrict__ As, const double* __restrict__ Bs, int ld,
                                          int tm, int tn, int ksteps, Epi epi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int wn_count = (tn + WN - 1) / WN;
  const int wm = warp / wn_count, wn = warp - wm * wn_count;
  const int tr0 = wm * WM, tc0 = wn * WN;
  if (tr0 >= tm) return;
  double c[WM][WN][2];
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < WN; ++j) c[i][j][0] = c[i][j][1] = 0.0;
  // out-of-range tiles of a partial warp tile read tile 0 (valid memory) and are discarded
  int ao[WM], bo[WN];
#pragma unroll
  for (int i = 0; i < WM; ++i) {
    const int r = (tr0 + i < tm ? tr0 + i : 0) * 8 + g;
    ao[i] = AT ? (t * ld + r) : (r * ld + t);
  }
#pragma unroll
  for (int j = 0; j < WN; ++j) {
    const int cc = (tc0 + j < tn ? tc0 + j : 0) * 8 + g;
    bo[j] = BT ? (cc * ld + t) : (t * ld + cc);
  }
  const int astep = AT ? 4 * ld : 4, bstep = BT ? 4 : 4 * ld;
#pragma unroll 2
  for (int ks = 0; ks < ksteps; ++ks) {
    double a[WM], b[WN];
#pragma unroll
    for (int i = 0; i < WM; ++i) a[i] = As[ao[i] + ks * astep];
#pragma unroll
    for (int j = 0; j < WN; ++j) b[j] = Bs[bo[j] + ks * bstep];
#pragma unroll
    for (int i = 0; i < WM; ++i)
#pragma unroll
      for (int j = 0; j < WN; ++j) dmma884(c[i][j][0], c[i][j][1], a[i], b[j]);
  }
#pragma unroll
  for (int i = 0; i < WM; ++i) {
    if (tr0 + i >= tm) break;
#pragma unroll
    for (int j = 0; j < WN; ++j) {
      if (tc0 + j >= tn) break;
      epi((tr0 + i) * 8 + g, (tc0 + j) * 8 + 2 * t, c[i][j][0], c[i][j][1]);
    }
  }
}

// zero-padded copy of an (nr x nc) matrix (element (r, c) at src(r, c)) into an n8r x ld buffer
template <class Src>
__device__ __forceinline__ void slab_fill(double* dst, int ld, int rows8, int nr, int nc, Src src) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int r = warp; r < rows8; r += nw)
    for (int c0 = lane; c0 < ld; c0 += 32) dst[r * ld + c0] = (r < nr && c0 < nc) ? src(r, c0) : 0.0;
}

template <int WM, int WN, int STAGE>
__global__ void __launch_bounds__(FD3_MAXWARPS * 32)
fd3_kernel(const Fd3Item* __restrict__ items, int nitems, int n8, const double* __restrict__ src,
           double* dst, double alpha, int accumulate) {
  pdl_begin();
  extern __shared__ __align__(16) double fd3_smem[];
  // which interior, which slab
  int it = 0;
  {
    int lo = 0, hi = nitems - 1;
    const int b = blockIdx.x;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if ((STAGE == 1 ? items[mid].slab1 : items[mid].slab0) <= b) lo = mid; else hi = mid - 1;
    }
    it = lo;
  }
  const Fd3Item I = items[it];
  const int s = blockIdx.x - (STAGE == 1 ? I.slab1 : I.slab0);
  const int n0 = I.n[0], n1 = I.n[1], n2 = I.n[2];
  const int ld = n8 + 4;
  double* S = fd3_smem;            // the slab, then the second product's left operand source
  double* X = S + n8 * ld;         // first product
  double* L = X + n8 * ld;         // left factor
  double* R = L + n8 * ld;         // right factor (stage 1: the slab of D)
  const long long n12 = (long long)n1 * n2;
  if (STAGE != 1) {
    // slab i0 = s: rows i1, columns i2
    const long long base = (long long)s * n12;
    const int tm = (n1 + 7) >> 3, tn = (n2 + 7) >> 3;
    if (STAGE == 0)
      slab_fill(S, ld, tm * 8, n1, n2, [&](int r, int c) { return __ldg(&src[__ldg(&I.idx[base + (long long)r * n2 + c])]); });
    else
      slab_fill(S, ld, tm * 8, n1, n2, [&](int r, int c) { return I.buf1[base + (long long)r * n2 + c]; });
    slab_fill(L, ld, tm * 8, n1, n1, [&](int r, int c) { return __ldg(&I.T[1][r * n1 + c]); });
    slab_fill(R, ld, tn * 8, n2, n2, [&](int r, int c) { return __ldg(&I.T[2][r * n2 + c]); });
    __syncthreads();
    const int k1 = (n1 + 3) >> 2, k2 = (n2 + 3) >> 2;
    auto keep = [&](int r, int c, double v0, double v1) {
      *reinterpret_cast<double2*>(&X[r * ld + c]) = make_double2(v0, v1);
    };
    if (STAGE == 0) {
      // X = T1^T S ; Y = X T2
      slab_gemm<WM, WN, true, false>(L, S, ld, tm, tn, k1, keep);
      __syncthreads();
      double* out = I.buf0 + base;
      slab_gemm<WM, WN, false, false>(X, R, ld, tm, tn, k2, [&](int r, int c, double v0, double v1) {
        if (r < n1) {
          if (c < n2) out[(long long)r * n2 + c] = v0;
          if (c + 1 < n2) out[(long long)r * n2 + c + 1] = v1;
        }
      });
    } else {
      // X = T1 S ; out = X T2^T -> scatter
      slab_gemm<WM, WN, false, false>(L, S, ld, tm, tn, k1, keep);
      __syncthreads();
      const int* idx = I.idx + base;
      slab_gemm<WM, WN, false, true>(X, R, ld, tm, tn, k2, [&](int r, int c, double v0, double v1) {
        if (r < n1) {
          if (c < n2) {
            double* d = dst + __ldg(&idx[(long long)r * n2 + c]);
            const double sv = __dmul_rn(alpha, v0);
            *d = accumulate ? __dadd_rn(*d, sv) : sv;
          }
          if (c + 1 < n2) {
            double* d = dst + __ldg(&idx[(long long)r * n2 + c + 1]);
            const double sv = __dmul_rn(alpha, v1);
            *d = accumulate ? __dadd_rn(*d, sv) : sv;
          }
        }
      });
    }
  } else {
    // slab i1 = s: rows i0 (stride n1 n2), columns i2
    const long long base = (long long)s * n2;
    const int tm = (n0 + 7) >> 3, tn = (n2 + 7) >> 3;
    slab_fill(S, ld, tm * 8, n0, n2, [&](int r, int c) { return I.buf0[base + (long long)r * n12 + c]; });
    slab_fill(L, ld, tm * 8, n0, n0, [&](int r, int c) { return __ldg(&I.T[0][r * n0 + c]); });
    slab_fill(R, ld, tm * 8, n0, n2, [&](int r, int c) { return __ldg(&I.D[base + (long long)r * n12 + c]); });
    __syncthreads();
    const int k0 = (n0 + 3) >> 2;
    // X = (T0^T S) ./ D   (padding stays zero: 0 / 0 is never formed)
    slab_gemm<WM, WN, true, false>(L, S, ld, tm, tn, k0, [&](int r, int c, double v0, double v1) {
      const double d0 = R[r * ld + c], d1 = R[r * ld + c + 1];
      const double q0 = (r < n0 && c < n2) ? __ddiv_rn(v0, d0) : 0.0;
      const double q1 = (r < n0 && c + 1 < n2) ? __ddiv_rn(v1, d1) : 0.0;
      *reinterpret_cast<double2*>(&X[r * ld + c]) = make_double2(q0, q1);
    });
    __syncthreads();
    double* out = I.buf1 + base;
    slab_gemm<WM, WN, false, false>(L, X, ld, tm, tn, k0, [&](int r, int c, double v0, double v1) {
      if (r < n0) {
        if (c < n2) out[(long long)r * n12 + c] = v0;
        if (c + 1 < n2) out[(long long)r * n12 + c + 1] = v1;
      }
    });
  }
}

template <int WM, int WN>
void launch_fd3_t(cudaStream_t s, const Fd3Plan& P, int stage, const double* r, double* u, double alpha,
                  int accumulate) {
  static bool attr = false;
  const size_t smem_max = 4ull * FD3_NMAX * (FD3_NMAX + 4) * sizeof(double);
  if (!attr) {
    cudaFuncSetAttribute(fd3_kernel<WM, WN, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
    cudaFuncSetAttribute(fd3_kernel<WM, WN, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
    cudaFuncSetAttribute(fd3_kernel<WM, WN, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
    attr = true;
  }
  const size_t smem = 4ull * P.n8 * (P.n8 + 4) * sizeof(double);
  const int t8 = P.n8 / 8;
  const int warps = ((t8 + WM - 1) / WM) * ((t8 + WN - 1) / WN);
  if (stage == 0)
    launch_k(fd3_kernel<WM, WN, 0>, dim3(P.slabs0), dim3(32 * warps), smem, s, P.d_items, P.nitems, P.n8, r,
             (double*)nullptr, alpha, accumulate);
  else if (stage == 1)
    launch_k(fd3_kernel<WM, WN, 1>, dim3(P.slabs1), dim3(32 * warps), smem, s, P.d_items, P.nitems, P.n8, r,
             (double*)nullptr, alpha, accumulate);
  else
    launch_k(fd3_kernel<WM, WN, 2>, dim3(P.slabs0), dim3(32 * warps), smem, s, P.d_items, P.nitems, P.n8, r, u,
             alpha, accumulate);
}

}  // namespace

// warp tile per side: 3 x 3 tiles (9 warps at n8 = 72), 2 x 2 below 5 tiles
int fd3_warp_tile(int n8) { return n8 / 8 >= 5 ? 3 : (n8 / 8 >= 2 ? 2 : 1); }

void launch_fd3(cudaStream_t s, const Fd3Plan& P, int stage, const double* r, double* u, double alpha,
                int accumulate) {
  switch (fd3_warp_tile(P.n8)) {
    case 3: launch_fd3_t<3, 3>(s, P, stage, r, u, alpha, accumulate); break;
    case 2: launch_fd3_t<2, 2>(s, P, stage, r, u, alpha, accumulate); break;
    default: launch_fd3_t<1, 1>(s, P, stage, r, u, alpha, accumulate); break;
  }
}

void fd3_set_carveout(int pct) {
  for (const void* f : {(const void*)fd3_kernel<3, 3, 0>, (const void*)fd3_kernel<3, 3, 1>, (const void*)fd3_kernel<3, 3, 2>,
                        (const void*)fd3_kernel<2, 2, 0>, (const void*)fd3_kernel<2, 2, 1>, (const void*)fd3_kernel<2, 2, 2>,
                        (const void*)fd3_kernel<1, 1, 0>, (const void*)fd3_kernel<1, 1, 1>, (const void*)fd3_kernel<1, 1, 2>})
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  cudaGetLastError();
}

}  // namespace igb
