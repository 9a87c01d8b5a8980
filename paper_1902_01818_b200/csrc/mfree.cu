// mfree.cu -- matrix-free finest-level operator for conforming multi-patch spaces on affine patches.
//
// The reference assembles such patches by Kronecker products (assembly.py:333-344: per patch
// K = sum_a det/s_a^2 (x)_i (K_i if i == a else M_i), 1-D mass / stiffness of the B-spline spaces)
// and reduces them to free DoFs, summing shared interface copies and dropping Dirichlet rows and
// columns.  y = A x is applied here by sum factorisation instead of reading A:
//
//   3-D:  U = M3 X, V = K3 X               (along axis 2; X = the block copy of x, 0 on Dirichlet)
//         W1 = M2 U, W2 = c1 K2 U + c2 M2 V  (along axis 1)
//         Y = c0 K1 W1 + M1 W2              (along axis 0)
//   2-D:  U = M2 X, V = K2 X;  Y = c0 K1 U + c1 M1 V
//   y_f = sum over the block copies of f of Y (root copy first, fixed order: deterministic)
//
// Every pass reads (2p+1) neighbours along one axis per output (L1/L2 hits) and streams whole
// arrays once: ~80 bytes per DoF against 12 bytes per nonzero of A (343 per 3-D row at p = 3).
// Measured and dropped: the passes along axes 2 and 1 fused per plane in shared memory plus the
// axis-0 pass fused with the copy sum (two launches instead of four): 5.5 vs 5.2 ms per cfg5 solve.
#include <algorithm>
#include <cstdlib>

#include "kernels.cuh"

namespace igb {
namespace {

__device__ __forceinline__ int mf_patch(const MfArgs& a, long long b) {
  int k = 0;
  while (k + 1 < a.npatch && a.off[k + 1] <= b) ++k;
  return k;
}

// band row of the 1-D matrix of (patch k, axis d): entries j - i + p for j in [i - p, i + p]
__device__ __forceinline__ const double* mf_row(const double* pool, const MfArgs& a, int k, int d, int i) {
  return pool + a.band[k][d] + (long long)i * (2 * a.p + 1);
}

// The tap loops are compiled for the degree (P = p, 2P + 1 taps, all loads issued before the sums;
// P = 0: any degree, runtime loop); positions inside a patch are 32-bit (unsigned division).
// pass along the last axis: U = M X, V = K X, X read through the block -> free map
template <int DIM, int P>
__global__ void __launch_bounds__(256) mf_last_kernel(const __grid_constant__ MfArgs a, const double* __restrict__ x,
                                                      double* U, double* V) {
  pdl_begin();
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.nblk) return;
  const int k = mf_patch(a, b);
  const unsigned n = (unsigned)a.n[k][DIM - 1];
  const int i = (int)((unsigned)(b - a.off[k]) % n);
  const long long base = b - i;  // first entry of this line
  const double* m = mf_row(a.Mb, a, k, DIM - 1, i);
  const double* kk = mf_row(a.Kb, a, k, DIM - 1, i);
  double u = 0.0, v = 0.0;
  if (P > 0) {
    int f[2 * P + 1];
    double xv[2 * P + 1], mw[2 * P + 1], kw[2 * P + 1];
#pragma unroll
    for (int t = 0; t <= 2 * P; ++t) {
      const int j = i + t - P;
      const bool in = j >= 0 && j < (int)n;
      f[t] = in ? __ldg(a.bfree + base + j) : -1;
      mw[t] = in ? __ldg(m + t) : 0.0;
      kw[t] = in ? __ldg(kk + t) : 0.0;
    }
#pragma unroll
    for (int t = 0; t <= 2 * P; ++t) xv[t] = f[t] >= 0 ? __ldg(x + f[t]) : 0.0;
#pragma unroll
    for (int t = 0; t <= 2 * P; ++t) {
      u = fma(mw[t], xv[t], u);
      v = fma(kw[t], xv[t], v);
    }
  } else {
    for (int t = -a.p; t <= a.p; ++t) {
      const int j = i + t;
      if (j < 0 || j >= (int)n) continue;
      const int f = __ldg(a.bfree + base + j);
      const double xv = f >= 0 ? __ldg(x + f) : 0.0;
      u = fma(__ldg(m + t + a.p), xv, u);
      v = fma(__ldg(kk + t + a.p), xv, v);
    }
  }
  U[b] = u;
  V[b] = v;
}

// 3-D middle pass along axis 1: W1 = M2 U, W2 = c1 K2 U + c2 M2 V
template <int P>
__global__ void __launch_bounds__(256) mf_mid_kernel(const __grid_constant__ MfArgs a, const double* __restrict__ U,
                                                     const double* __restrict__ V, double* W1, double* W2) {
  pdl_begin();
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.nblk) return;
  const int k = mf_patch(a, b);
  const int n1 = a.n[k][1], n2 = a.n[k][2];
  const unsigned loc = (unsigned)(b - a.off[k]);
  const int i = (int)((loc / (unsigned)n2) % (unsigned)n1);
  const long long base = b - (long long)i * n2;
  const double* m = mf_row(a.Mb, a, k, 1, i);
  const double* kk = mf_row(a.Kb, a, k, 1, i);
  double mu = 0.0, ku = 0.0, mv = 0.0;
  if (P > 0) {
    double uv[2 * P + 1], vv[2 * P + 1], mw[2 * P + 1], kw[2 * P + 1];
#pragma unroll
    for (int t = 0; t <= 2 * P; ++t) {
      const int j = i + t - P;
      const bool in = j >= 0 && j < n1;
      uv[t] = in ? __ldg(U + base + (long long)j * n2) : 0.0;
      vv[t] = in ? __ldg(V + base + (long long)j * n2) : 0.0;
      mw[t] = in ? __ldg(m + t) : 0.0;
      kw[t] = in ? __ldg(kk + t) : 0.0;
    }
#pragma unroll
    for (int t = 0; t <= 2 * P; ++t) {
      mu = fma(mw[t], uv[t], mu);
      ku = fma(kw[t], uv[t], ku);
      mv = fma(mw[t], vv[t], mv);
    }
  } else {
    for (int t = -a.p; t <= a.p; ++t) {
      const int j = i + t;
      if (j < 0 || j >= n1) continue;
      const double uv = __ldg(U + base + (long long)j * n2), vv = __ldg(V + base + (long long)j * n2);
      const double mw = __ldg(m + t + a.p), kw = __ldg(kk + t + a.p);
      mu = fma(mw, uv, mu);
      ku = fma(kw, uv, ku);
      mv = fma(mw, vv, mv);
    }
  }
  W1[b] = mu;
  W2[b] = fma(a.c[k][1], ku, a.c[k][2] * mv);
}

// pass along axis 0: Y = c0 K1 P + M1 Q (3-D: P = W1, Q = W2; 2-D: P = U, Q = c1 V)
template <int DIM, int PD>
__global__ void __launch_bounds__(256) mf_first_kernel(const __grid_constant__ MfArgs a, const double* __restrict__ P,
                                                       const double* __restrict__ Q, double* Y) {
  pdl_begin();
  const long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= a.nblk) return;
  const int k = mf_patch(a, b);
  const unsigned stride = DIM == 3 ? (unsigned)a.n[k][1] * (unsigned)a.n[k][2] : (unsigned)a.n[k][1];
  const int n0 = a.n[k][0];
  const unsigned loc = (unsigned)(b - a.off[k]);
  const int i = (int)(loc / stride);
  const long long base = b - (long long)i * stride;
  const double* m = mf_row(a.Mb, a, k, 0, i);
  const double* kk = mf_row(a.Kb, a, k, 0, i);
  double kp = 0.0, mq = 0.0;
  if (PD > 0) {
    double pv[2 * PD + 1], qv[2 * PD + 1], mw[2 * PD + 1], kw[2 * PD + 1];
#pragma unroll
    for (int t = 0; t <= 2 * PD; ++t) {
      const int j = i + t - PD;
      const bool in = j >= 0 && j < n0;
      pv[t] = in ? __ldg(P + base + (long long)j * stride) : 0.0;
      qv[t] = in ? __ldg(Q + base + (long long)j * stride) : 0.0;
      mw[t] = in ? __ldg(m + t) : 0.0;
      kw[t] = in ? __ldg(kk + t) : 0.0;
    }
#pragma unroll
    for (int t = 0; t <= 2 * PD; ++t) {
      kp = fma(kw[t], pv[t], kp);
      mq = fma(mw[t], qv[t], mq);
    }
  } else {
    for (int t = -a.p; t <= a.p; ++t) {
      const int j = i + t;
      if (j < 0 || j >= n0) continue;
      kp = fma(__ldg(kk + t + a.p), __ldg(P + base + (long long)j * stride), kp);
      mq = fma(__ldg(m + t + a.p), __ldg(Q + base + (long long)j * stride), mq);
    }
  }
  const double cq = DIM == 3 ? 1.0 : a.c[k][1];
  Y[b] = fma(a.c[k][0], kp, cq * mq);
}

// y = z + sign * A x over free DoFs: sum of the block copies (root first, then the others)
__global__ void __launch_bounds__(256) mf_sum_kernel(const __grid_constant__ MfArgs a, const double* __restrict__ Yb,
                                                     const double* z, double* y, int sign) {
  pdl_begin();
  const int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= a.nfree) return;
  double s = __ldg(Yb + __ldg(a.froot + f));
  const int t1 = __ldg(a.xptr + f + 1);
  for (int t = __ldg(a.xptr + f); t < t1; ++t) s += __ldg(Yb + __ldg(a.xblk + t));
  if (sign == 0) y[f] = s;
  else if (sign < 0) y[f] = z ? __dsub_rn(z[f], s) : -s;
  else y[f] = __dadd_rn(z[f], s);
}

}  // namespace

template <int P>
void mf_carveout_p(int pct) {
  const void* fns[] = {(const void*)mf_last_kernel<2, P>, (const void*)mf_last_kernel<3, P>, (const void*)mf_mid_kernel<P>,
                       (const void*)mf_first_kernel<2, P>, (const void*)mf_first_kernel<3, P>};
  for (const void* f : fns) cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

void mf_set_carveout(int pct) {
  mf_carveout_p<0>(pct);
  mf_carveout_p<2>(pct);
  mf_carveout_p<3>(pct);
  mf_carveout_p<4>(pct);
  cudaFuncSetAttribute((const void*)mf_sum_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  cudaGetLastError();
}

template <int P>
static void mf_apply_p(cudaStream_t s, const MfArgs& a, const double* x, const double* z, double* y, int sign,
                       double* const scratch[4]) {
  const dim3 gb((unsigned)((a.nblk + 255) / 256)), gf((unsigned)((a.nfree + 255) / 256)), blk(256);
  double *U = scratch[0], *V = scratch[1], *W1 = scratch[2], *W2 = scratch[3];
  if (a.dim == 3) {
    launch_k(mf_last_kernel<3, P>, gb, blk, 0, s, a, x, U, V);
    launch_k(mf_mid_kernel<P>, gb, blk, 0, s, a, (const double*)U, (const double*)V, W1, W2);
    launch_k(mf_first_kernel<3, P>, gb, blk, 0, s, a, (const double*)W1, (const double*)W2, U);
  } else {
    launch_k(mf_last_kernel<2, P>, gb, blk, 0, s, a, x, U, V);
    launch_k(mf_first_kernel<2, P>, gb, blk, 0, s, a, (const double*)U, (const double*)V, W1);
    U = W1;
  }
  launch_k(mf_sum_kernel, gf, blk, 0, s, a, (const double*)U, z, y, sign);
}

void launch_mf_apply(cudaStream_t s, const MfArgs& a, const double* x, const double* z, double* y, int sign,
                     double* const scratch[4]) {
  switch (a.p) {   // the sums run over the same taps in the same order for every variant
    case 2: mf_apply_p<2>(s, a, x, z, y, sign, scratch); break;
    case 3: mf_apply_p<3>(s, a, x, z, y, sign, scratch); break;
    case 4: mf_apply_p<4>(s, a, x, z, y, sign, scratch); break;
    default: mf_apply_p<0>(s, a, x, z, y, sign, scratch); break;
  }
}

}  // namespace igb
