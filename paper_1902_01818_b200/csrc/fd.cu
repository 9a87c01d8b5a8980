// fd.cu -- fused 2-D fast diagonalisation on a thread-block cluster (sm_100a).
//
// SCMS interior solve (smoothers.py:272-301, square-transform form of
// ScmsInteriorSolver): X = T0 ((T0^T R T1) ./ D) T1^T with R = r[idx], and
// u[idx] (+)= alpha X.  One cluster of G CTAs per interior; CTA c owns the rows
// [c rb, c rb + rb) (rb <= FDC_RB) of every intermediate, thread j owns column j:
//
//   1  B  = T0^T R          left T0[:, rows]^T   right R (gathered from r)
//   2  A  = (B T1) ./ D     left B (own rows)    right T1          -> A rows to scratch
//      cluster barrier (A complete in L2)
//   3  B' = T0 A            left T0[rows, :]     right A (scratch)
//   4  X  = B' T1^T         left B' (own rows)   right T1^T        -> u[idx] (+)= alpha X
//
// Left operands live in shared memory as [m][i] (a 10-double row per m: one
// broadcast load feeds 10 FMAs of the thread's column); right operands stream
// through a double-buffered [FDC_KC][FDC_NMAX] shared chunk, loaded into
// registers one chunk ahead.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace igb {

namespace {

constexpr int FDC_RB = 10;     // rows per CTA
constexpr int FDC_KC = 16;     // right-operand rows per chunk
constexpr size_t FDC_SMEM = 8 * (2 * FDC_NMAX * FDC_RB + 2 * FDC_KC * FDC_NMAX);

template <class Load>
__device__ __forceinline__ void fdc_gemm(double (&acc)[FDC_RB], const double (*L)[FDC_RB], int K, int j, bool active,
                                         double (*rch)[FDC_KC][FDC_NMAX], Load ld) {
#pragma unroll
  for (int i = 0; i < FDC_RB; ++i) acc[i] = 0.0;
  double pre[FDC_KC];
#pragma unroll
  for (int k = 0; k < FDC_KC; ++k) pre[k] = ld(min(k, K - 1));  // clamped rows are never consumed
  const int nch = (K + FDC_KC - 1) / FDC_KC;
  for (int q = 0; q < nch; ++q) {
    double (*buf)[FDC_NMAX] = rch[q & 1];
#pragma unroll
    for (int k = 0; k < FDC_KC; ++k) buf[k][j] = pre[k];
    __syncthreads();
    if (q + 1 < nch) {
      const int m0 = (q + 1) * FDC_KC;
#pragma unroll
      for (int k = 0; k < FDC_KC; ++k) pre[k] = ld(min(m0 + k, K - 1));
    }
    const int m0 = q * FDC_KC;
    const int kn = min(FDC_KC, K - m0);
    if (kn == FDC_KC) {
#pragma unroll 8
      for (int k = 0; k < FDC_KC; ++k) {
        const double x = buf[k][j];
        const double* l = L[m0 + k];
#pragma unroll
        for (int i = 0; i < FDC_RB; ++i) acc[i] = fma(l[i], x, acc[i]);
      }
    } else {
      for (int k = 0; k < kn; ++k) {
        const double x = buf[k][j];
        const double* l = L[m0 + k];
#pragma unroll
        for (int i = 0; i < FDC_RB; ++i) acc[i] = fma(l[i], x, acc[i]);
      }
    }
  }
}

__global__ void __launch_bounds__(FDC_NT, 1) fd_cluster_kernel(const FdCluster* __restrict__ items, const double* r,
                                                            double* u, double alpha, int accumulate) {
  extern __shared__ __align__(16) double fdc_smem[];
  double (*lop)[FDC_RB] = reinterpret_cast<double (*)[FDC_RB]>(fdc_smem);
  double (*outT)[FDC_RB] = lop + FDC_NMAX;
  double (*rch)[FDC_KC][FDC_NMAX] = reinterpret_cast<double (*)[FDC_KC][FDC_NMAX]>(fdc_smem + 2 * FDC_NMAX * FDC_RB);
  const cg::cluster_group cluster = cg::this_cluster();
  const int G = (int)cluster.num_blocks(), c = (int)cluster.block_rank();
  const FdCluster it = items[blockIdx.x / G];
  const int n0 = it.n0, n1 = it.n1;
  const int rb = (n0 + G - 1) / G, r0 = c * rb, nr = max(0, min(rb, n0 - r0));
  const int j = threadIdx.x;
  const bool active = j < n1;
  const int jj = active ? j : n1 - 1;  // idle columns load a valid dummy (never stored)
  double acc[FDC_RB];

  // left-operand fill: all of a thread's loads are issued before any store (one round trip)
  constexpr int FILL = (FDC_NMAX * FDC_RB + FDC_NT - 1) / FDC_NT;
  auto fill = [&](bool rows) {
    double v[FILL];
#pragma unroll
    for (int q = 0; q < FILL; ++q) {
      const int e = j + q * FDC_NT, m = e / FDC_RB, i = e - m * FDC_RB;
      const int mm = min(m, n0 - 1), ii = min(i, max(nr - 1, 0));
      v[q] = __ldg(it.T0 + (rows ? (size_t)(r0 + ii) * n0 + mm : (size_t)mm * n0 + r0 + ii));
    }
#pragma unroll
    for (int q = 0; q < FILL; ++q) {
      const int e = j + q * FDC_NT, m = e / FDC_RB, i = e - m * FDC_RB;
      if (m < n0) lop[m][i] = i < nr ? v[q] : 0.0;
    }
  };
  // 1: B = T0^T R      lop[m][i] = T0[m][r0 + i]
  fill(false);
  __syncthreads();
  fdc_gemm(acc, lop, n0, j, active, rch, [&](int m) { return r[__ldg(it.idx + (size_t)m * n1 + jj)]; });
#pragma unroll
  for (int i = 0; i < FDC_RB; ++i) outT[j][i] = acc[i];
  __syncthreads();
  // 2: A = (B T1) ./ D   left outT[m][i] = B[i][m]
  fdc_gemm(acc, outT, n1, j, active, rch, [&](int m) { return __ldg(it.T1 + (size_t)m * n1 + jj); });
  if (active) {
#pragma unroll
    for (int i = 0; i < FDC_RB; ++i)
      if (i < nr) {
        const size_t o = (size_t)(r0 + i) * n1 + j;
        __stcg(it.scratch + o, __ddiv_rn(acc[i], __ldg(it.D + o)));
      }
  }
  cluster.sync();  // every row of A written (release/acquire at cluster scope)
  // 3: B' = T0 A        lop[m][i] = T0[r0 + i][m]
  fill(true);
  int gi[FDC_RB];  // epilogue targets, fetched two products ahead (idx -> u chain off the critical path)
#pragma unroll
  for (int i = 0; i < FDC_RB; ++i) gi[i] = __ldg(it.idx + (size_t)(r0 + min(i, max(nr - 1, 0))) * n1 + jj);
  __syncthreads();
  fdc_gemm(acc, lop, n0, j, active, rch, [&](int m) { return __ldcg(it.scratch + (size_t)m * n1 + jj); });
  __syncthreads();
#pragma unroll
  for (int i = 0; i < FDC_RB; ++i) outT[j][i] = acc[i];
  __syncthreads();
  // 4: X = B' T1^T      right T1[j][m]
  fdc_gemm(acc, outT, n1, j, active, rch, [&](int m) { return __ldg(it.T1 + (size_t)jj * n1 + m); });
  if (active) {
#pragma unroll
    for (int i = 0; i < FDC_RB; ++i)
      if (i < nr) {
        const double v = __dmul_rn(alpha, acc[i]);
        u[gi[i]] = accumulate ? __dadd_rn(u[gi[i]], v) : v;
      }
  }
}

}  // namespace

int fd_cluster_size(int n0max) { return (n0max + FDC_RB - 1) / FDC_RB; }

void set_carveout_panel(int pct);  // panel.cu

void set_carveout_panel_fd(int pct) {
  cudaFuncSetAttribute(fd_cluster_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  cudaGetLastError();
  set_carveout_panel(pct);
}

void launch_fd_cluster(cudaStream_t s, const FdCluster* d_items, int nitems, int G, const double* r, double* u,
                       double alpha, int accumulate) {
  if (nitems <= 0) return;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fd_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(fd_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FDC_SMEM);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nitems * G, 1, 1);
  cfg.blockDim = dim3(FDC_NT, 1, 1);
  cfg.dynamicSmemBytes = FDC_SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attrs[1];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = G;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  cfg.attrs = attrs;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, fd_cluster_kernel, d_items, r, u, alpha, accumulate);
}

}  // namespace igb
