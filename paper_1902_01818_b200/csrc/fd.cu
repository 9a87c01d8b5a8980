// fd.cu -- fused 2-D fast diagonalisation (sm_100a).
//
// SCMS interior solve (smoothers.py:272-301, square-transform form of
// ScmsInteriorSolver): X = T0 ((T0^T R T1) ./ D) T1^T with R = r[idx], and
// u[idx] (+)= alpha X.  Two launches per SCMS application, split where rows of the
// middle intermediate are exchanged:
//
//   fd_front   1  B  = T0^T R          left T0[:, rows]^T   right R (gathered from r)
//              2  A  = (B T1) ./ D     left B (own rows)    right T1      -> rows of A to scratch
//   fd_back    3  B' = T0 A            left T0[rows, :]     right A (scratch, L2)
//              4  X  = B' T1^T         left B' (own rows)   right T1^T    -> u[idx] (+)= alpha X
//
// Every CTA owns RB rows of one interior (all interiors of a level in one grid, ~1 CTA
// per SM) and thread j owns column j.  Left operands live in shared memory as [m][i] (RB
// doubles per m: broadcast loads feeding RB FMAs of the thread's column); each product's
// right operand is copied whole into shared memory by cp.async (one latency per product).
#include <cuda_runtime.h>

#include <cstdlib>

#include "kernels.cuh"

namespace igb {

namespace {

constexpr int FDC_KC = 16;  // gathered-operand rows per chunk

// NM = largest interior side of the variant, NT = threads (one column each, NT >= NM).
// WHOLE: products 2-4 copy their right operand whole into shared memory (NM = 160); else every
// product streams it in chunks (NM = 264: a 264^2 operand does not fit).
template <int RB, int NM, bool WHOLE>
size_t fd_smem(int kmax) {
  const size_t rs = WHOLE ? (size_t)(kmax > 2 * FDC_KC ? kmax : 2 * FDC_KC) * NM : (size_t)2 * FDC_KC * NM;
  return 8 * (2 * (size_t)NM * RB + rs);
}

// Gathered right operand (R = r[idx], step 1): 16-row chunks, each thread loading its column
// of the next chunk into registers while the current one is multiplied (plain loads; 8-byte
// cp.async copies of a gather measured slower).  rch: two [FDC_KC][FDC_NMAX] chunks.
template <int RB, int NM, class Load>
__device__ __forceinline__ void fdc_gemm_chunked(double (&acc)[RB], const double (*L)[RB], int K, int j,
                                                 double* rch_base, Load ld) {
  double (*rch)[FDC_KC][NM] = reinterpret_cast<double (*)[FDC_KC][NM]>(rch_base);
#pragma unroll
  for (int i = 0; i < RB; ++i) acc[i] = 0.0;
  double pre[FDC_KC];
#pragma unroll
  for (int k = 0; k < FDC_KC; ++k) pre[k] = ld(min(k, K - 1));  // clamped rows are never consumed
  const int nch = (K + FDC_KC - 1) / FDC_KC;
  for (int q = 0; q < nch; ++q) {
    double (*buf)[NM] = rch[q & 1];
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
    for (int k = 0; k < kn; ++k) {
      const double x = buf[k][j];
      const double* l = L[m0 + k];
#pragma unroll
      for (int i = 0; i < RB; ++i) acc[i] = fma(l[i], x, acc[i]);
    }
  }
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}

// acc[i] = sum_m L[m][i] * Rt(m, j) for m < K.  The whole right operand is copied into the
// shared buffer Rs ([m][FDC_NMAX]) at once -- every thread issues cp.async for its column of
// all K rows (8-byte copies, so gathered operands work too) -- one memory latency per product,
// then the multiply runs from shared memory.  The caller synchronises before Rs is reused.
template <int RB, int NM, class Addr>
__device__ __forceinline__ void fdc_gemm(double (&acc)[RB], const double (*L)[RB], int K, int j, bool active,
                                         double* Rs, Addr addr) {
  if (active) {
#pragma unroll 4
    for (int m = 0; m < K; ++m) cp_async8(Rs + m * NM + j, addr(m));
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncthreads();
#pragma unroll
  for (int i = 0; i < RB; ++i) acc[i] = 0.0;
  const double* x = Rs + j;
#pragma unroll 8
  for (int m = 0; m < K; ++m) {
    const double xm = x[m * NM];
    const double* l = L[m];
#pragma unroll
    for (int i = 0; i < RB; ++i) acc[i] = fma(l[i], xm, acc[i]);
  }
}

struct FdCtx {
  FdCluster it;
  int r0, nr, n0, n1, j, jj;
  bool active;
};

__device__ __forceinline__ FdCtx fd_locate(const FdBatch& bt) {
  FdCtx c;
  int item = 0;
#pragma unroll 1
  for (int i = 1; i < bt.nitems; ++i)
    if ((int)blockIdx.x >= bt.cta0[i]) item = i;
  c.it = bt.items[item];
  c.n0 = c.it.n0;
  c.n1 = c.it.n1;
  c.r0 = ((int)blockIdx.x - bt.cta0[item]) * bt.rb;
  c.nr = max(0, min(bt.rb, c.n0 - c.r0));
  c.j = threadIdx.x;
  c.active = c.j < c.n1;
  c.jj = c.active ? c.j : c.n1 - 1;  // idle columns load a valid dummy (never stored)
  return c;
}

// left-operand fill: lop[m][i] = T0[m][r0+i] (cols) or T0[r0+i][m] (rows); every load of a
// thread is issued before its stores (one round trip)
template <int RB, int NM, int NT>
__device__ __forceinline__ void fd_fill(double (*lop)[RB], const FdCtx& c, bool rows) {
  constexpr int FILL = (NM * RB + NT - 1) / NT;
  double v[FILL];
#pragma unroll
  for (int q = 0; q < FILL; ++q) {
    const int e = c.j + q * NT, m = e / RB, i = e - m * RB;
    const int mm = min(m, c.n0 - 1), ii = min(i, max(c.nr - 1, 0));
    v[q] = __ldg(c.it.T0 + (rows ? (size_t)(c.r0 + ii) * c.n0 + mm : (size_t)mm * c.n0 + c.r0 + ii));
  }
#pragma unroll
  for (int q = 0; q < FILL; ++q) {
    const int e = c.j + q * NT, m = e / RB, i = e - m * RB;
    if (m < c.n0) lop[m][i] = i < c.nr ? v[q] : 0.0;
  }
}

template <int RB, int NM, int NT, bool WHOLE>
__global__ void __launch_bounds__(NT, 2) fd_front_kernel(const __grid_constant__ FdBatch bt, const double* r) {
  pdl_begin();
  extern __shared__ __align__(16) double fdc_smem[];
  double (*lop)[RB] = reinterpret_cast<double (*)[RB]>(fdc_smem);
  double (*outT)[RB] = lop + NM;
  double* Rs = fdc_smem + 2 * NM * RB;  // right operand (whole [kmax][NM], or two chunks)
  const FdCtx c = fd_locate(bt);
  const int n1 = c.n1, jj = c.jj;
  double acc[RB];
  // 1: B = T0^T R
  fd_fill<RB, NM, NT>(lop, c, false);
  __syncthreads();
  if (c.j == 0)  // step 2's operand: into L2 while step 1 runs
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(c.it.T1), "r"((unsigned)(8 * n1 * n1) & ~15u)
                 : "memory");
  fdc_gemm_chunked<RB, NM>(acc, lop, c.n0, c.j, Rs, [&](int m) { return r[__ldg(c.it.idx + (size_t)m * n1 + jj)]; });
  if (c.j < NM) {
#pragma unroll
    for (int i = 0; i < RB; ++i) outT[c.j][i] = acc[i];
  }
  __syncthreads();
  // 2: A = (B T1) ./ D    left outT[m][i] = B[i][m]
  if (WHOLE)
    fdc_gemm<RB, NM>(acc, outT, n1, c.j, c.active, Rs, [&](int m) { return c.it.T1 + (size_t)m * n1 + jj; });
  else
    fdc_gemm_chunked<RB, NM>(acc, outT, n1, c.j, Rs, [&](int m) { return __ldg(c.it.T1 + (size_t)m * n1 + jj); });
  if (c.active) {
#pragma unroll
    for (int i = 0; i < RB; ++i)
      if (i < c.nr) {
        const size_t o = (size_t)(c.r0 + i) * n1 + c.j;
        c.it.scratch[o] = __ddiv_rn(acc[i], __ldg(c.it.D + o));
      }
  }
}

// interface pieces (linsolve.py:33-53 on the pieces of smoothers.py:316-319): u[idx] (+)=
// alpha inv r[idx], warp per row -- the same work as piece_gemv_kernel, in the back launch
__device__ void fd_piece_rows(const PieceRowBlock& b, const double* r, double* u, double alpha, int accumulate) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp >= b.nrows) return;
  const int i = b.row0 + warp;
  const double* row = b.inv + (long long)i * b.m;
  double s = 0.0;
  for (int j = lane; j < b.m; j += 32) s = fma(__ldg(&row[j]), __ldg(&r[__ldg(&b.idx[j])]), s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    const int gi = __ldg(&b.idx[i]);
    const double v = __dmul_rn(alpha, s);
    u[gi] = accumulate ? __dadd_rn(u[gi], v) : v;
  }
}

template <int RB, int NM, int NT, bool WHOLE>
__global__ void __launch_bounds__(NT, 2) fd_back_kernel(const __grid_constant__ FdBatch bt, const double* r,
                                                        double* u, double alpha, int accumulate) {
  pdl_begin();
  if ((int)blockIdx.x >= bt.cta0[bt.nitems]) {
    fd_piece_rows(bt.pieces[blockIdx.x - bt.cta0[bt.nitems]], r, u, alpha, accumulate);
    return;
  }
  extern __shared__ __align__(16) double fdc_smem[];
  double (*lop)[RB] = reinterpret_cast<double (*)[RB]>(fdc_smem);
  double (*outT)[RB] = lop + NM;
  double* Rs = fdc_smem + 2 * NM * RB;
  const FdCtx c = fd_locate(bt);
  const int n1 = c.n1, jj = c.jj;
  double acc[RB];
  // 3: B' = T0 A
  fd_fill<RB, NM, NT>(lop, c, true);
  int gi[RB];  // epilogue targets, fetched two products ahead
#pragma unroll
  for (int i = 0; i < RB; ++i) gi[i] = __ldg(c.it.idx + (size_t)(c.r0 + min(i, max(c.nr - 1, 0))) * n1 + jj);
  __syncthreads();
  if (WHOLE)
    fdc_gemm<RB, NM>(acc, lop, c.n0, c.j, c.active, Rs, [&](int m) { return c.it.scratch + (size_t)m * n1 + jj; });
  else
    fdc_gemm_chunked<RB, NM>(acc, lop, c.n0, c.j, Rs, [&](int m) { return c.it.scratch[(size_t)m * n1 + jj]; });
  if (c.j < NM) {
#pragma unroll
    for (int i = 0; i < RB; ++i) outT[c.j][i] = acc[i];
  }
  __syncthreads();
  // 4: X = B' T1^T       right T1[j][m]
  if (WHOLE)
    fdc_gemm<RB, NM>(acc, outT, n1, c.j, c.active, Rs, [&](int m) { return c.it.T1 + (size_t)jj * n1 + m; });
  else
    fdc_gemm_chunked<RB, NM>(acc, outT, n1, c.j, Rs, [&](int m) { return __ldg(c.it.T1 + (size_t)jj * n1 + m); });
  if (c.active) {
#pragma unroll
    for (int i = 0; i < RB; ++i)
      if (i < c.nr) {
        const double v = __dmul_rn(alpha, acc[i]);
        u[gi[i]] = accumulate ? __dadd_rn(u[gi[i]], v) : v;
      }
  }
}

template <int RB, int NM, int NT, bool WHOLE>
void launch_rb(cudaStream_t s, const FdBatch& bt, const double* r, double* u, double alpha, int accumulate) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fd_front_kernel<RB, NM, NT, WHOLE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)fd_smem<RB, NM, WHOLE>(NM));
    cudaFuncSetAttribute(fd_back_kernel<RB, NM, NT, WHOLE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)fd_smem<RB, NM, WHOLE>(NM));
    attr = true;
  }
  const int grid = bt.cta0[bt.nitems];
  const size_t smem = fd_smem<RB, NM, WHOLE>(bt.kmax);
  launch_k(fd_front_kernel<RB, NM, NT, WHOLE>, dim3(grid), dim3(NT), smem, s, bt, r);
  launch_k(fd_back_kernel<RB, NM, NT, WHOLE>, dim3(grid + bt.npieces), dim3(NT), smem, s, bt, r, u, alpha,
           accumulate);
}

}  // namespace

int fd_rows_per_cta(int total_rows) {
  static const int forced = std::getenv("IGB_FD_RB") ? std::atoi(std::getenv("IGB_FD_RB")) : 0;
  if (forced == 2 || forced == 4 || forced == 8) return forced;
  // about one CTA per SM for the level's interiors together (the right operand fills shared memory)
  const int want = (total_rows + 147) / 148;
  return want <= 2 ? 2 : (want <= 4 ? 4 : 8);
}

void launch_fd_batch(cudaStream_t s, const FdBatch& bt, const double* r, double* u, double alpha, int accumulate) {
  if (bt.nitems <= 0) return;
  if (bt.large) {
    switch (bt.rb) {
      case 2: launch_rb<2, FDL_NMAX, FDL_NT, false>(s, bt, r, u, alpha, accumulate); break;
      case 4: launch_rb<4, FDL_NMAX, FDL_NT, false>(s, bt, r, u, alpha, accumulate); break;
      default: launch_rb<8, FDL_NMAX, FDL_NT, false>(s, bt, r, u, alpha, accumulate); break;
    }
    return;
  }
  switch (bt.rb) {
    case 2: launch_rb<2, FDC_NMAX, FDC_NT, true>(s, bt, r, u, alpha, accumulate); break;
    case 4: launch_rb<4, FDC_NMAX, FDC_NT, true>(s, bt, r, u, alpha, accumulate); break;
    default: launch_rb<8, FDC_NMAX, FDC_NT, true>(s, bt, r, u, alpha, accumulate); break;
  }
}

void set_carveout_panel(int pct);  // panel.cu

void set_carveout_panel_fd(int pct) {
  for (const void* f :
       {(const void*)fd_front_kernel<2, FDC_NMAX, FDC_NT, true>, (const void*)fd_back_kernel<2, FDC_NMAX, FDC_NT, true>,
        (const void*)fd_front_kernel<4, FDC_NMAX, FDC_NT, true>, (const void*)fd_back_kernel<4, FDC_NMAX, FDC_NT, true>,
        (const void*)fd_front_kernel<8, FDC_NMAX, FDC_NT, true>, (const void*)fd_back_kernel<8, FDC_NMAX, FDC_NT, true>,
        (const void*)fd_front_kernel<2, FDL_NMAX, FDL_NT, false>, (const void*)fd_back_kernel<2, FDL_NMAX, FDL_NT, false>,
        (const void*)fd_front_kernel<4, FDL_NMAX, FDL_NT, false>, (const void*)fd_back_kernel<4, FDL_NMAX, FDL_NT, false>,
        (const void*)fd_front_kernel<8, FDL_NMAX, FDL_NT, false>, (const void*)fd_back_kernel<8, FDL_NMAX, FDL_NT, false>})
    cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  cudaGetLastError();
  set_carveout_panel(pct);
}

}  // namespace igb
