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

__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// Warp tile of a slab product: which tiles this warp owns.
template <int WM, int WN>
struct WarpTile {
  int tr0, tc0, g, t;
  bool active;
  __device__ __forceinline__ WarpTile(int tm, int tn) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    g = lane >> 2;
    t = lane & 3;
    const int wn_count = (tn + WN - 1) / WN;
    const int wm = warp / wn_count;
    tr0 = wm * WM;
    tc0 = (warp - wm * wn_count) * WN;
    active = tr0 < tm;
  }
};

// c(M x N) += op(A)(M x K) op(B)(K x N), operands in shared memory with pitch ld.
// AT: A is stored transposed (A(m,k) = As[k*ld + m]); BT: B(k,n) = Bs[n*ld + k].
// tm, tn: number of 8-row / 8-column tiles; ksteps: K / 4 (padding is zero).  Lane (g, t) ends
// up with outputs (row 8 i + g, columns 8 j + 2 t, + 1) of tile (i, j) in c[i][j][0..1].
template <int WM, int WN, bool AT, bool BT>
__device__ __forceinline__ void slab_gemm(const WarpTile<WM, WN>& w, const double* __restrict__ As,
                                          const double* __restrict__ Bs, int ld, int tm, int tn, int ksteps,
                                          double (&c)[WM][WN][2]) {
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < WN; ++j) c[i][j][0] = c[i][j][1] = 0.0;
  if (!w.active) return;
  // out-of-range tiles of a partial warp tile read tile 0 (valid memory) and are discarded
  int ao[WM], bo[WN];
#pragma unroll
  for (int i = 0; i < WM; ++i) {
    const int r = (w.tr0 + i < tm ? w.tr0 + i : 0) * 8 + w.g;
    ao[i] = AT ? (w.t * ld + r) : (r * ld + w.t);
  }
#pragma unroll
  for (int j = 0; j < WN; ++j) {
    const int cc = (w.tc0 + j < tn ? w.tc0 + j : 0) * 8 + w.g;
    bo[j] = BT ? (cc * ld + w.t) : (w.t * ld + cc);
  }
  const int astep = AT ? 4 * ld : 4, bstep = BT ? 4 : 4 * ld;
#pragma unroll 4
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
}

// every owned output pair: f(i, j, row, col) with col even
template <int WM, int WN, class F>
__device__ __forceinline__ void for_tiles(const WarpTile<WM, WN>& w, int tm, int tn, F f) {
  if (!w.active) return;
#pragma unroll
  for (int i = 0; i < WM; ++i) {
    if (w.tr0 + i >= tm) break;
#pragma unroll
    for (int j = 0; j < WN; ++j) {
      if (w.tc0 + j >= tn) break;
      f(i, j, (w.tr0 + i) * 8 + w.g, (w.tc0 + j) * 8 + 2 * w.t);
    }
  }
}

// zero-padded asynchronous copy of an (nr x nc) matrix with row stride rs into a rows8 x ld
// buffer; all copies of the CTA are in flight together (cp.async), padding is stored directly
__device__ __forceinline__ void slab_fill(double* dst, int ld, int rows8, int nr, int nc, const double* src,
                                          long long rs) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int r = warp; r < rows8; r += nw)
    for (int c0 = lane; c0 < ld; c0 += 32) {
      if (r < nr && c0 < nc) cp_async8(&dst[r * ld + c0], src + r * rs + c0);
      else dst[r * ld + c0] = 0.0;
    }
}
// the same through an index list: element (r, c) = src[idx[r * nc + c]]; index loads batched
// four rows deep so their latency is paid once per batch, not once per row
__device__ __forceinline__ void slab_fill_gather(double* dst, int ld, int rows8, int nr, int nc,
                                                 const double* __restrict__ src, const int* __restrict__ idx) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  constexpr int RB = 4, CB = 3;   // ld <= 96
  for (int r0 = warp; r0 < rows8; r0 += RB * nw) {
    int id[RB][CB];
#pragma unroll
    for (int a = 0; a < RB; ++a)
#pragma unroll
      for (int b = 0; b < CB; ++b) {
        const int r = r0 + a * nw, c0 = lane + 32 * b;
        id[a][b] = (r < nr && c0 < nc) ? __ldg(&idx[(long long)r * nc + c0]) : -1;
      }
#pragma unroll
    for (int a = 0; a < RB; ++a)
#pragma unroll
      for (int b = 0; b < CB; ++b) {
        const int r = r0 + a * nw, c0 = lane + 32 * b;
        if (r < rows8 && c0 < ld) {
          if (id[a][b] >= 0) cp_async8(&dst[r * ld + c0], src + id[a][b]);
          else dst[r * ld + c0] = 0.0;
        }
      }
  }
}

// lr_shared: T1 and T2 are the same matrix for every interior (equal spaces along the slab's two
// axes), so one copy serves as left and right factor and stage 1 reads D from global memory: two
// buffers instead of three, two CTAs per SM at n8 = 72.
template <int WM, int WN, int STAGE>
__global__ void __launch_bounds__(FD3_MAXWARPS * 32, 2)
fd3_kernel(const Fd3Item* __restrict__ items, int nitems, int n8, int lr_shared, const double* __restrict__ src,
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
  double* S = fd3_smem;            // the slab; overwritten by the first product
  double* L = S + n8 * ld;         // left factor
  double* R = lr_shared ? L : L + n8 * ld;   // right factor (stage 1, three buffers: the slab of D)
  const long long n12 = (long long)n1 * n2;
  double c[WM][WN][2];
  if (STAGE != 1) {
    // slab i0 = s: rows i1, columns i2
    const long long base = (long long)s * n12;
    const int tm = (n1 + 7) >> 3, tn = (n2 + 7) >> 3;
    const WarpTile<WM, WN> w(tm, tn);
    if (STAGE == 0) slab_fill_gather(S, ld, tm * 8, n1, n2, src, I.idx + base);
    else slab_fill(S, ld, tm * 8, n1, n2, I.buf1 + base, n2);
    slab_fill(L, ld, tm * 8, n1, n1, I.T[1], n1);
    if (!lr_shared) slab_fill(R, ld, tn * 8, n2, n2, I.T[2], n2);
    cp_async_wait_all();
    __syncthreads();
    const int k1 = (n1 + 3) >> 2, k2 = (n2 + 3) >> 2;
    // first product (T1^T S or T1 S), in place: every warp holds its outputs until all have read S
    if (STAGE == 0) slab_gemm<WM, WN, true, false>(w, L, S, ld, tm, tn, k1, c);
    else slab_gemm<WM, WN, false, false>(w, L, S, ld, tm, tn, k1, c);
    __syncthreads();
    for_tiles(w, tm, tn, [&](int i, int j, int r, int cc) {
      *reinterpret_cast<double2*>(&S[r * ld + cc]) = make_double2(c[i][j][0], c[i][j][1]);
    });
    __syncthreads();
    if (STAGE == 0) {
      // Y = S T2
      slab_gemm<WM, WN, false, false>(w, S, R, ld, tm, tn, k2, c);
      double* out = I.buf0 + base;
      for_tiles(w, tm, tn, [&](int i, int j, int r, int cc) {
        if (r < n1) {
          if (cc < n2) out[(long long)r * n2 + cc] = c[i][j][0];
          if (cc + 1 < n2) out[(long long)r * n2 + cc + 1] = c[i][j][1];
        }
      });
    } else {
      // out = S T2^T -> u[idx] (+)= alpha out; targets and old values are fetched in batches
      const int* idx = I.idx + base;
      int id[WM][WN][2];
      for_tiles(w, tm, tn, [&](int i, int j, int r, int cc) {
        id[i][j][0] = (r < n1 && cc < n2) ? __ldg(&idx[(long long)r * n2 + cc]) : -1;
        id[i][j][1] = (r < n1 && cc + 1 < n2) ? __ldg(&idx[(long long)r * n2 + cc + 1]) : -1;
      });
      slab_gemm<WM, WN, false, true>(w, S, R, ld, tm, tn, k2, c);
      // old values and stores one tile row at a time (register budget of two CTAs per SM)
      if (w.active) {
#pragma unroll
        for (int i = 0; i < WM; ++i) {
          if (w.tr0 + i >= tm) break;
          double old[WN][2];
#pragma unroll
          for (int j = 0; j < WN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              old[j][h] = (accumulate && w.tc0 + j < tn && id[i][j][h] >= 0) ? dst[id[i][j][h]] : 0.0;
#pragma unroll
          for (int j = 0; j < WN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              if (w.tc0 + j < tn && id[i][j][h] >= 0)
                dst[id[i][j][h]] = __dadd_rn(old[j][h], __dmul_rn(alpha, c[i][j][h]));
        }
      }
    }
  } else {
    // slab i1 = s: rows i0 (stride n1 n2), columns i2
    const long long base = (long long)s * n2;
    const int tm = (n0 + 7) >> 3, tn = (n2 + 7) >> 3;
    const WarpTile<WM, WN> w(tm, tn);
    slab_fill(S, ld, tm * 8, n0, n2, I.buf0 + base, n12);
    slab_fill(L, ld, tm * 8, n0, n0, I.T[0], n0);
    if (!lr_shared) slab_fill(R, ld, tm * 8, n0, n2, I.D + base, n12);
    cp_async_wait_all();
    __syncthreads();
    const int k0 = (n0 + 3) >> 2;
    // S = (T0^T S) ./ D   (padding stays zero: 0 / 0 is never formed)
    slab_gemm<WM, WN, true, false>(w, L, S, ld, tm, tn, k0, c);
    __syncthreads();
    if (w.active) {
      const double* Dg = I.D + base;
#pragma unroll
      for (int i = 0; i < WM; ++i) {
        if (w.tr0 + i >= tm) break;
        const int r = (w.tr0 + i) * 8 + w.g;
        double dv[WN][2];
#pragma unroll
        for (int j = 0; j < WN; ++j) {
          const int cc = (w.tc0 + j) * 8 + 2 * w.t;
          const bool in0 = w.tc0 + j < tn && r < n0 && cc < n2, in1 = w.tc0 + j < tn && r < n0 && cc + 1 < n2;
          if (lr_shared) {  // denominators straight from global memory (L2)
            dv[j][0] = in0 ? __ldg(&Dg[(long long)r * n12 + cc]) : 1.0;
            dv[j][1] = in1 ? __ldg(&Dg[(long long)r * n12 + cc + 1]) : 1.0;
          } else if (w.tc0 + j < tn) {
            const double2 d = *reinterpret_cast<const double2*>(&R[r * ld + cc]);
            dv[j][0] = in0 ? d.x : 1.0;
            dv[j][1] = in1 ? d.y : 1.0;
          }
        }
#pragma unroll
        for (int j = 0; j < WN; ++j) {
          if (w.tc0 + j >= tn) break;
          const int cc = (w.tc0 + j) * 8 + 2 * w.t;
          const double q0 = (r < n0 && cc < n2) ? __ddiv_rn(c[i][j][0], dv[j][0]) : 0.0;
          const double q1 = (r < n0 && cc + 1 < n2) ? __ddiv_rn(c[i][j][1], dv[j][1]) : 0.0;
          *reinterpret_cast<double2*>(&S[r * ld + cc]) = make_double2(q0, q1);
        }
      }
    }
    __syncthreads();
    slab_gemm<WM, WN, false, false>(w, L, S, ld, tm, tn, k0, c);
    double* out = I.buf1 + base;
    for_tiles(w, tm, tn, [&](int i, int j, int r, int cc) {
      if (r < n0) {
        if (cc < n2) out[(long long)r * n12 + cc] = c[i][j][0];
        if (cc + 1 < n2) out[(long long)r * n12 + cc + 1] = c[i][j][1];
      }
    });
  }
}

template <int WM, int WN>
void launch_fd3_t(cudaStream_t s, const Fd3Plan& P, int stage, const double* r, double* u, double alpha,
                  int accumulate) {
  static bool attr = false;
  const size_t smem_max = 3ull * FD3_NMAX * (FD3_NMAX + 4) * sizeof(double);
  if (!attr) {
    cudaFuncSetAttribute(fd3_kernel<WM, WN, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
    cudaFuncSetAttribute(fd3_kernel<WM, WN, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
    cudaFuncSetAttribute(fd3_kernel<WM, WN, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
    attr = true;
  }
  const size_t smem = (P.lr_shared ? 2ull : 3ull) * P.n8 * (P.n8 + 4) * sizeof(double);
  const int t8 = P.n8 / 8;
  const int warps = ((t8 + WM - 1) / WM) * ((t8 + WN - 1) / WN);
  if (stage == 0)
    launch_k(fd3_kernel<WM, WN, 0>, dim3(P.slabs0), dim3(32 * warps), smem, s, P.d_items, P.nitems, P.n8, P.lr_shared, r,
             (double*)nullptr, alpha, accumulate);
  else if (stage == 1)
    launch_k(fd3_kernel<WM, WN, 1>, dim3(P.slabs1), dim3(32 * warps), smem, s, P.d_items, P.nitems, P.n8, P.lr_shared, r,
             (double*)nullptr, alpha, accumulate);
  else
    launch_k(fd3_kernel<WM, WN, 2>, dim3(P.slabs0), dim3(32 * warps), smem, s, P.d_items, P.nitems, P.n8, P.lr_shared, r, u,
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
