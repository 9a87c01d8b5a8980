// flow.cu -- dependency-driven triangular sweep over the whole GPU (Gauss-Seidel in the
// reference's natural order for levels whose rows are long and whose dependency levels are
// wide: 3-D patches, high-degree 2-D).
//
// Replaces SuperLU dgstrs on tril(A) / triu(A) as called by GaussSeidel.apply_forward /
// apply_backward (reference smoothers.py:171-200; factor built at :178-184 with natural
// permutations, so the solve is a plain substitution in row order).
//
// Design (no barrier of any kind inside the sweep):
//  * rows are listed in dependency-level order (level = 1 + max level of the rows they read),
//    padded so that the RPW = 32 / G rows a warp takes at once never straddle a level;
//  * the grid is persistent and fully co-resident; warp w takes list groups w, w + W, ...,
//    so every warp walks its rows in increasing level order;
//  * each solution value is published in a global copy xg[par][row] that reads as a
//    signalling-NaN sentinel until produced; a row's lanes load their dependencies from it
//    (ld.relaxed.gpu: the L2 coherence point) and re-poll the sentinel ones.  A value and its
//    "ready" flag are one 8-byte word, so no fence is needed.
// Progress: the lowest unfinished list entry has all its dependencies at lower levels (done),
// and its warp has finished every earlier entry it owns, so it is running -- with all CTAs
// resident no warp can wait forever.  Every poll has a clock64 watchdog that reports and
// traps instead of hanging the device.
// The two halves of xg alternate between sweeps of the same level and direction (device-side
// parity flipped by the last CTA to finish): the producer writes the value into the current
// half and the sentinel into the other, which is the next sweep's current half.
#include <cstdio>

#include "kernels.cuh"

namespace igb {
namespace {

constexpr int FLOW_MINB = 2;  // resident CTAs per SM the register budget is sized for (3: spills, measured 1.5x slower)
constexpr unsigned long long FLOW_PENDING = 0x7FF4DEADBEEF5678ULL;

__device__ __forceinline__ double ld_relaxed(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ double ld_nc_f64(const double* p) {
  double v;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_nc_s32(const int* p) {
  int v;
  asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double ld_f64_volatile(const double* p) {
  double v;
  asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ bool is_pending(double v) {
  return (unsigned long long)__double_as_longlong(v) == FLOW_PENDING;
}
__device__ __noinline__ void flow_stuck(int col, int row) {
  printf("[igb flow] block %d thread %d: value of row %d (needed by row %d) never produced\n", (int)blockIdx.x,
         (int)threadIdx.x, col, row);
  __trap();
}
// G lanes per row, K entries per lane held in registers per chunk (longer rows loop).
// The next row's list metadata is fetched while the current row waits for its dependencies,
// and the right-hand side / inverse diagonal loads are pinned at the top of the row (volatile
// asm: the compiler may not sink them to their use after the poll loop).
template <int G, int K>
__global__ void __launch_bounds__(FLOW_NT, FLOW_MINB) flow_sweep_kernel(FlowArgs a) {
  pdl_begin();
  constexpr int RPW = 32 / G;
  const int lane = threadIdx.x & 31, sub = lane / G, gl = lane % G;
  const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const int par = *(volatile const int*)a.par_ctr;  // stable for the whole launch
  const double* xg_cur = a.xg + (size_t)par * a.n;
  double* xg_set = a.xg + (size_t)par * a.n;
  double* xg_clr = a.xg + (size_t)(par ^ 1) * a.n;
  const long long stride = nwarps * RPW;

  long long q0 = gwarp * RPW;
  int nrow = -1, ns = 0, ne = 0, ncc = -1, nel = -1;
  if (q0 < a.nq) {
    nrow = ld_nc_s32(a.row + q0 + sub);
    ns = ld_nc_s32(a.eptr + q0 + sub);
    ne = ld_nc_s32(a.eptr + q0 + sub + 1);
    if (a.crit) ncc = ld_nc_s32(a.crit + q0 + sub);
    if (a.elate) nel = ld_nc_s32(a.elate + q0 + sub);
  }
  for (; q0 < a.nq; q0 += stride) {
    const long long q = q0 + sub;
    const int row = nrow, s = ns, e = ne, cc = ncc;
    const int el = (a.elate && row >= 0) ? nel : e;  // early entries [s, el)
    long long c0 = 0, t0 = 0;
    if (a.trace && gl == 0) {
      t0 = gtime();
      c0 = clock64();
    }
    // first probe of the critical dependency: its L2 round trip runs under the loads issued below
    double cv = 0.0;
    const bool crit_wait = a.crit && gl == 0 && row >= 0 && cc >= 0;
    if (crit_wait) cv = ld_relaxed(xg_cur + cc);
    double rhs = 0.0, uold = 0.0, idg = 0.0;
    if (gl == 0 && row >= 0) {
      rhs = ld_nc_f64(a.res + row);
      idg = ld_nc_f64(a.idiag + q);
      if (a.accumulate) uold = ld_f64_volatile(a.u + row);
    }
    if (q0 + stride < a.nq) {  // next row's metadata
      nrow = ld_nc_s32(a.row + q + stride);
      ns = ld_nc_s32(a.eptr + q + stride);
      ne = ld_nc_s32(a.eptr + q + stride + 1);
      if (a.crit) ncc = ld_nc_s32(a.crit + q + stride);
      if (a.elate) nel = ld_nc_s32(a.elate + q + stride);
      // ... and its entries, right-hand side and old value into L2: a row is a chain of memory round
      // trips (entries -> values -> late entries -> late values), and on wide levels (cfg5's finest:
      // 733 rows per level for 2,368 warps) the sweep is bound by the time a warp spends per row;
      // with the coefficient stream already in L2 two of those trips cost 0.3 us instead of ~1.2
      if (a.prefetch) {
        const char* pc = reinterpret_cast<const char*>(a.ecol + ns);
        const char* pv = reinterpret_cast<const char*>(a.eval + ns);
        const int bc = (ne - ns) * 4;
        for (int o = gl * 128; o < bc; o += G * 128) prefetch_l2(pc + o);
        for (int o = gl * 128; o < 2 * bc; o += G * 128) prefetch_l2(pv + o);
        if (gl == 0 && nrow >= 0) {
          prefetch_l2(a.res + nrow);
          if (a.accumulate) prefetch_l2(a.u + nrow);
        }
      }
    }
    // first chunk of the row's coefficients: in flight while the critical dependency is awaited
    int c[K];
    double v[K], x[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int idx = s + gl + k * G;
      c[k] = idx < el ? __ldcs(a.ecol + idx) : -1;
      v[k] = idx < el ? __ldcs(a.eval + idx) : 0.0;
    }
    if (crit_wait) {  // wait for the latest dependency first (one poller per row)
      if (is_pending(cv)) {
        const long long w0 = clock64();
        while (is_pending(ld_relaxed(xg_cur + cc))) {
          if (a.backoff) __nanosleep(a.backoff);
          if (clock64() - w0 > (1LL << 31)) flow_stuck(cc, row);
        }
      }
    }
    if (a.crit) __syncwarp();
    long long cc0 = 0;
    if (a.trace && gl == 0) cc0 = clock64();
    double acc = 0.0;
    for (int base = s; base < el; base += G * K) {
      if (base > s) {
#pragma unroll
        for (int k = 0; k < K; ++k) {
          const int idx = base + gl + k * G;
          c[k] = idx < el ? __ldcs(a.ecol + idx) : -1;
          v[k] = idx < el ? __ldcs(a.eval + idx) : 0.0;
        }
      }
#pragma unroll
      for (int k = 0; k < K; ++k) x[k] = c[k] >= 0 ? ld_relaxed(xg_cur + c[k]) : 0.0;
      // re-poll every still-pending value of this lane together: one L2 round trip per
      // attempt, not one per pending entry once the last dependency has landed
      unsigned pend = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) pend |= (c[k] >= 0 && is_pending(x[k])) ? 1u << k : 0u;
      if (pend) {
        const long long w0 = clock64();
        do {
#pragma unroll
          for (int k = 0; k < K; ++k)
            if (pend >> k & 1u) x[k] = ld_relaxed(xg_cur + c[k]);
#pragma unroll
          for (int k = 0; k < K; ++k)
            if ((pend >> k & 1u) && !is_pending(x[k])) pend &= ~(1u << k);
          if (pend && clock64() - w0 > (1LL << 31)) {
            int bad = -1;
#pragma unroll
            for (int k = 0; k < K; ++k)
              if (pend >> k & 1u) bad = c[k];
            flow_stuck(bad, row);
          }
        } while (pend);
      }
#pragma unroll
      for (int k = 0; k < K; ++k) acc = fma(v[k], x[k], acc);
    }
    long long c1 = 0;
    if (a.trace && gl == 0) c1 = clock64();
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, G);
    // late entries (the newest dependencies): every lane of the row loads and polls all of them
    // (same addresses: one request per warp) and adds them serially in a fixed order, so the
    // early reduction above never waits for them
    if (row >= 0 && el < e) {
      constexpr int LM = 8;
      int lc[LM];
      double lv[LM], lx[LM];
      const int nl = e - el;
      for (int j0 = 0; j0 < nl; j0 += LM) {
#pragma unroll
        for (int j = 0; j < LM; ++j) {
          const int idx = el + j0 + j;
          lc[j] = j0 + j < nl ? ld_nc_s32(a.ecol + idx) : -1;
          lv[j] = j0 + j < nl ? ld_nc_f64(a.eval + idx) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < LM; ++j) lx[j] = lc[j] >= 0 ? ld_relaxed(xg_cur + lc[j]) : 0.0;
        unsigned pend = 0;
#pragma unroll
        for (int j = 0; j < LM; ++j) pend |= (lc[j] >= 0 && is_pending(lx[j])) ? 1u << j : 0u;
        if (pend) {
          const long long w0 = clock64();
          do {
#pragma unroll
            for (int j = 0; j < LM; ++j)
              if (pend >> j & 1u) lx[j] = ld_relaxed(xg_cur + lc[j]);
#pragma unroll
            for (int j = 0; j < LM; ++j)
              if ((pend >> j & 1u) && !is_pending(lx[j])) pend &= ~(1u << j);
            if (pend && clock64() - w0 > (1LL << 31)) {
              int bad = -1;
#pragma unroll
              for (int j = 0; j < LM; ++j)
                if (pend >> j & 1u) bad = lc[j];
              flow_stuck(bad, row);
            }
          } while (pend);
        }
#pragma unroll
        for (int j = 0; j < LM; ++j) acc = fma(lv[j], lx[j], acc);
      }
    }
    if (gl == 0 && row >= 0) {
      const double xv = (rhs - acc) * idg;
      st_relaxed(xg_set + row, xv);
      xg_clr[row] = __longlong_as_double((long long)FLOW_PENDING);
      a.u[row] = a.accumulate ? uold + xv : xv;
      if (a.trace) {  // [start time, crit seen - start, ready - crit seen, stored - ready (cycles), stored time]
        const long long c2 = clock64();
        a.trace[5 * q] = t0;
        a.trace[5 * q + 1] = cc0 - c0;
        a.trace[5 * q + 2] = c1 - cc0;
        a.trace[5 * q + 3] = c2 - c1;
        a.trace[5 * q + 4] = gtime();
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // the last CTA flips the parity for the next sweep
    __threadfence();
    if (atomicAdd(a.done_ctr, 1u) == gridDim.x - 1) {
      *a.done_ctr = 0u;
      *(volatile int*)a.par_ctr = par ^ 1;
      __threadfence();
    }
  }
}

template <int G, int K>
const void* flow_fn() {
  return (const void*)flow_sweep_kernel<G, K>;
}
const void* flow_kernel_for(int G) {
  switch (G) {
    case 8: return flow_fn<8, 4>();
    case 16: return flow_fn<16, 4>();
    default: return flow_fn<32, 6>();
  }
}

}  // namespace

int flow_max_ctas() {
  static int cap = -1;
  if (cap < 0) {
    int dev = 0, sms = 0, per = 0, best = 1 << 30;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    for (int G : {8, 16, 32}) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, flow_kernel_for(G), FLOW_NT, 0);
      best = per < best ? per : best;
    }
    cudaGetLastError();
    cap = best * sms;
    if (cap < 1) cap = 1;
  }
  return cap;
}

void flow_set_carveout(int pct) {
  for (int G : {8, 16, 32})
    cudaFuncSetAttribute(flow_kernel_for(G), cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  cudaGetLastError();
}

void launch_flow_sweep(cudaStream_t s, const FlowArgs& a) {
  const dim3 grid(a.ctas), block(FLOW_NT);
  switch (a.G) {
    case 8: launch_k(flow_sweep_kernel<8, 4>, grid, block, 0, s, a); break;
    case 16: launch_k(flow_sweep_kernel<16, 4>, grid, block, 0, s, a); break;
    default: launch_k(flow_sweep_kernel<32, 6>, grid, block, 0, s, a); break;
  }
}

}  // namespace igb
