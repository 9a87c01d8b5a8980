// line.cu -- line sweep: Gauss-Seidel in the reference's natural order along grid lines
// (plan and rationale: line_plan.h).
//
// Replaces SuperLU dgstrs on tril(A) / triu(A) as called by GaussSeidel.apply_forward /
// apply_backward (reference smoothers.py:171-200; natural permutations, so a plain substitution).
//
//  * persistent grid, one bundle (a run of lines, e.g. a plane of a 3-D patch) per CTA at a time,
//    bundles dealt round-robin (CTA c: bundles c, c + G, ...), lines dealt to warps round-robin;
//  * a warp walks its line row by row: all lanes gather the row's entries (32 per chunk), a
//    butterfly reduction leaves the same sum in every lane, and every lane finishes the row with
//    the three newest same-line values it keeps in registers -- the line's own dependency chain
//    never leaves the warp;
//  * a value is published in the bundle's shared-memory array (read by the CTA's other warps) and
//    in the global copy xg[par][position] (read by other bundles); both read as a signalling-NaN
//    sentinel until produced (value and ready flag in one 8-byte word, no fences); readers re-poll;
//  * the next row's entries are loaded into registers while the current row waits, and an L2 bulk
//    prefetch runs LINE_PF rows ahead.
// Progress: the lowest unfinished position has all dependencies done; its bundle's CTA has finished
// every lower bundle it owns (they hold lower positions) and its line's warp every lower line of
// the bundle, so it is running.  Every poll has a clock64 watchdog (report + trap, no hang).
// The halves of xg alternate between sweeps of the same level and direction (device-side parity,
// flipped by the last CTA), as in flow.cu.
#include <cstdio>

#include "kernels.cuh"

namespace igb {
namespace {

constexpr unsigned long long LINE_PENDING = 0x7FF4DEADBEEF9ABCULL;
constexpr int LINE_PF = 6;  // rows of L2 bulk prefetch ahead

__device__ __forceinline__ bool pend(double v) { return (unsigned long long)__double_as_longlong(v) == LINE_PENDING; }
__device__ __forceinline__ double ld_relaxed(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ double lds_vol(const double* p) { return *(const volatile double*)p; }
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __noinline__ void line_stuck(int code, int p) {
  printf("[igb line] block %d thread %d: value %s %d (needed by position %d) never produced\n", (int)blockIdx.x,
         (int)threadIdx.x, code < 0 ? "in shared slot" : "at position", code < 0 ? -1 - code : code, p);
  __trap();
}

template <int C>
struct RowData {
  int cc[C];
  double cv[C];
  int nch;
};

template <int C>
__device__ __forceinline__ void load_row(const LineArgs& a, int p, int lane, RowData<C>& r) {
  const int c0 = __ldg(a.cptr + p), c1 = __ldg(a.cptr + p + 1);
  r.nch = c1 - c0;
  const size_t base = (size_t)c0 * 32 + lane;
#pragma unroll
  for (int k = 0; k < C; ++k) {
    r.cc[k] = k < r.nch ? __ldg(a.ccol + base + 32 * k) : -1 - a.rb_max;
    r.cv[k] = k < r.nch ? __ldg(a.cval + base + 32 * k) : 0.0;
  }
}

template <int C>
__global__ void __launch_bounds__(LINE_NT, 1) line_sweep_kernel(LineArgs a) {
  pdl_begin();
  extern __shared__ __align__(16) double xs[];  // [rb_max + 1]; slot rb_max always 0
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int par = *(volatile const int*)a.par_ctr;
  const double* xg_cur = a.xg + (size_t)par * a.n;
  double* xg_set = a.xg + (size_t)par * a.n;
  double* xg_clr = a.xg + (size_t)(par ^ 1) * a.n;
  if (threadIdx.x == 0) xs[a.rb_max] = 0.0;
  for (int b = blockIdx.x; b < a.nb; b += gridDim.x) {
    const int bs = a.bstart[b], be = a.bstart[b + 1];
    for (int i = threadIdx.x; i < be - bs; i += blockDim.x) xs[i] = __longlong_as_double((long long)LINE_PENDING);
    __syncthreads();
    for (int l = a.bline[b] + warp; l < a.bline[b + 1]; l += W) {
      const int p0 = a.lstart[l], p1 = a.lstart[l + 1];
      double x1 = 0.0, x2 = 0.0, x3 = 0.0;
      RowData<C> cur, nxt;
      load_row<C>(a, p0, lane, cur);
      for (int p = p0; p < p1; ++p) {
        const int row = a.upper ? a.n - 1 - p : p;
        double rhs = 0.0, idg = 0.0, o1 = 0.0, o2 = 0.0, o3 = 0.0, uold = 0.0;
        rhs = __ldg(a.res + row);
        idg = __ldg(a.idiag + p);
        o1 = __ldg(a.own + 3 * (size_t)p);
        o2 = __ldg(a.own + 3 * (size_t)p + 1);
        o3 = __ldg(a.own + 3 * (size_t)p + 2);
        if (a.accumulate && lane == 0) uold = a.u[row];
        if (p + 1 < p1) load_row<C>(a, p + 1, lane, nxt);
        if (lane == 0 && p + LINE_PF < p1) {
          const int cpf = __ldg(a.cptr + p + LINE_PF), cpe = __ldg(a.cptr + p + LINE_PF + 1);
          if (cpe > cpf) {
            prefetch_l2(a.cval + (size_t)cpf * 32, (unsigned)(cpe - cpf) * 256u);
            prefetch_l2(a.ccol + (size_t)cpf * 32, (unsigned)(cpe - cpf) * 128u);
          }
        }
        // gather the row's values (shared: the bundle; global: other bundles); re-poll pending ones
        double xv[C];
#pragma unroll
        for (int k = 0; k < C; ++k) xv[k] = cur.cc[k] < 0 ? lds_vol(xs + (-1 - cur.cc[k])) : ld_relaxed(xg_cur + cur.cc[k]);
        unsigned pm = 0;
#pragma unroll
        for (int k = 0; k < C; ++k) pm |= pend(xv[k]) ? 1u << k : 0u;
        if (pm) {
          const long long w0 = clock64();
          do {
#pragma unroll
            for (int k = 0; k < C; ++k)
              if (pm >> k & 1u) {
                xv[k] = cur.cc[k] < 0 ? lds_vol(xs + (-1 - cur.cc[k])) : ld_relaxed(xg_cur + cur.cc[k]);
                if (!pend(xv[k])) pm &= ~(1u << k);
              }
            if (pm && clock64() - w0 > (1LL << 31)) {
              int bad = 0;
#pragma unroll
              for (int k = 0; k < C; ++k)
                if (pm >> k & 1u) bad = cur.cc[k];
              line_stuck(bad, p);
            }
          } while (pm);
        }
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < C; ++k) acc = fma(cur.cv[k], xv[k], acc);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);  // same sum in every lane
        double s = rhs - acc;
        s = fma(-o3, x3, s);
        s = fma(-o2, x2, s);
        s = fma(-o1, x1, s);
        const double x = s * idg;
        if (lane == 0) {
          *(volatile double*)(xs + (p - bs)) = x;
          st_relaxed(xg_set + p, x);
          xg_clr[p] = __longlong_as_double((long long)LINE_PENDING);
          a.u[row] = a.accumulate ? uold + x : x;
        }
        x3 = x2;
        x2 = x1;
        x1 = x;
        cur = nxt;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {  // the last CTA flips the parity for the next sweep
    __threadfence();
    if (atomicAdd(a.done_ctr, 1u) == gridDim.x - 1) {
      *a.done_ctr = 0u;
      *(volatile int*)a.par_ctr = par ^ 1;
      __threadfence();
    }
  }
}

template <class F>
void for_line_variants(F&& f) {
  f(line_sweep_kernel<2>);
  f(line_sweep_kernel<4>);
  f(line_sweep_kernel<6>);
  f(line_sweep_kernel<8>);
}

}  // namespace

int line_chunk_variant(int C) { return C <= 2 ? 2 : C <= 4 ? 4 : C <= 6 ? 6 : C <= 8 ? 8 : -1; }

int line_max_ctas(size_t smem) {
  int dev = 0, sms = 0, per = 0, best = 1 << 30;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for_line_variants([&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, LINE_NT, smem);
    best = per < best ? per : best;
  });
  cudaGetLastError();
  return best < 1 ? 0 : best * sms;
}

void launch_line_sweep(cudaStream_t s, const LineArgs& a) {
  const dim3 grid(a.ctas), block(LINE_NT);
  const size_t smem = 8 * ((size_t)a.rb_max + 1);
  switch (line_chunk_variant(a.C)) {
    case 2: launch_k(line_sweep_kernel<2>, grid, block, smem, s, a); break;
    case 4: launch_k(line_sweep_kernel<4>, grid, block, smem, s, a); break;
    case 6: launch_k(line_sweep_kernel<6>, grid, block, smem, s, a); break;
    default: launch_k(line_sweep_kernel<8>, grid, block, smem, s, a); break;
  }
}

}  // namespace igb
