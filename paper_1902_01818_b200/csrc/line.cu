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
#include "line_plan.h"

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

__device__ __forceinline__ double fetch(const double* xs, const double* xg, int code) {
  return code < 0 ? lds_vol(xs + (-1 - code)) : ld_relaxed(xg + code);
}

__device__ __forceinline__ void prefetch_line_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Per-warp row pipeline (iteration t works on four rows at once):
//   A  row t+3: load its early entry codes; bulk-prefetch the record of the row a.pf rows further
//               along this warp's row sequence into L2;
//   B  row t+2: issue the gathers of its early values (shared / global), load their coefficients;
//   C  row t+1: re-poll early values still pending (together), FMA, butterfly reduction -> acc in
//               every lane; issue the gathers of its late values, load its scalars;
//   D  row t:   re-poll its late values (together), finish
//               s = rhs - acc - sum late (oldest first) - own(3, 2, 1), publish x.
// Only D waits on the newest values, so the gathers and the reduction run ahead of the
// critical path; every per-row array the pipeline reads is in the row's record (one contiguous
// block, prefetched as one bulk copy) or in res / u (prefetched by line).
template <int C>
struct StA {
  int p, row;
  int cc[C];
};
template <int C>
struct StB {
  int p, row;
  int cc[C];
  double cv[C], xv[C];
};
struct StD {
  int p, row;
  long long cw;  // trace: cycles re-polling early values
  double acc;
  int lc[LINE_LATE];
  double lv[LINE_LATE], lx[LINE_LATE];
  double rhs, idg, o1, o2, o3, uold;
};

// This warp's row sequence within a bundle: lines l0, l0 + W, ...; positions in order.
struct RowIter {
  int l, p, end;
  __device__ __forceinline__ void init(const LineArgs& a, int l0, int lend) {
    l = l0;
    p = end = -1;
    if (l < lend) {
      p = a.lstart[l];
      end = a.lstart[l + 1];
    }
  }
  __device__ __forceinline__ int next(const LineArgs& a, int W, int lend) {  // current (-1: done), advance
    const int cur = p;
    if (cur < 0) return -1;
    if (++p == end) {
      l += W;
      if (l < lend) {
        p = a.lstart[l];
        end = a.lstart[l + 1];
      } else {
        p = -1;
      }
    }
    return cur;
  }
};

template <int C>
__global__ void __launch_bounds__(LINE_NT, 1) line_sweep_kernel(LineArgs a) {
  pdl_begin();
  extern __shared__ __align__(16) double xs[];  // [rb_max + 1]; slot rb_max always 0
  constexpr int RB = line_rec_bytes(C);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int par = *(volatile const int*)a.par_ctr;
  const double* xg_cur = a.xg + (size_t)par * a.n;
  double* xg_set = a.xg + (size_t)par * a.n;
  double* xg_clr = a.xg + (size_t)(par ^ 1) * a.n;
  const int zero_code = -1 - a.rb_max;
  if (threadIdx.x == 0) xs[a.rb_max] = 0.0;
  auto rec = [&](int p) { return a.rec + (size_t)p * RB; };
  for (int b = blockIdx.x; b < a.nb; b += gridDim.x) {
    const int bs = a.bstart[b], be = a.bstart[b + 1];
    const int lend = a.bline[b + 1];
    for (int i = threadIdx.x; i < be - bs; i += blockDim.x) xs[i] = __longlong_as_double((long long)LINE_PENDING);
    RowIter it, pf;
    it.init(a, a.bline[b] + warp, lend);
    pf.init(a, a.bline[b] + warp, lend);
    // L2 prefetch of the first a.pf records of this warp's sequence (the pipeline keeps a.pf ahead)
    for (int k = 0; k < a.pf; ++k) {
      const int q = pf.next(a, W, lend);
      if (q >= 0 && lane == 0) {
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rec(q)), "r"((unsigned)RB) : "memory");
        prefetch_line_l2(a.res + (a.upper ? a.n - 1 - q : q));
      }
    }
    __syncthreads();
    auto stage_a = [&](StA<C>& A, int p) {
      A.p = p;
      if (p < 0) return;
      A.row = a.upper ? a.n - 1 - p : p;
      const int* cc = reinterpret_cast<const int*>(rec(p));
#pragma unroll
      for (int k = 0; k < C; ++k) A.cc[k] = __ldg(cc + 32 * k + lane);
      const int q = pf.next(a, W, lend);
      if (q >= 0 && lane == 0) {
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(rec(q)), "r"((unsigned)RB) : "memory");
        const int qr = a.upper ? a.n - 1 - q : q;
        prefetch_line_l2(a.res + qr);
        if (a.accumulate) prefetch_line_l2(a.u + qr);
      }
    };
    auto stage_b = [&](StB<C>& B, const StA<C>& A) {
      B.p = A.p;
      B.row = A.row;
      if (A.p < 0) return;
      const double* cv = reinterpret_cast<const double*>(rec(A.p) + line_off_cv(C));
#pragma unroll
      for (int k = 0; k < C; ++k) {
        B.cc[k] = A.cc[k];
        B.xv[k] = fetch(xs, xg_cur, A.cc[k]);
        B.cv[k] = __ldg(cv + 32 * k + lane);
      }
    };
    auto poll = [&](int code, double v, int p) {
      if (!pend(v)) return v;
      const long long w0 = clock64();
      do {
        v = fetch(xs, xg_cur, code);
        if (clock64() - w0 > (1LL << 31)) line_stuck(code, p);
      } while (pend(v));
      return v;
    };
    auto stage_c = [&](StD& D, StB<C>& B) {
      D.p = B.p;
      D.row = B.row;
      if (B.p < 0) return;
      const int p = B.p;
      const char* r = rec(p);
      const int* meta = reinterpret_cast<const int*>(r + line_off_meta(C));
      const double* lvv = reinterpret_cast<const double*>(r + line_off_lv(C));
      const double* own = reinterpret_cast<const double*>(r + line_off_own(C));
      // late values and scalars of this row first (consumed one iteration later, in D)
#pragma unroll
      for (int j = 0; j < LINE_LATE; ++j) {
        D.lc[j] = __ldg(meta + j);
        D.lv[j] = __ldg(lvv + j);
      }
#pragma unroll
      for (int j = 0; j < LINE_LATE; ++j) D.lx[j] = fetch(xs, xg_cur, D.lc[j]);
      const int ovs = __ldg(meta + LINE_LATE), ovn = __ldg(meta + LINE_LATE + 1);
      D.rhs = __ldg(a.res + B.row);
      D.o1 = __ldg(own);
      D.o2 = __ldg(own + 1);
      D.o3 = __ldg(own + 2);
      D.idg = __ldg(own + 3);
      D.uold = (a.accumulate && lane == 0) ? a.u[B.row] : 0.0;
      // early values still pending: re-polled together, one round trip per attempt
      unsigned pm = 0;
#pragma unroll
      for (int k = 0; k < C; ++k) pm |= pend(B.xv[k]) ? 1u << k : 0u;
      D.cw = 0;
      if (a.trace && __any_sync(0xffffffffu, pm)) D.cw = -clock64();
      if (pm) {
        const long long w0 = clock64();
        unsigned nap = 0;  // backoff: a waiting warp must not take issue slots from the working ones
        do {
          if (nap) __nanosleep(nap);
          nap = nap ? min(nap * 2u, 1024u) : 32u;
#pragma unroll
          for (int k = 0; k < C; ++k)
            if (pm >> k & 1u) B.xv[k] = fetch(xs, xg_cur, B.cc[k]);
#pragma unroll
          for (int k = 0; k < C; ++k)
            if ((pm >> k & 1u) && !pend(B.xv[k])) pm &= ~(1u << k);
          if (pm && clock64() - w0 > (1LL << 31)) {
            int bad = 0;
#pragma unroll
            for (int k = 0; k < C; ++k)
              if (pm >> k & 1u) bad = B.cc[k];
            line_stuck(bad, p);
          }
        } while (pm);
      }
      if (D.cw) D.cw += clock64();
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < C; ++k) acc = fma(B.cv[k], B.xv[k], acc);
      for (int k = 0; k < ovn; ++k) {  // long rows (interface rows): the overflow chunks synchronously
        const size_t at = ((size_t)ovs + k) * 32 + lane;
        const int code = __ldg(a.ocol + at);
        acc = fma(__ldg(a.oval + at), poll(code, fetch(xs, xg_cur, code), p), acc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);  // same sum in every lane
      D.acc = acc;
    };
    StA<C> A;
    StB<C> B;
    StD D;
    double x1 = 0.0, x2 = 0.0, x3 = 0.0;
    // prologue: fill the pipeline
    stage_a(A, it.next(a, W, lend));
    stage_b(B, A);
    stage_a(A, it.next(a, W, lend));
    stage_c(D, B);
    stage_b(B, A);
    stage_a(A, it.next(a, W, lend));
    long long pc[5] = {0, 0, 0, 0, 0}, rows_done = 0;
    long long tc = a.prof ? clock64() : 0;
    auto mark = [&](int i) {
      if (a.prof) {
        const long long now = clock64();
        pc[i] += now - tc;
        tc = now;
      }
    };
    while (D.p >= 0) {
      ++rows_done;
      // D: finish row t (late values re-polled together, added oldest first, then the own line's)
      unsigned pm = 0;
#pragma unroll
      for (int j = 0; j < LINE_LATE; ++j) pm |= pend(D.lx[j]) ? 1u << j : 0u;
      const long long dw0 = a.trace ? clock64() : 0;
      if (pm) {
        const long long w0 = clock64();
        int tries = 0;
        do {
          if (++tries > 8) __nanosleep(32);
#pragma unroll
          for (int j = 0; j < LINE_LATE; ++j)
            if (pm >> j & 1u) D.lx[j] = fetch(xs, xg_cur, D.lc[j]);
#pragma unroll
          for (int j = 0; j < LINE_LATE; ++j)
            if ((pm >> j & 1u) && !pend(D.lx[j])) pm &= ~(1u << j);
          if (pm && clock64() - w0 > (1LL << 31)) line_stuck(D.lc[0], D.p);
        } while (pm);
      }
      mark(0);
      double s = D.rhs - D.acc;
#pragma unroll
      for (int j = 0; j < LINE_LATE; ++j) s = fma(-D.lv[j], D.lx[j], s);
      s = fma(-D.o3, x3, s);
      s = fma(-D.o2, x2, s);
      s = fma(-D.o1, x1, s);
      const double x = s * D.idg;
      if (lane == 0) {
        *(volatile double*)(xs + (D.p - bs)) = x;
        st_relaxed(xg_set + D.p, x);
        if (a.trace) {
          long long gt;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
          a.trace[3 * (size_t)D.p] = gt;
          a.trace[3 * (size_t)D.p + 1] = clock64() - dw0;
          a.trace[3 * (size_t)D.p + 2] = D.cw;
        }
        xg_clr[D.p] = __longlong_as_double((long long)LINE_PENDING);
        a.u[D.row] = a.accumulate ? D.uold + x : x;
      }
      x3 = x2;
      x2 = x1;
      x1 = x;
      mark(1);
      stage_c(D, B);
      mark(2);
      stage_b(B, A);
      mark(3);
      stage_a(A, it.next(a, W, lend));
      mark(4);
    }
    if (a.prof && lane == 0 && rows_done) {
      for (int i = 0; i < 5; ++i) atomicAdd((unsigned long long*)a.prof + i, (unsigned long long)pc[i]);
      atomicAdd((unsigned long long*)a.prof + 5, (unsigned long long)rows_done);
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
}

}  // namespace

// register chunks of the record layout (line_plan.cpp picks 2, 4 or 6)
int line_chunk_variant(int C) { return C <= 2 ? 2 : C <= 4 ? 4 : 6; }

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
    default: launch_k(line_sweep_kernel<6>, grid, block, smem, s, a); break;
  }
}

}  // namespace igb
