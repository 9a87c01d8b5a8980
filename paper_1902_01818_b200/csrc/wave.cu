// wave.cu -- Gauss-Seidel in the reference's natural order with the dependency chain kept inside
// one CTA per grid plane (wave_plan.h), sm_100a.
//
// Replaces SuperLU dgstrs on tril(A) / triu(A) as called by GaussSeidel.apply_forward /
// apply_backward (reference smoothers.py:171-200) on levels whose rows are long and whose
// dependency levels are wide (3-D patches): there the flow sweep (flow.cu) pays one L2 round trip
// per dependency level (0.85-1.2 us), because every level of the lattice reads the level before.
//
// One persistent CTA per SM, 32 warps in three roles:
//   compute warps (WAVE_NI): sweep one bundle (plane) at a time, frame by frame.  Lane (slot r,
//     part gl) gathers KI values of the bundle's solution vector from shared memory, the GI parts
//     are reduced by shuffles, lane gl == 0 finishes the row
//         x = (rhs - (external sum + internal sum)) / a_ii,
//     stores it to shared memory and publishes it (global copy xg, u), and one named barrier ends
//     the frame.  The lane records stream through a private cp.async ring PF frames ahead, so the
//     chain never waits for global memory.
//   poller warps (WAVE_NP): fetch what lane gl == 0 needs for the coming slots -- header, right-hand
//     side, old u, and the row's external sum (polled from the global copy eg until produced) --
//     into a shared-memory queue, RQ slots ahead of the compute warps.
//   external warps (the rest): the flow sweep's loop over the rows that have external entries, in
//     global dependency-level order, values polled from xg; they publish the sums in eg.
// Bundles are handed out in position order by a ticket counter; the planner bounds the number of
// bundles that must be held at once by the number of CTAs, and every CTA is resident, so the
// lowest unfinished row always has a running owner: no deadlock, no grid-wide barrier.  Every
// wait has a clock64 watchdog that reports and traps instead of hanging the device.
#include <cstdio>

#include "kernels.cuh"
#include "wave_plan.h"

namespace igb {
namespace {

constexpr unsigned long long WAVE_PENDING = 0x7FF4DEADBEEF2468ULL;
constexpr int GI = WAVE_GI, SP = WAVE_SP, NI = WAVE_NI, PQ = WAVE_PQ, LK = WAVE_LK, LN = WAVE_LN, RQ = WAVE_RQ;
constexpr int NCOMP = NI * 32;          // compute lanes
constexpr int NP = 6;                   // poller warps
constexpr int NQ = NP * 32 / PQ;        // poller quads (rows in flight)
constexpr int NE = WAVE_NT / 32 - NI - 1 - NP;   // external warps per CTA (one warp publishes)
constexpr int PF = 16;                  // frames of lane records in flight
constexpr int EK = 6;                   // external entries per lane and chunk

__device__ __forceinline__ double ld_relaxed(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
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
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ bool is_pending(double v) {
  return (unsigned long long)__double_as_longlong(v) == WAVE_PENDING;
}
__device__ __forceinline__ double pending() { return __longlong_as_double((long long)WAVE_PENDING); }
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bar_compute() { asm volatile("bar.sync 1, %0;" ::"n"(NCOMP) : "memory"); }
__device__ unsigned long long wave_progress[4];  // frames, external rows, bundles handed out (diagnostics of the watchdog)
__device__ __noinline__ void wave_stuck(const char* what, int a, int b) {
  volatile unsigned long long* wp = wave_progress;
  const unsigned long long f0 = wp[0], e0 = wp[1], b0 = wp[2];
  printf("[igb wave] block %d thread %d: %s (%d, %d) never arrived; frames done %llu, external rows %llu, bundles %llu\n",
         (int)blockIdx.x, (int)threadIdx.x, what, a, b, f0, e0, b0);
  const long long w0 = clock64();
  while (clock64() - w0 < (1LL << 31)) {}   // let every other stuck thread report before the trap
  __trap();
}

struct WaveCtrl {
  int bundle;   // bundle being swept (-1: none left)
  int seq;      // bumped at every hand-out
  int cons;     // rows of the bundle published and freed (pollers' flow control)
  int cnt;      // rows of the bundle computed (compute warps, before the frame's barrier)
  int fseq;     // frames of the bundle finished (thread 0, after the barrier)
  int pad[3];
};

__global__ void __launch_bounds__(WAVE_NT, 1) wave_sweep_kernel(WaveArgs a) {
  pdl_begin();
  extern __shared__ __align__(16) unsigned char wave_smem[];
  // shared-memory carve-up
  double* xs = reinterpret_cast<double*>(wave_smem);                       // [xs_len]
  WaveRecA* ringA = reinterpret_cast<WaveRecA*>(xs + a.xs_len);            // [PF][NCOMP]
  WaveRecB* ringB = reinterpret_cast<WaveRecB*>(ringA + PF * NCOMP);
  double* rq_rhs = reinterpret_cast<double*>(ringB + PF * NCOMP);         // [RQ] value + ready flag
  double* rq_ext = rq_rhs + RQ;   // the row's result x (compute lane -> publisher)
  double* rq_idg = rq_ext + RQ;
  double* rq_uold = rq_idg + RQ;
  int* rq_row = reinterpret_cast<int*>(rq_uold + RQ);
  int* rq_loc = rq_row + RQ;
  volatile WaveCtrl* ctrl = reinterpret_cast<volatile WaveCtrl*>(rq_loc + RQ);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int par = *(volatile const int*)a.par_ctr;  // stable for the whole launch
  const double* xg_cur = a.xg + (size_t)par * a.n;
  double* xg_set = a.xg + (size_t)par * a.n;
  double* xg_clr = a.xg + (size_t)(par ^ 1) * a.n;
  const double* eg_cur = a.eg + (size_t)par * a.n;
  double* eg_set = a.eg + (size_t)par * a.n;
  double* eg_clr = a.eg + (size_t)(par ^ 1) * a.n;

  for (int i = tid; i < RQ; i += WAVE_NT) rq_rhs[i] = pending();
  if (a.dbg && blockIdx.x == 0 && tid < 4) wave_progress[tid] = 0;
  if (tid == 0) {
    ctrl->bundle = -1;
    ctrl->seq = 0;
    ctrl->cons = 0;
    ctrl->cnt = 0;
    ctrl->fseq = 0;
  }
  __syncthreads();

  if (warp < NI) {
    // ------------------------------------------------------------------ compute warps
    // The frame loop is one dependent chain per warp (shared-memory gather -> fma -> shuffles ->
    // finish -> store -> barrier), so every instruction in it costs its full latency: the lane only
    // computes; publishing x (global copy, u) and freeing the queue slot is the publisher warp's job.
    const int L = tid, gl = L % GI;
    int seq = 0;
    long long d_frames = 0, d_cyc = 0, d_bund = 0;
    for (;;) {
      if (tid == 0) {
        const int b = atomicAdd(a.ticket, 1);
        const int bb = b < a.nb ? b : -1;
        if (a.dbg) atomicAdd(&wave_progress[2], 1ULL);
        if (bb >= 0) {
          ctrl->cons = 0;
          ctrl->cnt = 0;
          ctrl->fseq = 0;
          xs[ld_nc_s32(a.b_start + bb + 1) - ld_nc_s32(a.b_start + bb)] = 0.0;
        }
        ctrl->bundle = bb;
        __threadfence_block();
        ctrl->seq = seq + 1;
      }
      ++seq;
      bar_compute();
      const int b = ctrl->bundle;
      if (b < 0) break;
      const int fr0 = ld_nc_s32(a.b_frame + b), fr1 = ld_nc_s32(a.b_frame + b + 1);
      const WaveRecA* pa = a.recA + (size_t)fr0 * NCOMP + L;
      const WaveRecB* pb = a.recB + (size_t)fr0 * NCOMP + L;
#pragma unroll 1
      for (int i = 0; i < PF; ++i) {
        if (fr0 + i < fr1) {
          cp_async16(&ringA[i * NCOMP + L], pa);
          cp_async16(&ringB[i * NCOMP + L], pb);
        }
        cp_async_commit();
        pa += NCOMP;
        pb += NCOMP;
      }
      const long long t_b = a.dbg ? clock64() : 0;
      int left = fr1 - fr0 - PF;     // frames still to prefetch
      WaveRecA* ra = ringA + L;
      WaveRecB* rb = ringB + L;
      int e = 0;
#pragma unroll 1
      for (int f = fr0; f < fr1; ++f) {
        cp_async_wait<PF - 1>();
        const WaveRecA A = *ra;
        const WaveRecB B = *rb;
        const double x0 = xs[B.i0], x1 = xs[B.i1], x2 = xs[B.i2];
        const bool mine = gl == 0 && B.ord != 0;
        const int q = (int)B.ord - 1;
        double bq = 0.0;
        if (mine) {  // the pollers' hand-over for this row (normally there already)
          volatile double* vr = rq_rhs + q;
          bq = *vr;
          if (is_pending(bq)) {
            const long long w0 = clock64();
            while (is_pending(bq = *vr))
              if (clock64() - w0 > (1LL << 31)) wave_stuck("queue slot of bundle / frame", b, f - fr0);
          }
        }
        double acc = __dmul_rn(A.c0, x0);
        acc = fma(A.c1, x1, acc);
        acc = fma(B.c2, x2, acc);
        if (left > 0) {
          cp_async16(ra, pa);
          cp_async16(rb, pb);
          pa += NCOMP;
          pb += NCOMP;
        }
        --left;
        cp_async_commit();
        if (++e == PF) {
          e = 0;
          ra = ringA + L;
          rb = ringB + L;
        } else {
          ra += NCOMP;
          rb += NCOMP;
        }
#pragma unroll
        for (int o = GI / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, GI);
        if (mine) {
          const double xv = (bq - acc) * *(volatile double*)(rq_idg + q);
          xs[*(volatile int*)(rq_loc + q)] = xv;
          *(volatile double*)(rq_ext + q) = xv;
        }
        bar_compute();
        if (tid == 0) ctrl->fseq = f - fr0 + 1;
      }
      cp_async_wait<0>();
      if (a.dbg && tid == 0) {
        d_cyc += clock64() - t_b;
        d_frames += fr1 - fr0;
        ++d_bund;
      }
      // the publisher frees the queue; the next bundle may not start before it is empty
      if (tid == 0) {
        const int rows = ld_nc_s32(a.b_start + b + 1) - ld_nc_s32(a.b_start + b);
        const long long w0 = clock64();
        while (ctrl->cons < rows)
          if (clock64() - w0 > (1LL << 31)) wave_stuck("publisher of bundle", b, ctrl->cons);
      }
    }
    if (a.dbg && tid == 0) {
      atomicAdd((unsigned long long*)a.dbg + 0, (unsigned long long)d_frames);
      atomicAdd((unsigned long long*)a.dbg + 1, (unsigned long long)d_cyc);
      atomicAdd((unsigned long long*)a.dbg + 3, (unsigned long long)d_bund);
    }
  } else if (warp == NI) {
    // ------------------------------------------------------------------ publisher warp
    // after every frame: the rows just computed go to the global copy (and u), their queue slots
    // are freed
    int seq = 0;
    for (;;) {
      {
        const long long w0 = clock64();
        while (ctrl->seq == seq) {
          __nanosleep(64);
          if (clock64() - w0 > (1LL << 32)) wave_stuck("bundle hand-out (publisher)", seq, 0);
        }
      }
      ++seq;
      __threadfence_block();
      const int b = ctrl->bundle;
      if (b < 0) break;
      const int fr0 = ld_nc_s32(a.b_frame + b);
      const int nfr = ld_nc_s32(a.b_frame + b + 1) - fr0;
      int fs = 0, o0 = 0;
      while (fs < nfr) {
        int fnow = ctrl->fseq;
        if (fnow == fs) {
          const long long w0 = clock64();
          while ((fnow = ctrl->fseq) == fs)
            if (clock64() - w0 > (1LL << 32)) wave_stuck("frame of bundle (publisher)", b, fs);
        }
        __threadfence_block();
        const int o1 = ld_nc_s32(a.f_end + fr0 + fnow - 1);   // rows of the bundle in its first fnow frames
        for (int o = o0 + lane; o < o1; o += 32) {
          const int q = o % RQ;
          const double xv = *(volatile double*)(rq_ext + q);
          const int row = *(volatile int*)(rq_row + q);
          st_relaxed(xg_set + row, xv);
          xg_clr[row] = pending();
          a.u[row] = a.accumulate ? *(volatile double*)(rq_uold + q) + xv : xv;
          *(volatile double*)(rq_rhs + q) = pending();
        }
        __syncwarp();
        if (lane == 0 && o1 > o0) {
          __threadfence_block();
          ctrl->cons = o1;
          if (a.dbg) atomicAdd(&wave_progress[0], (unsigned long long)(fnow - fs));
        }
        o0 = o1;
        fs = fnow;
      }
    }
  } else if (warp < NI + 1 + NP) {
    // ------------------------------------------------------------------ poller warps
    // a quad of lanes per row: header, right-hand side, old u, the external warps' sum, and the
    // row's late entries (LK per lane), polled from xg and added here
    // Every quad walks its own rows (u0 + g, + NQ, ...) at its own pace, but the warp runs ONE
    // instruction stream: a loop in which each quad polls what its current row still misses,
    // delivers the row when complete and moves on.  A quad must not hold back its warp mates (their
    // rows may belong to earlier frames, and the awaited values may depend on those through the
    // external warps), and divergent per-quad spin loops would multiply the issue slots the
    // pollers take from the compute warps.
    const int g = (tid - NCOMP - 32) / PQ, ql = tid & (PQ - 1);
    int seq = 0;
    long long d_xw = 0, d_ew = 0, d_rows = 0, d_fc = 0;
    for (;;) {
      {
        const long long w0 = clock64();
        while (ctrl->seq == seq) {
          __nanosleep(64);
          if (clock64() - w0 > (1LL << 32)) wave_stuck("bundle hand-out", seq, 0);
        }
      }
      ++seq;
      __threadfence_block();
      const int b = ctrl->bundle;
      if (b < 0) break;
      const int u0 = ld_nc_s32(a.b_start + b), u1 = ld_nc_s32(a.b_start + b + 1);
      int4 hn = make_int4(-1, 0, 0, 0);
      int lcn[LK];
      double lvn[LK];
      auto fetch = [&](int u) {
        if (u < u1) {
          hn = *reinterpret_cast<const int4*>(a.hdr + u);
#pragma unroll
          for (int k = 0; k < LK; ++k) {
            lcn[k] = ld_nc_s32(a.lcol + (size_t)u * LN + ql * LK + k);
            lvn[k] = ld_nc_f64(a.lval + (size_t)u * LN + ql * LK + k);
          }
        }
      };
      int u = u0 + g;
      bool have = false, extp = false;
      int4 h = hn;
      int lc[LK];
      double lv[LK], x[LK];
      double rhs = 0.0, uo = 0.0, ext = 0.0;
      unsigned pend = 0;
      long long t_have = 0;
#pragma unroll
      for (int k = 0; k < LK; ++k) { lc[k] = -1; lv[k] = 0.0; x[k] = 0.0; }
      fetch(u);
      for (;;) {
        if (!have && u < u1) {  // take the prefetched row, start its loads
          h = hn;
#pragma unroll
          for (int k = 0; k < LK; ++k) { lc[k] = lcn[k]; lv[k] = lvn[k]; }
          fetch(u + NQ);
          const int row = h.x;
          rhs = 0.0; uo = 0.0; ext = 0.0;
          if (ql == 0) rhs = ld_nc_f64(a.res + row);
          if (ql == 1 && a.accumulate) uo = a.u[row];
          extp = ql == 2 && ((h.y >> 16) & 1);
          if (extp) ext = ld_relaxed(eg_cur + row);
          pend = 0;
#pragma unroll
          for (int k = 0; k < LK; ++k) {
            x[k] = 0.0;
            if (lc[k] >= 0) {
              x[k] = ld_relaxed(xg_cur + lc[k]);
              pend |= 1u << k;
            }
          }
          have = true;
          t_have = clock64();

        }
        if (have) {  // what arrived since the last pass; reload the rest
#pragma unroll
          for (int k = 0; k < LK; ++k)
            if (pend >> k & 1u) {
              if (!is_pending(x[k])) pend &= ~(1u << k);
              else x[k] = ld_relaxed(xg_cur + lc[k]);
            }
          if (extp) {
            if (!is_pending(ext)) extp = false;
            else ext = ld_relaxed(eg_cur + h.x);
          }
          if ((pend || extp) && clock64() - t_have > (1LL << 31)) {
            printf("[igb wave] bundle %d rows [%d, %d) row u %d waits for rows %d %d %d (mask %u, ext %d), cons %d\n", b, u0,
                   u1, u, lc[0], lc[1], lc[2], pend, (int)extp, ctrl->cons);
            wave_stuck("late value / external sum for row", h.x, (int)pend);
          }
        }
        const unsigned rdy = __ballot_sync(0xffffffffu, have && pend == 0 && !extp);
        const bool quad_ready = ((rdy >> (lane & ~(PQ - 1))) & 0xFu) == 0xFu;
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < LK; ++k) acc = fma(lv[k], x[k], acc);
        acc += __shfl_xor_sync(0xffffffffu, acc, 1, PQ);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2, PQ);
        const double uo0 = __shfl_sync(0xffffffffu, uo, 1, PQ);
        const double ext0 = __shfl_sync(0xffffffffu, ext, 2, PQ);
        int delivered = 0;
        if (quad_ready && ql == 0) {
          const int o = u - u0;
          if (o + SP + 1 <= ctrl->cons + RQ) {
            const int q = o % RQ;
            rq_idg[q] = __hiloint2double(h.w, h.z);
            rq_uold[q] = uo0;
            rq_row[q] = h.x;
            rq_loc[q] = h.y & 0xffff;
            __threadfence_block();
            *(volatile double*)(rq_rhs + q) = rhs - (ext0 + acc);
            delivered = 1;
            if (a.dbg && g == 0) {
              ++d_rows;
              d_xw += clock64() - t_have;
            }
          } else if (a.dbg && g == 0) {
            ++d_fc;
          }
        }
        delivered = __shfl_sync(0xffffffffu, delivered, 0, PQ);
        if (delivered) {
          have = false;
          u += NQ;
        }
        if (__all_sync(0xffffffffu, !have && u >= u1)) break;
        if (!__any_sync(0xffffffffu, delivered) && a.pbackoff) __nanosleep(a.pbackoff);
      }
    }
    if (a.dbg && g == 0 && ql == 0) {
      atomicAdd((unsigned long long*)a.dbg + 4, (unsigned long long)d_xw);
      atomicAdd((unsigned long long*)a.dbg + 5, (unsigned long long)d_ew);
      atomicAdd((unsigned long long*)a.dbg + 6, (unsigned long long)d_rows);
      atomicAdd((unsigned long long*)a.dbg + 7, (unsigned long long)d_fc);
    }
  } else {
    // ------------------------------------------------------------------ external warps (cf. flow.cu)
    const long long gwarp = (long long)blockIdx.x * NE + (warp - NI - 1 - NP);
    const long long nwarps = (long long)gridDim.x * NE;
    long long q = gwarp;
    int nrow = -1, ns = 0, ne = 0, nel = 0, ncc = -1;
    if (q < a.nq) {
      nrow = ld_nc_s32(a.e_row + q);
      ns = ld_nc_s32(a.eptr + q);
      ne = ld_nc_s32(a.eptr + q + 1);
      nel = ld_nc_s32(a.elate + q);
      ncc = ld_nc_s32(a.crit + q);
    }
    for (; q < a.nq; q += nwarps) {
      const int row = nrow, s = ns, e = ne, el = nel, cc = ncc;
      if (q + nwarps < a.nq) {  // next row's metadata
        nrow = ld_nc_s32(a.e_row + q + nwarps);
        ns = ld_nc_s32(a.eptr + q + nwarps);
        ne = ld_nc_s32(a.eptr + q + nwarps + 1);
        nel = ld_nc_s32(a.elate + q + nwarps);
        ncc = ld_nc_s32(a.crit + q + nwarps);
      }
      // first chunk of coefficients while the critical dependency is awaited
      int c[EK];
      double v[EK], x[EK];
#pragma unroll
      for (int k = 0; k < EK; ++k) {
        const int idx = s + lane + k * 32;
        c[k] = idx < el ? __ldcs(a.ecol + idx) : -1;
        v[k] = idx < el ? __ldcs(a.eval + idx) : 0.0;
      }
      if (lane == 0 && cc >= 0 && is_pending(ld_relaxed(xg_cur + cc))) {
        const long long w0 = clock64();
        while (is_pending(ld_relaxed(xg_cur + cc))) {
          if (a.backoff) __nanosleep(a.backoff);
          if (clock64() - w0 > (1LL << 31)) wave_stuck("critical value / row", cc, row);
        }
      }
      __syncwarp();
      double acc = 0.0;
      for (int base = s; base < el; base += 32 * EK) {
        if (base > s) {
#pragma unroll
          for (int k = 0; k < EK; ++k) {
            const int idx = base + lane + k * 32;
            c[k] = idx < el ? __ldcs(a.ecol + idx) : -1;
            v[k] = idx < el ? __ldcs(a.eval + idx) : 0.0;
          }
        }
#pragma unroll
        for (int k = 0; k < EK; ++k) x[k] = c[k] >= 0 ? ld_relaxed(xg_cur + c[k]) : 0.0;
        unsigned pend = 0;
#pragma unroll
        for (int k = 0; k < EK; ++k) pend |= (c[k] >= 0 && is_pending(x[k])) ? 1u << k : 0u;
        if (pend) {
          const long long w0 = clock64();
          do {
            if (a.backoff) __nanosleep(a.backoff);
#pragma unroll
            for (int k = 0; k < EK; ++k)
              if (pend >> k & 1u) x[k] = ld_relaxed(xg_cur + c[k]);
#pragma unroll
            for (int k = 0; k < EK; ++k)
              if ((pend >> k & 1u) && !is_pending(x[k])) pend &= ~(1u << k);
            if (pend && clock64() - w0 > (1LL << 31)) wave_stuck("early value for row", row, (int)pend);
          } while (pend);
        }
#pragma unroll
        for (int k = 0; k < EK; ++k) acc = fma(v[k], x[k], acc);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      // late entries of the list (newer than crit_lag levels, beyond the pollers' LN): every lane
      // loads and polls all of them and adds them serially in a fixed order
      if (el < e) {
        constexpr int LM = 4;
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
              if (a.backoff) __nanosleep(a.backoff);
#pragma unroll
              for (int j = 0; j < LM; ++j)
                if (pend >> j & 1u) lx[j] = ld_relaxed(xg_cur + lc[j]);
#pragma unroll
              for (int j = 0; j < LM; ++j)
                if ((pend >> j & 1u) && !is_pending(lx[j])) pend &= ~(1u << j);
              if (pend && clock64() - w0 > (1LL << 31)) wave_stuck("late value for row", row, (int)pend);
            } while (pend);
          }
#pragma unroll
          for (int j = 0; j < LM; ++j) acc = fma(lv[j], lx[j], acc);
        }
      }
      if (lane == 0) {
        st_relaxed(eg_set + row, acc);
        eg_clr[row] = pending();
        if (a.dbg) atomicAdd(&wave_progress[1], 1ULL);
      }
    }
  }
  __syncthreads();
  if (tid == 0) {  // the last CTA flips the parity and rewinds the ticket for the next sweep
    __threadfence();
    if (atomicAdd(a.done_ctr, 1u) == gridDim.x - 1) {
      *a.done_ctr = 0u;
      *(volatile int*)a.ticket = 0;
      *(volatile int*)a.par_ctr = par ^ 1;
      __threadfence();
    }
  }
}

}  // namespace

size_t wave_smem_bytes(int rb_max) {
  const size_t xs_len = ((size_t)rb_max + 1 + 1) & ~(size_t)1;
  return xs_len * 8 + (size_t)PF * NCOMP * 32 + (size_t)RQ * 40 + 16;
}
int wave_xs_len(int rb_max) { return (int)(((size_t)rb_max + 1 + 1) & ~(size_t)1); }

int wave_max_ctas(size_t smem) {
  int dev = 0, sms = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(wave_sweep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, wave_sweep_kernel, WAVE_NT, smem);
  cudaGetLastError();
  return per * sms;
}

void wave_set_carveout(int pct) {
  cudaFuncSetAttribute(wave_sweep_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
  cudaGetLastError();
}

void launch_wave_sweep(cudaStream_t s, const WaveArgs& a) {
  launch_k(wave_sweep_kernel, dim3(a.ctas), dim3(WAVE_NT), wave_smem_bytes(a.rb_max), s, a);
}

}  // namespace igb
