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

namespace igb {
namespace {

constexpr unsigned long long WAVE_PENDING = 0x7FF4DEADBEEF2468ULL;
constexpr int GI = WAVE_GI, SP = WAVE_SP, NI = WAVE_NI;
constexpr int NCOMP = NI * 32;          // compute lanes
constexpr int NP = 3;                   // poller warps
constexpr int NPOLL = NP * 32;
constexpr int NE = WAVE_NT / 32 - NI - NP;   // external warps per CTA
constexpr int PF = 16;                  // frames of lane records in flight
constexpr int RQ = SP * 16;             // queue slots between pollers and compute lanes
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
__device__ __noinline__ void wave_stuck(const char* what, int a, int b) {
  printf("[igb wave] block %d thread %d: %s (%d, %d) never arrived\n", (int)blockIdx.x, (int)threadIdx.x, what, a, b);
  __trap();
}

struct WaveCtrl {
  int bundle;   // bundle being swept (-1: none left)
  int seq;      // bumped at every hand-out
  int cons;     // global slots consumed by the compute warps
  int pad;
};

__global__ void __launch_bounds__(WAVE_NT, 1) wave_sweep_kernel(WaveArgs a) {
  pdl_begin();
  extern __shared__ __align__(16) unsigned char wave_smem[];
  // shared-memory carve-up
  double* xs = reinterpret_cast<double*>(wave_smem);                       // [xs_len]
  WaveRecA* ringA = reinterpret_cast<WaveRecA*>(xs + a.xs_len);            // [PF][NCOMP]
  WaveRecB* ringB = reinterpret_cast<WaveRecB*>(ringA + PF * NCOMP);
  double* rq_rhs = reinterpret_cast<double*>(ringB + PF * NCOMP);         // [RQ] value + ready flag
  double* rq_ext = rq_rhs + RQ;
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
  if (tid == 0) {
    ctrl->bundle = -1;
    ctrl->seq = 0;
    ctrl->cons = 0;
  }
  __syncthreads();

  if (warp < NI) {
    // ------------------------------------------------------------------ compute warps
    const int L = tid, r = L / GI, gl = L % GI;
    int seq = 0;
    for (;;) {
      if (tid == 0) {
        const int b = atomicAdd(a.ticket, 1);
        const int bb = b < a.nb ? b : -1;
        if (bb >= 0) {
          ctrl->cons = ld_nc_s32(a.b_frame + bb) * SP;
          xs[ld_nc_s32(a.b_rows + bb)] = 0.0;
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
#pragma unroll 1
      for (int i = 0; i < PF; ++i) {
        if (fr0 + i < fr1) {
          cp_async16(&ringA[i * NCOMP + L], a.recA + (size_t)(fr0 + i) * NCOMP + L);
          cp_async16(&ringB[i * NCOMP + L], a.recB + (size_t)(fr0 + i) * NCOMP + L);
        }
        cp_async_commit();
      }
      int e = 0;
#pragma unroll 1
      for (int f = fr0; f < fr1; ++f) {
        cp_async_wait<PF - 1>();
        const WaveRecA A = ringA[e * NCOMP + L];
        const WaveRecB B = ringB[e * NCOMP + L];
        const double x0 = xs[B.i0], x1 = xs[B.i1], x2 = xs[B.i2];
        double acc = __dmul_rn(A.c0, x0);
        acc = fma(A.c1, x1, acc);
        acc = fma(B.c2, x2, acc);
        if (f + PF < fr1) {
          cp_async16(&ringA[e * NCOMP + L], a.recA + (size_t)(f + PF) * NCOMP + L);
          cp_async16(&ringB[e * NCOMP + L], a.recB + (size_t)(f + PF) * NCOMP + L);
        }
        cp_async_commit();
        e = e + 1 == PF ? 0 : e + 1;
#pragma unroll
        for (int o = GI / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, GI);
        if (gl == 0) {
          const int q = (f * SP + r) % RQ;
          volatile double* vr = rq_rhs + q;
          double rhs = *vr;
          if (is_pending(rhs)) {
            const long long w0 = clock64();
            while (is_pending(rhs = *vr))
              if (clock64() - w0 > (1LL << 31)) wave_stuck("queue slot of frame/slot", f, r);
          }
          const int row = *(volatile int*)(rq_row + q);
          if (row >= 0) {
            const double ext = *(volatile double*)(rq_ext + q);
            const double idg = *(volatile double*)(rq_idg + q);
            const double xv = (rhs - (ext + acc)) * idg;
            xs[*(volatile int*)(rq_loc + q)] = xv;
            st_relaxed(xg_set + row, xv);
            xg_clr[row] = pending();
            a.u[row] = a.accumulate ? *(volatile double*)(rq_uold + q) + xv : xv;
          }
          *vr = pending();
        }
        bar_compute();
        if (tid == 0) ctrl->cons = (f + 1) * SP;
      }
      cp_async_wait<0>();
    }
  } else if (warp < NI + NP) {
    // ------------------------------------------------------------------ poller warps
    const int j = tid - NCOMP;
    int seq = 0;
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
      const int s1 = ld_nc_s32(a.b_frame + b + 1) * SP;
      int s = ld_nc_s32(a.b_frame + b) * SP + j;
      int4 h = make_int4(-1, 0, 0, 0);
      if (s < s1) h = *reinterpret_cast<const int4*>(a.slot + s);
      for (; s < s1; s += NPOLL) {
        const int row = h.x;
        const int loc = h.y & 0xffff, has_ext = (h.y >> 16) & 1;
        const double idg = __hiloint2double(h.w, h.z);
        if (s + NPOLL < s1) h = *reinterpret_cast<const int4*>(a.slot + s + NPOLL);
        double rhs = 0.0, uo = 0.0, ext = 0.0;
        if (row >= 0) {
          rhs = ld_nc_f64(a.res + row);
          if (a.accumulate) uo = a.u[row];
          if (has_ext) {
            ext = ld_relaxed(eg_cur + row);
            if (is_pending(ext)) {
              const long long w0 = clock64();
              while (is_pending(ext = ld_relaxed(eg_cur + row))) {
                if (a.backoff) __nanosleep(a.backoff);
                if (clock64() - w0 > (1LL << 31)) wave_stuck("external sum of row / slot", row, s);
              }
            }
          }
        }
        if (s >= ctrl->cons + RQ) {
          const long long w0 = clock64();
          while (s >= ctrl->cons + RQ) {
            __nanosleep(32);
            if (clock64() - w0 > (1LL << 32)) wave_stuck("queue space for slot", s, ctrl->cons);
          }
        }
        const int q = s % RQ;
        rq_ext[q] = ext;
        rq_idg[q] = idg;
        rq_uold[q] = uo;
        rq_row[q] = row;
        rq_loc[q] = loc;
        __threadfence_block();
        *(volatile double*)(rq_rhs + q) = rhs;
      }
    }
  } else {
    // ------------------------------------------------------------------ external warps (cf. flow.cu)
    const long long gwarp = (long long)blockIdx.x * NE + (warp - NI - NP);
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
      // late entries (the newest dependencies): every lane loads and polls all of them (same
      // addresses: one request per warp) and adds them serially in a fixed order
      if (el < e) {
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
