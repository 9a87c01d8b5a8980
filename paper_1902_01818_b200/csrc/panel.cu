// panel.cu -- row-panel triangular sweep for the Gauss-Seidel smoother (sm_100a).
//
// Solves T c = r (T = tril(A) forward / triu(A) backward, smoothers.py:178-190) in
// position space, one panel of B = 32 G rows per step, on one thread-block cluster
// of G CTAs x 16 warps (plan: panel_plan.h).  Per panel k:
//
//   phase A  r_i = res_i - sum_{q < kB} T_iq c_q       half-warp per row, ring in smem
//            (+ entries older than the ring, gathered one panel ahead from global)
//            -> r_i stored into every CTA's rbuf (DSMEM);   cluster barrier
//   phase B  c_i = sum_j Tinv_kk[i][j] r_j              warp per row pair (q, b-1-q),
//            Tinv slice of this CTA staged by a TMA bulk copy issued one
//            panels ahead -> c_i stored into every CTA's ring (DSMEM), u, xg;
//            cluster barrier
//
// Everything but c is x-independent and streamed ahead: the per-panel critical
// path is two cluster barriers plus a 16-lane and a 32-lane reduction.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace igb {

namespace {

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init1(unsigned long long* b) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(b)) : "memory");
}
// The inverse blocks are read once per sweep (147 MB per direction on cfg2's finest level, more than
// L2): load them with an evict-first L2 policy so they do not push the matrices and vectors the
// rest of the cycle reuses out of L2.
__device__ __forceinline__ unsigned long long evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                          unsigned long long policy, bool hint) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(bar)), "r"(bytes) : "memory");
  if (hint)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            saddr(dst)),
        "l"(src), "r"(bytes), "r"(saddr(bar)), "l"(policy)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(saddr(dst)),
        "l"(src), "r"(bytes), "r"(saddr(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "PWAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra PWAIT_%=;\n}" ::"r"(saddr(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

__device__ __forceinline__ unsigned mapa(unsigned local, int rank) {
  unsigned r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
// store one double into (remote) shared memory; completion is signalled on the
// receiver's mbarrier as 8 transaction bytes
__device__ __forceinline__ void st_async(unsigned raddr, double v, unsigned rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
               "l"(__double_as_longlong(v)), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void mbar_arm(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(unsigned long long* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(saddr(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Wait for a phase of an exchange mbarrier.  Watchdog: a protocol error must not hang
// the device -- after ~2^31 cycles report and trap (the launch fails with an error).
__device__ __noinline__ void exchange_stuck(int what, int t, unsigned parity) {
  printf("[igb panel] cluster %d CTA %d thread %d: %s exchange of local panel %d (parity %u) never completed\n",
         (int)(blockIdx.x / cg::this_cluster().num_blocks()), (int)cg::this_cluster().block_rank(), (int)threadIdx.x,
         what ? "solution" : "residual", t, parity);
  __trap();
}
__device__ __forceinline__ void mbar_wait_cluster(unsigned long long* b, unsigned parity, int what = 0, int t = 0) {
  if (mbar_try(b, parity)) return;
  const long long t0 = clock64();
  while (!mbar_try(b, parity))
    if (clock64() - t0 > (1LL << 31)) exchange_stuck(what, t, parity);
}

// Global solution copy: two halves selected by the sweep parity; a value not yet produced in
// this sweep reads as PANEL_PENDING (a signalling NaN no arithmetic produces).  The producer
// writes the value into the current half and PENDING into the other (ready for the next sweep
// of this level and direction, which starts only after this kernel has finished).
constexpr unsigned long long PANEL_PENDING = 0x7FF4DEADBEEF1234ULL;
__device__ __forceinline__ bool pending(double v) {
  return (unsigned long long)__double_as_longlong(v) == PANEL_PENDING;
}
__device__ __noinline__ void poll_stuck(int pos) {
  printf("[igb panel] cluster %d CTA %d thread %d: solution value at position %d never produced\n",
         (int)(blockIdx.x / cg::this_cluster().num_blocks()), (int)cg::this_cluster().block_rank(),
         (int)threadIdx.x, pos);
  __trap();
}
__device__ __forceinline__ double poll_value(const double* xg, int pos, double v) {
  if (!pending(v)) return v;
  const long long t0 = clock64();
  do {
    v = __ldcg(xg + pos);
    if (clock64() - t0 > (1LL << 31)) poll_stuck(pos);
  } while (pending(v));
  return v;
}

template <int KA, int KF>
struct PanelSet {
  double b, u0;
  int xm, xc;                  // destination mask of this lane's phase-B row; values due in bar_x
                               // (low 16 bits) | far slots of panel t+2 (bits 16..)
  int kf;                      // far slots in use for the next panel (fv/fc/fx)
  double ev[KA];
  int ec[KA];
  double fv[KF > 0 ? KF : 1];  // far coefficients of the NEXT panel
  int fc[KF > 0 ? KF : 1];
  double fx[KF > 0 ? KF : 1];  // their solution values (loaded one panel ahead)
};

// Synchronisation: no CTA-wide or cluster-wide barrier per panel.  Every value
// a CTA needs from its peers arrives by st.async with a complete_tx on a local
// mbarrier: bar_r[t & 1] counts the b_t residuals of panel t (broadcast to every
// CTA), bar_x the solution values of panel t this CTA reads later (xcnt[t][cta];
// each value goes only to the CTAs whose rows reference it).  Thread 0 re-arms a
// barrier right after its phase completes, before its warp produces anything the
// next phase depends on.  Ordering argument: a CTA sends r(t+2) only after the
// x(t+1) it needs, which were produced after every CTA sent r(t+1), i.e. after
// every warp finished panel t (wait_r(t), phase B(t)) -- the planner gives every
// CTA at least one value of every panel so this holds; hence bar_r needs two
// parities, rbuf two buffers, and after wait_r(t) every local warp is past phase
// B(t-1) (so the TMA stage of panel t-1 may be refilled).  x(t+1) is produced only
// after every CTA sent r(t+1), i.e. after its wait_x(t): one bar_x suffices.
//
// Clusters: cluster c sweeps panels [split[c], split[c+1]); values of earlier ranges and
// values older than the ring come from the global copy, fetched one panel ahead and polled
// until produced.  Dependencies point only to earlier positions, so a cluster never waits
// for a later one.


// warps per CTA by inverse-chunk count: B = 512 (16 warps) or B = 256 (8 warps, more
// registers per thread for the entry-heavy 3-D rows)
template <int KBC>
__host__ __device__ constexpr int panel_warps() { return KBC == 17 ? 16 : 8; }

template <int KBC, int KA, int KF>
__global__ void __launch_bounds__(panel_warps<KBC>() * 32, 1) panel_sweep_kernel(PanelArgs a) {
  pdl_begin();
  using Set = PanelSet<KA, KF>;
  extern __shared__ __align__(128) double psm[];
  constexpr int W = panel_warps<KBC>();
  constexpr int S = PANEL_STAGES;
  const int B = a.B, R = a.R, n = a.n;
  const cg::cluster_group cluster = cg::this_cluster();
  const int G = (int)cluster.num_blocks(), s = (int)cluster.block_rank();
  const int ci = blockIdx.x / G;
  const int p0 = a.split[ci], p1 = a.split[ci + 1];  // this cluster's panels ...
  const int rs = a.rstart[ci], re = a.rstart[ci + 1];  // ... cover positions [rs, re), B each from rs
  const int T = p1 - p0;
  const int tid = threadIdx.x, w = tid >> 5, l = tid & 31, h = l >> 4, hl = l & 15;
  const int pq = w * G + s;  // pair index: rows pq and b-1-pq of every panel
  double* ring = psm;
  double* rbuf = ring + R;                    // [2][B]
  double* lin_s = rbuf + 2 * B;               // [S][W][KBC][32]
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(lin_s + (size_t)S * W * KBC * 32);
  unsigned long long* full = bars;            // [S] TMA stages
  unsigned long long* bar_r = bars + S;      // [2]
  unsigned long long* bar_x = bars + S + 2;
  const size_t cta_lin = (size_t)W * KBC * 32;
  const unsigned lin_bytes = (unsigned)(cta_lin * 8);
  auto panel_rows = [&](int t) { return min(B, re - (rs + t * B)); };  // local panel index t

  for (int i = tid; i < R + 2 * B; i += W * 32) psm[i] = 0.0;
  if (tid == 0) {
    for (int i = 0; i < S + 3; ++i) mbar_init1(&bars[i]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_arm(&bar_r[0], 8u * panel_rows(0));
    if (T > 1) mbar_arm(&bar_r[1], 8u * panel_rows(1));
    mbar_arm(bar_x, 8u * (__ldg(a.xcnt + (size_t)p0 * G + s) & 0xffff));
  }
  // lane hl sends to CTA hl of the cluster (G <= 16)
  const int peer = hl < G ? hl : 0;
  const unsigned peer_psm = mapa(saddr(psm), peer);
  const unsigned peer_bar_r = mapa(saddr(bar_r), peer), peer_bar_x = mapa(saddr(bar_x), peer);  // + 8 (t & 1)
  cluster.sync();

  const double* lin_g = a.lin + ((size_t)p0 * G + s) * cta_lin;  // panel p0 of this CTA
  const unsigned long long l2pol = evict_first_policy();
  const bool hint = !(a.ablate & 128);
  const size_t lin_panel = (size_t)G * cta_lin;
  if (tid == 0 && !(a.ablate & 1)) {
    for (int t = 0; t < S - 1 && t < T; ++t)
      bulk_load(lin_s + (size_t)t * cta_lin, lin_g + t * lin_panel, lin_bytes, &full[t], l2pol, hint);
    for (int t = S - 1; t < S - 1 + a.pf && t < T; ++t) bulk_prefetch_l2(lin_g + t * lin_panel, lin_bytes);
  }

  const size_t ent_cta = (size_t)W * KA * 32, far_cta = (size_t)W * KF * 32;
  const size_t ent_off = ((size_t)s * W + w) * KA * 32 + l, far_off = ((size_t)s * W + w) * KF * 32 + l;
  const int rmask = R - 1;
  const int par = KF > 0 ? *a.par_ctr : 0;  // sweep parity: stable for the whole launch
  const double* xg_cur = a.xg + (size_t)par * n;
  double* xg_set = a.xg + (size_t)par * n;
  double* xg_clr = a.xg + (size_t)(par ^ 1) * n;

  // set of local panel t: rhs + old u + near entries of t, far entries of t+1
  auto load = [&](Set& X, int t, int kf_next) {
    const int k = p0 + t, k0 = rs + t * B, b = panel_rows(t);
    const int ia = s * (B / G) + 2 * w + h;  // phase-A row (contiguous chunk per CTA)
    const int pr = h ? b - 1 - pq : pq;
    const int p = min(k0 + max(pr, 0), n - 1);  // clamped: invalid rows load a finite dummy
    const int row = a.upper ? n - 1 - p : p;
    const int pa = min(k0 + ia, n - 1);
    X.b = __ldg(a.res + (a.upper ? n - 1 - pa : pa));
    if (a.accumulate) X.u0 = a.u[row];
    X.xm = __ldg(a.xmask + p);
    X.xc = __ldg(a.xcnt + (size_t)k * G + s);
    const size_t eo = (size_t)k * G * ent_cta + ent_off;
#pragma unroll
    for (int j = 0; j < KA; ++j) {
      X.ev[j] = __ldg(a.ev + eo + j * 32);
      X.ec[j] = __ldg(a.ec + eo + j * 32);
    }
    if (KF > 0) {
      const int kn = k + 1 < p1 ? k + 1 : a.npan;  // panel npan is a zero pad
      const size_t fo = (size_t)kn * G * far_cta + far_off;
      X.kf = kf_next;
#pragma unroll
      for (int j = 0; j < KF; ++j) {
        X.fv[j] = 0.0;
        X.fc[j] = -1;
        if (j < kf_next) {  // warp-uniform: most panels need at most one slot
          X.fv[j] = __ldg(a.fv + fo + j * 32);
          X.fc[j] = __ldg(a.fc + fo + j * 32);
        }
      }
    }
  };

  Set A, Bs;
  load(A, 0, KF);
#pragma unroll
  for (int j = 0; j < (KF > 0 ? KF : 1); ++j) {
    Bs.fv[j] = 0.0;
    Bs.fx[j] = 0.0;  // slots skipped by the kf test keep finite (zero or older) values
    A.fx[j] = 0.0;
  }
  Bs.kf = 0;
  if (KF > 0) {  // the range's first panel: its far entries (other ranges) belong to no earlier set
    const size_t fo = (size_t)p0 * G * far_cta + far_off;
    Bs.kf = KF;
#pragma unroll
    for (int j = 0; j < KF; ++j) {
      Bs.fv[j] = __ldg(a.fv + fo + j * 32);
      Bs.fc[j] = __ldg(a.fc + fo + j * 32);
      if (Bs.fc[j] >= 0) Bs.fx[j] = __ldcg(xg_cur + Bs.fc[j]);
    }
  }
  const long long t_start = clock64();
  long long tm[6] = {0, 0, 0, 0, 0, 0};
  long long tprev = t_start;
  auto mark = [&](int i) {
    if (a.dbg) {
      const long long now = clock64();
      tm[i] += now - tprev;
      tprev = now;
    }
  };

  auto step = [&](Set& X, Set& Y, int t) {
    const int k0 = rs + t * B, b = panel_rows(t);
    if (t > 0 && !(a.ablate & 64)) {  // x of panel t-1 complete in this CTA's ring
      mbar_wait_cluster(bar_x, (unsigned)((t - 1) & 1), 1, t - 1);
      if (tid == 0) mbar_arm(bar_x, 8u * (X.xc & 0xffff));
    }
    mark(0);
    // far part of panel t (values gathered during panel t-1; re-polled if not produced yet)
    double sA = 0.0;
    if (KF > 0) {
#pragma unroll
      for (int j = 0; j < KF; ++j) {
        if (j < Y.kf && Y.fc[j] >= 0) Y.fx[j] = poll_value(xg_cur, Y.fc[j], Y.fx[j]);
        sA = fma(Y.fv[j], Y.fx[j], sA);
      }
    }
    mark(1);
    // ---- phase A: off-panel part, half-warp per row
    const int r1 = pq, r2 = b - 1 - pq;
    const bool v1 = pq < (b + 1) / 2, v2 = pq < b / 2;
    const bool vh = h ? v2 : v1;
    const int pr = h ? r2 : r1;
    if (!(a.ablate & 16)) {
#pragma unroll
      for (int j = 0; j < KA; ++j) sA = fma(X.ev[j], ring[X.ec[j]], sA);
    }
    sA += __shfl_xor_sync(0xffffffffu, sA, 8);
    sA += __shfl_xor_sync(0xffffffffu, sA, 4);
    sA += __shfl_xor_sync(0xffffffffu, sA, 2);
    sA += __shfl_xor_sync(0xffffffffu, sA, 1);
    const int rb = (t & 1) * B;
    const int ia = s * (B / G) + 2 * w + h;
    if (ia < b && hl < G && !(a.ablate & 64)) st_async(peer_psm + 8u * (R + rb + ia), X.b - sA, peer_bar_r + 8u * (t & 1));
    // issued while the residual exchange is in flight: next panel's set, old values
    if (KF > 0) {
#pragma unroll
      for (int j = 0; j < KF; ++j)  // panel t+1: positions < tB - R + B (final)
        if (j < X.kf) {  // padded slots (fc < 0) hold 0: never PENDING times a zero coefficient
          if (X.fc[j] >= 0) X.fx[j] = __ldcg(xg_cur + X.fc[j]);
          else X.fx[j] = 0.0;
        }
    }
    if (t + 1 < T) load(Y, t + 1, (a.ablate & 256) ? KF : X.xc >> 16);  // 256: every far slot (diagnostic)
    mark(2);
    // ---- phase B: inverse block, warp per row pair
    if (!(a.ablate & 64)) mbar_wait_cluster(&bar_r[t & 1], (unsigned)((t >> 1) & 1), 0, t);
    else __syncthreads();
    if (tid == 0) {
      if (t + 2 < T && !(a.ablate & 64)) mbar_arm(&bar_r[t & 1], 8u * panel_rows(t + 2));
      const int tn = t + S - 1;  // stage of panel t-1: every local warp is past it (wait_r)
      if (!(a.ablate & 1)) {
        if (tn < T)
          bulk_load(lin_s + (size_t)(tn & (S - 1)) * cta_lin, lin_g + tn * lin_panel, lin_bytes, &full[tn & (S - 1)],
                    l2pol, hint);
        if (a.pf && tn + a.pf < T) bulk_prefetch_l2(lin_g + (tn + a.pf) * lin_panel, lin_bytes);
      }
    }
    mark(3);
    if (!(a.ablate & 1)) mbar_wait_parity(&full[t & (S - 1)], (unsigned)((t / S) & 1));
    mark(4);
    const double* L = lin_s + (size_t)(t & (S - 1)) * cta_lin + (size_t)w * KBC * 32 + l;
    const double* rv = rbuf + rb + l;
    // row r1 uses chunks [0, nc1), row r2 chunks [nc1, nc1 + nc2); both read r at column 32c + lane
    const int nc1 = v1 ? (r1 + 32) >> 5 : 0, nc2 = v2 ? (r2 + 32) >> 5 : 0;
    const double* L2 = L + 32 * nc1;
    double a1 = 0.0, a2 = 0.0, a3 = 0.0, a4 = 0.0;
    if (a.ablate & 4) {
      a1 = rv[0];
      a2 = rv[32];
    } else {
#pragma unroll
      for (int c = 0; c < KBC - 1; c += 2) {
        const double x0 = rv[32 * c], x1 = rv[32 * c + 32];
        if (c < nc1) a1 = fma(L[32 * c], x0, a1);
        if (c + 1 < nc1) a3 = fma(L[32 * c + 32], x1, a3);
        if (c < nc2) a2 = fma(L2[32 * c], x0, a2);
        if (c + 1 < nc2) a4 = fma(L2[32 * c + 32], x1, a4);
      }
      a1 += a3;
      a2 += a4;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    const double xv = h ? a2 : a1;
    if (vh) {
      if (hl < G && (X.xm >> hl & 1) && !(a.ablate & 64)) st_async(peer_psm + 8u * ((k0 + pr) & rmask), xv, peer_bar_x);
      if (hl == 0 && !(a.ablate & 32)) {
        const int p = k0 + pr;
        const int row = a.upper ? n - 1 - p : p;
        a.u[row] = a.accumulate ? X.u0 + xv : xv;
        if (KF > 0) {
          __stcg(xg_set + p, xv);
          __stcg(xg_clr + p, __longlong_as_double((long long)PANEL_PENDING));
        }
      }
    }
    mark(5);
  };
  for (int t = 0; t < T; t += 2) {
    step(A, Bs, t);
    if (t + 1 < T) step(Bs, A, t + 1);
  }
  // every x of the last panel has landed here before anyone leaves the cluster
  if (!(a.ablate & 64)) mbar_wait_cluster(bar_x, (unsigned)((T - 1) & 1), 1, T - 1);
  cluster.sync();
  if (KF > 0 && tid == 0) {  // the last CTA of the grid flips the parity for the next sweep
    __threadfence();
    if (atomicAdd(a.done_ctr, 1u) == gridDim.x - 1) {
      *a.done_ctr = 0u;
      *a.par_ctr = par ^ 1;
      __threadfence();
    }
  }
  if (a.dbg && s == 0 && tid == 0) {
    a.dbg[0] = T;
    a.dbg[1] = clock64() - t_start;
    for (int i = 0; i < 6; ++i) a.dbg[2 + i] = tm[i];
  }
}

template <int KBC, int KA, int KF>
void launch_one(cudaStream_t st, const PanelArgs& a) {
  auto kern = panel_sweep_kernel<KBC, KA, KF>;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.G * a.nclu, 1, 1);
  cfg.blockDim = dim3(panel_warps<KBC>() * 32, 1, 1);
  cfg.dynamicSmemBytes = panel_smem_bytes(a);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = a.G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, kern, a);
}

// variants: B = 512: KA in {2,4,8,12}, KF in {0,1,4}, and KA 14 with KF 0;  B = 256: KA in {4,8,12},
// KF in {0,4,8}, and KA 14 with KF 0 / 4, KA 18 with KF 0
template <int KA>
void dispatch_kf17(cudaStream_t st, const PanelArgs& a) {
  switch (a.KF) {
    case 0: launch_one<17, KA, 0>(st, a); break;
    case 1: launch_one<17, KA, 1>(st, a); break;
    case 5:
      if constexpr (KA == 8) {
        launch_one<17, 8, 5>(st, a);
        break;
      }
      [[fallthrough]];
    default: launch_one<17, KA, 4>(st, a); break;
  }
}
template <int KA>
void dispatch_kf9(cudaStream_t st, const PanelArgs& a) {
  switch (a.KF) {
    case 0: launch_one<9, KA, 0>(st, a); break;
    case 4: launch_one<9, KA, 4>(st, a); break;
    case 10:
      if constexpr (KA == 12) {
        launch_one<9, 12, 10>(st, a);
        break;
      }
      [[fallthrough]];
    default: launch_one<9, KA, 8>(st, a); break;
  }
}

template <class F>
void for_all_variants(int KBC, F&& f) {
  auto per_ka = [&](auto ka) {
    constexpr int K = decltype(ka)::value;
    if (KBC == 17) {
      f(panel_sweep_kernel<17, K, 0>);
      f(panel_sweep_kernel<17, K, 1>);
      f(panel_sweep_kernel<17, K, 4>);
    } else if (K >= 4) {
      f(panel_sweep_kernel<9, (K >= 4 ? K : 4), 0>);
      f(panel_sweep_kernel<9, (K >= 4 ? K : 4), 4>);
      f(panel_sweep_kernel<9, (K >= 4 ? K : 4), 8>);
    }
  };
  per_ka(std::integral_constant<int, 2>{});
  per_ka(std::integral_constant<int, 4>{});
  per_ka(std::integral_constant<int, 8>{});
  per_ka(std::integral_constant<int, 12>{});
  if (KBC == 17) f(panel_sweep_kernel<17, 14, 0>);  // long single-range rows (p = 8 backward: ~208 near)
  if (KBC == 17) f(panel_sweep_kernel<17, 8, 5>);   // p = 6 backward: up to 78 far entries per row
  if (KBC == 9) f(panel_sweep_kernel<9, 12, 10>);   // p = 8 backward, several ranges: 136 far entries
  if (KBC == 9) {  // small 3-D levels: interface rows with up to 279 near entries
    f(panel_sweep_kernel<9, 14, 0>);
    f(panel_sweep_kernel<9, 14, 4>);
    f(panel_sweep_kernel<9, 18, 0>);
  }
}

}  // namespace

size_t panel_smem_bytes(const PanelArgs& a) {
  const size_t W = a.KBC == 17 ? 16 : 8;
  return 8 * ((size_t)a.R + 2 * (size_t)a.B + (size_t)PANEL_STAGES * W * a.KBC * 32) + 8 * ((size_t)PANEL_STAGES + 3);
}

bool panel_prepare(int G, int KBC) {
  if (KBC != 17 && KBC != 9) return false;
  bool ok = true;
  for_all_variants(KBC, [&](auto kern) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024) != cudaSuccess)
      ok = false;
    if (G > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
      ok = false;
  });
  if (!ok) {
    cudaGetLastError();
    return false;
  }
  // can a cluster of G CTAs with (nearly) all shared memory be resident?
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G, 1, 1);
  cfg.blockDim = dim3((KBC == 17 ? 16 : 8) * 32, 1, 1);
  cfg.dynamicSmemBytes = 220 * 1024;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  cudaError_t e = KBC == 17 ? cudaOccupancyMaxActiveClusters(&nclusters, panel_sweep_kernel<17, 2, 0>, &cfg)
                            : cudaOccupancyMaxActiveClusters(&nclusters, panel_sweep_kernel<9, 4, 0>, &cfg);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return nclusters >= 1;
}

void set_carveout_panel(int pct) {
  for (int kbc : {17, 9})
    for_all_variants(kbc, [&](auto kern) { cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct); });
  cudaGetLastError();
}

int panel_max_clusters(int G, int KBC, size_t smem) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G * 8, 1, 1);
  cfg.blockDim = dim3((KBC == 17 ? 16 : 8) * 32, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclusters = 0;
  cudaError_t e = KBC == 17 ? cudaOccupancyMaxActiveClusters(&nclusters, panel_sweep_kernel<17, 2, 4>, &cfg)
                            : cudaOccupancyMaxActiveClusters(&nclusters, panel_sweep_kernel<9, 4, 8>, &cfg);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  return nclusters < 1 ? 1 : nclusters;
}

void launch_panel_sweep(cudaStream_t st, const PanelArgs& a) {
  if (a.KBC == 17) {
    switch (a.KA) {
      case 2: dispatch_kf17<2>(st, a); break;
      case 4: dispatch_kf17<4>(st, a); break;
      case 8: dispatch_kf17<8>(st, a); break;
      case 14: launch_one<17, 14, 0>(st, a); break;
      default: dispatch_kf17<12>(st, a); break;
    }
  } else {
    switch (a.KA) {
      case 4: dispatch_kf9<4>(st, a); break;
      case 8: dispatch_kf9<8>(st, a); break;
      case 14:
        if (a.KF == 0) launch_one<9, 14, 0>(st, a);
        else launch_one<9, 14, 4>(st, a);
        break;
      case 18: launch_one<9, 18, 0>(st, a); break;
      default: dispatch_kf9<12>(st, a); break;
    }
  }
}

}  // namespace igb
