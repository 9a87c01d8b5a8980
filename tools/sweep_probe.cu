// sweep_probe.cu -- isolate the per-step cost of the level-sweep structure.
// Synthetic: T steps, NT threads, TPR threads/row, KMAX entries/thread, loads from a
// stream in the same interleaved layout, ring in smem, barrier per step.
// MODE bits: 1 = loads, 2 = dot, 4 = shuffle+store, 8 = 4-set rotation (else 1 set, no prefetch)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/sweep_probe.cu -o tools/sweep_probe.bin
#include <cstdio>
#include <cuda_runtime.h>

constexpr int NT = 384, KMAX = 8;
struct Set { double v[KMAX]; int c[KMAX]; double b, invd; };

template <int MODE, int TPR>
__global__ void __launch_bounds__(NT) probe(const double2* vs, const int2* cs, const double* rp, double* xp,
                                            int T, int nrows, long long* out) {
  __shared__ double ring[4096];
  const int tid = threadIdx.x, rho = tid / TPR, tau = tid % TPR;
  for (int i = tid; i < 4096; i += NT) ring[i] = 0.0;
  __syncthreads();
  const int nthr = nrows * TPR;
  const long long step_elems = (long long)nthr * (KMAX / 2);
  auto load = [&](Set& S, int t) {
    if (!(MODE & 1) || tid >= nthr) return;
    const double2* v2 = vs + (long long)t * step_elems + tid;
    const int2* c2 = cs + (long long)t * step_elems + tid;
#pragma unroll
    for (int j = 0; j < KMAX / 2; ++j) {
      const double2 a = __ldg(v2 + j * nthr);
      const int2 b = __ldg(c2 + j * nthr);
      S.v[2 * j] = a.x; S.v[2 * j + 1] = a.y; S.c[2 * j] = b.x; S.c[2 * j + 1] = b.y;
    }
    S.b = __ldg(rp + (long long)t * nrows + rho);
    S.invd = 0.5;
  };
  auto compute = [&](const Set& S, int t) {
    double s0 = 0, s1 = 0;
    double s;
    if ((MODE & 16) && rho < nrows) {  // tree: all products independent
      double p[KMAX];
#pragma unroll
      for (int k = 0; k < KMAX; ++k) p[k] = S.v[k] * ring[S.c[k] & 4095];
#pragma unroll
      for (int w = KMAX / 2; w > 0; w >>= 1)
#pragma unroll
        for (int k = 0; k < w; ++k) p[k] += p[k + w];
      s = p[0];
    } else {
      if ((MODE & 2) && rho < nrows) {
#pragma unroll
        for (int k = 0; k < KMAX; k += 2) {
          s0 = fma(S.v[k], ring[S.c[k] & 4095], s0);
          s1 = fma(S.v[k + 1], ring[S.c[k + 1] & 4095], s1);
        }
      }
      s = s0 + s1;
    }
    if (MODE & 4) {
      for (int o = TPR >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (tau == 0 && rho < nrows) {
        const double xi = (S.b - s) * S.invd;
        ring[(t * nrows + rho) & 4095] = xi;
        xp[(long long)t * nrows + rho] = xi;
      }
    }
  };
  Set A, B, C, D;
  for (int k = 0; k < KMAX; ++k) { A.v[k] = B.v[k] = C.v[k] = D.v[k] = 0; A.c[k] = B.c[k] = C.c[k] = D.c[k] = k; }
  A.b = B.b = C.b = D.b = A.invd = B.invd = C.invd = D.invd = 0;
  long long t0 = clock64();
  if (MODE & 8) {
    load(A, 0); load(B, 1); load(C, 2);
    for (int t = 0; t < T; t += 4) {
      load(D, t + 3); __syncthreads(); compute(A, t);
      load(A, t + 4); __syncthreads(); compute(B, t + 1);
      load(B, t + 5); __syncthreads(); compute(C, t + 2);
      load(C, t + 6); __syncthreads(); compute(D, t + 3);
    }
  } else {
    for (int t = 0; t < T; ++t) {
      load(A, t); __syncthreads(); compute(A, t);
    }
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / T;
}

template <int MODE, int TPR>
void run(const double2* vs, const int2* cs, const double* rp, double* xp, int T, int nrows, long long* out,
         const char* name) {
  probe<MODE, TPR><<<1, NT>>>(vs, cs, rp, xp, T, nrows, out);
  probe<MODE, TPR><<<1, NT>>>(vs, cs, rp, xp, T, nrows, out);
  long long h;
  cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("%-34s TPR %d rows %3d: %5lld cyc/step\n", name, TPR, nrows, h);
}

__global__ void lat(long long* out, double a, float af) {
  double x = a, y = a * 0.5;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { x = fma(x, 1.0000001, y); }
  long long t1 = clock64();
  double z = a;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { z = z + 1.0000001; }
  long long t2 = clock64();
  float f = af;
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { f = fmaf(f, 1.0000001f, 0.5f); }
  long long t3 = clock64();
  out[0] = (t1 - t0) / 1000; out[1] = (t2 - t1) / 1000; out[2] = (t3 - t2) / 1000;
  out[3] = (long long)(x + z + f);
}

// Early/late split: warps 0..LW-1 own rows (late part: 2 entries + partial from smem),
// the other warps compute the early partial sums of the next step into smem.
template <int TPR>
__global__ void __launch_bounds__(NT) probe_split(const double2* vs, const int2* cs, const double* rp, double* xp,
                                                  int T, int nrows, long long* out) {
  __shared__ double ring[4096];
  __shared__ double part[2][256];
  const int tid = threadIdx.x;
  for (int i = tid; i < 4096; i += NT) ring[i] = 0.0;
  for (int i = tid; i < 512; i += NT) (&part[0][0])[i] = 0.0;
  __syncthreads();
  const int nthr = nrows * TPR;            // early-part threads (helpers), TPR per row
  const bool helper = tid >= 128 && tid - 128 < nthr;
  const int htid = tid - 128, hrho = htid / TPR, htau = htid % TPR;
  const bool owner = tid < nrows;          // late part: one thread per row
  const long long step_elems = (long long)nthr * (KMAX / 2);
  Set A, B;
  for (int k = 0; k < KMAX; ++k) { A.v[k] = B.v[k] = 0; A.c[k] = B.c[k] = k; }
  A.b = B.b = 0; A.invd = B.invd = 0.5;
  auto load = [&](Set& S, int t) {
    if (!helper) return;
    const double2* v2 = vs + (long long)t * step_elems + htid;
    const int2* c2 = cs + (long long)t * step_elems + htid;
#pragma unroll
    for (int j = 0; j < KMAX / 2; ++j) {
      const double2 a = __ldg(v2 + j * nthr);
      const int2 b = __ldg(c2 + j * nthr);
      S.v[2 * j] = a.x; S.v[2 * j + 1] = a.y; S.c[2 * j] = b.x; S.c[2 * j + 1] = b.y;
    }
  };
  double lv0 = 0.1, lv1 = 0.2, b = 0.0;
  long long t0 = clock64();
  load(A, 0);
  for (int t = 0; t < T; t += 2) {
    // helpers: early part of step t+1 (uses ring values of steps <= t-1)
    load(B, t + 1);
    {
      double s0 = 0, s1 = 0;
      if (helper) {
#pragma unroll
        for (int k = 0; k < KMAX; k += 2) { s0 = fma(A.v[k], ring[A.c[k] & 4095], s0); s1 = fma(A.v[k + 1], ring[A.c[k + 1] & 4095], s1); }
      }
      double s = s0 + s1;
      for (int o = TPR >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (helper && htau == 0) part[(t + 1) & 1][hrho] = s;
    }
    if (owner) {  // late part of step t: 2 entries from the previous step + partial
      const double xi = (b - part[t & 1][tid] - lv0 * ring[(tid + 3) & 4095] - lv1 * ring[(tid + 5) & 4095]) * 0.5;
      ring[(t * nrows + tid) & 4095] = xi;
      xp[(long long)t * nrows + tid] = xi;
    }
    __syncthreads();
    load(A, t + 2);
    {
      double s0 = 0, s1 = 0;
      if (helper) {
#pragma unroll
        for (int k = 0; k < KMAX; k += 2) { s0 = fma(B.v[k], ring[B.c[k] & 4095], s0); s1 = fma(B.v[k + 1], ring[B.c[k + 1] & 4095], s1); }
      }
      double s = s0 + s1;
      for (int o = TPR >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (helper && htau == 0) part[t & 1][hrho] = s;
    }
    if (owner) {
      const double xi = (b - part[(t + 1) & 1][tid] - lv0 * ring[(tid + 3) & 4095] - lv1 * ring[(tid + 5) & 4095]) * 0.5;
      ring[((t + 1) * nrows + tid) & 4095] = xi;
      xp[(long long)(t + 1) * nrows + tid] = xi;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / T;
}

int main() {
  const int T = 1300, nrows = 52;
  const long long elems = (long long)(T + 8) * nrows * 8 * (KMAX / 2);
  double2* vs; int2* cs; double* rp; double* xp; long long* out;
  cudaMalloc(&vs, elems * 16); cudaMalloc(&cs, elems * 8);
  cudaMalloc(&rp, (T + 8) * 256 * 8); cudaMalloc(&xp, (T + 8) * 256 * 8); cudaMalloc(&out, 64);
  cudaMemset(vs, 0, elems * 16); cudaMemset(cs, 0, elems * 8); cudaMemset(rp, 0, (T + 8) * 256 * 8);
  {
    lat<<<1, 32>>>(out, 1.5, 1.5f);
    long long h[4];
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    printf("dependent DFMA %lld cyc, DADD %lld cyc, FFMA %lld cyc (incl. loop overhead)\n", h[0], h[1], h[2]);
  }
  {
    probe_split<4><<<1, NT>>>(vs, cs, rp, xp, T, nrows, out);
    probe_split<4><<<1, NT>>>(vs, cs, rp, xp, T, nrows, out);
    long long h;
    cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
    printf("early/late split (helpers 6 warps, 1-set loads) rows 52: %lld cyc/step\n", h);
  }
  run<0, 4>(vs, cs, rp, xp, T, nrows, out, "barrier only");
  run<22, 4>(vs, cs, rp, xp, T, nrows, out, "tree-dot+shfl+store");
  run<31, 4>(vs, cs, rp, xp, T, nrows, out, "loads(4 sets)+tree-dot+shfl+store");
  run<4, 4>(vs, cs, rp, xp, T, nrows, out, "shfl+store");
  run<6, 4>(vs, cs, rp, xp, T, nrows, out, "dot+shfl+store");
  run<7, 4>(vs, cs, rp, xp, T, nrows, out, "loads(1 set)+dot+shfl+store");
  run<15, 4>(vs, cs, rp, xp, T, nrows, out, "loads(4 sets)+dot+shfl+store");
  run<9, 4>(vs, cs, rp, xp, T, nrows, out, "loads(4 sets) only");
  run<15, 2>(vs, cs, rp, xp, T, nrows, out, "loads(4 sets)+dot+shfl+store");
  run<15, 8>(vs, cs, rp, xp, T, 40, out, "loads(4 sets)+dot+shfl+store");
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
