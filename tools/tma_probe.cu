// tma_probe.cu -- single-CTA latency/throughput probe for the sweep design:
//  (1) cp.async.bulk (TMA) global->shared of B bytes, issue->complete latency (clock64)
//  (2) same with D copies in flight (pipelined throughput)
//  (3) cp.async.ca 8B gather latency, (4) plain ld.global latency.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/tma_probe.cu -o /tmp/tma_probe
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int MODE>
__device__ __forceinline__ void mwait(unsigned long long* b, unsigned parity) {
  if (MODE == 0) {
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}"
                 ::"r"(sa(b)), "r"(parity) : "memory");
  } else if (MODE == 1) {
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}"
                 ::"r"(sa(b)), "r"(parity) : "memory");
  } else {
    asm volatile("{\n .reg .pred p;\nW_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 20;\n @!p bra W_%=;\n}"
                 ::"r"(sa(b)), "r"(parity) : "memory");
  }
}

template <int MODE>
__global__ void probe(const unsigned char* src, long long span, int bytes, int depth, int iters,
                      long long* out, const double* gsrc) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ unsigned long long bars[16];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 16; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  unsigned phase[16] = {0};
  long long off = 0;
  // pipelined: keep `depth` copies in flight
  for (int it = 0; it < iters + depth - 1; ++it) {
    if (it < iters) {
      const int s = it % depth;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bars[s])), "r"(bytes));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(sm + (size_t)s * bytes)), "l"(src + off), "r"(bytes), "r"(sa(&bars[s])) : "memory");
      off += bytes;
      if (off + bytes > span) off = 0;
    }
    if (it >= depth - 1) {
      const int w = it - (depth - 1);
      const int s = w % depth;
      mwait<MODE>(&bars[s], phase[s]);
      phase[s] ^= 1;
    }
  }
  long long t1 = clock64();
  out[0] = (t1 - t0) / iters;
  // cp.async 8B latency (dependent chain)
  double* d = reinterpret_cast<double*>(sm);
  long long t2 = clock64();
  int idx = 0;
  for (int i = 0; i < 64; ++i) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa(d)), "l"(gsrc + idx) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    idx = ((int)d[0] + i * 4099) & ((1 << 20) - 1);
  }
  long long t3 = clock64();
  out[1] = (t3 - t2) / 64;
  // plain load chain
  long long t4 = clock64();
  idx = 0;
  double acc = 0;
  for (int i = 0; i < 64; ++i) {
    const double v = gsrc[idx];
    acc += v;
    idx = ((int)v + i * 4099 + 7) & ((1 << 20) - 1);
  }
  long long t5 = clock64();
  out[2] = (t5 - t4) / 64;
  out[3] = (long long)acc;
}

int main() {
  const long long span = 256ll << 20;
  unsigned char* src;
  double* g;
  long long* out;
  cudaMalloc(&src, span);
  cudaMemset(src, 0, span);
  cudaMalloc(&g, 8 << 20);
  cudaMemset(g, 0, 8 << 20);
  cudaMalloc(&out, 64);
  cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  const int sizes[] = {4096, 16384, 32768};
  const int depths[] = {1, 2, 4, 8};
  for (int b : sizes)
    for (int dd : depths) {
      if ((long long)b * dd > 200 * 1024) continue;
      for (int mode = 0; mode < 3; ++mode)
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) probe<0><<<1, 32, (size_t)b * dd>>>(src, span, b, dd, 200, out, g);
        if (mode == 1) probe<1><<<1, 32, (size_t)b * dd>>>(src, span, b, dd, 200, out, g);
        if (mode == 2) probe<2><<<1, 32, (size_t)b * dd>>>(src, span, b, dd, 200, out, g);
        long long h[4];
        cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
        if (rep == 1)
          printf("mode %d bulk %6d B depth %d: %6lld cyc/copy (%.1f B/cyc) | cp.async8 lat %lld | ldg lat %lld\n", mode, b, dd,
                 h[0], (double)b / h[0], h[1], h[2]);
      }
    }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
