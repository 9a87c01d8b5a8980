// tma_bw_probe.cu -- TMA bulk-copy bandwidth (global -> shared) per SM, for CTAs inside one
// thread-block cluster (one GPC) vs spread over the device, and for plain coalesced loads.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/tma_bw_probe.cu -o tools/tma_bw_probe.bin
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// each CTA streams `iters` chunks of `chunk` bytes (distinct addresses), S stages
__global__ void __launch_bounds__(512, 1) tma_bw(const char* src, size_t span, int chunk, int iters, int nsplit,
                                                 long long* out) {
  extern __shared__ __align__(128) char sm[];
  __shared__ unsigned long long bar[2];
  const int tid = threadIdx.x;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const size_t base = (size_t)blockIdx.x * iters * chunk;
  auto issue = [&](int it) {
    const int st = it & 1;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&bar[st])), "r"(chunk) : "memory");
    const int part = chunk / nsplit;
    for (int p = 0; p < nsplit; ++p) {
      const char* g = src + (base + (size_t)it * chunk + (size_t)p * part) % span;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              saddr(sm + st * chunk + p * part)),
          "l"(g), "r"(part), "r"(saddr(&bar[st]))
          : "memory");
    }
  };
  long long t0 = clock64();
  if (tid == 0) issue(0);
  for (int it = 0; it < iters; ++it) {
    if (tid == 0 && it + 1 < iters) issue(it + 1);
    const unsigned par = (it >> 1) & 1;
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                     saddr(&bar[it & 1])),
                 "r"(par)
                 : "memory");
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
}

// plain coalesced loads (each warp 16B/lane), summed to defeat DCE
__global__ void __launch_bounds__(512, 1) ldg_bw(const double2* src, size_t span16, int chunk, int iters,
                                                 long long* out, double* sink) {
  const int tid = threadIdx.x;
  const size_t base = (size_t)blockIdx.x * iters * (chunk / 16);
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const size_t o = base + (size_t)it * (chunk / 16);
    for (int k = tid; k < chunk / 16; k += 512) {
      const double2 v = __ldcs(src + (o + k) % span16);
      acc += v.x + v.y;
    }
  }
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345.678) sink[0] = acc;
}

void run(bool cluster, int nblk, int chunk, int nsplit, const char* src, size_t span, long long* out,
         long long* hout) {
  const int iters = 200;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nblk);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = 2 * chunk;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = nblk;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = cluster ? 1 : 0;
  cudaFuncSetAttribute(tma_bw, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(tma_bw, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * chunk);
  for (int r = 0; r < 2; ++r) cudaLaunchKernelEx(&cfg, tma_bw, src, span, chunk, iters, nsplit, out);
  cudaError_t e = cudaMemcpy(hout, out, nblk * 8, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < nblk; ++i) mx = hout[i] > mx ? hout[i] : mx;
  printf("TMA %-8s ctas %3d chunk %6d split %d: %6.1f B/clk per SM, %7.1f B/clk total %s\n", cluster ? "cluster" : "spread",
         nblk, chunk, nsplit, (double)chunk * iters / mx, (double)chunk * iters * nblk / mx, e ? cudaGetErrorString(e) : "");
}

int main() {
  const size_t span = (size_t)2 << 30;  // 2 GiB: beyond L2
  char* src;
  cudaMalloc(&src, span);
  cudaMemset(src, 1, span);
  long long* out;
  cudaMalloc(&out, 1024 * 8);
  long long hout[1024];
  double* sink;
  cudaMalloc(&sink, 8);
  for (int chunk : {16384, 65536})
    for (int nsplit : {1, 4}) {
      run(true, 16, chunk, nsplit, src, span, out, hout);
      run(false, 16, chunk, nsplit, src, span, out, hout);
      run(true, 8, chunk, nsplit, src, span, out, hout);
      run(false, 1, chunk, nsplit, src, span, out, hout);
      run(false, 148, chunk, nsplit, src, span, out, hout);
    }
  for (int nblk : {1, 16, 148}) {
    const int chunk = 65536, iters = 200;
    for (int r = 0; r < 2; ++r)
      ldg_bw<<<nblk, 512>>>((const double2*)src, span / 16, chunk, iters, out, sink);
    cudaMemcpy(hout, out, nblk * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < nblk; ++i) mx = hout[i] > mx ? hout[i] : mx;
    printf("LDG.128 spread ctas %3d: %6.1f B/clk per SM, %7.1f total\n", nblk, (double)chunk * iters / mx,
           (double)chunk * iters * nblk / mx);
  }
  return 0;
}
