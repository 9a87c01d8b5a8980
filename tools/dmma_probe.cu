// dmma_probe.cu -- fp64 throughput of mma.sync.m8n8k4.f64 (DMMA) against DFMA on sm_100a,
// per SM and whole GPU, for several warps per CTA and independent accumulator counts.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/dmma_probe.cu -o tools/dmma_probe.bin
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int ACC>
__global__ void dmma_loop(int iters, double* out, long long* cyc) {
  double c[ACC][2];
#pragma unroll
  for (int i = 0; i < ACC; ++i) c[i][0] = c[i][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-3;
  __syncthreads();
  long long t0 = clock64();
  for (int j = 0; j < iters; ++j) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) dmma(c[i][0], c[i][1], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <int ACC>
__global__ void dfma_loop(int iters, double* out, long long* cyc) {
  double c[ACC];
#pragma unroll
  for (int i = 0; i < ACC; ++i) c[i] = i;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9 * threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
  for (int j = 0; j < iters; ++j) {
#pragma unroll
    for (int i = 0; i < ACC; ++i) c[i] = fma(c[i], a, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ACC; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}

template <typename F>
static void run(const char* name, F launch, int blocks, int threads, int iters, double flop_per_thread_iter,
                double* out, long long* cyc) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch(blocks, threads, iters);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  launch(blocks, threads, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double flops = flop_per_thread_iter * iters * (double)threads * blocks;
  printf("%-10s blocks %4d threads %4d: %8.3f ms  %7.2f TF/s  %7.2f flop/clk/SM (cta0 %lld cyc)\n", name, blocks,
         threads, ms, flops / ms * 1e-9, flop_per_thread_iter * iters * threads / (double)h *
         (blocks >= 148 ? (blocks / 148) : 1), h);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 8 * 1024 * 8);
  cudaMalloc(&cyc, 64);
  const int iters = 4000;
  for (int blocks : {1, 148, 296}) {
    for (int threads : {32, 128, 256, 512}) {
      // DMMA: 256 FMA = 512 flop per warp instruction -> 16 flop per thread per DMMA
      run("dmma x1", [&](int b, int t, int it) { dmma_loop<1><<<b, t>>>(it, out, cyc); }, blocks, threads, iters, 16.0 * 1, out, cyc);
      run("dmma x4", [&](int b, int t, int it) { dmma_loop<4><<<b, t>>>(it, out, cyc); }, blocks, threads, iters, 16.0 * 4, out, cyc);
      run("dmma x9", [&](int b, int t, int it) { dmma_loop<9><<<b, t>>>(it, out, cyc); }, blocks, threads, iters, 16.0 * 9, out, cyc);
      run("dfma x8", [&](int b, int t, int it) { dfma_loop<8><<<b, t>>>(it, out, cyc); }, blocks, threads, iters, 2.0 * 8, out, cyc);
      run("dfma x16", [&](int b, int t, int it) { dfma_loop<16><<<b, t>>>(it, out, cyc); }, blocks, threads, iters, 2.0 * 16, out, cyc);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
