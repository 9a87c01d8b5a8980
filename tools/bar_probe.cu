// bar_probe.cu -- cycles per iteration of {smem RMW; __syncthreads} loops, one CTA.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/bar_probe.cu -o tools/bar_probe.bin
#include <cstdio>
#include <cuda_runtime.h>

__global__ void bar_loop(int iters, long long* out, int mode) {
  __shared__ double y[4096];
  const int tid = threadIdx.x;
  for (int i = tid; i < 4096; i += blockDim.x) y[i] = i;
  __syncthreads();
  long long t0 = clock64();
  double acc = 0;
  for (int j = 0; j < iters; ++j) {
    if (mode >= 1) {
      const double yj = y[j & 4095];
      const int r = (tid * 7 + j) & 4095;
      if (mode == 1) y[r] = y[r] - 0.5 * yj;
      else y[r] = __dsub_rn(y[r], __dmul_rn(0.5, yj));
      acc += yj;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) { out[0] = (t1 - t0) / iters; out[1] = (long long)acc; }
}

__global__ void ddiv_loop(int iters, long long* out, double d) {
  long long t0 = clock64();
  double v = 1.2345;
  for (int j = 0; j < iters; ++j) v = __ddiv_rn(v + 1.0, d);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = (t1 - t0) / iters; out[1] = (long long)v; }
}

int main() {
  long long* out;
  cudaMalloc(&out, 64);
  const int threads[] = {32, 96, 128, 256, 1024};
  for (int mode = 0; mode < 3; ++mode)
    for (int nt : threads) {
      bar_loop<<<1, nt>>>(2000, out, mode);
      long long h[2];
      cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
      printf("mode %d threads %4d: %lld cyc/iter\n", mode, nt, h[0]);
    }
  ddiv_loop<<<1, 32>>>(2000, out, 3.0);
  long long h[2];
  cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  printf("dependent __ddiv_rn: %lld cyc\n", h[0]);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
