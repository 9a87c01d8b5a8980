// lat_probe.cu -- dependent-chain latency of fp64 ops and LDS on sm_100a (one warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(long long* out, double a, int n) {
  __shared__ double sm[1024];
  for (int i = threadIdx.x; i < 1024; i += 32) sm[i] = (i % 7) * 1e-30;
  __syncwarp();
  double x = a, y = a * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, 1.0000001, y);
  long long t1 = clock64();
  double z = a;
  for (int i = 0; i < n; ++i) z = z + 1.0000001;
  long long t2 = clock64();
  double w = a;
  int idx = 0;
  for (int i = 0; i < n; ++i) { w = fma(w, 1.0, sm[idx]); idx = (int)(sm[idx] * 1e30) & 1023; }
  long long t3 = clock64();
  float f = (float)a;
  for (int i = 0; i < n; ++i) f = fmaf(f, 1.0000001f, 0.5f);
  long long t4 = clock64();
  out[0] = (t1 - t0) / n; out[1] = (t2 - t1) / n; out[2] = (t3 - t2) / n; out[3] = (t4 - t3) / n;
  out[4] = (long long)(x + z + w + f);
}
int main() {
  long long* d; cudaMalloc(&d, 64); long long h[5];
  lat<<<1, 32>>>(d, 1.5, 4000); lat<<<1, 32>>>(d, 1.5, 4000);
  cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
  printf("DFMA chain %lld cyc/op | DADD chain %lld | LDS->DFMA->idx chain %lld | FFMA chain %lld\n", h[0], h[1], h[2], h[3]);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
