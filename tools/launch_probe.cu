// launch_probe.cu -- per-launch cost of near-empty kernels by launch shape (stream order,
// CUDA-event timed over 200 back-to-back launches, and the same captured in a CUDA graph).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/launch_probe.cu -o tools/launch_probe.bin
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void tiny(double* out) {
  __shared__ double flag;  // static: valid for launches without dynamic shared memory
  if (threadIdx.x == 0) flag = blockIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && flag < -1) out[0] = flag;
}

float time_launches(int grid, int block, size_t smem, int cluster, bool graph) {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  double* out;
  cudaMalloc(&out, 8);
  cudaFuncSetAttribute(tiny, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(tiny, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = cluster > 0 ? 1 : 0;
  const int N = 200;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaGraphExec_t ge = nullptr;
  if (graph) {
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, tiny, out);
    if (cudaStreamEndCapture(s, &g) != cudaSuccess || cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
      printf("capture/instantiate failed: %s\n", cudaGetErrorString(cudaGetLastError()));
      return -1;
    }
    cudaGraphDestroy(g);
    cudaGraphLaunch(ge, s);
  } else {
    for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, tiny, out);
  }
  cudaStreamSynchronize(s);
  cudaEventRecord(a, s);
  if (graph) cudaGraphLaunch(ge, s);
  else
    for (int i = 0; i < N; ++i) cudaLaunchKernelEx(&cfg, tiny, out);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e) {
    printf("error %s\n", cudaGetErrorString(e));
    exit(1);
  }
  return ms * 1000 / N;
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  struct Case { int grid, block; size_t smem; int cluster; const char* name; } cases[] = {
      {4, 160, 0, 0, "4 CTAs, no smem"},
      {4, 160, 110 * 1024, 0, "4 CTAs, 110 KB smem"},
      {4, 160, 110 * 1024, 1, "4 CTAs, 110 KB, cluster 1"},
      {4, 160, 0, 1, "4 CTAs, no smem, cluster 1"},
      {60, 160, 110 * 1024, 15, "60 CTAs, 110 KB, cluster 15"},
      {16, 512, 210 * 1024, 16, "16 CTAs, 213 KB, cluster 16"},
      {16, 512, 0, 16, "16 CTAs, no smem, cluster 16"},
      {148, 256, 0, 0, "148 CTAs, no smem"},
  };
  for (bool graph : {false, true})
    for (auto& c : cases)
      printf("%-6s %-34s %7.2f us/launch\n", graph ? "graph" : "stream", c.name,
             time_launches(c.grid, c.block, c.smem, c.cluster, graph));
  return 0;
}
