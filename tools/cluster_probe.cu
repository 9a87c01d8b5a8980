// cluster_probe.cu -- cycles per iteration of {DSMEM broadcast store; cluster barrier} on sm_100a.
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

template <int MODE>
__global__ void __cluster_dims__(1, 1, 1) dummy() {}

template <int MODE>
__global__ void loop(int iters, long long* out) {
  __shared__ double ring[1024];
  auto cl = cg::this_cluster();
  const int n = cl.num_blocks();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) ring[i] = 0;
  double* peers[8];
  for (int r = 0; r < 8; ++r) peers[r] = r < n ? cl.map_shared_rank(ring, r) : ring;
  cl.sync();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE >= 1 && threadIdx.x < 64) {
      const double v = ring[(threadIdx.x + it) & 1023] + 1.0;
      for (int r = 0; r < n; ++r) peers[r][(threadIdx.x * 7 + it) & 1023] = v;
    }
    if (MODE == 2) {
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    } else if (MODE == 3) {
      asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    } else {
      cl.sync();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = (t1 - t0) / iters;
}

template <int MODE>
void run(int cs, long long* d, const char* name) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = 0;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr; cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, loop<MODE>, 2000, d);
  cudaLaunchKernelEx(&cfg, loop<MODE>, 2000, d);
  long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-40s cluster %d: %lld cyc/iter (%s)\n", name, cs, h, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  for (int cs : {1, 2, 4, 8}) {
    run<0>(cs, d, "cg cluster.sync only");
    run<1>(cs, d, "DSMEM broadcast + cg cluster.sync");
    run<2>(cs, d, "DSMEM broadcast + arrive.release/wait.acq");
    run<3>(cs, d, "DSMEM broadcast + arrive.relaxed/wait");
  }
  return 0;
}
