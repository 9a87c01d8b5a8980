// dsmem_probe.cu -- cost of cluster exchanges on B200: all-to-all of M values per CTA
// per round through st.async + mbarrier complete_tx, vs barrier.cluster.
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/dsmem_probe.cu -o tools/dsmem_probe.bin
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned saddr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(unsigned a, int r) {
  unsigned d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(r));
  return d;
}
__device__ __forceinline__ void arm(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void waitp(unsigned long long* b, unsigned par) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(saddr(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void waitp_relaxed(unsigned long long* b, unsigned par) {
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(saddr(b)), "r"(par) : "memory");
}

// MODE 5: values staged locally, __syncthreads, G threads each bulk-copy one slice
//         (cp.async.bulk shared::cta -> shared::cluster, complete_tx on the peer's mbarrier)
// MODE 0: st.async b64, MODE 1: st.async v2.b64 (16 B), MODE 2: barrier.cluster only,
// MODE 3: plain DSMEM stores + barrier.cluster, MODE 4: st.async b64 but only warp 0 waits then bar.sync
// M = values each CTA receives per round (spread over senders)
template <int MODE>
__global__ void __launch_bounds__(512, 1) probe(int rounds, int M, long long* out) {
  __shared__ __align__(16) double buf[2][1024];
  __shared__ __align__(16) double stage[2][1024];
  __shared__ unsigned long long bar[2];
  cg::cluster_group cl = cg::this_cluster();
  const int G = cl.num_blocks(), s = cl.block_rank(), tid = threadIdx.x;
  const int vals_per_msg = MODE == 1 ? 2 : 1;
  // sender slots: each CTA sends M/G values to every CTA -> M/G/vals messages per destination
  const int msgs_per_dst = M / G / vals_per_msg;
  const int nsend = msgs_per_dst * G;  // messages sent by this CTA per round
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    arm(&bar[0], 8u * M);
  }
  for (int i = tid; i < 2048; i += 512) (&buf[0][0])[i] = 0;
  cl.sync();
  const int dst = tid % G, k = tid / G;  // thread -> (destination, message index)
  const bool sender = tid < nsend;
  const unsigned rb0 = mapa(saddr(&buf[0][0]), dst), rbar0 = mapa(saddr(&bar[0]), dst);
  double v = s + 1.0;
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    const int ph = r & 1;
    if (MODE == 5) {
      // my M/G values per destination are identical for every destination here: stage M/G values once
      if (tid < M / G) stage[ph][tid] = v;
      __syncthreads();
      if (tid < G) {
        const unsigned bytes = 8u * (M / G);
        const unsigned dsto = mapa(saddr(&buf[ph][s * (M / G)]), tid);
        const unsigned dbar = mapa(saddr(&bar[0]), tid);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dsto),
                     "r"(saddr(&stage[ph][0])), "r"(bytes), "r"(dbar)
                     : "memory");
      }
      waitp(&bar[0], ph);
      if (tid == 0) arm(&bar[0], 8u * M);
      v += buf[ph][tid & 1023] * 1e-30;
    } else if (MODE <= 1 || MODE == 4) {
      if (sender) {
        const unsigned off = 8u * (ph * 1024 + (s * msgs_per_dst + k) * vals_per_msg);
        if (MODE == 1)
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(rb0 + off),
                       "d"(v), "d"(v), "r"(rbar0 + 8u * 0)
                       : "memory");
        else
          asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(rb0 + off),
                       "l"(__double_as_longlong(v)), "r"(rbar0)
                       : "memory");
      }
      if (MODE == 4) {
        if (tid < 32) waitp(&bar[0], ph);
        __syncthreads();
      } else {
        waitp(&bar[0], ph);
      }
      if (tid == 0) arm(&bar[0], 8u * M);
      v += buf[ph][tid & 1023] * 1e-30;
    } else {
      if (MODE == 3 && sender) {
        double* rb = cl.map_shared_rank(&buf[0][0], dst);
        rb[ph * 1024 + s * msgs_per_dst + k] = v;
      }
      asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
      asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
      v += buf[ph][tid & 1023] * 1e-30;
    }
  }
  long long t1 = clock64();
  if (MODE <= 1 || MODE >= 4) {
    // drain: last arm is pending, nothing more arrives; make sure no one exits early
  }
  cl.sync();
  if (s == 0 && tid == 0) out[0] = (t1 - t0) / rounds;
  if (v == -1) out[1] = 1;
}

template <int MODE>
void run(int G, int M, long long* out, const char* name) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(512);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = G;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, probe<MODE>, 2000, M, out);
  long long h = 0;
  cudaError_t e = cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
  printf("%-40s G %2d M %4d: %6lld cyc/round  %s\n", name, G, M, h, e ? cudaGetErrorString(e) : "");
}

int main() {
  long long* out;
  cudaMalloc(&out, 64);
  for (int G : {2, 4, 8, 16}) {
    run<2>(G, 16, out, "barrier.cluster only");
    run<3>(G, 512, out, "plain DSMEM stores + barrier.cluster");
    for (int M : {16, 64, 256, 512}) run<0>(G, M, out, "st.async b64 + mbarrier (all wait)");
    for (int M : {64, 512}) run<1>(G, M, out, "st.async v2.b64 + mbarrier");
    for (int M : {64, 512}) run<4>(G, M, out, "st.async b64, warp0 waits + bar.sync");
    for (int M : {64, 256, 512, 1024}) if (M / G >= 2) run<5>(G, M, out, "bulk smem->smem per destination");
  }
  return 0;
}
