// DSMEM atomic throughput probe: random u32 atomic adds into the distributed shared memory
// of a thread-block cluster (remote ranks via mapa / atom.shared::cluster).
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int LOCAL_ONLY>
__global__ void k_dsmem(uint32_t *out, uint32_t sbins, uint64_t ops_per_thread) {
  extern __shared__ __align__(16) uint32_t tab[];
  cg::cluster_group cl = cg::this_cluster();
  for (uint32_t i = threadIdx.x; i < sbins; i += blockDim.x) tab[i] = 0;
  cl.sync();
  uint32_t nr = cl.num_blocks();
  uint32_t base = (uint32_t)__cvta_generic_to_shared(tab);
  uint32_t x = hash32(threadIdx.x + blockIdx.x * blockDim.x);
  for (uint64_t k = 0; k < ops_per_thread; k++) {
    x = hash32(x + (uint32_t)k);
    uint32_t rank = LOCAL_ONLY ? cl.block_rank() : (x >> 24) % nr;
    uint32_t a = base + 4 * ((x & 0xFFFFFF) % sbins), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    asm volatile("red.shared::cluster.add.u32 [%0], %1;" ::"r"(ra), "r"(1u) : "memory");
  }
  cl.sync();
  for (uint32_t i = threadIdx.x; i < sbins; i += blockDim.x) if (tab[i] == 12345678) out[0] = 1;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *out; cudaMalloc(&out, 4);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int thr = 512; const uint64_t per = 4096; const uint32_t sbins = 40000; size_t smem = sbins * 4;
  int csv[] = {1, 2, 4, 8, 16};
  for (int cs : csv) {
    for (int local = 0; local < 2; local++) {
      auto kern = local ? k_dsmem<1> : k_dsmem<0>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (cs > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      int blocks = (sms / cs) * cs;
      cfg.gridDim = dim3(blocks); cfg.blockDim = dim3(thr); cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      float ms = 0;
      for (int w = 0; w < 2; w++) {
        cudaEventRecord(a);
        cudaError_t e = cudaLaunchKernelEx(&cfg, kern, out, sbins, per);
        cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
        if (e != cudaSuccess) { printf("cs=%d launch: %s\n", cs, cudaGetErrorString(e)); break; }
      }
      cudaError_t e = cudaGetLastError();
      printf("cluster %2d %s: blocks %d  %.3f Gop/s  (%s)\n", cs, local ? "local " : "remote", blocks,
             (double)blocks * thr * per / ms / 1e6, cudaGetErrorString(e));
    }
  }
  return 0;
}
