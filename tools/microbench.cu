// microbench.cu — throughput probes that decide the attribution kernel's design (not part of
// the product).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb tools/microbench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

// 1) REDG u64 / u32 at pseudo-random addresses within `bins`
template <typename T>
__global__ void k_redg(T *h, uint32_t bins, uint64_t ops, uint32_t seed) {
  uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k = tid; k < ops; k += nt) {
    uint32_t a = hash32((uint32_t)k ^ seed) % bins;
    atomicAdd(h + a, (T)1);
  }
}
// 2) ATOMS u32 / u64 at pseudo-random addresses within a smem table of `sbins` entries
template <typename T>
__global__ void k_atoms(T *out, uint32_t sbins, uint64_t ops_per_thread, uint32_t seed) {
  extern __shared__ __align__(16) uint8_t sm[];
  T *tab = reinterpret_cast<T *>(sm);
  for (uint32_t i = threadIdx.x; i < sbins; i += blockDim.x) tab[i] = 0;
  __syncthreads();
  uint32_t x = hash32(threadIdx.x + blockIdx.x * blockDim.x + seed);
  for (uint64_t k = 0; k < ops_per_thread; k++) {
    x = hash32(x + (uint32_t)k);
    atomicAdd(tab + (x % sbins), (T)1);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < sbins; i += blockDim.x) if (tab[i] == 12345678) out[0] = 1;
}
// 3) streaming read of 16-B records, trivial use
__global__ void k_stream(const uint4 *p, uint64_t n, uint32_t *out) {
  uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t k = tid; k < n; k += nt) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + k));
    acc ^= v.x + v.w;
  }
  if (acc == 0x12345678) out[0] = acc;
}
// 4) streaming read + a dependent gather into a `gbins`-entry table (the granule map)
__global__ void k_stream_gather(const uint4 *p, uint64_t n, const uint32_t *g, uint32_t gbins, uint32_t *out) {
  uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t k = tid; k < n; k += nt) {
    uint4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p + k));
    acc ^= __ldg(g + (v.x % gbins));
  }
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  const uint64_t OPS = 1ull << 30;
  unsigned long long *h64; uint32_t *h32;
  CK(cudaMalloc(&h64, 8ull << 23)); CK(cudaMalloc(&h32, 4ull << 23));
  uint32_t binsv[] = {1u << 10, 1u << 14, 1u << 17, 6u << 20, 8u << 20};
  for (uint32_t bins : binsv) {
    for (int w = 0; w < 2; w++) {
      cudaEventRecord(a);
      k_redg<unsigned long long><<<sms * 8, 256>>>(h64, bins, OPS, 7);
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    }
    printf("REDG u64 bins=%8u : %.3f Gop/s\n", bins, OPS / ms / 1e6);
    cudaEventRecord(a);
    k_redg<unsigned int><<<sms * 8, 256>>>(h32, bins, OPS, 7);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("REDG u32 bins=%8u : %.3f Gop/s\n", bins, OPS / ms / 1e6);
  }
  uint32_t sbinsv[] = {1024, 8192, 24576};
  for (uint32_t sb : sbinsv) {
    uint64_t per = 1 << 12;
    int thr = 512;
    size_t sm32 = sb * 4, sm64 = sb * 8;
    CK(cudaFuncSetAttribute(k_atoms<unsigned int>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000));
    CK(cudaFuncSetAttribute(k_atoms<unsigned long long>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000));
    for (int w = 0; w < 2; w++) {
      cudaEventRecord(a);
      k_atoms<unsigned int><<<sms * 2, thr, sm32>>>(h32, sb, per, 3);
      cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    }
    printf("ATOMS u32 sbins=%6u : %.3f Gop/s\n", sb, (double)sms * 2 * thr * per / ms / 1e6);
    cudaEventRecord(a);
    k_atoms<unsigned long long><<<sms * 2, thr, sm64>>>((unsigned long long *)h64, sb, per, 3);
    cudaEventRecord(b); cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
    printf("ATOMS u64 sbins=%6u : %.3f Gop/s\n", sb, (double)sms * 2 * thr * per / ms / 1e6);
    CK(cudaGetLastError());
  }
  uint64_t n = 1ull << 31;  // 32 GB of 16-B records
  uint4 *rec; CK(cudaMalloc(&rec, n * 16)); CK(cudaMemset(rec, 1, n * 16));
  uint32_t *g; CK(cudaMalloc(&g, 4u << 20)); CK(cudaMemset(g, 0, 4u << 20));
  for (int w = 0; w < 2; w++) {
    cudaEventRecord(a); k_stream<<<sms * 8, 256>>>(rec, n, h32); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  }
  printf("stream 16B records: %.1f GB/s\n", n * 16 / ms / 1e6);
  for (int w = 0; w < 2; w++) {
    cudaEventRecord(a); k_stream_gather<<<sms * 8, 256>>>(rec, n, g, 1u << 19, h32); cudaEventRecord(b);
    cudaEventSynchronize(b); cudaEventElapsedTime(&ms, a, b);
  }
  printf("stream + gather(2MB table): %.1f GB/s\n", n * 16 / ms / 1e6);
  CK(cudaGetLastError());
  return 0;
}
