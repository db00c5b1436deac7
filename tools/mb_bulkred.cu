// Probe: throughput of 1-D TMA bulk reductions (cp.reduce.async.bulk .add.u64, 16 B each) at
// random 16-B-aligned global addresses, issued per lane, vs plain red.global.add.u64.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

template <int LANES>
__global__ void k_bulk(unsigned long long *h, uint32_t rows, uint64_t ops_per_thread) {
  __shared__ __align__(16) unsigned long long buf[1024 * 2];
  buf[2 * threadIdx.x] = 1;
  buf[2 * threadIdx.x + 1] = 0;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  uint32_t s = (uint32_t)__cvta_generic_to_shared(buf + 2 * threadIdx.x);
  uint32_t x = hash32(threadIdx.x + blockIdx.x * 977);
  int lane = threadIdx.x & 31;
  for (uint64_t k = 0; k < ops_per_thread; k++) {
    x = hash32(x + (uint32_t)k);
    if (lane < LANES) {
      unsigned long long *g = h + 2ull * (x % rows);
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], 16;" ::"l"(g), "r"(s) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if ((k & 7) == 7) asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void k_red(unsigned long long *h, uint32_t rows, uint64_t ops_per_thread) {
  uint32_t x = hash32(threadIdx.x + blockIdx.x * 977);
  for (uint64_t k = 0; k < ops_per_thread; k++) {
    x = hash32(x + (uint32_t)k);
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(h + 2ull * (x % rows)), "l"(1ull));
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *h; cudaMalloc(&h, 64ull << 20); cudaMemset(h, 0, 64ull << 20);
  uint32_t rows = (64u << 20) / 16;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int thr : {256, 1024}) {
    uint64_t per = 2048;
    for (int w = 0; w < 2; w++) { cudaEventRecord(a); k_bulk<32><<<sms, thr>>>(h, rows, per); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b);
    printf("bulk red 16B, 32 lanes/warp, %4d thr/CTA: %.3f Gop/s  (%s)\n", thr, (double)sms * thr * per / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    for (int w = 0; w < 2; w++) { cudaEventRecord(a); k_bulk<1><<<sms, thr>>>(h, rows, per); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b);
    printf("bulk red 16B, 1 lane/warp,  %4d thr/CTA: %.3f Gop/s\n", thr, (double)sms * (thr / 32) * per / ms / 1e6);
    for (int w = 0; w < 2; w++) { cudaEventRecord(a); k_red<<<sms, thr>>>(h, rows, per); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b);
    printf("red.global u64,             %4d thr/CTA: %.3f Gop/s\n", thr, (double)sms * thr * per / ms / 1e6);
  }
  return 0;
}
