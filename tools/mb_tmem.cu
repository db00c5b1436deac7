// mb_tmem.cu — probe: can a TMA-filled record ring be moved smem -> TMEM with tcgen05.cp
// (128x128b: one 16-B record per TMEM lane) and read back with tcgen05.ld.32x32b.x4?
// Checks the layout (record r of a 128-record block -> lane r, 4 consecutive columns) and
// times the smem->TMEM->register path against plain LDS.128.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mb_tmem tools/mb_tmem.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor, SWIZZLE_NONE, K-major: core matrix = 8 rows x 16 B (128 B
// contiguous); SBO = byte distance between core matrices along M (here 128 B: the next 8
// records), LBO unused for a 16-B-wide matrix; version 1 (bits 46-47) for sm_100.
__device__ __forceinline__ uint64_t desc_none(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  return d;
}

__global__ void __launch_bounds__(128) k_probe(uint32_t *out, int sbo, int lbo, int reps, long long *cyc) {
  __shared__ __align__(1024) uint4 buf[128 * 16];
  __shared__ uint32_t taddr_s;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  for (int i = t; i < 128 * 16; i += 128) buf[i] = make_uint4(i, i + 100000, i + 200000, i + 300000);
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t taddr = taddr_s;
  // 16 blocks of 128 records -> columns 4b..4b+3
  if (t == 0) {
    for (int b = 0; b < 16; b++) {
      uint64_t d = desc_none(smem_u32(buf + b * 128), lbo, sbo);
      asm volatile("tcgen05.cp.cta_group::1.128x128b [%0], %1;" ::"r"(taddr + 4 * b), "l"(d));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(
          smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int b = 0; b < 16; b++) {
    uint32_t r0, r1, r2, r3;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(taddr + ((uint32_t)(32 * w) << 16) + 4 * b));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    int rec = b * 128 + 32 * w + lane;
    out[rec * 4 + 0] = r0; out[rec * 4 + 1] = r1; out[rec * 4 + 2] = r2; out[rec * 4 + 3] = r3;
  }
  // timing: repeated TMEM loads of 16 blocks vs LDS.128 of the same records
  long long c0 = clock64();
  uint32_t acc = 0;
  for (int k = 0; k < reps; k++)
    for (int b = 0; b < 16; b++) {
      uint32_t r0, r1, r2, r3;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                   : "r"(taddr + ((uint32_t)(32 * w) << 16) + 4 * b));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc += r0 ^ r1 ^ r2 ^ r3;
    }
  long long c1 = clock64();
  for (int k = 0; k < reps; k++)
    for (int b = 0; b < 16; b++) {
      uint32_t x, y, z, q;
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(x), "=r"(y), "=r"(z), "=r"(q)
                   : "r"(smem_u32(&buf[b * 128 + 32 * w + lane])));
      acc += x ^ y ^ z ^ q;
    }
  long long c2 = clock64();
  if (t == 0) { cyc[0] = c1 - c0; cyc[1] = c2 - c1; }
  if (acc == 0x12345678) out[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(taddr));
}

int main() {
  uint32_t *d_out; long long *d_cyc;
  cudaMalloc(&d_out, 2048 * 16); cudaMalloc(&d_cyc, 16);
  static uint32_t h[2048 * 4];
  int cfgs[][2] = {{128, 0}, {128, 2048}, {128, 128}, {2048, 128}};
  for (auto &c : cfgs) {
    cudaMemset(d_out, 0xFF, 2048 * 16);
    k_probe<<<1, 128>>>(d_out, c[0], c[1], 1000, d_cyc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("sbo=%d lbo=%d: %s\n", c[0], c[1], cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    long long cy[2]; cudaMemcpy(cy, d_cyc, 16, cudaMemcpyDeviceToHost);
    int bad = 0, first = -1;
    for (int r = 0; r < 2048; r++)
      if (h[r * 4] != (uint32_t)r || h[r * 4 + 1] != (uint32_t)r + 100000 || h[r * 4 + 2] != (uint32_t)r + 200000 ||
          h[r * 4 + 3] != (uint32_t)r + 300000) { bad++; if (first < 0) first = r; }
    printf("sbo=%d lbo=%d: %d/2048 records wrong (first %d: %u %u %u %u); cycles per 16-block pass: tmem %.1f lds %.1f\n",
           c[0], c[1], bad, first, first >= 0 ? h[first * 4] : 0, first >= 0 ? h[first * 4 + 1] : 0,
           first >= 0 ? h[first * 4 + 2] : 0, first >= 0 ? h[first * 4 + 3] : 0, cy[0] / 1000.0, cy[1] / 1000.0);
  }
  return 0;
}
