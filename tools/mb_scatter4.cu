// Probe: TMA reduce-scatter of 4 rows (cp.reduce.async.bulk.tensor.2d ... add.tile::scatter4)
// into a u64 [rows][16] tensor, 16-B boxes (2 slots) per row, random rows.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}

__global__ void k_s4(const __grid_constant__ CUtensorMap tm, uint32_t rows, uint64_t ops, int lanes) {
  __shared__ __align__(128) unsigned long long buf[256 * 16];
  unsigned long long *my = buf + 16 * threadIdx.x;  // 4 rows x 2 u64, 128-B aligned
  for (int q = 0; q < 8; q++) my[q] = (q & 1) ? 0 : 1;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  uint32_t s = (uint32_t)__cvta_generic_to_shared(my);
  uint32_t x = hash32(threadIdx.x + blockIdx.x * 977);
  int lane = threadIdx.x & 31;
  for (uint64_t k = 0; k < ops; k++) {
    x = hash32(x + (uint32_t)k);
    if (lane < lanes) {
      int col = 2 * (x & 7);
      int r0 = x % rows, r1 = (x * 3) % rows, r2 = (x * 7) % rows, r3 = (x * 13) % rows;
      asm volatile(
          "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile::scatter4.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];"
          ::"l"(&tm), "r"(col), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(s) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    if ((k & 7) == 7) asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t rows = 500000;
  unsigned long long *h; cudaMalloc(&h, (size_t)rows * 128); cudaMemset(h, 0, (size_t)rows * 128);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
  if (!enc) { printf("no encoder\n"); return 1; }
  CUtensorMap tm;
  cuuint64_t dims[2] = {16, rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {2, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, h, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)r);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  float ms;
  for (int lanes : {32, 8, 1}) {
    uint64_t per = 1024;
    for (int w = 0; w < 2; w++) { cudaEventRecord(a); k_s4<<<sms * 4, 256>>>(tm, rows, per, lanes); cudaEventRecord(b); cudaEventSynchronize(b); }
    cudaEventElapsedTime(&ms, a, b);
    double ops = (double)sms * 4 * 8 * lanes * per;
    printf("scatter4 reduce, %2d lanes/warp: %.3f Gop/s = %.3f G rows/s (%s)\n", lanes, ops / ms / 1e6, 4 * ops / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  }
  // check correctness: total added = 4 rows x 1 per op (only even column = 1)
  return 0;
}
