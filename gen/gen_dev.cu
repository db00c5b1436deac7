/* gen_dev.cu — device build of the counter-based record generator (INPUT GENERATION ONLY;
 * see gen_core.h).  Used to materialise multi-GB workloads directly in HBM, untimed.
 * Bit-identical to gen_host.c (tests/test_gen.py checks a memcmp on sampled ranges). */
#include <cuda_runtime.h>
#include "gen_core.h"

__global__ void gen_kernel(gen_tables T, uint64_t k0, uint64_t n, gen_record *out)
{
  uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += stride) {
    gen_record r = gen_one(&T, k0 + x);
    uint4 v;
    v.x = (uint32_t)r.pc; v.y = (uint32_t)(r.pc >> 32);
    v.z = r.count; v.w = (uint32_t)r.stall | ((uint32_t)r.stream << 16);
    reinterpret_cast<uint4 *>(out)[x] = v;
  }
}

extern "C" int gen_records_device(const gen_tables *T_dev_ptrs, uint64_t k0, uint64_t n,
                                  void *d_out, void *stream)
{
  if (n == 0) return 0;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint64_t blocks = (n + 255) / 256;
  if (blocks > (uint64_t)sms * 16) blocks = (uint64_t)sms * 16;
  gen_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(*T_dev_ptrs, k0, n, (gen_record *)d_out);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
