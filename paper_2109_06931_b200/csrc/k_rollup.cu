// k_rollup.cu — a-5 roll-up (§5.1: "propagating values up"; flat view
// per function P:936-937) with the fused a-10 derived-metric epilogue (§6.1 P:944-948:
// W = (S - S_stall)/S; stall percentages P:918; readings R3-R5, R18).
//
// One warp per row.  The row's instruction list (load-time CSR: every instruction whose
// scope chain contains the row's scope) is walked two instructions at a time: each
// half-warp reads one 128-B histogram row (lane = slot), adds it into its accumulator and
// adds the instruction's valid-sample total S(i) into the class-mix accumulator of lane
// class(i).  The 16 sums, the 16 mix entries and the 33 derived columns are written by the
// same warp; nothing goes back to HBM between roll-up and epilogue.
#include <cuda_runtime.h>
#include <stdint.h>

#include "gpa_internal.cuh"

namespace gpa {
namespace {

constexpr unsigned FULL = 0xFFFFFFFFu;

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7FF8000000000000ll); }
__device__ __forceinline__ bool is_lat(int r) { return r >= 1 && r <= 11 && r != 9; }  // R4

__global__ void __launch_bounds__(256) k_rollup(const uint32_t *__restrict__ ptr, const uint32_t *__restrict__ lst,
                                                uint32_t rows, int identity, const uint64_t *__restrict__ H,
                                                const uint8_t *__restrict__ cls, uint64_t *__restrict__ out_hist,
                                                uint64_t *__restrict__ out_mix, double *__restrict__ metrics) {
  const int lane = threadIdx.x & 31, half = lane >> 4, sl = lane & 15;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t r = warp; r < rows; r += nwarps) {
    uint32_t lo = identity ? r : __ldg(ptr + r), hi = identity ? r + 1 : __ldg(ptr + r + 1);
    unsigned long long acc = 0, mix = 0;
    for (uint32_t j0 = lo; j0 < hi; j0 += 2) {
      uint32_t j = j0 + half;
      bool ok = j < hi;
      uint32_t i = ok ? (identity ? j : __ldg(lst + j)) : 0;
      unsigned long long h = ok ? __ldg(H + ((uint64_t)i << 4) + sl) : 0ull;
      acc += h;
      unsigned long long s = sl < GPA_VALID_SLOTS ? h : 0ull;  // S(i) over the half-warp
      s += __shfl_xor_sync(FULL, s, 8);
      s += __shfl_xor_sync(FULL, s, 4);
      s += __shfl_xor_sync(FULL, s, 2);
      s += __shfl_xor_sync(FULL, s, 1);
      if (ok && __ldg(cls + i) == sl) mix += s;
    }
    acc += __shfl_down_sync(FULL, acc, 16);
    mix += __shfl_down_sync(FULL, mix, 16);
    if (lane < 16) {
      if (out_hist) out_hist[(uint64_t)r * GPA_SLOTS + lane] = acc;
      if (out_mix) out_mix[(uint64_t)r * GPA_SLOTS + lane] = mix;
    }
    if (metrics) {
      unsigned long long S = lane < GPA_VALID_SLOTS ? acc : 0ull;
      unsigned long long L = (lane < GPA_VALID_SLOTS && is_lat(lane)) ? acc : 0ull;
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        S += __shfl_xor_sync(FULL, S, o);
        L += __shfl_xor_sync(FULL, L, o);
      }
      unsigned long long v0 = __shfl_sync(FULL, acc, 0), v9 = __shfl_sync(FULL, acc, 9),
                         v15 = __shfl_sync(FULL, acc, 15);
      double *m = metrics + (uint64_t)r * GPA_NUM_DERIVED;
      double Sd = __ull2double_rn(S);
      bool z = S == 0;
      if (lane == 0) {
        m[0] = Sd;
        m[1] = z ? qnan() : __ddiv_rn(__ull2double_rn(v0), Sd);          // W
        m[2] = z ? qnan() : __ddiv_rn(__ull2double_rn(v0 + v9), Sd);     // latency hiding
        m[3] = z ? qnan() : __ddiv_rn(__ull2double_rn(L), Sd);           // latency stall
        m[16] = __ull2double_rn(v15);                                     // invalid samples
      }
      if (lane < GPA_VALID_SLOTS) m[4 + lane] = z ? qnan() : __ddiv_rn(__ull2double_rn(acc), Sd);
      if (lane < 16) m[17 + lane] = z ? qnan() : __ddiv_rn(__ull2double_rn(mix), Sd);
    }
  }
}

// CCT rows: fp64 vectors; S and the latency sum fold slots left to right (R3, R4).
__global__ void __launch_bounds__(256) k_derive_f64(const double *__restrict__ V, uint64_t rows,
                                                    double *__restrict__ metrics) {
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += (uint64_t)gridDim.x * blockDim.x) {
    const double2 *p = reinterpret_cast<const double2 *>(V + r * GPA_SLOTS);
    double v[16];
#pragma unroll
    for (int q = 0; q < 8; q++) {
      double2 t = __ldg(p + q);
      v[2 * q] = t.x;
      v[2 * q + 1] = t.y;
    }
    double S = 0.0, L = 0.0;
#pragma unroll
    for (int q = 0; q < GPA_VALID_SLOTS; q++) S = __dadd_rn(S, v[q]);
#pragma unroll
    for (int q = 0; q < GPA_VALID_SLOTS; q++)
      if (is_lat(q)) L = __dadd_rn(L, v[q]);
    double *m = metrics + r * GPA_NUM_DERIVED;
    bool z = S == 0.0;
    m[0] = S;
    m[1] = z ? qnan() : __ddiv_rn(v[0], S);
    m[2] = z ? qnan() : __ddiv_rn(__dadd_rn(v[0], v[9]), S);
    m[3] = z ? qnan() : __ddiv_rn(L, S);
#pragma unroll
    for (int q = 0; q < GPA_VALID_SLOTS; q++) m[4 + q] = z ? qnan() : __ddiv_rn(v[q], S);
    m[16] = v[15];
#pragma unroll
    for (int q = 0; q < 16; q++) m[17 + q] = qnan();  // no mix for CCT rows (R5)
  }
}

}  // namespace

cudaError_t launch_rollup(const uint32_t *d_ptr, const uint32_t *d_inst, uint32_t rows, bool identity,
                          const uint64_t *d_hist, const uint8_t *d_class, uint64_t *d_out_hist,
                          uint64_t *d_out_mix, double *d_metrics, int sm_count, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  uint64_t want = ((uint64_t)rows + 7) / 8;  // 8 warps per block
  uint64_t cap = (uint64_t)sm_count * 8;
  unsigned blocks = (unsigned)(want < cap ? want : cap);
  k_rollup<<<blocks, 256, 0, st>>>(d_ptr, d_inst, rows, identity ? 1 : 0, d_hist, d_class, d_out_hist, d_out_mix,
                                   d_metrics);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_derive_f64(const double *d_v, uint64_t rows, double *d_metrics, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  uint64_t blocks = (rows + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_derive_f64<<<(unsigned)blocks, 256, 0, st>>>(d_v, rows, d_metrics);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace gpa
