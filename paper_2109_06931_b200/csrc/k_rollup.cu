// k_rollup.cu — a-5 roll-up (§5.1: "propagating values up"; flat view
// per function P:936-937) with the fused a-10 derived-metric epilogue (§6.1 P:944-948:
// W = (S - S_stall)/S; stall percentages P:918; readings R3-R5, R18).
//
// Each row's instruction list (load-time CSR: every instruction whose scope chain contains
// the row's scope) is summed by a quad of lanes; the instruction's valid-sample total S(i)
// goes to the mix entry of class(i).  The 16 sums, the 16 mix entries and the 33 derived
// columns are written by the same quad: nothing returns to HBM between roll-up and epilogue.
#include <cuda_runtime.h>
#include <stdint.h>

#include "gpa_internal.cuh"

// Blocks per SM of the roll-up grids: short-lived blocks (a few items each) rather than one
// resident wave, so that the CCT's kernels on the high-priority stream find an SM as soon as a
// roll-up block retires while the scopes are rolled up concurrently on the side stream.
#ifndef GPA_ROLL_BLOCKS_PER_SM
#define GPA_ROLL_BLOCKS_PER_SM 64
#endif

namespace gpa {
namespace {

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7FF8000000000000ll); }
__device__ __forceinline__ bool is_lat(int r) { return r >= 1 && r <= 11 && r != 9; }  // R4

// Quad layout: 4 lanes per work item, lane q owns slots 4q..4q+3 of a 128-B histogram row
// (two 16-B loads), so a warp works on 8 rows / chunks at once.  Rows longer than
// kRollChunk instructions are split into chunks at load time; their partial sums meet in a
// u64 scratch row (integer adds: exact in any order) and a second pass finalises them.
__device__ __forceinline__ unsigned quad_mask() { return 0xFu << (threadIdx.x & 28); }

struct Acc {
  unsigned long long h[4], m[4];
};

// S(i) and the class-mix contribution of instruction i, added into a
__device__ __forceinline__ void acc_inst(Acc &a, const uint64_t *__restrict__ H, const uint8_t *__restrict__ cls,
                                         uint32_t i, int q, unsigned qm) {
  const ulonglong2 *p = reinterpret_cast<const ulonglong2 *>(H + ((uint64_t)i << 4) + 4 * q);
  ulonglong2 x = __ldg(p), y = __ldg(p + 1);
  a.h[0] += x.x; a.h[1] += x.y; a.h[2] += y.x; a.h[3] += y.y;
  unsigned long long s = q < 3 ? (x.x + x.y + y.x + y.y) : 0ull;  // slots 0..11
  s += __shfl_xor_sync(qm, s, 1, 4);
  s += __shfl_xor_sync(qm, s, 2, 4);
  uint32_t k = __ldg(cls + i);
  if ((int)(k >> 2) == q) a.m[k & 3] += s;
}

__device__ __forceinline__ void finalize(const Acc &a, uint32_t r, int q, unsigned qm, uint64_t *__restrict__ out_hist,
                                         uint64_t *__restrict__ out_mix, double *__restrict__ metrics) {
  if (out_hist) {
    ulonglong2 *o = reinterpret_cast<ulonglong2 *>(out_hist + (uint64_t)r * GPA_SLOTS + 4 * q);
    o[0] = make_ulonglong2(a.h[0], a.h[1]);
    o[1] = make_ulonglong2(a.h[2], a.h[3]);
  }
  if (out_mix) {
    ulonglong2 *o = reinterpret_cast<ulonglong2 *>(out_mix + (uint64_t)r * GPA_SLOTS + 4 * q);
    o[0] = make_ulonglong2(a.m[0], a.m[1]);
    o[1] = make_ulonglong2(a.m[2], a.m[3]);
  }
  if (!metrics) return;
  unsigned long long S = 0, L = 0;
#pragma unroll
  for (int t = 0; t < 4; t++) {
    int r2 = 4 * q + t;
    if (r2 < GPA_VALID_SLOTS) S += a.h[t];
    if (r2 < GPA_VALID_SLOTS && is_lat(r2)) L += a.h[t];
  }
  S += __shfl_xor_sync(qm, S, 1, 4);
  S += __shfl_xor_sync(qm, S, 2, 4);
  L += __shfl_xor_sync(qm, L, 1, 4);
  L += __shfl_xor_sync(qm, L, 2, 4);
  unsigned long long v9 = __shfl_sync(qm, a.h[1], 2, 4);   // slot 9 lives in lane 2
  unsigned long long v15 = __shfl_sync(qm, a.h[3], 3, 4);  // slot 15 lives in lane 3
  double *m = metrics + (uint64_t)r * GPA_NUM_DERIVED;
  const double Sd = __ull2double_rn(S);
  const bool z = S == 0;
  if (q == 0) {
    m[0] = Sd;
    m[1] = z ? qnan() : __ddiv_rn(__ull2double_rn(a.h[0]), Sd);       // W
    m[2] = z ? qnan() : __ddiv_rn(__ull2double_rn(a.h[0] + v9), Sd);  // latency hiding (R4)
    m[3] = z ? qnan() : __ddiv_rn(__ull2double_rn(L), Sd);            // latency stall (R4)
    m[16] = __ull2double_rn(v15);                                      // invalid samples
  }
#pragma unroll
  for (int t = 0; t < 4; t++) {
    int r2 = 4 * q + t;
    if (r2 < GPA_VALID_SLOTS) m[4 + r2] = z ? qnan() : __ddiv_rn(__ull2double_rn(a.h[t]), Sd);
    m[17 + r2] = z ? qnan() : __ddiv_rn(__ull2double_rn(a.m[t]), Sd);
  }
}

// pass 1: one quad per chunk (or per instruction when `identity`)
__global__ void __launch_bounds__(256) k_rollup(const uint32_t *__restrict__ chunk, const uint32_t *__restrict__ lst,
                                                uint32_t n_items, int identity,
                                                const uint32_t *__restrict__ multi_slot, const uint64_t *__restrict__ H,
                                                const uint8_t *__restrict__ cls, uint64_t *__restrict__ out_hist,
                                                uint64_t *__restrict__ out_mix, double *__restrict__ metrics,
                                                unsigned long long *__restrict__ scratch) {
  const int q = threadIdx.x & 3;
  const unsigned qm = quad_mask();
  const uint32_t nq = (gridDim.x * blockDim.x) >> 2;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 2; w < n_items; w += nq) {
    uint32_t row, b, e;
    if (identity) {
      row = w; b = w; e = w + 1;
    } else {
      row = __ldg(chunk + 3 * w); b = __ldg(chunk + 3 * w + 1); e = __ldg(chunk + 3 * w + 2);
    }
    Acc a = {{0, 0, 0, 0}, {0, 0, 0, 0}};
    uint32_t j = b;
    for (; j + 4 <= e; j += 4) {  // four independent rows in flight per lane
      uint32_t i0 = identity ? j : __ldg(lst + j), i1 = identity ? j + 1 : __ldg(lst + j + 1);
      uint32_t i2 = identity ? j + 2 : __ldg(lst + j + 2), i3 = identity ? j + 3 : __ldg(lst + j + 3);
      acc_inst(a, H, cls, i0, q, qm);
      acc_inst(a, H, cls, i1, q, qm);
      acc_inst(a, H, cls, i2, q, qm);
      acc_inst(a, H, cls, i3, q, qm);
    }
    for (; j < e; j++) acc_inst(a, H, cls, identity ? j : __ldg(lst + j), q, qm);
    const uint32_t slot = identity ? NONE : __ldg(multi_slot + row);
    if (slot == NONE) {
      finalize(a, row, q, qm, out_hist, out_mix, metrics);
    } else {
      unsigned long long *sp = scratch + (uint64_t)slot * 32;
#pragma unroll
      for (int t = 0; t < 4; t++) {
        if (a.h[t]) atomicAdd(sp + 4 * q + t, a.h[t]);
        if (a.m[t]) atomicAdd(sp + 16 + 4 * q + t, a.m[t]);
      }
    }
  }
}

// pass 2: one quad per multi-chunk row: finalise from the scratch sums
__global__ void __launch_bounds__(256) k_rollup_fin(const uint32_t *__restrict__ multi_rows, uint32_t n_multi,
                                                    const unsigned long long *__restrict__ scratch,
                                                    uint64_t *__restrict__ out_hist, uint64_t *__restrict__ out_mix,
                                                    double *__restrict__ metrics) {
  const int q = threadIdx.x & 3;
  const unsigned qm = quad_mask();
  const uint32_t nq = (gridDim.x * blockDim.x) >> 2;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 2; w < n_multi; w += nq) {
    const unsigned long long *sp = scratch + (uint64_t)w * 32;
    Acc a;
#pragma unroll
    for (int t = 0; t < 4; t++) {
      a.h[t] = sp[4 * q + t];
      a.m[t] = sp[16 + 4 * q + t];
    }
    finalize(a, __ldg(multi_rows + w), q, qm, out_hist, out_mix, metrics);
  }
}

// ---- all scope kinds in one launch (gpa_derive_scopes) ----------------------------------------
// items [0, n_ident): INST rows ident_lo + w (identity); then the merged chunk list of the tree
// kinds (kind, row, begin, end into the concatenated instruction lists), ordered by function.
struct ScopeOuts {
  uint64_t *hist[5];
  uint64_t *mix[5];
  double *met[5];
  const uint32_t *mslot[5];  // per tree kind: row -> merged multi slot (NONE = single chunk)
};

__global__ void __launch_bounds__(256) k_rollup_multi(const uint4 *__restrict__ chunk, uint32_t n_chunk,
                                                      uint32_t ident_lo, uint32_t n_ident,
                                                      const uint32_t *__restrict__ lst, const uint64_t *__restrict__ H,
                                                      const uint8_t *__restrict__ cls, ScopeOuts O,
                                                      unsigned long long *__restrict__ scratch) {
  const int q = threadIdx.x & 3;
  const unsigned qm = quad_mask();
  const uint32_t nq = (gridDim.x * blockDim.x) >> 2;
  const uint32_t items = n_ident + n_chunk;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 2; w < items; w += nq) {
    uint32_t kind, row, b, e;
    const bool ident = w < n_ident;
    if (ident) {
      kind = 0; row = ident_lo + w; b = row; e = row + 1;
    } else {
      const uint4 c = __ldg(chunk + (w - n_ident));
      kind = c.x; row = c.y; b = c.z; e = c.w;
    }
    Acc a = {{0, 0, 0, 0}, {0, 0, 0, 0}};
    uint32_t j = b;
    for (; j + 4 <= e; j += 4) {
      uint32_t i0 = ident ? j : __ldg(lst + j), i1 = ident ? j + 1 : __ldg(lst + j + 1);
      uint32_t i2 = ident ? j + 2 : __ldg(lst + j + 2), i3 = ident ? j + 3 : __ldg(lst + j + 3);
      acc_inst(a, H, cls, i0, q, qm);
      acc_inst(a, H, cls, i1, q, qm);
      acc_inst(a, H, cls, i2, q, qm);
      acc_inst(a, H, cls, i3, q, qm);
    }
    for (; j < e; j++) acc_inst(a, H, cls, ident ? j : __ldg(lst + j), q, qm);
    const uint32_t slot = ident ? NONE : __ldg(O.mslot[kind] + row);
    if (slot == NONE) {
      finalize(a, row, q, qm, O.hist[kind], O.mix[kind], O.met[kind]);
    } else {
      unsigned long long *sp = scratch + (uint64_t)slot * 32;
#pragma unroll
      for (int t = 0; t < 4; t++) {
        if (a.h[t]) atomicAdd(sp + 4 * q + t, a.h[t]);
        if (a.m[t]) atomicAdd(sp + 16 + 4 * q + t, a.m[t]);
      }
    }
  }
}

// multi-chunk rows: (kind, row) pairs, slots m0 .. m0 + n of the merged multi list
__global__ void __launch_bounds__(256) k_rollup_fin_multi(const uint2 *__restrict__ mrows, uint32_t n_multi,
                                                          const unsigned long long *__restrict__ scratch, ScopeOuts O) {
  const int q = threadIdx.x & 3;
  const unsigned qm = quad_mask();
  const uint32_t nq = (gridDim.x * blockDim.x) >> 2;
  for (uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 2; w < n_multi; w += nq) {
    const unsigned long long *sp = scratch + (uint64_t)w * 32;
    Acc a;
#pragma unroll
    for (int t = 0; t < 4; t++) {
      a.h[t] = sp[4 * q + t];
      a.m[t] = sp[16 + 4 * q + t];
    }
    const uint2 kr = __ldg(mrows + w);
    finalize(a, kr.y, q, qm, O.hist[kr.x], O.mix[kr.x], O.met[kr.x]);
  }
}

// CCT rows: fp64 vectors; S and the latency sum fold slots left to right (R3, R4).
// d_rows (asynchronous trees): the row count on the device; above `rows` (~0: the build did not
// fit) means no row
__global__ void __launch_bounds__(256) k_derive_f64(const double *__restrict__ V, uint64_t rows,
                                                    double *__restrict__ metrics,
                                                    const unsigned long long *__restrict__ d_rows) {
  if (d_rows) {
    const unsigned long long r = *d_rows;
    rows = r > rows ? 0 : r;
  }
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

cudaError_t launch_rollup(const RollSet *set, uint32_t rows, const uint64_t *d_hist, const uint8_t *d_class,
                          uint64_t *d_out_hist, uint64_t *d_out_mix, double *d_metrics, int sm_count,
                          cudaStream_t st, uint32_t c0, uint32_t c1, uint32_t m0, uint32_t m1) {
  if (rows == 0) return cudaSuccess;
  const bool identity = set == nullptr;
  if (!identity) {
    c1 = c1 < set->n_chunks ? c1 : set->n_chunks;
    m1 = m1 < set->n_multi ? m1 : set->n_multi;
    if (c0 >= c1) return cudaSuccess;
  }
  const uint32_t items = identity ? rows : c1 - c0;
  unsigned long long *scratch = nullptr;  // slots [m0, m1) of the n_multi multi-chunk rows
  const uint32_t n_multi = identity || m0 >= m1 ? 0 : m1 - m0;
  if (n_multi) {
    cudaError_t e = pool_alloc((void **)&scratch, (size_t)n_multi * 32 * 8, st);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(scratch, 0, (size_t)n_multi * 32 * 8, st);
  }
  uint64_t want = ((uint64_t)items * 4 + 255) / 256;
  uint64_t cap = (uint64_t)sm_count * GPA_ROLL_BLOCKS_PER_SM;
  unsigned blocks = (unsigned)(want < cap ? want : cap);
  k_rollup<<<blocks, 256, 0, st>>>(identity ? nullptr : set->d_chunk + 3ull * c0, identity ? nullptr : set->d_inst,
                                   items, identity ? 1 : 0, identity ? nullptr : set->d_multi_slot, d_hist, d_class,
                                   d_out_hist, d_out_mix, d_metrics, scratch ? scratch - (size_t)m0 * 32 : nullptr);
  count_launches(1);
  cudaError_t e = cudaGetLastError();
  if (n_multi) {
    uint64_t b2 = ((uint64_t)n_multi * 4 + 255) / 256;
    k_rollup_fin<<<(unsigned)(b2 < cap ? b2 : cap), 256, 0, st>>>(set->d_multi_rows + m0, n_multi, scratch, d_out_hist,
                                                                   d_out_mix, d_metrics);
    count_launches(1);
    cudaError_t e2 = cudaGetLastError();
    cudaError_t e3 = cudaFreeAsync(scratch, st);
    if (e == cudaSuccess) e = e2 != cudaSuccess ? e2 : e3;
  }
  return e;
}

cudaError_t launch_rollup_multi(const MultiRoll &M, uint32_t c0, uint32_t c1, uint32_t m0, uint32_t m1, uint32_t ident_lo,
                                uint32_t n_ident, const uint64_t *d_hist, const uint8_t *d_class,
                                uint64_t *const hist[5], uint64_t *const mix[5], double *const met[5], int sm_count,
                                cudaStream_t st) {
  ScopeOuts O;
  for (int k = 0; k < 5; k++) {
    O.hist[k] = hist[k];
    O.mix[k] = mix[k];
    O.met[k] = met[k];
    O.mslot[k] = M.d_mslot[k];
  }
  const uint32_t n_chunk = c1 > c0 ? c1 - c0 : 0, n_multi = m1 > m0 ? m1 - m0 : 0;
  const uint32_t items = n_ident + n_chunk;
  if (items == 0) return cudaSuccess;
  unsigned long long *scratch = nullptr;
  if (n_multi) {
    cudaError_t e = pool_alloc((void **)&scratch, (size_t)n_multi * 32 * 8, st);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(scratch, 0, (size_t)n_multi * 32 * 8, st);
  }
  uint64_t want = ((uint64_t)items * 4 + 255) / 256;
  uint64_t cap = (uint64_t)sm_count * GPA_ROLL_BLOCKS_PER_SM;
  unsigned blocks = (unsigned)(want < cap ? want : cap);
  k_rollup_multi<<<blocks, 256, 0, st>>>(reinterpret_cast<const uint4 *>(M.d_chunk) + c0, n_chunk, ident_lo, n_ident,
                                         M.d_lst, d_hist, d_class, O, scratch ? scratch - (size_t)m0 * 32 : nullptr);
  count_launches(1);
  cudaError_t e = cudaGetLastError();
  if (n_multi) {
    uint64_t b2 = ((uint64_t)n_multi * 4 + 255) / 256;
    k_rollup_fin_multi<<<(unsigned)(b2 < cap ? b2 : cap), 256, 0, st>>>(
        reinterpret_cast<const uint2 *>(M.d_mrows) + m0, n_multi, scratch, O);
    count_launches(1);
    cudaError_t e2 = cudaGetLastError();
    cudaError_t e3 = cudaFreeAsync(scratch, st);
    if (e == cudaSuccess) e = e2 != cudaSuccess ? e2 : e3;
  }
  return e;
}

cudaError_t launch_derive_f64(const double *d_v, uint64_t rows, double *d_metrics, cudaStream_t st,
                              const unsigned long long *d_rows) {
  if (rows == 0) return cudaSuccess;
  uint64_t blocks = (rows + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_derive_f64<<<(unsigned)blocks, 256, 0, st>>>(d_v, rows, d_metrics, d_rows);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace gpa
