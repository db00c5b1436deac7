// k_prof.cu — f1: per-profile function histograms and cross-profile statistics
// (§4.5 P:481-487 "sum, min, mean, max, std. deviation, and coefficient of
// variation"; profiles = GPU streams / ranks / threads; reading R25).
//
// k_attr_prof_tma (granule map): see below.
// k_attr_prof: register streaming (4 records per lane in flight), pc -> instruction through
//   the granule map (or binary search), -> function, -> (profile, function, slot) bin.  A
//   warp's records usually share the profile (streams are contiguous) and often the function,
//   so lanes with equal 64-bit keys are combined (match.any) before one u64 L2 reduction.
// k_prof_stats: one thread per (function, slot); exact u64 / u128 sums over the profiles,
//   then one correctly rounded conversion per statistic (bit-identical to the oracle).
#include <cuda_runtime.h>
#include <stdint.h>

#include "gpa_internal.cuh"
#include "kern_common.cuh"

namespace gpa {
namespace {

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr int kThreads = 256, kUnroll = 4;


template <int MODE>
__global__ void __launch_bounds__(kThreads)
    k_attr_prof(AttrTables T, const uint32_t *__restrict__ inst_func, uint32_t n_func, const uint4 *__restrict__ rec,
                uint64_t n, uint32_t n_prof, unsigned long long *__restrict__ PH, unsigned long long *__restrict__ PU) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * kThreads) >> 5;
  for (uint64_t base = warp * 32 * kUnroll; base < n; base += nwarps * 32 * kUnroll) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; u++) {
      uint64_t k = base + (uint64_t)u * 32 + lane;
      v[u] = k < n ? ld_stream(rec + k) : make_uint4(0, 0, 0, 0);
    }
    uint32_t f[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; u++) {
      uint32_t i = lookup<MODE>(T, ((uint64_t)v[u].y << 32) | v[u].x);
      f[u] = i == NONE ? NONE : (inst_func ? __ldg(inst_func + i) : i);  // inst_func NULL: instruction rows
    }
#pragma unroll
    for (int u = 0; u < kUnroll; u++) {
      uint64_t k = base + (uint64_t)u * 32 + lane;
      uint32_t cnt = v[u].z, stall = v[u].w & 0xFFFFu, stream = v[u].w >> 16;
      uint32_t slot = stall < GPA_VALID_SLOTS ? stall : GPA_SLOT_INVALID;
      uint64_t p = stream < n_prof ? stream : n_prof;
      unsigned long long *target =
          f[u] == NONE ? PU + (p << 4 | slot) : PH + (((p * n_func + f[u]) << 4) | slot);
      const bool live = k < n && cnt;
      unsigned long long key = live ? (unsigned long long)(uintptr_t)target : 0ull;
      unsigned peers = __match_any_sync(FULL, key);
      int gmax = __reduce_max_sync(FULL, (unsigned)__popc(peers));
      unsigned long long total = cnt;
      if (gmax > 1) {
        unsigned rest = peers & ~(1u << lane);
        for (int t = 1; t < gmax; t++) {
          int src = rest ? __ffs(rest) - 1 : lane;
          uint32_t x = __shfl_sync(FULL, cnt, src);
          if (rest) {
            total += x;
            rest &= rest - 1;
          }
        }
      }
      if (live && lane == __ffs(peers) - 1) atomicAdd(target, total);
    }
  }
}

// k_attr_prof_tma: the TMA-fed variant used with the granule map.  Each CTA takes a contiguous
// range of record tiles; streams are contiguous in the input (one profile's records follow
// each other), so a CTA meets only a few profiles.  Its shared memory holds u32 counters for
// K "profile lanes" x n_func functions x 12 slots, lane k = profile p_first + k where p_first
// is the profile of the CTA's first record; other records, unattributed ones and invalid
// stalls go straight to L2.  One gather (granule -> function, built at load) per record.
// 31 consumer warps x 3 records per lane in two 46.5 KiB stages, one tile of lookahead (the geometry
// of K_attr_code32) and 96 KiB of counters, so ring + table stay under the 196 KiB carve-out and
// ~30 KiB of L1 caches the granule -> function gathers: C4 (1e9 records, 384 profiles) 3.65 ->
// 2.61 ms = 0.94 of the HBM peak (16 warps x 2 x 4 stages with 160 KiB of counters before)
#ifndef GPA_PROF_TAB
#define GPA_PROF_TAB (96 * 1024)
#endif
#ifndef GPA_PROF_NC
#define GPA_PROF_NC 31
#endif
#ifndef GPA_PROF_R
#define GPA_PROF_R 3
#endif
#ifndef GPA_PROF_NST
#define GPA_PROF_NST 2
#endif
#ifndef GPA_PROF_LOOK
#define GPA_PROF_LOOK 1
#endif
constexpr int kProfTab = GPA_PROF_TAB;  // bytes of shared counters
using RingProf = Ring<GPA_PROF_NC, GPA_PROF_R, GPA_PROF_NST>;
constexpr int kProfLook = GPA_PROF_LOOK;

template <class RG>
__global__ void __launch_bounds__(RG::kThreads, 1)
    k_attr_prof_tma(AttrTables T, const uint32_t *__restrict__ gfunc, uint32_t n_func, const uint4 *__restrict__ rec,
                    uint64_t n, uint32_t n_prof, uint32_t K, unsigned long long *__restrict__ PH,
                    unsigned long long *__restrict__ PU) {
  // K > 0: each CTA takes a contiguous range of tiles (it meets few profiles: the shared table
  // pays).  K == 0 (instruction rows, everything to L2): tiles are dealt round-robin so all CTAs
  // stay inside the same stretch of the stream (a profile or two) and the reduction targets stay
  // L2-resident instead of spreading over 148 profiles' rows.
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int S = RG::kTile, NST = RG::kStages, NC = RG::kConsumers, R = RG::kPerLane, D = kProfLook + 1;
  uint4 *ring = reinterpret_cast<uint4 *>(smem);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + RG::kBytes);
  uint64_t *empty = full + NST;
  uint32_t *tab = reinterpret_cast<uint32_t *>(smem + RG::kBytes + 2 * NST * 8);
  const uint32_t tab_s = smem_u32(tab);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t ntiles = (n + S - 1) / S;
  const bool rr = K == 0;
  const uint64_t t0 = rr ? blockIdx.x : ntiles * blockIdx.x / gridDim.x;
  const uint64_t t1 = rr ? ntiles : ntiles * (blockIdx.x + 1) / gridDim.x;
  const uint64_t step = rr ? gridDim.x : 1;
  const uint32_t nt = K * n_func * GPA_VALID_SLOTS;
  for (uint32_t x = threadIdx.x; x < nt; x += blockDim.x) tab[x] = 0;
  uint32_t pf = 0;
  if (t0 < t1) {
    uint32_t s0 = __ldg(reinterpret_cast<const uint32_t *>(rec + t0 * S) + 3) >> 16;
    pf = s0 < n_prof ? s0 : n_prof;
  }
  ring_init(full, empty, NST, NC);
  __syncthreads();
  if (warp == NC) {
    if (lane == 0) ring_produce<RG>(ring, full, empty, rec, n, t0, step, t1);
    return;
  }
  uint4 v[D][R];
  uint32_t c[D][R];
  auto fetch = [&](uint32_t it, uint4 *vv, uint32_t *cc) {
    uint32_t st = it % NST, ph = (it / NST) & 1;
    mbar_wait(full + st, ph);
    const uint4 *src = ring + (size_t)st * S + warp * 32 + lane;
#pragma unroll
    for (int u = 0; u < R; u++) vv[u] = src[u * NC * 32];  // beyond the tile end: masked below
    __syncwarp();
    if (lane == 0) ring_release(empty + st);
#pragma unroll
    for (int u = 0; u < R; u++) {
      uint64_t g = ((((uint64_t)vv[u].y << 32) | vv[u].x) - T.base) >> T.gshift;
      cc[u] = g < T.n_gran ? __ldg(gfunc + g) : NONE;
    }
  };
#pragma unroll
  for (int q = 0; q < kProfLook; q++)
    if (t0 + q * step < t1) fetch(q, v[q], c[q]);
  for (uint32_t it0 = 0;; it0 += D) {
#pragma unroll
    for (int q = 0; q < D; q++) {
      const uint32_t it = it0 + q;
      const uint64_t tile = t0 + it * step;
      if (tile >= t1) goto done;
      if (tile + kProfLook * step < t1) fetch(it + kProfLook, v[(q + kProfLook) % D], c[(q + kProfLook) % D]);
      const uint64_t left = n - tile * S;
      const uint32_t m = (uint32_t)(left < (uint64_t)S ? left : (uint64_t)S);
      uint32_t old[R], idx[R];
#pragma unroll
      for (int u = 0; u < R; u++) {
        const uint32_t j = (uint32_t)(u * NC + warp) * 32 + lane;
        const uint32_t f = c[q][u], cnt = v[q][u].z, stall = v[q][u].w & 0xFFFFu, sid = v[q][u].w >> 16;
        const uint32_t slot = stall < GPA_VALID_SLOTS ? stall : GPA_SLOT_INVALID;
        const uint32_t p = sid < n_prof ? sid : n_prof;
        const uint32_t k = p - pf;  // profile lane (wraps to a huge value below pf)
        idx[u] = NONE;
        old[u] = 0;
        if (j < m) {
          if (f != NONE && slot < (uint32_t)GPA_VALID_SLOTS && k < K) {
            idx[u] = (k * n_func + f) * GPA_VALID_SLOTS + slot;
            old[u] = atoms_add(tab_s + idx[u] * 4, cnt);
          } else if (f == NONE) {
            red_add_u64(PU + ((uint64_t)p << 4 | slot), cnt);
          } else {
            red_add_u64(PH + (((uint64_t)p * n_func + f) << 4 | slot), cnt);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < R; u++) {
        if (idx[u] != NONE && old[u] + v[q][u].z < old[u]) {  // u32 wrap: repay 2^32 in L2
          uint32_t x = idx[u], slot = x % GPA_VALID_SLOTS, kf = x / GPA_VALID_SLOTS;
          red_add_u64(PH + (((uint64_t)(pf + kf / n_func) * n_func + kf % n_func) << 4 | slot), 1ull << 32);
        }
      }
    }
  }
done:
  asm volatile("bar.sync 1, %0;" ::"r"(NC * 32) : "memory");
  for (uint32_t x = threadIdx.x; x < nt; x += NC * 32) {
    uint32_t val = tab[x];
    if (val) {
      uint32_t slot = x % GPA_VALID_SLOTS, kf = x / GPA_VALID_SLOTS;
      red_add_u64(PH + (((uint64_t)(pf + kf / n_func) * n_func + kf % n_func) << 4 | slot), val);
    }
  }
}

// correctly rounded unsigned 128-bit -> double
__device__ __forceinline__ double u128_to_double(unsigned __int128 x) {
  uint64_t hi = (uint64_t)(x >> 64);
  if (hi == 0) return __ull2double_rn((uint64_t)x);
  int lz = __clzll((long long)hi);
  int shift = 64 - lz;                           // bits to drop so the value fits in 64
  uint64_t m = (uint64_t)(x >> shift);
  uint64_t sticky = ((x & (((unsigned __int128)1 << shift) - 1)) != 0) ? 1ull : 0ull;
  return ldexp(__ull2double_rn(m | sticky), shift);
}

__global__ void k_prof_stats(const uint64_t *__restrict__ PH, uint32_t n_prof, uint32_t rows,
                             double *__restrict__ out) {
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < (uint64_t)rows * GPA_SLOTS;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t f = x >> 4;
    const int r = (int)(x & 15);
    unsigned __int128 sum = 0, sq = 0;
    uint64_t mn = ~0ull, mx = 0;
    for (uint32_t p = 0; p < n_prof; p++) {
      uint64_t v = __ldg(PH + ((uint64_t)p * rows + f) * GPA_SLOTS + r);
      sum += v;
      sq += (unsigned __int128)v * v;
      mn = v < mn ? v : mn;
      mx = v > mx ? v : mx;
    }
    const double P = __uint2double_rn(n_prof), S = u128_to_double(sum);
    const unsigned __int128 num = (unsigned __int128)n_prof * sq - sum * sum;  // P·Σx² − (Σx)²
    const double mean = n_prof ? __ddiv_rn(S, P) : 0.0;
    const double sd = n_prof ? __ddiv_rn(__dsqrt_rn(u128_to_double(num)), P) : 0.0;
    double *o = out + f * 6 * GPA_SLOTS;
    o[0 * GPA_SLOTS + r] = S;
    o[1 * GPA_SLOTS + r] = n_prof ? __ull2double_rn(mn) : 0.0;
    o[2 * GPA_SLOTS + r] = mean;
    o[3 * GPA_SLOTS + r] = __ull2double_rn(mx);
    o[4 * GPA_SLOTS + r] = sd;
    o[5 * GPA_SLOTS + r] = mean == 0.0 ? 0.0 : __ddiv_rn(sd, mean);
  }
}

// fp64 cube statistics (R28): left-fold sum, min, max, mean, two-pass population std, cv
__global__ void k_prof_stats_f64(const double *__restrict__ X, uint32_t n_prof, uint64_t rows,
                                 double *__restrict__ out) {
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < rows * GPA_SLOTS;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t f = x >> 4;
    const int r = (int)(x & 15);
    double sum = 0.0, mn = 0.0, mx = 0.0;
    for (uint32_t p = 0; p < n_prof; p++) {
      const double v = __ldg(X + ((uint64_t)p * rows + f) * GPA_SLOTS + r);
      sum = __dadd_rn(sum, v);
      if (p == 0 || v < mn) mn = v;
      if (p == 0 || v > mx) mx = v;
    }
    const double mean = n_prof ? __ddiv_rn(sum, __uint2double_rn(n_prof)) : 0.0;
    double ss = 0.0;
    for (uint32_t p = 0; p < n_prof; p++) {
      const double d = __dsub_rn(__ldg(X + ((uint64_t)p * rows + f) * GPA_SLOTS + r), mean);
      ss = __dadd_rn(ss, __dmul_rn(d, d));
    }
    const double sd = n_prof ? __dsqrt_rn(__ddiv_rn(ss, __uint2double_rn(n_prof))) : 0.0;
    double *o = out + f * 6 * GPA_SLOTS;
    o[0 * GPA_SLOTS + r] = sum;
    o[1 * GPA_SLOTS + r] = mn;
    o[2 * GPA_SLOTS + r] = mean;
    o[3 * GPA_SLOTS + r] = mx;
    o[4 * GPA_SLOTS + r] = sd;
    o[5 * GPA_SLOTS + r] = mean == 0.0 ? 0.0 : __ddiv_rn(sd, mean);
  }
}

}  // namespace

cudaError_t launch_attribute_profiles_inst(const AttrTables &T, uint32_t n_inst, const gpa_sample *d_samples,
                                           uint64_t n, uint32_t n_prof, unsigned long long *d_ph,
                                           unsigned long long *d_pu, int sm_count, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const uint4 *rec = reinterpret_cast<const uint4 *>(d_samples);
  // large calls: the current profile's hot (instruction, slot) bins in shared memory (k_attr.cu)
  if (prof_code_ok(T, n)) return launch_prof_inst_code(T, d_samples, n, n_prof, d_ph, d_pu, sm_count, st);
  if (T.mode == 0 && n >= 4096) {  // TMA ring, granule -> instruction, one u64 L2 reduction per record
    using RG = RingProf;
    const size_t smem = RG::kBytes + 2 * RG::kStages * 8;
    cudaError_t e = cudaFuncSetAttribute(k_attr_prof_tma<RG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    uint64_t ntiles = (n + RG::kTile - 1) / RG::kTile;
    unsigned blocks = (unsigned)(ntiles < (uint64_t)sm_count ? ntiles : (uint64_t)sm_count);
    k_attr_prof_tma<RG><<<blocks, RG::kThreads, smem, st>>>(T, T.gmap, n_inst, rec, n, n_prof, 0, d_ph, d_pu);
    count_launches(1);
    return cudaGetLastError();
  }
  uint64_t per_block = (uint64_t)kThreads * kUnroll;
  uint64_t want = (n + per_block - 1) / per_block;
  uint64_t cap = (uint64_t)sm_count * (2048 / kThreads);
  unsigned blocks = (unsigned)(want < cap ? want : cap);
  if (T.mode == 0) k_attr_prof<0><<<blocks, kThreads, 0, st>>>(T, nullptr, n_inst, rec, n, n_prof, d_ph, d_pu);
  else k_attr_prof<1><<<blocks, kThreads, 0, st>>>(T, nullptr, n_inst, rec, n, n_prof, d_ph, d_pu);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_profile_stats_f64(const double *d_x, uint32_t n_prof, uint64_t rows, double *d_stats,
                                     cudaStream_t st) {
  if (!rows) return cudaSuccess;
  uint64_t blocks = (rows * GPA_SLOTS + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_prof_stats_f64<<<(unsigned)blocks, 256, 0, st>>>(d_x, n_prof, rows, d_stats);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_attribute_profiles(const AttrTables &T, const uint32_t *d_inst_func, const uint32_t *d_gfunc,
                                      uint32_t n_func, const gpa_sample *d_samples, uint64_t n, uint32_t n_prof,
                                      unsigned long long *d_ph, unsigned long long *d_pu, int sm_count,
                                      cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const uint32_t K0 = n_func ? (uint32_t)(kProfTab / ((size_t)n_func * GPA_VALID_SLOTS * 4)) : 0;
  if (T.mode == 0 && n >= 4096 && K0 >= 1) {  // else: register streaming with warp aggregation
    using RG = RingProf;
    const uint32_t K = K0 > 16 ? 16 : K0;
    const size_t smem = RG::kBytes + 2 * RG::kStages * 8 + (size_t)K * n_func * GPA_VALID_SLOTS * 4;
    cudaError_t e = cudaFuncSetAttribute(k_attr_prof_tma<RG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    uint64_t ntiles = (n + RG::kTile - 1) / RG::kTile;
    unsigned blocks = (unsigned)(ntiles < (uint64_t)sm_count ? ntiles : (uint64_t)sm_count);
    k_attr_prof_tma<RG><<<blocks, RG::kThreads, smem, st>>>(T, d_gfunc, n_func, reinterpret_cast<const uint4 *>(d_samples),
                                                          n, n_prof, K, d_ph, d_pu);
    count_launches(1);
    return cudaGetLastError();
  }
  uint64_t per_block = (uint64_t)kThreads * kUnroll;
  uint64_t want = (n + per_block - 1) / per_block;
  uint64_t cap = (uint64_t)sm_count * (2048 / kThreads);
  unsigned blocks = (unsigned)(want < cap ? want : cap);
  const uint4 *rec = reinterpret_cast<const uint4 *>(d_samples);
  if (T.mode == 0) k_attr_prof<0><<<blocks, kThreads, 0, st>>>(T, d_inst_func, n_func, rec, n, n_prof, d_ph, d_pu);
  else k_attr_prof<1><<<blocks, kThreads, 0, st>>>(T, d_inst_func, n_func, rec, n, n_prof, d_ph, d_pu);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_profile_stats(const uint64_t *d_ph, uint32_t n_prof, uint32_t rows, double *d_stats,
                                 cudaStream_t st) {
  if (!rows) return cudaSuccess;
  uint64_t blocks = ((uint64_t)rows * GPA_SLOTS + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_prof_stats<<<(unsigned)blocks, 256, 0, st>>>(d_ph, n_prof, rows, d_stats);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace gpa
