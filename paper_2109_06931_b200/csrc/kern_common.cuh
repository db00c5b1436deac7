// kern_common.cuh — device helpers shared by the libgpa kernels (streaming loads, L2
// reductions, shared atomics, mbarriers, 1-D TMA bulk copies and the record ring).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gpa_internal.cuh"

namespace gpa {
namespace {

// ---- device helpers ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 ld_stream(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

__device__ __forceinline__ void red_add_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v));
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t atoms_add(uint32_t saddr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(saddr), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ uint32_t ld_shared_u32(uint32_t saddr) {
  uint32_t v;
  asm volatile("ld.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(saddr) : "memory");
  return v;
}

__device__ __forceinline__ uint2 ld_shared_v2(uint32_t saddr) {
  uint2 v;
  asm volatile("ld.shared::cta.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(saddr) : "memory");
  return v;
}

__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(smem_u32(b)),
      "r"(parity), "r"(0x989680u)
      : "memory");
}
// same, on a 32-bit shared address
__device__ __forceinline__ void mbar_wait_s(uint32_t b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE_%=;\n\t"
      "bra WAIT_%=;\n\t"
      "DONE_%=:\n\t}" ::"r"(b),
      "r"(parity), "r"(0x989680u)
      : "memory");
}
__device__ __forceinline__ void ring_release_s(uint32_t empty_bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(empty_bar) : "memory");
}
__device__ __forceinline__ uint4 lds128(uint32_t saddr) {
  uint4 r;
  asm volatile("ld.shared::cta.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(saddr) : "memory");
  return r;
}
// predicated shared atomic add (returns old, or `dflt` when !p)
__device__ __forceinline__ uint32_t atoms_add_if(bool p, uint32_t saddr, uint32_t v, uint32_t dflt) {
  uint32_t old = dflt;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q atom.shared::cta.add.u32 %0, [%1], %3;\n\t}"
               : "+r"(old) : "r"(saddr), "r"((uint32_t)p), "r"(v) : "memory");
  return old;
}
// predicated L2 reduction with a cache policy
__device__ __forceinline__ void red_add_u64_if(bool p, unsigned long long *a, unsigned long long v, uint64_t pol) {
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %0, 0;\n\t@q red.global.add.L2::cache_hint.u64 [%1], %2, %3;\n\t}"
               ::"r"((uint32_t)p), "l"(a), "l"(v), "l"(pol) : "memory");
}

// consumer side of a ring stage: order this warp's generic-proxy reads of the stage before the
// producer's next async-proxy (TMA) write into it, then count the warp as done
__device__ __forceinline__ void ring_release(uint64_t *empty_bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_arrive(empty_bar);
}
// 1-D bulk copy global -> shared through the TMA engine, completion counted on `bar`
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// pc -> instruction (a-2, R6): granule map (MODE 0) or binary search over the sorted
// instruction starts (MODE 1); NONE outside every [addr, addr + len)
template <int MODE>
__device__ __forceinline__ uint32_t lookup(const AttrTables &T, uint64_t pc) {
  if (MODE == 0) {
    uint64_t g = (pc - T.base) >> T.gshift;  // pc < base wraps to a huge g
    return g < T.n_gran ? __ldg(T.gmap + g) : NONE;
  } else {
    if (!(pc >= T.base && pc < T.end)) return NONE;
    uint32_t lo = 0, hi = T.n_inst;
    while (lo < hi) {
      uint32_t mid = (lo + hi) >> 1;
      if (__ldg(T.inst_addr + mid) <= pc) lo = mid + 1; else hi = mid;
    }
    uint32_t j = lo - 1;  // lo >= 1 because pc >= base = inst_addr[0]
    return pc - __ldg(T.inst_addr + j) < (uint64_t)__ldg(T.inst_len + j) ? j : NONE;
  }
}

// ---- TMA ring geometry ----------------------------------------------------------------------------
template <int NC, int R, int NST>
struct Ring {
  static constexpr int kConsumers = NC, kPerLane = R, kStages = NST;
  static constexpr int kTile = NC * 32 * R;  // records per stage
  static constexpr size_t kBytes = (size_t)NST * kTile * 16;
  static constexpr int kThreads = (NC + 1) * 32;
};

// producer warp body: one elected lane drives the bulk-copy engine over this CTA's tiles
// (tiles t0, t0+step, ... < t1 of S records; the last tile of the stream may be partial)
// ring stress testing (gpa_set_ring_stress): pseudo-random sleeps of 0..(stress*0.5) us that let the
// producer run ahead of slow consumers and vice versa; 0 in production
__device__ __forceinline__ void stress_sleep(uint32_t stress, uint32_t a, uint32_t b) {
  if (stress) {
    uint32_t h = (a * 0x9E3779B1u) ^ (b * 0x85EBCA77u) ^ stress;
    h ^= h >> 15;
    h *= 0x2C1B3C6Du;
    h ^= h >> 12;
    if (h & 1u) __nanosleep((h >> 8) % (stress * 500u + 1u));
  }
}

template <class RG>
__device__ __forceinline__ void ring_produce(uint4 *ring, uint64_t *full, uint64_t *empty, const uint4 *rec,
                                             uint64_t n, uint64_t t0, uint64_t step, uint64_t t1, uint32_t stress = 0) {
  constexpr int S = RG::kTile, NST = RG::kStages;
  uint64_t policy;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
  uint32_t it = 0;
  for (uint64_t tile = t0; tile < t1; tile += step, ++it) {
    uint32_t st = it % NST, ph = (it / NST) & 1;
    if (it >= (uint32_t)NST) mbar_wait(empty + st, ph ^ 1);
    stress_sleep(stress, (uint32_t)tile, 0xFFFFu);
    uint64_t left = n - tile * S;
    uint32_t bytes = (uint32_t)((left < (uint64_t)S ? left : (uint64_t)S) * 16);
    mbar_arrive_expect_tx(full + st, bytes);
    bulk_g2s(ring + (size_t)st * S, rec + tile * S, bytes, full + st, policy);
  }
}

// Producer with the tile index published in tile_of[stage] before arming the stage (the arrive
// releases it; consumers read it after their acquiring wait).  Dynamic order: the next tile of the
// whole stream comes from a global counter (atomicAdd), so CTAs that start late or run slowly take
// fewer tiles.  The end is a stage armed without a copy whose tile index is >= ntiles.
template <class RG>
__device__ __forceinline__ void ring_produce_dyn(uint4 *ring, uint64_t *full, uint64_t *empty, uint32_t *tile_of,
                                                 const uint4 *rec, uint64_t n, uint32_t ntiles, unsigned int *ctr,
                                                 uint32_t stress = 0) {
  constexpr int S = RG::kTile, NST = RG::kStages;
  uint64_t policy;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
  // ctr == nullptr: static order (tile blockIdx.x + it * gridDim.x), else the index of the
  // following tile is fetched one stage ahead, so the atomic's round trip overlaps the wait
  uint32_t next = ctr ? atomicAdd(ctr, 1u) : blockIdx.x;
  for (uint32_t it = 0;; ++it) {
    uint32_t st = it % NST, ph = (it / NST) & 1;
    const uint32_t tile = next;
    if (tile < ntiles) next = ctr ? atomicAdd(ctr, 1u) : tile + gridDim.x;
    if (it >= (uint32_t)NST) mbar_wait(empty + st, ph ^ 1);
    stress_sleep(stress, tile, 0xFFFFu);
    tile_of[st] = tile;
    if (tile >= ntiles) {
      mbar_arrive(full + st);  // end marker: no bytes
      return;
    }
    uint64_t left = n - (uint64_t)tile * S;
    uint32_t bytes = (uint32_t)((left < (uint64_t)S ? left : (uint64_t)S) * 16);
    mbar_arrive_expect_tx(full + st, bytes);
    bulk_g2s(ring + (size_t)st * S, rec + (uint64_t)tile * S, bytes, full + st, policy);
  }
}

__device__ __forceinline__ void ring_init(uint64_t *full, uint64_t *empty, int nst, uint32_t consumers) {
  if (threadIdx.x == 0) {
    for (int q = 0; q < nst; q++) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, consumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}

// ---- scans ---------------------------------------------------------------------------------
constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 2;
constexpr int kScanTile = kScanThreads * kScanItems;

// block-wide exclusive scan of one u32 per thread; returns the block total in *total
__device__ __forceinline__ uint32_t block_exscan(uint32_t v, uint32_t *total) {
  __shared__ uint32_t wsum[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  __syncthreads();
  if (lane == 31) wsum[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t s = lane < nw ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(kFull, s, o);
      if (lane >= o) s += y;
    }
    wsum[lane] = s;  // inclusive warp-prefix
  }
  __syncthreads();
  *total = wsum[nw - 1];
  return x - v + (wid ? wsum[wid - 1] : 0);
}

// multi-block exclusive scan of u32 values in place (k_scan_reduce -> k_scan_top -> k_scan_down;
// up to 65536 tiles of kScanTile); the grand total goes to *total
__global__ void __launch_bounds__(kScanThreads) k_scan_reduce(const uint32_t *v, uint64_t m, uint32_t *bs) {
  uint64_t i0 = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < kScanItems; q++) s += i0 + q < m ? v[i0 + q] : 0;
  uint32_t tot;
  block_exscan(s, &tot);
  if (threadIdx.x == 0) bs[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_top(uint32_t *bs, uint32_t nb, unsigned long long *total) {
  uint32_t running = 0;
  for (uint32_t base = 0; base < nb; base += blockDim.x) {
    uint32_t i = base + threadIdx.x;
    uint32_t v = i < nb ? bs[i] : 0, tot;
    uint32_t ex = block_exscan(v, &tot);
    if (i < nb) bs[i] = running + ex;
    running += tot;
  }
  if (threadIdx.x == 0) total[0] = running;
}

__global__ void __launch_bounds__(kScanThreads) k_scan_down(uint32_t *v, uint64_t m, const uint32_t *bs) {
  uint64_t i0 = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  uint32_t x[kScanItems], s = 0;
#pragma unroll
  for (int q = 0; q < kScanItems; q++) {
    x[q] = i0 + q < m ? v[i0 + q] : 0;
    s += x[q];
  }
  uint32_t tot;
  uint32_t ex = block_exscan(s, &tot) + bs[blockIdx.x];
#pragma unroll
  for (int q = 0; q < kScanItems; q++) {
    if (i0 + q < m) v[i0 + q] = ex;
    ex += x[q];
  }
}

// single-pass exclusive scan of u32 values in place (decoupled look-back): each CTA takes the
// next tile by ticket, publishes its aggregate, then warp 0 walks back over the predecessors'
// published (aggregate | inclusive) words 32 at a time until it meets an inclusive prefix, and
// publishes its own inclusive prefix.  One read and one write per element.
#ifndef GPA_SCAN_ITEMS
#define GPA_SCAN_ITEMS 24  // 8: f4 on B3 2.36 ms, 16: 2.30, 24: 2.27 (fewer tiles in the look-back chain)
#endif
constexpr int kLbThreads = 512, kLbItems = GPA_SCAN_ITEMS, kLbTile = kLbThreads * kLbItems;
static_assert(kLbItems % 4 == 0, "scan items per thread: whole 16-B vectors");

__global__ void __launch_bounds__(kLbThreads) k_scan_lb(uint32_t *__restrict__ v, uint64_t m,
                                                       unsigned long long *state, uint32_t *ctr,
                                                       unsigned long long *total) {
  const unsigned long long kLbAgg = 1ull << 32, kLbInc = 2ull << 32;  // published: aggregate / inclusive
  __shared__ uint32_t s_tile, s_excl;
  if (threadIdx.x == 0) s_tile = atomicAdd(ctr, 1u);
  __syncthreads();
  const uint32_t tile = s_tile;
  const uint64_t i0 = (uint64_t)tile * kLbTile + (uint64_t)threadIdx.x * kLbItems;
  uint32_t x[kLbItems], sum = 0;
  if (i0 + kLbItems <= m) {
#pragma unroll
    for (int k4 = 0; k4 < kLbItems / 4; k4++) {
      const uint4 a = *reinterpret_cast<const uint4 *>(v + i0 + 4 * k4);
      x[4 * k4] = a.x; x[4 * k4 + 1] = a.y; x[4 * k4 + 2] = a.z; x[4 * k4 + 3] = a.w;
    }
  } else {
#pragma unroll
    for (int q = 0; q < kLbItems; q++) x[q] = i0 + q < m ? v[i0 + q] : 0;
  }
#pragma unroll
  for (int q = 0; q < kLbItems; q++) sum += x[q];
  uint32_t agg;
  uint32_t ex = block_exscan(sum, &agg);
  volatile unsigned long long *vs = state;
  if (threadIdx.x == 0) vs[tile] = (tile == 0 ? kLbInc : kLbAgg) | agg;
  if (tile > 0 && threadIdx.x < 32) {
    const int lane = threadIdx.x;
    uint32_t excl = 0;
    int64_t p = (int64_t)tile - 1;
    for (;;) {
      const int64_t q = p - lane;
      const unsigned long long w = q >= 0 ? vs[q] : kLbInc;  // before the first tile: prefix 0
      const uint32_t flag = (uint32_t)(w >> 32);
      if (__any_sync(kFull, flag == 0)) continue;           // a predecessor has not published yet
      const unsigned inc = __ballot_sync(kFull, flag == 2);
      const int stop = inc ? __ffs(inc) - 1 : 31;
      uint32_t val = lane <= stop ? (uint32_t)w : 0u;
#pragma unroll
      for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(kFull, val, o);
      excl += val;
      if (inc) break;
      p -= 32;
    }
    if (lane == 0) {
      s_excl = excl;
      vs[tile] = kLbInc | (uint32_t)(excl + agg);
    }
  }
  __syncthreads();
  uint32_t run = (tile ? s_excl : 0u) + ex;
  if (i0 + kLbItems <= m) {
    uint32_t y[kLbItems];
#pragma unroll
    for (int q = 0; q < kLbItems; q++) {
      y[q] = run;
      run += x[q];
    }
#pragma unroll
    for (int k4 = 0; k4 < kLbItems / 4; k4++)
      *reinterpret_cast<uint4 *>(v + i0 + 4 * k4) = make_uint4(y[4 * k4], y[4 * k4 + 1], y[4 * k4 + 2], y[4 * k4 + 3]);
  } else {
#pragma unroll
    for (int q = 0; q < kLbItems; q++)
      if (i0 + q < m) {
        v[i0 + q] = run;
        run += x[q];
      }
  }
  const uint64_t n_tiles = (m + kLbTile - 1) / kLbTile;
  if (threadIdx.x == 0 && tile == (n_tiles ? n_tiles - 1 : 0)) total[0] = (uint32_t)((tile ? s_excl : 0u) + agg);
}

}  // namespace

void count_launches(uint64_t k);

namespace {
// host side: exclusive scan of m u32 values (m <= 2^27; v 16-B aligned) in place on `st`; the
// total lands in *total (device); scratch = kScanScratchWords u32
inline cudaError_t scan_u32(uint32_t *v, uint64_t m, uint32_t *scratch, unsigned long long *total, cudaStream_t st) {
  uint64_t nt = (m + kLbTile - 1) / kLbTile;
  if (nt > 32768) return cudaErrorInvalidValue;
  if (nt == 0) nt = 1;
  unsigned long long *state = reinterpret_cast<unsigned long long *>(scratch);
  uint32_t *ctr = scratch + 2 * nt;
  cudaError_t e = cudaMemsetAsync(scratch, 0, (2 * nt + 1) * 4, st);
  if (e != cudaSuccess) return e;
  k_scan_lb<<<(unsigned)nt, kLbThreads, 0, st>>>(v, m, state, ctr, total);
  count_launches(1);
  return cudaGetLastError();
}
}  // namespace
}  // namespace gpa