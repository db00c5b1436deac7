// k_attr.cu — a-1..a-3: PC-sample decode, pc -> instruction lookup, per-instruction x
// stall-reason histogram (§4.2 P:365-374 "an instruction address, a stall reason,
// and a count"; §4.5 P:475-479 raw metric = sum; §5 P:614-617 disjoint relocated ranges).
//
// attr_choice() picks the kernel of a call (numbering of gpa_set_attr_kernel):
// from 2^20 records K_attr_direct (9) where the whole module fits shared memory (C2); else from
// max(4e6, 8 x n_inst) records on (granule-map structures) a large-call kernel with a per-call
// plan (sample -> shared-memory hot set); below that register streaming (1).  A call is one pool
// allocation, one fill kernel, the plan kernels, the main kernel and one fold (k_fold_all: the
// CTAs' tables are stored as slabs and summed byte-wise, acc and the granule scratch folded).
//
// Why privatise: measured on B200 (tools/microbench.cu), u64 reductions into L2 cost ~1.3 SM
// cycles of LSU issue per lane (~1.9e11/s at spread addresses), far below the ~4.1e11 records/s
// the HBM roofline allows; shared-memory u32 atomics sustain ~1.3e12/s.  Every large-call kernel
// streams record tiles HBM -> shared memory with 1-D TMA bulk copies (cp.async.bulk, L2
// evict-first) into an mbarrier ring driven by one producer lane; consumer warps read their
// records from shared memory, free the stage (proxy fence + arrive) and count hot records with
// shared atomics, the rest with L2 reductions.  Results are identical for every kernel.
//
//  7 K_attr_probe (structures up to 2^18 granules, C3/C4): a 2-way set-associative table of 8192
//     granules in shared memory (key = the granule) with a row of 12 byte counters each: the record
//     path has no global load at all (probe, shared atomic or L2 reduction into a granule-indexed
//     scratch); k_sample_gran / k_place choose the table per plan.
//  8 K_attr_code32 (larger structures, C5): 102 400 byte-packed (instruction, slot) bins found
//     through a 32-bit per-granule code (base << 12 | hot-slot mask); non-hot records go to the
//     granule-indexed scratch.  k_sample_bins / k_vhist / k_pick / k_assign_bins / k_codemap32
//     choose the bins per plan.
//  9 K_attr_direct (modules of up to ~13.8 k granules, C2): every granule's 12 byte counters in
//     shared memory, no plan; also k_attr_prof_code (f1 instruction rows with a plan's hot bins).
//  Byte / half-word counters: a carry out of a packed counter is visible in the atomic's old value
//  and repaid exactly in L2 (acc), so any count is exact.  Plans are reusable (gpa_attr_plan_*).
//  3 / 5 / 6 K_attr_bins<32 / 8 / 16>: the round-1 kernel (64-bit code map: instruction + hot
//     info) with u32 / u8 / u16 bins.  4 K_attr_hot: hot 12-slot rows.  2 K_attr_tma: TMA ring,
//     warp-aggregated L2 reductions only.  1 K_attr_stream: register streaming (small calls and
//     binary-search structures).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <stdint.h>
#include <stdlib.h>

#include "gpa_internal.cuh"
#include "kern_common.cuh"

// record paths: predicated atomics instead of hot / cold branches (1) or branches (0); K_attr_code32
// measured 12.25 / 12.12 ms with branches against 12.38 / 12.40 ms predicated (C5, same box)
#ifndef GPA_CODE_PRED
#define GPA_CODE_PRED 0
#endif
// K_attr_probe: predicated (C4 2.69 -> 2.59 ms, 0.91 -> 0.94 of peak; C3 unchanged)
#ifndef GPA_PROBE_PRED
#define GPA_PROBE_PRED 1
#endif
// K_attr_code32: unconditional code gather (sentinel entry) and 32-bit scratch row offsets
#ifndef GPA_DIRECT_MIN  // records from which K_attr_direct runs (structures it holds whole)
#define GPA_DIRECT_MIN (1 << 20)
#endif
#ifndef GPA_CODE_LEAN
#define GPA_CODE_LEAN 1
#endif
// L2 evict-last hint on the code gathers: off (C5 12.01 -> 11.95 ms without it: the hint's policy
// register is re-staged into uniform registers per gather)
#ifndef GPA_CODE_HINT
#define GPA_CODE_HINT 0
#endif

namespace gpa {
namespace {

constexpr unsigned FULL = 0xFFFFFFFFu;
std::atomic<int> g_ring_stress{0};  // gpa_set_ring_stress (testing): TMA-ring timing perturbation, 0 = off


// Warp-aggregated accumulate: lanes with equal `key` sum their counts; the lowest lane of
// each group issues one u64 reduction.  key == FULL marks an idle lane.
__device__ __forceinline__ void warp_accumulate(uint32_t key, uint32_t cnt, unsigned long long *target) {
  const int lane = threadIdx.x & 31;
  unsigned peers = __match_any_sync(FULL, key);
  int gmax = __reduce_max_sync(FULL, (unsigned)__popc(peers));
  unsigned long long total = cnt;
  if (gmax > 1) {
    unsigned rest = peers & ~(1u << lane);
    for (int t = 1; t < gmax; t++) {
      int src = rest ? __ffs(rest) - 1 : lane;
      uint32_t v = __shfl_sync(FULL, cnt, src);
      if (rest) {
        total += v;
        rest &= rest - 1;
      }
    }
  }
  if (key != FULL && lane == __ffs(peers) - 1) red_add_u64(target, total);
}

__device__ __forceinline__ void accumulate_one(uint32_t i, uint4 v, bool live, unsigned long long *H,
                                               unsigned long long *U) {
  uint32_t cnt = v.z, stall = v.w & 0xFFFFu;
  uint32_t slot = stall < GPA_VALID_SLOTS ? stall : GPA_SLOT_INVALID;
  uint32_t key = (!live || cnt == 0) ? FULL : (i == NONE ? (0xFFFFFFE0u | slot) : (i << 4 | slot));
  warp_accumulate(key, cnt, i == NONE ? U + slot : H + ((uint64_t)i << 4 | slot));
}

// ---- K_attr_stream: register streaming ---------------------------------------------------------
constexpr int kStreamThreads = 256, kStreamUnroll = 4;

template <int MODE, bool REC>
__global__ void __launch_bounds__(kStreamThreads)
    k_attr_stream(AttrTables T, const uint4 *__restrict__ rec, uint64_t n, unsigned long long *__restrict__ H,
                  unsigned long long *__restrict__ U, uint32_t *__restrict__ rec_inst) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * kStreamThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * kStreamThreads) >> 5;
  for (uint64_t base = warp * 32 * kStreamUnroll; base < n; base += nwarps * 32 * kStreamUnroll) {
    uint4 v[kStreamUnroll];
#pragma unroll
    for (int u = 0; u < kStreamUnroll; u++) {
      uint64_t k = base + (uint64_t)u * 32 + lane;
      v[u] = k < n ? ld_stream(rec + k) : make_uint4(0, 0, 0, 0);
    }
    uint32_t inst[kStreamUnroll];
#pragma unroll
    for (int u = 0; u < kStreamUnroll; u++) inst[u] = lookup<MODE>(T, ((uint64_t)v[u].y << 32) | v[u].x);
#pragma unroll
    for (int u = 0; u < kStreamUnroll; u++) {
      uint64_t k = base + (uint64_t)u * 32 + lane;
      if (REC && k < n) rec_inst[k] = inst[u];
      accumulate_one(inst[u], v[u], k < n, H, U);
    }
  }
}

// ---- K_attr_tma: TMA ring + warp-aggregated L2 reductions ----------------------------------------
using RingTma = Ring<16, 4, 4>;

template <int MODE, bool REC>
__global__ void __launch_bounds__(RingTma::kThreads, 1)
    k_attr_tma(AttrTables T, const uint4 *__restrict__ rec, uint64_t n, unsigned long long *__restrict__ H,
               unsigned long long *__restrict__ U, uint32_t *__restrict__ rec_inst) {
  extern __shared__ __align__(128) uint8_t smem[];
  using RG = RingTma;
  constexpr int S = RG::kTile, NST = RG::kStages, NC = RG::kConsumers, R = RG::kPerLane;
  uint4 *ring = reinterpret_cast<uint4 *>(smem);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + RG::kBytes);
  uint64_t *empty = full + NST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  ring_init(full, empty, NST, NC);
  __syncthreads();
  if (warp == NC) {
    if (lane == 0) ring_produce<RG>(ring, full, empty, rec, n, blockIdx.x, gridDim.x, (n + RG::kTile - 1) / RG::kTile);
    return;
  }
  const uint64_t ntiles = (n + S - 1) / S;
  uint32_t it = 0;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    uint32_t st = it % NST, ph = (it / NST) & 1;
    mbar_wait(full + st, ph);
    uint64_t left = n - tile * S;
    uint32_t m = (uint32_t)(left < (uint64_t)S ? left : (uint64_t)S);
    uint4 v[R];
#pragma unroll
    for (int u = 0; u < R; u++) v[u] = ring[(size_t)st * S + (u * NC + warp) * 32 + lane];
    __syncwarp();
    if (lane == 0) ring_release(empty + st);
    uint32_t inst[R];
#pragma unroll
    for (int u = 0; u < R; u++) inst[u] = lookup<MODE>(T, ((uint64_t)v[u].y << 32) | v[u].x);
#pragma unroll
    for (int u = 0; u < R; u++) {
      uint32_t j = (uint32_t)(u * NC + warp) * 32 + lane;
      if (REC && j < m) rec_inst[tile * S + j] = inst[u];
      accumulate_one(inst[u], v[u], j < m, H, U);
    }
  }
}

// ---- K_attr_hot: heavy-hitter rows in shared memory ---------------------------------------------
constexpr int kHotSlots = GPA_VALID_SLOTS;
constexpr int kHotRows = 3328;                     // 3328 x 12 x 4 B = 156 KiB
using RingHot = Ring<16, 2, 4>;                    // 4 x 16 KiB stages
constexpr int kLook = 2;                           // tiles of records + codes in flight ahead
#ifndef GPA_SAMPLE_CHUNK_LOG
#define GPA_SAMPLE_CHUNK_LOG 7  // 16 384 runs of 128 records: the sample spans ~16 k launch bursts (tools/sample_sweep.sh)
#endif
constexpr int kSampleChunk = 1 << GPA_SAMPLE_CHUNK_LOG, kSampleChunks = (1 << 21) / kSampleChunk;
constexpr uint64_t kHotMinRecords = (uint64_t)kSampleChunks * kSampleChunk;
#ifndef GPA_SAMPLE_DIV
#define GPA_SAMPLE_DIV 256
#endif
#ifndef GPA_SAMPLE_MAX_LOG
#define GPA_SAMPLE_MAX_LOG 21
#endif
constexpr int kVBins = 4096;

__global__ void k_sample(AttrTables T, const uint4 *__restrict__ rec, uint64_t n, uint32_t *__restrict__ scnt) {
  const uint64_t total = (uint64_t)kSampleChunks * kSampleChunk;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c = x / kSampleChunk, o = x % kSampleChunk;
    uint64_t k = c * (n - kSampleChunk) / (kSampleChunks - 1) + o;
    uint4 v = ld_stream(rec + k);
    uint32_t i = lookup<0>(T, ((uint64_t)v.y << 32) | v.x);
    if (i != NONE) atomicAdd(scnt + i, 1u);
  }
}

// histogram of the per-instruction sample counts (capped at kVBins-1), block-privatised
__global__ void __launch_bounds__(1024) k_vhist(const uint32_t *__restrict__ scnt, uint32_t n_inst,
                                                uint32_t *__restrict__ V) {
  __shared__ uint32_t h[kVBins];
  for (int c = threadIdx.x; c < kVBins; c += blockDim.x) h[c] = 0;
  __syncthreads();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_inst; i += gridDim.x * blockDim.x) {
    uint32_t c = scnt[i];
    if (c) atomicAdd(h + (c < kVBins - 1 ? c : kVBins - 1), 1u);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < kVBins; c += blockDim.x)
    if (h[c]) atomicAdd(V + c, h[c]);
}

// thr[0] = smallest t >= 1 whose suffix count sum_{c >= t} V[c] fits in `rows` (or the top
// bucket if even it does not fit; k_assign then caps the rows); thr[1] = 0 (rows assigned).
// One CTA of 1024 threads; thread t owns the 4 bins c = 4095-4t .. 4092-4t.
__global__ void __launch_bounds__(1024) k_pick(const uint32_t *__restrict__ V, uint32_t *__restrict__ thr,
                                               uint32_t rows) {
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t n_over;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) n_over = 0;
  uint32_t v[4], s = 0;
#pragma unroll
  for (int q = 0; q < 4; q++) {
    v[q] = V[kVBins - 1 - (4 * t + q)];
    s += v[q];
  }
  uint32_t x = s;  // inclusive scan over threads = suffix sums over bins
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t z = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(FULL, z, o);
      if (lane >= o) z += y;
    }
    wsum[lane] = z;
  }
  __syncthreads();
  uint32_t run = x - s + (w ? wsum[w - 1] : 0);
  uint32_t over = 0;  // bins c >= 1 whose suffix sum exceeds rows
#pragma unroll
  for (int q = 0; q < 4; q++) {
    run += v[q];
    int c = kVBins - 1 - (4 * t + q);
    over += (c >= 1 && run > rows);
  }
  if (over) atomicAdd(&n_over, over);
  __syncthreads();
  if (t == 0) {
    uint32_t th = 1 + n_over;  // suffix sums are non-increasing in c
    thr[0] = th > kVBins - 1 ? kVBins - 1 : th;
    thr[1] = 0;
  }
}

__global__ void k_assign(const uint32_t *__restrict__ scnt, uint32_t n_inst, uint32_t *__restrict__ thr,
                         uint32_t *__restrict__ hot_row, uint32_t *__restrict__ row_inst, uint32_t rows) {
  const uint32_t t = thr[0];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_inst; i += gridDim.x * blockDim.x) {
    uint32_t c = scnt[i], r = NONE;
    if (c && (c < kVBins - 1 ? c : kVBins - 1) >= t) {
      uint32_t q = atomicAdd(thr + 1, 1u);
      if (q < rows) {
        r = q;
        row_inst[q] = i;
      }
    }
    hot_row[i] = r;
  }
}

// code: cold instruction i -> i << 4 (low nibble 0), hot row r -> r << 4 | 1, unmapped -> ~0
__global__ void k_codemap(const uint32_t *__restrict__ gmap, uint64_t n_gran, const uint32_t *__restrict__ hot_row,
                          uint32_t *__restrict__ code) {
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_gran; g += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t m = gmap[g];
    uint32_t r = m == NONE ? NONE : hot_row[m];
    code[g] = m == NONE ? 0xFFFFFFFFu : (r != NONE ? (r << 4 | 1u) : (m << 4));
  }
}

template <class RG, int ROWS, bool REC>
__global__ void __launch_bounds__(RG::kThreads, 1)
    k_attr_hot(uint64_t base, uint64_t n_gran, uint32_t gshift, const uint32_t *__restrict__ code,
               const uint4 *__restrict__ rec, uint64_t n, unsigned long long *__restrict__ H,
               unsigned long long *__restrict__ U, uint32_t *__restrict__ rec_inst,
               const uint32_t *__restrict__ row_inst, const uint32_t *__restrict__ thr) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int S = RG::kTile, NST = RG::kStages, NC = RG::kConsumers, R = RG::kPerLane, D = kLook + 1;
  constexpr size_t TAB = (size_t)ROWS * kHotSlots * 4;
  uint4 *ring = reinterpret_cast<uint4 *>(smem);
  uint32_t *tab = reinterpret_cast<uint32_t *>(smem + RG::kBytes);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + RG::kBytes + TAB);
  uint64_t *empty = full + NST;
  const uint32_t tab_s = smem_u32(tab);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t ntiles = (n + S - 1) / S;
  const uint32_t nhot = min(thr[1], (uint32_t)ROWS);
  for (uint32_t x = threadIdx.x; x < nhot * kHotSlots; x += blockDim.x) tab[x] = 0;
  ring_init(full, empty, NST, NC);
  __syncthreads();
  if (warp == NC) {
    if (lane == 0) ring_produce<RG>(ring, full, empty, rec, n, blockIdx.x, gridDim.x, (n + RG::kTile - 1) / RG::kTile);
    return;
  }
  uint4 v[D][R];
  uint32_t c[D][R];
  const uint64_t G = gridDim.x;
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
      uint64_t g = ((((uint64_t)vv[u].y << 32) | vv[u].x) - base) >> gshift;
      cc[u] = g < n_gran ? __ldg(code + g) : 0xFFFFFFFFu;
    }
  };
#pragma unroll
  for (int q = 0; q < kLook; q++)
    if (blockIdx.x + q * G < ntiles) fetch(q, v[q], c[q]);
  for (uint32_t it0 = 0;; it0 += D) {
#pragma unroll
    for (int q = 0; q < D; q++) {
      const uint32_t it = it0 + q;
      const uint64_t tile = blockIdx.x + it * G;
      if (tile >= ntiles) goto done;
      if (tile + kLook * G < ntiles) fetch(it + kLook, v[(q + kLook) % D], c[(q + kLook) % D]);
      const uint64_t left = n - tile * S;
      const uint32_t m = (uint32_t)(left < (uint64_t)S ? left : (uint64_t)S);
      uint32_t old[R];
      bool added[R];
#pragma unroll
      for (int u = 0; u < R; u++) {
        const uint32_t j = (uint32_t)(u * NC + warp) * 32 + lane;
        const uint32_t cd = c[q][u], cnt = v[q][u].z, stall = v[q][u].w & 0xFFFFu;
        const uint32_t slot = stall < GPA_VALID_SLOTS ? stall : GPA_SLOT_INVALID;
        const uint32_t nib = cd & 15u;
        const bool live = j < m;
        if (REC && live)
          rec_inst[tile * S + j] = nib == 15u ? NONE : (nib == 1u ? __ldg(row_inst + (cd >> 4)) : (cd >> 4));
        old[u] = 0;
        added[u] = false;
        if (live) {
          if (nib == 1u && slot < (uint32_t)kHotSlots) {
            old[u] = atoms_add(tab_s + ((cd >> 4) * kHotSlots + slot) * 4, cnt);
            added[u] = true;
          } else if (nib == 0u) {
            red_add_u64(H + (cd | slot), cnt);
          } else if (nib == 15u) {
            red_add_u64(U + slot, cnt);
          } else {  // hot instruction, invalid stall slot
            red_add_u64(H + ((uint64_t)__ldg(row_inst + (cd >> 4)) << 4 | slot), cnt);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < R; u++) {
        // old + cnt wrapped the u32 shared counter: repay 2^32 in L2
        if (added[u] && old[u] + v[q][u].z < old[u])
          red_add_u64(H + ((uint64_t)__ldg(row_inst + (c[q][u] >> 4)) << 4 | (v[q][u].w & 0xFFFFu)), 1ull << 32);
      }
    }
  }
done:
  asm volatile("bar.sync 1, %0;" ::"r"(NC * 32) : "memory");
  for (uint32_t x = threadIdx.x; x < nhot * kHotSlots; x += NC * 32) {
    uint32_t val = tab[x];
    if (val) red_add_u64(H + ((uint64_t)__ldg(row_inst + x / kHotSlots) << 4 | (x % kHotSlots)), val);
  }
}

// ---- K_attr_bins: heavy-hitter BINS in shared memory (default) ---------------------------------
// Same pipeline as K_attr_hot, but the shared table holds individual (instruction, slot) bins
// rather than whole 12-slot rows: 128 KiB cover the 32 768 most-sampled bins (C5: ~70 % of
// records vs 67 % for 3 328 rows in 156 KiB), so fewer records fall back to L2 reductions.
// Per call: k_sample_bins counts sampled records per bin; the top kHotBins bins are chosen by
// the same value histogram / threshold; k_assign_bins gives each instruction a 12-bit mask of
// its hot slots and a base index (atomic cursor) and records bin_of[idx] = inst<<4 | slot;
// k_codemap_bins builds a per-call 64-bit code per granule: low word inst<<4 (or ~0 unmapped),
// high word base<<12 | mask (0 for unmapped granules and instructions without hot bins).  A record's table index is base + popc(mask & below(slot)).
#ifndef GPA_HOT_BINS
#define GPA_HOT_BINS 32768
#endif
constexpr int kHotBins = GPA_HOT_BINS;               // x 4 B = 128 KiB (the rest of the SM's 256 KiB is L1 for the code-map gathers)
static_assert((kHotBins & (kHotBins - 1)) == 0, "GPA_HOT_BINS: shared words must be a power of two");
static_assert((uint64_t)kHotBins * 4 <= (1u << 20), "GPA_HOT_BINS: byte-bin index must fit the 20-bit code base field");
static_assert((size_t)kHotBins * 4 + 2 * 31 * 64 * 16 + 64 <= 227 * 1024, "GPA_HOT_BINS: table + ring exceed shared memory");
// 31 consumer warps x 2 records per lane (tile = 1984 records, 2 x 31 KiB stages) + the producer
// = 1024 threads, 1 tile of lookahead: C5 15.6 -> 14.9 ms, C4 3.71 -> 3.21 ms against 16 x 2 x 4
// stages with lookahead 2 (DESIGN.md §7 geometry sweep; fewer stage releases per record, each of
// which costs a proxy fence that waits for the warp's outstanding memory operations)
using RingBins = Ring<31, 2, 2>;
constexpr int kLookBins = 1;

// cnt[key] += 1 for every lane whose key != NONE, one atomic per distinct key of the warp (all 32
// lanes must call it: the sample loops run whole warps, chunks x kSampleChunk being a multiple of 32)
__device__ __forceinline__ void sample_add(uint32_t *cnt, uint32_t key) {
  const unsigned peers = __match_any_sync(FULL, key);
  if (key != NONE && (threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1)) atomicAdd(cnt + key, (uint32_t)__popc(peers));
}

// `chunks` runs of kSampleChunk records, evenly spaced over the call's records
__global__ void k_sample_bins(AttrTables T, const uint4 *__restrict__ rec, uint64_t n, uint32_t chunks,
                              uint32_t *__restrict__ scnt) {
  const uint64_t total = (uint64_t)chunks * kSampleChunk;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c = x / kSampleChunk, o = x % kSampleChunk;
    uint64_t k = c * (n - kSampleChunk) / (chunks - 1) + o;
    uint4 v = ld_stream(rec + k);
    uint32_t i = lookup<0>(T, ((uint64_t)v.y << 32) | v.x);
    uint32_t stall = v.w & 0xFFFFu;
    // sampled runs are bursts of one kernel: lanes often share a bin, so one atomic per distinct bin
    // and warp (a hot bin's counter would otherwise serialise thousands of same-address atomics)
    sample_add(scnt, i != NONE && stall < GPA_VALID_SLOTS ? i * kHotSlots + stall : NONE);
  }
}

__global__ void k_assign_bins(const uint32_t *__restrict__ scnt, uint32_t n_inst, uint32_t *__restrict__ thr,
                              uint32_t *__restrict__ hot_info, uint32_t *__restrict__ bin_of, uint32_t K) {
  const uint32_t t = thr[0];
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_inst; i += gridDim.x * blockDim.x) {
    uint32_t mask = 0;
#pragma unroll
    for (int r = 0; r < kHotSlots; r++) {
      uint32_t c = scnt[(uint64_t)i * kHotSlots + r];
      if (c && (c < kVBins - 1 ? c : kVBins - 1) >= t) mask |= 1u << r;
    }
    uint32_t info = 0;
    if (mask) {
      uint32_t k = __popc(mask);
      uint32_t base = atomicAdd(thr + 1, k);
      if (base + k <= K) {
        info = base << 12 | mask;
        for (uint32_t m = mask, q = base; m; m &= m - 1, q++) bin_of[q] = i << 4 | (__ffs(m) - 1);
      }
    }
    hot_info[i] = info;
  }
}

__global__ void k_codemap_bins(const uint32_t *__restrict__ gmap, uint64_t n_gran,
                               const uint32_t *__restrict__ hot_info, unsigned long long *__restrict__ code) {
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_gran; g += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t m = gmap[g];
    code[g] = m == NONE ? 0xFFFFFFFFull : ((unsigned long long)hot_info[m] << 32 | (m << 4));
  }
}

__device__ __forceinline__ uint32_t ldg_keep_u32(const uint32_t *p, uint64_t pol) {
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ unsigned long long ldg_keep(const unsigned long long *p, uint64_t pol) {
  unsigned long long v;
  asm volatile("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ void red_add_u64_keep(unsigned long long *p, unsigned long long v, uint64_t pol) {
  asm volatile("red.global.add.L2::cache_hint.u64 [%0], %1, %2;" ::"l"(p), "l"(v), "l"(pol) : "memory");
}

// Bins packed into 32-bit shared words: BITS = 32 (one bin per word), 16 or 8 (two / four bins
// per word).  Bin idx lives in word idx & (NW-1), part idx / NW (interleaved, so the consecutive
// bins of one instruction fall in different banks).  A packed add of cnt < 2^BITS into part k can
// carry across the part boundaries above it; every carry is visible in the atomic's old value:
// a carry out of part j (< P-1) leaves part j short by 2^BITS and part j+1 one too high, so the
// adder repays R_j += 2^BITS and R_{j+1} -= 1 in L2 (u64, modular), and a carry out of the word
// repays R_{P-1} += 2^BITS.  Final H = L2 repayments + the flushed parts: exact for any count.
template <int BITS>
struct Pack {
  static constexpr int P = 32 / BITS;
  static constexpr uint32_t kBoundary = BITS == 8 ? 0x01010100u : (BITS == 16 ? 0x00010000u : 0u);
  static constexpr uint32_t kPartMask = BITS == 32 ? 0xFFFFFFFFu : ((1u << BITS) - 1u);
};

// repayments go to acc[idx] (u64, one per bin, L2-resident): fire-and-forget reductions with no
// dependent load of the bin's (instruction, slot); k_fold_acc adds acc into H once per call
template <int BITS, int NW>
__device__ __forceinline__ void repay_carries(unsigned long long *acc, uint32_t w, uint32_t old, uint32_t delta,
                                              uint64_t pol) {
  constexpr int P = Pack<BITS>::P;
  const unsigned long long s = (unsigned long long)old + delta;
  const uint32_t cin = old ^ delta ^ (uint32_t)s;  // carry into each bit position
#pragma unroll
  for (int j = 0; j < P; j++) {
    const bool cross = j < P - 1 ? ((cin >> (BITS * (j + 1))) & 1u) : (uint32_t)(s >> 32);
    if (cross) {
      red_add_u64_keep(acc + (uint32_t)j * NW + w, 1ull << BITS, pol);
      if (j < P - 1) red_add_u64_keep(acc + (uint32_t)(j + 1) * NW + w, ~0ull, pol);  // -1 (mod 2^64)
    }
  }
}

// H[bin_of[b]] += acc[b] for every assigned bin
__global__ void k_fold_acc(const unsigned long long *__restrict__ acc, const uint32_t *__restrict__ bin_of,
                           const uint32_t *__restrict__ thr, uint32_t K, unsigned long long *__restrict__ H) {
  const uint32_t nb = min(thr[1], K);
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
    const unsigned long long v = acc[b];
    const uint32_t t = bin_of[b];
    if (v && t != NONE) red_add_u64(H + t, v);  // other streams may add into H concurrently
  }
}

template <class RG, int NW, int BITS, bool REC, int LOOK = kLook>
__global__ void __launch_bounds__(RG::kThreads, 1)
    k_attr_bins(uint64_t base, uint64_t n_gran, uint32_t gshift, const unsigned long long *__restrict__ code,
                const uint4 *__restrict__ rec, uint64_t n, unsigned long long *__restrict__ H,
                unsigned long long *__restrict__ U, uint32_t *__restrict__ rec_inst,
                unsigned long long *__restrict__ acc, const uint32_t *__restrict__ thr) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int S = RG::kTile, NST = RG::kStages, NC = RG::kConsumers, R = RG::kPerLane, D = LOOK + 1;
  constexpr int P = Pack<BITS>::P;
  static_assert((NW & (NW - 1)) == 0, "NW must be a power of two");
  static_assert((uint64_t)NW * P <= (1u << 20), "bin index must fit the code map's 20-bit base field");
  constexpr uint32_t kLogNW = __builtin_ctz(NW);
  uint4 *ring = reinterpret_cast<uint4 *>(smem);
  uint32_t *tab = reinterpret_cast<uint32_t *>(smem + RG::kBytes);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + RG::kBytes + (size_t)NW * 4);
  uint64_t *empty = full + NST;
  const uint32_t tab_s = smem_u32(tab);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t ntiles = (n + S - 1) / S;
  const uint32_t nb = min(thr[1], (uint32_t)NW * P);
  const uint32_t nw = min(nb, (uint32_t)NW);
  for (uint32_t x = threadIdx.x; x < nw; x += blockDim.x) tab[x] = 0;
  ring_init(full, empty, NST, NC);
  __syncthreads();
  if (warp == NC) {
    if (lane == 0) ring_produce<RG>(ring, full, empty, rec, n, blockIdx.x, gridDim.x, (n + RG::kTile - 1) / RG::kTile);
    return;
  }
  uint4 v[D][R];
  unsigned long long c[D][R];
  const uint64_t G = gridDim.x;
  uint64_t keep;  // L2 evict-last for the code map (the record stream is evict-first)
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
  auto fetch = [&](uint32_t it, uint4 *vv, unsigned long long *cc) {
    uint32_t st = it % NST, ph = (it / NST) & 1;
    mbar_wait(full + st, ph);
    const uint4 *src = ring + (size_t)st * S + warp * 32 + lane;
#pragma unroll
    for (int u = 0; u < R; u++) vv[u] = src[u * NC * 32];  // beyond the tile end: masked below
    __syncwarp();
    if (lane == 0) ring_release(empty + st);
#pragma unroll
    for (int u = 0; u < R; u++) {
      uint64_t g = ((((uint64_t)vv[u].y << 32) | vv[u].x) - base) >> gshift;
      cc[u] = g < n_gran ? ldg_keep(code + g, keep) : 0xFFFFFFFFull;  // unmapped: low word ~0, no hot mask
    }
  };
#pragma unroll
  for (int q = 0; q < LOOK; q++)
    if (blockIdx.x + q * G < ntiles) fetch(q, v[q], c[q]);
  for (uint32_t it0 = 0;; it0 += D) {
#pragma unroll
    for (int q = 0; q < D; q++) {
      const uint32_t it = it0 + q;
      const uint64_t tile = blockIdx.x + it * G;
      if (tile >= ntiles) goto done;
      if (tile + LOOK * G < ntiles) fetch(it + LOOK, v[(q + LOOK) % D], c[(q + LOOK) % D]);
      const uint64_t left = n - tile * S;
      const uint32_t m = (uint32_t)(left < (uint64_t)S ? left : (uint64_t)S);
      uint32_t old[R], idx[R], delta[R];
#pragma unroll
      for (int u = 0; u < R; u++) {
        const uint32_t j = (uint32_t)(u * NC + warp) * 32 + lane;
        const uint32_t lo = (uint32_t)c[q][u], hi = (uint32_t)(c[q][u] >> 32);
        const uint32_t cnt = v[q][u].z, stall = v[q][u].w & 0xFFFFu;
        const uint32_t slot = stall < GPA_VALID_SLOTS ? stall : GPA_SLOT_INVALID;
        const bool live = j < m;
        if (REC && live) rec_inst[tile * S + j] = lo == 0xFFFFFFFFu ? NONE : lo >> 4;
        const uint32_t mask = hi & 0xFFFu;
        const bool hot = slot < (uint32_t)kHotSlots && ((mask >> slot) & 1u) && (BITS == 32 || cnt <= Pack<BITS>::kPartMask);
        idx[u] = (hi >> 12) + __popc(mask & ((1u << slot) - 1u));
        old[u] = 0;
        delta[u] = 0;
        if (live) {
          if (hot) {
            delta[u] = BITS == 32 ? cnt : cnt << (BITS * (idx[u] >> kLogNW));
            old[u] = atoms_add(tab_s + (idx[u] & (NW - 1)) * 4, delta[u]);
          } else {
            red_add_u64_keep(lo == 0xFFFFFFFFu ? U + slot : H + (lo | slot), cnt, keep);
            idx[u] = NONE;
          }
        } else {
          idx[u] = NONE;
        }
      }
#pragma unroll
      for (int u = 0; u < R; u++) {
        // a carry across a part boundary or out of the word: repay in L2
        const unsigned long long s = (unsigned long long)old[u] + delta[u];
        const uint32_t crossed = ((old[u] ^ delta[u] ^ (uint32_t)s) & Pack<BITS>::kBoundary) | (uint32_t)(s >> 32);
        if (idx[u] != NONE && crossed) repay_carries<BITS, NW>(acc, idx[u] & (NW - 1), old[u], delta[u], keep);
      }
    }
  }
done:
  asm volatile("bar.sync 1, %0;" ::"r"(NC * 32) : "memory");
  for (uint32_t x = threadIdx.x; x < nw; x += NC * 32) {
    const uint32_t word = tab[x];
#pragma unroll
    for (int p = 0; p < P; p++) {
      const uint32_t val = (word >> (BITS * p)) & Pack<BITS>::kPartMask;
      if (val && (uint32_t)p * NW + x < nb) red_add_u64_keep(acc + (uint32_t)p * NW + x, val, keep);  // coalesced
    }
  }
}

template <int BITS>
cudaError_t launch_bins(const AttrTables &T, const uint4 *rec, uint64_t n, unsigned long long *H,
                        unsigned long long *U, uint32_t *ri, int sm_count, cudaStream_t st) {
  constexpr int NW = kHotBins;                       // shared 32-bit words (128 KiB)
  constexpr uint32_t K = (uint32_t)NW * (32 / BITS);  // bins
  // stream-ordered scratch: scnt[n_inst*12] | hot_info[n_inst] | bin_of[K] | V[4096] | thr[4] | code[n_gran] (u64)
  // | acc[K] (u64)
  const size_t ni = T.n_inst, nbins = ni * kHotSlots;
  size_t words = nbins + ni + K + kVBins + 4;
  words = (words + 1) & ~(size_t)1;  // 8-B align the code map
  uint32_t *w = nullptr;
  cudaError_t e = pool_alloc((void **)&w, words * 4 + T.n_gran * 8 + (size_t)K * 8, st);
  if (e != cudaSuccess) return e;
  uint32_t *scnt = w, *hot_info = w + nbins, *bin_of = hot_info + ni, *V = bin_of + K, *thr = V + kVBins;
  unsigned long long *code = reinterpret_cast<unsigned long long *>(w + words);
  unsigned long long *acc = code + T.n_gran;
  cudaMemsetAsync(acc, 0, (size_t)K * 8, st);
  cudaMemsetAsync(scnt, 0, nbins * 4, st);
  cudaMemsetAsync(V, 0, kVBins * 4, st);
  cudaMemsetAsync(bin_of, 0xFF, (size_t)K * 4, st);  // unassigned table entries map to NONE
  // sample min(2^21, max(2^18, n/256)) records: the pre-pass then stays a small fraction of a
  // mid-size call (C2, 1e7 records)
  const uint64_t ns = std::min<uint64_t>(std::min<uint64_t>((uint64_t)kSampleChunks * kSampleChunk, 1ull << GPA_SAMPLE_MAX_LOG),
                                         std::max<uint64_t>(1ull << 18, n / GPA_SAMPLE_DIV));
  const uint32_t chunks = (uint32_t)std::max<uint64_t>(2, ns / kSampleChunk);
  k_sample_bins<<<sm_count * 4, 256, 0, st>>>(T, rec, n, chunks, scnt);
  k_vhist<<<sm_count, 1024, 0, st>>>(scnt, (uint32_t)nbins, V);
  k_pick<<<1, 1024, 0, st>>>(V, thr, K);
  k_assign_bins<<<sm_count * 2, 256, 0, st>>>(scnt, (uint32_t)ni, thr, hot_info, bin_of, K);
  k_codemap_bins<<<sm_count * 4, 256, 0, st>>>(T.gmap, T.n_gran, hot_info, code);
  using RG = RingBins;
  auto kern = ri ? k_attr_bins<RG, NW, BITS, true, kLookBins> : k_attr_bins<RG, NW, BITS, false, kLookBins>;
  const size_t smem = RG::kBytes + (size_t)NW * 4 + 2 * RG::kStages * 8;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) {
    kern<<<sm_count, RG::kThreads, smem, st>>>(T.base, T.n_gran, T.gshift, code, rec, n, H, U, ri, acc, thr);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) {
    k_fold_acc<<<(K + 255) / 256, 256, 0, st>>>(acc, bin_of, thr, K, H);
    e = cudaGetLastError();
  }
  count_launches(7);
  cudaError_t e2 = cudaFreeAsync(w, st);
  return e != cudaSuccess ? e : e2;
}

// ---- store flush of a CTA's byte-counter table ----------------------------------------------------
// At the end of K_attr_probe / K_attr_code32 every CTA stores its table of packed byte counters to a
// slab of its own (coalesced 16-B stores) instead of one L2 reduction per non-zero counter (up to
// 98 k per CTA, ~15 M per launch, ~75 us at the measured 1.9e11 reductions/s).  k_fold_all then
// sums the slabs byte-wise into acc (byte j of word x = counter 4x + j).
// Words [nw, NWALL) of the slab (table words this plan leaves unused, never zeroed in shared memory)
// are stored as 0.  NWALL is a multiple of 4.
template <uint32_t NWALL>
__device__ __forceinline__ void dump_table(const uint32_t *tab, uint32_t nw, uint32_t *slab, uint32_t nthr) {
  static_assert(NWALL % 4 == 0, "slab rows are stored as 16-B vectors");
  for (uint32_t x = threadIdx.x; x < NWALL / 4; x += nthr) {
    uint4 v = reinterpret_cast<const uint4 *>(tab)[x];
    if (4 * x + 4 > nw) {
      v.x = 4 * x + 0 < nw ? v.x : 0u;
      v.y = 4 * x + 1 < nw ? v.y : 0u;
      v.z = 4 * x + 2 < nw ? v.z : 0u;
      v.w = 4 * x + 3 < nw ? v.w : 0u;
    }
    reinterpret_cast<uint4 *>(slab)[x] = v;
  }
}

// The end of a call in one launch.  Blocks [0, tb): table words, kFoldParts x 32 threads per 32
// words: the CTA slabs of the last launch are summed byte-wise (byte j of word x = counter 4x + j;
// two bytes at a time in 16-bit lanes, <= 256 slabs of 255 per lane before a spill), the parts
// combined in shared memory, then either added to acc (fin == 0: a chunk of a multi-launch call;
// the dynamic tile counter is reset for the next launch) or, with acc, reduced into H through the
// plan (fin == 1: K_attr_probe entry -> granule -> instruction; K_attr_code32 bin -> (instruction,
// slot)).  Blocks [tb, grid) (fin == 1 only): the granule scratch Hg -> H / U (gap granules and
// the out-of-module row -> U).
constexpr int kFoldParts = 8;
struct FoldArgs {
  const uint32_t *dump;
  uint32_t nw, tb;
  int slabs, fin, variant;
  unsigned long long *acc;
  unsigned int *ctr;
  const unsigned long long *best;       // 7
  const uint32_t *bin_of, *thr;         // 8
  const uint32_t *gmap;
  const unsigned long long *Hg;
  uint64_t n_gran;
  unsigned long long *H, *U;
};

__global__ void __launch_bounds__(kFoldParts * 32) k_fold_all(FoldArgs F) {
  __shared__ uint32_t part[kFoldParts][32][4];
  if (blockIdx.x >= F.tb) {  // Hg -> H / U, 16 lanes per granule row
    const uint64_t nb = gridDim.x - F.tb;
    for (uint64_t t = (uint64_t)(blockIdx.x - F.tb) * blockDim.x + threadIdx.x; t < (F.n_gran + 1) * 16; t += nb * blockDim.x) {
      const unsigned long long v = F.Hg[t];
      if (!v) continue;
      const uint64_t g = t >> 4;
      const uint32_t sl = (uint32_t)(t & 15), i = g < F.n_gran ? __ldg(F.gmap + g) : NONE;
      red_add_u64(i == NONE ? F.U + sl : F.H + ((uint64_t)i << 4 | sl), v);
    }
    return;
  }
  const uint32_t wl = threadIdx.x & 31, pt = threadIdx.x >> 5;
  const uint32_t x = blockIdx.x * 32 + wl;
  if (!F.fin && blockIdx.x == 0 && threadIdx.x == 0 && F.ctr) *F.ctr = 0;  // the next launch's tile counter
  uint32_t s4[4] = {0, 0, 0, 0};
  if (x < F.nw) {
    for (int c0 = pt; c0 < F.slabs; c0 += kFoldParts * 256) {
      uint32_t ev = 0, od = 0;  // bytes 0, 2 / 1, 3 in 16-bit lanes
      const int c1 = min(F.slabs, c0 + kFoldParts * 256);
#pragma unroll 8
      for (int c = c0; c < c1; c += kFoldParts) {
        const uint32_t w = __ldcs(F.dump + (size_t)c * F.nw + x);
        ev += w & 0x00FF00FFu;
        od += (w >> 8) & 0x00FF00FFu;
      }
      s4[0] += ev & 0xFFFFu;
      s4[1] += od & 0xFFFFu;
      s4[2] += ev >> 16;
      s4[3] += od >> 16;
    }
  }
#pragma unroll
  for (int j = 0; j < 4; j++) part[pt][wl][j] = s4[j];
  __syncthreads();
  if (pt >= 4 || x >= F.nw) return;
  unsigned long long t = 0;
#pragma unroll
  for (int q = 0; q < kFoldParts; q++) t += part[q][wl][pt];
  const uint32_t bin = 4 * x + pt;  // this thread alone owns the counter (the main kernel's repayments are done)
  if (!F.fin) {
    if (t) F.acc[bin] += t;
    return;
  }
  t += F.acc[bin];
  if (!t) return;
  if (F.variant == 7) {  // acc index = 12 e + slot
    const uint32_t e = bin / GPA_VALID_SLOTS, sl = bin - e * GPA_VALID_SLOTS;
    const unsigned long long b = F.best[e];
    if (!b) return;
    const uint32_t i = F.gmap[0xFFFFFFFFu - (uint32_t)b];  // placed granules are mapped (k_sample_gran)
    red_add_u64(F.H + ((uint64_t)i << 4 | sl), t);
  } else if (F.variant == 9) {  // acc index = 12 g + slot; gap granules -> U
    const uint32_t g = bin / GPA_VALID_SLOTS, sl = bin - g * GPA_VALID_SLOTS;
    if (g >= F.n_gran) return;
    const uint32_t i = F.gmap[g];
    red_add_u64(i == NONE ? F.U + sl : F.H + ((uint64_t)i << 4 | sl), t);
  } else {
    if (bin >= F.thr[1]) return;
    const uint32_t b = F.bin_of[bin];
    if (b != NONE) red_add_u64(F.H + b, t);
  }
}

// fill n 32-bit words at each of up to 4 ranges with a value (16-B aligned ranges)
struct FillSet {
  uint32_t *p[4];
  uint64_t n[4];
  uint32_t v[4];
};
__global__ void k_fill(FillSet F) {
  const uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (uint64_t)gridDim.x * blockDim.x;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const uint32_t v = F.v[j];
    const uint4 v4 = make_uint4(v, v, v, v);
    for (uint64_t x = gt; x < F.n[j] / 4; x += gs) reinterpret_cast<uint4 *>(F.p[j])[x] = v4;
    for (uint64_t x = F.n[j] / 4 * 4 + gt; x < F.n[j]; x += gs) F.p[j][x] = v;
  }
}

// ---- K_attr_probe: granule-keyed rows of byte counters, no global load in the record loop ---------
// Each CTA holds a 2-way set-associative table of kProbeM granules (the key is the granule index
// itself; set = (g ^ g >> 12) mod 4096, one 64-bit shared load returns both ways) and, per entry,
// a row of 12 byte-wide counters (one per valid stall slot).  A hit with count < 256 is added to
// its byte counter with a shared atomic; a carry across a byte boundary or out of the word is
// visible in the atomic's old value and repaid through acc (as for the packed bins above).  Every
// other record is reduced into a granule-indexed scratch histogram Hg[g][slot] in L2 (records
// outside the module into the extra row Hg[n_gran], which folds into U).  So the per-record path
// reads the record from the TMA ring, probes the table and issues one shared atomic or one L2
// reduction: no gather, no wait on global memory; the kernel is issue-bound, so the record path
// is written for a small instruction count.  k_fold_all then adds the slabs, acc and Hg into
// H (instruction = gmap[g]; gap granules -> U).  The table is chosen per call from a sample:
// each set keeps its two most-sampled granules.
constexpr int kProbeSetsLog = 12, kProbeSets = 1 << kProbeSetsLog;  // 4096 sets x 2 ways
constexpr int kProbeM = 2 * kProbeSets;                               // entries: 32 KiB keys + 96 KiB rows
constexpr int kProbeRowBytes = GPA_VALID_SLOTS;                       // byte counter of (e, slot) at 12 e + slot
constexpr int kProbeWords = kProbeM * kProbeRowBytes / 4;
constexpr uint32_t kEmpty = 0xFFFFFFFFu;
#ifndef GPA_PROBE_NC
#define GPA_PROBE_NC 31
#endif
#ifndef GPA_PROBE_R
#define GPA_PROBE_R 3
#endif
#ifndef GPA_PROBE_NST
#define GPA_PROBE_NST 2
#endif
using RingProbe = Ring<GPA_PROBE_NC, GPA_PROBE_R, GPA_PROBE_NST>;

__host__ __device__ __forceinline__ uint32_t probe_set(uint32_t g) { return (g ^ (g >> kProbeSetsLog)) & (kProbeSets - 1); }

// sampled records per mapped granule
__global__ void k_sample_gran(AttrTables T, const uint4 *__restrict__ rec, uint64_t n, uint32_t chunks,
                              uint32_t *__restrict__ gcnt) {
  const uint64_t total = (uint64_t)chunks * kSampleChunk;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c = x / kSampleChunk, o = x % kSampleChunk;
    uint64_t k = c * (n - kSampleChunk) / (chunks - 1) + o;
    uint4 v = ld_stream(rec + k);
    uint64_t g = ((((uint64_t)v.y << 32) | v.x) - T.base) >> T.gshift;
    sample_add(gcnt, g < T.n_gran && (v.w & 0xFFFFu) < GPA_VALID_SLOTS && __ldg(T.gmap + g) != NONE ? (uint32_t)g : NONE);
  }
}

// way 0 of each set keeps its most-sampled granule, way 1 the next one (ties: the smaller granule);
// best[] holds (count << 32 | ~g), 0 = empty
__global__ void k_place(const uint32_t *__restrict__ gcnt, uint64_t n_gran, int way, unsigned long long *__restrict__ best) {
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_gran; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = gcnt[g];
    if (!c) continue;
    const uint32_t st = probe_set((uint32_t)g);
    const unsigned long long v = (unsigned long long)c << 32 | (0xFFFFFFFFu - (uint32_t)g);
    if (way == 1 && best[2 * st] == v) continue;  // the way-0 winner
    atomicMax(best + 2 * st + way, v);
  }
}

__device__ __forceinline__ uint32_t best_gran(unsigned long long b) { return b ? 0xFFFFFFFFu - (uint32_t)b : kEmpty; }

struct ProbeArgs {
  uint32_t base_lo, base_hi, span, gshift, n_gran;  // span = n_gran << gshift, one 4 GiB window (probe_ok)
  uint32_t stress;                                  // ring stress test (gpa_set_ring_stress), 0 = off
};

// one record: granule (n_gran when outside the module), 2-way probe, shared byte add or L2 reduction.
// The module lies in one aligned 4 GiB window (probe_ok), so pc is in the module iff its high word
// is base_hi and its low word minus base_lo is below span.
template <bool REC>
__device__ __forceinline__ void probe_record(const ProbeArgs &A, uint4 v, bool live, uint32_t key_s, uint32_t cnt_s,
                                             unsigned long long *Hg, unsigned long long *acc, uint64_t keep,
                                             uint32_t *ri, const uint32_t *gmap) {
  const uint32_t dlo = v.x - A.base_lo;
  const uint32_t g = (v.y == A.base_hi && dlo < A.span) ? dlo >> A.gshift : A.n_gran;
  const uint32_t set = probe_set(g);
  const uint2 kk = ld_shared_v2(key_s + set * 8);
  const uint32_t cnt = v.z, st16 = v.w & 0xFFFFu;
  if (REC && live) *ri = g == A.n_gran ? NONE : __ldg(gmap + g);
  const bool w1 = kk.y == g;
  const bool hot = live && (kk.x == g || w1) && st16 < (uint32_t)GPA_VALID_SLOTS && cnt < 256u;
  const uint32_t baddr = set * (2 * kProbeRowBytes) + (w1 ? (uint32_t)kProbeRowBytes : 0u) + st16;
  const uint32_t sh = (baddr << 3) & 24u;
  const uint32_t delta = cnt << sh;
  if (GPA_PROBE_PRED) {  // straight-line: predicated shared atomic / L2 reduction, a carry (rare) branches
    const uint32_t old = atoms_add_if(hot, cnt_s + (baddr & ~3u), delta, 0u);
    const uint32_t slot = st16 < (uint32_t)GPA_VALID_SLOTS ? st16 : (uint32_t)GPA_SLOT_INVALID;
    red_add_u64_if(live && !hot, Hg + (g * GPA_SLOTS + slot), cnt, keep);  // 32-bit row offset (probe_ok)
    if (hot && ((old >> sh) & 0xFFu) + cnt > 255u) repay_carries<8, 1>(acc + (baddr & ~3u), 0, old, delta, keep);
    return;
  }
  if (hot) {
    const uint32_t old = atoms_add(cnt_s + (baddr & ~3u), delta);
    // the byte's old value + cnt > 255: a carry left the byte (maybe further): repay through acc
    if (((old >> sh) & 0xFFu) + cnt > 255u) {
      const unsigned long long sum = (unsigned long long)old + delta;
      const uint32_t cin = old ^ delta ^ (uint32_t)sum;
      unsigned long long *a = acc + (baddr & ~3u);  // acc index = 12 e + slot; this word's first slot
#pragma unroll
      for (int jb = 0; jb < 4; jb++) {
        const bool cross = jb < 3 ? ((cin >> (8 * (jb + 1))) & 1u) : (uint32_t)(sum >> 32);
        if (cross) {
          red_add_u64_keep(a + jb, 256ull, keep);
          if (jb < 3) red_add_u64_keep(a + jb + 1, ~0ull, keep);  // -1 (mod 2^64)
        }
      }
    }
  } else if (live) {
    const uint32_t slot = st16 < (uint32_t)GPA_VALID_SLOTS ? st16 : (uint32_t)GPA_SLOT_INVALID;
    red_add_u64(Hg + ((uint64_t)g * GPA_SLOTS + slot), cnt);
  }
}

template <class RG, bool REC>
__global__ void __launch_bounds__(RG::kThreads, 1)
    k_attr_probe(ProbeArgs A, const uint32_t *__restrict__ gmap, const uint4 *__restrict__ rec, uint64_t n,
                 unsigned long long *__restrict__ Hg, uint32_t *__restrict__ rec_inst,
                 const unsigned long long *__restrict__ best, unsigned long long *__restrict__ acc,
                 unsigned int *__restrict__ tile_ctr, uint32_t *__restrict__ dump) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int S = RG::kTile, NST = RG::kStages, NC = RG::kConsumers, R = RG::kPerLane;
  uint4 *ring = reinterpret_cast<uint4 *>(smem);
  uint2 *keys = reinterpret_cast<uint2 *>(smem + RG::kBytes);  // [set]: (way0 granule, way1 granule)
  uint32_t *cnt8 = reinterpret_cast<uint32_t *>(keys + kProbeSets);
  uint64_t *full = reinterpret_cast<uint64_t *>(cnt8 + kProbeWords);
  uint64_t *empty = full + NST;
  uint32_t *tile_of = reinterpret_cast<uint32_t *>(empty + NST);
  const uint32_t key_s = smem_u32(keys), cnt_s = smem_u32(cnt8), full_s = smem_u32(full), empty_s = smem_u32(empty);
  const uint32_t tile_s = smem_u32(tile_of);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ntiles = (uint32_t)((n + S - 1) / S);
  for (uint32_t x = threadIdx.x; x < kProbeSets; x += blockDim.x)
    keys[x] = make_uint2(best_gran(best[2 * x]), best_gran(best[2 * x + 1]));
  for (uint32_t x = threadIdx.x; x < kProbeWords; x += blockDim.x) cnt8[x] = 0;
  ring_init(full, empty, NST, NC);
  __syncthreads();
  if (warp == NC) {
    if (lane == 0) ring_produce_dyn<RG>(ring, full, empty, tile_of, rec, n, ntiles, tile_ctr, A.stress);
    return;
  }
  uint64_t keep;  // L2 evict-last for Hg / acc (the record stream is evict-first)
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
  const uint32_t ring_s = smem_u32(ring) + (warp * 32 + lane) * 16;
  const uint32_t last_m = (uint32_t)(n - (uint64_t)(ntiles - 1) * S);  // records in the stream's last tile
  uint32_t *ri = nullptr;
  for (uint32_t it = 0;; ++it) {
    const uint32_t st = it % NST, ph = (it / NST) & 1;
    mbar_wait_s(full_s + st * 8, ph);
    const uint32_t tile = ld_shared_u32(tile_s + st * 4);
    if (tile >= ntiles) break;
    stress_sleep(A.stress, it, warp);
    uint4 v[R];
#pragma unroll
    for (int u = 0; u < R; u++) v[u] = lds128(ring_s + (st * S + u * NC * 32) * 16);  // beyond the tile end: masked
    __syncwarp();
    if (lane == 0) ring_release_s(empty_s + st * 8);
    if (tile != ntiles - 1 || last_m == (uint32_t)S) {
#pragma unroll
      for (int u = 0; u < R; u++) {
        if (REC) ri = rec_inst + (uint64_t)tile * S + (u * NC + warp) * 32 + lane;
        probe_record<REC>(A, v[u], true, key_s, cnt_s, Hg, acc, keep, ri, gmap);
      }
    } else {  // the stream's partial last tile
#pragma unroll
      for (int u = 0; u < R; u++) {
        const uint32_t j = (uint32_t)(u * NC + warp) * 32 + lane;
        if (REC) ri = rec_inst + (uint64_t)tile * S + j;
        probe_record<REC>(A, v[u], j < last_m, key_s, cnt_s, Hg, acc, keep, ri, gmap);
      }
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(NC * 32) : "memory");
  dump_table<kProbeWords>(cnt8, kProbeWords, dump + (size_t)blockIdx.x * kProbeWords, NC * 32);  // word x: bytes = acc[4x ..]
}

// module span < 2^32 inside one aligned 4 GiB window (32-bit granule arithmetic; < 2^27 granules, so
// a granule-scratch row offset 16 g + slot fits 32 bits)
bool probe_ok(const AttrTables &T) {
  const uint64_t span = T.n_gran << T.gshift;
  return T.mode == 0 && T.n_gran < (1ull << 27) && span < (1ull << 32) && (T.base >> 32) == ((T.base + span - 1) >> 32);
}


// ---- K_attr_direct: every granule's row of byte counters in shared memory (small structures) ------
// When the whole module fits (n_gran x 12 byte counters next to a 2-stage ring: up to ~13.8 k
// granules, C2's 12 129), the CTA table is indexed by the granule itself: no plan (no sample,
// no placement), no probe, no gather.  A record with a valid slot and count < 256 in the module is
// one shared byte add (carries repaid through acc as in K_attr_probe); every other record (invalid
// slot, count >= 256, outside the module) is reduced into the granule scratch Hg.  Gap granules are
// counted like the rest and go to U in the fold (gmap[g] = NONE).
using RingDirect = Ring<31, 2, 2>;
constexpr size_t kDirectSmemMax = 232448;  // the opt-in dynamic shared memory of one sm_100 CTA

__host__ __device__ inline uint32_t direct_words(uint64_t n_gran) {  // table words, a multiple of 4
  return (uint32_t)(((n_gran * GPA_VALID_SLOTS + 3) / 4 + 3) & ~3ull);
}
__host__ __device__ inline size_t direct_smem(uint64_t n_gran) {
  return RingDirect::kBytes + (size_t)direct_words(n_gran) * 4 + 2 * RingDirect::kStages * 8 + 4 * RingDirect::kStages;
}

template <class RG, bool REC>
__global__ void __launch_bounds__(RG::kThreads, 1)
    k_attr_direct(ProbeArgs A, const uint32_t *__restrict__ gmap, const uint4 *__restrict__ rec, uint64_t n,
                  unsigned long long *__restrict__ Hg, uint32_t *__restrict__ rec_inst,
                  unsigned long long *__restrict__ acc, unsigned int *__restrict__ tile_ctr, uint32_t *__restrict__ dump,
                  uint32_t tw) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int S = RG::kTile, NST = RG::kStages, NC = RG::kConsumers, R = RG::kPerLane;
  uint4 *ring = reinterpret_cast<uint4 *>(smem);
  uint32_t *tab = reinterpret_cast<uint32_t *>(smem + RG::kBytes);
  uint64_t *full = reinterpret_cast<uint64_t *>(tab + tw);
  uint64_t *empty = full + NST;
  uint32_t *tile_of = reinterpret_cast<uint32_t *>(empty + NST);
  uint32_t tab_s = smem_u32(tab);
  asm volatile("mov.b32 %0, %0;" : "+r"(tab_s));
  const uint32_t full_s = smem_u32(full), empty_s = smem_u32(empty), tile_s = smem_u32(tile_of);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ntiles = (uint32_t)((n + S - 1) / S);
  for (uint32_t x = threadIdx.x; x < tw / 4; x += blockDim.x) reinterpret_cast<uint4 *>(tab)[x] = make_uint4(0, 0, 0, 0);
  ring_init(full, empty, NST, NC);
  __syncthreads();
  if (warp == NC) {
    if (lane == 0) ring_produce_dyn<RG>(ring, full, empty, tile_of, rec, n, ntiles, tile_ctr, A.stress);
    return;
  }
  uint64_t keep;  // L2 evict-last for Hg / acc (the record stream is evict-first)
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
  const uint32_t ring_s = smem_u32(ring) + (warp * 32 + lane) * 16;
  const uint32_t last_m = (uint32_t)(n - (uint64_t)(ntiles - 1) * S);
  for (uint32_t it = 0;; ++it) {
    const uint32_t st = it % NST, ph = (it / NST) & 1;
    mbar_wait_s(full_s + st * 8, ph);
    const uint32_t tile = ld_shared_u32(tile_s + st * 4);
    if (tile >= ntiles) break;
    stress_sleep(A.stress, it, warp);
    uint4 v[R];
#pragma unroll
    for (int u = 0; u < R; u++) v[u] = lds128(ring_s + (st * S + u * NC * 32) * 16);  // beyond the tile end: masked
    __syncwarp();
    if (lane == 0) ring_release_s(empty_s + st * 8);
    const bool partial = tile == ntiles - 1 && last_m != (uint32_t)S;
#pragma unroll
    for (int u = 0; u < R; u++) {
      const uint32_t j = (uint32_t)(u * NC + warp) * 32 + lane;
      const bool live = !partial || j < last_m;
      const uint32_t dlo = v[u].x - A.base_lo;
      const uint32_t g = (v[u].y == A.base_hi && dlo < A.span) ? dlo >> A.gshift : A.n_gran;
      const uint32_t cnt = v[u].z, st16 = v[u].w & 0xFFFFu;
      if (REC && live) rec_inst[(uint64_t)tile * S + j] = g == A.n_gran ? NONE : __ldg(gmap + g);
      const bool hot = live && g < A.n_gran && st16 < (uint32_t)GPA_VALID_SLOTS && cnt < 256u;
      const uint32_t baddr = g * GPA_VALID_SLOTS + st16;
      const uint32_t sh = (baddr & 3u) << 3, delta = cnt << sh;
      if (hot) {
        const uint32_t old = atoms_add(tab_s + (baddr & ~3u), delta);
        if (((old >> sh) & 0xFFu) + cnt > 255u) repay_carries<8, 1>(acc + (baddr & ~3u), 0, old, delta, keep);
      } else if (live) {
        const uint32_t slot = st16 < (uint32_t)GPA_VALID_SLOTS ? st16 : (uint32_t)GPA_SLOT_INVALID;
        red_add_u64(Hg + (g * GPA_SLOTS + slot), cnt);
      }
    }
  }
  asm volatile("bar.sync 1, %0;" ::"r"(NC * 32) : "memory");
  uint32_t *slab = dump + (size_t)blockIdx.x * tw;
  for (uint32_t x = threadIdx.x; x < tw / 4; x += NC * 32)
    reinterpret_cast<uint4 *>(slab)[x] = reinterpret_cast<const uint4 *>(tab)[x];
}

bool direct_ok(const AttrTables &T) { return probe_ok(T) && direct_smem(T.n_gran) <= kDirectSmemMax; }

// ---- f1 at instruction level with K_attr_code32's hot bins ------------
// The per-profile cube PH[(P+1)][n_inst][16] (profile = the record's stream field, P = overflow).
// A CTA takes a contiguous range of tiles (one profile's records are contiguous in the stream, so it
// meets a few profiles in turn) and counts the current profile's records that fall into the call
// plan's hot (instruction, slot) bins in K_attr_code32's byte-packed shared table; every other
// record is one L2 reduction into the cube (instruction = gmap[g]).  When a whole tile belongs to
// another profile, the consumer warps meet at a named barrier, flush the table into the old
// profile's rows (bin -> (instruction, slot) through the plan's bin_of) and continue with the new
// profile.  A byte carry is repaid in the cube directly (+256 at the bin, -1 at the next byte's bin,
// unassigned bins skipped on both sides, so they cancel).  Exact for any plan.
__device__ __forceinline__ void prof_repay(unsigned long long *row, const uint32_t *__restrict__ bin_of, uint32_t nb,
                                           uint32_t word, uint32_t old, uint32_t delta) {
  const unsigned long long s = (unsigned long long)old + delta;
  const uint32_t cin = old ^ delta ^ (uint32_t)s;
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const bool cross = j < 3 ? ((cin >> (8 * (j + 1))) & 1u) : (uint32_t)(s >> 32);
    if (!cross) continue;
    const uint32_t b0 = 4 * word + j, t0 = b0 < nb ? __ldg(bin_of + b0) : NONE;
    if (t0 != NONE) red_add_u64(row + t0, 256ull);
    if (j < 3) {
      const uint32_t t1 = b0 + 1 < nb ? __ldg(bin_of + b0 + 1) : NONE;
      if (t1 != NONE) red_add_u64(row + t1, ~0ull);  // -1 (mod 2^64)
    }
  }
}

template <class RG, int NW>
__global__ void __launch_bounds__(RG::kThreads, 1)
    k_attr_prof_code(ProbeArgs A, const uint32_t *__restrict__ gmap, const uint32_t *__restrict__ code,
                     const uint32_t *__restrict__ bin_of, const uint32_t *__restrict__ thr, const uint4 *__restrict__ rec,
                     uint64_t n, uint32_t n_inst, uint32_t n_prof, unsigned long long *__restrict__ PH,
                     unsigned long long *__restrict__ PU) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int S = RG::kTile, NST = RG::kStages, NC = RG::kConsumers, R = RG::kPerLane;
  uint4 *ring = reinterpret_cast<uint4 *>(smem);
  uint32_t *tab = reinterpret_cast<uint32_t *>(smem + RG::kBytes);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + RG::kBytes + (size_t)NW * 4);
  uint64_t *empty = full + NST;
  uint32_t *tile_of = reinterpret_cast<uint32_t *>(empty + NST);
  uint32_t tab_s = smem_u32(tab);
  asm volatile("mov.b32 %0, %0;" : "+r"(tab_s));
  const uint32_t full_s = smem_u32(full), empty_s = smem_u32(empty), tile_s = smem_u32(tile_of);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ntiles = (uint32_t)((n + S - 1) / S);
  const uint32_t t0 = (uint32_t)((uint64_t)ntiles * blockIdx.x / gridDim.x);
  const uint32_t t1 = (uint32_t)((uint64_t)ntiles * (blockIdx.x + 1) / gridDim.x);
  const uint32_t nb = min(thr[1], (uint32_t)NW * 4);
  for (uint32_t x = threadIdx.x; x < NW; x += blockDim.x) tab[x] = 0;
  ring_init(full, empty, NST, NC);
  __syncthreads();
  if (warp == NC) {
    if (lane == 0) ring_produce<RG>(ring, full, empty, rec, n, t0, 1, t1);
    return;
  }
  const uint32_t ring_s = smem_u32(ring) + (warp * 32 + lane) * 16;
  const uint32_t last_m = (uint32_t)(n - (uint64_t)(ntiles - 1) * S);
  const uint64_t rows = (uint64_t)n_inst * GPA_SLOTS;  // u64 per profile
  // the profile the table counts: the CTA's first record's (clamped to the overflow profile)
  uint32_t pcur = n_prof;
  if (t0 < t1) {
    const uint32_t s0 = __ldg(reinterpret_cast<const uint32_t *>(rec + (uint64_t)t0 * S) + 3) >> 16;
    pcur = s0 < n_prof ? s0 : n_prof;
  }
  auto flush = [&](uint32_t p) {  // table -> PH[p], zeroed; all consumer warps
    asm volatile("bar.sync 1, %0;" ::"r"(NC * 32) : "memory");
    unsigned long long *row = PH + (uint64_t)p * rows;
    for (uint32_t x = threadIdx.x; x < NW; x += NC * 32) {
      const uint32_t word = tab[x];
      if (!word) continue;
      tab[x] = 0;
#pragma unroll
      for (int q = 0; q < 4; q++) {
        const uint32_t val = (word >> (8 * q)) & 0xFFu, b = 4 * x + q;
        if (val && b < nb) {
          const uint32_t t = __ldg(bin_of + b);
          if (t != NONE) red_add_u64(row + t, val);
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NC * 32) : "memory");
  };
  for (uint32_t it = 0; t0 + it < t1; ++it) {
    const uint32_t tile = t0 + it;
    const uint32_t st = it % NST, ph = (it / NST) & 1;
    mbar_wait_s(full_s + st * 8, ph);
    const bool last = tile == ntiles - 1;
    const uint32_t m = last ? last_m : (uint32_t)S;
    // a tile wholly of another profile: switch the table to it (uniform: every warp reads the same words)
    const uint32_t pa = ld_shared_u32(smem_u32(ring) + (st * S) * 16 + 12) >> 16;
    const uint32_t pz = ld_shared_u32(smem_u32(ring) + (st * S + m - 1) * 16 + 12) >> 16;
    const uint32_t qa = pa < n_prof ? pa : n_prof, qz = pz < n_prof ? pz : n_prof;
    uint4 v[R];
#pragma unroll
    for (int u = 0; u < R; u++) v[u] = lds128(ring_s + (st * S + u * NC * 32) * 16);
    __syncwarp();
    if (lane == 0) ring_release_s(empty_s + st * 8);
    if (qa == qz && qa != pcur) {
      flush(pcur);
      pcur = qa;
    }
    uint32_t g[R], c[R];
#pragma unroll
    for (int u = 0; u < R; u++) {
      const uint32_t dlo = v[u].x - A.base_lo;
      g[u] = (v[u].y == A.base_hi && dlo < A.span) ? dlo >> A.gshift : A.n_gran;
      c[u] = __ldg(code + g[u]);  // code[n_gran] = 0
    }
    unsigned long long *row = PH + (uint64_t)pcur * rows;
#pragma unroll
    for (int u = 0; u < R; u++) {
      const uint32_t j = (uint32_t)(u * NC + warp) * 32 + lane;
      const bool live = j < m;
      const uint32_t cnt = v[u].z, st16 = v[u].w & 0xFFFFu, sid = v[u].w >> 16;
      const uint32_t p = sid < n_prof ? sid : n_prof;
      const uint32_t mask = c[u] & 0xFFFu;
      const bool hot = live && p == pcur && st16 < (uint32_t)GPA_VALID_SLOTS && ((mask >> st16) & 1u) && cnt < 256u;
      const uint32_t idx = (c[u] >> 12) + __popc(mask & ((1u << st16) - 1u));
      const uint32_t word = idx >> 2, sh = (idx & 3u) << 3, delta = cnt << sh;
      if (hot) {
        const uint32_t old = atoms_add(tab_s + word * 4, delta);
        if (((old >> sh) & 0xFFu) + cnt > 255u) prof_repay(row, bin_of, nb, word, old, delta);
      } else if (live && cnt) {
        const uint32_t slot = st16 < (uint32_t)GPA_VALID_SLOTS ? st16 : (uint32_t)GPA_SLOT_INVALID;
        const uint32_t i = g[u] < A.n_gran ? __ldg(gmap + g[u]) : NONE;
        red_add_u64(i == NONE ? PU + ((uint64_t)p << 4 | slot) : PH + (uint64_t)p * rows + ((uint64_t)i << 4 | slot), cnt);
      }
    }
  }
  flush(pcur);
}


// ---- K_attr_code32: packed bins located through a 32-bit per-granule code ------------------------
// The byte-packed bins of K_attr_bins<8> (131 072 bins in 128 KiB), but the per-call code map holds
// only the hot information of the granule's instruction (base << 12 | 12-bit hot-slot mask; 0 =
// no hot slot / unmapped): 4 B per granule, so twice as many codes per L1 line as the 64-bit map.
// Records that are not hot (cold slots, cold or unmapped granules, counts >= 256) are reduced
// into the granule-indexed scratch Hg of K_attr_probe (no instruction index needed), folded into
// H / U after the kernel.
__global__ void k_codemap32(const uint32_t *__restrict__ gmap, uint64_t n_gran, const uint32_t *__restrict__ hot_info,
                            uint32_t *__restrict__ code) {
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g <= n_gran; g += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t m = g < n_gran ? gmap[g] : NONE;
    code[g] = m == NONE ? 0u : hot_info[m];
  }
}

template <class RG, int NW, int PACK, bool REC, int LOOK = 1>
__global__ void __launch_bounds__(RG::kThreads, 1)
    k_attr_code32(ProbeArgs A, const uint32_t *__restrict__ gmap, const uint32_t *__restrict__ code,
                  const uint4 *__restrict__ rec, uint64_t n, unsigned long long *__restrict__ Hg,
                  uint32_t *__restrict__ rec_inst, unsigned long long *__restrict__ acc, const uint32_t *__restrict__ thr,
                  unsigned int *__restrict__ tile_ctr, uint32_t *__restrict__ dump) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int S = RG::kTile, NST = RG::kStages, NC = RG::kConsumers, R = RG::kPerLane, D = LOOK + 1;
  // PACK 0: bin idx in word idx % NW, byte idx / NW (NW a power of two: the consecutive bins of one
  // instruction fall in different banks); PACK 1: word idx / 4, byte idx % 4 (any NW)
  static_assert(PACK == 1 || (NW & (NW - 1)) == 0, "interleaved bins need a power-of-two word count");
  constexpr uint32_t kLogNW = PACK ? 0 : __builtin_ctz(NW);
  uint32_t *tab = reinterpret_cast<uint32_t *>(smem + RG::kBytes);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + RG::kBytes + (size_t)NW * 4);
  uint64_t *empty = full + NST;
  uint32_t *tile_of = reinterpret_cast<uint32_t *>(empty + NST);
  uint4 *ring = reinterpret_cast<uint4 *>(smem);
  uint32_t tab_s = smem_u32(tab);
  if (GPA_CODE_LEAN) asm volatile("mov.b32 %0, %0;" : "+r"(tab_s));  // a plain register, not re-derived per use
  const uint32_t full_s = smem_u32(full), empty_s = smem_u32(empty), tile_s = smem_u32(tile_of);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t ntiles = (uint32_t)((n + S - 1) / S);
  const uint32_t nb = min(thr[1], (uint32_t)NW * 4);
  const uint32_t nw = PACK ? min((nb + 3) / 4, (uint32_t)NW) : min(nb, (uint32_t)NW);
  for (uint32_t x = threadIdx.x; x < nw; x += blockDim.x) tab[x] = 0;
  ring_init(full, empty, NST, NC);
  __syncthreads();
  if (warp == NC) {
    if (lane == 0) ring_produce_dyn<RG>(ring, full, empty, tile_of, rec, n, ntiles, tile_ctr, A.stress);
    return;
  }
  uint64_t keep;  // L2 evict-last for the code map and the reductions (the record stream is evict-first)
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(keep));
  const uint32_t ring_s = smem_u32(ring) + (warp * 32 + lane) * 16;
  const uint32_t last_m = (uint32_t)(n - (uint64_t)(ntiles - 1) * S);
  uint4 v[D][R];
  uint32_t g[D][R], c[D][R], tid[D];
  bool ended = false;  // the end marker has been read: fetch no further stage
  auto fetch = [&](uint32_t it, uint4 *vv, uint32_t *gg, uint32_t *cc, uint32_t &tt) {
    const uint32_t st = it % NST, ph = (it / NST) & 1;
    mbar_wait_s(full_s + st * 8, ph);
    tt = ld_shared_u32(tile_s + st * 4);
    if (tt >= ntiles) {
      ended = true;
      return;
    }
    stress_sleep(A.stress, it, warp);
#pragma unroll
    for (int u = 0; u < R; u++) vv[u] = lds128(ring_s + (st * S + u * NC * 32) * 16);  // beyond the end: masked
    __syncwarp();
    if (lane == 0) ring_release_s(empty_s + st * 8);
#pragma unroll
    for (int u = 0; u < R; u++) {
      const uint32_t dlo = vv[u].x - A.base_lo;
      gg[u] = (vv[u].y == A.base_hi && dlo < A.span) ? dlo >> A.gshift : A.n_gran;
      if (GPA_CODE_LEAN) cc[u] = GPA_CODE_HINT ? ldg_keep_u32(code + gg[u], keep) : __ldg(code + gg[u]);  // code[n_gran] = 0
      else cc[u] = gg[u] < A.n_gran ? ldg_keep_u32(code + gg[u], keep) : 0u;
    }
  };
#pragma unroll
  for (int q = 0; q < D; q++) tid[q] = ntiles;
#pragma unroll
  for (int q = 0; q < LOOK; q++)
    if (!ended) fetch(q, v[q], g[q], c[q], tid[q]);
  for (uint32_t it0 = 0;; it0 += D) {
#pragma unroll
    for (int q = 0; q < D; q++) {
      const uint32_t it = it0 + q;
      const uint32_t tile = tid[q];
      if (tile >= ntiles) goto done;
      if (!ended) fetch(it + LOOK, v[(q + LOOK) % D], g[(q + LOOK) % D], c[(q + LOOK) % D], tid[(q + LOOK) % D]);
      const bool last = tile == ntiles - 1;
#pragma unroll
      for (int u = 0; u < R; u++) {
        const uint32_t j = (uint32_t)(u * NC + warp) * 32 + lane;
        const bool live = !last || j < last_m;
        const uint32_t cnt = v[q][u].z, st16 = v[q][u].w & 0xFFFFu, cd = c[q][u], gq = g[q][u];
        if (REC && live) rec_inst[(uint64_t)tile * S + j] = gq == A.n_gran ? NONE : __ldg(gmap + gq);
        const uint32_t mask = cd & 0xFFFu;
        const bool hot = live && st16 < (uint32_t)GPA_VALID_SLOTS && ((mask >> st16) & 1u) && cnt < 256u;
        const uint32_t idx = (cd >> 12) + __popc(mask & ((1u << st16) - 1u));
        const uint32_t word = PACK ? idx >> 2 : idx & (NW - 1);
        const uint32_t sh = PACK ? (idx & 3u) << 3 : (idx >> kLogNW) << 3;
        const uint32_t delta = cnt << sh;
        if (PACK && GPA_CODE_PRED) {
          // straight-line: a predicated shared atomic (hot) and a predicated L2 reduction (the rest),
          // no divergent branches; only a carry (rare) branches
          const uint32_t old = atoms_add_if(hot, tab_s + word * 4, delta, 0u);
          const uint32_t slot = st16 < (uint32_t)GPA_VALID_SLOTS ? st16 : (uint32_t)GPA_SLOT_INVALID;
          red_add_u64_if(live && !hot, Hg + ((uint64_t)gq * GPA_SLOTS + slot), cnt, keep);
          if (hot && ((old >> sh) & 0xFFu) + cnt > 255u) repay_carries<8, 1>(acc + 4 * word, 0, old, delta, keep);
        } else if (hot) {
          const uint32_t old = atoms_add(tab_s + word * 4, delta);
          if (((old >> sh) & 0xFFu) + cnt > 255u) {
            if (PACK) repay_carries<8, 1>(acc + 4 * word, 0, old, delta, keep);  // bins 4 word .. 4 word + 3
            else repay_carries<8, NW>(acc, word, old, delta, keep);
          }
        } else if (live) {
          const uint32_t slot = st16 < (uint32_t)GPA_VALID_SLOTS ? st16 : (uint32_t)GPA_SLOT_INVALID;
          if (GPA_CODE_LEAN) red_add_u64(Hg + (gq * GPA_SLOTS + slot), cnt);  // 32-bit row offset: n_gran < 2^27
          else red_add_u64(Hg + ((uint64_t)gq * GPA_SLOTS + slot), cnt);
        }
      }
      tid[q] = ntiles;  // consumed
    }
  }
done:
  asm volatile("bar.sync 1, %0;" ::"r"(NC * 32) : "memory");
  if (PACK) {
    dump_table<NW>(tab, nw, dump + (size_t)blockIdx.x * NW, NC * 32);  // word x: bytes = acc[4x ..]
  } else {
    for (uint32_t x = threadIdx.x; x < nw; x += NC * 32) {
      const uint32_t word = tab[x];
#pragma unroll
      for (int p = 0; p < 4; p++) {
        const uint32_t val = (word >> (8 * p)) & 0xFFu;
        const uint32_t bin = (uint32_t)p * NW + x;
        if (val && bin < nb) red_add_u64_keep(acc + bin, val, keep);
      }
    }
  }
}

#ifndef GPA_CODE_NC
#define GPA_CODE_NC 31
#endif
// 25 600 words = 102 400 byte bins, packed four consecutive bins per word: with the 93 KiB ring
// the CTA stays under the 196 KiB shared-memory carve-out, leaving ~60 KiB of L1 for the code
// gathers (C5: 12.54 ms with 32 768 interleaved words in the 228 KiB carve-out -> 12.12 ms;
// 26 624+ words cross into the larger carve-out again: 12.73 ms)
#ifndef GPA_CODE_NW
#define GPA_CODE_NW 25600
#endif
#ifndef GPA_CODE_PACK
#define GPA_CODE_PACK 1
#endif
#ifndef GPA_CODE_R
#define GPA_CODE_R 3
#endif
#ifndef GPA_CODE_NST
#define GPA_CODE_NST 2
#endif
#ifndef GPA_CODE_LOOK
#define GPA_CODE_LOOK 1
#endif
using RingCode = Ring<GPA_CODE_NC, GPA_CODE_R, GPA_CODE_NST>;

}  // namespace

// ---- attribution plans: the pre-pass of K_attr_probe / K_attr_code32 (which granules / bins live
// in shared memory), built from a sample of records and reusable for any number of calls and
// chunks: the result is exact for every plan, only the speed depends on how well it fits ------------
constexpr uint32_t kCodeK = (uint32_t)GPA_CODE_NW * 4;  // K_attr_code32 byte bins

// records sampled to build a plan: n/256, at least 2^17, at most 2^21 for the probe table (7) and
// 2^22 for the 131 072 byte bins of 8, whose ranking needs the finer counts (C5: 12.77 -> 12.7 ms;
// C4 with 7 got slower with 2^22)
// floor 2^17 (C2 1e7 records: 0.087 -> 0.083 ms against 2^18; 2^16 0.089; C3 0.324 -> 0.319 ms)
#ifndef GPA_SAMPLE_MIN_LOG
#define GPA_SAMPLE_MIN_LOG 17
#endif
static uint64_t plan_sample(uint64_t n, int variant) {
  const int cap = variant == 8 ? GPA_SAMPLE_MAX_LOG + 1 : GPA_SAMPLE_MAX_LOG;
  return std::min<uint64_t>(1ull << cap, std::max<uint64_t>(1ull << GPA_SAMPLE_MIN_LOG, n / GPA_SAMPLE_DIV));
}

size_t plan_bytes(const AttrTables &T, int variant) {
  if (variant == 9) return 16;                                                   // none
  if (variant == 7) return (size_t)kProbeM * 8;                                  // best[M]
  return ((size_t)kCodeK + 4 + T.n_gran + 1) * 4;  // bin_of[K] | thr[4] | code[n_gran + 1] (code[n_gran] = 0: out of module)
}

// ---- host side of a call: few API calls (a mid-size call, C2's 1e7 records, is otherwise paced by
// the host: ~20 allocations / memsets / launches took longer to issue than the GPU work they held) --
static size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }
static uint32_t table_words(const AttrPlan &p) {
  return p.variant == 7 ? (uint32_t)kProbeWords : p.variant == 9 ? direct_words(p.n_gran) : (uint32_t)GPA_CODE_NW;
}
// per-counter accumulators (acc): one per shared byte counter (7, 9) or bin (8)
static size_t acc_count(const AttrPlan &p) {
  return p.variant == 7 ? (size_t)kProbeM * GPA_VALID_SLOTS : p.variant == 9 ? (size_t)table_words(p) * 4 : (size_t)kCodeK;
}

// transient scratch of a plan build: gcnt[n_gran] (7) | scnt[n_inst*12] hot_info[n_inst] V[4096] (8)
static size_t build_bytes(const AttrTables &T, int variant) {
  if (variant == 9) return 0;
  if (variant == 7) return al256((size_t)T.n_gran * 4);
  return al256(((size_t)T.n_inst * kHotSlots + T.n_inst + kVBins) * 4);
}

// accumulators of one call (or of all chunks of a host-records call): acc (per shared counter) |
// Hg (granule x slot, + the out-of-module row) | one table slab per CTA | the dynamic tile counter
static size_t acc_bytes(const AttrPlan &p, int sm_count) {
  const size_t na = acc_count(p) * 8;
  const size_t nh = (size_t)(p.n_gran + 1) * 128;
  return al256(na + nh) + al256((size_t)sm_count * table_words(p) * 4) + 256;
}

static void plan_ptrs(const AttrTables &T, int variant, void *mem, AttrPlan *p) {
  p->variant = variant;
  p->n_gran = T.n_gran;
  if (variant == 7) {
    p->best = reinterpret_cast<unsigned long long *>(mem);
  } else {
    p->bin_of = reinterpret_cast<uint32_t *>(mem);
    p->thr = p->bin_of + kCodeK;
    p->code = p->thr + 4;
  }
}

static void acc_ptrs(const AttrPlan &p, void *mem, int sm_count, AttrAcc *a) {
  const size_t na = acc_count(p) * 8;
  const size_t nh = (size_t)(p.n_gran + 1) * 128;
  uint8_t *b = reinterpret_cast<uint8_t *>(mem);
  a->acc = reinterpret_cast<unsigned long long *>(b);
  a->Hg = a->acc + na / 8;
  a->dump = reinterpret_cast<uint32_t *>(b + al256(na + nh));
  a->slabs = sm_count;
  a->ctr = reinterpret_cast<unsigned int *>(b + al256(na + nh) + al256((size_t)sm_count * table_words(p) * 4));
}

struct Fills {
  FillSet F{};
  int k = 0;
  void add(void *p, size_t words, uint32_t v) {
    F.p[k] = reinterpret_cast<uint32_t *>(p);
    F.n[k] = words;
    F.v[k] = v;
    k++;
  }
  cudaError_t launch(int sm_count, cudaStream_t st) {
    k_fill<<<sm_count * 8, 256, 0, st>>>(F);
    count_launches(1);
    return cudaGetLastError();
  }
};

static void build_fills(const AttrTables &T, const AttrPlan &p, void *w, Fills &f) {
  if (p.variant == 9) return;  // no plan
  if (p.variant == 7) {
    f.add(w, T.n_gran, 0u);                      // gcnt
    f.add(p.best, (size_t)kProbeM * 2, 0u);      // best
  } else {
    f.add(w, (size_t)T.n_inst * kHotSlots + T.n_inst + kVBins, 0u);  // scnt | hot_info | V
    f.add(p.bin_of, kCodeK, 0xFFFFFFFFu);         // unassigned bins map to NONE
  }
}

static void acc_fills(const AttrPlan &p, const AttrAcc &a, Fills &f) {
  const size_t na = acc_count(p) * 8;
  f.add(a.acc, (na + (size_t)(p.n_gran + 1) * 128) / 4, 0u);  // acc | Hg (the slabs are stored whole)
  f.add(a.ctr, 4, 0u);
}

// the sample -> table kernels (scratch zeroed)
static cudaError_t build_kernels(const AttrTables &T, const AttrPlan &p, const uint4 *rec, uint64_t n, void *w,
                                 int sm_count, cudaStream_t st) {
  if (p.variant == 9) return cudaSuccess;  // no plan
  const uint32_t chunks = (uint32_t)std::max<uint64_t>(2, plan_sample(n, p.variant) / kSampleChunk);
  if (p.variant == 7) {
    uint32_t *gcnt = reinterpret_cast<uint32_t *>(w);
    const unsigned gb = (unsigned)std::min<uint64_t>((T.n_gran + 255) / 256, (uint64_t)sm_count * 8);
    k_sample_gran<<<sm_count * 4, 256, 0, st>>>(T, rec, n, chunks, gcnt);
    k_place<<<gb, 256, 0, st>>>(gcnt, T.n_gran, 0, p.best);
    k_place<<<gb, 256, 0, st>>>(gcnt, T.n_gran, 1, p.best);
    count_launches(3);
    return cudaGetLastError();
  }
  const size_t ni = T.n_inst, nbins = ni * kHotSlots;
  uint32_t *scnt = reinterpret_cast<uint32_t *>(w), *hot_info = scnt + nbins, *V = hot_info + ni;
  k_sample_bins<<<sm_count * 4, 256, 0, st>>>(T, rec, n, chunks, scnt);
  k_vhist<<<sm_count, 1024, 0, st>>>(scnt, (uint32_t)nbins, V);
  k_pick<<<1, 1024, 0, st>>>(V, p.thr, kCodeK);
  k_assign_bins<<<sm_count * 2, 256, 0, st>>>(scnt, (uint32_t)ni, p.thr, hot_info, p.bin_of, kCodeK);
  k_codemap32<<<sm_count * 4, 256, 0, st>>>(T.gmap, T.n_gran, hot_info, p.code);
  count_launches(5);
  return cudaGetLastError();
}

cudaError_t plan_build(const AttrTables &T, int variant, const uint4 *rec, uint64_t n, void *mem, AttrPlan *p,
                       int sm_count, cudaStream_t st) {
  plan_ptrs(T, variant, mem, p);
  if (variant == 9) return cudaSuccess;  // no plan
  void *w = nullptr;
  cudaError_t e = pool_alloc(&w, build_bytes(T, variant), st);
  if (e != cudaSuccess) return e;
  Fills f;
  build_fills(T, *p, w, f);
  e = f.launch(sm_count, st);
  if (e == cudaSuccess) e = build_kernels(T, *p, rec, n, w, sm_count, st);
  cudaError_t e2 = cudaFreeAsync(w, st);
  return e != cudaSuccess ? e : e2;
}

cudaError_t plan_begin(const AttrPlan &p, AttrAcc *a, int sm_count, cudaStream_t st) {
  void *mem = nullptr;
  cudaError_t e = pool_alloc(&mem, acc_bytes(p, sm_count), st);
  if (e != cudaSuccess) return e;
  acc_ptrs(p, mem, sm_count, a);
  Fills f;
  acc_fills(p, *a, f);
  return f.launch(sm_count, st);
}

// cudaFuncSetAttribute once per kernel and device (it costs a few microseconds of host time per call)
template <class K>
static cudaError_t smem_attr_once(K kern, size_t smem, int slot) {
  static std::atomic<uint64_t> done[4];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = 1ull << (dev & 63);
  if (done[slot].load(std::memory_order_relaxed) & bit) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) done[slot].fetch_or(bit, std::memory_order_relaxed);
  return e;
}

static FoldArgs fold_args(const AttrTables &T, const AttrPlan &p, const AttrAcc &a, int slabs, int fin,
                          unsigned long long *H, unsigned long long *U) {
  FoldArgs F{};
  F.dump = a.dump;
  F.nw = table_words(p);
  F.tb = (F.nw + 31) / 32;
  F.slabs = slabs;
  F.fin = fin;
  F.variant = p.variant;
  F.acc = a.acc;
  F.ctr = a.ctr;
  F.best = p.best;
  F.bin_of = p.bin_of;
  F.thr = p.thr;
  F.gmap = T.gmap;
  F.Hg = a.Hg;
  F.n_gran = T.n_gran;
  F.H = H;
  F.U = U;
  return F;
}

// one launch of the main kernel; fold != 0: its slabs -> acc (and the tile counter reset) right away,
// as every launch of a multi-launch call must; a single-launch call leaves them to plan_end
static cudaError_t plan_launch(const AttrTables &T, const AttrPlan &p, const AttrAcc &a, const uint4 *rec, uint64_t n,
                               uint32_t *ri, int sm_count, cudaStream_t st, bool fold) {
  if (n == 0) return cudaSuccess;
  const ProbeArgs A{(uint32_t)T.base, (uint32_t)(T.base >> 32), (uint32_t)(T.n_gran << T.gshift), T.gshift,
                    (uint32_t)T.n_gran, (uint32_t)g_ring_stress.load(std::memory_order_relaxed)};
  cudaError_t e;
  if (p.variant == 9) {
    using RG = RingDirect;
    auto kern = ri ? k_attr_direct<RG, true> : k_attr_direct<RG, false>;
    const size_t smem = direct_smem(T.n_gran);
    // the table size varies per structure: set the attribute whenever this structure needs more
    static std::atomic<size_t> set_for[2];
    if (smem > set_for[ri ? 1 : 0].load(std::memory_order_relaxed)) {
      if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDirectSmemMax)) != cudaSuccess)
        return e;
      set_for[ri ? 1 : 0].store(kDirectSmemMax, std::memory_order_relaxed);
    }
    kern<<<sm_count, RG::kThreads, smem, st>>>(A, T.gmap, rec, n, a.Hg, ri, a.acc, a.ctr, a.dump, table_words(p));
  } else if (p.variant == 7) {
    using RG = RingProbe;
    auto kern = ri ? k_attr_probe<RG, true> : k_attr_probe<RG, false>;
    const size_t smem = RG::kBytes + (size_t)kProbeSets * 8 + (size_t)kProbeWords * 4 + 2 * RG::kStages * 8 + 4 * RG::kStages;
    if ((e = smem_attr_once(kern, smem, ri ? 1 : 0)) != cudaSuccess) return e;
    // dynamic tile order for the probe kernel (C4: 2.82 -> 2.71 ms); the counter is zero here
    kern<<<sm_count, RG::kThreads, smem, st>>>(A, T.gmap, rec, n, a.Hg, ri, p.best, a.acc, a.ctr, a.dump);
  } else {
    using RG = RingCode;
    auto kern = ri ? k_attr_code32<RG, GPA_CODE_NW, GPA_CODE_PACK, true, GPA_CODE_LOOK>
                   : k_attr_code32<RG, GPA_CODE_NW, GPA_CODE_PACK, false, GPA_CODE_LOOK>;
    const size_t smem = RG::kBytes + (size_t)GPA_CODE_NW * 4 + 2 * RG::kStages * 8 + 4 * RG::kStages;
    if ((e = smem_attr_once(kern, smem, ri ? 3 : 2)) != cudaSuccess) return e;
    // static tile order for the code-map kernel (C5: 12.54 ms vs 13.16 ms with the dynamic order)
    kern<<<sm_count, RG::kThreads, smem, st>>>(A, T.gmap, p.code, rec, n, a.Hg, ri, a.acc, p.thr, nullptr, a.dump);
  }
  count_launches(1);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  if (fold && (p.variant != 8 || GPA_CODE_PACK)) {
    const FoldArgs F = fold_args(T, p, a, sm_count, 0, nullptr, nullptr);
    k_fold_all<<<F.tb, kFoldParts * 32, 0, st>>>(F);
    count_launches(1);
  }
  return cudaGetLastError();
}

cudaError_t plan_run(const AttrTables &T, const AttrPlan &p, const AttrAcc &a, const uint4 *rec, uint64_t n,
                     uint32_t *ri, int sm_count, cudaStream_t st) {
  return plan_launch(T, p, a, rec, n, ri, sm_count, st, true);
}

// fold the accumulators (+ `slabs` table slabs not yet folded) into H / U in one launch
static cudaError_t plan_fold_final(const AttrTables &T, const AttrPlan &p, const AttrAcc &a, int slabs,
                                   unsigned long long *H, unsigned long long *U, int sm_count, cudaStream_t st) {
  const FoldArgs F = fold_args(T, p, a, slabs, 1, H, U);
  const uint64_t b2 = std::min<uint64_t>(((T.n_gran + 1) * 16 + 255) / 256, (uint64_t)sm_count * 16);
  k_fold_all<<<F.tb + (unsigned)b2, kFoldParts * 32, 0, st>>>(F);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t plan_end(const AttrTables &T, const AttrPlan &p, AttrAcc *a, unsigned long long *H, unsigned long long *U,
                     int sm_count, cudaStream_t st) {
  cudaError_t e = plan_fold_final(T, p, *a, 0, H, U, sm_count, st);
  cudaError_t e2 = cudaFreeAsync(a->acc, st);
  a->acc = a->Hg = nullptr;
  return e != cudaSuccess ? e : e2;
}

// one call with a transient plan built from the call's own records: one allocation, one fill, the
// plan kernels, the main kernel and one fold
cudaError_t launch_planned(const AttrTables &T, int variant, const uint4 *rec, uint64_t n, unsigned long long *H,
                           unsigned long long *U, uint32_t *ri, int sm_count, cudaStream_t st) {
  AttrPlan p;
  p.variant = variant;
  p.n_gran = T.n_gran;
  const size_t b0 = al256(plan_bytes(T, variant)), b1 = build_bytes(T, variant), b2 = acc_bytes(p, sm_count);
  uint8_t *mem = nullptr;
  bool cached = false;  // the structure's reusable scratch (no pool call), else a pool block
  cudaError_t e = scratch_get(T.cache, b0 + b1 + b2, st, (void **)&mem, &cached);
  if (e != cudaSuccess) return e;
  plan_ptrs(T, variant, mem, &p);
  AttrAcc a;
  acc_ptrs(p, mem + b0 + b1, sm_count, &a);
  Fills f;
  build_fills(T, p, mem + b0, f);
  acc_fills(p, a, f);
  e = f.launch(sm_count, st);
  if (e == cudaSuccess) e = build_kernels(T, p, rec, n, mem + b0, sm_count, st);
  if (e == cudaSuccess) e = plan_launch(T, p, a, rec, n, ri, sm_count, st, false);
  if (e == cudaSuccess) e = plan_fold_final(T, p, a, (p.variant != 8 || GPA_CODE_PACK) ? sm_count : 0, H, U, sm_count, st);
  cudaError_t e2 = scratch_put(T.cache, mem, cached, st);
  return e != cudaSuccess ? e : e2;
}

namespace {

template <class RG, int ROWS>
cudaError_t run_hot(const AttrTables &T, const uint4 *rec, uint64_t n, unsigned long long *H, unsigned long long *U,
                    uint32_t *ri, const uint32_t *code, const uint32_t *row_inst, const uint32_t *thr, int sm_count,
                    cudaStream_t st) {
  auto kern = ri ? k_attr_hot<RG, ROWS, true> : k_attr_hot<RG, ROWS, false>;
  const size_t smem = RG::kBytes + (size_t)ROWS * kHotSlots * 4 + 2 * RG::kStages * 8;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<sm_count, RG::kThreads, smem, st>>>(T.base, T.n_gran, T.gshift, code, rec, n, H, U, ri, row_inst, thr);
  return cudaGetLastError();
}

std::atomic<int> g_attr_kernel{-1};  // gpa_set_attr_kernel; -1 = read GPA_ATTR_VARIANT once (0 if unset)

int attr_variant() {  // 0 auto, 1 stream, 2 tma, 3 shared bins, 4 shared rows (when applicable)
  if (g_attr_kernel.load(std::memory_order_relaxed) < 0) {
    const char *e = getenv("GPA_ATTR_VARIANT");
    int expect = -1;
    g_attr_kernel.compare_exchange_strong(expect, e ? atoi(e) : 0);
  }
  return g_attr_kernel.load(std::memory_order_relaxed);
}

cudaError_t launch_hot(const AttrTables &T, const uint4 *rec, uint64_t n, unsigned long long *H,
                       unsigned long long *U, uint32_t *ri, int sm_count, cudaStream_t st) {
  // stream-ordered scratch: scnt[n_inst] | hot_row[n_inst] | row_inst[K] | V[4096] | thr[4] | code[n_gran]
  size_t ni = T.n_inst;
  size_t words = 2 * ni + kHotRows + kVBins + 4 + T.n_gran;
  uint32_t *w = nullptr;
  cudaError_t e = pool_alloc((void **)&w, words * 4, st);
  if (e != cudaSuccess) return e;
  uint32_t *scnt = w, *hot_row = w + ni, *row_inst = hot_row + ni, *V = row_inst + kHotRows, *thr = V + kVBins,
           *code = thr + 4;
  cudaMemsetAsync(scnt, 0, ni * 4, st);
  cudaMemsetAsync(V, 0, kVBins * 4, st);
  k_sample<<<sm_count * 4, 256, 0, st>>>(T, rec, n, scnt);
  k_vhist<<<sm_count, 1024, 0, st>>>(scnt, (uint32_t)ni, V);
  k_pick<<<1, 1024, 0, st>>>(V, thr, kHotRows);
  k_assign<<<sm_count * 2, 256, 0, st>>>(scnt, (uint32_t)ni, thr, hot_row, row_inst, kHotRows);
  k_codemap<<<sm_count * 4, 256, 0, st>>>(T.gmap, T.n_gran, hot_row, code);
  e = run_hot<RingHot, kHotRows>(T, rec, n, H, U, ri, code, row_inst, thr, sm_count, st);
  count_launches(6);
  cudaError_t e2 = cudaFreeAsync(w, st);
  return e != cudaSuccess ? e : e2;
}

template <int MODE>
cudaError_t launch_tma(const AttrTables &T, const uint4 *rec, uint64_t n, unsigned long long *H,
                       unsigned long long *U, uint32_t *ri, int sm_count, cudaStream_t st) {
  auto kern = ri ? k_attr_tma<MODE, true> : k_attr_tma<MODE, false>;
  size_t smem = RingTma::kBytes + 2 * RingTma::kStages * 8;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  uint64_t ntiles = (n + RingTma::kTile - 1) / RingTma::kTile;
  unsigned blocks = (unsigned)(ntiles < (uint64_t)sm_count ? ntiles : (uint64_t)sm_count);
  kern<<<blocks, RingTma::kThreads, smem, st>>>(T, rec, n, H, U, ri);
  count_launches(1);
  return cudaGetLastError();
}

template <int MODE>
cudaError_t launch_stream(const AttrTables &T, const uint4 *rec, uint64_t n, unsigned long long *H,
                          unsigned long long *U, uint32_t *ri, int sm_count, cudaStream_t st) {
  uint64_t per_block = (uint64_t)kStreamThreads * kStreamUnroll;
  uint64_t want = (n + per_block - 1) / per_block;
  uint64_t cap = (uint64_t)sm_count * (2048 / kStreamThreads);  // one full wave of resident blocks
  unsigned blocks = (unsigned)(want < cap ? want : cap);
  if (ri) k_attr_stream<MODE, true><<<blocks, kStreamThreads, 0, st>>>(T, rec, n, H, U, ri);
  else k_attr_stream<MODE, false><<<blocks, kStreamThreads, 0, st>>>(T, rec, n, H, U, nullptr);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace

void set_attr_kernel(int which) { g_attr_kernel.store(which, std::memory_order_relaxed); }
void set_ring_stress(int level) { g_ring_stress.store(level, std::memory_order_relaxed); }

// the kernel a call of n records runs (1..8, gpa_set_attr_kernel numbering)
int attr_choice(const AttrTables &T, uint64_t n) {
  const int var = attr_variant();
  const bool hot_ok = T.mode == 0 && n >= kHotMinRecords && T.n_inst >= 1024;
  // automatic choice: the large-call kernels' per-call pre-pass (sample, table / code map; growing
  // with the structure) pays off from ~4e6 records and 8 records per instruction on (measured
  // crossovers: C2 ~2e6, C3 ~4e6, C5 ~5e6 records; tools/attr_variants.py); below that the
  // register-streaming kernel is fastest.  Among the large-call kernels: the probe table (8192
  // granules in shared memory, no gather) while the structure is small enough for it to hold most
  // sampled records (C3, C4: ~0.92), else the byte bins found through the 32-bit code map (C5)
  //
  const bool bins_auto = hot_ok && n >= 4000000ull && n >= 8ull * T.n_inst;
  // the whole module in shared memory (K_attr_direct, no plan): from GPA_DIRECT_MIN records on
  if ((var == 0 && n >= (uint64_t)GPA_DIRECT_MIN || var == 9) && direct_ok(T)) return 9;
  if (var == 0 && bins_auto) return probe_ok(T) ? (T.n_gran <= (1ull << 18) ? 7 : 8) : 3;
  if (var >= 3 && var <= 6 && hot_ok) return var;
  if ((var == 7 || var == 8) && hot_ok && probe_ok(T)) return var;
  return (var == 1 || n < 4096 || (var == 0 && T.mode == 0)) ? 1 : 2;
}

// CTAs of the persistent attribution kernels: all SMs, or fewer (environment GPA_ATTR_CTAS) so that
// kernels of other streams (a previous batch's analysis) find free SMs while a batch is attributed
int attr_ctas(int sm_count) {
  static const int v = [] {
    const char *e = getenv("GPA_ATTR_CTAS");
    return e ? atoi(e) : 0;
  }();
  return v > 0 && v < sm_count ? v : sm_count;
}

// f1 instruction level with the hot bins of a call plan (k_attr_prof_code); false: not applicable
bool prof_code_ok(const AttrTables &T, uint64_t n) {
  return probe_ok(T) && n >= 4000000ull && T.n_inst >= 1024 && getenv("GPA_PROF_INST_L2") == nullptr;
}

cudaError_t launch_prof_inst_code(const AttrTables &T, const gpa_sample *d_samples, uint64_t n, uint32_t n_prof,
                                  unsigned long long *PH, unsigned long long *PU, int sm_count, cudaStream_t st) {
  const uint4 *rec = reinterpret_cast<const uint4 *>(d_samples);
  AttrPlan p;
  p.variant = 8;
  p.n_gran = T.n_gran;
  const size_t b0 = al256(plan_bytes(T, 8)), b1 = build_bytes(T, 8);
  uint8_t *mem = nullptr;
  cudaError_t e = pool_alloc((void **)&mem, b0 + b1, st);
  if (e != cudaSuccess) return e;
  plan_ptrs(T, 8, mem, &p);
  Fills f;
  build_fills(T, p, mem + b0, f);
  e = f.launch(sm_count, st);
  if (e == cudaSuccess) e = build_kernels(T, p, rec, n, mem + b0, sm_count, st);
  if (e == cudaSuccess) {
    using RG = RingCode;
    auto kern = k_attr_prof_code<RG, GPA_CODE_NW>;
    const size_t smem = RG::kBytes + (size_t)GPA_CODE_NW * 4 + 2 * RG::kStages * 8 + 4 * RG::kStages;
    e = smem_attr_once(kern, smem, 3);
    const ProbeArgs A{(uint32_t)T.base, (uint32_t)(T.base >> 32), (uint32_t)(T.n_gran << T.gshift), T.gshift,
                      (uint32_t)T.n_gran, 0u};
    const uint64_t ntiles = (n + RG::kTile - 1) / RG::kTile;
    const unsigned blocks = (unsigned)std::min<uint64_t>(ntiles, (uint64_t)sm_count);
    if (e == cudaSuccess) {
      kern<<<blocks, RG::kThreads, smem, st>>>(A, T.gmap, p.code, p.bin_of, p.thr, rec, n, (uint32_t)T.n_inst, n_prof,
                                               PH, PU);
      count_launches(1);
      e = cudaGetLastError();
    }
  }
  cudaError_t e2 = cudaFreeAsync(mem, st);
  return e != cudaSuccess ? e : e2;
}

cudaError_t launch_attribute(const AttrTables &T, const gpa_sample *d_samples, uint64_t n,
                             unsigned long long *d_hist, unsigned long long *d_unattr, uint32_t *d_rec_inst,
                             int sm_count, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const uint4 *rec = reinterpret_cast<const uint4 *>(d_samples);
  switch (attr_choice(T, n)) {
    case 9:
    case 8:
    case 7: return launch_planned(T, attr_choice(T, n), rec, n, d_hist, d_unattr, d_rec_inst, attr_ctas(sm_count), st);
    case 6: return launch_bins<16>(T, rec, n, d_hist, d_unattr, d_rec_inst, sm_count, st);
    case 5: return launch_bins<8>(T, rec, n, d_hist, d_unattr, d_rec_inst, sm_count, st);
    case 4: return launch_hot(T, rec, n, d_hist, d_unattr, d_rec_inst, sm_count, st);
    case 3: return launch_bins<32>(T, rec, n, d_hist, d_unattr, d_rec_inst, sm_count, st);
    case 2:
      return T.mode == 0 ? launch_tma<0>(T, rec, n, d_hist, d_unattr, d_rec_inst, sm_count, st)
                         : launch_tma<1>(T, rec, n, d_hist, d_unattr, d_rec_inst, sm_count, st);
    default:
      return T.mode == 0 ? launch_stream<0>(T, rec, n, d_hist, d_unattr, d_rec_inst, sm_count, st)
                         : launch_stream<1>(T, rec, n, d_hist, d_unattr, d_rec_inst, sm_count, st);
  }
}

}  // namespace gpa
