// k_attr.cu — a-1..a-3: PC-sample decode, pc -> instruction lookup, per-instruction x
// stall-reason histogram (§4.2; §4.5; §5).
//
// One persistent, grid-stride kernel streams the 16-B records (one 128-bit non-allocating
// load each, several in flight per thread), maps pc -> instruction through the load-time
// granule map (L2/L1-resident; exact range semantics, reading R6), and adds `count` to
// H[inst][slot] (or U[slot]) with a u64 reduction in L2.  Records of a warp that hit the
// same bin are combined first (match.any + shuffles), so a hot bin costs one L2 atomic per
// warp instead of one per record.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "gpa_internal.cuh"

namespace gpa {
namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;  // records in flight per thread per iteration
constexpr unsigned FULL = 0xFFFFFFFFu;

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

template <int MODE>
__device__ __forceinline__ uint32_t lookup(const AttrTables &T, uint64_t pc) {
  if (!(pc >= T.base && pc < T.end)) return NONE;
  if (MODE == 0) {
    return __ldg(T.gmap + ((pc - T.base) >> T.gshift));
  } else {
    // largest start <= pc (binary search over the sorted starts), then the length check
    uint32_t lo = 0, hi = T.n_inst;
    while (lo < hi) {
      uint32_t mid = (lo + hi) >> 1;
      if (__ldg(T.inst_addr + mid) <= pc) lo = mid + 1; else hi = mid;
    }
    uint32_t j = lo - 1;  // lo >= 1 because pc >= base = inst_addr[0]
    return pc - __ldg(T.inst_addr + j) < (uint64_t)__ldg(T.inst_len + j) ? j : NONE;
  }
}

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

template <int MODE, bool REC>
__global__ void __launch_bounds__(kThreads) k_attribute(AttrTables T, const uint4 *__restrict__ rec, uint64_t n,
                                                        unsigned long long *__restrict__ H,
                                                        unsigned long long *__restrict__ U,
                                                        uint32_t *__restrict__ rec_inst) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * kThreads + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * kThreads) >> 5;
  const uint64_t step = nwarps * 32 * kUnroll;
  // each warp owns 32*kUnroll consecutive records per iteration (coalesced 16-B loads)
  for (uint64_t base = warp * 32 * kUnroll; base < n; base += step) {
    uint4 v[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; u++) {
      uint64_t k = base + (uint64_t)u * 32 + lane;
      v[u] = k < n ? ld_stream(rec + k) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; u++) {
      uint64_t k = base + (uint64_t)u * 32 + lane;
      bool live = k < n;
      uint64_t pc = ((uint64_t)v[u].y << 32) | v[u].x;
      uint32_t cnt = v[u].z;
      uint32_t stall = v[u].w & 0xFFFFu;
      uint32_t slot = stall < GPA_VALID_SLOTS ? stall : GPA_SLOT_INVALID;
      uint32_t i = lookup<MODE>(T, pc);
      if (REC && live) rec_inst[k] = i;
      uint32_t key = !live ? FULL : (i == NONE ? (0xFFFFFFE0u | slot) : (i << 4 | slot));
      unsigned long long *target = i == NONE ? U + slot : H + ((uint64_t)i << 4 | slot);
      // live records with count 0 contribute nothing; keep them idle
      if (cnt == 0) key = FULL;
      warp_accumulate(key, cnt, target);
    }
  }
}


// ---- v2: TMA-fed persistent kernel ----------------------------------------------------------
// One CTA per SM.  A producer warp streams tiles of S records HBM -> shared memory with 1-D
// bulk copies (cp.async.bulk, the TMA engine) into an NST-stage ring guarded by mbarriers,
// with an L2 evict-first policy so the stream does not push the histogram and the granule
// map out of L2.  NC consumer warps copy their R records per tile to registers, release the
// stage at once (so the next bulk copy can land), issue all R granule-map gathers before
// using any (R independent L2 round trips in flight per lane), then accumulate.
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
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
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

template <int NC, int R, int NST>
struct TmaCfg {
  static constexpr int kConsumers = NC;
  static constexpr int kPerLane = R;
  static constexpr int kStages = NST;
  static constexpr int kTile = NC * 32 * R;                   // records per stage
  static constexpr int kThreads = (NC + 1) * 32;
  static constexpr size_t kSmem = (size_t)NST * kTile * 16 + 2 * NST * sizeof(uint64_t);
};

template <class C, int MODE, bool REC, bool AGG>
__global__ void __launch_bounds__(C::kThreads, 1)
    k_attribute_tma(AttrTables T, const uint4 *__restrict__ rec, uint64_t n, unsigned long long *__restrict__ H,
                    unsigned long long *__restrict__ U, uint32_t *__restrict__ rec_inst) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int S = C::kTile, NST = C::kStages, NC = C::kConsumers, R = C::kPerLane;
  uint4 *ring = reinterpret_cast<uint4 *>(smem);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)NST * S * 16);
  uint64_t *empty = full + NST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t ntiles = (n + S - 1) / S;
  if (threadIdx.x == 0) {
    for (int q = 0; q < NST; q++) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == NC) {  // producer warp: one elected lane drives the bulk-copy engine
    if (lane == 0) {
      uint64_t policy;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      uint32_t it = 0;
      for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        uint32_t st = it % NST, ph = (it / NST) & 1;
        if (it >= (uint32_t)NST) mbar_wait(empty + st, ph ^ 1);
        uint64_t left = n - tile * S;
        uint32_t bytes = (uint32_t)((left < (uint64_t)S ? left : (uint64_t)S) * 16);
        mbar_arrive_expect_tx(full + st, bytes);
        bulk_g2s(ring + (size_t)st * S, rec + tile * S, bytes, full + st, policy);
      }
    }
    return;
  }
  uint32_t it = 0;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
    uint32_t st = it % NST, ph = (it / NST) & 1;
    mbar_wait(full + st, ph);
    uint64_t left = n - tile * S;
    uint32_t m = (uint32_t)(left < (uint64_t)S ? left : (uint64_t)S);
    uint4 v[R];
#pragma unroll
    for (int u = 0; u < R; u++) {
      uint32_t j = (uint32_t)(u * NC + warp) * 32 + lane;
      v[u] = j < m ? ring[(size_t)st * S + j] : make_uint4(0, 0, 0, 0);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);   // registers hold the records: stage free
    uint32_t inst[R];
#pragma unroll
    for (int u = 0; u < R; u++) inst[u] = lookup<MODE>(T, ((uint64_t)v[u].y << 32) | v[u].x);
#pragma unroll
    for (int u = 0; u < R; u++) {
      uint32_t j = (uint32_t)(u * NC + warp) * 32 + lane;
      bool live = j < m;
      uint32_t i = inst[u], cnt = v[u].z, stall = v[u].w & 0xFFFFu;
      uint32_t slot = stall < GPA_VALID_SLOTS ? stall : GPA_SLOT_INVALID;
      if (REC && live) rec_inst[tile * S + j] = i;
      unsigned long long *target = i == NONE ? U + slot : H + ((uint64_t)i << 4 | slot);
      if (AGG) {
        uint32_t key = (!live || cnt == 0) ? FULL : (i == NONE ? (0xFFFFFFE0u | slot) : (i << 4 | slot));
        warp_accumulate(key, cnt, target);
      } else if (live && cnt) {
        red_add_u64(target, cnt);
      }
    }
  }
}

using CfgA = TmaCfg<16, 4, 6>;

template <class C, int MODE, bool REC, bool AGG>
cudaError_t launch_tma(const AttrTables &T, const uint4 *rec, uint64_t n, unsigned long long *H,
                       unsigned long long *U, uint32_t *ri, int sm_count, cudaStream_t st) {
  auto kern = k_attribute_tma<C, MODE, REC, AGG>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
  if (e != cudaSuccess) return e;
  uint64_t ntiles = (n + C::kTile - 1) / C::kTile;
  unsigned blocks = (unsigned)(ntiles < (uint64_t)sm_count ? ntiles : (uint64_t)sm_count);
  kern<<<blocks, C::kThreads, C::kSmem, st>>>(T, rec, n, H, U, ri);
  return cudaGetLastError();
}

int attr_variant() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("GPA_ATTR_VARIANT");
    v = e ? atoi(e) : 6;
  }
  return v;
}

// ---- v3: heavy-hitter rows privatised in shared memory ---------------------------------------
// Measured on B200 (tools/microbench.cu): u64 reductions into L2 sustain ~1.9e11/s at spread
// addresses and far less on hot addresses, while the HBM roofline needs ~4.3e11 records/s;
// shared-memory u32 atomics sustain ~1.3e12/s.  So the histogram rows of the hottest
// instructions are privatised per CTA in shared memory:
//   1. k_sample    count instruction hits in 64 evenly spaced chunks of the stream (2^21 records)
//   2. k_vhist / k_pick / k_assign   pick up to KROWS instructions with the largest counts
//   3. k_codemap   per-call copy of the granule map: code = hot row | 0x80000000, or the
//                  instruction index (one gather still resolves a record)
//   4. k_attr_hot  stream records (registers, software-pipelined one iteration ahead); hot
//                  valid-slot records -> u32 shared atomics, others -> u64 L2 reductions;
//                  a u32 wrap (old + cnt < old) is repaid as +2^32 in L2, so the result is
//                  exact for any counts; each CTA flushes its rows once at the end.
// The hot set only changes where a count is added first, never the result (bit-exact).
constexpr int kHotRows = 4608;                 // 4608 rows x 12 slots x 4 B = 216 KiB smem
constexpr int kHotSlots = GPA_VALID_SLOTS;
constexpr size_t kHotSmem = (size_t)kHotRows * kHotSlots * 4;
constexpr int kSampleChunks = 64, kSampleChunk = 1 << 15;
constexpr int kVBins = 4096;
constexpr int kHotThreads = 768;
constexpr int kHotR = 4;

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

__global__ void k_vhist(const uint32_t *__restrict__ scnt, uint32_t n_inst, uint32_t *__restrict__ V) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_inst; i += gridDim.x * blockDim.x) {
    uint32_t c = scnt[i];
    if (c) atomicAdd(V + (c < kVBins - 1 ? c : kVBins - 1), 1u);
  }
}

// smallest threshold t >= 1 whose suffix count fits in kHotRows (or the top bucket)
__global__ void k_pick(const uint32_t *__restrict__ V, uint32_t *__restrict__ thr, uint32_t rows) {
  if (threadIdx.x == 0) {
    uint32_t acc = 0, t = kVBins - 1;
    for (int c = kVBins - 1; c >= 1; c--) {
      if (acc + V[c] > rows) break;
      acc += V[c];
      t = c;
    }
    thr[0] = t;
    thr[1] = 0;  // rows assigned so far
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

__global__ void k_codemap(const uint32_t *__restrict__ gmap, uint64_t n_gran, const uint32_t *__restrict__ hot_row,
                          uint32_t *__restrict__ code) {
  for (uint64_t g = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n_gran; g += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t m = gmap[g];
    uint32_t r = m == NONE ? NONE : hot_row[m];
    code[g] = m == NONE ? NONE : (r != NONE ? (0x80000000u | r) : m);
  }
}

template <bool REC>
__device__ __forceinline__ void hot_accumulate(uint32_t *tab, const uint32_t *__restrict__ row_inst, uint32_t c,
                                               uint4 v, bool live, uint64_t k, unsigned long long *__restrict__ H,
                                               unsigned long long *__restrict__ U, uint32_t *__restrict__ rec_inst) {
  uint32_t cnt = v.z, stall = v.w & 0xFFFFu;
  uint32_t slot = stall < GPA_VALID_SLOTS ? stall : GPA_SLOT_INVALID;
  bool hot = c != NONE && (c & 0x80000000u);
  if (REC && live) rec_inst[k] = c == NONE ? NONE : (hot ? __ldg(row_inst + (c & 0x7FFFFFFFu)) : c);
  if (!live || cnt == 0) return;
  if (c == NONE) {
    red_add_u64(U + slot, cnt);
  } else if (hot && slot < (uint32_t)kHotSlots) {
    uint32_t r = c & 0x7FFFFFFFu;
    uint32_t old = atomicAdd(tab + r * kHotSlots + slot, cnt);
    if (old + cnt < old) red_add_u64(H + ((uint64_t)__ldg(row_inst + r) << 4 | slot), 1ull << 32);
  } else {
    uint32_t i = hot ? __ldg(row_inst + (c & 0x7FFFFFFFu)) : c;
    red_add_u64(H + ((uint64_t)i << 4 | slot), cnt);
  }
}

template <bool REC>
__global__ void __launch_bounds__(kHotThreads, 1)
    k_attr_hot(uint64_t base, uint64_t end, uint32_t gshift, const uint32_t *__restrict__ code,
               const uint4 *__restrict__ rec, uint64_t n, unsigned long long *__restrict__ H,
               unsigned long long *__restrict__ U, uint32_t *__restrict__ rec_inst,
               const uint32_t *__restrict__ row_inst, const uint32_t *__restrict__ thr) {
  extern __shared__ __align__(16) uint32_t tab[];
  const uint32_t nhot = min(thr[1], (uint32_t)kHotRows);
  for (uint32_t x = threadIdx.x; x < nhot * kHotSlots; x += blockDim.x) tab[x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t step = nwarps * 32 * kHotR;
  uint4 nxt[kHotR];
  uint64_t b = warp * 32 * kHotR;
#pragma unroll
  for (int u = 0; u < kHotR; u++) {
    uint64_t k = b + (uint64_t)u * 32 + lane;
    nxt[u] = k < n ? ld_stream(rec + k) : make_uint4(0, 0, 0, 0);
  }
  for (; b < n; b += step) {
    uint4 v[kHotR];
#pragma unroll
    for (int u = 0; u < kHotR; u++) v[u] = nxt[u];
#pragma unroll
    for (int u = 0; u < kHotR; u++) {          // prefetch the next iteration's records
      uint64_t k = b + step + (uint64_t)u * 32 + lane;
      nxt[u] = k < n ? ld_stream(rec + k) : make_uint4(0, 0, 0, 0);
    }
    uint32_t c[kHotR];
#pragma unroll
    for (int u = 0; u < kHotR; u++) {
      uint64_t pc = ((uint64_t)v[u].y << 32) | v[u].x;
      c[u] = (pc >= base && pc < end) ? __ldg(code + ((pc - base) >> gshift)) : NONE;
    }
#pragma unroll
    for (int u = 0; u < kHotR; u++) {
      uint64_t k = b + (uint64_t)u * 32 + lane;
      hot_accumulate<REC>(tab, row_inst, c[u], v[u], k < n, k, H, U, rec_inst);
    }
  }
  __syncthreads();
  for (uint32_t x = threadIdx.x; x < nhot * kHotSlots; x += blockDim.x) {
    uint32_t val = tab[x];
    if (val) red_add_u64(H + ((uint64_t)__ldg(row_inst + x / kHotSlots) << 4 | (x % kHotSlots)), val);
  }
}

// v3b: the same accumulation with a three-deep software pipeline per thread: records of
// iteration i+2 are loaded from HBM while the granule codes of iteration i+1 are gathered from
// L2 and iteration i is accumulated, so neither latency is exposed.  Shared atomics are issued
// before any of their results are examined (wrap checks last).
template <bool REC, int R>
__global__ void __launch_bounds__(kHotThreads, 1)
    k_attr_hot2(uint64_t base, uint64_t end, uint32_t gshift, const uint32_t *__restrict__ code,
                const uint4 *__restrict__ rec, uint64_t n, unsigned long long *__restrict__ H,
                unsigned long long *__restrict__ U, uint32_t *__restrict__ rec_inst,
                const uint32_t *__restrict__ row_inst, const uint32_t *__restrict__ thr) {
  extern __shared__ __align__(16) uint32_t tab[];
  const uint32_t nhot = min(thr[1], (uint32_t)kHotRows);
  for (uint32_t x = threadIdx.x; x < nhot * kHotSlots; x += blockDim.x) tab[x] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t step = nwarps * 32 * R;
  auto load = [&](uint64_t b, uint4 *dst) {
#pragma unroll
    for (int u = 0; u < R; u++) {
      uint64_t k = b + (uint64_t)u * 32 + lane;
      dst[u] = k < n ? ld_stream(rec + k) : make_uint4(0, 0, 0, 0);
    }
  };
  auto gather = [&](const uint4 *v, uint32_t *c) {
#pragma unroll
    for (int u = 0; u < R; u++) {
      uint64_t pc = ((uint64_t)v[u].y << 32) | v[u].x;
      c[u] = (pc >= base && pc < end) ? __ldg(code + ((pc - base) >> gshift)) : NONE;
    }
  };
  uint64_t b = warp * 32 * R;
  uint4 va[R], vb[R], vc[R];
  uint32_t ca[R], cb[R];
  load(b, va);
  load(b + step, vb);
  gather(va, ca);
  for (; b < n; b += step) {
    load(b + 2 * step, vc);
    gather(vb, cb);
    uint32_t old[R];
    bool hot[R];
#pragma unroll
    for (int u = 0; u < R; u++) {
      uint64_t k = b + (uint64_t)u * 32 + lane;
      bool live = k < n;
      uint32_t c = ca[u], cnt = va[u].z, stall = va[u].w & 0xFFFFu;
      uint32_t slot = stall < GPA_VALID_SLOTS ? stall : GPA_SLOT_INVALID;
      bool h = c != NONE && (c & 0x80000000u);
      if (REC && live) rec_inst[k] = c == NONE ? NONE : (h ? __ldg(row_inst + (c & 0x7FFFFFFFu)) : c);
      hot[u] = live && cnt && h && slot < (uint32_t)kHotSlots;
      old[u] = hot[u] ? atomicAdd(tab + (c & 0x7FFFFFFFu) * kHotSlots + slot, cnt) : 0u;
      if (live && cnt && !hot[u]) {
        uint32_t i = h ? __ldg(row_inst + (c & 0x7FFFFFFFu)) : c;
        red_add_u64(c == NONE ? U + slot : H + ((uint64_t)i << 4 | slot), cnt);
      }
    }
#pragma unroll
    for (int u = 0; u < R; u++) {
      if (hot[u] && old[u] + va[u].z < old[u]) {
        uint32_t stall = va[u].w & 0xFFFFu;
        red_add_u64(H + ((uint64_t)__ldg(row_inst + (ca[u] & 0x7FFFFFFFu)) << 4 | stall), 1ull << 32);
      }
    }
#pragma unroll
    for (int u = 0; u < R; u++) {
      va[u] = vb[u];
      vb[u] = vc[u];
      ca[u] = cb[u];
    }
  }
  __syncthreads();
  for (uint32_t x = threadIdx.x; x < nhot * kHotSlots; x += blockDim.x) {
    uint32_t val = tab[x];
    if (val) red_add_u64(H + ((uint64_t)__ldg(row_inst + x / kHotSlots) << 4 | (x % kHotSlots)), val);
  }
}

// v3c: records fed by the TMA engine.  Measured (ncu, v3b): gathers issued behind
// streaming loads complete in issue order from the L1TEX queue, so register prefetching
// cannot hide the HBM latency from the granule-code gather.  Here a producer warp streams
// record tiles into a shared-memory ring with cp.async.bulk (UBLKCP, outside the LSU queue);
// consumer warps read their records from shared memory, release the stage, issue the code
// gathers of tile i+1 and accumulate tile i meanwhile.  Ring (3 x 24 KiB) and the hot-row
// table (3200 rows x 48 B) share the 227 KiB of shared memory.
constexpr int kT3Warps = 24, kT3Rpl = 2, kT3Stages = 3;
constexpr int kT3Tile = kT3Warps * 32 * kT3Rpl;                 // records per stage
constexpr int kT3Rows = 3200;
constexpr size_t kT3Ring = (size_t)kT3Stages * kT3Tile * 16;
constexpr size_t kT3Smem = kT3Ring + (size_t)kT3Rows * kHotSlots * 4 + 2 * kT3Stages * 8;

template <bool REC>
__global__ void __launch_bounds__((kT3Warps + 1) * 32, 1)
    k_attr_hot3(uint64_t base, uint64_t end, uint32_t gshift, const uint32_t *__restrict__ code,
                const uint4 *__restrict__ rec, uint64_t n, unsigned long long *__restrict__ H,
                unsigned long long *__restrict__ U, uint32_t *__restrict__ rec_inst,
                const uint32_t *__restrict__ row_inst, const uint32_t *__restrict__ thr) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int S = kT3Tile, NST = kT3Stages, NC = kT3Warps, R = kT3Rpl;
  uint4 *ring = reinterpret_cast<uint4 *>(smem);
  uint32_t *tab = reinterpret_cast<uint32_t *>(smem + kT3Ring);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kT3Ring + (size_t)kT3Rows * kHotSlots * 4);
  uint64_t *empty = full + NST;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t ntiles = (n + S - 1) / S;
  const uint32_t nhot = min(thr[1], (uint32_t)kT3Rows);
  for (uint32_t x = threadIdx.x; x < nhot * kHotSlots; x += blockDim.x) tab[x] = 0;
  if (threadIdx.x == 0) {
    for (int q = 0; q < NST; q++) {
      mbar_init(full + q, 1);
      mbar_init(empty + q, NC);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == NC) {
    if (lane == 0) {
      uint64_t policy;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      uint32_t it = 0;
      for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        uint32_t st = it % NST, ph = (it / NST) & 1;
        if (it >= (uint32_t)NST) mbar_wait(empty + st, ph ^ 1);
        uint64_t left = n - tile * S;
        uint32_t bytes = (uint32_t)((left < (uint64_t)S ? left : (uint64_t)S) * 16);
        mbar_arrive_expect_tx(full + st, bytes);
        bulk_g2s(ring + (size_t)st * S, rec + tile * S, bytes, full + st, policy);
      }
    }
    return;
  }
  // consumers: tile i+1's records and code gathers overlap tile i's accumulation
  uint4 va[R], vb[R];
  uint32_t ca[R], cb[R];
  uint64_t ka = 0;
  uint32_t ma = 0;
  auto fetch = [&](uint32_t it, uint64_t tile, uint4 *v, uint32_t *c, uint32_t &m) {
    uint32_t st = it % NST, ph = (it / NST) & 1;
    mbar_wait(full + st, ph);
    uint64_t left = n - tile * S;
    m = (uint32_t)(left < (uint64_t)S ? left : (uint64_t)S);
#pragma unroll
    for (int u = 0; u < R; u++) {
      uint32_t j = (uint32_t)(u * NC + warp) * 32 + lane;
      v[u] = j < m ? ring[(size_t)st * S + j] : make_uint4(0, 0, 0, 0);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + st);
#pragma unroll
    for (int u = 0; u < R; u++) {
      uint64_t pc = ((uint64_t)v[u].y << 32) | v[u].x;
      c[u] = (pc >= base && pc < end) ? __ldg(code + ((pc - base) >> gshift)) : NONE;
    }
  };
  uint32_t it = 0;
  uint64_t tile = blockIdx.x;
  if (tile < ntiles) {
    fetch(it, tile, va, ca, ma);
    ka = tile * S;
  }
  while (tile < ntiles) {
    uint64_t nt = tile + gridDim.x;
    uint32_t mb = 0;
    if (nt < ntiles) fetch(it + 1, nt, vb, cb, mb);
    uint32_t old[R];
    bool hot[R];
#pragma unroll
    for (int u = 0; u < R; u++) {
      uint32_t j = (uint32_t)(u * NC + warp) * 32 + lane;
      bool live = j < ma;
      uint32_t c = ca[u], cnt = va[u].z, stall = va[u].w & 0xFFFFu;
      uint32_t slot = stall < GPA_VALID_SLOTS ? stall : GPA_SLOT_INVALID;
      bool h = c != NONE && (c & 0x80000000u);
      if (REC && live) rec_inst[ka + j] = c == NONE ? NONE : (h ? __ldg(row_inst + (c & 0x7FFFFFFFu)) : c);
      hot[u] = live && cnt && h && slot < (uint32_t)kHotSlots;
      old[u] = hot[u] ? atomicAdd(tab + (c & 0x7FFFFFFFu) * kHotSlots + slot, cnt) : 0u;
      if (live && cnt && !hot[u]) {
        uint32_t i = h ? __ldg(row_inst + (c & 0x7FFFFFFFu)) : c;
        red_add_u64(c == NONE ? U + slot : H + ((uint64_t)i << 4 | slot), cnt);
      }
    }
#pragma unroll
    for (int u = 0; u < R; u++) {
      if (hot[u] && old[u] + va[u].z < old[u]) {
        uint32_t stall = va[u].w & 0xFFFFu;
        red_add_u64(H + ((uint64_t)__ldg(row_inst + (ca[u] & 0x7FFFFFFFu)) << 4 | stall), 1ull << 32);
      }
    }
#pragma unroll
    for (int u = 0; u < R; u++) {
      va[u] = vb[u];
      ca[u] = cb[u];
    }
    ma = mb;
    ka = nt * S;
    tile = nt;
    ++it;
  }
  asm volatile("bar.sync 1, %0;" ::"r"(NC * 32) : "memory");
  for (uint32_t x = threadIdx.x; x < nhot * kHotSlots; x += NC * 32) {
    uint32_t val = tab[x];
    if (val) red_add_u64(H + ((uint64_t)__ldg(row_inst + x / kHotSlots) << 4 | (x % kHotSlots)), val);
  }
}

cudaError_t launch_hot(const AttrTables &T, const uint4 *rec, uint64_t n, unsigned long long *H,
                       unsigned long long *U, uint32_t *ri, int sm_count, cudaStream_t st) {
  // scratch (stream-ordered): scnt[n_inst] | hot_row[n_inst] | row_inst[K] | V[4096] | thr[2] | code[n_gran]
  size_t ni = T.n_inst;
  size_t words = 2 * ni + kHotRows + kVBins + 4 + T.n_gran;
  uint32_t *w = nullptr;
  cudaError_t e = cudaMallocAsync((void **)&w, words * 4, st);
  if (e != cudaSuccess) return e;
  uint32_t *scnt = w, *hot_row = w + ni, *row_inst = hot_row + ni, *V = row_inst + kHotRows, *thr = V + kVBins,
           *code = thr + 4;
  cudaMemsetAsync(scnt, 0, ni * 4, st);
  cudaMemsetAsync(V, 0, kVBins * 4, st);
  k_sample<<<sm_count * 4, 256, 0, st>>>(T, rec, n, scnt);
  k_vhist<<<sm_count * 2, 256, 0, st>>>(scnt, (uint32_t)ni, V);
  uint32_t rows = attr_variant() == 6 ? kT3Rows : kHotRows;
  k_pick<<<1, 32, 0, st>>>(V, thr, rows);
  k_assign<<<sm_count * 2, 256, 0, st>>>(scnt, (uint32_t)ni, thr, hot_row, row_inst, rows);
  k_codemap<<<sm_count * 4, 256, 0, st>>>(T.gmap, T.n_gran, hot_row, code);
  if (attr_variant() == 6) {
    auto kern = ri ? k_attr_hot3<true> : k_attr_hot3<false>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kT3Smem);
    if (e == cudaSuccess) {
      kern<<<sm_count, (kT3Warps + 1) * 32, kT3Smem, st>>>(T.base, T.end, T.gshift, code, rec, n, H, U, ri, row_inst,
                                                            thr);
      e = cudaGetLastError();
    }
  } else {
    auto kern = attr_variant() == 5 ? (ri ? k_attr_hot2<true, 4> : k_attr_hot2<false, 4>)
                                    : (ri ? k_attr_hot<true> : k_attr_hot<false>);
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kHotSmem);
    if (e == cudaSuccess) {
      kern<<<sm_count, kHotThreads, kHotSmem, st>>>(T.base, T.end, T.gshift, code, rec, n, H, U, ri, row_inst, thr);
      e = cudaGetLastError();
    }
  }
  count_launches(6);
  cudaError_t e2 = cudaFreeAsync(w, st);
  return e != cudaSuccess ? e : e2;
}


}  // namespace

cudaError_t launch_attribute(const AttrTables &T, const gpa_sample *d_samples, uint64_t n,
                             unsigned long long *d_hist, unsigned long long *d_unattr, uint32_t *d_rec_inst,
                             int sm_count, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const uint4 *rec = reinterpret_cast<const uint4 *>(d_samples);
  int var = attr_variant();  // 1: register-streaming kernel; 2: TMA ring + warp aggregation;
                             // 3: TMA ring, one reduction per record; 4: shared-memory
                             // heavy-hitter rows (v3) for large calls
  if (var >= 4 && T.mode == 0 && n >= (uint64_t)kSampleChunks * kSampleChunk && T.n_inst >= 1024)
    return launch_hot(T, rec, n, d_hist, d_unattr, d_rec_inst, sm_count, st);
  if (var >= 4) var = 2;
  count_launches(1);
  if (var >= 2 && n >= 4096) {
    bool agg = var == 2;
#define GPA_TMA(M, RI, A) return launch_tma<CfgA, M, RI, A>(T, rec, n, d_hist, d_unattr, d_rec_inst, sm_count, st)
    if (T.mode == 0) {
      if (d_rec_inst) { if (agg) GPA_TMA(0, true, true); else GPA_TMA(0, true, false); }
      else { if (agg) GPA_TMA(0, false, true); else GPA_TMA(0, false, false); }
    } else {
      if (d_rec_inst) { if (agg) GPA_TMA(1, true, true); else GPA_TMA(1, true, false); }
      else { if (agg) GPA_TMA(1, false, true); else GPA_TMA(1, false, false); }
    }
#undef GPA_TMA
  }
  uint64_t per_block = (uint64_t)kThreads * kUnroll;
  uint64_t want = (n + per_block - 1) / per_block;
  uint64_t cap = (uint64_t)sm_count * (2048 / kThreads);  // one full wave of resident blocks
  unsigned blocks = (unsigned)(want < cap ? want : cap);
  if (T.mode == 0) {
    if (d_rec_inst) k_attribute<0, true><<<blocks, kThreads, 0, st>>>(T, rec, n, d_hist, d_unattr, d_rec_inst);
    else k_attribute<0, false><<<blocks, kThreads, 0, st>>>(T, rec, n, d_hist, d_unattr, nullptr);
  } else {
    if (d_rec_inst) k_attribute<1, true><<<blocks, kThreads, 0, st>>>(T, rec, n, d_hist, d_unattr, d_rec_inst);
    else k_attribute<1, false><<<blocks, kThreads, 0, st>>>(T, rec, n, d_hist, d_unattr, nullptr);
  }
  return cudaGetLastError();
}

}  // namespace gpa
