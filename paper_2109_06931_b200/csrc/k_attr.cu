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
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
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
    v = e ? atoi(e) : 2;
  }
  return v;
}

}  // namespace

cudaError_t launch_attribute(const AttrTables &T, const gpa_sample *d_samples, uint64_t n,
                             unsigned long long *d_hist, unsigned long long *d_unattr, uint32_t *d_rec_inst,
                             int sm_count, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const uint4 *rec = reinterpret_cast<const uint4 *>(d_samples);
  count_launches(1);
  int var = attr_variant();  // 1: register-streaming kernel; 2: TMA ring + warp aggregation;
                             // 3: TMA ring, one reduction per record
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
