// k_blame.cu — f4: GPU-idleness blame over trace lines (§6.2 P:970-976:
// "identifies times when all GPU streams are idle and at least one CPU thread is active ...
// partitions the cost of GPU idleness among routines being executed by active CPU threads";
// DESIGN.md reading R27: equal shares, state of a line = ctx of its last change point).
//
// Data-parallel interval sweep, exact in integers:
//   1. k_blame_prep   per event in line order: line, activity change (-1/0/+1), kind, rank packed in
//                     one u32; validation (time order, routine ids).
//   2. k_merge        log2(lines per rank) rounds of stable merge-path merges of adjacent
//                     sorted runs (the lines) within each rank -> one time-ordered sequence
//                     per rank (times + event ids), 32 outputs per thread.
//   3. k_blame_delta  per sorted position: the change of "GPU lines active" (high 16 bits)
//                     and "CPU lines active" (low 16 bits) packed into one u32; exclusive
//                     scan (mod 2^32) then gives both counts on every elementary interval.
//   4. k_blame_pieces per elementary interval [t_j, t_j+1): GPU-idle time and blameable time
//                     per rank (block-reduced), blameable flags -> scan -> compaction of the
//                     blameable pieces (duration, k).
//   5. k_blame_segwork per CPU segment (listed by k_blame_compact) (an active change point to the next one of its line):
//                     num[rank][routine][k] += duration over the blameable pieces it spans (u64
//                     reductions, run-length aggregated); segments longer than 256 pieces queue
//                     their remaining chunks for k_blame_overflow.
//   6. k_blame_fin    blame = sum_k num/k (ascending k), share = blame / total.
#include <cuda_runtime.h>
#include <stdint.h>

#include "gpa_internal.cuh"
#include "kern_common.cuh"

namespace gpa {
namespace {

constexpr int kMergeChunk = kMergeChunkHost;
constexpr int kPieceThreads = 256, kPieceItems = 8;

__device__ __forceinline__ uint64_t upper_bound_u64(const uint64_t *a, uint64_t n, uint64_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// per event, in line order (coalesced): info = scope << 4 | active << 3 | kind << 2 | (d + 1) with
// active = the line is active after this change point and d = its change of activity (-1, 0, +1);
// validation flags: err bit 0 = a line goes back in time, bit 1 = CPU routine id >= n_routines
__global__ void k_blame_prep(const uint64_t *__restrict__ line_off, const uint8_t *__restrict__ line_kind,
                             const uint32_t *__restrict__ line_scope, uint32_t n_lines, uint64_t n,
                             const uint64_t *__restrict__ time, const uint32_t *__restrict__ ctx,
                             uint32_t n_routines, uint32_t *__restrict__ info, uint32_t *__restrict__ err) {
  constexpr int kItems = 8;
  const uint64_t T = blockDim.x;
  uint32_t bad = 0;
  for (uint64_t b0 = (uint64_t)blockIdx.x * T * kItems; b0 < n; b0 += (uint64_t)gridDim.x * T * kItems) {
    uint64_t e = b0 + threadIdx.x;
    if (e >= n) break;
    uint32_t l = (uint32_t)(upper_bound_u64(line_off, n_lines + 1, e) - 1);
#pragma unroll
    for (int q = 0; q < kItems; q++, e += T) {
      if (e >= n) break;
      while (line_off[l + 1] <= e) l++;
      const uint64_t first = line_off[l], last = line_off[l + 1] - 1;
      const uint32_t c = ctx[e], kind = line_kind[l];
      const bool an = c != NONE && e != last;
      const bool ap = e != first && ctx[e - 1] != NONE;
      if (e != first && time[e] < time[e - 1]) bad |= 1;
      if (kind && an && c >= n_routines) bad |= 2;
      info[e] = line_scope[l] << 4 | (uint32_t)an << 3 | kind << 2 | (uint32_t)((int)an - (int)ap + 1);
    }
  }
  if (bad) atomicOr(err, bad);
}

// one round: output run p = merge of A = [a0, a1) and B = [a1, b1) (B empty: copy).  One CTA
// per tile of kMergeTile outputs: the tile's merge-path split is found in global memory, both
// input windows are staged in shared memory with coalesced loads, every thread merges
// kMergeItems outputs from shared memory (A first on ties: stable), and the tile is written
// back through shared memory with coalesced stores.
constexpr int kMergeThreads = 256, kMergeItems = kMergeChunk / kMergeThreads;

// merge-path split of every tile start (thread per tile; all searches in flight at once)
__global__ void k_merge_split(const MergePair *__restrict__ pairs, const uint64_t *__restrict__ tile_start,
                              uint32_t np, const uint64_t *__restrict__ st, uint64_t *__restrict__ split,
                              uint32_t *__restrict__ tile_pair) {
  const uint64_t n_tiles = tile_start[np];
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c <= n_tiles;
       c += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t i = 0;
    if (c < n_tiles) {
      const uint32_t p = (uint32_t)(upper_bound_u64(tile_start, np + 1, c) - 1);
      tile_pair[c] = p;
      const MergePair q = pairs[p];
      const uint64_t na = q.a1 - q.a0, nb = q.b1 - q.a1;
      const uint64_t d = (c - tile_start[p]) * kMergeChunk;
      const uint64_t *A = st + q.a0, *B = st + q.a1;
      uint64_t lo = d > nb ? d - nb : 0, hi = min(d, na);
      while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if (A[mid] <= B[d - 1 - mid]) lo = mid + 1; else hi = mid;
      }
      i = lo;
    }
    split[c] = i;  // split[n_tiles] unused (tile ends are computed from the pair)
  }
}
static_assert(kMergeItems * kMergeThreads == kMergeChunk, "tile");

struct MergeTile {
  uint64_t a0, a1, d0, i0, j0;
  int la, m;
};

__device__ __forceinline__ MergeTile merge_tile(const MergePair *__restrict__ pairs,
                                                const uint64_t *__restrict__ tile_start,
                                                const uint32_t *__restrict__ tile_pair,
                                                const uint64_t *__restrict__ split, uint64_t c) {
  const uint32_t p = tile_pair[c];
  const MergePair q = pairs[p];
  const uint64_t na = q.a1 - q.a0, nb = q.b1 - q.a1;
  const uint64_t d0 = (c - tile_start[p]) * kMergeChunk, d1 = min(d0 + kMergeChunk, na + nb);
  const bool last = c + 1 == tile_start[p + 1];
  const uint64_t i0 = split[c], i1 = last ? na : split[c + 1];
  return MergeTile{q.a0, q.a1, d0, i0, d0 - i0, (int)(i1 - i0), (int)(d1 - d0)};
}

__device__ __forceinline__ void cp_async8(void *s, const void *g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async4(void *s, const void *g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(s)), "l"(g) : "memory");
}

// Tiles are double-buffered: while a CTA merges tile c from one buffer, the asynchronous copies
// (cp.async, no registers) of its next tile land in the other.
__global__ void __launch_bounds__(kMergeThreads) k_merge(const MergePair *__restrict__ pairs,
                                                       const uint64_t *__restrict__ tile_start, uint32_t np,
                                                       const uint64_t *__restrict__ st,
                                                       const uint32_t *__restrict__ si, uint64_t *__restrict__ dt,
                                                       uint32_t *__restrict__ di,
                                                       const uint64_t *__restrict__ split,
                                                       const uint32_t *__restrict__ tile_pair) {
  __shared__ __align__(16) uint64_t skb[2][kMergeChunk];
  __shared__ __align__(16) uint32_t svb[2][kMergeChunk];
  const uint64_t n_tiles = tile_start[np];
  auto issue = [&](uint64_t c, int buf) {
    const MergeTile T = merge_tile(pairs, tile_start, tile_pair, split, c);
#pragma unroll
    for (int u = 0; u < kMergeItems; u++) {
      const int x = (int)threadIdx.x + u * kMergeThreads;
      if (x < T.m) {
        const uint64_t src = x < T.la ? T.a0 + T.i0 + x : T.a1 + T.j0 + (x - T.la);
        cp_async8(&skb[buf][x], st + src);
        if (si) cp_async4(&svb[buf][x], si + src);
        else svb[buf][x] = (uint32_t)src;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int buf = 0;
  if (blockIdx.x < n_tiles) issue(blockIdx.x, 0);
  for (uint64_t c = blockIdx.x; c < n_tiles; c += gridDim.x, buf ^= 1) {
    if (c + gridDim.x < n_tiles) issue(c + gridDim.x, buf ^ 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    const MergeTile T = merge_tile(pairs, tile_start, tile_pair, split, c);
    uint64_t *sk = skb[buf];
    uint32_t *sv = svb[buf];
    const int la = T.la, m = T.m, lb = m - la;
    const uint64_t d0 = T.d0;
    const int dd = min((int)threadIdx.x * kMergeItems, m);
    int lo = dd > lb ? dd - lb : 0, hi = min(dd, la);
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (sk[mid] <= sk[la + dd - 1 - mid]) lo = mid + 1; else hi = mid;
    }
    int i = lo, j = dd - lo;
    uint64_t rk[kMergeItems];
    uint32_t rv[kMergeItems];
    uint64_t ka = i < la ? sk[i] : 0, kb = j < lb ? sk[la + j] : 0;  // heads kept in registers
#pragma unroll
    for (int o = 0; o < kMergeItems; o++) {
      if (dd + o < m) {
        const bool takeA = j >= lb || (i < la && ka <= kb);
        if (takeA) {
          rk[o] = ka;
          rv[o] = sv[i];
          if (++i < la) ka = sk[i];
        } else {
          rk[o] = kb;
          rv[o] = sv[la + j];
          if (++j < lb) kb = sk[la + j];
        }
      }
    }
    __syncthreads();
    // stage the tile for coalesced stores; XOR swizzles keep the stride-8 writes conflict-free
#pragma unroll
    for (int o = 0; o < kMergeItems; o++)
      if (dd + o < m) {
        const int x = dd + o;
        sk[x ^ ((x >> 3) & 15)] = rk[o];
        sv[x ^ ((x >> 3) & 31)] = rv[o];
      }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kMergeItems; u++) {
      const int x = (int)threadIdx.x + u * kMergeThreads;
      if (x < m) {
        __stcs(dt + T.a0 + d0 + x, (unsigned long long)sk[x ^ ((x >> 3) & 15)]);
        __stcs(di + T.a0 + d0 + x, sv[x ^ ((x >> 3) & 31)]);
      }
    }
    __syncthreads();
  }
}

__global__ void k_blame_delta(uint64_t n, const uint32_t *__restrict__ ord, const uint32_t *__restrict__ info,
                              uint32_t *__restrict__ delta, uint32_t *__restrict__ scan, uint32_t *__restrict__ psc) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t e = ord[j], f = info[e];
    const int d = (int)(f & 3) - 1;
    const uint32_t pk = (f & 4) ? (uint32_t)d : (uint32_t)(d * 65536);
    delta[j] = pk;
    scan[j] = pk;
    psc[j] = f >> 4;
  }
}

__device__ __forceinline__ unsigned long long block_sum_u64(unsigned long long v) {
  __shared__ unsigned long long ws[32];
  for (int o = 16; o; o >>= 1) v += __shfl_down_sync(kFull, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) ws[wid] = v;
  __syncthreads();
  unsigned long long t = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += ws[w];
  return t;
}

// elementary intervals: GPU-idle / blameable time per rank, blameable flags (into bflag)
__global__ void __launch_bounds__(kPieceThreads) k_blame_pieces(uint64_t n, const uint64_t *__restrict__ st,
                                                              const uint32_t *__restrict__ delta,
                                                              const uint32_t *__restrict__ scan,
                                                              const uint32_t *__restrict__ psc,
                                                              uint32_t *__restrict__ bflag,
                                                              unsigned long long *__restrict__ acc /*[2*S]*/,
                                                              uint32_t n_scopes) {
  const uint64_t tiles = (n + kPieceThreads * kPieceItems - 1) / (kPieceThreads * kPieceItems);
  for (uint64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const uint64_t j0 = tile * kPieceThreads * kPieceItems;
    const uint32_t sc0 = psc[j0];
    unsigned long long idle = 0, blam = 0;
#pragma unroll
    for (int q = 0; q < kPieceItems; q++) {
      const uint64_t j = j0 + (uint64_t)q * kPieceThreads + threadIdx.x;
      if (j >= n) break;
      const uint32_t P = scan[j] + delta[j], sc = psc[j];
      const uint32_t cov = P >> 16, k = P & 0xFFFF;
      uint64_t dur = 0;
      if (j + 1 < n && psc[j + 1] == sc) dur = st[j + 1] - st[j];
      const bool gi = dur && cov == 0, b = gi && k;
      bflag[j] = b;
      if (gi) {
        if (sc == sc0) {
          idle += dur;
          blam += b ? dur : 0;
        } else {
          atomicAdd(acc + sc, (unsigned long long)dur);
          if (b) atomicAdd(acc + n_scopes + sc, (unsigned long long)dur);
        }
      }
    }
    idle = block_sum_u64(idle);
    blam = block_sum_u64(blam);
    if (threadIdx.x == 0) {
      if (idle) atomicAdd(acc + sc0, idle);
      if (blam) atomicAdd(acc + n_scopes + sc0, blam);
    }
  }
}

// compaction of the blameable pieces: (duration, k) at their scan index; every change point e
// also learns the index of the first blameable piece at or after it (bpos[e], a scatter through
// the sorted order) so a CPU segment [e, e+1) spans pieces [bpos[e], bpos[e+1]).  Active CPU
// change points (segment starts) of CTA r's kSegRegion sorted positions are listed in region r
// of seg[] (shared-memory counter, no global atomics; order inside a region is irrelevant because
// the segments' contributions are integer sums); seg_n[r] = their number.
constexpr int kSegRegion = 8192, kCompactThreads = 256;
constexpr uint32_t kSegTabBytes = 96 * 1024;

__global__ void __launch_bounds__(kCompactThreads) k_blame_compact(
    uint64_t n, const uint64_t *__restrict__ st, const uint32_t *__restrict__ delta, const uint32_t *__restrict__ scan,
    const uint32_t *__restrict__ ord, const uint32_t *__restrict__ info, const uint32_t *__restrict__ ctx,
    const uint32_t *__restrict__ bidx, uint64_t *__restrict__ pdur, uint32_t *__restrict__ pk,
    uint32_t *__restrict__ bpos, uint32_t n_routines, uint2 *__restrict__ seg, uint32_t *__restrict__ seg_n) {
  __shared__ uint32_t cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  const uint64_t r0 = (uint64_t)blockIdx.x * kSegRegion;
  uint2 *out = seg + r0;
  for (int i = threadIdx.x; i < kSegRegion; i += kCompactThreads) {
    const uint64_t j = r0 + i;
    bool act = false;
    uint32_t e = 0, f = 0;
    if (j < n) {
      e = ord[j];
      const uint32_t b = bidx[j];
      f = info[e];
      bpos[e] = b;
      act = (f & 12) == 12;  // active CPU change point: a segment starts here
      if (j + 1 < n && bidx[j + 1] != b) {
        const uint32_t P = scan[j] + delta[j];
        pdur[b] = st[j + 1] - st[j];
        pk[b] = P & 0xFFFF;
      }
    }
    const unsigned m = __ballot_sync(kFull, act);
    const int lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (m && lane == 0) base = atomicAdd(&cnt, (uint32_t)__popc(m));
    base = __shfl_sync(kFull, base, 0);
    if (act) out[base + __popc(m & ((1u << lane) - 1))] = make_uint2(e, (f >> 4) * n_routines + ctx[e]);
  }
  __syncthreads();
  if (threadIdx.x == 0) seg_n[blockIdx.x] = cnt;
}

// CPU segments: thread per change point e; an active CPU change point starts a segment that
// spans the blameable pieces [bidx[pos[e]], bidx[pos[e+1]]).  The thread adds up to kSegChunk of
// them (run-length aggregated by k) into num[rank][routine][k]; the rest of a longer segment is
// queued in chunks of kSegChunk for k_blame_overflow, so no thread serialises a long segment.
constexpr uint32_t kSegChunk = 256;

__device__ __forceinline__ void blame_add(unsigned long long *num, uint64_t rbase, uint32_t p0, uint32_t p1,
                                          const uint64_t *__restrict__ pdur, const uint32_t *__restrict__ pk) {
  uint32_t key = ~0u;
  unsigned long long run = 0;
  constexpr int B = 8;  // pieces loaded per batch (independent loads in flight)
  for (uint32_t p = p0; p < p1; p += B) {
    uint32_t kk[B];
    uint64_t dd[B];
#pragma unroll
    for (int q = 0; q < B; q++)
      if (p + q < p1) {
        kk[q] = pk[p + q];
        dd[q] = pdur[p + q];
      }
#pragma unroll
    for (int q = 0; q < B; q++)
      if (p + q < p1) {
        if (kk[q] != key) {
          if (run) red_add_u64(num + rbase + key, run);
          key = kk[q];
          run = 0;
        }
        run += dd[q];
      }
  }
  if (run) red_add_u64(num + rbase + key, run);
}

// CTA r takes the segments listed in region r (all from kSegRegion consecutive sorted positions,
// so nearly always one rank): rows of that rank accumulate in a shared-memory table
// [routine][k] (tab_n > 0) flushed with one u64 reduction per non-zero entry; other ranks and
// overflow chunks go straight to L2.
__device__ __forceinline__ void blame_add_smem(unsigned long long *row, uint32_t p0, uint32_t p1,
                                               const uint64_t *__restrict__ pdur, const uint32_t *__restrict__ pk) {
  constexpr int B = 8;
  for (uint32_t p = p0; p < p1; p += B) {
    uint32_t kk[B];
    uint64_t dd[B];
#pragma unroll
    for (int q = 0; q < B; q++)
      if (p + q < p1) {
        kk[q] = pk[p + q];
        dd[q] = pdur[p + q];
      }
#pragma unroll
    for (int q = 0; q < B; q++)
      if (p + q < p1) atomicAdd(row + kk[q], (unsigned long long)dd[q]);
  }
}

__global__ void __launch_bounds__(kCompactThreads) k_blame_segwork(
    const uint32_t *__restrict__ seg_n, const uint2 *__restrict__ seg, const uint32_t *__restrict__ bpos,
    const uint64_t *__restrict__ pdur, const uint32_t *__restrict__ pk, uint32_t n_routines, uint32_t kw,
    uint32_t tab_n, unsigned long long *__restrict__ num, uint2 *__restrict__ ovf, uint32_t *__restrict__ n_ovf) {
  extern __shared__ unsigned long long tab[];
  const uint32_t m = seg_n[blockIdx.x];
  if (m == 0) return;  // uniform over the CTA
  const uint2 *in = seg + (uint64_t)blockIdx.x * kSegRegion;
  const uint32_t tsc = in[0].y / n_routines;
  for (uint32_t x = threadIdx.x; x < tab_n; x += kCompactThreads) tab[x] = 0;
  __syncthreads();
  for (uint32_t x = threadIdx.x; x < m; x += kCompactThreads) {
    const uint2 sg = in[x];
    const uint32_t e = sg.x, p0 = bpos[e], p1 = bpos[e + 1];
    if (p0 == p1) continue;
    const uint32_t pm = p1 - p0 > kSegChunk ? p0 + kSegChunk : p1;
    if (tab_n && sg.y / n_routines == tsc) blame_add_smem(tab + (uint64_t)(sg.y % n_routines) * kw, p0, pm, pdur, pk);
    else blame_add(num, (uint64_t)sg.y * kw, p0, pm, pdur, pk);
    for (uint32_t q = pm; q < p1; q += kSegChunk)
      ovf[atomicAdd(n_ovf, 1u)] = make_uint2((uint32_t)(blockIdx.x * kSegRegion + x), q);
  }
  __syncthreads();
  const uint64_t tb = (uint64_t)tsc * n_routines * kw;
  for (uint32_t x = threadIdx.x; x < tab_n; x += kCompactThreads)
    if (tab[x]) red_add_u64(num + tb + x, tab[x]);
}

__global__ void k_blame_overflow(const uint32_t *__restrict__ n_ovf, const uint2 *__restrict__ ovf,
                                 const uint2 *__restrict__ seg, const uint32_t *__restrict__ bpos,
                                 const uint64_t *__restrict__ pdur, const uint32_t *__restrict__ pk, uint32_t kw,
                                 unsigned long long *__restrict__ num) {
  const uint32_t m = *n_ovf;
  for (uint32_t x = blockIdx.x * blockDim.x + threadIdx.x; x < m; x += gridDim.x * blockDim.x) {
    const uint2 v = ovf[x];
    const uint2 sg = seg[v.x];
    const uint32_t p1 = bpos[sg.x + 1];
    blame_add(num, (uint64_t)sg.y * kw, v.y, min(v.y + kSegChunk, p1), pdur, pk);
  }
}

__global__ void k_blame_fin(uint32_t n_scopes, uint32_t n_routines, uint32_t kmax,
                            const unsigned long long *__restrict__ num, const unsigned long long *__restrict__ acc,
                            double *__restrict__ blame, double *__restrict__ share, uint64_t *__restrict__ total,
                            uint64_t *__restrict__ gpu_idle) {
  const uint64_t n = (uint64_t)n_scopes * n_routines;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) {
    const unsigned long long *v = num + x * (kmax + 1);
    double b = 0.0;
    for (uint32_t k = 1; k <= kmax; k++) b = __dadd_rn(b, __ddiv_rn((double)v[k], (double)k));
    const uint32_t s = (uint32_t)(x / n_routines);
    const uint64_t t = acc[n_scopes + s];
    if (blame) blame[x] = b;
    if (share) share[x] = t ? __ddiv_rn(b, (double)t) : __longlong_as_double(0x7FF8000000000000ll);
    if (x % n_routines == 0) {
      if (total) total[s] = t;
      if (gpu_idle) gpu_idle[s] = acc[s];
    }
  }
}

unsigned grid_for(uint64_t n, unsigned threads = 256) {
  uint64_t b = (n + threads - 1) / threads;
  return (unsigned)(b < 148 * 16 ? (b ? b : 1) : 148 * 16);
}

}  // namespace

cudaError_t blame_prep(const BlameArgs &a, uint32_t n_lines, cudaStream_t st) {
  k_blame_prep<<<grid_for(a.n, 256 * 8), 256, 0, st>>>(a.line_off, a.line_kind, a.line_scope, n_lines, a.n, a.time,
                                                        a.ctx, a.n_routines, a.info, a.err);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t blame_merge(const MergePair *pairs, const uint64_t *chunk_start, uint32_t np, uint64_t n_chunks,
                        const uint64_t *st_in, const uint32_t *si, uint64_t *dt, uint32_t *di, uint64_t *split,
                        cudaStream_t st) {
  uint32_t *tile_pair = reinterpret_cast<uint32_t *>(split + n_chunks + 1);
  k_merge_split<<<grid_for(n_chunks + 1), 256, 0, st>>>(pairs, chunk_start, np, st_in, split, tile_pair);
  k_merge<<<(unsigned)(n_chunks < 148 * 16 ? (n_chunks ? n_chunks : 1) : 148 * 16), kMergeThreads, 0, st>>>(
      pairs, chunk_start, np, st_in, si, dt, di, split, tile_pair);
  count_launches(2);
  return cudaGetLastError();
}

cudaError_t blame_sweep(const BlameArgs &a, cudaStream_t st) {
  const uint64_t n = a.n;
  k_blame_delta<<<grid_for(n), 256, 0, st>>>(n, a.ord, a.info, a.delta, a.scan, a.psc);
  count_launches(1);
  cudaError_t e = scan_u32(a.scan, n, a.bs, a.tots + 0, st);
  if (e != cudaSuccess) return e;
  const uint64_t tiles = (n + kPieceThreads * kPieceItems - 1) / (kPieceThreads * kPieceItems);
  k_blame_pieces<<<(unsigned)(tiles == 0 ? 1 : (tiles < 148 * 8 ? tiles : 148 * 8)), kPieceThreads, 0, st>>>(
      n, a.st, a.delta, a.scan, a.psc, a.bidx, a.acc, a.n_scopes);
  count_launches(1);
  if ((e = scan_u32(a.bidx, n, a.bs, a.tots + 1, st)) != cudaSuccess) return e;
  const unsigned regions = (unsigned)((n + kSegRegion - 1) / kSegRegion);
  if (regions) {
    k_blame_compact<<<regions, kCompactThreads, 0, st>>>(n, a.st, a.delta, a.scan, a.ord, a.info, a.ctx, a.bidx,
                                                         a.pdur, a.pk, a.pos, a.n_routines, a.seg, a.seg_n);
    const uint64_t tab = (uint64_t)a.n_routines * (a.kmax + 1);
    const uint32_t tab_n = tab * 8 <= kSegTabBytes ? (uint32_t)tab : 0;
    if (tab_n * 8 > 48 * 1024 &&
        (e = cudaFuncSetAttribute(k_blame_segwork, cudaFuncAttributeMaxDynamicSharedMemorySize, kSegTabBytes)) !=
            cudaSuccess)
      return e;
    k_blame_segwork<<<regions, kCompactThreads, tab_n * 8, st>>>(a.seg_n, a.seg, a.pos, a.pdur, a.pk, a.n_routines,
                                                                  a.kmax + 1, tab_n, a.num, a.ovf, a.err + 1);
    k_blame_overflow<<<148 * 4, 256, 0, st>>>(a.err + 1, a.ovf, a.seg, a.pos, a.pdur, a.pk, a.kmax + 1, a.num);
    count_launches(3);
  }
  const uint64_t ns = (uint64_t)a.n_scopes * a.n_routines;
  k_blame_fin<<<grid_for(ns), 256, 0, st>>>(a.n_scopes, a.n_routines, a.kmax, a.num, a.acc, a.blame, a.share,
                                            a.total, a.gpu_idle);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace gpa
