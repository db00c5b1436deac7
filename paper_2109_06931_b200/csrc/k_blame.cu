// k_blame.cu — f4: GPU-idleness blame over trace lines (§6.2 P:970-976:
// "identifies times when all GPU streams are idle and at least one CPU thread is active ...
// partitions the cost of GPU idleness among routines being executed by active CPU threads";
// DESIGN.md reading R27: equal shares, state of a line = ctx of its last change point).
//
// Data-parallel interval sweep, exact in integers:
//   1. k_line_of      event -> line.
//   2. k_merge        log2(lines per rank) rounds of stable merge-path merges of adjacent
//                     sorted runs (the lines) within each rank -> one time-ordered sequence
//                     per rank (times + event ids), 32 outputs per thread.
//   3. k_blame_delta  per sorted position: +-1 change of "GPU lines active" (high 16 bits)
//                     and "CPU lines active" (low 16 bits) packed into one u32; exclusive
//                     scan (mod 2^32) then gives both counts on every elementary interval.
//   4. k_blame_pieces per elementary interval [t_j, t_j+1): GPU-idle time and blameable time
//                     per rank (block-reduced), blameable flags -> scan -> compaction of the
//                     blameable pieces (duration, k).
//   5. k_blame_segs   per CPU segment (an active change point to the next one of its line):
//                     the number of blameable pieces it spans; exclusive scan = work offsets.
//   6. k_blame_work   one work item per (segment, blameable piece): num[rank][routine][k] +=
//                     duration (u64 reductions, run-length aggregated per thread).
//   7. k_blame_fin    blame = sum_k num/k (ascending k), share = blame / total.
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

__device__ __forceinline__ uint64_t upper_bound_u32(const uint32_t *a, uint64_t n, uint32_t x) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    uint64_t mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_line_of(const uint64_t *__restrict__ line_off, uint32_t n_lines, uint64_t n,
                          uint32_t *__restrict__ line_of) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x)
    line_of[e] = (uint32_t)(upper_bound_u64(line_off, n_lines + 1, e) - 1);
}

// one round: output run p = merge of A = [a0, a1) and B = [a1, b1) (B empty: copy)
__global__ void k_merge(const MergePair *__restrict__ pairs, const uint64_t *__restrict__ chunk_start, uint32_t np,
                        const uint64_t *__restrict__ st, const uint32_t *__restrict__ si, uint64_t *__restrict__ dt,
                        uint32_t *__restrict__ di) {
  const uint64_t n_chunks = chunk_start[np];
  for (uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n_chunks;
       c += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t p = (uint32_t)(upper_bound_u64(chunk_start, np + 1, c) - 1);
    const MergePair q = pairs[p];
    const uint64_t na = q.a1 - q.a0, nb = q.b1 - q.a1;
    const uint64_t d = (c - chunk_start[p]) * kMergeChunk, dend = min(d + kMergeChunk, na + nb);
    const uint64_t *A = st + q.a0, *B = st + q.a1;
    // merge path: i = number of A elements among the first d outputs (A first on ties)
    uint64_t lo = d > nb ? d - nb : 0, hi = min(d, na);
    while (lo < hi) {
      uint64_t mid = (lo + hi) >> 1;
      if (A[mid] <= B[d - 1 - mid]) lo = mid + 1; else hi = mid;
    }
    uint64_t i = lo, j = d - lo;
    for (uint64_t o = d; o < dend; o++) {
      const bool takeA = j >= nb || (i < na && A[i] <= B[j]);
      const uint64_t src = takeA ? q.a0 + i : q.a1 + j;
      dt[q.a0 + o] = st[src];
      di[q.a0 + o] = si ? si[src] : (uint32_t)src;
      if (takeA) i++; else j++;
    }
  }
}

__global__ void k_blame_delta(uint64_t n, const uint32_t *__restrict__ ord, const uint32_t *__restrict__ line_of,
                              const uint64_t *__restrict__ line_off, const uint8_t *__restrict__ line_kind,
                              const uint32_t *__restrict__ line_scope, const uint64_t *__restrict__ time,
                              const uint32_t *__restrict__ ctx, uint32_t n_routines, uint32_t *__restrict__ pos,
                              uint32_t *__restrict__ delta, uint32_t *__restrict__ scan, uint32_t *__restrict__ psc,
                              uint32_t *__restrict__ err) {
  uint32_t bad = 0;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t e = ord[j], l = line_of[e];
    pos[e] = (uint32_t)j;
    const uint64_t first = line_off[l], last = line_off[l + 1] - 1;
    const uint32_t c = ctx[e];
    const bool an = c != NONE && e != last;
    const bool ap = e != first && ctx[e - 1] != NONE;
    if (e != first && time[e] < time[e - 1]) bad |= 1;
    const uint8_t kind = line_kind[l];
    if (kind && an && c >= n_routines) bad |= 2;
    const int d = (int)an - (int)ap;
    const uint32_t pk = kind == 0 ? (uint32_t)(d * 65536) : (uint32_t)d;
    delta[j] = pk;
    scan[j] = pk;
    psc[j] = line_scope[l];
  }
  if (bad) atomicOr(err, bad);
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

// compaction of the blameable pieces: (duration, k) at their scan index
__global__ void k_blame_compact(uint64_t n, const uint64_t *__restrict__ st, const uint32_t *__restrict__ delta,
                                const uint32_t *__restrict__ scan, const uint32_t *__restrict__ psc,
                                const uint32_t *__restrict__ bidx, uint64_t *__restrict__ pdur,
                                uint32_t *__restrict__ pk) {
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j + 1 < n; j += (uint64_t)gridDim.x * blockDim.x) {
    if (bidx[j + 1] == bidx[j]) continue;  // not blameable
    const uint32_t P = scan[j] + delta[j];
    pdur[bidx[j]] = st[j + 1] - st[j];
    pk[bidx[j]] = P & 0xFFFF;
  }
}

// CPU segments: number of blameable pieces spanned by the segment starting at event e
__global__ void k_blame_segs(uint64_t n, const uint32_t *__restrict__ line_of, const uint64_t *__restrict__ line_off,
                             const uint8_t *__restrict__ line_kind, const uint32_t *__restrict__ ctx,
                             const uint32_t *__restrict__ pos, const uint32_t *__restrict__ bidx,
                             uint32_t *__restrict__ cnt) {
  for (uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t l = line_of[e];
    uint32_t c = 0;
    if (line_kind[l] && ctx[e] != NONE && e + 1 < line_off[l + 1]) c = bidx[pos[e + 1]] - bidx[pos[e]];
    cnt[e] = c;
  }
}

constexpr int kWorkItems = 16;

__global__ void k_blame_work(uint64_t n, const unsigned long long *__restrict__ W_total,
                             const uint32_t *__restrict__ woff, const uint32_t *__restrict__ pos,
                             const uint32_t *__restrict__ bidx, const uint64_t *__restrict__ pdur,
                             const uint32_t *__restrict__ pk, const uint32_t *__restrict__ line_of,
                             const uint32_t *__restrict__ line_scope, const uint32_t *__restrict__ ctx,
                             uint32_t n_routines, uint32_t kw, unsigned long long *__restrict__ num) {
  const uint64_t W = *W_total;
  for (uint64_t w0 = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) * kWorkItems; w0 < W;
       w0 += (uint64_t)gridDim.x * blockDim.x * kWorkItems) {
    const uint64_t w1 = min(w0 + kWorkItems, W);
    uint64_t e = upper_bound_u32(woff, n, (uint32_t)w0) - 1;
    uint64_t key = ~0ull, run = 0;
    uint32_t seg_end = (e + 1 < n) ? woff[e + 1] : (uint32_t)W;
    uint64_t base = 0;
    for (uint64_t w = w0; w < w1; w++) {
      if (w >= seg_end || w == w0) {
        if (w != w0) {
          e = upper_bound_u32(woff, n, (uint32_t)w) - 1;
          seg_end = (e + 1 < n) ? woff[e + 1] : (uint32_t)W;
        }
        base = ((uint64_t)line_scope[line_of[e]] * n_routines + ctx[e]) * kw;
      }
      const uint32_t piece = bidx[pos[e]] + (uint32_t)(w - woff[e]);
      const uint64_t k2 = base + pk[piece];
      const uint64_t dur = pdur[piece];
      if (k2 != key) {
        if (run) red_add_u64(num + key, run);
        key = k2;
        run = 0;
      }
      run += dur;
    }
    if (run) red_add_u64(num + key, run);
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

cudaError_t blame_line_of(const uint64_t *line_off, uint32_t n_lines, uint64_t n, uint32_t *line_of, cudaStream_t st) {
  k_line_of<<<grid_for(n), 256, 0, st>>>(line_off, n_lines, n, line_of);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t blame_merge(const MergePair *pairs, const uint64_t *chunk_start, uint32_t np, uint64_t n_chunks,
                        const uint64_t *st_in, const uint32_t *si, uint64_t *dt, uint32_t *di, cudaStream_t st) {
  k_merge<<<grid_for(n_chunks), 256, 0, st>>>(pairs, chunk_start, np, st_in, si, dt, di);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t blame_sweep(const BlameArgs &a, cudaStream_t st) {
  const uint64_t n = a.n;
  k_blame_delta<<<grid_for(n), 256, 0, st>>>(n, a.ord, a.line_of, a.line_off, a.line_kind, a.line_scope, a.time,
                                             a.ctx, a.n_routines, a.pos, a.delta, a.scan, a.psc, a.err);
  count_launches(1);
  cudaError_t e = scan_u32(a.scan, n, a.bs, a.tots + 0, st);
  if (e != cudaSuccess) return e;
  const uint64_t tiles = (n + kPieceThreads * kPieceItems - 1) / (kPieceThreads * kPieceItems);
  k_blame_pieces<<<(unsigned)(tiles == 0 ? 1 : (tiles < 148 * 8 ? tiles : 148 * 8)), kPieceThreads, 0, st>>>(
      n, a.st, a.delta, a.scan, a.psc, a.bidx, a.acc, a.n_scopes);
  count_launches(1);
  if ((e = scan_u32(a.bidx, n, a.bs, a.tots + 1, st)) != cudaSuccess) return e;
  k_blame_compact<<<grid_for(n), 256, 0, st>>>(n, a.st, a.delta, a.scan, a.psc, a.bidx, a.pdur, a.pk);
  k_blame_segs<<<grid_for(n), 256, 0, st>>>(n, a.line_of, a.line_off, a.line_kind, a.ctx, a.pos, a.bidx, a.cnt);
  count_launches(2);
  if ((e = scan_u32(a.cnt, n, a.bs, a.tots + 2, st)) != cudaSuccess) return e;
  k_blame_work<<<148 * 8, 256, 0, st>>>(n, a.tots + 2, a.cnt, a.pos, a.bidx, a.pdur, a.pk, a.line_of, a.line_scope,
                                        a.ctx, a.n_routines, a.kmax + 1, a.num);
  const uint64_t ns = (uint64_t)a.n_scopes * a.n_routines;
  k_blame_fin<<<grid_for(ns), 256, 0, st>>>(a.n_scopes, a.n_routines, a.kmax, a.num, a.acc, a.blame, a.share,
                                            a.total, a.gpu_idle);
  count_launches(2);
  return cudaGetLastError();
}

}  // namespace gpa
