// k_cct.cu — a-6..a-9: approximate GPU calling-context tree (§5.3).
//
//  Step 1  k_weights      w_e = valid samples on call instruction e (R10)
//  Step 2  k_propagate    zero-weight propagation to the least fixpoint (R11), the
//                                 same rule on the condensed DAG (guard, R12), W_X, and the
//                                 exact context count by a path DP over the static DAG levels
//  Step 3  load time      Tarjan condensation (gpa_host.cu)
//  Step 4  k_roots, k_level_count / scan / k_level_write: breadth-first split of
//                                 the DAG into the tree, one level at a time (count children,
//                                 exclusive scan = BFS numbering R17, write children with
//                                 f(child) = f(parent) * w_e / W_callee, R13);
//                  k_excl         excl = f * S_function (0 for SCC contexts, R14);
//                  k_incl_level   incl = excl + children's incl in child order, deepest
//                                 level first.
// Every fp64 operation is one correctly rounded __d*_rn call in the oracle's order.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <stdint.h>

#include "gpa_internal.cuh"
#include "kern_common.cuh"

namespace gpa {
namespace {

constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr unsigned long long SAT = 1ull << 62;

__global__ void k_weights(const uint32_t *__restrict__ call_inst, uint32_t n_call, const uint64_t *__restrict__ H,
                          uint64_t *__restrict__ w, uint32_t lo = 0, uint32_t hi = 0xFFFFFFFFu) {
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n_call; e += gridDim.x * blockDim.x) {
    const uint32_t ci = call_inst[e];
    if (ci < lo || ci >= hi) continue;  // another rank's call site (gpa_cct_inputs)
    const uint64_t *h = H + ((uint64_t)ci << 4);
    uint64_t s = 0;
#pragma unroll
    for (int r = 0; r < GPA_VALID_SLOTS; r++) s += h[r];
    w[e] = s;
  }
}

struct PropArgs {
  uint32_t n_func, n_dag, n_lev, exact, do_count, n_call;
  const uint64_t *S_f;
  const uint32_t *fin_ptr, *fin_e, *caller, *scc_of, *din_ptr, *din_e, *dmem_ptr, *dmem, *dlev_ptr, *dlev_node;
  const uint8_t *nontriv;
  uint64_t *w, *W, *paths;
  uint8_t *fact, *dact;
  unsigned long long *count;
  uint32_t *q0, *q1;  // worklists, max(n_func, n_dag) entries each
  uint32_t n_ext;     // external call sites (din_e entries)
  uint32_t stage_dp;  // SM only: the DP's static tables fit behind the mutable state
  uint32_t batch;     // gridDim.x problems (R30): block b works on problem b's slices
  uint64_t fstride, dstride, pstride;  // activity bytes per problem (func, DAG); paths + q u64 per problem
};

// set byte flag[i] to 1; true if it was 0 (byte flags live in 32-bit words: atomicOr)
__device__ __forceinline__ bool set_flag(volatile uint8_t *flag, uint32_t i) {
  uintptr_t a = (uintptr_t)(flag + i);
  unsigned *word = (unsigned *)(a & ~(uintptr_t)3);
  const unsigned sh = 8u * (unsigned)(a & 3);
  return ((atomicOr(word, 1u << sh) >> sh) & 0xFFu) == 0;
}

// Single CTA: the call graph is small (<= a few thousand functions); rounds are separated
// by __syncthreads, which also orders the memory updates inside the CTA.  SM = true: the
// mutable state (w, function / DAG activity, path counts) lives in shared memory for the
// whole kernel (every fixpoint round then costs shared-memory, not L2, latency) and is
// written back at the end; the read-only graph tables stay in global memory (L1-cached).
template <bool SM>
__global__ void __launch_bounds__(1024) k_propagate(PropArgs A0) {
  PropArgs A = A0;
  if (A.batch) {  // one independent problem per block (per-profile trees, R30)
    const uint64_t b = blockIdx.x;
    A.S_f += b * A.n_func * GPA_SLOTS;
    A.w += b * A.n_call;
    A.W += b * A.n_dag;
    A.fact += b * A.fstride;
    A.dact += b * A.dstride;
    A.paths += b * A.pstride;
    A.q0 = reinterpret_cast<uint32_t *>(A.paths + A.n_dag + 1);
    A.q1 = A.q0 + (A.pstride - A.n_dag - 1);
  }
  __shared__ unsigned long long red[32];
  extern __shared__ __align__(16) uint8_t psm[];
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  volatile uint8_t *fact = A.fact;
  volatile uint8_t *dact = A.dact;
  volatile uint64_t *w = A.w;
  volatile uint64_t *paths = A.paths;
  if (SM) {
    uint64_t *ws = reinterpret_cast<uint64_t *>(psm);
    uint64_t *ps = ws + A.n_call;
    uint8_t *fs = reinterpret_cast<uint8_t *>(ps + A.n_dag);
    for (uint32_t e = t; e < A.n_call; e += nt) ws[e] = A.w[e];
    w = ws;
    paths = ps;
    fact = fs;
    dact = fs + A.n_func;
  }
  // a function is active if any valid slot of S_f is non-zero: six independent 16-B loads per
  // function row (a dependent 12-load loop behind volatile stores serialised on L2 latency)
  {
    uint8_t *fw = const_cast<uint8_t *>(fact);
#pragma unroll 2
    for (uint32_t f = t; f < A.n_func; f += nt) {
      const ulonglong2 *row = reinterpret_cast<const ulonglong2 *>(A.S_f + (uint64_t)f * GPA_SLOTS);
      ulonglong2 v[GPA_VALID_SLOTS / 2];
#pragma unroll
      for (int q = 0; q < GPA_VALID_SLOTS / 2; q++) v[q] = __ldg(row + q);
      unsigned long long o = 0;
#pragma unroll
      for (int q = 0; q < GPA_VALID_SLOTS / 2; q++) o |= v[q].x | v[q].y;
      fw[f] = o != 0;
    }
  }
  // Step 2: "if a function has samples and none of its incoming call edges has a non-zero
  // weight, we assign each of its incoming call edges a weight of one; we repeat this
  // propagation through callers".  A function's in-edges are written only when that
  // function is processed, so each active function needs processing exactly once: a worklist
  // of the initially active functions, then of the callers each round activates (the least
  // fixpoint of R11, O(F + E) work; rounds = length of the longest zero-weight chain).
  // Exact counts skip it ("For call graphs based on samples", R24).
  __shared__ uint32_t qn[2];
  auto run_worklist = [&](uint32_t n_items, volatile uint8_t *act, const uint32_t *in_ptr, const uint32_t *in_e,
                          bool dag) {
    __syncthreads();
    if (t == 0) qn[0] = 0;
    __syncthreads();
    for (uint32_t x = t; x < n_items; x += nt)
      if (act[x]) A.q0[atomicAdd(&qn[0], 1u)] = x;
    uint32_t cur = 0;
    for (;;) {
      __syncthreads();
      const uint32_t m = qn[cur];
      if (m == 0) break;
      if (t == 0) qn[cur ^ 1] = 0;
      __syncthreads();
      uint32_t *qc = cur ? A.q1 : A.q0, *qx = cur ? A.q0 : A.q1;
      for (uint32_t i = t; i < m; i += nt) {
        const uint32_t x = qc[i], a = in_ptr[x], b = in_ptr[x + 1];
        if (a == b) continue;
        bool zero = true;
        for (uint32_t k = a; k < b; k++) zero &= w[in_e[k]] == 0;
        if (!zero) continue;
        for (uint32_t k = a; k < b; k++) {
          const uint32_t e = in_e[k];
          w[e] = 1;
          const uint32_t u = dag ? A.scc_of[A.caller[e]] : A.caller[e];
          if (set_flag(act, u)) qx[atomicAdd(&qn[cur ^ 1], 1u)] = u;
        }
      }
      __threadfence_block();
      cur ^= 1;
    }
  };
  if (!A.exact) run_worklist(A.n_func, fact, A.fin_ptr, A.fin_e, false);
  // DAG activity, then the guard (R12): the same rule on external in-edges of DAG nodes
  // (samples mode only, like Step 2)
  __syncthreads();
  for (uint32_t X = t; X < A.n_dag; X += nt) dact[X] = 0;
  __syncthreads();
  for (uint32_t f = t; f < A.n_func; f += nt)  // a DAG node is active if any member is
    if (fact[f]) dact[A.scc_of[f]] = 1;
  if (!A.exact) run_worklist(A.n_dag, dact, A.din_ptr, A.din_e, true);
  // W_X = total weight of the external calls into X
  __syncthreads();
  for (uint32_t X = t; X < A.n_dag; X += nt) {
    uint64_t s = 0;
    for (uint32_t k = A.din_ptr[X]; k < A.din_ptr[X + 1]; k++) s += w[A.din_e[k]];
    A.W[X] = s;
  }
  if (SM) {  // write the shared state back for the tree builders
    for (uint32_t e = t; e < A.n_call; e += nt) A.w[e] = w[e];
    for (uint32_t f = t; f < A.n_func; f += nt) A.fact[f] = fact[f];
    for (uint32_t X = t; X < A.n_dag; X += nt) A.dact[X] = dact[X];
  }
  // exact context count: paths from active roots through edges with w > 0, level by level
  // (skipped when the caller builds the tree into a static-bound allocation and reads the
  // size back afterwards)
  if (!A.do_count) return;
  if (SM && A.stage_dp) {
    // The level loop is a chain of dependent reads; with the weights final, stage per
    // external in-edge its source DAG node (or NONE when w = 0) and per level slot the node
    // and its in-edge range in shared memory in one coalesced pass, so each of the
    // dag_levels rounds costs shared-memory latency only.
    uint32_t *src = reinterpret_cast<uint32_t *>(psm + 8ull * (A.n_call + A.n_dag) + ((A.n_func + A.n_dag + 7) & ~7u));
    uint32_t *lx = src + A.n_ext, *la = lx + A.n_dag, *lb = la + A.n_dag;
    __syncthreads();
    for (uint32_t k = t; k < A.n_ext; k += nt) {
      const uint32_t e = A.din_e[k];
      src[k] = w[e] ? A.scc_of[A.caller[e]] : 0xFFFFFFFFu;
    }
    for (uint32_t q = t; q < A.n_dag; q += nt) {
      const uint32_t X = A.dlev_node[q];
      lx[q] = X;
      la[q] = A.din_ptr[X];
      lb[q] = A.din_ptr[X + 1];
    }
    __syncthreads();
    uint32_t q0 = 0;
    for (uint32_t L = 0; L < A.n_lev; L++) {
      const uint32_t q1 = A.dlev_ptr[L + 1];
      for (uint32_t q = q0 + t; q < q1; q += nt) {
        const uint32_t X = lx[q], a = la[q], b = lb[q];
        unsigned long long p = 0;
        if (a == b) {
          p = dact[X] ? 1 : 0;
        } else {
          for (uint32_t k = a; k < b; k++)
            if (src[k] != 0xFFFFFFFFu) p = min(SAT, p + paths[src[k]]);
        }
        paths[X] = p;
      }
      q0 = q1;
      __syncthreads();
    }
  } else {
    for (uint32_t L = 0; L < A.n_lev; L++) {
      __syncthreads();
      for (uint32_t q = A.dlev_ptr[L] + t; q < A.dlev_ptr[L + 1]; q += nt) {
        uint32_t X = A.dlev_node[q];
        uint32_t a = A.din_ptr[X], b = A.din_ptr[X + 1];
        unsigned long long p = 0;
        if (a == b) {
          p = dact[X] ? 1 : 0;
        } else {
          for (uint32_t k = a; k < b; k++) {
            uint32_t e = A.din_e[k];
            if (w[e]) p = min(SAT, p + paths[A.scc_of[A.caller[e]]]);
          }
        }
        paths[X] = p;
      }
    }
  }
  __syncthreads();
  unsigned long long tot = 0;
  for (uint32_t X = t; X < A.n_dag; X += nt) {
    unsigned long long per = A.nontriv[X] ? 1ull + (A.dmem_ptr[X + 1] - A.dmem_ptr[X]) : 1ull;
    unsigned long long p = paths[X];
    tot = min(SAT, tot + (p > SAT / per ? SAT : p * per));
  }
  for (int o = 16; o; o >>= 1) tot = min(SAT, tot + __shfl_xor_sync(FULL, tot, o));
  if ((t & 31) == 0) red[t >> 5] = tot;
  __syncthreads();
  if (t < 32) {
    tot = t < (nt >> 5) ? red[t] : 0;
    for (int o = 16; o; o >>= 1) tot = min(SAT, tot + __shfl_xor_sync(FULL, tot, o));
    if (t == 0) A.count[0] = tot;
  }
}

// roots: active DAG nodes without external in-edges, in DAG order (R15)
__global__ void __launch_bounds__(1024) k_roots(uint32_t n_dag, const uint32_t *din_ptr, const uint8_t *dact,
                                                const uint8_t *nontriv, uint32_t *parent, uint32_t *site,
                                                uint32_t *node, uint8_t *kind, double *frac,
                                                unsigned long long *n_out) {
  uint32_t running = 0;
  for (uint32_t base = 0; base < n_dag; base += blockDim.x) {
    uint32_t X = base + threadIdx.x;
    uint32_t flag = X < n_dag && din_ptr[X] == din_ptr[X + 1] && dact[X];
    uint32_t tot;
    uint32_t pos = running + block_exscan(flag, &tot);
    if (flag) {
      parent[pos] = NONE;
      site[pos] = NONE;
      node[pos] = X;
      kind[pos] = nontriv[X] ? GPA_CTX_SCC : GPA_CTX_FUNC;
      frac[pos] = 1.0;
    }
    running += tot;
  }
  if (threadIdx.x == 0) n_out[0] = running;
}

struct LevelArgs {
  const uint32_t *fout_ptr, *fout_e, *callee, *scc_of, *dmem_ptr, *dmem;
  const uint8_t *nontriv;
  const uint64_t *w, *W;
  uint32_t *parent, *site, *node, *first_child, *n_children;
  uint8_t *kind;
  double *frac;
};

__device__ __forceinline__ uint32_t func_of_ctx(const LevelArgs &A, uint8_t k, uint32_t nd) {
  return k == GPA_CTX_SCC_MEMBER ? nd : A.dmem[A.dmem_ptr[nd]];
}

__device__ __forceinline__ uint32_t child_count(const LevelArgs &A, uint64_t c) {
  uint8_t k = A.kind[c];
  uint32_t nd = A.node[c];
  if (k == GPA_CTX_SCC) return A.dmem_ptr[nd + 1] - A.dmem_ptr[nd];
  uint32_t g = func_of_ctx(A, k, nd), cnt = 0;
  for (uint32_t q = A.fout_ptr[g]; q < A.fout_ptr[g + 1]; q++) cnt += A.w[A.fout_e[q]] != 0;
  return cnt;
}

__global__ void k_level_count(LevelArgs A, uint64_t a, uint64_t b, uint32_t *tmp) {
  for (uint64_t c = a + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < b; c += (uint64_t)gridDim.x * blockDim.x)
    tmp[c - a] = child_count(A, c);
}

__global__ void k_level_write(LevelArgs A, uint64_t a, uint64_t b, const uint32_t *off) {
  for (uint64_t c = a + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; c < b; c += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t o = b + off[c - a];
    uint8_t k = A.kind[c];
    uint32_t nd = A.node[c];
    double f = A.frac[c];
    uint32_t cnt = 0;
    if (k == GPA_CTX_SCC) {  // members in ascending function id (R14)
      for (uint32_t q = A.dmem_ptr[nd]; q < A.dmem_ptr[nd + 1]; q++, cnt++) {
        uint64_t d = o + cnt;
        A.parent[d] = (uint32_t)c;
        A.site[d] = NONE;
        A.node[d] = A.dmem[q];
        A.kind[d] = GPA_CTX_SCC_MEMBER;
        A.frac[d] = f;
      }
    } else {  // external calls with w > 0, ascending call instruction (R15, R17)
      uint32_t g = func_of_ctx(A, k, nd);
      for (uint32_t q = A.fout_ptr[g]; q < A.fout_ptr[g + 1]; q++) {
        uint32_t e = A.fout_e[q];
        uint64_t we = A.w[e];
        if (!we) continue;
        uint32_t Y = A.scc_of[A.callee[e]];
        uint64_t d = o + cnt++;
        A.parent[d] = (uint32_t)c;
        A.site[d] = e;
        A.node[d] = Y;
        A.kind[d] = A.nontriv[Y] ? GPA_CTX_SCC : GPA_CTX_FUNC;
        A.frac[d] = __dmul_rn(f, __ddiv_rn(__ull2double_rn(we), __ull2double_rn(A.W[Y])));  // R13
      }
    }
    A.first_child[c] = (uint32_t)o;
    A.n_children[c] = cnt;
  }
}

__global__ void k_excl(uint64_t n, const uint8_t *kind, const uint32_t *node, const double *frac,
                       const uint32_t *dmem_ptr, const uint32_t *dmem, const uint64_t *S_f, double *excl) {
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n * GPA_SLOTS;
       x += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c = x >> 4;
    int r = (int)(x & 15);
    uint8_t k = kind[c];
    double v = 0.0;
    if (k != GPA_CTX_SCC) {
      uint32_t g = k == GPA_CTX_SCC_MEMBER ? node[c] : dmem[dmem_ptr[node[c]]];
      v = __dmul_rn(frac[c], __ull2double_rn(S_f[(uint64_t)g * GPA_SLOTS + r]));
    }
    excl[x] = v;
  }
}

__global__ void k_incl_level(uint64_t a, uint64_t b, const uint32_t *first_child, const uint32_t *n_children,
                             const double *excl, double *incl) {
  for (uint64_t x = a * GPA_SLOTS + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < b * GPA_SLOTS;
       x += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t c = x >> 4;
    int r = (int)(x & 15);
    double v = excl[x];
    uint32_t d0 = first_child[c], nc = n_children[c];
    for (uint32_t d = d0; d < d0 + nc; d++) v = __dadd_rn(v, incl[(uint64_t)d * GPA_SLOTS + r]);
    incl[x] = v;
  }
}

// f1 at CCT level (R28): profile p's excl = frac * p's function histogram; incl level by level
__global__ void k_cct_prof_excl(uint64_t n, uint32_t P1, uint32_t n_func, const uint8_t *__restrict__ kind,
                                const uint32_t *__restrict__ node, const double *__restrict__ frac,
                                const uint32_t *__restrict__ dmem_ptr, const uint32_t *__restrict__ dmem,
                                const uint64_t *__restrict__ PH, double *__restrict__ excl) {
  const uint64_t per = n * GPA_SLOTS;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < per * P1;
       x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = x / per, y = x - p * per, c = y >> 4;
    const int r = (int)(y & 15);
    const uint8_t k = kind[c];
    double v = 0.0;
    if (k != GPA_CTX_SCC) {
      const uint32_t g = k == GPA_CTX_SCC_MEMBER ? node[c] : dmem[dmem_ptr[node[c]]];
      v = __dmul_rn(frac[c], __ull2double_rn(PH[(p * n_func + g) * GPA_SLOTS + r]));
    }
    excl[x] = v;
  }
}

__global__ void k_cct_prof_incl_level(uint64_t n, uint64_t a, uint64_t b, uint32_t P1,
                                      const uint32_t *__restrict__ first_child, const uint32_t *__restrict__ n_children,
                                      const double *__restrict__ excl, double *__restrict__ incl) {
  const uint64_t w = (b - a) * GPA_SLOTS;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < w * P1; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t p = x / w, y = a * GPA_SLOTS + (x - p * w), c = y >> 4;
    const int r = (int)(y & 15);
    const double *I = incl + p * n * GPA_SLOTS;
    double v = excl[p * n * GPA_SLOTS + y];
    const uint32_t d0 = first_child[c], nc = n_children[c];
    for (uint32_t d = d0; d < d0 + nc; d++) v = __dadd_rn(v, I[(uint64_t)d * GPA_SLOTS + r]);
    incl[p * n * GPA_SLOTS + y] = v;
  }
}

// Whole Step 4 in one CTA for small trees (the common case: C1, C2, C4, C5 have <= 2^15
// contexts): roots, every BFS level (count -> block scan -> write), excl, and the reverse
// incl fold, separated by __syncthreads instead of kernel launches and host syncs.
constexpr int kSmallLevels = 1024;
constexpr uint64_t kSmallMax = 1ull << 16;

__device__ __forceinline__ void write_children(const LevelArgs &A, uint64_t c, uint64_t o) {
  uint8_t k = A.kind[c];
  uint32_t nd = A.node[c];
  double f = A.frac[c];
  uint32_t cnt = 0;
  if (k == GPA_CTX_SCC) {
    for (uint32_t q = A.dmem_ptr[nd]; q < A.dmem_ptr[nd + 1]; q++, cnt++) {
      uint64_t d = o + cnt;
      A.parent[d] = (uint32_t)c;
      A.site[d] = NONE;
      A.node[d] = A.dmem[q];
      A.kind[d] = GPA_CTX_SCC_MEMBER;
      A.frac[d] = f;
    }
  } else {
    uint32_t g = func_of_ctx(A, k, nd);
    for (uint32_t q = A.fout_ptr[g]; q < A.fout_ptr[g + 1]; q++) {
      uint32_t e = A.fout_e[q];
      uint64_t we = A.w[e];
      if (!we) continue;
      uint32_t Y = A.scc_of[A.callee[e]];
      uint64_t d = o + cnt++;
      A.parent[d] = (uint32_t)c;
      A.site[d] = e;
      A.node[d] = Y;
      A.kind[d] = A.nontriv[Y] ? GPA_CTX_SCC : GPA_CTX_FUNC;
      A.frac[d] = __dmul_rn(f, __ddiv_rn(__ull2double_rn(we), __ull2double_rn(A.W[Y])));  // R13
    }
  }
  A.first_child[c] = (uint32_t)o;
  A.n_children[c] = cnt;
}

__global__ void __launch_bounds__(1024) k_cct_small(LevelArgs A, uint32_t n_dag, const uint32_t *din_ptr,
                                                    const uint8_t *dact, uint32_t *lev_out,
                                                    unsigned long long *built, uint64_t cap) {
  __shared__ uint32_t lev[kSmallLevels + 1];
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  uint32_t running = 0;
  for (uint32_t base = 0; base < n_dag; base += nt) {  // roots in DAG order (R15)
    uint32_t X = base + t;
    uint32_t flag = X < n_dag && din_ptr[X] == din_ptr[X + 1] && dact[X];
    uint32_t tot;
    uint32_t pos = running + block_exscan(flag, &tot);
    if (flag && pos < cap) {
      A.parent[pos] = NONE;
      A.site[pos] = NONE;
      A.node[pos] = X;
      A.kind[pos] = A.nontriv[X] ? GPA_CTX_SCC : GPA_CTX_FUNC;
      A.frac[pos] = 1.0;
    }
    running += tot;
  }
  __syncthreads();
  uint32_t a = 0, b = running, L = 0;
  if (t == 0) lev[0] = 0;
  while (b > a && L < kSmallLevels) {
    if (t == 0) lev[L + 1] = b;
    L++;
    uint32_t next = b;
    for (uint32_t base = a; base < b; base += nt) {
      uint32_t c = base + t;
      uint32_t cnt = c < b ? child_count(A, c) : 0;
      uint32_t tot;
      uint32_t off = block_exscan(cnt, &tot);
      if (c < b && next + off + cnt <= cap) write_children(A, c, next + off);
      next += tot;
    }
    __syncthreads();
    a = b;
    b = next;
    if (b > cap) break;  // more contexts than the arrays hold (the host falls back)
  }
  __syncthreads();
  for (uint32_t l = t; l <= L; l += nt) lev_out[l + 1] = lev[l];  // lev_out[0] = number of levels
  if (t == 0) lev_out[0] = L;
  if (t == 0) built[0] = (b > a || b > cap) ? ~0ull : b;  // ~0: level or capacity overflow (host falls back)
  if ((b > a || b > cap) && t == 0) lev_out[0] = 0;        // nothing for the fold to walk
}

// k_cct_small with its working set in shared memory (used when it fits): per external call
// site (in each caller's ascending call-instruction order) the child it creates — node, kind,
// site and the ratio w_e / W_Y (R13; frac = parent's frac * ratio, the same two roundings as
// write_children) — the number of weighted external calls of every function, and the kind /
// node / frac of the current and next BFS level (up to kSmallCap contexts each; contexts
// beyond that are read back from global memory).  Same numbering and results as k_cct_small.
constexpr uint32_t kSmallCap = 3072;
constexpr uint8_t kSkip = 0xFF;

__host__ __device__ inline size_t small2_smem(uint32_t n_func, uint32_t m) {
  return (size_t)m * 8 + (size_t)m * 4 * 2 + 2ull * kSmallCap * 8 + 2ull * kSmallCap * 4 + (size_t)n_func * 2 +
         (size_t)m + 2ull * kSmallCap + 64;
}

__global__ void __launch_bounds__(1024) k_cct_small2(LevelArgs A, uint32_t n_func, uint32_t m, uint32_t n_dag,
                                                     const uint32_t *din_ptr, const uint8_t *dact, uint32_t *lev_out,
                                                     unsigned long long *built, uint32_t stage, uint32_t par,
                                                     uint64_t cap) {
  extern __shared__ __align__(16) uint8_t sm2[];
  __shared__ uint32_t lev[kSmallLevels + 1];
  double *eratio = reinterpret_cast<double *>(sm2);
  double *cfrac = eratio + m, *nfrac = cfrac + kSmallCap;
  uint32_t *enode = reinterpret_cast<uint32_t *>(nfrac + kSmallCap);
  uint32_t *esite = enode + m;
  uint32_t *cnode = esite + m, *nnode = cnode + kSmallCap;
  uint16_t *nzc = reinterpret_cast<uint16_t *>(nnode + kSmallCap);
  uint8_t *ekind = reinterpret_cast<uint8_t *>(nzc + n_func);
  uint8_t *ckind = ekind + m, *nkind = ckind + kSmallCap;
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  // stage = 1: the static tables every level reads (DAG members, external calls per function)
  // are copied to shared memory once, so a level costs shared-memory latency only
  const uint32_t *dmem_ptr = A.dmem_ptr, *dmem = A.dmem, *fout_ptr = A.fout_ptr;
  if (stage) {
    uint32_t *sp = reinterpret_cast<uint32_t *>(sm2 + ((small2_smem(n_func, m) + 15) & ~(size_t)15));
    uint32_t *sdp = sp, *sdm = sdp + n_dag + 1, *sfp = sdm + n_func;
    for (uint32_t x = t; x <= n_dag; x += nt) sdp[x] = A.dmem_ptr[x];
    for (uint32_t x = t; x < n_func; x += nt) sdm[x] = A.dmem[x];
    for (uint32_t x = t; x <= n_func; x += nt) sfp[x] = A.fout_ptr[x];
    dmem_ptr = sdp;
    dmem = sdm;
    fout_ptr = sfp;
    __syncthreads();
  }
  for (uint32_t q = t; q < m; q += nt) {  // the child each weighted external call creates
    const uint32_t e = A.fout_e[q];
    const uint64_t we = A.w[e];
    const uint32_t Y = A.scc_of[A.callee[e]];
    esite[q] = e;
    enode[q] = Y;
    ekind[q] = we ? (A.nontriv[Y] ? GPA_CTX_SCC : GPA_CTX_FUNC) : kSkip;
    eratio[q] = we ? __ddiv_rn(__ull2double_rn(we), __ull2double_rn(A.W[Y])) : 0.0;  // R13
  }
  __syncthreads();
  for (uint32_t g = t; g < n_func; g += nt) {
    uint32_t c = 0;
    for (uint32_t q = fout_ptr[g]; q < fout_ptr[g + 1]; q++) c += ekind[q] != kSkip;
    nzc[g] = (uint16_t)c;
  }
  // par = 1: children are written thread-per-child (a level's contexts keep their first child's
  // index in loff; a child finds its parent by binary search and its call site in wq, the
  // weighted external calls of every function compacted in call-instruction order from wptr)
  uint32_t *wptr = nullptr, *wq = nullptr, *loff = nullptr;
  if (par) {
    uint32_t *pp = reinterpret_cast<uint32_t *>(sm2 + par);
    wptr = pp;
    wq = wptr + n_func + 1;
    loff = wq + m;
    __syncthreads();
    uint32_t run = 0;
    for (uint32_t base = 0; base < n_func; base += nt) {
      const uint32_t g = base + t;
      uint32_t tot;
      const uint32_t o = run + block_exscan(g < n_func ? (uint32_t)nzc[g] : 0u, &tot);
      if (g < n_func) wptr[g] = o;
      run += tot;
    }
    if (t == 0) wptr[n_func] = run;
    __syncthreads();
    for (uint32_t g = t; g < n_func; g += nt) {
      uint32_t k = wptr[g];
      for (uint32_t q = fout_ptr[g]; q < fout_ptr[g + 1]; q++)
        if (ekind[q] != kSkip) wq[k++] = q;
    }
  }
  uint32_t running = 0;
  for (uint32_t base = 0; base < n_dag; base += nt) {  // roots in DAG order (R15)
    uint32_t X = base + t;
    uint32_t flag = X < n_dag && din_ptr[X] == din_ptr[X + 1] && dact[X];
    uint32_t tot;
    uint32_t pos = running + block_exscan(flag, &tot);
    if (flag && pos < cap) {
      const uint8_t k = A.nontriv[X] ? GPA_CTX_SCC : GPA_CTX_FUNC;
      A.parent[pos] = NONE;
      A.site[pos] = NONE;
      A.node[pos] = X;
      A.kind[pos] = k;
      A.frac[pos] = 1.0;
      if (pos < kSmallCap) {
        ckind[pos] = k;
        cnode[pos] = X;
        cfrac[pos] = 1.0;
      }
    }
    running += tot;
  }
  __syncthreads();
  uint32_t a = 0, b = running, L = 0;
  if (t == 0) lev[0] = 0;
  bool over = b > cap;  // more contexts than the arrays hold: stop, the host falls back
  while (!over && b > a && L < kSmallLevels) {
    if (t == 0) lev[L + 1] = b;
    L++;
    uint32_t next = b;
    if (par && b - a <= kSmallCap) {
      // phase A: child counts -> offsets (BFS numbering, R17) per context of the level
      for (uint32_t base = a; base < b; base += nt) {
        const uint32_t c = base + t;
        uint32_t cnt = 0;
        if (c < b) {
          const uint8_t k = ckind[c - a];
          const uint32_t nd = cnode[c - a];
          cnt = k == GPA_CTX_SCC ? dmem_ptr[nd + 1] - dmem_ptr[nd]
                                 : (uint32_t)nzc[k == GPA_CTX_SCC_MEMBER ? nd : dmem[dmem_ptr[nd]]];
        }
        uint32_t tot;
        const uint32_t o = next + block_exscan(cnt, &tot);
        if (c < b) {
          loff[c - a] = o;
          A.first_child[c] = o;
          A.n_children[c] = cnt;
        }
        next += tot;
      }
      __syncthreads();
      if (next > cap) {
        over = true;
        break;
      }
      // phase B: one thread per child
      const uint32_t w = b - a;
      for (uint32_t d = b + t; d < next; d += nt) {
        uint32_t lo = 0, hi = w;  // last context i with loff[i] <= d
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (loff[mid] <= d) lo = mid + 1; else hi = mid;
        }
        const uint32_t i = lo - 1, c = a + i, j = d - loff[i];
        const uint8_t k = ckind[i];
        const uint32_t nd = cnode[i];
        const double f = cfrac[i];
        uint8_t ck;
        uint32_t cn;
        double cf;
        A.parent[d] = c;
        if (k == GPA_CTX_SCC) {  // members in ascending function id (R14)
          ck = GPA_CTX_SCC_MEMBER;
          cn = dmem[dmem_ptr[nd] + j];
          cf = f;
          A.site[d] = NONE;
        } else {  // the j-th weighted external call in call-instruction order (R15, R17)
          const uint32_t g = k == GPA_CTX_SCC_MEMBER ? nd : dmem[dmem_ptr[nd]];
          const uint32_t q = wq[wptr[g] + j];
          ck = ekind[q];
          cn = enode[q];
          cf = __dmul_rn(f, eratio[q]);
          A.site[d] = esite[q];
        }
        A.node[d] = cn;
        A.kind[d] = ck;
        A.frac[d] = cf;
        if (d - b < kSmallCap) {
          nkind[d - b] = ck;
          nnode[d - b] = cn;
          nfrac[d - b] = cf;
        }
      }
    } else
    for (uint32_t base = a; base < b; base += nt) {
      const uint32_t c = base + t;
      uint8_t k = 0;
      uint32_t nd = 0, cnt = 0, g = 0;
      double f = 0.0;
      if (c < b) {
        if (c - a < kSmallCap) {
          k = ckind[c - a];
          nd = cnode[c - a];
          f = cfrac[c - a];
        } else {
          k = A.kind[c];
          nd = A.node[c];
          f = A.frac[c];
        }
        if (k == GPA_CTX_SCC) {
          cnt = dmem_ptr[nd + 1] - dmem_ptr[nd];
        } else {
          g = k == GPA_CTX_SCC_MEMBER ? nd : dmem[dmem_ptr[nd]];
          cnt = nzc[g];
        }
      }
      uint32_t tot;
      const uint32_t o = next + block_exscan(cnt, &tot);
      if (c < b && o + cnt <= cap) {
        if (k == GPA_CTX_SCC) {  // members in ascending function id (R14)
          uint32_t d = o;
          for (uint32_t q = dmem_ptr[nd]; q < dmem_ptr[nd + 1]; q++, d++) {
            const uint32_t mf = dmem[q];
            A.parent[d] = c;
            A.site[d] = NONE;
            A.node[d] = mf;
            A.kind[d] = GPA_CTX_SCC_MEMBER;
            A.frac[d] = f;
            if (d - b < kSmallCap) {
              nkind[d - b] = GPA_CTX_SCC_MEMBER;
              nnode[d - b] = mf;
              nfrac[d - b] = f;
            }
          }
        } else {  // weighted external calls, ascending call instruction (R15, R17)
          uint32_t d = o;
          for (uint32_t q = fout_ptr[g]; q < fout_ptr[g + 1]; q++) {
            const uint8_t ek = ekind[q];
            if (ek == kSkip) continue;
            const double fr = __dmul_rn(f, eratio[q]);
            A.parent[d] = c;
            A.site[d] = esite[q];
            A.node[d] = enode[q];
            A.kind[d] = ek;
            A.frac[d] = fr;
            if (d - b < kSmallCap) {
              nkind[d - b] = ek;
              nnode[d - b] = enode[q];
              nfrac[d - b] = fr;
            }
            d++;
          }
        }
        A.first_child[c] = o;
        A.n_children[c] = cnt;
      }
      next += tot;
    }
    __syncthreads();
    {  // the next level becomes the current one
      uint8_t *tk = ckind; ckind = nkind; nkind = tk;
      uint32_t *tn = cnode; cnode = nnode; nnode = tn;
      double *tf = cfrac; cfrac = nfrac; nfrac = tf;
    }
    a = b;
    b = next;
    over = over || b > cap;
  }
  __syncthreads();
  for (uint32_t l = t; l <= L; l += nt) lev_out[l + 1] = lev[l];  // lev_out[0] = number of levels
  if (t == 0) lev_out[0] = over ? 0 : L;                            // overflow: nothing to fold
  if (t == 0) built[0] = (over || b > a) ? ~0ull : b;  // ~0: level or capacity overflow (host falls back)
}

// Exact counts from instrumentation: block b's execution count goes to slot 0 of
// every instruction of the block.  One thread per block; blocks are short and disjoint.
__global__ void k_block_counts(uint32_t n_blocks, const uint32_t *__restrict__ start, const uint64_t *__restrict__ cnt,
                               uint32_t n_inst, unsigned long long *__restrict__ H) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < n_blocks; b += gridDim.x * blockDim.x) {
    uint32_t lo = start[b], hi = min(start[b + 1], n_inst);
    unsigned long long c = cnt[b];
    if (c)
      for (uint32_t i = lo; i < hi; i++) atomicAdd(H + ((uint64_t)i << 4), c);
  }
}

// Step 4 for large trees in ONE cooperative launch: the grid walks the BFS levels itself,
// separated by grid-wide barriers (no host round trip per level).  Per level [a, b):
//   A  block i counts the children of its contiguous chunk and scans them locally
//   B  block 0 scans the per-block totals -> the next level's size
//   C  every block writes its chunk's children at b + block offset + local offset
// then excl for every context, then incl level by level from the deepest.
// Dataflow incl fold (no level barriers).  The excl pass computes excl for every (context, slot)
// and zeroes the context's arrival counter; then the 16 lanes (slots) of each leaf context store
// incl = excl and climb: after their stores they count their context in at the parent (fence +
// one atomic per context); the child that arrives last (count == the parent's n_children)
// computes the parent's incl = excl + the children's incl in index order -- the same fp64
// operations in the same order as the level fold and the oracle, so the result is bit-identical --
// and climbs on.  No thread ever waits for another, so there is no deadlock; the critical path is
// one store-fence-atomic-load round trip per tree level instead of a barrier plus the level's loads.
// Threads x = 16 c + r: the 16 lanes of a half-warp hold one context (blockDim and strides are
// multiples of 16).
__device__ __forceinline__ double excl_of(const LevelArgs &A, const uint64_t *__restrict__ S_f, uint64_t c, int r) {
  const uint8_t k = A.kind[c];
  if (k == GPA_CTX_SCC) return 0.0;  // excl (R14)
  const uint32_t g = k == GPA_CTX_SCC_MEMBER ? A.node[c] : A.dmem[A.dmem_ptr[A.node[c]]];
  return __dmul_rn(A.frac[c], __ull2double_rn(S_f[(uint64_t)g * GPA_SLOTS + r]));
}

// climb from context c (lane r of its half-warp) with incl(c) = v; returns when this half-warp is
// not the last arrival at an ancestor, or after storing a root's incl
__device__ __forceinline__ void fold_climb(const LevelArgs &A, const double *__restrict__ excl, double *incl,
                                           uint32_t *arrived, uint32_t c, uint32_t r, double v) {
  const unsigned hmask = 0xFFFFu << (threadIdx.x & 16);
  for (;;) {
    const uint32_t p = A.parent[c];
    uint32_t nc = 0, d0 = 0;
    if (p != NONE) {
      nc = A.n_children[p];
      d0 = A.first_child[p];
    }
    __stcg(incl + (uint64_t)c * GPA_SLOTS + r, v);
    if (p == NONE) return;
    if (nc == 1) {  // an only child is trivially the last arrival: no fence, no counter (recursion chains)
      v = __dadd_rn(__ldcg(excl + (uint64_t)p * GPA_SLOTS + r), v);
      c = p;
      continue;
    }
    // release: this lane's incl is visible device-wide before the context is counted in (acq_rel,
    // not __threadfence: that is fence.sc plus an L1 invalidation; every load here goes to L2)
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    __syncwarp(hmask);
    uint32_t last = 0;
    if (r == 0) last = atomicAdd(arrived + p, 1u) + 1u == nc;
    last = __shfl_sync(hmask, last, 0, 16);
    if (!last) return;
    asm volatile("fence.acq_rel.gpu;" ::: "memory");  // acquire: every sibling's incl is visible
    v = __ldcg(excl + (uint64_t)p * GPA_SLOTS + r);
    const double *ci = incl + (uint64_t)d0 * GPA_SLOTS + r;
    uint32_t d = 0;
    for (; d + 4 <= nc; d += 4) {  // four loads in flight, added in index order
      const double a0 = __ldcg(ci + (uint64_t)d * GPA_SLOTS), a1 = __ldcg(ci + (uint64_t)(d + 1) * GPA_SLOTS);
      const double a2 = __ldcg(ci + (uint64_t)(d + 2) * GPA_SLOTS), a3 = __ldcg(ci + (uint64_t)(d + 3) * GPA_SLOTS);
      v = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(v, a0), a1), a2), a3);
    }
    for (; d < nc; d++) v = __dadd_rn(v, __ldcg(ci + (uint64_t)d * GPA_SLOTS));
    c = p;
  }
}

namespace cg = cooperative_groups;
constexpr int kCoopThreads = 512;

__global__ void __launch_bounds__(kCoopThreads) k_cct_coop(LevelArgs A, uint32_t n_dag, const uint32_t *din_ptr,
                                                          const uint8_t *dact, const uint64_t *S_f, uint64_t n_total,
                                                          double *excl, double *incl, uint32_t *tmp, uint32_t *bsum,
                                                          uint32_t *lev, uint32_t max_lev,
                                                          unsigned long long *built) {
  cg::grid_group grid = cg::this_grid();
  const uint32_t t = threadIdx.x, nt = blockDim.x, B = gridDim.x, bi = blockIdx.x;
  __shared__ uint32_t s_off;
  if (bi == 0) {  // roots in DAG order (R15)
    uint32_t running = 0;
    for (uint32_t base = 0; base < n_dag; base += nt) {
      uint32_t X = base + t;
      uint32_t flag = X < n_dag && din_ptr[X] == din_ptr[X + 1] && dact[X];
      uint32_t tot;
      uint32_t pos = running + block_exscan(flag, &tot);
      if (flag) {
        A.parent[pos] = NONE;
        A.site[pos] = NONE;
        A.node[pos] = X;
        A.kind[pos] = A.nontriv[X] ? GPA_CTX_SCC : GPA_CTX_FUNC;
        A.frac[pos] = 1.0;
      }
      running += tot;
    }
    if (t == 0) {
      lev[0] = 0;
      lev[1] = running;
    }
  }
  grid.sync();
  uint32_t L = 0;
  for (; L < max_lev; L++) {
    const uint32_t a = lev[L], b = lev[L + 1];
    if (b == a) break;
    const uint32_t m = b - a, chunk = (m + B - 1) / B;
    const uint32_t c0 = a + min(m, bi * chunk), c1 = a + min(m, (bi + 1) * chunk);
    uint32_t run = 0;  // A: local counts + scan
    for (uint32_t base = c0; base < c1; base += nt) {
      uint32_t c = base + t;
      uint32_t cnt = c < c1 ? child_count(A, c) : 0;
      uint32_t tot;
      uint32_t off = block_exscan(cnt, &tot);
      if (c < c1) tmp[c - a] = run + off;
      run += tot;
    }
    if (t == 0) bsum[bi] = run;
    grid.sync();
    {  // B: every block sums the totals of the blocks before it (block 0 also the level size),
       // instead of block 0 scanning them behind one more grid barrier
      uint32_t v = 0, vall = 0, tot, tot2;
      for (uint32_t i = t; i < B; i += nt) {
        const uint32_t x = __ldcg(bsum + i);
        if (i < bi) v += x;
        vall += x;
      }
      block_exscan(v, &tot);
      block_exscan(vall, &tot2);
      if (t == 0) {
        s_off = tot;
        if (bi == 0) lev[L + 2] = b + tot2;
      }
    }
    __syncthreads();  // C: write the children
    for (uint32_t c = c0 + t; c < c1; c += nt) write_children(A, c, (uint64_t)b + s_off + tmp[c - a]);
    grid.sync();
  }
  const uint64_t gt = (uint64_t)bi * nt + t, gs = (uint64_t)B * nt;
  for (uint64_t x = gt; x < n_total * GPA_SLOTS; x += gs) excl[x] = excl_of(A, S_f, x >> 4, (int)(x & 15));
  grid.sync();
  // incl: deepest level first, children in order.  (The dataflow fold of the small trees, fold_climb,
  // measured 4.4x slower here: with millions of contexts each thread walks hundreds of leaves, and
  // every climb step is a serial store-fence-atomic round trip, while a level pass is bandwidth-bound.)
  for (int l = (int)L - 1; l >= 0; l--) {
    for (uint64_t x = (uint64_t)lev[l] * GPA_SLOTS + gt; x < (uint64_t)lev[l + 1] * GPA_SLOTS; x += gs) {
      uint64_t c = x >> 4;
      int r = (int)(x & 15);
      double v = excl[x];
      uint32_t d0 = A.first_child[c], nc = A.n_children[c];
      for (uint32_t d = d0; d < d0 + nc; d++) v = __dadd_rn(v, incl[(uint64_t)d * GPA_SLOTS + r]);
      incl[x] = v;
    }
    grid.sync();
  }
  if (bi == 0 && t == 0) built[0] = L < max_lev ? lev[L] : ~0ull;
}

// excl for every context, then incl level by level (deepest first), over the whole grid with
// grid-wide barriers; the level boundaries come from k_cct_small (lev[0] = levels,
// lev[1 + l] = first context of level l).
__global__ void __launch_bounds__(512) k_cct_fold(LevelArgs A, const uint32_t *__restrict__ lev,
                                                 const uint64_t *__restrict__ S_f, double *excl, double *incl) {
  cg::grid_group grid = cg::this_grid();
  const uint32_t L = lev[0];
  const uint64_t n = lev[1 + L];
  const uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, gs = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t x = gt; x < n * GPA_SLOTS; x += gs) {  // excl (R14)
    uint64_t c = x >> 4;
    int r = (int)(x & 15);
    uint8_t k = A.kind[c];
    double v = 0.0;
    if (k != GPA_CTX_SCC) {
      uint32_t g = k == GPA_CTX_SCC_MEMBER ? A.node[c] : A.dmem[A.dmem_ptr[A.node[c]]];
      v = __dmul_rn(A.frac[c], __ull2double_rn(S_f[(uint64_t)g * GPA_SLOTS + r]));
    }
    excl[x] = v;
  }
  grid.sync();
  for (int l = (int)L - 1; l >= 0; l--) {  // incl: children in index order
    for (uint64_t x = (uint64_t)lev[1 + l] * GPA_SLOTS + gt; x < (uint64_t)lev[2 + l] * GPA_SLOTS; x += gs) {
      uint64_t c = x >> 4;
      int r = (int)(x & 15);
      double v = excl[x];
      uint32_t d0 = A.first_child[c], nc = A.n_children[c];
      for (uint32_t d = d0; d < d0 + nc; d++) v = __dadd_rn(v, incl[(uint64_t)d * GPA_SLOTS + r]);
      incl[x] = v;
    }
    grid.sync();
  }
}

// The same excl + level-by-level incl fold on ONE thread-block cluster (8-16 SMs) with hardware
// cluster barriers between levels instead of grid-wide barriers: small trees have tens of
// levels with little work each, so the barrier latency dominates.  Values written by other
// CTAs of the cluster are read through L2 (ld.cg) after the barrier's release/acquire.
__global__ void __launch_bounds__(1024) k_cct_fold_cl(LevelArgs A, const uint32_t *__restrict__ lev,
                                                    const uint64_t *__restrict__ S_f, double *excl, double *incl) {
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t L = lev[0];
  const uint64_t n = lev[1 + L];
  const uint64_t gt = (uint64_t)cl.block_rank() * blockDim.x + threadIdx.x, gs = (uint64_t)cl.num_blocks() * blockDim.x;
  for (uint64_t x = gt; x < n * GPA_SLOTS; x += gs) {  // excl (R14)
    uint64_t c = x >> 4;
    int r = (int)(x & 15);
    uint8_t k = A.kind[c];
    double v = 0.0;
    if (k != GPA_CTX_SCC) {
      uint32_t g = k == GPA_CTX_SCC_MEMBER ? A.node[c] : A.dmem[A.dmem_ptr[A.node[c]]];
      v = __dmul_rn(A.frac[c], __ull2double_rn(S_f[(uint64_t)g * GPA_SLOTS + r]));
    }
    excl[x] = v;
  }
  cl.sync();
  for (int l = (int)L - 1; l >= 0; l--) {  // incl: children in index order
    for (uint64_t x = (uint64_t)lev[1 + l] * GPA_SLOTS + gt; x < (uint64_t)lev[2 + l] * GPA_SLOTS; x += gs) {
      uint64_t c = x >> 4;
      int r = (int)(x & 15);
      double v = __ldcg(excl + x);
      uint32_t d0 = A.first_child[c], nc = A.n_children[c];
      for (uint32_t d = d0; d < d0 + nc; d++) v = __dadd_rn(v, __ldcg(incl + (uint64_t)d * GPA_SLOTS + r));
      incl[x] = v;
    }
    cl.sync();
  }
}

__global__ void k_cct_excl_lev(LevelArgs A, const uint32_t *__restrict__ lev, const uint64_t *__restrict__ S_f,
                               double *__restrict__ excl, uint32_t *__restrict__ arrived) {
  const uint64_t n = lev[1 + lev[0]];
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n * GPA_SLOTS; x += (uint64_t)gridDim.x * blockDim.x) {
    excl[x] = excl_of(A, S_f, x >> 4, (int)(x & 15));
    if ((x & 15) == 0) arrived[x >> 4] = 0;
  }
}

__global__ void k_cct_fold_up(LevelArgs A, const uint32_t *__restrict__ lev, const double *__restrict__ excl,
                              double *incl, uint32_t *arrived) {
  const uint64_t n = lev[1 + lev[0]];
  const uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= n * GPA_SLOTS) return;
  const uint32_t c = (uint32_t)(x >> 4);
  if (A.n_children[c] != 0) return;
  fold_climb(A, excl, incl, arrived, c, (uint32_t)(x & 15), excl[x]);
}

unsigned grid_for(uint64_t work, unsigned threads) {
  uint64_t b = (work + threads - 1) / threads;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b ? b : 1);
}

LevelArgs level_args(const gpa_structure_s *s, gpa_cct_s *c) {
  LevelArgs A;
  A.fout_ptr = s->d_fout_ptr; A.fout_e = s->d_fout_e; A.callee = s->d_call_callee; A.scc_of = s->d_scc_of;
  A.dmem_ptr = s->d_dmem_ptr; A.dmem = s->d_dmem; A.nontriv = s->d_dag_nontrivial;
  A.w = c->w; A.W = c->W;
  A.parent = c->parent; A.site = c->site; A.node = c->node; A.first_child = c->first_child;
  A.n_children = c->n_children; A.kind = c->kind; A.frac = c->frac;
  return A;
}

}  // namespace

cudaError_t launch_cct_prof_excl(const gpa_structure_s *s, const gpa_cct_s *c, const uint64_t *d_ph, uint32_t P1,
                                 double *d_excl, cudaStream_t st) {
  k_cct_prof_excl<<<grid_for(c->n * GPA_SLOTS * P1, 256), 256, 0, st>>>(
      c->n, P1, s->info.n_func, c->kind, c->node, c->frac, s->d_dmem_ptr, s->d_dmem, d_ph, d_excl);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_cct_prof_incl_level(const gpa_cct_s *c, uint64_t a, uint64_t b, uint32_t P1, const double *d_excl,
                                       double *d_incl, cudaStream_t st) {
  if (b <= a) return cudaSuccess;
  k_cct_prof_incl_level<<<grid_for((b - a) * GPA_SLOTS * P1, 256), 256, 0, st>>>(c->n, a, b, P1, c->first_child,
                                                                                  c->n_children, d_excl, d_incl);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_cct_weights_range(const gpa_structure_s *s, const uint64_t *d_hist, uint32_t lo, uint32_t hi,
                                     uint64_t *d_w, cudaStream_t st) {
  uint32_t n = s->info.n_call;
  if (!n || lo >= hi) return cudaSuccess;
  k_weights<<<grid_for(n, 256), 256, 0, st>>>(s->d_call_inst, n, d_hist, d_w, lo, hi);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_cct_weights(const gpa_structure_s *s, const uint64_t *d_hist, uint64_t *d_w, cudaStream_t st) {
  uint32_t n = s->info.n_call;
  if (!n) return cudaSuccess;
  k_weights<<<grid_for(n, 256), 256, 0, st>>>(s->d_call_inst, n, d_hist, d_w);
  count_launches(1);
  return cudaGetLastError();
}

constexpr size_t kPropSmem = 200 * 1024;

cudaError_t launch_cct_propagate(const gpa_structure_s *s, const uint64_t *d_S_f, uint64_t *d_w,
                                 uint8_t *d_func_active, uint8_t *d_dag_active, uint64_t *d_W,
                                 unsigned long long *d_count, bool exact, bool count, cudaStream_t st,
                                 uint32_t n_batch, uint64_t fstride, uint64_t dstride) {
  static_assert(sizeof(unsigned long long) == sizeof(uint64_t), "u64");
  if (n_batch && count) return cudaErrorInvalidValue;  // the path count is a single-problem output
  uint64_t *paths = nullptr;
  const size_t nq = std::max<size_t>(s->info.n_func, s->info.n_dag) + 1;
  const uint64_t pstride = (s->info.n_dag + 1) + nq;  // u64 words: paths, then two u32 worklists of nq
  const uint32_t nb = n_batch ? n_batch : 1;
  cudaError_t e = pool_alloc((void **)&paths, sizeof(uint64_t) * pstride * nb, st);
  if (e != cudaSuccess) return e;
  PropArgs A;
  A.batch = n_batch ? 1u : 0u;
  A.fstride = fstride;
  A.dstride = dstride;
  A.pstride = pstride;
  A.n_func = s->info.n_func; A.n_dag = s->info.n_dag; A.n_lev = s->info.dag_levels; A.exact = exact ? 1 : 0; A.do_count = count ? 1 : 0;
  A.S_f = d_S_f; A.fin_ptr = s->d_fin_ptr; A.fin_e = s->d_fin_e; A.caller = s->d_call_caller;
  A.scc_of = s->d_scc_of; A.din_ptr = s->d_din_ptr; A.din_e = s->d_din_e; A.dmem_ptr = s->d_dmem_ptr;
  A.dmem = s->d_dmem; A.dlev_ptr = s->d_dlev_ptr; A.dlev_node = s->d_dlev_node; A.nontriv = s->d_dag_nontrivial;
  A.w = d_w; A.W = d_W; A.paths = paths; A.fact = d_func_active; A.dact = d_dag_active; A.count = d_count;
  A.n_call = s->info.n_call;
  A.q0 = reinterpret_cast<uint32_t *>(paths + s->info.n_dag + 1);
  A.q1 = A.q0 + nq;
  A.n_ext = s->n_ext_calls;
  size_t sm = 8ull * (A.n_call + A.n_dag) + A.n_func + A.n_dag + 8;
  const size_t sm_dp = 8ull * (A.n_call + A.n_dag) + ((A.n_func + A.n_dag + 7) & ~7ull) + 4ull * A.n_ext +
                       12ull * A.n_dag;
  A.stage_dp = count && sm_dp <= kPropSmem ? 1u : 0u;
  if (A.stage_dp) sm = std::max(sm, sm_dp);
  if (sm <= kPropSmem) {
    if (sm > 48 * 1024 &&
        (e = cudaFuncSetAttribute(k_propagate<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kPropSmem)) !=
            cudaSuccess)
      return e;
    k_propagate<true><<<nb, 1024, sm, st>>>(A);
  } else {
    k_propagate<false><<<nb, 1024, 0, st>>>(A);
  }
  count_launches(1);
  e = cudaGetLastError();
  cudaError_t e2 = cudaFreeAsync(paths, st);
  return e != cudaSuccess ? e : e2;
}

cudaError_t launch_cct_roots(const gpa_structure_s *s, const uint8_t *d_dag_active, gpa_cct_s *c,
                             unsigned long long *d_n, cudaStream_t st) {
  k_roots<<<1, 1024, 0, st>>>(s->info.n_dag, s->d_din_ptr, d_dag_active, s->d_dag_nontrivial, c->parent, c->site,
                              c->node, c->kind, c->frac, d_n);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_cct_level(const gpa_structure_s *s, gpa_cct_s *c, uint64_t a, uint64_t b, uint32_t *d_tmp,
                             uint32_t *d_bs, unsigned long long *d_next, cudaStream_t st) {
  LevelArgs A = level_args(s, c);
  uint64_t m = b - a;
  k_level_count<<<grid_for(m, 256), 256, 0, st>>>(A, a, b, d_tmp);
  uint64_t nb = (m + kScanTile - 1) / kScanTile;
  if (nb > 65536) return cudaErrorInvalidValue;
  k_scan_reduce<<<(unsigned)nb, kScanThreads, 0, st>>>(d_tmp, m, d_bs);
  k_scan_top<<<1, kScanThreads, 0, st>>>(d_bs, (uint32_t)nb, d_next);
  k_scan_down<<<(unsigned)nb, kScanThreads, 0, st>>>(d_tmp, m, d_bs);
  k_level_write<<<grid_for(m, 256), 256, 0, st>>>(A, a, b, d_tmp);
  count_launches(5);
  return cudaGetLastError();
}

cudaError_t launch_block_counts(uint32_t n_blocks, const uint32_t *d_start, const uint64_t *d_cnt, uint32_t n_inst,
                                uint64_t *d_hist, cudaStream_t st) {
  if (!n_blocks) return cudaSuccess;
  k_block_counts<<<grid_for(n_blocks, 256), 256, 0, st>>>(n_blocks, d_start, d_cnt, n_inst,
                                                          (unsigned long long *)d_hist);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_cct_coop(const gpa_structure_s *s, gpa_cct_s *c, uint32_t *d_tmp, uint32_t *d_bsum, uint32_t *d_lev,
                            uint32_t max_lev, unsigned long long *d_built, int sm_count, cudaStream_t st) {
  LevelArgs A = level_args(s, c);
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cct_coop, kCoopThreads, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorCooperativeLaunchTooLarge;
  unsigned blocks = (unsigned)(sm_count * (per_sm < 2 ? per_sm : 2));
  uint32_t n_dag = s->info.n_dag;
  const uint32_t *din_ptr = s->d_din_ptr;
  const uint8_t *dact = c->dag_active;
  const uint64_t *S_f = c->S_f;
  uint64_t n_total = c->n;
  double *excl = c->excl, *incl = c->incl;
  void *args[] = {&A, &n_dag, &din_ptr, &dact, &S_f, &n_total, &excl, &incl, &d_tmp, &d_bsum, &d_lev, &max_lev, &d_built};
  e = cudaLaunchCooperativeKernel((void *)k_cct_coop, dim3(blocks), dim3(kCoopThreads), args, 0, st);
  count_launches(1);
  return e;
}

cudaError_t launch_cct_small(const gpa_structure_s *s, gpa_cct_s *c, uint32_t *d_lev, unsigned long long *d_built,
                             int sm_count, cudaStream_t st) {
  LevelArgs A = level_args(s, c);
  const uint32_t m_ext = s->n_ext_calls;
  const size_t sm2 = small2_smem(s->info.n_func, m_ext);
  const size_t sm2s = ((sm2 + 15) & ~(size_t)15) + 4ull * (s->info.n_dag + 1 + 2ull * s->info.n_func + 1);
  const uint32_t stage = sm2s <= 200 * 1024 ? 1u : 0u;
  cudaError_t e = cudaSuccess;
  if (sm2 <= 200 * 1024 && s->info.n_func < 65536) {
    size_t smx = stage ? sm2s : sm2;
    // thread-per-child level writes when their tables fit as well (wptr, wq, loff)
    const size_t par_at = (smx + 15) & ~(size_t)15;
    const size_t par_bytes = 4ull * (s->info.n_func + 1 + m_ext + kSmallCap);
    const uint32_t par = par_at + par_bytes <= 227 * 1024 - 8 * 1024 ? (uint32_t)par_at : 0u;
    if (par) smx = par_at + par_bytes;
    e = cudaFuncSetAttribute(k_cct_small2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smx);
    if (e != cudaSuccess) return e;
    k_cct_small2<<<1, 1024, smx, st>>>(A, s->info.n_func, m_ext, s->info.n_dag, s->d_din_ptr, c->dag_active, d_lev,
                                       d_built, stage, par, c->n);
  } else {
    k_cct_small<<<1, 1024, 0, st>>>(A, s->info.n_dag, s->d_din_ptr, c->dag_active, d_lev, d_built, c->n);
  }
  count_launches(1);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const uint32_t *lev = d_lev;
  const uint64_t *S_f = c->S_f;
  double *excl = c->excl, *incl = c->incl;
  static const bool level_fold = getenv("GPA_CCT_LEVEL_FOLD") != nullptr;  // A/B switch: the cluster level fold
  if (!level_fold) {  // dataflow fold over every (context, slot) of the capacity c->n
    uint32_t *arrived = nullptr;
    if ((e = pool_alloc((void **)&arrived, c->n * 4, st)) != cudaSuccess) return e;
    k_cct_excl_lev<<<grid_for(c->n * GPA_SLOTS, 256), 256, 0, st>>>(A, lev, S_f, excl, arrived);
    k_cct_fold_up<<<(unsigned)((c->n * GPA_SLOTS + 255) / 256), 256, 0, st>>>(A, lev, excl, incl, arrived);
    count_launches(2);
    e = cudaGetLastError();
    cudaError_t e2 = cudaFreeAsync(arrived, st);
    return e != cudaSuccess ? e : e2;
  }
  // largest cluster the device accepts for k_cct_fold_cl (16, else 8); 0 = none (cooperative grid)
  static std::atomic<int> cluster{-1};
  int cs0 = cluster.load(std::memory_order_relaxed);
  if (cs0 < 0) {
    cs0 = cudaFuncSetAttribute(k_cct_fold_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess ? 16 : 8;
    cudaGetLastError();
  }
  for (int cs = cs0; cs >= 8; cs /= 2) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(1024);
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, k_cct_fold_cl, A, lev, S_f, excl, incl);
    if (e == cudaSuccess) {
      count_launches(1);
      cluster.store(cs, std::memory_order_relaxed);
      return cudaSuccess;
    }
    cudaGetLastError();
  }
  cluster.store(0, std::memory_order_relaxed);
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cct_fold, 512, 0);
  if (e != cudaSuccess) return e;
  unsigned blocks = (unsigned)(sm_count * (per_sm < 2 ? (per_sm < 1 ? 1 : per_sm) : 2));
  void *args[] = {&A, &lev, &S_f, &excl, &incl};
  e = cudaLaunchCooperativeKernel((void *)k_cct_fold, dim3(blocks), dim3(512), args, 0, st);
  count_launches(1);
  return e;
}

bool cct_small_ok(const gpa_structure_s *s, uint64_t n) {
  return n <= kSmallMax && 2ull * s->info.dag_levels + 2 < (uint64_t)kSmallLevels;
}

cudaError_t launch_cct_excl(const gpa_structure_s *s, gpa_cct_s *c, cudaStream_t st) {
  if (!c->n) return cudaSuccess;
  k_excl<<<grid_for(c->n * GPA_SLOTS, 256), 256, 0, st>>>(c->n, c->kind, c->node, c->frac, s->d_dmem_ptr, s->d_dmem,
                                                        c->S_f, c->excl);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_cct_incl_level(gpa_cct_s *c, uint64_t a, uint64_t b, cudaStream_t st) {
  if (b <= a) return cudaSuccess;
  k_incl_level<<<grid_for((b - a) * GPA_SLOTS, 256), 256, 0, st>>>(a, b, c->first_child, c->n_children, c->excl,
                                                                  c->incl);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace gpa
