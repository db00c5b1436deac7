// k_cctp.cu — f1 extension (reading R30): an approximate CCT per profile ("for each GPU kernel
// invocation"), unified by call path ("unify the tree of call paths
// from each profile into a single tree").
//
// Every profile's tree is a subtree of the tree built from the union of the profiles' Step-2
// results (an edge that carries weight in some profile, a DAG node active in some profile): a
// path of profile p starts at a root active in p and follows edges with w_p > 0, all of which the
// union tree has.  So the unified tree is the union tree restricted to the contexts present in
// at least one profile, in the union tree's breadth-first order (roots in DAG order, members by
// function id, calls by call instruction — the order every profile tree uses):
//   k_prof_call_weights   per-profile call-site weights from the records (Step 1, R10)
//   k_union_inputs        Step-1 inputs of the union tree (activity markers, edge flags)
//   k_multi_frac          per level of the union tree: presence and frac of every profile,
//                         f(child) = f(parent) * (w_p / W_p) — the per-profile tree's roundings
//   k_multi_compact       unified ids of the contexts present in some profile (after a scan)
//   k_multi_excl / k_multi_incl_level   excl = f * S_f,p (R14), incl folded in child order
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "gpa_internal.cuh"
#include "kern_common.cuh"

namespace gpa {
namespace {

// records of calls into [P+1][n_call] (profile = stream field, overflow profile P), valid slots only
template <int MODE>
__global__ void k_prof_call_weights(AttrTables T, const uint32_t *__restrict__ inst_call, const uint4 *__restrict__ rec,
                                    uint64_t n, uint32_t n_prof, uint32_t n_call, unsigned long long *__restrict__ wp) {
  // four records in flight per thread (the loads are independent; one at a time left HBM idle)
  constexpr int U = 4;
  const uint64_t G = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t k0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k0 < n; k0 += U * G) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) v[u] = k0 + u * G < n ? ld_stream(rec + k0 + u * G) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; u++) {
      const uint32_t stall = v[u].w & 0xFFFFu, prof = v[u].w >> 16;
      if (stall >= GPA_VALID_SLOTS || v[u].z == 0) continue;  // (count 0 also marks a padding lane)
      const uint32_t i = lookup<MODE>(T, ((uint64_t)v[u].y << 32) | v[u].x);
      if (i == NONE) continue;
      const uint32_t e = __ldg(inst_call + i);
      if (e == NONE) continue;
      atomicAdd(wp + (uint64_t)(prof < n_prof ? prof : n_prof) * n_call + e, (unsigned long long)v[u].z);
    }
  }
}

// union inputs: slot 0 of S = 1 for functions active in some profile or whose DAG node is (the
// guard of R12 activates a caller's DAG node without its function), w = 1 for edges with weight
// in some profile (after each profile's Step 2).  Step 2 only adds weight and activity, so the
// union tree contains every profile's tree (possibly more paths, which no profile marks present)
__global__ void k_union_inputs(uint32_t P, uint32_t n_func, uint32_t n_call, uint64_t fs, uint64_t ds,
                               const uint32_t *__restrict__ scc_of, const uint8_t *__restrict__ fact,
                               const uint8_t *__restrict__ dact, const uint64_t *__restrict__ w,
                               uint64_t *__restrict__ S_u, uint64_t *__restrict__ w_u) {
  // one warp per function / call site, its lanes striding the profiles
  const uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (t < n_func) {
    const uint32_t X = scc_of[t];
    uint32_t a = 0;
    for (uint32_t p = lane; p < P; p += 32) a |= fact[p * fs + t] | dact[p * ds + X];
    a = __any_sync(0xFFFFFFFFu, a != 0);
    if (lane < GPA_SLOTS) S_u[(uint64_t)t * GPA_SLOTS + lane] = (lane == 0 && a) ? 1ull : 0ull;
  }
  if (t < n_call) {
    bool any = false;
    for (uint32_t p = lane; p < P; p += 32) any = any || w[(uint64_t)p * n_call + t] != 0;
    any = __any_sync(0xFFFFFFFFu, any);
    if (lane == 0) w_u[t] = any ? 1ull : 0ull;
  }
}

// does any profile mark union context c present?  (all lanes of the warp, the result in all)
__device__ __forceinline__ bool warp_any_present(const uint8_t *__restrict__ pres, uint64_t c, uint32_t P) {
  uint32_t a = 0;
  for (uint32_t p = threadIdx.x & 31; p < P; p += 32) a |= pres[c * P + p];
  return __any_sync(0xFFFFFFFFu, a != 0);
}

struct MultiArgs {
  uint32_t P, n_call, n_dag;
  const uint32_t *parent, *site, *node;  // union tree
  const uint8_t *kind;
  const uint64_t *w, *W;                 // per profile after Step 2: [P][n_call], [P][n_dag]
  const uint8_t *dact;                   // [P][ds]
  uint64_t ds;
  uint8_t *pres;                         // [n][P]
  double *frac;                          // [n][P]
};

// contexts [a, b) of the union tree x profiles: presence and frac top-down
__global__ void k_multi_frac(MultiArgs A, uint64_t a, uint64_t b) {
  const uint64_t m = (b - a) * A.P;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < m; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = a + x / A.P;
    const uint32_t p = (uint32_t)(x % A.P);
    const uint32_t pc = A.parent[c];
    uint8_t pr = 0;
    double f = 0.0;
    if (pc == NONE) {  // a root: active in p (roots are the DAG nodes without external in-edges, R15)
      pr = A.dact[p * A.ds + A.node[c]];
      f = 1.0;
    } else if (A.pres[(uint64_t)pc * A.P + p]) {
      const double fp = A.frac[(uint64_t)pc * A.P + p];
      if (A.kind[c] == GPA_CTX_SCC_MEMBER) {
        pr = 1;
        f = fp;
      } else {
        const uint64_t we = A.w[(uint64_t)p * A.n_call + A.site[c]];
        if (we) {
          pr = 1;
          f = __dmul_rn(fp, __ddiv_rn(__ull2double_rn(we), __ull2double_rn(A.W[(uint64_t)p * A.n_dag + A.node[c]])));  // R13
        }
      }
    }
    A.pres[c * A.P + p] = pr;
    A.frac[c * A.P + p] = pr ? f : 0.0;
  }
}

// any-profile flag per union context (the scan input)
__global__ void k_multi_any(const uint8_t *__restrict__ pres, uint64_t n, uint32_t P, uint32_t *__restrict__ flag) {
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;  // one warp per context
  for (uint64_t c = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < n; c += nw) {
    const bool a = warp_any_present(pres, c, P);
    if ((threadIdx.x & 31) == 0) flag[c] = a ? 1u : 0u;
  }
}

struct CompactArgs {
  uint64_t n;
  uint32_t P;
  const uint32_t *parent, *site, *node, *first_child, *n_children;  // union tree
  const uint8_t *kind, *pres;
  const uint32_t *uid;        // exclusive scan of the any-flags
  const double *frac;         // [n][P]
  uint32_t *u_parent, *u_site, *u_node, *u_first_child, *u_n_children;
  uint8_t *u_kind;
  double *u_frac;             // [n_u][P]
};

__global__ void k_multi_compact(CompactArgs A) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;  // one warp per context
  for (uint64_t c = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < A.n; c += nw) {
    if (!warp_any_present(A.pres, c, A.P)) continue;
    const uint32_t u = A.uid[c];
    if (lane == 0) {
      const uint32_t pc = A.parent[c];
      A.u_parent[u] = pc == NONE ? NONE : A.uid[pc];
      A.u_site[u] = A.site[c];
      A.u_node[u] = A.node[c];
      A.u_kind[u] = A.kind[c];
    }
    for (uint32_t p = lane; p < A.P; p += 32) A.u_frac[(uint64_t)u * A.P + p] = A.frac[c * A.P + p];
    // present children are a contiguous run of unified ids: the first present child of c
    const uint32_t d0 = A.first_child[c], nc = A.n_children[c];
    uint32_t cnt = 0, first = NONE;
    for (uint32_t d = d0; d < d0 + nc; d++) {
      if (warp_any_present(A.pres, d, A.P)) {
        if (first == NONE) first = A.uid[d];
        cnt++;
      }
    }
    if (lane == 0) {
      A.u_first_child[u] = first == NONE ? 0u : first;
      A.u_n_children[u] = cnt;
    }
  }
}

// excl[u][p][r] = frac * S_f,p[g][r] for FUNC / SCC_MEMBER contexts (0 for SCC contexts, R14)
__global__ void k_multi_excl(uint64_t n_u, uint32_t P, uint32_t n_func, const uint8_t *__restrict__ kind,
                             const uint32_t *__restrict__ node, const uint32_t *__restrict__ dmem_ptr,
                             const uint32_t *__restrict__ dmem, const double *__restrict__ frac,
                             const uint64_t *__restrict__ Sp, double *__restrict__ excl) {
  const uint64_t m = n_u * P * GPA_SLOTS;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < m; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t up = x >> 4;            // (u, p)
    const uint64_t u = up / P;
    const uint32_t p = (uint32_t)(up % P), r = (uint32_t)(x & 15);
    const uint8_t k = kind[u];
    double v = 0.0;
    const double f = frac[up];
    if (k != GPA_CTX_SCC && f != 0.0) {
      const uint32_t g = k == GPA_CTX_SCC_MEMBER ? node[u] : dmem[dmem_ptr[node[u]]];
      v = __dmul_rn(f, __ull2double_rn(Sp[((uint64_t)p * n_func + g) * GPA_SLOTS + r]));
    }
    excl[x] = v;
  }
}

// unified contexts [a, b): incl = excl + children's incl in child order (absent children are 0)
__global__ void k_multi_incl_level(uint64_t a, uint64_t b, uint32_t P, const uint32_t *__restrict__ first_child,
                                   const uint32_t *__restrict__ n_children, const double *__restrict__ excl,
                                   double *__restrict__ incl) {
  const uint64_t m = (b - a) * P * GPA_SLOTS;
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < m; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t y = a * P * GPA_SLOTS + x;
    const uint64_t u = y / ((uint64_t)P * GPA_SLOTS);
    const uint64_t rest = y - u * P * GPA_SLOTS;  // p * 16 + r
    double v = excl[y];
    const uint32_t d0 = first_child[u], nc = n_children[u];
    for (uint32_t d = d0; d < d0 + nc; d++) v = __dadd_rn(v, incl[(uint64_t)d * P * GPA_SLOTS + rest]);
    incl[y] = v;
  }
}

unsigned grid_of(uint64_t work) {
  uint64_t b = (work + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b ? b : 1);
}

}  // namespace

cudaError_t launch_prof_call_weights(const AttrTables &T, const uint32_t *inst_call, const gpa_sample *d_samples,
                                     uint64_t n, uint32_t n_prof, uint32_t n_call, unsigned long long *wp,
                                     int sm_count, cudaStream_t st) {
  if (n == 0 || n_call == 0) return cudaSuccess;
  const uint4 *rec = reinterpret_cast<const uint4 *>(d_samples);
  const unsigned blocks = (unsigned)std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count * 8);
  if (T.mode == 0) k_prof_call_weights<0><<<blocks, 256, 0, st>>>(T, inst_call, rec, n, n_prof, n_call, wp);
  else k_prof_call_weights<1><<<blocks, 256, 0, st>>>(T, inst_call, rec, n, n_prof, n_call, wp);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_union_inputs(const gpa_structure_s *s, uint32_t P, const uint8_t *fact, uint64_t fs,
                                const uint8_t *dact, uint64_t ds, const uint64_t *w, uint64_t *S_u, uint64_t *w_u,
                                cudaStream_t st) {
  const uint32_t n_func = s->info.n_func, n_call = s->info.n_call;
  const uint32_t m = n_func > n_call ? n_func : n_call;
  if (m == 0) return cudaSuccess;
  k_union_inputs<<<(unsigned)(((uint64_t)m * 32 + 255) / 256), 256, 0, st>>>(P, n_func, n_call, fs, ds, s->d_scc_of, fact,
                                                                           dact, w, S_u, w_u);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_multi_tree(const gpa_structure_s *s, const gpa_cct_s *sup, uint32_t P, const uint64_t *Sp,
                              const uint64_t *w, const uint64_t *W, const uint8_t *dact, uint64_t ds, uint8_t *pres,
                              double *frac,
                              uint32_t *flag, uint32_t *scan_scratch, unsigned long long *d_total, cudaStream_t st) {
  MultiArgs A{P, s->info.n_call, s->info.n_dag, sup->parent, sup->site, sup->node, sup->kind, w, W, dact, ds, pres, frac};
  for (size_t L = 0; L + 1 < sup->level_start.size(); L++) {
    const uint64_t a = sup->level_start[L], b = sup->level_start[L + 1];
    if (b > a) {
      k_multi_frac<<<grid_of((b - a) * P), 256, 0, st>>>(A, a, b);
      count_launches(1);
    }
  }
  k_multi_any<<<grid_of(sup->n * 32), 256, 0, st>>>(pres, sup->n, P, flag);
  count_launches(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return scan_u32(flag, sup->n, scan_scratch, d_total, st);
}

cudaError_t launch_multi_compact(const gpa_cct_s *sup, uint32_t P, const uint8_t *pres, const uint32_t *uid,
                                 const double *frac, gpa_cct_multi_s *m, cudaStream_t st) {
  CompactArgs A{sup->n, P, sup->parent, sup->site, sup->node, sup->first_child, sup->n_children, sup->kind, pres, uid,
                frac, m->parent, m->site, m->node, m->first_child, m->n_children, m->kind, m->frac};
  k_multi_compact<<<grid_of(sup->n * 32), 256, 0, st>>>(A);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_multi_values(const gpa_structure_s *s, gpa_cct_multi_s *m, const uint64_t *Sp, cudaStream_t st) {
  if (m->n == 0) return cudaSuccess;
  const uint32_t P = m->n_profiles;
  k_multi_excl<<<grid_of(m->n * P * GPA_SLOTS), 256, 0, st>>>(m->n, P, s->info.n_func, m->kind, m->node, s->d_dmem_ptr,
                                                              s->d_dmem, m->frac, Sp, m->excl);
  count_launches(1);
  for (size_t L = m->level_start.size() - 1; L-- > 0;) {
    const uint64_t a = m->level_start[L], b = m->level_start[L + 1];
    if (b > a) {
      k_multi_incl_level<<<grid_of((b - a) * P * GPA_SLOTS), 256, 0, st>>>(a, b, P, m->first_child, m->n_children,
                                                                         m->excl, m->incl);
      count_launches(1);
    }
  }
  return cudaGetLastError();
}

}  // namespace gpa
