// k_sparse.cu — f3: profile-major / CCT-major sparse cubes (§5.2
// P:797-832, Fig. sf) of the per-profile histogram cube Hp[p][c][m] (profiles x function
// rows x slots).  Each plane is a CSR-like segment: values + leaf ids, and a sparse index of
// (id, start) pairs over the non-empty inner entries, closed by a sentinel (NONE, end).
//   CMS: plane = context c, inner = metric m, leaf = profile p   ("vals, pids, midxs")
//   PMS: plane = profile p, inner = context c, leaf = metric m  ("vals, mids, cidxs")
// Like hpcprof-mpi's "exscan operations ... to find the right offsets": count the
// non-zeros of every (plane, inner) cell, exclusive-scan the counts into value offsets and the
// index entries (+1 sentinel per plane) into index offsets, then every cell writes its run.
#include <cuda_runtime.h>
#include <stdint.h>

#include "gpa_internal.cuh"
#include "kern_common.cuh"

namespace gpa {
namespace {

// cell x = (plane, inner) in plane-major order; leaf values are read with stride `ls`
struct Geo {
  uint32_t P, C, cms;
  __host__ __device__ uint64_t cells() const { return cms ? (uint64_t)C * GPA_SLOTS : (uint64_t)P * C; }
  __host__ __device__ uint32_t inner_n() const { return cms ? GPA_SLOTS : C; }
  __host__ __device__ uint32_t leaf_n() const { return cms ? P : GPA_SLOTS; }
  __device__ __forceinline__ uint64_t at(uint64_t x, uint32_t l) const {  // index into Hp
    if (cms) {
      uint64_t c = x >> 4, m = x & 15;
      return ((uint64_t)l * C + c) * GPA_SLOTS + m;
    }
    return x * GPA_SLOTS + l;  // x = p*C + c
  }
};

__global__ void k_sparse_count(Geo g, const uint64_t *__restrict__ H, uint32_t *__restrict__ nv,
                               uint32_t *__restrict__ ni) {
  const uint64_t n = g.cells();
  const uint32_t inner = g.inner_n(), leaves = g.leaf_n();
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t k = 0;
    for (uint32_t l = 0; l < leaves; l++) k += __ldg(H + g.at(x, l)) != 0;
    nv[x] = k;
    ni[x] = (k != 0) + ((x % inner) == inner - 1);  // the last cell of a plane also holds the sentinel
  }
}

__global__ void k_sparse_write(Geo g, const uint64_t *__restrict__ H, const uint32_t *__restrict__ ov,
                               const uint32_t *__restrict__ oi, const unsigned long long *__restrict__ tot,
                               uint64_t *__restrict__ plane_off, uint64_t *__restrict__ index_off,
                               uint64_t *__restrict__ vals, uint32_t *__restrict__ ids,
                               uint64_t *__restrict__ index_start, uint32_t *__restrict__ index_id) {
  const uint64_t n = g.cells();
  const uint32_t inner = g.inner_n(), leaves = g.leaf_n();
  for (uint64_t x = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; x < n; x += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t b = (uint32_t)(x % inner);
    uint64_t v = ov[x], i = oi[x];
    if (b == 0) {
      plane_off[x / inner] = v;
      index_off[x / inner] = i;
    }
    const uint64_t v0 = v;
    for (uint32_t l = 0; l < leaves; l++) {
      uint64_t h = __ldg(H + g.at(x, l));
      if (h) {
        vals[v] = h;
        ids[v] = l;
        v++;
      }
    }
    if (v > v0) {
      index_id[i] = b;
      index_start[i] = v0;
      i++;
    }
    if (b == inner - 1) {  // sentinel: end of the plane
      index_id[i] = NONE;
      index_start[i] = v;
    }
    if (x == 0) {
      plane_off[n / inner] = tot[0];
      index_off[n / inner] = tot[1];
    }
  }
}

unsigned grid(uint64_t n) {
  uint64_t b = (n + 255) / 256;
  return (unsigned)(b < 148 * 16 ? (b ? b : 1) : 148 * 16);
}

}  // namespace

cudaError_t sparse_count(const uint64_t *H, uint32_t P, uint32_t C, bool cms, uint32_t *ov, uint32_t *oi,
                         uint32_t *bs, unsigned long long *tot, cudaStream_t st) {
  Geo g{P, C, cms ? 1u : 0u};
  const uint64_t n = g.cells();
  k_sparse_count<<<grid(n), 256, 0, st>>>(g, H, ov, oi);
  count_launches(1);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  e = scan_u32(ov, n, bs, tot, st);
  if (e != cudaSuccess) return e;
  return scan_u32(oi, n, bs, tot + 1, st);
}

cudaError_t sparse_write(const uint64_t *H, uint32_t P, uint32_t C, bool cms, const uint32_t *ov, const uint32_t *oi,
                         const unsigned long long *tot, uint64_t *plane_off, uint64_t *index_off, uint64_t *vals,
                         uint32_t *ids, uint64_t *index_start, uint32_t *index_id, cudaStream_t st) {
  Geo g{P, C, cms ? 1u : 0u};
  k_sparse_write<<<grid(g.cells()), 256, 0, st>>>(g, H, ov, oi, tot, plane_off, index_off, vals, ids, index_start,
                                                  index_id);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace gpa
