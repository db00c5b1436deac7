// gpa_host.cu — the C ABI of libgpa (include/gpa.h): argument checking, structure
// validation and load-time table construction (pc->instruction granule map, roll-up CSR,
// call-graph CSR, Tarjan SCC condensation, DAG levels), and the host orchestration of the
// kernels in k_attr.cu / k_rollup.cu / k_cct.cu.
//
// Paper: Zhou et al., arXiv 2109.06931.  Citations: P:<line>.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <chrono>
#include <vector>

#include "gpa.h"
#include "gpa_internal.cuh"

using namespace gpa;

static thread_local std::string g_err;
static std::atomic<unsigned long long> g_launches{0};

void gpa::count_launches(uint64_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

static std::mutex g_pool_mu;
static cudaMemPool_t g_pools[64] = {};

// bytes the library's memory pool keeps reserved (environment GPA_POOL_KEEP_BYTES, default 8 GiB)
static uint64_t pool_keep() {
  static const uint64_t keep = [] {
    const char *e = getenv("GPA_POOL_KEEP_BYTES");
    return e ? strtoull(e, nullptr, 10) : (8ull << 30);
  }();
  return keep;
}

// return reserved pool memory above the release threshold to the driver (after large frees)
static void pool_trim(int dev) {
  static const bool off = getenv("GPA_POOL_NO_TRIM") != nullptr;  // (diagnostics)
  if (off) return;
  std::lock_guard<std::mutex> lock(g_pool_mu);
  if (dev >= 0 && dev < 64 && g_pools[dev]) cudaMemPoolTrimTo(g_pools[dev], pool_keep());
}

cudaError_t gpa::pool_alloc(void **p, size_t bytes, cudaStream_t st) {
  std::mutex &mu = g_pool_mu;
  cudaMemPool_t *pools = g_pools;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone)
    return cudaMallocAsync(p, bytes, st);  // inside a CUDA-graph capture: a graph memory node
  if (dev < 0 || dev >= 64) return cudaMallocAsync(p, bytes, st);
  {
    std::lock_guard<std::mutex> lock(mu);
    if (!pools[dev]) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      e = cudaMemPoolCreate(&pools[dev], &props);
      if (e != cudaSuccess) return e;
      // keep up to pool_keep() bytes reserved between calls (default 8 GiB: the scratch of the
      // largest calls measured — f4 blame over 31 M events, a 4.19 M-context exact tree — so
      // repeated calls never go back to the driver; with 1 GiB f4 took 19.5 ms instead of 2.3);
      // memory above it is returned to the driver at synchronization points and after
      // gpa_free_cct / gpa_free_sparse, so a larger one-off does not stay reserved
      uint64_t keep = pool_keep();
      cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  static const bool dbg = getenv("GPA_DEBUG_POOL") != nullptr;  // (diagnostics) slow pool calls
  if (!dbg) return cudaMallocFromPoolAsync(p, bytes, pools[dev], st);
  const auto t0 = std::chrono::steady_clock::now();
  e = cudaMallocFromPoolAsync(p, bytes, pools[dev], st);
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (ms > 0.5) fprintf(stderr, "gpa pool_alloc %zu bytes: %.3f ms\n", bytes, ms);
  return e;
}

static gpa_status fail(gpa_status st, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

#define CU(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      if (e_ == cudaErrorMemoryAllocation) {                                             \
        cudaGetLastError();                                                              \
        return fail(GPA_ERR_OUT_OF_MEMORY, "%s: %s", #call, cudaGetErrorString(e_));     \
      }                                                                                  \
      return fail(GPA_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_));                \
    }                                                                                    \
  } while (0)

namespace {

struct DeviceGuard {
  int prev = -1;
  cudaError_t err = cudaSuccess;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) err = cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

namespace {
struct PoolScratch {  // stream-ordered scratch, released on the stream at scope exit
  cudaStream_t st;
  std::vector<void *> ptrs;
  explicit PoolScratch(cudaStream_t s) : st(s) {}
  template <class T>
  cudaError_t get(T **p, uint64_t count) {
    void *q = nullptr;
    cudaError_t e = pool_alloc(&q, count ? count * sizeof(T) : 8, st);
    if (e == cudaSuccess) ptrs.push_back(q);
    *p = (T *)q;
    return e;
  }
  ~PoolScratch() {
    for (void *p : ptrs)
      if (cudaFreeAsync(p, st) != cudaSuccess) cudaGetLastError();
  }
};
}  // namespace

// Everything validation derives on the way (needed again by the loader).
struct Derived {
  std::vector<uint32_t> inst_func;     // function of each instruction
  std::vector<uint32_t> func_of_scope; // function owning each FUNCTION scope
  std::vector<uint32_t> call_caller;   // caller function of each call site
};

gpa_status validate(const gpa_structure_desc *d, Derived *out) {
  if (!d) return fail(GPA_ERR_INVALID_ARG, "desc is NULL");
  const uint32_t ni = d->n_inst, ns = d->n_scope, nf = d->n_func, nc = d->n_call;
  if (ni && (!d->inst_addr || !d->inst_len || !d->inst_class || !d->inst_scope))
    return fail(GPA_ERR_INVALID_ARG, "instruction arrays are NULL with n_inst=%u", ni);
  if (ns && (!d->scope_parent || !d->scope_kind))
    return fail(GPA_ERR_INVALID_ARG, "scope arrays are NULL with n_scope=%u", ns);
  if (nf && !d->func_scope) return fail(GPA_ERR_INVALID_ARG, "func_scope is NULL with n_func=%u", nf);
  if (nc && (!d->call_inst || !d->call_callee))
    return fail(GPA_ERR_INVALID_ARG, "call arrays are NULL with n_call=%u", nc);
  if (ni > (1u << 28) - 16) return fail(GPA_ERR_STRUCTURE, "n_inst=%u exceeds 2^28-16", ni);
  // instructions: disjoint ranges in ascending order (reading R6)
  for (uint32_t i = 0; i < ni; i++) {
    if (d->inst_len[i] == 0) return fail(GPA_ERR_STRUCTURE, "inst_len[%u] == 0", i);
    if (d->inst_addr[i] > UINT64_MAX - d->inst_len[i])
      return fail(GPA_ERR_STRUCTURE, "instruction %u range overflows 2^64", i);
    if (i && d->inst_addr[i - 1] + d->inst_len[i - 1] > d->inst_addr[i])
      return fail(GPA_ERR_STRUCTURE, "instruction %u overlaps or precedes instruction %u", i, i - 1);
    if (d->inst_class[i] >= GPA_CLASSES) return fail(GPA_ERR_STRUCTURE, "inst_class[%u] > 15", i);
  }
  // scope tree: FUNCTION roots, LINE leaves, no cycles
  for (uint32_t s = 0; s < ns; s++) {
    uint8_t k = d->scope_kind[s];
    uint32_t p = d->scope_parent[s];
    if (k > GPA_KIND_LINE) return fail(GPA_ERR_STRUCTURE, "scope_kind[%u]=%u", s, k);
    if ((k == GPA_KIND_FUNCTION) != (p == NONE))
      return fail(GPA_ERR_STRUCTURE, "scope %u: FUNCTION scopes (only) must be roots", s);
    if (p != NONE) {
      if (p >= ns) return fail(GPA_ERR_STRUCTURE, "scope_parent[%u]=%u out of range", s, p);
      if (d->scope_kind[p] == GPA_KIND_LINE) return fail(GPA_ERR_STRUCTURE, "scope %u has a LINE parent", s);
    }
  }
  std::vector<uint8_t> state(ns, 0);  // 0 new, 1 on the current walk, 2 reaches a root
  std::vector<uint32_t> walk;
  for (uint32_t s = 0; s < ns; s++) {
    walk.clear();
    uint32_t x = s;
    while (x != NONE && state[x] == 0) {
      state[x] = 1;
      walk.push_back(x);
      x = d->scope_parent[x];
    }
    if (x != NONE && state[x] == 1) return fail(GPA_ERR_STRUCTURE, "scope tree has a cycle through %u", x);
    for (uint32_t y : walk) state[y] = 2;
  }
  out->func_of_scope.assign(ns, NONE);
  for (uint32_t f = 0; f < nf; f++) {
    uint32_t s = d->func_scope[f];
    if (s >= ns || d->scope_kind[s] != GPA_KIND_FUNCTION)
      return fail(GPA_ERR_STRUCTURE, "func_scope[%u]=%u is not a FUNCTION scope", f, s);
    if (out->func_of_scope[s] != NONE) return fail(GPA_ERR_STRUCTURE, "FUNCTION scope %u claimed twice", s);
    out->func_of_scope[s] = f;
  }
  for (uint32_t s = 0; s < ns; s++)
    if (d->scope_kind[s] == GPA_KIND_FUNCTION && out->func_of_scope[s] == NONE)
      return fail(GPA_ERR_STRUCTURE, "FUNCTION scope %u is not claimed by any function", s);
  // instruction -> LINE scope -> ... -> FUNCTION root -> function
  out->inst_func.resize(ni);
  std::vector<uint32_t> root(ns, NONE);
  for (uint32_t i = 0; i < ni; i++) {
    uint32_t s = d->inst_scope[i];
    if (s >= ns || d->scope_kind[s] != GPA_KIND_LINE)
      return fail(GPA_ERR_STRUCTURE, "inst_scope[%u]=%u is not a LINE scope", i, s);
    if (root[s] == NONE) {
      uint32_t x = s;
      while (d->scope_parent[x] != NONE) x = d->scope_parent[x];
      root[s] = x;
    }
    out->inst_func[i] = out->func_of_scope[root[s]];
  }
  // call sites: direct calls, one per call instruction (reading R22)
  out->call_caller.resize(nc);
  std::vector<uint8_t> is_call(ni, 0);
  for (uint32_t e = 0; e < nc; e++) {
    if (d->call_inst[e] >= ni) return fail(GPA_ERR_STRUCTURE, "call_inst[%u] out of range", e);
    if (d->call_callee[e] >= nf) return fail(GPA_ERR_STRUCTURE, "call_callee[%u] out of range", e);
    if (is_call[d->call_inst[e]]++) return fail(GPA_ERR_STRUCTURE, "two call sites on instruction %u", d->call_inst[e]);
    out->call_caller[e] = out->inst_func[d->call_inst[e]];
  }
  return GPA_OK;
}

// Tarjan's SCC algorithm, iterative form.  comp[v] = component id in completion order.
uint32_t tarjan(uint32_t n, const std::vector<uint32_t> &ptr, const std::vector<uint32_t> &dst,
                std::vector<uint32_t> &comp) {
  std::vector<uint32_t> index(n, NONE), low(n, 0), stack, it(n, 0);
  std::vector<uint8_t> on(n, 0);
  std::vector<uint32_t> call;
  uint32_t next = 0, ncomp = 0;
  comp.assign(n, NONE);
  for (uint32_t r = 0; r < n; r++) {
    if (index[r] != NONE) continue;
    call.push_back(r);
    index[r] = low[r] = next++;
    stack.push_back(r);
    on[r] = 1;
    it[r] = ptr[r];
    while (!call.empty()) {
      uint32_t v = call.back();
      if (it[v] < ptr[v + 1]) {
        uint32_t u = dst[it[v]++];
        if (index[u] == NONE) {
          index[u] = low[u] = next++;
          stack.push_back(u);
          on[u] = 1;
          it[u] = ptr[u];
          call.push_back(u);
        } else if (on[u]) {
          low[v] = std::min(low[v], index[u]);
        }
      } else {
        call.pop_back();
        if (!call.empty()) low[call.back()] = std::min(low[call.back()], low[v]);
        if (low[v] == index[v]) {
          uint32_t u;
          do {
            u = stack.back();
            stack.pop_back();
            on[u] = 0;
            comp[u] = ncomp;
          } while (u != v);
          ncomp++;
        }
      }
    }
  }
  return ncomp;
}

template <class T>
gpa_status upload(gpa_structure_s *s, T **dptr, const T *h, size_t n) {
  *dptr = nullptr;
  size_t bytes = sizeof(T) * (n ? n : 1);
  CU(cudaMalloc((void **)dptr, bytes));
  s->allocs.push_back(*dptr);
  s->info.device_bytes += bytes;
  if (n) CU(cudaMemcpy(*dptr, h, sizeof(T) * n, cudaMemcpyHostToDevice));
  return GPA_OK;
}

#define UP(dst, vec)                                                   \
  do {                                                                 \
    gpa_status st_ = upload(s, &(dst), (vec).data(), (vec).size());    \
    if (st_ != GPA_OK) return st_;                                     \
  } while (0)

void free_structure(gpa_structure_s *s) {
  if (!s) return;
  DeviceGuard g(s->device);
  scratch_release(&s->scratch);
  for (void *p : s->allocs) cudaFree(p);
  delete s;
}


gpa_status build(const gpa_structure_desc *d, const Derived &dv, gpa_structure_s *s) {
  const uint32_t ni = d->n_inst, ns = d->n_scope, nf = d->n_func, nc = d->n_call;
  gpa_structure_info &info = s->info;
  info.n_inst = ni; info.n_scope = ns; info.n_func = nf; info.n_call = nc;
  for (uint32_t x = 0; x < ns; x++) {
    if (d->scope_kind[x] == GPA_KIND_LINE) info.n_line++;
    if (d->scope_kind[x] == GPA_KIND_LOOP) info.n_loop++;
    if (d->scope_kind[x] == GPA_KIND_INLINE) info.n_inline++;
  }

  // ---- a-2: pc -> instruction map.  Granule 2^g = largest power of two that
  // divides every start offset and every length; each granule is then wholly inside one
  // instruction or wholly inside a gap, so the map reproduces [addr, addr+len) exactly.
  std::vector<uint64_t> addr(d->inst_addr, d->inst_addr + ni);
  std::vector<uint16_t> len(d->inst_len, d->inst_len + ni);
  std::vector<uint8_t> cls(d->inst_class, d->inst_class + ni);
  UP(s->d_inst_addr, addr);
  UP(s->d_inst_len, len);
  UP(s->d_inst_class, cls);
  AttrTables &T = s->attr;
  T.cache = &s->scratch;
  T.n_inst = ni;
  T.inst_addr = s->d_inst_addr;
  T.inst_len = s->d_inst_len;
  T.mode = 1;
  if (ni) {
    T.base = addr[0];
    T.end = addr[ni - 1] + len[ni - 1];
    uint64_t bits = 0;
    for (uint32_t i = 0; i < ni; i++) bits |= (addr[i] - T.base) | len[i];
    T.gshift = (uint32_t)__builtin_ctzll(bits);
    T.n_gran = (T.end - T.base) >> T.gshift;
    if (T.n_gran <= (1ull << 28)) {
      std::vector<uint32_t> gmap(T.n_gran, NONE);
      for (uint32_t i = 0; i < ni; i++) {
        uint64_t g0 = (addr[i] - T.base) >> T.gshift, g1 = (addr[i] + len[i] - T.base) >> T.gshift;
        for (uint64_t g = g0; g < g1; g++) gmap[g] = i;
      }
      UP(s->d_gmap, gmap);
      T.gmap = s->d_gmap;
      T.mode = 0;
      for (auto &x : gmap) x = x == NONE ? NONE : dv.inst_func[x];  // granule -> function
      UP(s->d_gfunc, gmap);
    }
  } else {
    T.base = 1;
    T.end = 0;  // empty range: every pc is unattributed
  }
  info.lookup_mode = T.mode;
  info.granule_shift = T.gshift;
  info.lookup_entries = T.mode == 0 ? T.n_gran : 0;

  // ---- a-5: roll-up CSR: row -> instructions whose scope chain
  // contains the row's scope.  LINE/LOOP/INLINE rows = scopes of that kind in ascending id;
  // FUNC rows = functions.
  std::vector<uint32_t> row_of(ns, NONE);
  RollSet *R = s->roll;
  for (uint32_t x = 0; x < ns; x++) {
    uint8_t k = d->scope_kind[x];
    int set = k == GPA_KIND_LINE ? ROLL_LINE : k == GPA_KIND_LOOP ? ROLL_LOOP : k == GPA_KIND_INLINE ? ROLL_INLINE : -1;
    if (set >= 0) {
      row_of[x] = (uint32_t)R[set].ids.size();
      R[set].ids.push_back(x);
    } else {
      row_of[x] = dv.func_of_scope[x];
    }
  }
  R[ROLL_FUNC].ids.resize(nf);
  std::iota(R[ROLL_FUNC].ids.begin(), R[ROLL_FUNC].ids.end(), 0u);
  auto set_of = [&](uint32_t x) -> int {
    uint8_t k = d->scope_kind[x];
    return k == GPA_KIND_LINE ? ROLL_LINE : k == GPA_KIND_LOOP ? ROLL_LOOP : k == GPA_KIND_INLINE ? ROLL_INLINE : ROLL_FUNC;
  };
  std::vector<std::vector<uint32_t>> ptr(ROLL_KINDS), lst(ROLL_KINDS);
  for (int k = 0; k < ROLL_KINDS; k++) {
    R[k].rows = (uint32_t)R[k].ids.size();
    ptr[k].assign(R[k].rows + 1, 0);
  }
  for (uint32_t i = 0; i < ni; i++)
    for (uint32_t x = d->inst_scope[i]; x != NONE; x = d->scope_parent[x]) ptr[set_of(x)][row_of[x] + 1]++;
  for (int k = 0; k < ROLL_KINDS; k++) {
    for (uint32_t r = 0; r < R[k].rows; r++) ptr[k][r + 1] += ptr[k][r];
    lst[k].resize(ptr[k][R[k].rows]);
  }
  {
    std::vector<std::vector<uint32_t>> fill(ptr);
    for (uint32_t i = 0; i < ni; i++)
      for (uint32_t x = d->inst_scope[i]; x != NONE; x = d->scope_parent[x]) {
        int k = set_of(x);
        lst[k][fill[k][row_of[x]]++] = i;
      }
  }
  // function layout (P:711-714 distributed statistics, gpa_derive_metrics_range): first / last
  // instruction of every function and whether each function is one contiguous run
  {
    std::vector<uint32_t> lo(nf, ni), hi(nf, 0), cnt(nf, 0);
    for (uint32_t i = 0; i < ni; i++) {
      const uint32_t f = dv.inst_func[i];
      lo[f] = std::min(lo[f], i);
      hi[f] = std::max(hi[f], i);
      cnt[f]++;
    }
    bool contig = true;
    for (uint32_t f = 0; f < nf; f++) contig = contig && (cnt[f] == 0 || hi[f] - lo[f] + 1 == cnt[f]);
    s->h_func_lo = lo;
    s->funcs_contiguous = contig;
    s->h_func_starts.clear();
    for (uint32_t f = 0; f < nf; f++)
      if (cnt[f]) s->h_func_starts.push_back(lo[f]);
    std::sort(s->h_func_starts.begin(), s->h_func_starts.end());
  }
  // function of every row of every kind (LINE / LOOP / INLINE: the scope's FUNCTION ancestor)
  std::vector<std::vector<uint32_t>> row_func(ROLL_KINDS);
  for (int k = 0; k < ROLL_KINDS; k++) row_func[k].assign(R[k].rows, 0);
  for (uint32_t x = 0; x < ns; x++) {
    const int k = set_of(x);
    if (k == ROLL_FUNC) continue;
    uint32_t y = x;
    while (d->scope_parent[y] != NONE) y = d->scope_parent[y];
    row_func[k][row_of[x]] = dv.func_of_scope[y];
  }
  for (uint32_t f = 0; f < nf; f++) row_func[ROLL_FUNC][f] = f;
  std::vector<std::vector<uint32_t>> h_chunks(ROLL_KINDS), h_mrows(ROLL_KINDS);
  for (int k = 0; k < ROLL_KINDS; k++) {
    UP(R[k].d_ptr, ptr[k]);
    UP(R[k].d_inst, lst[k]);
    // chunks of <= kRollChunk instructions; rows with several chunks get a scratch slot.  Rows
    // are visited in their function's instruction order (key = the function's first instruction)
    std::vector<uint32_t> rord(R[k].rows);
    std::iota(rord.begin(), rord.end(), 0u);
    auto key = [&](uint32_t r) { return s->h_func_lo[row_func[k][r]]; };
    std::stable_sort(rord.begin(), rord.end(), [&](uint32_t a, uint32_t b) { return key(a) < key(b); });
    std::vector<uint32_t> chunk, mslot(R[k].rows, NONE), mrows;
    R[k].h_chunk_key.clear();
    R[k].h_multi_key.clear();
    for (uint32_t r : rord) {
      uint32_t b = ptr[k][r], e = ptr[k][r + 1];
      if (e - b > kRollChunk) {
        mslot[r] = (uint32_t)mrows.size();
        mrows.push_back(r);
        R[k].h_multi_key.push_back(key(r));
      }
      if (b == e) { chunk.push_back(r); chunk.push_back(b); chunk.push_back(e); R[k].h_chunk_key.push_back(key(r)); }
      for (uint32_t x = b; x < e; x += kRollChunk) {
        chunk.push_back(r);
        chunk.push_back(x);
        chunk.push_back(std::min(e, x + kRollChunk));
        R[k].h_chunk_key.push_back(key(r));
      }
    }
    R[k].n_chunks = (uint32_t)(chunk.size() / 3);
    R[k].n_multi = (uint32_t)mrows.size();
    UP(R[k].d_chunk, chunk);
    UP(R[k].d_multi_slot, mslot);
    UP(R[k].d_multi_rows, mrows);
    h_chunks[k] = std::move(chunk);
    h_mrows[k] = std::move(mrows);
  }
  // the four kinds merged for gpa_derive_scopes: chunks and multi rows in function order (ties:
  // LINE, LOOP, INLINE, FUNC), instruction lists concatenated
  {
    MultiRoll &M = s->multi;
    std::vector<uint32_t> off(ROLL_KINDS + 1, 0);
    for (int k = 0; k < ROLL_KINDS; k++) off[k + 1] = off[k] + (uint32_t)lst[k].size();
    std::vector<uint32_t> all_lst(off[ROLL_KINDS]);
    for (int k = 0; k < ROLL_KINDS; k++) std::copy(lst[k].begin(), lst[k].end(), all_lst.begin() + off[k]);
    struct Item { uint32_t key, kind, a, b, c; };
    std::vector<Item> items, mitems;
    for (int k = 0; k < ROLL_KINDS; k++) {
      for (size_t c = 0; c < R[k].h_chunk_key.size(); c++)
        items.push_back({R[k].h_chunk_key[c], (uint32_t)k + 1, h_chunks[k][3 * c], h_chunks[k][3 * c + 1] + off[k],
                         h_chunks[k][3 * c + 2] + off[k]});
      for (size_t c = 0; c < h_mrows[k].size(); c++) mitems.push_back({R[k].h_multi_key[c], (uint32_t)k + 1, h_mrows[k][c], 0, 0});
    }
    auto by_key = [](const Item &x, const Item &y) { return x.key != y.key ? x.key < y.key : x.kind < y.kind; };
    std::stable_sort(items.begin(), items.end(), by_key);
    std::stable_sort(mitems.begin(), mitems.end(), by_key);
    std::vector<uint32_t> ch(4 * items.size()), mr(2 * mitems.size());
    M.h_chunk_key.resize(items.size());
    M.h_multi_key.resize(mitems.size());
    for (size_t i = 0; i < items.size(); i++) {
      ch[4 * i] = items[i].kind; ch[4 * i + 1] = items[i].a; ch[4 * i + 2] = items[i].b; ch[4 * i + 3] = items[i].c;
      M.h_chunk_key[i] = items[i].key;
    }
    std::vector<std::vector<uint32_t>> ms(ROLL_KINDS + 1);
    for (int k = 0; k < ROLL_KINDS; k++) ms[k + 1].assign(R[k].rows ? R[k].rows : 1, NONE);
    for (size_t i = 0; i < mitems.size(); i++) {
      mr[2 * i] = mitems[i].kind; mr[2 * i + 1] = mitems[i].a;
      M.h_multi_key[i] = mitems[i].key;
      ms[mitems[i].kind][mitems[i].a] = (uint32_t)i;
    }
    M.n_chunks = (uint32_t)items.size();
    M.n_multi = (uint32_t)mitems.size();
    if (ch.empty()) ch.assign(4, 0);
    if (mr.empty()) mr.assign(2, 0);
    if (all_lst.empty()) all_lst.assign(1, 0);
    UP(M.d_chunk, ch);
    UP(M.d_lst, all_lst);
    UP(M.d_mrows, mr);
    for (int k = 1; k <= ROLL_KINDS; k++) UP(M.d_mslot[k], ms[k]);
  }

  // ---- Step 1 structure: call graph from call instructions ---------------------
  std::vector<uint32_t> ci(d->call_inst, d->call_inst + nc), cc(d->call_callee, d->call_callee + nc);
  UP(s->d_call_inst, ci);
  UP(s->d_call_callee, cc);
  UP(s->d_call_caller, dv.call_caller);
  UP(s->d_inst_func, dv.inst_func);
  {
    std::vector<uint32_t> ic(ni ? ni : 1, NONE);
    for (uint32_t e = 0; e < nc; e++) ic[ci[e]] = e;  // one call site per call instruction (R22)
    UP(s->d_inst_call, ic);
  }
  std::vector<uint32_t> order(nc);
  std::iota(order.begin(), order.end(), 0u);
  std::sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return ci[a] < ci[b]; });
  std::vector<uint32_t> aptr(nf + 1, 0), adst(nc);  // adjacency for Tarjan
  std::vector<uint32_t> fin_ptr(nf + 1, 0), fin_e(nc);
  for (uint32_t e = 0; e < nc; e++) { aptr[dv.call_caller[e] + 1]++; fin_ptr[cc[e] + 1]++; }
  for (uint32_t f = 0; f < nf; f++) { aptr[f + 1] += aptr[f]; fin_ptr[f + 1] += fin_ptr[f]; }
  {
    std::vector<uint32_t> fa(aptr), fi(fin_ptr);
    for (uint32_t e : order) { adst[fa[dv.call_caller[e]]++] = cc[e]; fin_e[fi[cc[e]]++] = e; }
  }
  UP(s->d_fin_ptr, fin_ptr);
  UP(s->d_fin_e, fin_e);

  // ---- Step 3: Tarjan SCCs of the static call graph; DAG ids by ascending
  // smallest member (reading R17); non-trivial = >= 2 members or a self-call (R14).
  std::vector<uint32_t> comp;
  uint32_t ncomp = tarjan(nf, aptr, adst, comp);
  std::vector<uint32_t> cmin(ncomp, NONE), c2d(ncomp, NONE);
  for (uint32_t f = 0; f < nf; f++) cmin[comp[f]] = std::min(cmin[comp[f]], f);
  uint32_t nd = 0;
  for (uint32_t f = 0; f < nf; f++)
    if (cmin[comp[f]] == f) c2d[comp[f]] = nd++;
  s->h_scc_of.resize(nf);
  for (uint32_t f = 0; f < nf; f++) s->h_scc_of[f] = c2d[comp[f]];
  const std::vector<uint32_t> &scc = s->h_scc_of;
  info.n_dag = nd;
  std::vector<uint32_t> dmem_ptr(nd + 1, 0), dmem(nf);
  for (uint32_t f = 0; f < nf; f++) dmem_ptr[scc[f] + 1]++;
  for (uint32_t X = 0; X < nd; X++) dmem_ptr[X + 1] += dmem_ptr[X];
  {
    std::vector<uint32_t> fm(dmem_ptr);
    for (uint32_t f = 0; f < nf; f++) dmem[fm[scc[f]]++] = f;  // ascending function id
  }
  std::vector<uint8_t> nontriv(nd, 0);
  for (uint32_t X = 0; X < nd; X++) nontriv[X] = dmem_ptr[X + 1] - dmem_ptr[X] >= 2;
  for (uint32_t e = 0; e < nc; e++)
    if (dv.call_caller[e] == cc[e]) nontriv[scc[cc[e]]] = 1;
  for (uint32_t X = 0; X < nd; X++) info.n_scc += nontriv[X];
  // external edges: out-edges per function in call-instruction order; in-edges per DAG node
  std::vector<uint32_t> fout_ptr(nf + 1, 0), fout_e, din_ptr(nd + 1, 0), din_e;
  for (uint32_t e : order)
    if (scc[dv.call_caller[e]] != scc[cc[e]]) { fout_ptr[dv.call_caller[e] + 1]++; din_ptr[scc[cc[e]] + 1]++; }
  for (uint32_t f = 0; f < nf; f++) fout_ptr[f + 1] += fout_ptr[f];
  for (uint32_t X = 0; X < nd; X++) din_ptr[X + 1] += din_ptr[X];
  fout_e.resize(fout_ptr[nf]);
  din_e.resize(din_ptr[nd]);
  {
    std::vector<uint32_t> fo(fout_ptr), di(din_ptr);
    for (uint32_t e : order)
      if (scc[dv.call_caller[e]] != scc[cc[e]]) { fout_e[fo[dv.call_caller[e]]++] = e; din_e[di[scc[cc[e]]]++] = e; }
  }
  // static DAG levels (longest path from a source) and the all-edges context bound
  std::vector<uint32_t> indeg(nd, 0), level(nd, 0);
  std::vector<std::vector<uint32_t>> dsucc(nd);
  for (uint32_t e : din_e) { indeg[scc[cc[e]]]++; dsucc[scc[dv.call_caller[e]]].push_back(scc[cc[e]]); }
  std::vector<uint32_t> topo;
  for (uint32_t X = 0; X < nd; X++)
    if (!indeg[X]) topo.push_back(X);
  for (size_t q = 0; q < topo.size(); q++)
    for (uint32_t Y : dsucc[topo[q]]) {
      level[Y] = std::max(level[Y], level[topo[q]] + 1);
      if (--indeg[Y] == 0) topo.push_back(Y);
    }
  if (topo.size() != nd) return fail(GPA_ERR_INTERNAL, "condensed call graph is not a DAG");
  uint32_t nlev = 0;
  for (uint32_t X = 0; X < nd; X++) nlev = std::max(nlev, level[X] + 1);
  info.dag_levels = nlev;
  std::vector<uint32_t> dlev_ptr(nlev + 1, 0), dlev_node(nd);
  for (uint32_t X = 0; X < nd; X++) dlev_ptr[level[X] + 1]++;
  for (uint32_t L = 0; L < nlev; L++) dlev_ptr[L + 1] += dlev_ptr[L];
  {
    std::vector<uint32_t> fl(dlev_ptr);
    for (uint32_t X = 0; X < nd; X++) dlev_node[fl[level[X]]++] = X;
  }
  const uint64_t SAT = 1ull << 62;
  std::vector<uint64_t> paths(nd, 0);
  uint64_t bound = 0;
  for (uint32_t X : topo) {
    uint64_t p = din_ptr[X + 1] == din_ptr[X] ? 1 : 0;
    for (uint32_t k = din_ptr[X]; k < din_ptr[X + 1]; k++) p = std::min(SAT, p + paths[scc[dv.call_caller[din_e[k]]]]);
    paths[X] = p;
    uint64_t per = nontriv[X] ? 1 + (dmem_ptr[X + 1] - dmem_ptr[X]) : 1;
    bound = std::min(SAT, bound + (p > SAT / per ? SAT : p * per));
  }
  info.cct_path_bound = bound;
  UP(s->d_scc_of, s->h_scc_of);
  UP(s->d_fout_ptr, fout_ptr);
  UP(s->d_fout_e, fout_e);
  s->n_ext_calls = (uint32_t)fout_e.size();
  UP(s->d_din_ptr, din_ptr);
  UP(s->d_din_e, din_e);
  UP(s->d_dmem_ptr, dmem_ptr);
  UP(s->d_dmem, dmem);
  UP(s->d_dag_nontrivial, nontriv);
  UP(s->d_dlev_ptr, dlev_ptr);
  UP(s->d_dlev_node, dlev_node);
  CU(cudaDeviceSynchronize());
  return GPA_OK;
}

gpa_status check_dev_ptr(const void *p, int dev, const char *name) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(GPA_ERR_INVALID_ARG, "%s: not a CUDA pointer (%s)", name, cudaGetErrorString(e));
  }
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)
    return fail(GPA_ERR_INVALID_ARG, "%s is not device memory", name);
  if (a.type == cudaMemoryTypeDevice && a.device != dev)
    return fail(GPA_ERR_INVALID_ARG, "%s is on device %d, structure on %d", name, a.device, dev);
  return GPA_OK;
}

int sm_count(int dev) {
  static int cache[64] = {0};
  if (dev >= 0 && dev < 64 && cache[dev]) return cache[dev];
  int v = 148;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  if (dev >= 0 && dev < 64) cache[dev] = v;
  return v;
}

}  // namespace

#define CHECK(x)                         \
  do {                                   \
    gpa_status st_ = (x);                \
    if (st_ != GPA_OK) return st_;       \
  } while (0)

// ---- a-6..a-9 ---------------------------------------------------------------------------
// CCT memory is stream-ordered (the device's default memory pool, on the stream the tree was
// built on): allocation is a pool hit and freeing does not synchronize the device.
static void free_cct(gpa_cct_s *c) {
  if (!c) return;
  DeviceGuard g(c->device);
  for (void *p : c->allocs)
    if (cudaFreeAsync(p, c->stream) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(p);
    }
  const int dev = c->device;
  delete c;
  pool_trim(dev);  // whatever the stream has already released beyond the pool's threshold
}

// several arrays carved from ONE stream-ordered allocation (each 256-B aligned): a CCT call's
// dozen buffers cost one pool call instead of twelve (host time that small trees pay in full)
struct Carve {
  void **p;
  size_t bytes;
};
template <class T>
static Carve carve(T **p, size_t n) {
  return Carve{reinterpret_cast<void **>(p), sizeof(T) * (n ? n : 1)};
}
static cudaError_t alloc_block(gpa_cct_s *c, std::initializer_list<Carve> parts) {
  size_t tot = 0;
  for (const Carve &q : parts) tot += (q.bytes + 255) & ~(size_t)255;
  uint8_t *b = nullptr;
  cudaError_t e = pool_alloc((void **)&b, tot, c->stream);
  if (e != cudaSuccess) return e;
  c->allocs.push_back(b);
  for (const Carve &q : parts) {
    *q.p = b;
    b += (q.bytes + 255) & ~(size_t)255;
  }
  return cudaSuccess;
}

template <class T>
static cudaError_t calloc_dev(gpa_cct_s *c, T **p, size_t n) {
  *p = nullptr;
  cudaError_t e = pool_alloc((void **)p, sizeof(T) * (n ? n : 1), c->stream);
  if (e == cudaSuccess) c->allocs.push_back(*p);
  return e;
}

namespace gpa {
cudaError_t scratch_get(ScratchCache *c, size_t bytes, cudaStream_t st, void **out, bool *cached) {
  *cached = false;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) c = nullptr;  // graphs: pool
  if (c) {
    std::lock_guard<std::mutex> lock(c->mu);
    if (!c->busy) {
      cudaError_t e = cudaSuccess;
      if (!c->done) e = cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming);
      if (e == cudaSuccess && c->bytes < bytes) {  // grow: the old block is released after its last use
        if (c->mem) {
          if (c->last && c->last != st) cudaStreamWaitEvent(st, c->done, 0);
          cudaFreeAsync(c->mem, st);
          c->mem = nullptr;
          c->bytes = 0;
          c->last = st;
        }
        e = pool_alloc(&c->mem, bytes, st);
        if (e == cudaSuccess) c->bytes = bytes;
      }
      if (e == cudaSuccess && c->mem) {
        if (c->last && c->last != st) e = cudaStreamWaitEvent(st, c->done, 0);
        c->busy = true;
        *out = c->mem;
        *cached = true;
        return e;
      }
      cudaGetLastError();
    }
  }
  return pool_alloc(out, bytes, st);
}

cudaError_t scratch_put(ScratchCache *c, void *p, bool cached, cudaStream_t st) {
  if (!cached) return cudaFreeAsync(p, st);
  std::lock_guard<std::mutex> lock(c->mu);
  cudaError_t e = cudaEventRecord(c->done, st);
  c->last = st;
  c->busy = false;
  return e;
}

void scratch_release(ScratchCache *c) {
  std::lock_guard<std::mutex> lock(c->mu);
  if (c->mem) {
    if (c->done) cudaEventSynchronize(c->done);
    cudaFree(c->mem);
  }
  if (c->done) cudaEventDestroy(c->done);
  c->mem = nullptr;
  c->done = nullptr;
  c->bytes = 0;
}
}  // namespace gpa

extern "C" {

const char *gpa_version(void) { return "libgpa 0.1 (sm_100a)"; }
const char *gpa_last_error(void) { return g_err.c_str(); }
uint64_t gpa_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

gpa_status gpa_set_attr_kernel(int which) {
  if (which < 0 || which > 9) return fail(GPA_ERR_INVALID_ARG, "attribution kernel %d (0 auto, 1-9)", which);
  gpa::set_attr_kernel(which);
  return GPA_OK;
}

gpa_status gpa_set_ring_stress(int level) {
  if (level < 0 || level > 64) return fail(GPA_ERR_INVALID_ARG, "ring stress level %d (0 off, 1-64)", level);
  gpa::set_ring_stress(level);
  return GPA_OK;
}

gpa_status gpa_attr_kernel_choice(gpa_structure s, uint64_t n, int *which) {
  if (!s || !which) return fail(GPA_ERR_INVALID_ARG, "NULL argument");
  *which = attr_choice(s->attr, n);
  return GPA_OK;
}

gpa_status gpa_validate_structure(const gpa_structure_desc *desc) {
  Derived dv;
  return validate(desc, &dv);
}

gpa_status gpa_load_structure(const gpa_structure_desc *desc, int device, gpa_structure *out) {
  if (!out) return fail(GPA_ERR_INVALID_ARG, "out is NULL");
  *out = nullptr;
  Derived dv;
  CHECK(validate(desc, &dv));
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(GPA_ERR_INVALID_ARG, "device %d of %d", device, ndev);
  DeviceGuard g(device);
  CU(g.err);
  gpa_structure_s *s = new gpa_structure_s();
  s->device = device;
  gpa_status st = build(desc, dv, s);
  if (st != GPA_OK) {
    std::string msg = g_err;
    free_structure(s);
    g_err = msg;
    return st;
  }
  *out = s;
  return GPA_OK;
}

gpa_status gpa_get_structure_info(gpa_structure s, gpa_structure_info *out) {
  if (!s || !out) return fail(GPA_ERR_INVALID_ARG, "NULL argument");
  *out = s->info;
  return GPA_OK;
}

gpa_status gpa_scope_rows(gpa_structure s, gpa_scope scope, uint64_t *rows, uint32_t *h_ids) {
  if (!s || !rows) return fail(GPA_ERR_INVALID_ARG, "NULL argument");
  if (scope == GPA_SCOPE_INST) {
    *rows = s->info.n_inst;
    if (h_ids)
      for (uint32_t i = 0; i < s->info.n_inst; i++) h_ids[i] = i;
    return GPA_OK;
  }
  int k = scope == GPA_SCOPE_LINE ? ROLL_LINE : scope == GPA_SCOPE_LOOP ? ROLL_LOOP
        : scope == GPA_SCOPE_INLINE ? ROLL_INLINE : scope == GPA_SCOPE_FUNC ? ROLL_FUNC : -1;
  if (k < 0) return fail(GPA_ERR_INVALID_ARG, "scope %d has no static rows", (int)scope);
  *rows = s->roll[k].rows;
  if (h_ids && s->roll[k].rows) memcpy(h_ids, s->roll[k].ids.data(), sizeof(uint32_t) * s->roll[k].rows);
  return GPA_OK;
}

gpa_status gpa_get_scc(gpa_structure s, uint32_t *h_scc_of) {
  if (!s || (!h_scc_of && s->info.n_func)) return fail(GPA_ERR_INVALID_ARG, "NULL argument");
  if (s->info.n_func) memcpy(h_scc_of, s->h_scc_of.data(), sizeof(uint32_t) * s->info.n_func);
  return GPA_OK;
}

void gpa_free_structure(gpa_structure s) { free_structure(s); }

// ---- a-1..a-3 -------------------------------------------------------------------------
gpa_status gpa_attribute_samples(gpa_structure s, const gpa_sample *d_samples, uint64_t n,
                                 uint64_t *d_inst_hist, uint64_t *d_unattributed, uint32_t *d_rec_inst,
                                 gpa_stream_t stream) {
  if (!s) return fail(GPA_ERR_INVALID_ARG, "structure is NULL");
  if (n == 0) return GPA_OK;
  if (!d_samples || !d_unattributed || (!d_inst_hist && s->info.n_inst))
    return fail(GPA_ERR_INVALID_ARG, "NULL buffer with n=%llu", (unsigned long long)n);
  if ((uintptr_t)d_samples & 15) return fail(GPA_ERR_INVALID_ARG, "d_samples is not 16-byte aligned");
  DeviceGuard g(s->device);
  CU(g.err);
  CHECK(check_dev_ptr(d_samples, s->device, "d_samples"));
  CHECK(check_dev_ptr(d_unattributed, s->device, "d_unattributed"));
  if (d_inst_hist) CHECK(check_dev_ptr(d_inst_hist, s->device, "d_inst_hist"));
  if (d_rec_inst) CHECK(check_dev_ptr(d_rec_inst, s->device, "d_rec_inst"));
  CU(launch_attribute(s->attr, d_samples, n, (unsigned long long *)d_inst_hist,
                      (unsigned long long *)d_unattributed, d_rec_inst, sm_count(s->device),
                      (cudaStream_t)stream));
  return GPA_OK;
}

gpa_status gpa_attribute_samples_host(gpa_structure s, const gpa_sample *h_samples, uint64_t n,
                                      uint64_t *d_inst_hist, uint64_t *d_unattributed, gpa_stream_t stream) {
  if (!s) return fail(GPA_ERR_INVALID_ARG, "structure is NULL");
  if (n == 0) return GPA_OK;
  if (!h_samples || !d_unattributed || (!d_inst_hist && s->info.n_inst))
    return fail(GPA_ERR_INVALID_ARG, "NULL buffer with n=%llu", (unsigned long long)n);
  DeviceGuard g(s->device);
  CU(g.err);
  CHECK(check_dev_ptr(d_unattributed, s->device, "d_unattributed"));
  cudaStream_t st = (cudaStream_t)stream;
  // Pipeline: NBUF device staging buffers; H2D copy of chunk j on `cp` overlaps the
  // attribution kernel of chunk j-1 on `st`.
  const int NBUF = 3;
  const uint64_t CHUNK = 1ull << 22;  // records (64 MiB)
  uint64_t per = std::min<uint64_t>(CHUNK, n);
  cudaStream_t cp = nullptr;
  cudaEvent_t copied[NBUF] = {}, consumed[NBUF] = {};
  gpa_sample *buf[NBUF] = {};
  gpa_status ret = GPA_OK;
  void *plan_mem_err = nullptr;  // set below; released by cleanup() on an error path
  auto cleanup = [&]() {
    if (plan_mem_err) cudaFreeAsync(plan_mem_err, st);
    if (cp) cudaStreamSynchronize(cp);
    for (int b = 0; b < NBUF; b++) {
      if (buf[b]) cudaFreeAsync(buf[b], st);
      if (copied[b]) cudaEventDestroy(copied[b]);
      if (consumed[b]) cudaEventDestroy(consumed[b]);
    }
    if (cp) cudaStreamDestroy(cp);
    cudaStreamSynchronize(st);
  };
#define HC(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      ret = fail(e_ == cudaErrorMemoryAllocation ? GPA_ERR_OUT_OF_MEMORY : GPA_ERR_CUDA,  \
                 "%s: %s", #call, cudaGetErrorString(e_));                                \
      cudaGetLastError();                                                                 \
      cleanup();                                                                          \
      return ret;                                                                         \
    }                                                                                     \
  } while (0)
  HC(cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking));
  for (int b = 0; b < NBUF; b++) {
    HC(pool_alloc((void **)&buf[b], per * sizeof(gpa_sample), st));
    HC(cudaEventCreateWithFlags(&copied[b], cudaEventDisableTiming));
    HC(cudaEventCreateWithFlags(&consumed[b], cudaEventDisableTiming));
  }
  HC(cudaEventRecord(consumed[0], st));  // the staging buffers exist (stream-ordered) before any copy
  HC(cudaStreamWaitEvent(cp, consumed[0], 0));
  // the kernel is chosen for the whole call; a large-call kernel builds its plan once, from the
  // first chunk, accumulates every chunk and folds into H / U once at the end
  const int variant = attr_choice(s->attr, n);
  const bool planned = variant == 7 || variant == 8 || variant == 9;
  AttrPlan plan;
  AttrAcc acc;
  void *plan_mem = nullptr;
  for (uint64_t off = 0, j = 0; off < n; off += per, j++) {
    int b = (int)(j % NBUF);
    uint64_t m = std::min(per, n - off);
    if (j >= NBUF) HC(cudaStreamWaitEvent(cp, consumed[b], 0));
    HC(cudaMemcpyAsync(buf[b], h_samples + off, m * sizeof(gpa_sample), cudaMemcpyHostToDevice, cp));
    HC(cudaEventRecord(copied[b], cp));
    HC(cudaStreamWaitEvent(st, copied[b], 0));
    if (planned && j == 0) {
      HC(pool_alloc(&plan_mem, plan_bytes(s->attr, variant), st));
      plan_mem_err = plan_mem;
      HC(plan_build(s->attr, variant, reinterpret_cast<const uint4 *>(buf[b]), m, plan_mem, &plan, sm_count(s->device), st));
      HC(plan_begin(plan, &acc, sm_count(s->device), st));
    }
    if (planned)
      HC(plan_run(s->attr, plan, acc, reinterpret_cast<const uint4 *>(buf[b]), m, nullptr, sm_count(s->device), st));
    else
      HC(launch_attribute(s->attr, buf[b], m, (unsigned long long *)d_inst_hist,
                          (unsigned long long *)d_unattributed, nullptr, sm_count(s->device), st));
    HC(cudaEventRecord(consumed[b], st));
  }
  if (planned) {
    HC(plan_end(s->attr, plan, &acc, (unsigned long long *)d_inst_hist, (unsigned long long *)d_unattributed,
                sm_count(s->device), st));
    plan_mem_err = nullptr;
    HC(cudaFreeAsync(plan_mem, st));
    plan_mem = nullptr;
  }
#undef HC
  cleanup();
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(GPA_ERR_CUDA, "attribute_samples_host: %s", cudaGetErrorString(e));
  return GPA_OK;
}

// Steps 1-4 from the instruction histogram (d_inst_hist) or from precomputed Step-1
// inputs (d_func_hist = S_f, d_call_weight = w; gpa_reconstruct_cct_inputs)
// async_: the one-launch build is left pending (no synchronization; gpa_cct_finish reads the size)
static gpa_status reconstruct(gpa_structure s, bool from_hist, const uint64_t *d_inst_hist, const uint64_t *d_func_hist,
                              const uint64_t *d_call_weight, gpa_weight_mode mode, uint64_t max_contexts, gpa_cct *out,
                              uint64_t *n_contexts, gpa_stream_t stream, bool async_ = false) {
  if (!s || !n_contexts || (max_contexts && !out)) return fail(GPA_ERR_INVALID_ARG, "NULL argument");
  if (mode != GPA_WEIGHTS_SAMPLES && mode != GPA_WEIGHTS_EXACT) return fail(GPA_ERR_INVALID_ARG, "mode %d", (int)mode);
  if (out) *out = nullptr;
  DeviceGuard g(s->device);
  CU(g.err);
  cudaStream_t st = (cudaStream_t)stream;
  const gpa_structure_info &I = s->info;
  gpa_cct_s *c = new gpa_cct_s();
  c->device = s->device;
  c->stream = st;
  c->n_call = I.n_call; c->n_func = I.n_func; c->n_dag = I.n_dag;
  unsigned long long *d_cnt = nullptr;  // [0] total contexts, [1] next-level size
  gpa_status ret = GPA_OK;
#define CC(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      ret = fail(e_ == cudaErrorMemoryAllocation ? GPA_ERR_OUT_OF_MEMORY : GPA_ERR_CUDA,  \
                 "%s: %s", #call, cudaGetErrorString(e_));                                \
      cudaGetLastError();                                                                 \
      free_cct(c);                                                                        \
      return ret;                                                                         \
    }                                                                                     \
  } while (0)
  CC(alloc_block(c, {carve(&c->w, I.n_call), carve(&c->S_f, (size_t)I.n_func * SLOTS), carve(&c->func_active, I.n_func),
                      carve(&c->dag_active, I.n_dag), carve(&c->W, I.n_dag), carve(&d_cnt, 4)}));
  // Step 1: edge weights and per-function samples S_f (the FUNC roll-up), or the caller's
  // (copied: Step 2 rewrites w)
  if (from_hist) {
    CC(launch_cct_weights(s, d_inst_hist, c->w, st));
    CC(launch_rollup(&s->roll[ROLL_FUNC], s->roll[ROLL_FUNC].rows, d_inst_hist, s->d_inst_class, c->S_f, nullptr,
                     nullptr, sm_count(s->device), st));
  } else {
    if (I.n_call) CC(cudaMemcpyAsync(c->w, d_call_weight, sizeof(uint64_t) * I.n_call, cudaMemcpyDeviceToDevice, st));
    if (I.n_func)
      CC(cudaMemcpyAsync(c->S_f, d_func_hist, sizeof(uint64_t) * SLOTS * I.n_func, cudaMemcpyDeviceToDevice, st));
  }
  unsigned long long h_cnt[2] = {0, 0};
  const bool small_static = cct_small_ok(s, I.cct_path_bound);
  if (max_contexts && (small_static || cct_small_ok(s, kSmallContexts))) {
    // Small static bound: build straight into bound-sized arrays with one CTA and read the
    // size back once at the end (no separate path count, one host synchronization).  Larger
    // static bounds (C3: 4.19 M paths, ~37 k sampled contexts) try the same into kSmallContexts
    // slots first and fall back to the counted build only if the tree does not fit.
    CC(launch_cct_propagate(s, c->S_f, c->w, c->func_active, c->dag_active, c->W, d_cnt, mode == GPA_WEIGHTS_EXACT,
                            false, st));
    const uint64_t nb = small_static ? I.cct_path_bound : kSmallContexts;
    c->n = nb;
    uint32_t *d_lev = nullptr;
    CC(alloc_block(c, {carve(&c->parent, nb), carve(&c->site, nb), carve(&c->node, nb), carve(&c->first_child, nb),
                       carve(&c->n_children, nb), carve(&c->kind, nb), carve(&c->frac, nb), carve(&c->excl, nb * SLOTS),
                       carve(&c->incl, nb * SLOTS), carve(&d_lev, 1100)}));
    c->d_lev = d_lev; c->lev_fmt = 1; c->lev_len = 1100;
    CC(launch_cct_small(s, c, d_lev, d_cnt + 1, sm_count(s->device), st));
    if (async_) {  // gpa_reconstruct_cct_async: size (and a fall-back rebuild) left to gpa_cct_finish
      c->pending = true;
      c->d_built = d_cnt + 1;
      c->src = s;
      c->src_hist = d_inst_hist;
      c->src_mode = (int)mode;
      *n_contexts = nb;
      *out = c;
      return GPA_OK;
    }
    CC(cudaMemcpyAsync(h_cnt + 1, d_cnt + 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CC(cudaStreamSynchronize(st));
    if (h_cnt[1] > nb && small_static) {
      free_cct(c);
      return fail(GPA_ERR_INTERNAL, "tree of %llu contexts exceeds the static bound %llu", h_cnt[1],
                  (unsigned long long)nb);
    }
    if (h_cnt[1] <= nb) {
      c->n = h_cnt[1];
      *n_contexts = c->n;
      if (c->n > max_contexts) {
        free_cct(c);
        return fail(GPA_ERR_CAPACITY, "%llu contexts > max_contexts %llu", (unsigned long long)*n_contexts,
                    (unsigned long long)max_contexts);
      }
      *out = c;
      return GPA_OK;
    }
    // the optimistic build overflowed: the counted build below.  Step 2 rewrote w in place and
    // the activity it derived is not recoverable from w alone, so w is reset to the Step-1
    // weights first (the slots above stay allocated until gpa_free_cct)
    c->n = 0;
    c->d_lev = nullptr; c->lev_fmt = 0; c->lev_len = 0;
    if (from_hist) CC(launch_cct_weights(s, d_inst_hist, c->w, st));
    else if (I.n_call)
      CC(cudaMemcpyAsync(c->w, d_call_weight, sizeof(uint64_t) * I.n_call, cudaMemcpyDeviceToDevice, st));
  }
  // Step 2 + guard (R12) + W + context count (path DP over the DAG)
  CC(launch_cct_propagate(s, c->S_f, c->w, c->func_active, c->dag_active, c->W, d_cnt, mode == GPA_WEIGHTS_EXACT,
                          true, st));
  CC(cudaMemcpyAsync(h_cnt, d_cnt, sizeof(h_cnt), cudaMemcpyDeviceToHost, st));
  CC(cudaStreamSynchronize(st));
  *n_contexts = h_cnt[0];
  if (max_contexts == 0 || h_cnt[0] > max_contexts) {
    free_cct(c);
    if (max_contexts == 0) return GPA_OK;
    return fail(GPA_ERR_CAPACITY, "%llu contexts > max_contexts %llu", h_cnt[0], (unsigned long long)max_contexts);
  }
  const uint64_t n = h_cnt[0];
  if (n >= (1ull << 32) - 1) {
    free_cct(c);
    return fail(GPA_ERR_CAPACITY, "%llu contexts exceed the u32 context index", (unsigned long long)n);
  }
  c->n = n;
  CC(alloc_block(c, {carve(&c->parent, n), carve(&c->site, n), carve(&c->node, n), carve(&c->first_child, n),
                     carve(&c->n_children, n), carve(&c->kind, n), carve(&c->frac, n), carve(&c->excl, n * SLOTS),
                     carve(&c->incl, n * SLOTS)}));
  if (cct_small_ok(s, n)) {  // one CTA builds the whole tree: no per-level launches or syncs
    uint32_t *d_lev = nullptr;
    CC(calloc_dev(c, &d_lev, 1100));
    c->d_lev = d_lev; c->lev_fmt = 1; c->lev_len = 1100;
    CC(launch_cct_small(s, c, d_lev, d_cnt + 1, sm_count(s->device), st));
    *out = c;
    return GPA_OK;
  }
  uint32_t *d_tmp = nullptr, *d_bs = nullptr;
  CC(calloc_dev(c, &d_tmp, n + 1));
  CC(calloc_dev(c, &d_bs, 65536));
  {  // one cooperative launch walks every level (falls back to per-level launches if refused)
    const uint32_t max_lev = 2 * I.dag_levels + 4;
    uint32_t *d_lev = nullptr;
    CC(calloc_dev(c, &d_lev, max_lev + 2));
    cudaError_t e = launch_cct_coop(s, c, d_tmp, d_bs, d_lev, max_lev, d_cnt + 1, sm_count(s->device), st);
    if (e == cudaSuccess) {
      c->d_lev = d_lev; c->lev_fmt = 2; c->lev_len = max_lev + 2;
      CC(cudaMemcpyAsync(h_cnt + 1, d_cnt + 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
      CC(cudaStreamSynchronize(st));
      if (h_cnt[1] != n) {
        free_cct(c);
        return fail(GPA_ERR_INTERNAL, "cooperative BFS built %llu contexts, path count said %llu", h_cnt[1],
                    (unsigned long long)n);
      }
      *out = c;
      return GPA_OK;
    }
    cudaGetLastError();
  }
  // Step 4: breadth-first split of the DAG into the tree, level by level
  CC(launch_cct_roots(s, c->dag_active, c, d_cnt + 1, st));
  CC(cudaMemcpyAsync(h_cnt + 1, d_cnt + 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  CC(cudaStreamSynchronize(st));
  uint64_t a = 0, b = h_cnt[1];
  c->level_start.push_back(0);
  while (b > a) {
    c->level_start.push_back(b);
    if (b > n) { free_cct(c); return fail(GPA_ERR_INTERNAL, "BFS overran the counted contexts"); }
    CC(launch_cct_level(s, c, a, b, d_tmp, d_bs, d_cnt + 1, st));
    CC(cudaMemcpyAsync(h_cnt + 1, d_cnt + 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CC(cudaStreamSynchronize(st));
    a = b;
    b += h_cnt[1];
  }
  if (b != n) {
    free_cct(c);
    return fail(GPA_ERR_INTERNAL, "BFS built %llu contexts, path count said %llu", (unsigned long long)b,
                (unsigned long long)n);
  }
  CC(launch_cct_excl(s, c, st));
  for (size_t L = c->level_start.size() - 1; L-- > 0;)
    CC(launch_cct_incl_level(c, c->level_start[L], c->level_start[L + 1], st));
#undef CC
  *out = c;
  return GPA_OK;
}

gpa_status gpa_attribute_profiles(gpa_structure s, const gpa_sample *d_samples, uint64_t n, uint32_t n_profiles,
                                  uint64_t *d_prof_hist, uint64_t *d_prof_unattr, gpa_stream_t stream) {
  if (!s) return fail(GPA_ERR_INVALID_ARG, "structure is NULL");
  if (n == 0) return GPA_OK;
  if (!d_samples || !d_prof_unattr || (!d_prof_hist && s->info.n_func))
    return fail(GPA_ERR_INVALID_ARG, "NULL buffer with n=%llu", (unsigned long long)n);
  if ((uintptr_t)d_samples & 15) return fail(GPA_ERR_INVALID_ARG, "d_samples is not 16-byte aligned");
  if (n_profiles > 65536) return fail(GPA_ERR_INVALID_ARG, "n_profiles %u > 65536", n_profiles);
  DeviceGuard g(s->device);
  CU(g.err);
  CHECK(check_dev_ptr(d_samples, s->device, "d_samples"));
  CU(launch_attribute_profiles(s->attr, s->d_inst_func, s->d_gfunc, s->info.n_func, d_samples, n, n_profiles,
                               (unsigned long long *)d_prof_hist, (unsigned long long *)d_prof_unattr,
                               sm_count(s->device), (cudaStream_t)stream));
  return GPA_OK;
}

gpa_status gpa_profile_stats(gpa_structure s, const uint64_t *d_prof_hist, uint32_t n_profiles, double *d_stats,
                             gpa_stream_t stream) {
  if (!s) return fail(GPA_ERR_INVALID_ARG, "structure is NULL");
  if (!s->info.n_func) return GPA_OK;
  if (!d_prof_hist || !d_stats) return fail(GPA_ERR_INVALID_ARG, "NULL buffer");
  DeviceGuard g(s->device);
  CU(g.err);
  CU(launch_profile_stats(d_prof_hist, n_profiles, s->info.n_func, d_stats, (cudaStream_t)stream));
  return GPA_OK;
}

gpa_status gpa_attribute_profiles_inst(gpa_structure s, const gpa_sample *d_samples, uint64_t n, uint32_t n_profiles,
                                       uint64_t *d_prof_inst_hist, uint64_t *d_prof_unattr, gpa_stream_t stream) {
  if (!s) return fail(GPA_ERR_INVALID_ARG, "structure is NULL");
  if (n == 0) return GPA_OK;
  if (!d_samples || !d_prof_unattr || (!d_prof_inst_hist && s->info.n_inst))
    return fail(GPA_ERR_INVALID_ARG, "NULL buffer with n=%llu", (unsigned long long)n);
  if ((uintptr_t)d_samples & 15) return fail(GPA_ERR_INVALID_ARG, "d_samples is not 16-byte aligned");
  if (n_profiles > 65536) return fail(GPA_ERR_INVALID_ARG, "n_profiles %u > 65536", n_profiles);
  DeviceGuard g(s->device);
  CU(g.err);
  CHECK(check_dev_ptr(d_samples, s->device, "d_samples"));
  CU(launch_attribute_profiles_inst(s->attr, s->info.n_inst, d_samples, n, n_profiles,
                                    (unsigned long long *)d_prof_inst_hist, (unsigned long long *)d_prof_unattr,
                                    sm_count(s->device), (cudaStream_t)stream));
  return GPA_OK;
}

gpa_status gpa_profile_stats_rows(uint64_t rows, const uint64_t *d_prof_hist, uint32_t n_profiles, double *d_stats,
                                  int device, gpa_stream_t stream) {
  if (!rows) return GPA_OK;
  if (!d_prof_hist || !d_stats) return fail(GPA_ERR_INVALID_ARG, "NULL buffer");
  if (rows >= (1ull << 32)) return fail(GPA_ERR_UNSUPPORTED, "rows >= 2^32");
  DeviceGuard g(device);
  CU(g.err);
  CU(launch_profile_stats(d_prof_hist, n_profiles, (uint32_t)rows, d_stats, (cudaStream_t)stream));
  return GPA_OK;
}

gpa_status gpa_profile_stats_f64(uint64_t rows, const double *d_prof_vals, uint32_t n_profiles, double *d_stats,
                                 int device, gpa_stream_t stream) {
  if (!rows) return GPA_OK;
  if (!d_prof_vals || !d_stats) return fail(GPA_ERR_INVALID_ARG, "NULL buffer");
  DeviceGuard g(device);
  CU(g.err);
  CU(launch_profile_stats_f64(d_prof_vals, n_profiles, rows, d_stats, (cudaStream_t)stream));
  return GPA_OK;
}

// BFS level boundaries of a tree, whichever build path made it (synchronizes c->stream once)
static gpa_status cct_levels(gpa_cct_s *c) {
  if (!c->level_start.empty() || c->n == 0) return GPA_OK;
  if (!c->d_lev) return fail(GPA_ERR_INTERNAL, "tree has no level table");
  std::vector<uint32_t> h(c->lev_len);
  CU(cudaMemcpyAsync(h.data(), c->d_lev, 4ull * c->lev_len, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  std::vector<uint64_t> ls;
  if (c->lev_fmt == 1) {
    const uint32_t L = h[0];
    for (uint32_t l = 0; l <= L && 1 + l < c->lev_len; l++) ls.push_back(h[1 + l]);
  } else {
    ls.push_back(h[0]);
    for (uint32_t l = 1; l < c->lev_len && ls.back() < c->n; l++) ls.push_back(h[l]);
  }
  if (ls.empty() || ls.front() != 0 || ls.back() != c->n)
    return fail(GPA_ERR_INTERNAL, "inconsistent level table (%zu levels)", ls.size());
  c->level_start = ls;
  return GPA_OK;
}

gpa_status gpa_cct_profiles(gpa_structure s, gpa_cct cct, const uint64_t *d_prof_hist, uint32_t n_profiles,
                            double *d_prof_excl, double *d_prof_incl, gpa_stream_t stream) {
  if (!s || !cct) return fail(GPA_ERR_INVALID_ARG, "NULL handle");
  if (cct->pending) return fail(GPA_ERR_INVALID_ARG, "asynchronous tree: call gpa_cct_finish first");
  if (cct->n == 0) return GPA_OK;
  if (!d_prof_hist || !d_prof_excl || !d_prof_incl) return fail(GPA_ERR_INVALID_ARG, "NULL buffer");
  if (n_profiles > 65536) return fail(GPA_ERR_INVALID_ARG, "n_profiles %u > 65536", n_profiles);
  DeviceGuard g(s->device);
  CU(g.err);
  gpa_status r = cct_levels(cct);
  if (r != GPA_OK) return r;
  cudaStream_t st = (cudaStream_t)stream;
  const uint32_t P1 = n_profiles + 1;
  CU(launch_cct_prof_excl(s, cct, d_prof_hist, P1, d_prof_excl, st));
  for (size_t L = cct->level_start.size() - 1; L-- > 0;)
    CU(launch_cct_prof_incl_level(cct, cct->level_start[L], cct->level_start[L + 1], P1, d_prof_excl, d_prof_incl, st));
  return GPA_OK;
}

gpa_status gpa_idleness_blame(const gpa_trace_desc *d, const uint64_t *d_time, const uint32_t *d_ctx, double *d_blame,
                              double *d_share, uint64_t *d_total, uint64_t *d_gpu_idle, int device,
                              gpa_stream_t stream) {
  if (!d || (d->n_lines && (!d->line_off || !d->line_kind || !d->line_scope)))
    return fail(GPA_ERR_INVALID_ARG, "NULL trace descriptor array");
  if (d->n_scopes == 0 || d->n_routines == 0) return fail(GPA_ERR_INVALID_ARG, "n_scopes and n_routines must be > 0");
  const uint32_t L = d->n_lines, S = d->n_scopes, R = d->n_routines;
  if (L == 0 || d->line_off[0] != 0) return fail(GPA_ERR_INVALID_ARG, "line_off[0] must be 0 (and n_lines > 0)");
  std::vector<uint32_t> n_gpu(S, 0), n_cpu(S, 0);
  for (uint32_t l = 0; l < L; l++) {
    if (d->line_off[l + 1] < d->line_off[l]) return fail(GPA_ERR_INVALID_ARG, "line_off decreases at line %u", l);
    if (d->line_scope[l] >= S || (l && d->line_scope[l] < d->line_scope[l - 1]))
      return fail(GPA_ERR_INVALID_ARG, "line_scope[%u] out of range or not grouped", l);
    if (d->line_kind[l] > 1) return fail(GPA_ERR_INVALID_ARG, "line_kind[%u] = %u", l, d->line_kind[l]);
    (d->line_kind[l] ? n_cpu : n_gpu)[d->line_scope[l]]++;
  }
  uint32_t kmax = 1;
  for (uint32_t sc = 0; sc < S; sc++) {
    if (!n_gpu[sc]) return fail(GPA_ERR_INVALID_ARG, "scope %u has no GPU line", sc);
    if (n_gpu[sc] > 65535 || n_cpu[sc] > 65535) return fail(GPA_ERR_UNSUPPORTED, "scope %u has > 65535 lines", sc);
    kmax = std::max(kmax, n_cpu[sc]);
  }
  const uint64_t n = d->line_off[L];
  if (n > (1ull << 27)) return fail(GPA_ERR_UNSUPPORTED, "%llu events > 2^27", (unsigned long long)n);
  if (n * kmax >= (1ull << 32)) return fail(GPA_ERR_UNSUPPORTED, "events x CPU lines per scope >= 2^32");
  if (S >= (1u << 28)) return fail(GPA_ERR_UNSUPPORTED, "n_scopes >= 2^28");
  if (n && (!d_time || !d_ctx)) return fail(GPA_ERR_INVALID_ARG, "NULL event arrays");
  DeviceGuard g(device);
  CU(g.err);
  cudaStream_t st = (cudaStream_t)stream;

  // merge plan: per scope, the non-empty lines are the sorted runs; pair adjacent runs per round
  std::vector<std::vector<std::pair<uint64_t, uint64_t>>> runs(S);
  size_t max_runs = 1;
  for (uint32_t l = 0; l < L; l++)
    if (d->line_off[l + 1] > d->line_off[l]) runs[d->line_scope[l]].push_back({d->line_off[l], d->line_off[l + 1]});
  for (auto &r : runs) max_runs = std::max(max_runs, r.size());
  int rounds = 1;
  while ((size_t(1) << rounds) < max_runs) rounds++;
  std::vector<MergePair> pairs;
  std::vector<uint64_t> chunks;
  std::vector<uint32_t> round_np;
  for (int r = 0; r < rounds; r++) {
    uint32_t np = 0;
    uint64_t c = 0;
    chunks.push_back(0);
    for (auto &rs : runs) {
      std::vector<std::pair<uint64_t, uint64_t>> next;
      for (size_t i = 0; i < rs.size(); i += 2) {
        MergePair p{rs[i].first, rs[i].second, i + 1 < rs.size() ? rs[i + 1].second : rs[i].second};
        pairs.push_back(p);
        c += (p.b1 - p.a0 + kMergeChunkHost - 1) / kMergeChunkHost;
        chunks.push_back(c);
        next.push_back({p.a0, p.b1});
        np++;
      }
      rs.swap(next);
    }
    round_np.push_back(np);
  }

  PoolScratch mem(st);
  BlameArgs a{};
  a.n = n; a.n_scopes = S; a.n_routines = R; a.kmax = kmax;
  a.time = d_time; a.ctx = d_ctx;
  a.blame = d_blame; a.share = d_share; a.total = d_total; a.gpu_idle = d_gpu_idle;
  uint64_t *d_off = nullptr, *t0 = nullptr, *t1 = nullptr, *d_chunks = nullptr;
  uint8_t *d_kind = nullptr;
  uint32_t *d_scope = nullptr, *i0 = nullptr, *i1 = nullptr;
  MergePair *d_pairs = nullptr;
  const uint64_t nsr = (uint64_t)S * R * (kmax + 1);
  CU(mem.get(&d_off, L + 1));
  CU(mem.get(&d_kind, L));
  CU(mem.get(&d_scope, L));
  CU(mem.get(&d_pairs, pairs.size()));
  CU(mem.get(&d_chunks, chunks.size()));
  CU(mem.get(&t0, n)); CU(mem.get(&t1, n)); CU(mem.get(&i0, n)); CU(mem.get(&i1, n)); CU(mem.get(&a.info, n));
  CU(mem.get(&a.pos, n)); CU(mem.get(&a.delta, n)); CU(mem.get(&a.scan, n)); CU(mem.get(&a.psc, n));
  CU(mem.get(&a.bidx, n)); CU(mem.get(&a.pk, n)); CU(mem.get(&a.pdur, n));
  CU(mem.get(&a.ovf, n * kmax / 256 + 1));
  CU(mem.get(&a.seg, n));
  CU(mem.get(&a.seg_n, n / 8192 + 1));
  CU(mem.get(&a.bs, kScanScratchWords)); CU(mem.get(&a.err, 4)); CU(mem.get(&a.tots, 4));
  CU(mem.get(&a.acc, 2ull * S)); CU(mem.get(&a.num, nsr));
  uint64_t max_tiles = 0, *d_split = nullptr;
  for (size_t r = 0, cofs = 0; r < round_np.size(); cofs += round_np[r] + 1, r++)
    max_tiles = std::max(max_tiles, chunks[cofs + round_np[r]]);
  CU(mem.get(&d_split, 2 * max_tiles + 2));  // split [tiles+1] then the tile -> pair map (u32)
  CU(cudaMemcpyAsync(d_off, d->line_off, (L + 1) * 8, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(d_kind, d->line_kind, L, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(d_scope, d->line_scope, L * 4, cudaMemcpyHostToDevice, st));
  if (!pairs.empty()) CU(cudaMemcpyAsync(d_pairs, pairs.data(), pairs.size() * sizeof(MergePair), cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(d_chunks, chunks.data(), chunks.size() * 8, cudaMemcpyHostToDevice, st));
  CU(cudaMemsetAsync(a.err, 0, 16, st));
  CU(cudaMemsetAsync(a.acc, 0, 16ull * S, st));
  CU(cudaMemsetAsync(a.num, 0, nsr * 8, st));
  a.line_off = d_off; a.line_kind = d_kind; a.line_scope = d_scope;
  if (n) {
    CU(blame_prep(a, L, st));
    const uint64_t *src_t = d_time;
    const uint32_t *src_i = nullptr;
    uint64_t *dst_t = t0;
    uint32_t *dst_i = i0;
    size_t pofs = 0, cofs = 0;
    for (int r = 0; r < rounds; r++) {
      const uint32_t np = round_np[r];
      CU(blame_merge(d_pairs + pofs, d_chunks + cofs, np, chunks[cofs + np], src_t, src_i, dst_t, dst_i, d_split, st));
      pofs += np;
      cofs += np + 1;
      src_t = dst_t; src_i = dst_i;
      dst_t = dst_t == t0 ? t1 : t0;
      dst_i = dst_i == i0 ? i1 : i0;
    }
    a.st = src_t;
    a.ord = src_i;
  }
  CU(blame_sweep(a, st));
  uint32_t h_err = 0;
  CU(cudaMemcpyAsync(&h_err, a.err, 4, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  if (h_err & 1) return fail(GPA_ERR_INVALID_ARG, "a trace line goes back in time");
  if (h_err & 2) return fail(GPA_ERR_INVALID_ARG, "a CPU routine id is >= n_routines");
  return GPA_OK;
}

static void free_sparse(gpa_sparse_s *sp) {
  if (!sp) return;
  DeviceGuard g(sp->device);
  for (void *p : sp->allocs)
    if (cudaFreeAsync(p, sp->stream) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(p);
    }
  const int dev = sp->device;
  delete sp;
  pool_trim(dev);
}

gpa_status gpa_sparse_build(gpa_structure s, const uint64_t *d_prof_hist, uint32_t n_profiles, gpa_sparse_major major,
                            gpa_sparse *out, gpa_stream_t stream) {
  if (!s || !out) return fail(GPA_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  if (major != GPA_SPARSE_PMS && major != GPA_SPARSE_CMS) return fail(GPA_ERR_INVALID_ARG, "major %d", (int)major);
  const uint32_t P = n_profiles + 1, C = s->info.n_func;
  if (C && !d_prof_hist) return fail(GPA_ERR_INVALID_ARG, "d_prof_hist is NULL");
  if ((uint64_t)P * C * GPA_SLOTS >= (1ull << 32))
    return fail(GPA_ERR_UNSUPPORTED, "cube of %llu cells exceeds 2^32", (unsigned long long)P * C * GPA_SLOTS);
  DeviceGuard g(s->device);
  CU(g.err);
  cudaStream_t st = (cudaStream_t)stream;
  gpa_sparse_s *sp = new gpa_sparse_s();
  sp->device = s->device;
  sp->stream = st;
  sp->major = major;
  const bool cms = major == GPA_SPARSE_CMS;
  sp->n_planes = cms ? C : P;
  const uint64_t cells = cms ? (uint64_t)C * GPA_SLOTS : (uint64_t)P * C;
  auto alloc = [&](void **p, size_t bytes) {
    cudaError_t e = pool_alloc(p, bytes ? bytes : 8, st);
    if (e == cudaSuccess) sp->allocs.push_back(*p);
    return e;
  };
#define SC(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      gpa_status r_ = fail(e_ == cudaErrorMemoryAllocation ? GPA_ERR_OUT_OF_MEMORY : GPA_ERR_CUDA, "%s: %s", \
                           #call, cudaGetErrorString(e_));                                \
      cudaGetLastError();                                                                 \
      free_sparse(sp);                                                                    \
      return r_;                                                                          \
    }                                                                                     \
  } while (0)
  uint32_t *ov = nullptr, *oi = nullptr, *bs = nullptr;
  unsigned long long *tot = nullptr;
  SC(alloc((void **)&ov, cells * 4));
  SC(alloc((void **)&oi, cells * 4));
  SC(alloc((void **)&bs, kScanScratchWords * 4));
  SC(alloc((void **)&tot, 16));
  SC(alloc((void **)&sp->plane_off, (sp->n_planes + 1) * 8));
  SC(alloc((void **)&sp->index_off, (sp->n_planes + 1) * 8));
  if (cells == 0) {  // no function rows: every plane is empty except for its sentinel
    free_sparse(sp);
    return fail(GPA_ERR_UNSUPPORTED, "no function rows to encode");
  }
  SC(sparse_count(d_prof_hist, P, C, cms, ov, oi, bs, tot, st));
  unsigned long long h_tot[2] = {0, 0};
  SC(cudaMemcpyAsync(h_tot, tot, sizeof(h_tot), cudaMemcpyDeviceToHost, st));
  SC(cudaStreamSynchronize(st));
  sp->n_values = h_tot[0];
  sp->n_index = h_tot[1];
  SC(alloc((void **)&sp->vals, sp->n_values * 8));
  SC(alloc((void **)&sp->ids, sp->n_values * 4));
  SC(alloc((void **)&sp->index_start, sp->n_index * 8));
  SC(alloc((void **)&sp->index_id, sp->n_index * 4));
  SC(sparse_write(d_prof_hist, P, C, cms, ov, oi, tot, sp->plane_off, sp->index_off, sp->vals, sp->ids,
                  sp->index_start, sp->index_id, st));
#undef SC
  *out = sp;
  return GPA_OK;
}

gpa_status gpa_get_sparse_view(gpa_sparse sp, gpa_sparse_view *v) {
  if (!sp || !v) return fail(GPA_ERR_INVALID_ARG, "NULL argument");
  v->major = sp->major; v->n_planes = sp->n_planes; v->n_values = sp->n_values; v->n_index = sp->n_index;
  v->plane_off = sp->plane_off; v->index_off = sp->index_off; v->vals = sp->vals; v->ids = sp->ids;
  v->index_start = sp->index_start; v->index_id = sp->index_id;
  return GPA_OK;
}

void gpa_free_sparse(gpa_sparse sp) { free_sparse(sp); }

gpa_status gpa_block_counts(gpa_structure s, uint32_t n_blocks, const uint32_t *d_block_start,
                            const uint64_t *d_counts, uint64_t *d_inst_hist, gpa_stream_t stream) {
  if (!s) return fail(GPA_ERR_INVALID_ARG, "structure is NULL");
  if (n_blocks == 0) return GPA_OK;
  if (!d_block_start || !d_counts || !d_inst_hist) return fail(GPA_ERR_INVALID_ARG, "NULL buffer");
  DeviceGuard g(s->device);
  CU(g.err);
  CU(launch_block_counts(n_blocks, d_block_start, d_counts, s->info.n_inst, d_inst_hist, (cudaStream_t)stream));
  return GPA_OK;
}

gpa_status gpa_reconstruct_cct(gpa_structure s, const uint64_t *d_inst_hist, gpa_weight_mode mode,
                               uint64_t max_contexts, gpa_cct *out, uint64_t *n_contexts, gpa_stream_t stream) {
  if (s && !d_inst_hist && s->info.n_inst) return fail(GPA_ERR_INVALID_ARG, "d_inst_hist is NULL");
  if ((uintptr_t)d_inst_hist & 15) return fail(GPA_ERR_INVALID_ARG, "d_inst_hist must be 16-byte aligned");
  return reconstruct(s, true, d_inst_hist, nullptr, nullptr, mode, max_contexts, out, n_contexts, stream);
}

gpa_status gpa_reconstruct_cct_async(gpa_structure s, const uint64_t *d_inst_hist, gpa_weight_mode mode, gpa_cct *out,
                                     uint64_t *capacity, gpa_stream_t stream) {
  if (s && !d_inst_hist && s->info.n_inst) return fail(GPA_ERR_INVALID_ARG, "d_inst_hist is NULL");
  if ((uintptr_t)d_inst_hist & 15) return fail(GPA_ERR_INVALID_ARG, "d_inst_hist must be 16-byte aligned");
  if (!out || !capacity) return fail(GPA_ERR_INVALID_ARG, "NULL argument");
  return reconstruct(s, true, d_inst_hist, nullptr, nullptr, mode, ~0ull, out, capacity, stream, true);
}

gpa_status gpa_cct_finish(gpa_cct c, uint64_t *n_contexts, int *rebuilt) {
  if (!c || !n_contexts) return fail(GPA_ERR_INVALID_ARG, "NULL argument");
  if (rebuilt) *rebuilt = 0;
  if (!c->pending) {
    *n_contexts = c->n;
    return GPA_OK;
  }
  DeviceGuard g(c->device);
  CU(g.err);
  unsigned long long built = 0;
  CU(cudaMemcpyAsync(&built, c->d_built, sizeof built, cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (built <= c->n) {
    c->n = built;
    c->pending = false;
    *n_contexts = built;
    return GPA_OK;
  }
  if (c->src->info.cct_path_bound <= c->n)
    return fail(GPA_ERR_INTERNAL, "tree exceeds the static bound %llu", (unsigned long long)c->n);
  // the one-launch build did not fit its capacity: the counted build, on the same inputs and stream
  gpa_cct c2 = nullptr;
  uint64_t n2 = 0;
  CHECK(reconstruct(c->src, true, c->src_hist, nullptr, nullptr, (gpa_weight_mode)c->src_mode, ~0ull, &c2, &n2,
                    c->stream));
  std::swap(*c, *c2);
  free_cct(c2);  // the arrays of the pending build
  *n_contexts = c->n;
  if (rebuilt) *rebuilt = 1;
  return GPA_OK;
}

gpa_status gpa_get_cct_view(gpa_cct c, gpa_cct_view *v) {
  if (!c || !v) return fail(GPA_ERR_INVALID_ARG, "NULL argument");
  if (c->pending) return fail(GPA_ERR_INVALID_ARG, "asynchronous tree: call gpa_cct_finish first");
  v->n = c->n;
  v->parent = c->parent; v->site = c->site; v->node = c->node; v->kind = c->kind;
  v->first_child = c->first_child; v->n_children = c->n_children;
  v->frac = c->frac; v->excl = c->excl; v->incl = c->incl;
  v->n_call = c->n_call; v->n_func = c->n_func; v->n_dag = c->n_dag;
  v->call_weight = c->w; v->dag_weight = c->W; v->dag_active = c->dag_active;
  v->func_active = c->func_active; v->func_hist = c->S_f;
  return GPA_OK;
}

void gpa_free_cct(gpa_cct c) { free_cct(c); }

// ---- a-5 + a-10 -------------------------------------------------------------------------
gpa_status gpa_derive_metrics(gpa_structure s, gpa_scope scope, const uint64_t *d_inst_hist, gpa_cct cct,
                              uint64_t *d_scope_hist, uint64_t *d_scope_mix, double *d_metrics,
                              gpa_stream_t stream) {
  if (!s) return fail(GPA_ERR_INVALID_ARG, "structure is NULL");
  DeviceGuard g(s->device);
  CU(g.err);
  cudaStream_t st = (cudaStream_t)stream;
  if (scope == GPA_SCOPE_CCT_EXCL || scope == GPA_SCOPE_CCT_INCL) {
    if (!cct) return fail(GPA_ERR_INVALID_ARG, "CCT scope without a cct");
    if (d_scope_hist || d_scope_mix) return fail(GPA_ERR_INVALID_ARG, "CCT rows have no u64 histogram or mix");
    if (!d_metrics || cct->n == 0) return GPA_OK;
    // a pending (asynchronous) tree: rows = the size on the device, d_metrics holds the capacity
    CU(launch_derive_f64(scope == GPA_SCOPE_CCT_EXCL ? cct->excl : cct->incl, cct->n, d_metrics, st,
                         cct->pending ? cct->d_built : nullptr));
    return GPA_OK;
  }
  int k = scope == GPA_SCOPE_LINE ? ROLL_LINE : scope == GPA_SCOPE_LOOP ? ROLL_LOOP
        : scope == GPA_SCOPE_INLINE ? ROLL_INLINE : scope == GPA_SCOPE_FUNC ? ROLL_FUNC
        : scope == GPA_SCOPE_INST ? -1 : -2;
  if (k == -2) return fail(GPA_ERR_INVALID_ARG, "unknown scope %d", (int)scope);
  uint32_t rows = k < 0 ? s->info.n_inst : s->roll[k].rows;
  if (rows == 0 || (!d_scope_hist && !d_scope_mix && !d_metrics)) return GPA_OK;
  if (!d_inst_hist) return fail(GPA_ERR_INVALID_ARG, "d_inst_hist is NULL");
  if (((uintptr_t)d_inst_hist | (uintptr_t)d_scope_hist | (uintptr_t)d_scope_mix) & 15)
    return fail(GPA_ERR_INVALID_ARG, "histogram buffers must be 16-byte aligned");
  if ((uintptr_t)d_metrics & 7) return fail(GPA_ERR_INVALID_ARG, "d_metrics must be 8-byte aligned");
  CU(launch_rollup(k < 0 ? nullptr : &s->roll[k], rows, d_inst_hist, s->d_inst_class, d_scope_hist, d_scope_mix,
                   d_metrics, sm_count(s->device), st));
  return GPA_OK;
}


// ---- reusable attribution plans (gpa_attr_plan_*) -------------------------------------------------
struct gpa_attr_plan_s {
  int device = 0;
  const gpa_structure_s *s = nullptr;
  AttrPlan p;
  void *mem = nullptr;
};

gpa_status gpa_attr_plan_create(gpa_structure s, const gpa_sample *d_samples, uint64_t n, gpa_attr_plan *out,
                                gpa_stream_t stream) {
  if (!s || !out || (n && !d_samples)) return fail(GPA_ERR_INVALID_ARG, "NULL argument");
  if ((uintptr_t)d_samples & 15) return fail(GPA_ERR_INVALID_ARG, "d_samples is not 16-byte aligned");
  *out = nullptr;
  DeviceGuard g(s->device);
  CU(g.err);
  if (n) CHECK(check_dev_ptr(d_samples, s->device, "d_samples"));
  gpa_attr_plan_s *pl = new gpa_attr_plan_s();
  pl->device = s->device;
  pl->s = s;
  // the structure's large-call kernel (gpa_set_attr_kernel numbering); none for small samples or
  // structures without one (planned calls then run gpa_attribute_samples)
  const int v = attr_choice(s->attr, ~0ull >> 8);
  if ((v == 7 || v == 8 || v == 9) && n >= 4096) {
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaMalloc(&pl->mem, plan_bytes(s->attr, v));
    if (e == cudaSuccess) e = plan_build(s->attr, v, reinterpret_cast<const uint4 *>(d_samples), n, pl->mem, &pl->p,
                                         sm_count(s->device), st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      if (pl->mem) cudaFree(pl->mem);
      delete pl;
      cudaGetLastError();
      return fail(e == cudaErrorMemoryAllocation ? GPA_ERR_OUT_OF_MEMORY : GPA_ERR_CUDA, "gpa_attr_plan_create: %s",
                  cudaGetErrorString(e));
    }
  }
  *out = pl;
  return GPA_OK;
}

gpa_status gpa_attr_plan_variant(gpa_attr_plan p, int *which) {
  if (!p || !which) return fail(GPA_ERR_INVALID_ARG, "NULL argument");
  *which = p->p.variant;
  return GPA_OK;
}

gpa_status gpa_attribute_samples_planned(gpa_structure s, gpa_attr_plan p, const gpa_sample *d_samples, uint64_t n,
                                         uint64_t *d_inst_hist, uint64_t *d_unattributed, uint32_t *d_rec_inst,
                                         gpa_stream_t stream) {
  if (!s || !p) return fail(GPA_ERR_INVALID_ARG, "structure or plan is NULL");
  if (p->s != s) return fail(GPA_ERR_INVALID_ARG, "the plan was made for another structure");
  if (p->p.variant == 0) return gpa_attribute_samples(s, d_samples, n, d_inst_hist, d_unattributed, d_rec_inst, stream);
  if (n == 0) return GPA_OK;
  if (!d_samples || !d_unattributed || (!d_inst_hist && s->info.n_inst))
    return fail(GPA_ERR_INVALID_ARG, "NULL buffer with n=%llu", (unsigned long long)n);
  if ((uintptr_t)d_samples & 15) return fail(GPA_ERR_INVALID_ARG, "d_samples is not 16-byte aligned");
  DeviceGuard g(s->device);
  CU(g.err);
  CHECK(check_dev_ptr(d_samples, s->device, "d_samples"));
  CHECK(check_dev_ptr(d_unattributed, s->device, "d_unattributed"));
  if (d_inst_hist) CHECK(check_dev_ptr(d_inst_hist, s->device, "d_inst_hist"));
  if (d_rec_inst) CHECK(check_dev_ptr(d_rec_inst, s->device, "d_rec_inst"));
  cudaStream_t st = (cudaStream_t)stream;
  const int sm = sm_count(s->device);
  AttrAcc a;
  CU(plan_begin(p->p, &a, sm, st));
  cudaError_t e = plan_run(s->attr, p->p, a, reinterpret_cast<const uint4 *>(d_samples), n, d_rec_inst, sm, st);
  cudaError_t e2 = plan_end(s->attr, p->p, &a, (unsigned long long *)d_inst_hist,
                            (unsigned long long *)d_unattributed, sm, st);
  CU(e);
  CU(e2);
  return GPA_OK;
}

void gpa_attr_plan_free(gpa_attr_plan p) {
  if (!p) return;
  DeviceGuard g(p->device);
  if (p->mem) cudaFree(p->mem);
  delete p;
}

// ---- per-profile trees unified by call path (f1 extension, reading R30) ------------------------
static void free_cct_multi(gpa_cct_multi_s *m) {
  if (!m) return;
  DeviceGuard g(m->device);
  for (void *p : m->allocs)
    if (cudaFreeAsync(p, m->stream) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(p);
    }
  const int dev = m->device;
  delete m;
  pool_trim(dev);
}

static cudaError_t calloc_multi_bytes(gpa_cct_multi_s *m, void **p, size_t bytes) {
  *p = nullptr;
  cudaError_t e = pool_alloc(p, bytes ? bytes : 1, m->stream);
  if (e != cudaSuccess) return e;
  m->allocs.push_back(*p);
  return cudaMemsetAsync(*p, 0, bytes ? bytes : 1, m->stream);
}
#define calloc_multi(m, pp, n) calloc_multi_bytes((m), (void **)(pp), sizeof(**(pp)) * (size_t)(n))

gpa_status gpa_profile_call_weights(gpa_structure s, const gpa_sample *d_samples, uint64_t n, uint32_t n_profiles,
                                    uint64_t *d_prof_call_weight, gpa_stream_t stream) {
  if (!s) return fail(GPA_ERR_INVALID_ARG, "structure is NULL");
  if (n == 0 || s->info.n_call == 0) return GPA_OK;
  if (!d_samples || !d_prof_call_weight) return fail(GPA_ERR_INVALID_ARG, "NULL buffer");
  if ((uintptr_t)d_samples & 15) return fail(GPA_ERR_INVALID_ARG, "d_samples is not 16-byte aligned");
  if (n_profiles > 65535) return fail(GPA_ERR_INVALID_ARG, "n_profiles %u > 65535", n_profiles);
  DeviceGuard g(s->device);
  CU(g.err);
  CHECK(check_dev_ptr(d_samples, s->device, "d_samples"));
  CHECK(check_dev_ptr(d_prof_call_weight, s->device, "d_prof_call_weight"));
  CU(launch_prof_call_weights(s->attr, s->d_inst_call, d_samples, n, n_profiles, s->info.n_call,
                              (unsigned long long *)d_prof_call_weight, sm_count(s->device), (cudaStream_t)stream));
  return GPA_OK;
}

gpa_status gpa_reconstruct_cct_per_profile(gpa_structure s, const uint64_t *d_prof_func_hist,
                                           const uint64_t *d_prof_call_weight, uint32_t n_profiles,
                                           gpa_weight_mode mode, uint64_t max_contexts, gpa_cct_multi *out,
                                           uint64_t *n_contexts, gpa_stream_t stream) {
  if (!s || !out || !n_contexts) return fail(GPA_ERR_INVALID_ARG, "NULL argument");
  if (mode != GPA_WEIGHTS_SAMPLES && mode != GPA_WEIGHTS_EXACT) return fail(GPA_ERR_INVALID_ARG, "mode %d", (int)mode);
  const gpa_structure_info &I = s->info;
  const uint32_t P = n_profiles;
  if (P == 0 || P > 65535) return fail(GPA_ERR_INVALID_ARG, "n_profiles %u (1..65535)", P);
  if ((!d_prof_func_hist && I.n_func) || (!d_prof_call_weight && I.n_call)) return fail(GPA_ERR_INVALID_ARG, "NULL buffer");
  if ((uintptr_t)d_prof_func_hist & 15) return fail(GPA_ERR_INVALID_ARG, "d_prof_func_hist must be 16-byte aligned");
  *out = nullptr;
  *n_contexts = 0;
  DeviceGuard g(s->device);
  CU(g.err);
  cudaStream_t st = (cudaStream_t)stream;
  PoolScratch mem(st);
  const uint32_t nf = I.n_func, nc = I.n_call, nd = I.n_dag;
  // Steps 1-2 + guard + W of every profile (its own tree's inputs); w is rewritten by Step 2
  uint64_t *w = nullptr, *W = nullptr, *S_u = nullptr, *w_u = nullptr;
  uint8_t *fact = nullptr, *dact = nullptr;
  unsigned long long *d_cnt = nullptr;
  CU(mem.get(&w, (uint64_t)P * nc));
  CU(mem.get(&W, (uint64_t)P * nd));
  const uint64_t fs = (nf + 7ull) & ~7ull, ds = (nd + 7ull) & ~7ull;
  CU(mem.get(&fact, (uint64_t)P * fs));
  CU(mem.get(&dact, (uint64_t)P * ds));
  CU(mem.get(&S_u, (uint64_t)nf * SLOTS));
  CU(mem.get(&w_u, nc));
  CU(mem.get(&d_cnt, 4));
  if (nc) CU(cudaMemcpyAsync(w, d_prof_call_weight, sizeof(uint64_t) * P * nc, cudaMemcpyDeviceToDevice, st));
  // one block per profile (fact / dact rows padded to 8 bytes: the byte flags are set with word atomics)
  CU(launch_cct_propagate(s, d_prof_func_hist, w, fact, dact, W, d_cnt, mode == GPA_WEIGHTS_EXACT, false, st, P, fs, ds));
  // the union tree: activity and weighted edges of any profile (structure only: sample weights)
  CU(launch_union_inputs(s, P, fact, fs, dact, ds, w, S_u, w_u, st));
  gpa_cct sup = nullptr;
  uint64_t n_sup = 0;
  // the union tree holds every profile's tree; count-only calls still need it built
  CHECK(reconstruct(s, false, nullptr, S_u, w_u, GPA_WEIGHTS_SAMPLES, max_contexts ? max_contexts : kScanMaxWords, &sup, &n_sup,
                    stream));
  struct SupGuard {
    gpa_cct c;
    ~SupGuard() { free_cct(c); }
  } sg{sup};
  gpa_status r = cct_levels(sup);
  if (r != GPA_OK) return r;
  if (n_sup > kScanMaxWords) return fail(GPA_ERR_CAPACITY, "%llu union contexts", (unsigned long long)n_sup);
  if (n_sup == 0) {
    if (max_contexts) {
      gpa_cct_multi_s *m = new gpa_cct_multi_s();
      m->device = s->device;
      m->stream = st;
      m->n_profiles = P;
      *out = m;
    }
    return GPA_OK;
  }
  uint8_t *pres = nullptr;
  double *frac = nullptr;
  uint32_t *uid = nullptr, *scan_scratch = nullptr;
  CU(mem.get(&pres, n_sup * P));
  CU(mem.get(&frac, n_sup * P));
  CU(mem.get(&uid, n_sup + 1));
  CU(mem.get(&scan_scratch, kScanScratchWords));
  CU(launch_multi_tree(s, sup, P, d_prof_func_hist, w, W, dact, ds, pres, frac, uid, scan_scratch, d_cnt + 1, st));
  unsigned long long n_u = 0;
  CU(cudaMemcpyAsync(&n_u, d_cnt + 1, sizeof(n_u), cudaMemcpyDeviceToHost, st));
  // unified level starts: the scan value at every union-level start
  std::vector<uint32_t> lv(sup->level_start.size(), 0);
  for (size_t L = 0; L + 1 < sup->level_start.size(); L++)
    CU(cudaMemcpyAsync(&lv[L], uid + sup->level_start[L], 4, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  *n_contexts = n_u;
  if (max_contexts == 0) return GPA_OK;
  if (n_u > max_contexts)
    return fail(GPA_ERR_CAPACITY, "%llu contexts > max_contexts %llu", n_u, (unsigned long long)max_contexts);
  gpa_cct_multi_s *m = new gpa_cct_multi_s();
  m->device = s->device;
  m->stream = st;
  m->n = n_u;
  m->n_profiles = P;
  if (!lv.empty()) lv.back() = (uint32_t)n_u;
  for (uint32_t v : lv) m->level_start.push_back(v);
#define CM(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      free_cct_multi(m);                                                                  \
      cudaGetLastError();                                                                 \
      return fail(e_ == cudaErrorMemoryAllocation ? GPA_ERR_OUT_OF_MEMORY : GPA_ERR_CUDA, \
                  "%s: %s", #call, cudaGetErrorString(e_));                               \
    }                                                                                     \
  } while (0)
  CM(calloc_multi(m, &m->parent, n_u));
  CM(calloc_multi(m, &m->site, n_u));
  CM(calloc_multi(m, &m->node, n_u));
  CM(calloc_multi(m, &m->first_child, n_u));
  CM(calloc_multi(m, &m->n_children, n_u));
  CM(calloc_multi(m, &m->kind, n_u));
  CM(calloc_multi(m, &m->frac, n_u * P));
  CM(calloc_multi(m, &m->excl, n_u * P * SLOTS));
  CM(calloc_multi(m, &m->incl, n_u * P * SLOTS));
  CM(launch_multi_compact(sup, P, pres, uid, frac, m, st));
  CM(launch_multi_values(s, m, d_prof_func_hist, st));
#undef CM
  *out = m;
  return GPA_OK;
}

gpa_status gpa_get_cct_multi_view(gpa_cct_multi m, gpa_cct_multi_view *v) {
  if (!m || !v) return fail(GPA_ERR_INVALID_ARG, "NULL argument");
  v->n = m->n;
  v->n_profiles = m->n_profiles;
  v->parent = m->parent; v->site = m->site; v->node = m->node; v->kind = m->kind;
  v->first_child = m->first_child; v->n_children = m->n_children;
  v->frac = m->frac; v->excl = m->excl; v->incl = m->incl;
  return GPA_OK;
}

void gpa_free_cct_multi(gpa_cct_multi m) { free_cct_multi(m); }

// ---- distributed statistics: function-aligned instruction ranges ------------------
static gpa_status partition_bounds(uint32_t ni, const std::vector<uint32_t> &starts, bool contig, uint32_t n_parts,
                                   uint32_t *bounds) {
  if (!contig) return fail(GPA_ERR_STRUCTURE, "a function's instructions are not contiguous: no function-aligned split");
  bounds[0] = 0;
  for (uint32_t r = 1; r < n_parts; r++) {
    const uint64_t target = (uint64_t)ni * r / n_parts;
    // the function start nearest to the even split point, never before the previous bound
    auto it = std::lower_bound(starts.begin(), starts.end(), (uint32_t)target);
    uint32_t b = it == starts.end() ? ni : *it;
    if (it != starts.begin() && target - *(it - 1) < (uint64_t)b - target) b = *(it - 1);
    bounds[r] = std::max(b, bounds[r - 1]);
  }
  bounds[n_parts] = ni;
  return GPA_OK;
}

gpa_status gpa_partition_structure(const gpa_structure_desc *desc, uint32_t n_parts, uint32_t *h_inst_bounds) {
  if (!h_inst_bounds || n_parts == 0) return fail(GPA_ERR_INVALID_ARG, "n_parts must be > 0 with a bounds array");
  Derived dv;
  CHECK(validate(desc, &dv));
  const uint32_t ni = desc->n_inst, nf = desc->n_func;
  std::vector<uint32_t> lo(nf, ni), hi(nf, 0), cnt(nf, 0);
  for (uint32_t i = 0; i < ni; i++) {
    const uint32_t f = dv.inst_func[i];
    lo[f] = std::min(lo[f], i);
    hi[f] = std::max(hi[f], i);
    cnt[f]++;
  }
  bool contig = true;
  std::vector<uint32_t> starts;
  for (uint32_t f = 0; f < nf; f++) {
    contig = contig && (cnt[f] == 0 || hi[f] - lo[f] + 1 == cnt[f]);
    if (cnt[f]) starts.push_back(lo[f]);
  }
  std::sort(starts.begin(), starts.end());
  return partition_bounds(ni, starts, contig, n_parts, h_inst_bounds);
}

// [lo, hi) must be function-aligned: each end 0, n_inst or the first instruction of a function
static gpa_status check_range(gpa_structure s, uint32_t lo, uint32_t hi) {
  if (!s->funcs_contiguous) return fail(GPA_ERR_STRUCTURE, "functions are not contiguous: no instruction-range statistics");
  const uint32_t ni = s->info.n_inst;
  auto aligned = [&](uint32_t x) {
    return x == 0 || x == ni || std::binary_search(s->h_func_starts.begin(), s->h_func_starts.end(), x);
  };
  if (lo > hi || hi > ni || !aligned(lo) || !aligned(hi))
    return fail(GPA_ERR_INVALID_ARG, "instruction range [%u, %u) is not function-aligned in [0, %u]", lo, hi, ni);
  return GPA_OK;
}

// chunk / multi-row runs of roll-up kind k whose function starts in [lo, hi) (hi == n_inst: to the end,
// including functions without instructions)
static void range_runs(const RollSet &R, uint32_t lo, uint32_t hi, uint32_t ni, uint32_t *c0, uint32_t *c1,
                       uint32_t *m0, uint32_t *m1) {
  auto lb = [](const std::vector<uint32_t> &v, uint32_t x) {
    return (uint32_t)(std::lower_bound(v.begin(), v.end(), x) - v.begin());
  };
  *c0 = lb(R.h_chunk_key, lo);
  *c1 = hi >= ni ? (uint32_t)R.h_chunk_key.size() : lb(R.h_chunk_key, hi);
  *m0 = lb(R.h_multi_key, lo);
  *m1 = hi >= ni ? (uint32_t)R.h_multi_key.size() : lb(R.h_multi_key, hi);
}

gpa_status gpa_derive_metrics_range(gpa_structure s, gpa_scope scope, const uint64_t *d_inst_hist, uint32_t inst_lo,
                                    uint32_t inst_hi, uint64_t *d_scope_hist, uint64_t *d_scope_mix, double *d_metrics,
                                    gpa_stream_t stream) {
  if (!s) return fail(GPA_ERR_INVALID_ARG, "structure is NULL");
  int k = scope == GPA_SCOPE_LINE ? ROLL_LINE : scope == GPA_SCOPE_LOOP ? ROLL_LOOP
        : scope == GPA_SCOPE_INLINE ? ROLL_INLINE : scope == GPA_SCOPE_FUNC ? ROLL_FUNC
        : scope == GPA_SCOPE_INST ? -1 : -2;
  if (k == -2) return fail(GPA_ERR_INVALID_ARG, "scope %d has no instruction-range rows", (int)scope);
  CHECK(check_range(s, inst_lo, inst_hi));
  if (!d_scope_hist && !d_scope_mix && !d_metrics) return GPA_OK;
  if (!d_inst_hist) return fail(GPA_ERR_INVALID_ARG, "d_inst_hist is NULL");
  if (((uintptr_t)d_inst_hist | (uintptr_t)d_scope_hist | (uintptr_t)d_scope_mix) & 15)
    return fail(GPA_ERR_INVALID_ARG, "histogram buffers must be 16-byte aligned");
  if ((uintptr_t)d_metrics & 7) return fail(GPA_ERR_INVALID_ARG, "d_metrics must be 8-byte aligned");
  DeviceGuard g(s->device);
  CU(g.err);
  cudaStream_t st = (cudaStream_t)stream;
  if (k < 0) {  // INST rows = the range's instructions
    if (inst_hi == inst_lo) return GPA_OK;
    CU(launch_rollup(nullptr, inst_hi - inst_lo, d_inst_hist + (uint64_t)inst_lo * SLOTS, s->d_inst_class + inst_lo,
                     d_scope_hist ? d_scope_hist + (uint64_t)inst_lo * SLOTS : nullptr,
                     d_scope_mix ? d_scope_mix + (uint64_t)inst_lo * SLOTS : nullptr,
                     d_metrics ? d_metrics + (uint64_t)inst_lo * NCOLS : nullptr, sm_count(s->device), st));
    return GPA_OK;
  }
  uint32_t c0, c1, m0, m1;
  range_runs(s->roll[k], inst_lo, inst_hi, s->info.n_inst, &c0, &c1, &m0, &m1);
  CU(launch_rollup(&s->roll[k], s->roll[k].rows, d_inst_hist, s->d_inst_class, d_scope_hist, d_scope_mix, d_metrics,
                   sm_count(s->device), st, c0, c1, m0, m1));
  return GPA_OK;
}

gpa_status gpa_derive_scopes(gpa_structure s, const uint64_t *d_inst_hist, uint32_t inst_lo, uint32_t inst_hi,
                             const gpa_scope_out *outs, gpa_stream_t stream) {
  if (!s || !outs) return fail(GPA_ERR_INVALID_ARG, "NULL argument");
  const uint32_t ni = s->info.n_inst;
  const bool whole = inst_lo == 0 && inst_hi == ni;
  if (!whole) CHECK(check_range(s, inst_lo, inst_hi));
  else if (inst_lo > inst_hi) return fail(GPA_ERR_INVALID_ARG, "bad range");
  uint64_t *hist[5], *mix[5];
  double *met[5];
  bool any = false;
  for (int k = 0; k < 5; k++) {
    hist[k] = outs[k].scope_hist;
    mix[k] = outs[k].scope_mix;
    met[k] = outs[k].metrics;
    if (((uintptr_t)hist[k] | (uintptr_t)mix[k]) & 15)
      return fail(GPA_ERR_INVALID_ARG, "histogram buffers must be 16-byte aligned");
    if ((uintptr_t)met[k] & 7) return fail(GPA_ERR_INVALID_ARG, "metrics buffers must be 8-byte aligned");
    any = any || hist[k] || mix[k] || met[k];
  }
  if (!any) return GPA_OK;
  if (!d_inst_hist && ni) return fail(GPA_ERR_INVALID_ARG, "d_inst_hist is NULL");
  if ((uintptr_t)d_inst_hist & 15) return fail(GPA_ERR_INVALID_ARG, "d_inst_hist must be 16-byte aligned");
  DeviceGuard g(s->device);
  CU(g.err);
  const MultiRoll &M = s->multi;
  uint32_t c0 = 0, c1 = M.n_chunks, m0 = 0, m1 = M.n_multi;
  if (!whole) {
    auto lb = [](const std::vector<uint32_t> &v, uint32_t x) {
      return (uint32_t)(std::lower_bound(v.begin(), v.end(), x) - v.begin());
    };
    c0 = lb(M.h_chunk_key, inst_lo);
    c1 = inst_hi >= ni ? M.n_chunks : lb(M.h_chunk_key, inst_hi);
    m0 = lb(M.h_multi_key, inst_lo);
    m1 = inst_hi >= ni ? M.n_multi : lb(M.h_multi_key, inst_hi);
  }
  bool tree = false;
  for (int k = 1; k < 5; k++) tree = tree || hist[k] || mix[k] || met[k];
  if (!tree) c0 = c1 = m0 = m1 = 0;
  const bool inst = hist[0] || mix[0] || met[0];
  CU(launch_rollup_multi(M, c0, c1, m0, m1, inst_lo, inst ? inst_hi - inst_lo : 0, d_inst_hist, s->d_inst_class, hist,
                         mix, met, sm_count(s->device), (cudaStream_t)stream));
  return GPA_OK;
}

gpa_status gpa_cct_inputs(gpa_structure s, const uint64_t *d_inst_hist, uint32_t inst_lo, uint32_t inst_hi,
                          uint64_t *d_func_hist, uint64_t *d_call_weight, gpa_stream_t stream) {
  if (!s) return fail(GPA_ERR_INVALID_ARG, "structure is NULL");
  CHECK(check_range(s, inst_lo, inst_hi));
  if ((!d_inst_hist && s->info.n_inst) || (!d_func_hist && s->info.n_func) || (!d_call_weight && s->info.n_call))
    return fail(GPA_ERR_INVALID_ARG, "NULL buffer");
  if (((uintptr_t)d_inst_hist | (uintptr_t)d_func_hist) & 15)
    return fail(GPA_ERR_INVALID_ARG, "histogram buffers must be 16-byte aligned");
  DeviceGuard g(s->device);
  CU(g.err);
  cudaStream_t st = (cudaStream_t)stream;
  uint32_t c0, c1, m0, m1;
  range_runs(s->roll[ROLL_FUNC], inst_lo, inst_hi, s->info.n_inst, &c0, &c1, &m0, &m1);
  CU(launch_rollup(&s->roll[ROLL_FUNC], s->roll[ROLL_FUNC].rows, d_inst_hist, s->d_inst_class, d_func_hist, nullptr,
                   nullptr, sm_count(s->device), st, c0, c1, m0, m1));
  CU(launch_cct_weights_range(s, d_inst_hist, inst_lo, inst_hi, d_call_weight, st));
  return GPA_OK;
}

gpa_status gpa_reconstruct_cct_inputs(gpa_structure s, const uint64_t *d_func_hist, const uint64_t *d_call_weight,
                                      gpa_weight_mode mode, uint64_t max_contexts, gpa_cct *out, uint64_t *n_contexts,
                                      gpa_stream_t stream) {
  if (!s) return fail(GPA_ERR_INVALID_ARG, "structure is NULL");
  if ((!d_func_hist && s->info.n_func) || (!d_call_weight && s->info.n_call))
    return fail(GPA_ERR_INVALID_ARG, "NULL buffer");
  if ((uintptr_t)d_func_hist & 15) return fail(GPA_ERR_INVALID_ARG, "d_func_hist must be 16-byte aligned");
  return reconstruct(s, false, nullptr, d_func_hist, d_call_weight, mode, max_contexts, out, n_contexts, stream);
}
}  // extern "C"
