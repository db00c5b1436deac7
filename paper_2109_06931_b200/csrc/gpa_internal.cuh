// gpa_internal.cuh — internal types shared by the libgpa translation units.
// Public contract: include/gpa.h.  Nothing here is visible across the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <mutex>
#include <string>
#include <vector>

#include "gpa.h"

namespace gpa {

constexpr uint32_t NONE = GPA_NONE;
constexpr int SLOTS = GPA_SLOTS;
constexpr int VALID = GPA_VALID_SLOTS;
constexpr int NCOLS = GPA_NUM_DERIVED;

// roll-up row sets (index into gpa_structure_s::roll)
enum { ROLL_LINE = 0, ROLL_LOOP = 1, ROLL_INLINE = 2, ROLL_FUNC = 3, ROLL_KINDS = 4 };

// Tables the attribution kernel reads (passed by value as a kernel parameter).
// One device block reused by consecutive attribution calls on a structure (the per-call scratch:
// plan, accumulators, CTA slabs), so a call makes no pool allocation: a call on another stream
// than the previous one first waits for that call's event.  A call that finds it busy (another
// host thread) or too small allocates from the pool as before.
struct ScratchCache {
  std::mutex mu;
  void *mem = nullptr;
  size_t bytes = 0;
  bool busy = false;
  cudaStream_t last = nullptr;
  cudaEvent_t done = nullptr;
};
cudaError_t scratch_get(ScratchCache *c, size_t bytes, cudaStream_t st, void **out, bool *cached);
cudaError_t scratch_put(ScratchCache *c, void *p, bool cached, cudaStream_t st);
void scratch_release(ScratchCache *c);

struct AttrTables {
  uint64_t base;          // first instruction start
  uint64_t end;           // last instruction end (exclusive)
  uint32_t gshift;        // granule = 1 << gshift bytes
  uint32_t mode;          // 0 = granule map, 1 = binary search
  uint64_t n_gran;
  const uint32_t *gmap;   // [n_gran] instruction covering each granule, or NONE
  const uint64_t *inst_addr;
  const uint16_t *inst_len;
  uint32_t n_inst;
  ScratchCache *cache;    // host side: the structure's reusable call scratch (never read by kernels)
};

constexpr uint32_t kRollChunk = 32;  // instructions per roll-up work item

struct RollSet {
  uint32_t rows = 0;
  uint32_t *d_ptr = nullptr;    // [rows+1]
  uint32_t *d_inst = nullptr;   // [ptr[rows]]
  std::vector<uint32_t> ids;    // host: scope id (or function id) behind each row
  // work decomposition (load time): rows split into chunks of <= kRollChunk instructions
  uint32_t n_chunks = 0, n_multi = 0;
  uint32_t *d_chunk = nullptr;      // [3*n_chunks] (row, begin, end) into d_inst
  uint32_t *d_multi_slot = nullptr; // [rows] scratch slot of a row with > 1 chunk, else NONE
  uint32_t *d_multi_rows = nullptr; // [n_multi] the rows with > 1 chunk
  // chunks and multi-chunk rows are ordered by their row's function position (the first
  // instruction of the function; n_inst for an empty function), so the rows of the functions
  // inside an instruction range are a contiguous run of each (gpa_derive_metrics_range)
  std::vector<uint32_t> h_chunk_key, h_multi_key;
};

// the four tree kinds merged (gpa_derive_scopes): one chunk list in function order over the
// concatenated instruction lists, multi-chunk rows with merged slots
struct MultiRoll {
  uint32_t n_chunks = 0, n_multi = 0;
  uint32_t *d_chunk = nullptr;   // [4*n_chunks] (kind, row, begin, end); kind 1..4 = LINE, LOOP, INLINE, FUNC
  uint32_t *d_lst = nullptr;     // concatenated instruction lists
  uint32_t *d_mrows = nullptr;   // [2*n_multi] (kind, row)
  uint32_t *d_mslot[5] = {};     // per kind (index 1..4): row -> merged multi slot or NONE; [0] unused
  std::vector<uint32_t> h_chunk_key, h_multi_key;
};

}  // namespace gpa

struct gpa_structure_s {
  int device = 0;
  gpa_structure_info info{};
  gpa::AttrTables attr{};
  gpa::ScratchCache scratch;  // attr.cache
  // device tables
  uint64_t *d_inst_addr = nullptr;
  uint16_t *d_inst_len = nullptr;
  uint8_t *d_inst_class = nullptr;
  uint32_t *d_inst_func = nullptr;  // function of each instruction (per-profile histograms)
  uint32_t *d_inst_call = nullptr;  // call site of each call instruction, NONE elsewhere (per-profile weights)
  uint32_t *d_gfunc = nullptr;      // function of each granule of the pc map (NONE in gaps)
  uint32_t *d_gmap = nullptr;
  gpa::RollSet roll[gpa::ROLL_KINDS];
  gpa::MultiRoll multi;
  // call graph (function level)
  uint32_t *d_call_inst = nullptr, *d_call_callee = nullptr, *d_call_caller = nullptr;
  uint32_t *d_fin_ptr = nullptr, *d_fin_e = nullptr;    // in-edges per function
  uint32_t n_ext_calls = 0;                             // external (cross-DAG-node) call sites
  uint32_t *d_fout_ptr = nullptr, *d_fout_e = nullptr;  // external out-edges per function,
                                                        // ascending call instruction
  // condensed DAG
  uint32_t *d_scc_of = nullptr;                         // [n_func]
  uint32_t *d_din_ptr = nullptr, *d_din_e = nullptr;    // external in-edges per DAG node
  uint32_t *d_dmem_ptr = nullptr, *d_dmem = nullptr;    // members per DAG node (ascending)
  uint8_t *d_dag_nontrivial = nullptr;
  uint32_t *d_dlev_ptr = nullptr, *d_dlev_node = nullptr;  // DAG nodes grouped by level
  std::vector<uint32_t> h_scc_of;
  // function layout in the instruction order: first instruction of each function (n_inst when
  // empty), whether every function's instructions are contiguous, and the sorted function starts
  std::vector<uint32_t> h_func_lo, h_func_starts;
  bool funcs_contiguous = false;
  std::vector<void *> allocs;
};

// f1 extension (R30): per-profile trees unified by call path
struct gpa_cct_multi_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t n = 0;
  uint32_t n_profiles = 0;
  uint32_t *parent = nullptr, *site = nullptr, *node = nullptr, *first_child = nullptr, *n_children = nullptr;
  uint8_t *kind = nullptr;
  double *frac = nullptr, *excl = nullptr, *incl = nullptr;  // [n][P], [n][P][16], [n][P][16]
  std::vector<uint64_t> level_start;
  std::vector<void *> allocs;
};

struct gpa_sparse_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint32_t major = 0, n_planes = 0;
  uint64_t n_values = 0, n_index = 0;
  uint64_t *plane_off = nullptr, *index_off = nullptr, *vals = nullptr, *index_start = nullptr;
  uint32_t *ids = nullptr, *index_id = nullptr;
  std::vector<void *> allocs;
};

struct gpa_cct_s {
  int device = 0;
  cudaStream_t stream = nullptr;  // the build stream: allocations and frees are ordered on it
  uint64_t n = 0;
  uint32_t n_call = 0, n_func = 0, n_dag = 0;
  uint32_t *parent = nullptr, *site = nullptr, *node = nullptr, *first_child = nullptr,
           *n_children = nullptr;
  uint8_t *kind = nullptr;
  double *frac = nullptr, *excl = nullptr, *incl = nullptr;
  uint64_t *w = nullptr, *W = nullptr, *S_f = nullptr;
  uint8_t *dag_active = nullptr, *func_active = nullptr;
  std::vector<uint64_t> level_start;  // contexts of BFS level L: [level_start[L], level_start[L+1])
  // device level table of the one-kernel builds (read back lazily by gpa_cct_profiles):
  // lev_fmt 1 = k_cct_small (lev[0] = levels, lev[1 + l] = first context of level l),
  // lev_fmt 2 = k_cct_coop (lev[l] = first context of level l, up to lev_len entries)
  uint32_t *d_lev = nullptr;
  int lev_fmt = 0;
  uint32_t lev_len = 0;
  std::vector<void *> allocs;
  // gpa_reconstruct_cct_async: built into n (= capacity) slots, the size still on the device
  // (*d_built: contexts, or ~0 when the one-launch build did not fit) until gpa_cct_finish
  bool pending = false;
  unsigned long long *d_built = nullptr;
  gpa_structure src = nullptr;       // the inputs a counted rebuild needs (overflow only)
  const uint64_t *src_hist = nullptr;
  int src_mode = 0;
};

// ---- kernel launch accounting (gpa_kernel_launches) ------------------------------------------
namespace gpa {
void count_launches(uint64_t k);
void set_attr_kernel(int which);
void set_ring_stress(int level);
// Stream-ordered scratch from the library's own memory pool on the current device (release
// threshold = unlimited, so memory freed at one call is reused by the next without going
// back to the driver; the process's default pool is left untouched).
cudaError_t pool_alloc(void **p, size_t bytes, cudaStream_t st);
// scratch words a scan_u32 call (kern_common.cuh) needs: look-back state for up to 2^27
// elements + the tile ticket
constexpr size_t kScanScratchWords = 2 * 32768 + 4;
constexpr uint64_t kScanMaxWords = 1ull << 27;  // the largest scan_u32 input
}

// ---- kernels launchers (k_*.cu) -----------------------------------------------------------
namespace gpa {
int attr_choice(const AttrTables &T, uint64_t n);  // kernel a call of n records runs (gpa_attr_kernel_choice)
bool prof_code_ok(const AttrTables &T, uint64_t n);  // f1 instruction rows through a call plan's hot bins
cudaError_t launch_prof_inst_code(const AttrTables &T, const gpa_sample *d_samples, uint64_t n, uint32_t n_prof,
                                  unsigned long long *PH, unsigned long long *PU, int sm_count, cudaStream_t st);
// attribution plans of the large-call kernels 7 (probe table) and 8 (code map + byte bins), k_attr.cu
struct AttrPlan {
  int variant = 0;
  uint64_t n_gran = 0;
  unsigned long long *best = nullptr;                           // 7: table entries
  uint32_t *bin_of = nullptr, *thr = nullptr, *code = nullptr;  // 8: bins, bin count, code map
};
struct AttrAcc {
  unsigned long long *acc = nullptr, *Hg = nullptr;
  unsigned int *ctr = nullptr;  // dynamic tile counter (reset before every launch)
  uint32_t *dump = nullptr;     // one slab of shared-table words per CTA (flushed by store, folded into acc)
  int slabs = 0;
};
size_t plan_bytes(const AttrTables &T, int variant);
cudaError_t plan_build(const AttrTables &T, int variant, const uint4 *rec, uint64_t n, void *mem, AttrPlan *p,
                       int sm_count, cudaStream_t st);
cudaError_t plan_begin(const AttrPlan &p, AttrAcc *a, int sm_count, cudaStream_t st);
cudaError_t plan_run(const AttrTables &T, const AttrPlan &p, const AttrAcc &a, const uint4 *rec, uint64_t n,
                     uint32_t *ri, int sm_count, cudaStream_t st);
cudaError_t plan_end(const AttrTables &T, const AttrPlan &p, AttrAcc *a, unsigned long long *H, unsigned long long *U,
                     int sm_count, cudaStream_t st);
cudaError_t launch_attribute(const AttrTables &T, const gpa_sample *d_samples, uint64_t n,
                             unsigned long long *d_hist, unsigned long long *d_unattr,
                             uint32_t *d_rec_inst, int sm_count, cudaStream_t st);
// Row-wise roll-up with the fused derived-metric epilogue.  set == nullptr: identity rows
// (row r = instruction r, `rows` rows).
// [c0, c1) / [m0, m1): the chunk and multi-chunk-row runs to process (default: all).
cudaError_t launch_rollup(const RollSet *set, uint32_t rows, const uint64_t *d_hist, const uint8_t *d_class,
                          uint64_t *d_out_hist, uint64_t *d_out_mix, double *d_metrics, int sm_count,
                          cudaStream_t st, uint32_t c0 = 0, uint32_t c1 = 0xFFFFFFFFu, uint32_t m0 = 0,
                          uint32_t m1 = 0xFFFFFFFFu);
// w_e = sum_{r<12} H[call_inst[e]][r] for the call sites whose call instruction lies in [lo, hi)
cudaError_t launch_cct_weights_range(const gpa_structure_s *s, const uint64_t *d_hist, uint32_t lo, uint32_t hi,
                                     uint64_t *d_w, cudaStream_t st);
cudaError_t launch_derive_f64(const double *d_v, uint64_t rows, double *d_metrics, cudaStream_t st,
                              const unsigned long long *d_rows = nullptr);
// all scope kinds in one launch: INST rows [ident_lo, ident_lo + n_ident) and merged chunks [c0, c1),
// multi rows [m0, m1); outputs indexed by gpa_scope (0 INST .. 4 FUNC), NULL = not produced
cudaError_t launch_rollup_multi(const MultiRoll &M, uint32_t c0, uint32_t c1, uint32_t m0, uint32_t m1, uint32_t ident_lo,
                                uint32_t n_ident, const uint64_t *d_hist, const uint8_t *d_class,
                                uint64_t *const hist[5], uint64_t *const mix[5], double *const met[5], int sm_count,
                                cudaStream_t st);

// CCT pieces (k_cct.cu)
cudaError_t launch_cct_weights(const gpa_structure_s *s, const uint64_t *d_hist, uint64_t *d_w,
                               cudaStream_t st);
cudaError_t launch_cct_propagate(const gpa_structure_s *s, const uint64_t *d_S_f, uint64_t *d_w,
                                 uint8_t *d_func_active, uint8_t *d_dag_active, uint64_t *d_W,
                                 unsigned long long *d_count, bool exact, bool count, cudaStream_t st,
                                 uint32_t n_batch = 0, uint64_t fstride = 0, uint64_t dstride = 0);
// per-profile function histograms and cross-profile statistics (k_prof.cu)
cudaError_t launch_attribute_profiles(const AttrTables &T, const uint32_t *d_inst_func, const uint32_t *d_gfunc,
                                      uint32_t n_func,
                                      const gpa_sample *d_samples, uint64_t n, uint32_t n_prof,
                                      unsigned long long *d_ph, unsigned long long *d_pu, int sm_count,
                                      cudaStream_t st);
cudaError_t launch_attribute_profiles_inst(const AttrTables &T, uint32_t n_inst, const gpa_sample *d_samples,
                                           uint64_t n, uint32_t n_prof, unsigned long long *d_ph,
                                           unsigned long long *d_pu, int sm_count, cudaStream_t st);
cudaError_t launch_profile_stats_f64(const double *d_x, uint32_t n_prof, uint64_t rows, double *d_stats,
                                     cudaStream_t st);
cudaError_t launch_cct_prof_excl(const gpa_structure_s *s, const gpa_cct_s *c, const uint64_t *d_ph, uint32_t P1,
                                 double *d_excl, cudaStream_t st);
cudaError_t launch_cct_prof_incl_level(const gpa_cct_s *c, uint64_t a, uint64_t b, uint32_t P1, const double *d_excl,
                                       double *d_incl, cudaStream_t st);
cudaError_t launch_profile_stats(const uint64_t *d_ph, uint32_t n_prof, uint32_t rows, double *d_stats,
                                 cudaStream_t st);
// GPU-idleness blame (k_blame.cu)
constexpr int kMergeChunkHost = 2048;  // outputs per merge CTA tile (k_blame.cu)
struct MergePair {
  uint64_t a0, a1, b1;  // merge [a0, a1) with [a1, b1)
};
struct BlameArgs {
  uint64_t n;
  uint32_t n_scopes, n_routines, kmax;
  const uint32_t *ord;
  const uint64_t *line_off;
  const uint8_t *line_kind;
  const uint32_t *line_scope;
  const uint64_t *time;
  const uint32_t *ctx;
  const uint64_t *st;
  uint32_t *info, *pos /* bpos: first blameable piece at/after each change point */, *delta, *scan, *psc, *bidx, *pk, *bs, *err;
  uint64_t *pdur;
  uint2 *seg, *ovf;
  uint32_t *seg_n;
  unsigned long long *tots, *acc, *num;
  double *blame, *share;
  uint64_t *total, *gpu_idle;
};
cudaError_t blame_prep(const BlameArgs &a, uint32_t n_lines, cudaStream_t st);
cudaError_t blame_merge(const MergePair *pairs, const uint64_t *chunk_start, uint32_t np, uint64_t n_chunks,
                        const uint64_t *st_in, const uint32_t *si, uint64_t *dt, uint32_t *di, uint64_t *split,
                        cudaStream_t st);
cudaError_t blame_sweep(const BlameArgs &a, cudaStream_t st);

// sparse cubes (k_sparse.cu): counts + offsets (tot[0] values, tot[1] index entries), then the write
cudaError_t sparse_count(const uint64_t *H, uint32_t P, uint32_t C, bool cms, uint32_t *ov, uint32_t *oi,
                         uint32_t *bs, unsigned long long *tot, cudaStream_t st);
cudaError_t sparse_write(const uint64_t *H, uint32_t P, uint32_t C, bool cms, const uint32_t *ov, const uint32_t *oi,
                         const unsigned long long *tot, uint64_t *plane_off, uint64_t *index_off, uint64_t *vals,
                         uint32_t *ids, uint64_t *index_start, uint32_t *index_id, cudaStream_t st);
cudaError_t launch_block_counts(uint32_t n_blocks, const uint32_t *d_start, const uint64_t *d_cnt, uint32_t n_inst,
                                uint64_t *d_hist, cudaStream_t st);
cudaError_t launch_cct_roots(const gpa_structure_s *s, const uint8_t *d_dag_active, gpa_cct_s *c,
                             unsigned long long *d_n, cudaStream_t st);
cudaError_t launch_cct_level(const gpa_structure_s *s, gpa_cct_s *c, uint64_t a, uint64_t b,
                             uint32_t *d_tmp, uint32_t *d_blocksum, unsigned long long *d_next,
                             cudaStream_t st);
cudaError_t launch_cct_excl(const gpa_structure_s *s, gpa_cct_s *c, cudaStream_t st);
// whole Step 4 in one CTA when cct_small_ok (writes the built context count to *d_built; ~0 when
// the tree exceeds the c->n allocated slots or the level table)
constexpr uint64_t kSmallContexts = 1ull << 16;
bool cct_small_ok(const gpa_structure_s *s, uint64_t n);
// whole Step 4 in one cooperative grid launch (large trees); d_bsum >= 2*SMs entries
cudaError_t launch_cct_coop(const gpa_structure_s *s, gpa_cct_s *c, uint32_t *d_tmp, uint32_t *d_bsum, uint32_t *d_lev,
                            uint32_t max_lev, unsigned long long *d_built, int sm_count, cudaStream_t st);
cudaError_t launch_cct_small(const gpa_structure_s *s, gpa_cct_s *c, uint32_t *d_lev, unsigned long long *d_built,
                             int sm_count, cudaStream_t st);
cudaError_t launch_cct_incl_level(gpa_cct_s *c, uint64_t a, uint64_t b, cudaStream_t st);
// per-profile trees unified by call path (k_cctp.cu, R30)
cudaError_t launch_prof_call_weights(const AttrTables &T, const uint32_t *inst_call, const gpa_sample *d_samples,
                                     uint64_t n, uint32_t n_prof, uint32_t n_call, unsigned long long *wp,
                                     int sm_count, cudaStream_t st);
cudaError_t launch_union_inputs(const gpa_structure_s *s, uint32_t P, const uint8_t *fact, uint64_t fs,
                                const uint8_t *dact, uint64_t ds, const uint64_t *w, uint64_t *S_u, uint64_t *w_u,
                                cudaStream_t st);
cudaError_t launch_multi_tree(const gpa_structure_s *s, const gpa_cct_s *sup, uint32_t P, const uint64_t *Sp,
                              const uint64_t *w, const uint64_t *W, const uint8_t *dact, uint64_t ds, uint8_t *pres,
                              double *frac, uint32_t *flag, uint32_t *scan_scratch, unsigned long long *d_total, cudaStream_t st);
cudaError_t launch_multi_compact(const gpa_cct_s *sup, uint32_t P, const uint8_t *pres, const uint32_t *uid,
                                 const double *frac, gpa_cct_multi_s *m, cudaStream_t st);
cudaError_t launch_multi_values(const gpa_structure_s *s, gpa_cct_multi_s *m, const uint64_t *Sp, cudaStream_t st);
}  // namespace gpa
