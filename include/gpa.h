/*
 * gpa.h — C ABI of the B200-native GPU PC-sample attribution library (libgpa).
 *
 * Method: Zhou et al., "Measurement and Analysis of GPU-accelerated Applications
 * with HPCToolkit", Parallel Computing 2021 (arXiv 2109.06931).  Citations below
 * are "P:<line>" into /root/reference/PAPER.md (read-only copy of the paper's LaTeX)
 * plus the section they fall in; "Rn" refers to the numbered readings in DESIGN.md
 * §3 where the paper is silent or ambiguous.
 *
 * The library implements the data-parallel analysis path the paper describes:
 *   a-1..a-3  PC-sample decode, pc -> instruction range lookup, per-instruction x
 *             stall-reason histogram                        (§4.2, §4.5 P:475-479,
 *                                                           §5)
 *   a-4       cross-GPU combine (caller: NCCL reduce of the histogram; §5.1)
 *   a-5       roll-up to lines / loops / inlined code / functions  (§5.1)
 *   a-6..a-9  approximate GPU calling-context tree (§5.3, Steps 1-4)
 *   a-10      PC-sample-derived metrics, e.g. Warp Issue Rate W=(S-S_stall)/S (§6.1)
 *
 * Conventions shared by every entry point:
 *  - "d_" pointers are DEVICE pointers on the structure's device; "h_" pointers are host.
 *  - Every call that takes a cudaStream_t only ENQUEUES work on that stream unless its
 *    comment says it synchronizes.  Completion/ordering of caller buffers is the caller's job.
 *  - Errors are status codes; nothing aborts.  gpa_last_error() returns a thread-local
 *    message describing the most recent non-OK status on the calling thread.
 *  - Asynchronous device faults surface as GPA_ERR_CUDA at the next synchronizing call.
 *  - Handles are immutable after creation and may be used concurrently from several
 *    host threads / streams.
 */
#ifndef GPA_H
#define GPA_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define GPA_API __attribute__((visibility("default")))
#else
#define GPA_API
#endif

/* cudaStream_t without pulling in cuda_runtime.h (identical ABI: an opaque pointer). */
typedef struct CUstream_st *gpa_stream_t;

/* ---- constants (readings R2/R3/R5) -------------------------------------- */
#define GPA_SLOTS        16          /* histogram slots per instruction row                  */
#define GPA_VALID_SLOTS  12          /* slots 0..11 = stall reasons (R2); 12..14 always 0     */
#define GPA_SLOT_INVALID 15          /* a record whose stall field is >= 12 lands here (R2)   */
#define GPA_CLASSES      16          /* instruction classes (R5)                       */
#define GPA_NUM_DERIVED  33          /* derived columns per row (R3-R5, DESIGN.md §3 table)    */
#define GPA_NONE         0xFFFFFFFFu /* "no index" in every u32 index array                    */
#define GPA_NUM_STATS    6           /* cross-profile statistics: sum min mean max std cv (R25) */

/* Stall slots, modeled on CUPTI's PC-sampling stall enumeration (R2; the paper only says
 * "a stall reason").  Slot 0 = the warp issued (not stalled); W uses it. */
enum {
  GPA_STALL_NONE = 0, GPA_STALL_INST_FETCH = 1, GPA_STALL_EXEC_DEPENDENCY = 2,
  GPA_STALL_MEMORY_DEPENDENCY = 3, GPA_STALL_TEXTURE = 4, GPA_STALL_SYNC = 5,
  GPA_STALL_CONSTANT_MEMORY_DEPENDENCY = 6, GPA_STALL_PIPE_BUSY = 7,
  GPA_STALL_MEMORY_THROTTLE = 8, GPA_STALL_NOT_SELECTED = 9, GPA_STALL_OTHER = 10,
  GPA_STALL_SLEEPING = 11
};

typedef enum {
  GPA_OK = 0,
  GPA_ERR_INVALID_ARG = 1,   /* NULL pointer with n>0, misaligned sample buffer, bad enum,
                                pointer not on the handle's device                         */
  GPA_ERR_STRUCTURE = 2,     /* gpa_load_structure / gpa_validate_structure: malformed desc */
  GPA_ERR_CAPACITY = 3,      /* gpa_reconstruct_cct: more contexts than max_contexts        */
  GPA_ERR_OUT_OF_MEMORY = 4, /* device or host allocation failed                             */
  GPA_ERR_CUDA = 5,          /* a CUDA runtime call or kernel launch failed                  */
  GPA_ERR_INTERNAL = 6,      /* invariant violated inside the library (a bug)                */
  GPA_ERR_UNSUPPORTED = 7    /* feature not built                                            */
} gpa_status;

/* Scope kinds of the program-structure tree ("procedures, inlined functions,
 * loop nests, and source lines").  FUNCTION scopes are roots; LINE scopes are
 * leaves and every instruction's innermost scope (R7, R8). */
typedef enum { GPA_KIND_FUNCTION = 0, GPA_KIND_INLINE = 1, GPA_KIND_LOOP = 2,
               GPA_KIND_LINE = 3 } gpa_scope_kind;

/* Row sets gpa_derive_metrics can produce. */
typedef enum {
  GPA_SCOPE_INST = 0,     /* one row per instruction (rows = n_inst)                           */
  GPA_SCOPE_LINE = 1,     /* one row per LINE scope, ascending scope id (leaf rows, R8)          */
  GPA_SCOPE_LOOP = 2,     /* one row per LOOP scope, ascending scope id (inclusive, R8)          */
  GPA_SCOPE_INLINE = 3,   /* one row per INLINE scope, ascending scope id (inclusive, R8)        */
  GPA_SCOPE_FUNC = 4,     /* one row per function f (row f = func_scope[f]; inclusive; flat view
                             P:936-937)                                                          */
  GPA_SCOPE_CCT_EXCL = 5, /* one row per CCT context: exclusive apportioned samples  */
  GPA_SCOPE_CCT_INCL = 6  /* one row per CCT context: inclusive (context + descendants)          */
} gpa_scope;

/* CCT context kinds (R14). */
typedef enum { GPA_CTX_FUNC = 0, GPA_CTX_SCC = 1, GPA_CTX_SCC_MEMBER = 2 } gpa_ctx_kind;

/* Step-1 edge weights: call-instruction sample counts, or exact call counts.  With
 * GPA_WEIGHTS_EXACT the histogram holds exact execution counts (instrumentation, P:376-388;
 * see gpa_block_counts) and Step 2 and the DAG guard are skipped ("For call graphs
 * based on samples"; R24): with consistent counts the result equals samples mode. */
typedef enum { GPA_WEIGHTS_SAMPLES = 0, GPA_WEIGHTS_EXACT = 1 } gpa_weight_mode;

/* One PC sample as a sampler delivers it ("an instruction address, a stall
 * reason, and a count").  16 bytes, little-endian, 16-byte aligned (one 128-bit load).
 * pc: relocated module offset (R1).  stall: reason code; >= 12 is invalid data (R2).
 * stream: profile slot (GPU stream / rank); read but not used by the histogram. */
typedef struct {
  uint64_t pc;
  uint32_t count;
  uint16_t stall;
  uint16_t stream;
} gpa_sample;

/* Program structure of ONE load module (R1).  HOST arrays, copied by
 * gpa_load_structure; the caller keeps ownership and may free them after the call.
 * Validation (GPA_ERR_STRUCTURE) rejects: inst_addr not strictly ascending; inst_len == 0;
 * overlapping ranges ([addr,addr+len) must be disjoint, R6) or addr+len overflowing u64;
 * inst_scope not a LINE scope; scope_parent out of range / cyclic; a FUNCTION scope with a
 * parent or a non-FUNCTION scope without one; a LINE scope that is some scope's parent;
 * func_scope not a bijection onto the FUNCTION scopes; call_inst / call_callee out of range;
 * two call sites on the same instruction (direct calls only, R22); inst_class > 15;
 * scope_kind > 3; n_inst > 2^28 - 16. */
typedef struct {
  uint32_t n_inst;
  const uint64_t *inst_addr;    /* [n_inst] strictly ascending relocated start addresses    */
  const uint16_t *inst_len;     /* [n_inst] length in bytes (> 0)                            */
  const uint8_t  *inst_class;   /* [n_inst] class 0..15 (R5)                          */
  const uint32_t *inst_scope;   /* [n_inst] innermost scope, a LINE scope                    */
  uint32_t n_scope;
  const uint32_t *scope_parent; /* [n_scope] parent scope, GPA_NONE for FUNCTION scopes      */
  const uint8_t  *scope_kind;   /* [n_scope] gpa_scope_kind                                  */
  uint32_t n_func;
  const uint32_t *func_scope;   /* [n_func] the FUNCTION scope of function f                 */
  uint32_t n_call;
  const uint32_t *call_inst;    /* [n_call] instruction index of call site e          */
  const uint32_t *call_callee;  /* [n_call] callee function of call site e (direct calls)    */
} gpa_structure_desc;

typedef struct gpa_structure_s *gpa_structure;  /* device-resident, immutable after load */
typedef struct gpa_cct_s *gpa_cct;              /* library-owned CCT result               */

typedef struct {
  uint32_t n_inst, n_scope, n_line, n_loop, n_inline, n_func, n_call;
  uint32_t n_dag;          /* nodes of the SCC-condensed call graph (Step 3)       */
  uint32_t n_scc;          /* non-trivial SCCs (>= 2 members, or a self-call; R14)            */
  uint32_t dag_levels;     /* longest root->node chain in the condensed DAG (+1)              */
  uint64_t cct_path_bound; /* contexts if every call site had weight > 0 (saturating)         */
  uint32_t lookup_mode;    /* 0 = direct granule map, 1 = sorted-range binary search          */
  uint32_t granule_shift;  /* log2 of the granule size of the direct map                      */
  uint64_t lookup_entries; /* entries of the direct map (0 in mode 1)                         */
  uint64_t device_bytes;   /* device memory held by the handle                                */
} gpa_structure_info;

/* Read-only DEVICE views of a CCT (valid until gpa_free_cct).  Contexts are numbered in
 * breadth-first order (R17): roots first (ascending DAG id), then level by level; the
 * children of a context are contiguous, ordered by ascending call instruction (for call
 * children) or ascending member function id (for SCC members). */
typedef struct {
  uint64_t n;                  /* contexts                                                    */
  const uint32_t *parent;      /* [n] parent context or GPA_NONE for roots                   */
  const uint32_t *site;        /* [n] call site e that created it, GPA_NONE for roots/members */
  const uint32_t *node;        /* [n] DAG node id (FUNC/SCC) or function id (SCC_MEMBER)     */
  const uint8_t  *kind;        /* [n] gpa_ctx_kind                                            */
  const uint32_t *first_child; /* [n] index of first child (valid when n_children > 0)        */
  const uint32_t *n_children;  /* [n]                                                         */
  const double   *frac;        /* [n] apportioning fraction f (product form, R13)             */
  const double   *excl;        /* [n*16] f * S_function (0 for SCC contexts)                  */
  const double   *incl;        /* [n*16] excl + sum of children's incl, in child order        */
  /* Step-1..3 intermediates, exposed for verification: */
  uint32_t n_call, n_func, n_dag;
  const uint64_t *call_weight; /* [n_call] w_e after Step 2 and the DAG guard (R11, R12)      */
  const uint64_t *dag_weight;  /* [n_dag] W_X = sum of external in-edge weights              */
  const uint8_t  *dag_active;  /* [n_dag]                                                     */
  const uint8_t  *func_active; /* [n_func] after Step 2                                       */
  const uint64_t *func_hist;   /* [n_func*16] S_f                                             */
} gpa_cct_view;

/* ---- version / host-only queries ------------------------------------------------------ */
GPA_API const char *gpa_version(void);
/* Message for the most recent non-OK status on this thread ("" if none). */
GPA_API const char *gpa_last_error(void);
/* Kernels this process has launched through the library so far (all devices; a
 * diagnostic counter for benchmarks: launches inside a timed region = difference). */
GPA_API uint64_t gpa_kernel_launches(void);
/* Force the attribution kernel process-wide (testing / benchmarking; results are identical):
 * 0 automatic (default), 1 register streaming, 2 TMA ring with L2 reductions, 3 TMA ring with
 * shared-memory heavy-hitter bins (u32), 4 ... heavy-hitter rows, 5 / 6 ... bins packed four /
 * two per 32-bit word (carries repaid exactly), 7 TMA ring with a shared-memory probe table of
 * granule rows (no per-record gather), 8 byte-packed bins found through a 32-bit code map with
 * a granule-indexed scratch for the rest, 9 every granule's row of byte counters in shared memory
 * (no plan; modules of up to ~13.8 k granules) (3-8 only where applicable: granule map, >= 2^21
 * records, >= 1024 instructions; 7, 8 and 9 also need the module inside one aligned 4 GiB window
 * and < 2^27 granules; otherwise automatic).  Automatic = 9 from 2^20 records on where it
 * applies, else 7 (structures up to 2^18 granules) or 8 from max(4e6, 8 x n_inst) records on
 * (granule map), else 1 (2 for binary-search structures above 4096 records).  Also settable by
 * the environment variable GPA_ATTR_VARIANT before the first call.  DESIGN.md §7 describes the
 * kernels. */
GPA_API gpa_status gpa_set_attr_kernel(int which);
/* Testing only: level L in 1..64 makes the TMA-ring kernels (7, 8, 9) sleep pseudo-random times up to
 * L/2 us before each stage's bulk copy (producer) and before reading each stage (consumers), so
 * producer-ahead and consumer-ahead orders of the ring protocol are exercised; results must not
 * change.  0 (default) = off.  Process-wide. */
GPA_API gpa_status gpa_set_ring_stress(int level);
/* The kernel (1..9, numbering above) gpa_attribute_samples runs for a call of n records on s
 * under the current setting.  Host-only; *which is written on GPA_OK. */
GPA_API gpa_status gpa_attr_kernel_choice(gpa_structure s, uint64_t n, int *which);
/* Validate a structure description on the host only (no device touched).  Same checks and
 * status as gpa_load_structure. */
GPA_API gpa_status gpa_validate_structure(const gpa_structure_desc *desc);

/* ---- structure ------------------------------------------------------------------------ */
/* Validate desc, derive the load-time tables (pc->instruction map, roll-up CSR, call-graph
 * CSR, Tarjan SCC condensation of the STATIC call graph (Step 3: weights do not
 * change the SCCs), DAG levels) and upload them to `device`.  Synchronous. */
GPA_API gpa_status gpa_load_structure(const gpa_structure_desc *desc, int device, gpa_structure *out);
GPA_API gpa_status gpa_get_structure_info(gpa_structure s, gpa_structure_info *out);
/* Rows produced for `scope` and, if h_ids != NULL, the id behind each row: instruction
 * index (INST), scope id (LINE/LOOP/INLINE) or function id (FUNC).  Host only. */
GPA_API gpa_status gpa_scope_rows(gpa_structure s, gpa_scope scope, uint64_t *rows, uint32_t *h_ids);
/* h_scc_of[f] = DAG node of function f (DAG ids ascend with their smallest member). */
GPA_API gpa_status gpa_get_scc(gpa_structure s, uint32_t *h_scc_of);
GPA_API void gpa_free_structure(gpa_structure s);

/* ---- a-1..a-3: attribution -------------------------------------------------------------
 * For every record k in d_samples[0..n):  slot = stall < 12 ? stall : 15;
 *   i = the instruction with inst_addr[i] <= pc < inst_addr[i] + inst_len[i] (R6)
 *   found:  d_inst_hist[i*16 + slot] += count       (raw metric = sum)
 *   else:   d_unattributed[slot]     += count
 *   d_rec_inst[k] = i or GPA_NONE (only if d_rec_inst != NULL).
 * Outputs ACCUMULATE (+=, u64): the caller zeroes them; calling again on further chunks
 * or from several streams is how streams are chunked/resumed.  d_samples must be 16-byte
 * aligned.  n == 0 is a no-op.  Enqueue-only on `stream`. */
GPA_API gpa_status gpa_attribute_samples(gpa_structure s, const gpa_sample *d_samples, uint64_t n,
                                 uint64_t *d_inst_hist, uint64_t *d_unattributed,
                                 uint32_t *d_rec_inst, gpa_stream_t stream);
/* Same result from HOST records: the library streams h_samples to the device in chunks
 * (pipelined host->device copy overlapped with the attribution kernel) using internal
 * staging buffers.  h_samples may be pageable or pinned (pinned is copied directly).
 * Synchronizes `stream` before returning. */
GPA_API gpa_status gpa_attribute_samples_host(gpa_structure s, const gpa_sample *h_samples, uint64_t n,
                                      uint64_t *d_inst_hist, uint64_t *d_unattributed,
                                      gpa_stream_t stream);

/* ---- f1: per-profile histograms and cross-profile statistics ----------------------------
 * P:481-487 (§4.5): derived metrics "for combining metrics from different thread profiles ...
 * sum, min, mean, max, std. deviation, and coefficient of variation".  A profile is the
 * record's `stream` field (a GPU stream / rank / thread).
 * gpa_attribute_profiles: like gpa_attribute_samples, but per profile and per FUNCTION:
 *   d_prof_hist[(p*n_func + f)*16 + slot] += count for records of profile p attributed to an
 *   instruction of function f; unattributed records -> d_prof_unattr[p*16 + slot].  Records
 *   with stream >= n_profiles use profile row n_profiles, so both buffers hold n_profiles+1
 *   rows ((n_profiles+1)*n_func*16 and (n_profiles+1)*16 u64).  Accumulates; enqueue-only.
 * gpa_profile_stats: for every function f and slot r, over profiles p < n_profiles (R25,
 *   population convention, exact integer sums before one rounding):
 *   d_stats[(f*6 + k)*16 + r], k = 0 sum, 1 min, 2 mean = sum/P, 3 max,
 *   4 std = sqrt(P*sum(x^2) - sum(x)^2)/P, 5 cv = std/mean (0 when mean = 0).  Enqueue-only. */
GPA_API gpa_status gpa_attribute_profiles(gpa_structure s, const gpa_sample *d_samples, uint64_t n,
                                          uint32_t n_profiles, uint64_t *d_prof_hist, uint64_t *d_prof_unattr,
                                          gpa_stream_t stream);
GPA_API gpa_status gpa_profile_stats(gpa_structure s, const uint64_t *d_prof_hist, uint32_t n_profiles,
                                     double *d_stats, gpa_stream_t stream);

/* f1 at instruction and CCT level (SURVEY §8f f1 "per instruction, function or CCT context").
 * gpa_attribute_profiles_inst: as gpa_attribute_profiles with instruction rows:
 *   d_prof_inst_hist[(p*n_inst + i)*16 + slot] (n_profiles+1 rows of n_inst x 16 u64).
 * gpa_profile_stats_rows: the statistics of gpa_profile_stats for any u64 cube of `rows` rows
 *   ([n_profiles+1][rows][16], profiles 0..n_profiles-1 enter): d_stats [rows][6][16].
 * gpa_cct_profiles (reading R28): per-profile values on the tree `cct` (reconstructed from the
 *   aggregate histogram): d_prof_excl[(p*n + c)*16 + r] = frac(c) * d_prof_hist[p][g(c)][r] for
 *   FUNC / SCC_MEMBER contexts of function g (0 at SCC contexts), d_prof_incl = excl + children's
 *   incl in child order; d_prof_hist is gpa_attribute_profiles' function cube; both outputs are
 *   [n_profiles+1][n][16] f64.  Synchronizes the tree's build stream once (level table).
 * gpa_profile_stats_f64: statistics of an f64 cube [n_profiles+1][rows][16] over profiles
 *   0..n_profiles-1: sum (left fold in profile order), min, mean = sum/P, max, population std
 *   = sqrt(sum (x-mean)^2 / P) (two passes), cv = std/mean (0 when mean = 0) -> [rows][6][16].
 * All enqueue on `stream` (device memory of `device` for the two rows-only calls). */
GPA_API gpa_status gpa_attribute_profiles_inst(gpa_structure s, const gpa_sample *d_samples, uint64_t n,
                                               uint32_t n_profiles, uint64_t *d_prof_inst_hist,
                                               uint64_t *d_prof_unattr, gpa_stream_t stream);
GPA_API gpa_status gpa_profile_stats_rows(uint64_t rows, const uint64_t *d_prof_hist, uint32_t n_profiles,
                                          double *d_stats, int device, gpa_stream_t stream);
GPA_API gpa_status gpa_cct_profiles(gpa_structure s, gpa_cct cct, const uint64_t *d_prof_hist, uint32_t n_profiles,
                                    double *d_prof_excl, double *d_prof_incl, gpa_stream_t stream);
GPA_API gpa_status gpa_profile_stats_f64(uint64_t rows, const double *d_prof_vals, uint32_t n_profiles,
                                         double *d_stats, int device, gpa_stream_t stream);

/* ---- f3: sparse cubes (PMS / CMS) of the per-profile histograms -------------------------
 * PAPER.md §5.2: "Profile Major Sparse" and "CCT Major Sparse" formats, one modified
 * CSR per plane.  The cube is d_prof_hist of gpa_attribute_profiles with all n_profiles+1
 * profile rows (p x function row c x slot m).  GPA_SPARSE_CMS: plane = c, its values ordered
 * by (m, p) with ids[] = p, and a sparse metric index of (m, start) pairs; GPA_SPARSE_PMS:
 * plane = p, values ordered by (c, m) with ids[] = m, sparse context index of (c, start).
 * Every plane's index ends with a sentinel (GPA_NONE, end).  plane_off / index_off
 * [n_planes+1] are element offsets into the value / index arrays.  Library-owned result;
 * synchronizes `stream` (the non-zero count decides the allocation). */
typedef enum { GPA_SPARSE_PMS = 0, GPA_SPARSE_CMS = 1 } gpa_sparse_major;
typedef struct gpa_sparse_s *gpa_sparse;
typedef struct {
  uint32_t major, n_planes;
  uint64_t n_values, n_index;
  const uint64_t *plane_off;   /* [n_planes+1] */
  const uint64_t *index_off;   /* [n_planes+1] */
  const uint64_t *vals;        /* [n_values] non-zero values                       */
  const uint32_t *ids;         /* [n_values] profile id (CMS) or metric id (PMS)   */
  const uint64_t *index_start; /* [n_index] start of each inner run in vals        */
  const uint32_t *index_id;    /* [n_index] metric (CMS) / context (PMS) id; GPA_NONE = sentinel */
} gpa_sparse_view;
GPA_API gpa_status gpa_sparse_build(gpa_structure s, const uint64_t *d_prof_hist, uint32_t n_profiles,
                                    gpa_sparse_major major, gpa_sparse *out, gpa_stream_t stream);
GPA_API gpa_status gpa_get_sparse_view(gpa_sparse sp, gpa_sparse_view *out);
GPA_API void gpa_free_sparse(gpa_sparse sp);

/* ---- f4: GPU-idleness blame over trace lines ----------------------------------------------
 * PAPER.md §6.2: "identifies times when all GPU streams are idle and at least one
 * CPU thread is active. In such cases, it partitions the cost of GPU idleness among routines
 * being executed by active CPU threads" (normalized blame per CPU routine).  DESIGN.md R27:
 * a trace line is a sequence of change points (time, ctx), non-decreasing in time; on
 * [time[i], time[i+1]) the line is in state ctx[i] (GPA_NONE = idle); after its last change
 * point it is idle (the last ctx is ignored).  GPU lines are streams (ctx = any kernel id),
 * CPU lines are threads (ctx = routine id < n_routines, already mapped to the attribution
 * depth by the caller).  Lines are grouped into scopes (ranks).  Per scope, on every interval
 * where all its GPU lines are idle: gpu_idle += length; if k >= 1 of its CPU lines are
 * active: total += length and each active thread's routine gets length/k.  Outputs:
 * blame f64 [n_scopes][n_routines] = sum_k num_k / k with num_k the exact integer time
 * routine r was blamed while k threads were active (ascending k, one IEEE division and
 * addition each), share = blame / total (canonical NaN when total = 0), total and
 * gpu_idle u64 [n_scopes] (ns).  Any output pointer may be NULL.  Events are device arrays
 * d_time u64 [E] and d_ctx u32 [E], E = line_off[n_lines] <= 2^27, laid out line after line.
 * Errors: GPA_ERR_INVALID_ARG for a malformed line table (line_off not starting at 0 or
 * decreasing, line_scope decreasing or >= n_scopes, kind not 0/1, a scope without a GPU
 * line), a line going back in time or a CPU routine id >= n_routines (detected on the device;
 * the call synchronizes `stream`); GPA_ERR_UNSUPPORTED beyond the size limits (E > 2^27,
 * > 65535 lines of a kind per scope, E * max CPU lines per scope >= 2^32). */
typedef struct {
  uint32_t n_lines;
  const uint64_t *line_off;   /* HOST [n_lines+1] event offsets, line_off[0] = 0          */
  const uint8_t *line_kind;   /* HOST [n_lines] 0 = GPU stream, 1 = CPU thread            */
  const uint32_t *line_scope; /* HOST [n_lines] scope (rank) id, non-decreasing            */
  uint32_t n_scopes, n_routines;
} gpa_trace_desc;
GPA_API gpa_status gpa_idleness_blame(const gpa_trace_desc *desc, const uint64_t *d_time, const uint32_t *d_ctx,
                                      double *d_blame, double *d_share, uint64_t *d_total, uint64_t *d_gpu_idle,
                                      int device, gpa_stream_t stream);

/* ---- a-6..a-9: approximate GPU calling-context tree (§5.3) -----------------
 * From a per-instruction histogram: Step 1 edge weights w_e = sum_{r<12} H[call_inst[e]][r]
 * (R10); Step 2 zero-weight propagation to the least fixpoint (R11) and the
 * DAG guard (R12); Step 3 uses the load-time SCC condensation; Step 4 splits
 * the DAG into a tree, apportioning by f(child) = f(parent) * w_e / W_callee (P:880-881,
 * R13-R16).  max_contexts == 0: count only (*out untouched, *n_contexts = required).
 * More contexts than max_contexts -> GPA_ERR_CAPACITY with *n_contexts = required.
 * d_inst_hist must be 16-byte aligned.  Synchronizes `stream` (the context count decides
 * the allocation). */
GPA_API gpa_status gpa_reconstruct_cct(gpa_structure s, const uint64_t *d_inst_hist,
                               gpa_weight_mode mode, uint64_t max_contexts,
                               gpa_cct *out, uint64_t *n_contexts, gpa_stream_t stream);
/* Exact counts from instrumentation (execution frequency of each basic block,
 * propagated to its instructions): for block b, every instruction block_start[b] ..
 * block_start[b+1]-1 gains d_counts[b] in slot 0 of d_inst_hist (accumulated, u64).
 * d_block_start: DEVICE [n_blocks+1], ascending instruction indices (indices >= n_inst are
 * clipped).  Enqueue-only. */
GPA_API gpa_status gpa_block_counts(gpa_structure s, uint32_t n_blocks, const uint32_t *d_block_start,
                                    const uint64_t *d_counts, uint64_t *d_inst_hist, gpa_stream_t stream);
/* The same tree without a host synchronization (for a pipeline of batches: P:711-714 statistics
 * generated per batch while the next batch is attributed).  The tree is built in one launch into
 * *capacity context slots (the static path bound when it is small, else 2^16); its size stays on
 * the device.  Until gpa_cct_finish: gpa_derive_metrics with GPA_SCOPE_CCT_EXCL / _INCL writes the
 * rows of the built contexts only (d_metrics must hold *capacity rows; none when the build did
 * not fit); gpa_get_cct_view and gpa_cct_profiles fail with GPA_ERR_INVALID_ARG.  d_inst_hist must
 * stay unchanged until gpa_cct_finish (an overflowing build is redone from it).  Enqueue-only,
 * except structures whose trees the one-launch build cannot hold at all: then as
 * gpa_reconstruct_cct (synchronizes; *capacity = the context count, the tree finished). */
GPA_API gpa_status gpa_reconstruct_cct_async(gpa_structure s, const uint64_t *d_inst_hist, gpa_weight_mode mode,
                                             gpa_cct *out, uint64_t *capacity, gpa_stream_t stream);
/* Completes an asynchronous tree: synchronizes its stream and sets *n_contexts.  If the one-launch
 * build did not fit its capacity the tree is rebuilt with the counted path (synchronously, same
 * result as gpa_reconstruct_cct) and *rebuilt = 1 (may be NULL): CCT metrics derived before must
 * be derived again.  A finished or synchronous tree: *n_contexts = its size, *rebuilt = 0. */
GPA_API gpa_status gpa_cct_finish(gpa_cct c, uint64_t *n_contexts, int *rebuilt);
GPA_API gpa_status gpa_get_cct_view(gpa_cct c, gpa_cct_view *out);
/* Releases the tree's device memory in stream order on the stream gpa_reconstruct_cct was
 * called with (no device synchronization); work on other streams that still reads the views
 * must be ordered before that stream by the caller. */
GPA_API void gpa_free_cct(gpa_cct c);

/* ---- a-5 + a-10: roll-up and derived metrics -------------------------------------------
 * INST..FUNC: rows of `scope` (see gpa_scope_rows).  Row histogram (u64[16]) =
 *   sum of H over the instructions whose scope chain contains the row's scope (R8);
 *   mix (u64[16]) = per instruction class k, sum of S(i) = sum_{r<12} H[i][r] (R5).
 * CCT_EXCL / CCT_INCL: rows = contexts of `cct` (excl / incl vectors; no mix, no u64 out).
 * d_metrics[row*33 + c] (DESIGN.md §3 table; NaN = 0x7FF8000000000000 when S == 0, R18):
 *   0 S  1 W=v0/S  2 (v0+v9)/S  3 sum_{LAT} v/S  4..15 v[r]/S  16 v[15]
 *   17..32 mix[k]/S (NaN for CCT rows).
 * Any of d_scope_hist, d_scope_mix, d_metrics may be NULL.  For INST rows d_scope_hist
 * receives a copy of d_inst_hist.  d_inst_hist / d_scope_hist / d_scope_mix must be 16-byte
 * aligned, d_metrics 8-byte aligned (GPA_ERR_INVALID_ARG otherwise).  Enqueue-only. */
GPA_API gpa_status gpa_derive_metrics(gpa_structure s, gpa_scope scope, const uint64_t *d_inst_hist,
                              gpa_cct cct, uint64_t *d_scope_hist, uint64_t *d_scope_mix,
                              double *d_metrics, gpa_stream_t stream);

/* ---- f1 extension: a CCT per profile, unified by call path (reading R30) -----------------------
 * The paper reconstructs an approximate CCT "for each GPU kernel invocation" and unifies
 * the trees of all profiles into one.  Here a profile is a value of the records'
 * `stream` field (R25).  Per profile p the inputs are its function histogram S_f,p (the FUNC rows
 * of gpa_attribute_profiles) and its call-site weights w_p (gpa_profile_call_weights); Steps 2-4
 * run per profile exactly as gpa_reconstruct_cct_inputs would on (S_f,p, w_p).  The unified tree
 * holds every call path present in at least one profile's tree, numbered breadth first with the
 * order every tree uses (roots by DAG node, SCC members by function id, calls by call
 * instruction); frac / excl / incl of profile p at a unified context are p's own tree values
 * (bit for bit), 0 where p's tree lacks the path.
 *
 * gpa_profile_call_weights: adds, per record with a valid stall slot on a call instruction,
 *   its count to d_prof_call_weight[min(stream, n_profiles) * n_call + site] (DEVICE u64
 *   [(n_profiles+1) * n_call], accumulated; the last row collects stream ids >= n_profiles).
 * gpa_reconstruct_cct_per_profile: d_prof_func_hist DEVICE u64 [n_profiles][n_func][16] (16-byte
 *   aligned), d_prof_call_weight DEVICE u64 [n_profiles][n_call]; max_contexts bounds the unified
 *   tree and the union tree it is cut from (0: count only, *n_contexts = the unified count);
 *   GPA_ERR_CAPACITY when exceeded.  Synchronizes `stream`. */
typedef struct gpa_cct_multi_s *gpa_cct_multi;
typedef struct {
  uint64_t n;
  uint32_t n_profiles;
  const uint32_t *parent, *site, *node;   /* [n] (NONE for roots / no site) */
  const uint8_t *kind;                    /* [n] gpa_ctx_kind */
  const uint32_t *first_child, *n_children;
  const double *frac;                     /* [n][n_profiles] */
  const double *excl, *incl;              /* [n][n_profiles][16] */
} gpa_cct_multi_view;
GPA_API gpa_status gpa_profile_call_weights(gpa_structure s, const gpa_sample *d_samples, uint64_t n,
                                            uint32_t n_profiles, uint64_t *d_prof_call_weight, gpa_stream_t stream);
GPA_API gpa_status gpa_reconstruct_cct_per_profile(gpa_structure s, const uint64_t *d_prof_func_hist,
                                                   const uint64_t *d_prof_call_weight, uint32_t n_profiles,
                                                   gpa_weight_mode mode, uint64_t max_contexts, gpa_cct_multi *out,
                                                   uint64_t *n_contexts, gpa_stream_t stream);
GPA_API gpa_status gpa_get_cct_multi_view(gpa_cct_multi c, gpa_cct_multi_view *out);
GPA_API void gpa_free_cct_multi(gpa_cct_multi c);

/* ---- reusable attribution plans -----------------------------------------------------------------
 * The large-call attribution kernels (gpa_set_attr_kernel 7 / 8) first choose, from a sample of
 * the call's records, which granules / (instruction, slot) bins are counted in shared memory (a
 * "plan"; the rest go to L2).  gpa_attribute_samples builds a plan per call.  A plan built once
 * from representative records (e.g. the first batch of a profile stream: records of one
 * application are alike) can be reused for any number of later calls, removing the
 * per-call pre-pass; results are identical for every plan (exact counting), only speed differs.
 *
 * gpa_attr_plan_create: samples d_samples[0..n) (DEVICE, 16-byte aligned; n >= 4096 for a plan)
 *   and synchronizes `stream`.  Structures without a large-call kernel (binary-search lookup,
 *   module across a 4 GiB boundary) and small samples get an empty plan (variant 0): planned calls
 *   then behave as gpa_attribute_samples.  The plan holds device memory until gpa_attr_plan_free
 *   and must not outlive its structure.  Errors as gpa_attribute_samples. */
typedef struct gpa_attr_plan_s *gpa_attr_plan;
GPA_API gpa_status gpa_attr_plan_create(gpa_structure s, const gpa_sample *d_samples, uint64_t n,
                                        gpa_attr_plan *out, gpa_stream_t stream);
/* The kernel a plan runs (7 or 8, 0 = none). */
GPA_API gpa_status gpa_attr_plan_variant(gpa_attr_plan p, int *which);
/* gpa_attribute_samples with a prepared plan: same arguments, semantics (accumulates into
 * d_inst_hist / d_unattributed) and errors; enqueue-only.  Plans are read-only: one plan may serve
 * concurrent calls on different streams. */
GPA_API gpa_status gpa_attribute_samples_planned(gpa_structure s, gpa_attr_plan p, const gpa_sample *d_samples,
                                                 uint64_t n, uint64_t *d_inst_hist, uint64_t *d_unattributed,
                                                 uint32_t *d_rec_inst, gpa_stream_t stream);
GPA_API void gpa_attr_plan_free(gpa_attr_plan p);

/* ---- a-4 / a-5 across GPUs: statistics over function-aligned instruction ranges -------------
 * The paper reads measurements "in parallel, propagating values up the calling context tree"
 * and aggregates accumulators "by a second reduction operation" (reading R29 in
 * DESIGN.md): every scope row (LINE, LOOP, INLINE, FUNC)
 * lies inside one function, so when each function's instructions are contiguous, rank r of N can
 * receive the reduced histogram rows [b_r, b_{r+1}) of a function-aligned split (one
 * reduce-scatter instead of a reduce to one rank) and derive the rows of its own functions.
 *
 * gpa_partition_structure: HOST only (no device touched).  Writes h_inst_bounds[0..n_parts]:
 *   0 = b_0 <= b_1 <= ... <= b_n_parts = n_inst, each inner bound the first instruction of a
 *   function (the one nearest to r*n_inst/n_parts; empty parts possible).  Same checks as
 *   gpa_validate_structure; GPA_ERR_STRUCTURE when some function's instructions are not
 *   contiguous (then reduce to one rank and use gpa_derive_metrics). */
GPA_API gpa_status gpa_partition_structure(const gpa_structure_desc *desc, uint32_t n_parts,
                                           uint32_t *h_inst_bounds);
/* gpa_derive_metrics restricted to the rows of the functions whose instructions lie in
 * [inst_lo, inst_hi) (INST scope: rows inst_lo .. inst_hi-1).  Both ends must be 0, n_inst or
 * the first instruction of a function (GPA_ERR_INVALID_ARG otherwise; GPA_ERR_STRUCTURE when
 * functions are not contiguous); inst_hi == n_inst also takes functions without instructions.
 * Reads d_inst_hist rows of the range only; writes only the range's rows of the full-size
 * outputs (row numbering as gpa_derive_metrics).  No CCT scopes.  Enqueue-only. */
GPA_API gpa_status gpa_derive_metrics_range(gpa_structure s, gpa_scope scope, const uint64_t *d_inst_hist,
                                            uint32_t inst_lo, uint32_t inst_hi, uint64_t *d_scope_hist,
                                            uint64_t *d_scope_mix, double *d_metrics, gpa_stream_t stream);
/* All static scope kinds in one pass (one kernel launch + one for multi-chunk rows instead of one
 * or two per scope): outs[k] for k = GPA_SCOPE_INST .. GPA_SCOPE_FUNC (5 entries) gives that
 * scope's d_scope_hist / d_scope_mix / d_metrics exactly as gpa_derive_metrics would (any NULL;
 * an all-NULL entry skips the scope).  inst_lo = 0, inst_hi = n_inst: every row; otherwise the
 * rows of the function-aligned range, as gpa_derive_metrics_range.  Enqueue-only. */
typedef struct { uint64_t *scope_hist; uint64_t *scope_mix; double *metrics; } gpa_scope_out;
GPA_API gpa_status gpa_derive_scopes(gpa_structure s, const uint64_t *d_inst_hist, uint32_t inst_lo, uint32_t inst_hi,
                                     const gpa_scope_out *outs, gpa_stream_t stream);
/* CCT Step 1 on a range: S_f (d_func_hist[f*16 + r], u64) for the functions of
 * [inst_lo, inst_hi) and w_e (d_call_weight[e] = sum_{r<12} H[call_inst[e]][r], R10) for the call
 * sites whose call instruction lies in it; other entries are left untouched (zero them, then
 * the element-wise sum over a partition's ranks is the whole input).  Range rules as above;
 * d_inst_hist / d_func_hist 16-byte aligned.  Enqueue-only. */
GPA_API gpa_status gpa_cct_inputs(gpa_structure s, const uint64_t *d_inst_hist, uint32_t inst_lo,
                                  uint32_t inst_hi, uint64_t *d_func_hist, uint64_t *d_call_weight,
                                  gpa_stream_t stream);
/* gpa_reconstruct_cct from Step-1 inputs (S_f = d_func_hist [n_func*16], w = d_call_weight
 * [n_call], DEVICE, read only) instead of the instruction histogram: Steps 2-4
 * and the result are those of gpa_reconstruct_cct on a histogram with these S_f and w. */
GPA_API gpa_status gpa_reconstruct_cct_inputs(gpa_structure s, const uint64_t *d_func_hist,
                                              const uint64_t *d_call_weight, gpa_weight_mode mode,
                                              uint64_t max_contexts, gpa_cct *out, uint64_t *n_contexts,
                                              gpa_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* GPA_H */
