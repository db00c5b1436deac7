/*
 * gpa_oracle.c — plain, slow, obviously-correct CPU oracle for the PC-sample attribution
 * path of Zhou et al., "Measurement and Analysis of GPU-accelerated Applications with
 * HPCToolkit" (arXiv 2109.06931).  P:<n> = line n of the paper's LaTeX.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code, header,
 * table or constant with the CUDA library (paper_2109_06931_b200/csrc, include/gpa.h);
 * the constants below are restated from the paper and DESIGN.md §3.
 *
 * Compiled with -O2 -ffp-contract=off (no fused multiply-add: every fp64 operation is
 * one IEEE operation in the order written here).
 *
 * Parts and what pins them (tests/test_oracle_*.py):
 *   D1 oracle_attribute   — pinned by brute-force linear scan, conservation, shard invariance
 *   D2 oracle_rollup      — pinned by explicit range containment (SPEC-style resolve), sums
 *   D3-D6 oracle_cct      — pinned by hand-worked fixtures (tests/golden), brute-force path
 *                           enumeration with exact rationals, conservation, gprof identity
 *   D7 oracle_derive_*    — pinned by closed forms (P:948 W(100,75)=0.25, NaN at S=0, sums)
 *   D8 oracle_attribute_profiles / oracle_profile_stats — per-record brute force, SPEC stats
 *   D9 oracle_sparse_build — worked lookups, round trips through an independent decoder
 *   D11 oracle_cct_profiles / oracle_profile_stats_f64 — the single-profile identity with the
 *                           aggregate CCT, hand-worked fractions of the Fig.-4 fixture, numpy
 *                           two-pass statistics
 *   D10 oracle_blame       — SPEC's worked blame examples, a 1-ns brute force with exact
 *                           rationals, integer conservation
 * Parity is unpinned against the PAPER (pinned only against our own readings) for the stall
 * taxonomy (R2), the latency-hiding columns (R4) and the instruction mix (R5): the paper
 * gives no numbers for them.  See DESIGN.md §3.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <math.h>

#define O_SLOTS 16         /* slots per instruction row: 12 reasons, 3 reserved, 1 invalid */
#define O_VALID 12         /* stall reasons 0..11 (R2)                           */
#define O_INVALID 15       /* slot of a record whose stall code is >= 12 (R2)              */
#define O_NCOLS 33         /* derived columns                               */
#define O_NONE 0xFFFFFFFFu

typedef struct { uint64_t pc; uint32_t count; uint16_t stall; uint16_t stream; } o_record;

/* ======================================================================================
 * D1 — attribution ("Each PC sample ... includes an instruction address, a
 * stall reason, and a count"; P:616-617 functions relocated to unique addresses and split
 * into disjoint ranges; "A raw ... metric ... is simply the sum of all measured
 * values").  For each record: the instruction whose range [addr, addr+len) contains pc
 * (largest addr <= pc, found by binary search over the sorted starts) gets count added in
 * its stall slot; a pc in no range goes to the unattributed row U (reading R6).
 * ====================================================================================== */
static int64_t o_last_start_le(const uint64_t *inst_addr, uint32_t n_inst, uint64_t pc)
{
  /* upper_bound: first index with inst_addr[idx] > pc; answer is idx - 1 */
  uint64_t lo = 0, hi = n_inst;
  while (lo < hi) {
    uint64_t mid = lo + (hi - lo) / 2;
    if (inst_addr[mid] <= pc) lo = mid + 1; else hi = mid;
  }
  return (int64_t)lo - 1;
}

void oracle_attribute(uint32_t n_inst, const uint64_t *inst_addr, const uint16_t *inst_len,
                      const o_record *rec, uint64_t n,
                      uint64_t *H, uint64_t *U, uint32_t *rec_inst)
{
  for (uint64_t k = 0; k < n; k++) {
    uint64_t pc = rec[k].pc;
    uint32_t slot = rec[k].stall < O_VALID ? rec[k].stall : O_INVALID;
    int64_t j = o_last_start_le(inst_addr, n_inst, pc);
    if (j >= 0 && pc < inst_addr[j] + inst_len[j]) {
      H[(uint64_t)j * O_SLOTS + slot] += rec[k].count;
      if (rec_inst) rec_inst[k] = (uint32_t)j;
    } else {
      U[slot] += rec[k].count;
      if (rec_inst) rec_inst[k] = O_NONE;
    }
  }
}

/* D1 over T contiguous record ranges with thread-private histograms, merged serially
 * (integer addition: the result does not depend on T).  Used for the CPU baseline. */
typedef struct {
  uint32_t n_inst; const uint64_t *inst_addr; const uint16_t *inst_len;
  const o_record *rec; uint64_t n; uint64_t *H; uint64_t U[O_SLOTS];
} o_attr_job;

static void *o_attr_thread(void *p)
{
  o_attr_job *j = (o_attr_job *)p;
  oracle_attribute(j->n_inst, j->inst_addr, j->inst_len, j->rec, j->n, j->H, j->U, NULL);
  return NULL;
}

int oracle_attribute_mt(uint32_t n_inst, const uint64_t *inst_addr, const uint16_t *inst_len,
                        const o_record *rec, uint64_t n, uint64_t *H, uint64_t *U, int n_threads)
{
  if (n_threads < 1) n_threads = 1;
  o_attr_job *jobs = (o_attr_job *)calloc((size_t)n_threads, sizeof(o_attr_job));
  pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
  if (!jobs || !th) { free(jobs); free(th); return -1; }
  for (int t = 0; t < n_threads; t++) {
    uint64_t a = n * (uint64_t)t / (uint64_t)n_threads, b = n * (uint64_t)(t + 1) / (uint64_t)n_threads;
    jobs[t].n_inst = n_inst; jobs[t].inst_addr = inst_addr; jobs[t].inst_len = inst_len;
    jobs[t].rec = rec + a; jobs[t].n = b - a;
    jobs[t].H = (uint64_t *)calloc((size_t)n_inst * O_SLOTS + 1, sizeof(uint64_t));
    if (!jobs[t].H) return -1;
    pthread_create(&th[t], NULL, o_attr_thread, &jobs[t]);
  }
  for (int t = 0; t < n_threads; t++) {
    pthread_join(th[t], NULL);
    for (uint64_t x = 0; x < (uint64_t)n_inst * O_SLOTS; x++) H[x] += jobs[t].H[x];
    for (int s = 0; s < O_SLOTS; s++) U[s] += jobs[t].U[s];
    free(jobs[t].H);
  }
  free(jobs); free(th);
  return 0;
}

/* ======================================================================================
 * D2 — roll-up to lines, loops, inlined code and functions ("calling context
 * nodes are created based on program structure information for each instruction";
 * P:711-712 "propagating values up"; P:936-937 flat view per function).  Every scope on
 * the chain leaf(i) = inst_scope[i] -> ... -> FUNCTION root receives H[i] (reading R8:
 * LINE rows are leaves, LOOP/INLINE/FUNCTION rows inclusive).  MIX[s][class(i)] receives
 * S(i) = sum of the 12 valid slots of H[i] (instruction classes; reading R5).
 * Outputs are indexed by scope id and accumulate (+=).
 * ====================================================================================== */
void oracle_rollup(uint32_t n_inst, const uint32_t *inst_scope, const uint8_t *inst_class,
                   uint32_t n_scope, const uint32_t *scope_parent,
                   const uint64_t *H, uint64_t *Hs, uint64_t *MIX)
{
  (void)n_scope;
  for (uint32_t i = 0; i < n_inst; i++) {
    uint64_t S = 0;
    for (int r = 0; r < O_VALID; r++) S += H[(uint64_t)i * O_SLOTS + r];
    for (uint32_t s = inst_scope[i]; s != O_NONE; s = scope_parent[s]) {
      for (int r = 0; r < O_SLOTS; r++) Hs[(uint64_t)s * O_SLOTS + r] += H[(uint64_t)i * O_SLOTS + r];
      MIX[(uint64_t)s * O_SLOTS + inst_class[i]] += S;
    }
  }
}

/* inst -> function: walk the scope chain to its FUNCTION root, then invert func_scope. */
static void o_inst_func(uint32_t n_inst, const uint32_t *inst_scope, uint32_t n_scope,
                        const uint32_t *scope_parent, uint32_t n_func, const uint32_t *func_scope,
                        uint32_t *inst_func)
{
  uint32_t *func_of_scope = (uint32_t *)malloc(sizeof(uint32_t) * (n_scope + 1));
  for (uint32_t s = 0; s < n_scope; s++) func_of_scope[s] = O_NONE;
  for (uint32_t f = 0; f < n_func; f++) func_of_scope[func_scope[f]] = f;
  for (uint32_t i = 0; i < n_inst; i++) {
    uint32_t s = inst_scope[i];
    while (scope_parent[s] != O_NONE) s = scope_parent[s];
    inst_func[i] = func_of_scope[s];
  }
  free(func_of_scope);
}

void oracle_inst_func(uint32_t n_inst, const uint32_t *inst_scope, uint32_t n_scope,
                      const uint32_t *scope_parent, uint32_t n_func, const uint32_t *func_scope,
                      uint32_t *inst_func)
{
  o_inst_func(n_inst, inst_scope, n_scope, scope_parent, n_func, func_scope, inst_func);
}

/* ======================================================================================
 * D3-D6 — approximate GPU calling-context tree, §5.3 P:869-882 (four steps).
 * ====================================================================================== */
typedef struct {
  /* result contexts (BFS order, reading R17) */
  uint64_t n, cap;
  uint32_t *parent, *site, *node, *first_child, *n_children;
  uint8_t *kind;                 /* 0 FUNC, 1 SCC, 2 SCC_MEMBER (reading R14) */
  double *frac, *excl, *incl;    /* excl/incl: [n*16] */
  /* intermediates of Steps 1-3 */
  uint32_t n_func, n_call, n_dag;
  uint64_t *w_step1;             /* [n_call] Step 1 weights                     */
  uint64_t *w;                   /* [n_call] after Step 2 and the DAG guard     */
  uint8_t *func_active;          /* [n_func] after Step 2                       */
  uint64_t *S_f;                 /* [n_func*16]                                 */
  uint32_t *scc_of;              /* [n_func] DAG node of each function          */
  uint8_t *dag_nontrivial;       /* [n_dag]                                     */
  uint8_t *dag_active;           /* [n_dag]                                     */
  uint64_t *W;                   /* [n_dag] sum of external in-edge weights     */
  int status;                    /* 0 ok, 3 capacity exceeded (n = required)    */
} oracle_cct_result;

/* Tarjan's strongly-connected-components algorithm ("Identify strongly connected
 * components (SCCs) using Tarjan's algorithm"), textbook recursive form over the static
 * call graph (every call site, whatever its weight). */
typedef struct {
  uint32_t n_func; const uint32_t *out_ptr, *out_dst;
  uint32_t *index, *low, *stack, *comp; uint8_t *on_stack;
  uint32_t next_index, sp, n_comp;
} o_tarjan;

static void o_strongconnect(o_tarjan *t, uint32_t v)
{
  t->index[v] = t->low[v] = t->next_index++;
  t->stack[t->sp++] = v; t->on_stack[v] = 1;
  for (uint32_t k = t->out_ptr[v]; k < t->out_ptr[v + 1]; k++) {
    uint32_t u = t->out_dst[k];
    if (t->index[u] == O_NONE) {
      o_strongconnect(t, u);
      if (t->low[u] < t->low[v]) t->low[v] = t->low[u];
    } else if (t->on_stack[u]) {
      if (t->index[u] < t->low[v]) t->low[v] = t->index[u];
    }
  }
  if (t->low[v] == t->index[v]) {
    uint32_t u;
    do { u = t->stack[--t->sp]; t->on_stack[u] = 0; t->comp[u] = t->n_comp; } while (u != v);
    t->n_comp++;
  }
}

static int o_cmp_u64(const void *a, const void *b)
{
  uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

static int o_grow(oracle_cct_result *R)
{
  uint64_t nc = R->cap ? R->cap * 2 : 1024;
#define O_RE(p, T, m) do { void *q = realloc(R->p, sizeof(T) * (size_t)nc * (m)); if (!q) return -1; R->p = (T *)q; } while (0)
  O_RE(parent, uint32_t, 1); O_RE(site, uint32_t, 1); O_RE(node, uint32_t, 1);
  O_RE(first_child, uint32_t, 1); O_RE(n_children, uint32_t, 1); O_RE(kind, uint8_t, 1);
  O_RE(frac, double, 1); O_RE(excl, double, O_SLOTS); O_RE(incl, double, O_SLOTS);
#undef O_RE
  R->cap = nc;
  return 0;
}

static int o_append(oracle_cct_result *R, uint8_t kind, uint32_t node, uint32_t parent,
                    uint32_t site, double f)
{
  if (R->n == R->cap && o_grow(R)) return -1;
  uint64_t c = R->n++;
  R->kind[c] = kind; R->node[c] = node; R->parent[c] = parent; R->site[c] = site;
  R->frac[c] = f; R->first_child[c] = 0; R->n_children[c] = 0;
  return 0;
}

oracle_cct_result *oracle_cct_mode(uint32_t n_inst, const uint32_t *inst_scope,
                                   uint32_t n_scope, const uint32_t *scope_parent,
                                   uint32_t n_func, const uint32_t *func_scope,
                                   uint32_t n_call, const uint32_t *call_inst, const uint32_t *call_callee,
                                   const uint64_t *H, uint64_t max_contexts, int exact)
{
  oracle_cct_result *R = (oracle_cct_result *)calloc(1, sizeof(oracle_cct_result));
  R->n_func = n_func; R->n_call = n_call;
  uint32_t *inst_func = (uint32_t *)malloc(sizeof(uint32_t) * (n_inst + 1));
  o_inst_func(n_inst, inst_scope, n_scope, scope_parent, n_func, func_scope, inst_func);
  uint32_t *caller = (uint32_t *)malloc(sizeof(uint32_t) * (n_call + 1));
  for (uint32_t e = 0; e < n_call; e++) caller[e] = inst_func[call_inst[e]];

  /* ---- Step 1: static call graph from call instructions; edge weight = the call
   * instruction's sample count (sum of its valid stall slots, reading R10).  S_f = the
   * function's samples (all 16 slots; the 12 valid ones decide "has samples"). */
  R->w_step1 = (uint64_t *)calloc(n_call + 1, sizeof(uint64_t));
  R->w = (uint64_t *)calloc(n_call + 1, sizeof(uint64_t));
  for (uint32_t e = 0; e < n_call; e++) {
    uint64_t s = 0;
    for (int r = 0; r < O_VALID; r++) s += H[(uint64_t)call_inst[e] * O_SLOTS + r];
    R->w_step1[e] = s; R->w[e] = s;
  }
  R->S_f = (uint64_t *)calloc((size_t)n_func * O_SLOTS + 1, sizeof(uint64_t));
  for (uint32_t i = 0; i < n_inst; i++)
    for (int r = 0; r < O_SLOTS; r++) R->S_f[(uint64_t)inst_func[i] * O_SLOTS + r] += H[(uint64_t)i * O_SLOTS + r];

  /* in-edge lists per callee function, out-edge lists per caller (CSR) */
  uint32_t *in_ptr = (uint32_t *)calloc(n_func + 1, sizeof(uint32_t));
  uint32_t *in_e = (uint32_t *)malloc(sizeof(uint32_t) * (n_call + 1));
  uint32_t *out_ptr = (uint32_t *)calloc(n_func + 1, sizeof(uint32_t));
  uint32_t *out_e = (uint32_t *)malloc(sizeof(uint32_t) * (n_call + 1));
  uint32_t *out_dst = (uint32_t *)malloc(sizeof(uint32_t) * (n_call + 1));
  for (uint32_t e = 0; e < n_call; e++) { in_ptr[call_callee[e] + 1]++; out_ptr[caller[e] + 1]++; }
  for (uint32_t f = 0; f < n_func; f++) { in_ptr[f + 1] += in_ptr[f]; out_ptr[f + 1] += out_ptr[f]; }
  {
    uint32_t *fi = (uint32_t *)malloc(sizeof(uint32_t) * (n_func + 1));
    uint32_t *fo = (uint32_t *)malloc(sizeof(uint32_t) * (n_func + 1));
    memcpy(fi, in_ptr, sizeof(uint32_t) * n_func); memcpy(fo, out_ptr, sizeof(uint32_t) * n_func);
    /* out-edges of each caller in ascending call-instruction order (reading R17) */
    uint64_t *key = (uint64_t *)malloc(sizeof(uint64_t) * (n_call + 1));
    for (uint32_t e = 0; e < n_call; e++) key[e] = ((uint64_t)call_inst[e] << 32) | e;
    qsort(key, n_call, sizeof(uint64_t), o_cmp_u64);      /* sort sites by call_inst */
    uint32_t *order = (uint32_t *)malloc(sizeof(uint32_t) * (n_call + 1));
    for (uint32_t a = 0; a < n_call; a++) order[a] = (uint32_t)(key[a] & 0xFFFFFFFFu);
    free(key);
    for (uint32_t a = 0; a < n_call; a++) {
      uint32_t e = order[a];
      in_e[fi[call_callee[e]]++] = e;
      out_e[fo[caller[e]]] = e; out_dst[fo[caller[e]]++] = call_callee[e];
    }
    free(fi); free(fo); free(order);
  }

  /* ---- Step 2: "if a function has samples and none of its incoming call edges
   * has a non-zero weight, we assign each of its incoming call edges a weight of one; we
   * repeat this propagation through callers".  Worklist to the least fixpoint (R11). */
  R->func_active = (uint8_t *)calloc(n_func + 1, 1);
  uint32_t *work = (uint32_t *)malloc(sizeof(uint32_t) * (n_func + 1));
  uint32_t nwork = 0;
  for (uint32_t f = 0; f < n_func; f++) {
    uint64_t s = 0;
    for (int r = 0; r < O_VALID; r++) s += R->S_f[(uint64_t)f * O_SLOTS + r];
    R->func_active[f] = s > 0;
    if (R->func_active[f]) work[nwork++] = f;
  }
  if (exact) nwork = 0;   /* exact counts: Step 2 is "for call graphs based on samples" (R24) */
  while (nwork > 0) {
    uint32_t f = work[--nwork];
    if (in_ptr[f + 1] == in_ptr[f]) continue;                 /* no incoming edges */
    int all_zero = 1;
    for (uint32_t k = in_ptr[f]; k < in_ptr[f + 1]; k++) if (R->w[in_e[k]] != 0) all_zero = 0;
    if (!all_zero) continue;
    for (uint32_t k = in_ptr[f]; k < in_ptr[f + 1]; k++) {
      uint32_t e = in_e[k];
      R->w[e] = 1;
      if (!R->func_active[caller[e]]) { R->func_active[caller[e]] = 1; work[nwork++] = caller[e]; }
    }
  }

  /* ---- Step 3: Tarjan SCCs of the static call graph; an SCC node stands for
   * its members, external calls into a member are linked to the SCC node, intra-SCC edges
   * are removed.  A component is non-trivial if it has >= 2 members or a self-call (R14).
   * DAG nodes are numbered by ascending smallest member function (R17). */
  o_tarjan T;
  T.n_func = n_func; T.out_ptr = out_ptr; T.out_dst = out_dst;
  T.index = (uint32_t *)malloc(sizeof(uint32_t) * (n_func + 1));
  T.low = (uint32_t *)malloc(sizeof(uint32_t) * (n_func + 1));
  T.stack = (uint32_t *)malloc(sizeof(uint32_t) * (n_func + 1));
  T.comp = (uint32_t *)malloc(sizeof(uint32_t) * (n_func + 1));
  T.on_stack = (uint8_t *)calloc(n_func + 1, 1);
  T.next_index = 0; T.sp = 0; T.n_comp = 0;
  for (uint32_t f = 0; f < n_func; f++) T.index[f] = O_NONE;
  for (uint32_t f = 0; f < n_func; f++) if (T.index[f] == O_NONE) o_strongconnect(&T, f);
  uint32_t n_comp = T.n_comp;
  uint32_t *comp_min = (uint32_t *)malloc(sizeof(uint32_t) * (n_comp + 1));
  for (uint32_t c = 0; c < n_comp; c++) comp_min[c] = O_NONE;
  for (uint32_t f = 0; f < n_func; f++) if (f < comp_min[T.comp[f]]) comp_min[T.comp[f]] = f;
  /* components ordered by smallest member: walking f ascending meets each component first
   * at its smallest member */
  uint32_t *comp_to_dag = (uint32_t *)malloc(sizeof(uint32_t) * (n_comp + 1));
  uint32_t n_dag = 0;
  for (uint32_t f = 0; f < n_func; f++) if (comp_min[T.comp[f]] == f) comp_to_dag[T.comp[f]] = n_dag++;
  R->n_dag = n_dag;
  R->scc_of = (uint32_t *)malloc(sizeof(uint32_t) * (n_func + 1));
  for (uint32_t f = 0; f < n_func; f++) R->scc_of[f] = comp_to_dag[T.comp[f]];
  uint32_t *n_members = (uint32_t *)calloc(n_dag + 1, sizeof(uint32_t));
  for (uint32_t f = 0; f < n_func; f++) n_members[R->scc_of[f]]++;
  R->dag_nontrivial = (uint8_t *)calloc(n_dag + 1, 1);
  for (uint32_t X = 0; X < n_dag; X++) R->dag_nontrivial[X] = n_members[X] >= 2;
  for (uint32_t e = 0; e < n_call; e++) if (caller[e] == call_callee[e]) R->dag_nontrivial[R->scc_of[caller[e]]] = 1;

  /* active_X = any member active; external in-edges of X = call sites into a member of X
   * from outside X. */
  R->dag_active = (uint8_t *)calloc(n_dag + 1, 1);
  for (uint32_t f = 0; f < n_func; f++) if (R->func_active[f]) R->dag_active[R->scc_of[f]] = 1;
  /* Guard (reading R12): the Step-2 rule once more on the DAG, to its fixpoint (samples
   * mode only, like Step 2 itself; R24). */
  int changed = !exact;
  while (changed) {
    changed = 0;
    for (uint32_t X = 0; X < n_dag; X++) {
      if (!R->dag_active[X]) continue;
      int has_ext = 0, all_zero = 1;
      for (uint32_t e = 0; e < n_call; e++) {
        if (R->scc_of[call_callee[e]] == X && R->scc_of[caller[e]] != X) {
          has_ext = 1;
          if (R->w[e] != 0) all_zero = 0;
        }
      }
      if (has_ext && all_zero) {
        for (uint32_t e = 0; e < n_call; e++) {
          if (R->scc_of[call_callee[e]] == X && R->scc_of[caller[e]] != X) {
            R->w[e] = 1;
            if (!R->dag_active[R->scc_of[caller[e]]]) R->dag_active[R->scc_of[caller[e]]] = 1;
          }
        }
        changed = 1;
      }
    }
  }
  /* W_X = total weight of the external calls into X ("the total number of calls
   * from all call sites"). */
  R->W = (uint64_t *)calloc(n_dag + 1, sizeof(uint64_t));
  int *has_ext_in = (int *)calloc(n_dag + 1, sizeof(int));
  for (uint32_t e = 0; e < n_call; e++) {
    uint32_t X = R->scc_of[call_callee[e]];
    if (R->scc_of[caller[e]] != X) { R->W[X] += R->w[e]; has_ext_in[X] = 1; }
  }

  /* ---- Step 4: split the DAG into a tree; like gprof assume every
   * invocation takes the same time and apportion each function's samples among its call
   * sites by the ratio of calls from each site to all calls (product form, reading R13:
   * f(child) = f(parent) * w_e / W_callee).  Breadth-first; the queue order IS the context
   * numbering (R17).  SCC contexts hold no samples and have one SCC_MEMBER child per
   * member in ascending function id (R14); members carry f * S_member. */
  uint32_t *dag_members_ptr = (uint32_t *)calloc(n_dag + 1, sizeof(uint32_t));
  uint32_t *dag_members = (uint32_t *)malloc(sizeof(uint32_t) * (n_func + 1));
  for (uint32_t f = 0; f < n_func; f++) dag_members_ptr[R->scc_of[f] + 1]++;
  for (uint32_t X = 0; X < n_dag; X++) dag_members_ptr[X + 1] += dag_members_ptr[X];
  {
    uint32_t *fill = (uint32_t *)malloc(sizeof(uint32_t) * (n_dag + 1));
    memcpy(fill, dag_members_ptr, sizeof(uint32_t) * n_dag);
    for (uint32_t f = 0; f < n_func; f++) dag_members[fill[R->scc_of[f]]++] = f;
    free(fill);
  }
  int oom = 0;
  for (uint32_t X = 0; X < n_dag; X++)
    if (!has_ext_in[X] && R->dag_active[X])
      oom |= o_append(R, R->dag_nontrivial[X] ? 1 : 0, X, O_NONE, O_NONE, 1.0);
  for (uint64_t c = 0; c < R->n && !oom; c++) {
    R->first_child[c] = (uint32_t)R->n;
    if (R->kind[c] == 1) {                                     /* SCC context */
      for (int r = 0; r < O_SLOTS; r++) R->excl[c * O_SLOTS + r] = 0.0;
      uint32_t X = R->node[c];
      for (uint32_t k = dag_members_ptr[X]; k < dag_members_ptr[X + 1]; k++)
        oom |= o_append(R, 2, dag_members[k], (uint32_t)c, O_NONE, R->frac[c]);
    } else {                                                   /* a function's context */
      uint32_t g = R->kind[c] == 2 ? R->node[c] : dag_members[dag_members_ptr[R->node[c]]];
      for (int r = 0; r < O_SLOTS; r++)
        R->excl[c * O_SLOTS + r] = R->frac[c] * (double)R->S_f[(uint64_t)g * O_SLOTS + r];
      for (uint32_t k = out_ptr[g]; k < out_ptr[g + 1]; k++) {
        uint32_t e = out_e[k];
        uint32_t Y = R->scc_of[call_callee[e]];
        if (Y == R->scc_of[g] || R->w[e] == 0) continue;
        double q = (double)R->w[e] / (double)R->W[Y];
        oom |= o_append(R, R->dag_nontrivial[Y] ? 1 : 0, Y, (uint32_t)c, e, R->frac[c] * q);
      }
    }
    R->n_children[c] = (uint32_t)(R->n - R->first_child[c]);
  }
  /* inclusive = exclusive + children's inclusive, children folded in index order */
  for (uint64_t c = R->n; c-- > 0 && !oom;) {
    for (int r = 0; r < O_SLOTS; r++) R->incl[c * O_SLOTS + r] = R->excl[c * O_SLOTS + r];
    for (uint32_t d = R->first_child[c]; d < R->first_child[c] + R->n_children[c]; d++)
      for (int r = 0; r < O_SLOTS; r++) R->incl[c * O_SLOTS + r] += R->incl[(uint64_t)d * O_SLOTS + r];
  }
  R->status = oom ? 4 : (R->n > max_contexts ? 3 : 0);

  free(inst_func); free(caller); free(in_ptr); free(in_e); free(out_ptr); free(out_e); free(out_dst);
  free(work); free(T.index); free(T.low); free(T.stack); free(T.comp); free(T.on_stack);
  free(comp_min); free(comp_to_dag); free(n_members); free(has_ext_in);
  free(dag_members_ptr); free(dag_members);
  return R;
}

oracle_cct_result *oracle_cct(uint32_t n_inst, const uint32_t *inst_scope,
                              uint32_t n_scope, const uint32_t *scope_parent,
                              uint32_t n_func, const uint32_t *func_scope,
                              uint32_t n_call, const uint32_t *call_inst, const uint32_t *call_callee,
                              const uint64_t *H, uint64_t max_contexts)
{
  return oracle_cct_mode(n_inst, inst_scope, n_scope, scope_parent, n_func, func_scope, n_call, call_inst,
                         call_callee, H, max_contexts, 0);
}

/* Exact counts from instrumentation ("count the execution frequency of each basic
 * block ... propagate the counts to each instruction in the block"): every instruction of
 * block b (instructions block_start[b] .. block_start[b+1]-1) gains count[b] executions in
 * slot 0 of H (an executed instruction "issued"; reading R24). */
void oracle_block_counts(uint32_t n_blocks, const uint32_t *block_start, const uint64_t *count, uint64_t *H)
{
  for (uint32_t b = 0; b < n_blocks; b++)
    for (uint32_t i = block_start[b]; i < block_start[b + 1]; i++) H[(uint64_t)i * O_SLOTS + 0] += count[b];
}

void oracle_cct_free(oracle_cct_result *R)
{
  if (!R) return;
  free(R->parent); free(R->site); free(R->node); free(R->first_child); free(R->n_children);
  free(R->kind); free(R->frac); free(R->excl); free(R->incl);
  free(R->w_step1); free(R->w); free(R->func_active); free(R->S_f); free(R->scc_of);
  free(R->dag_nontrivial); free(R->dag_active); free(R->W);
  free(R);
}

/* ======================================================================================
 * D8 — per-profile histograms and cross-profile statistics.  P:481-487:
 * "Built-in derived metrics for combining metrics from different thread profiles ... include
 * sum, min, mean, max, std. deviation, and coefficient of variation"; a profile is an
 * application thread, rank or GPU stream — here the record's `stream` field.
 * Per profile p, function f, slot r: Hp[p][f][r] = sum of counts of p's records attributed
 * (D1) to an instruction of f; records with stream >= n_prof land in profile row n_prof.
 * Statistics over p = 0..n_prof-1 of x_p = Hp[p][f][r] (reading R25): population convention,
 * computed exactly in integers before one conversion:
 *   sum = Σx, min, max, mean = Σx / P, std = sqrt(P·Σx² − (Σx)²) / P, cv = std / mean
 *   (cv = 0 when mean = 0).  Output [f][6][16]: 0 sum, 1 min, 2 mean, 3 max, 4 std, 5 cv.
 * ====================================================================================== */
void oracle_attribute_profiles(uint32_t n_inst, const uint64_t *inst_addr, const uint16_t *inst_len,
                               const uint32_t *inst_func, uint32_t n_func, const o_record *rec, uint64_t n,
                               uint32_t n_prof, uint64_t *Hp, uint64_t *Up)
{
  for (uint64_t k = 0; k < n; k++) {
    uint64_t pc = rec[k].pc;
    uint32_t slot = rec[k].stall < O_VALID ? rec[k].stall : O_INVALID;
    uint32_t p = rec[k].stream < n_prof ? rec[k].stream : n_prof;
    int64_t j = o_last_start_le(inst_addr, n_inst, pc);
    if (j >= 0 && pc < inst_addr[j] + inst_len[j])
      Hp[((uint64_t)p * n_func + inst_func[j]) * O_SLOTS + slot] += rec[k].count;
    else
      Up[(uint64_t)p * O_SLOTS + slot] += rec[k].count;
  }
}

void oracle_profile_stats(uint32_t n_prof, uint32_t rows, const uint64_t *Hp, double *out)
{
  for (uint32_t f = 0; f < rows; f++) {
    for (int r = 0; r < O_SLOTS; r++) {
      unsigned __int128 sum = 0, sq = 0;
      uint64_t mn = UINT64_MAX, mx = 0;
      for (uint32_t p = 0; p < n_prof; p++) {
        uint64_t x = Hp[((uint64_t)p * rows + f) * O_SLOTS + r];
        sum += x;
        sq += (unsigned __int128)x * x;
        if (x < mn) mn = x;
        if (x > mx) mx = x;
      }
      double *o = out + (uint64_t)f * 6 * O_SLOTS;
      double P = (double)n_prof, S = (double)sum;
      unsigned __int128 num = (unsigned __int128)n_prof * sq - sum * sum;   /* P·Σx² − (Σx)² ≥ 0 */
      double mean = n_prof ? S / P : 0.0;
      double sd = n_prof ? sqrt((double)num) / P : 0.0;
      o[0 * O_SLOTS + r] = S;
      o[1 * O_SLOTS + r] = n_prof ? (double)mn : 0.0;
      o[2 * O_SLOTS + r] = mean;
      o[3 * O_SLOTS + r] = (double)mx;
      o[4 * O_SLOTS + r] = sd;
      o[5 * O_SLOTS + r] = mean == 0.0 ? 0.0 : sd / mean;
    }
  }
}

/* ======================================================================================
 * D9 — sparse cube formats (§5.2, Fig. sf).  The cube is
 * the per-profile histogram Hp[p][c][m] (p < P, c < C, m < 16; "context" = the function row,
 * metric = the slot).  Like CSR but over planes:
 *   CMS (context-major): plane c holds its non-zeros ordered by (metric, profile) as vals[]
 *     and pids[]; its sparse metric index is a list of (metric id, start) pairs for the
 *     non-empty metrics followed by a sentinel (GPA_NONE, end) ("we make midxs a sparse
 *     array: each entry is a pair of metric ID and this metric's starting index").
 *   PMS (profile-major): plane p holds its non-zeros ordered by (context, metric) as vals[]
 *     and mids[]; its sparse context index lists (context id, start) + sentinel.
 * plane_off[q] / index_off[q] give where plane q starts in the value / index arrays
 * ("a vector of ... offsets, one per ..."); element offsets, not bytes.
 * ====================================================================================== */
typedef struct {
  uint32_t n_planes; uint64_t n_values, n_index;
  uint64_t *plane_off, *index_off, *vals, *index_start;
  uint32_t *ids, *index_id;
} oracle_sparse;

oracle_sparse *oracle_sparse_build(const uint64_t *Hp, uint32_t P, uint32_t C, int cms)
{
  oracle_sparse *S = (oracle_sparse *)calloc(1, sizeof(oracle_sparse));
  uint32_t planes = cms ? C : P, inner = cms ? O_SLOTS : C, leaf = cms ? P : O_SLOTS;
  S->n_planes = planes;
  uint64_t nv = 0, ni = 0;
  for (uint64_t x = 0; x < (uint64_t)P * C * O_SLOTS; x++) nv += Hp[x] != 0;
  /* index entries: one per non-empty (plane, inner) pair, plus a sentinel per plane */
  for (uint32_t a = 0; a < planes; a++) {
    for (uint32_t b = 0; b < inner; b++) {
      int any = 0;
      for (uint32_t l = 0; l < leaf; l++) {
        uint64_t v = cms ? Hp[((uint64_t)l * C + a) * O_SLOTS + b] : Hp[((uint64_t)a * C + b) * O_SLOTS + l];
        if (v) any = 1;
      }
      ni += any;
    }
    ni += 1;
  }
  S->n_values = nv; S->n_index = ni;
  S->plane_off = (uint64_t *)malloc(sizeof(uint64_t) * (planes + 1));
  S->index_off = (uint64_t *)malloc(sizeof(uint64_t) * (planes + 1));
  S->vals = (uint64_t *)malloc(sizeof(uint64_t) * (nv + 1));
  S->ids = (uint32_t *)malloc(sizeof(uint32_t) * (nv + 1));
  S->index_start = (uint64_t *)malloc(sizeof(uint64_t) * (ni + 1));
  S->index_id = (uint32_t *)malloc(sizeof(uint32_t) * (ni + 1));
  uint64_t v0 = 0, i0 = 0;
  for (uint32_t a = 0; a < planes; a++) {
    S->plane_off[a] = v0; S->index_off[a] = i0;
    for (uint32_t b = 0; b < inner; b++) {
      uint64_t start = v0;
      for (uint32_t l = 0; l < leaf; l++) {
        uint64_t v = cms ? Hp[((uint64_t)l * C + a) * O_SLOTS + b] : Hp[((uint64_t)a * C + b) * O_SLOTS + l];
        if (v) { S->vals[v0] = v; S->ids[v0] = l; v0++; }
      }
      if (v0 > start) { S->index_id[i0] = b; S->index_start[i0] = start; i0++; }
    }
    S->index_id[i0] = O_NONE; S->index_start[i0] = v0; i0++;   /* sentinel: end of plane */
  }
  S->plane_off[planes] = v0; S->index_off[planes] = i0;
  return S;
}

void oracle_sparse_free(oracle_sparse *S)
{
  if (!S) return;
  free(S->plane_off); free(S->index_off); free(S->vals); free(S->ids); free(S->index_start); free(S->index_id);
  free(S);
}

/* ======================================================================================
 * D7 — derived metrics ("based on the number of total PC samples (S) and
 * stalled PC samples (S_stall), we can estimate the Warp Issue Rate (W) of schedulers as
 * W = (S - S_stall)/S"; "stall percentages").  S = sum of the 12 valid slots;
 * S_stall = S - v[0] (slot 0 = issued, reading R3).  Columns:
 *   0 S   1 W   2 latency-hiding (v0+v9)/S   3 latency-stall sum_{LAT} v/S (R4)
 *   4..15 v[r]/S   16 v[15] (invalid)   17..32 MIX[k]/S (R5; NaN for CCT rows)
 * S == 0: every ratio column is the canonical quiet NaN (R18).
 * ====================================================================================== */
static double o_nan(void)
{
  union { uint64_t u; double d; } x;
  x.u = 0x7FF8000000000000ull;
  return x.d;
}

/* latency stalls: every valid reason except issued (0) and not-selected (9) (R4) */
static int o_is_lat(int r) { return r >= 1 && r <= 11 && r != 9; }

void oracle_derive_u64(uint64_t rows, const uint64_t *V, const uint64_t *MIX, double *out)
{
  for (uint64_t i = 0; i < rows; i++) {
    const uint64_t *v = V + i * O_SLOTS;
    double *o = out + i * O_NCOLS;
    uint64_t S = 0, lat = 0;
    for (int r = 0; r < O_VALID; r++) S += v[r];
    for (int r = 0; r < O_VALID; r++) if (o_is_lat(r)) lat += v[r];
    double Sd = (double)S;
    o[0] = Sd;
    o[16] = (double)v[O_INVALID];
    if (S == 0) {
      for (int c = 1; c < O_NCOLS; c++) if (c != 16) o[c] = o_nan();
      continue;
    }
    o[1] = (double)v[0] / Sd;                      /* W = (S - S_stall)/S, S_stall = S - v0 */
    o[2] = (double)(v[0] + v[9]) / Sd;
    o[3] = (double)lat / Sd;
    for (int r = 0; r < O_VALID; r++) o[4 + r] = (double)v[r] / Sd;
    for (int k = 0; k < 16; k++) o[17 + k] = MIX ? (double)MIX[i * O_SLOTS + k] / Sd : o_nan();
  }
}

void oracle_derive_f64(uint64_t rows, const double *V, double *out)
{
  for (uint64_t i = 0; i < rows; i++) {
    const double *v = V + i * O_SLOTS;
    double *o = out + i * O_NCOLS;
    double S = 0.0, lat = 0.0;
    for (int r = 0; r < O_VALID; r++) S += v[r];
    for (int r = 0; r < O_VALID; r++) if (o_is_lat(r)) lat += v[r];
    o[0] = S;
    o[16] = v[O_INVALID];
    if (S == 0.0) {
      for (int c = 1; c < O_NCOLS; c++) if (c != 16) o[c] = o_nan();
      continue;
    }
    o[1] = v[0] / S;
    o[2] = (v[0] + v[9]) / S;
    o[3] = lat / S;
    for (int r = 0; r < O_VALID; r++) o[4 + r] = v[r] / S;
    for (int k = 0; k < 16; k++) o[17 + k] = o_nan();
  }
}

/* ======================================================================================
 * D10 — GPU-idleness blame ("it identifies times when all GPU streams are idle
 * and at least one CPU thread is active. In such cases, it partitions the cost of GPU
 * idleness among routines being executed by active CPU threads"; SPEC's blame_idleness:
 * equal division among the active CPU threads; reading R27).
 * A trace line is a sequence of change points (time, ctx), non-decreasing in time: from
 * time[i] to time[i+1] the line is in state ctx[i] (GPA NONE = idle); after its last change
 * point a line is idle.  Lines are grouped into scopes (ranks); for each scope, sweep the
 * union of its lines' change-point times: on every elementary interval [ta, tb) with all of
 * the scope's GPU lines idle, gpu_idle += tb-ta; if also k >= 1 CPU lines are active,
 * total += tb-ta and each active CPU line adds tb-ta to num[scope][its routine][k].
 * blame = sum_{k=1..kmax} num/k (one division and one addition per k, ascending k);
 * share = blame / total (NaN when total = 0).  Returns 0, or -1 when a line goes back in
 * time, a CPU routine id is >= n_routines, a scope has no GPU line, or the lines are not
 * grouped by non-decreasing scope.
 * ====================================================================================== */
static int o_cmp_u64b(const void *a, const void *b)
{
  uint64_t x = *(const uint64_t *)a, y = *(const uint64_t *)b;
  return x < y ? -1 : x > y;
}

int oracle_blame(uint32_t n_lines, const uint64_t *line_off, const uint8_t *line_kind, const uint32_t *line_scope,
                 const uint64_t *time, const uint32_t *ctx, uint32_t n_scopes, uint32_t n_routines, uint32_t kmax,
                 uint64_t *num, uint64_t *total, uint64_t *gpu_idle, double *blame, double *share)
{
  const uint64_t kw = (uint64_t)kmax + 1;
  memset(num, 0, sizeof(uint64_t) * n_scopes * n_routines * kw);
  memset(total, 0, sizeof(uint64_t) * n_scopes);
  memset(gpu_idle, 0, sizeof(uint64_t) * n_scopes);
  for (uint32_t l = 0; l < n_lines; l++) {
    if (line_scope[l] >= n_scopes || (l && line_scope[l] < line_scope[l - 1])) return -1;
    for (uint64_t e = line_off[l]; e < line_off[l + 1]; e++) {
      if (e > line_off[l] && time[e] < time[e - 1]) return -1;
      if (line_kind[l] == 1 && ctx[e] != O_NONE && ctx[e] >= n_routines && e + 1 < line_off[l + 1]) return -1;
    }
  }
  uint32_t l0 = 0;
  for (uint32_t sc = 0; sc < n_scopes; sc++) {
    uint32_t l1 = l0;
    while (l1 < n_lines && line_scope[l1] == sc) l1++;
    uint32_t n_gpu = 0, n_cpu = 0;
    uint64_t n_ev = 0;
    for (uint32_t l = l0; l < l1; l++) {
      if (line_kind[l] == 0) n_gpu++; else n_cpu++;
      n_ev += line_off[l + 1] - line_off[l];
    }
    if (n_gpu == 0 || n_cpu > kmax) return -1;
    uint64_t *ts = (uint64_t *)malloc(sizeof(uint64_t) * (n_ev ? n_ev : 1));
    uint64_t *cur = (uint64_t *)calloc(l1 - l0 + 1, sizeof(uint64_t));
    uint64_t m = 0;
    for (uint32_t l = l0; l < l1; l++)
      for (uint64_t e = line_off[l]; e < line_off[l + 1]; e++) ts[m++] = time[e];
    qsort(ts, m, sizeof(uint64_t), o_cmp_u64b);
    for (uint64_t i = 0; i + 1 < m; i++) {
      const uint64_t ta = ts[i], tb = ts[i + 1];
      if (ta == tb) continue;
      uint32_t cov = 0, k = 0;
      for (uint32_t l = l0; l < l1; l++) {   /* state of every line on [ta, tb) */
        const uint64_t len = line_off[l + 1] - line_off[l];
        while (cur[l - l0] < len && time[line_off[l] + cur[l - l0]] <= ta) cur[l - l0]++;
        const uint64_t c = cur[l - l0];
        const int active = c > 0 && c < len && ctx[line_off[l] + c - 1] != O_NONE;
        if (active) { if (line_kind[l] == 0) cov++; else k++; }
      }
      if (cov) continue;
      gpu_idle[sc] += tb - ta;
      if (!k) continue;
      total[sc] += tb - ta;
      for (uint32_t l = l0; l < l1; l++) {
        if (line_kind[l] != 1) continue;
        const uint64_t len = line_off[l + 1] - line_off[l], c = cur[l - l0];
        if (c > 0 && c < len && ctx[line_off[l] + c - 1] != O_NONE)
          num[((uint64_t)sc * n_routines + ctx[line_off[l] + c - 1]) * kw + k] += tb - ta;
      }
    }
    free(ts);
    free(cur);
    l0 = l1;
  }
  if (l0 != n_lines) return -1;
  for (uint32_t sc = 0; sc < n_scopes; sc++)
    for (uint32_t r = 0; r < n_routines; r++) {
      const uint64_t *v = num + ((uint64_t)sc * n_routines + r) * kw;
      double b = 0.0;
      for (uint32_t k = 1; k <= kmax; k++) b = b + (double)v[k] / (double)k;
      blame[(uint64_t)sc * n_routines + r] = b;
      share[(uint64_t)sc * n_routines + r] = total[sc] ? b / (double)total[sc] : o_nan();
    }
  return 0;
}

/* ======================================================================================
 * D11 — f1 at CCT level (SURVEY §8f f1 "per instruction, function or CCT context"; P:481-487
 * statistics over thread profiles of each CCT node; P:711-714 values propagated up the CCT).
 * Reading R28: the unified CCT is the tree reconstructed from the aggregate histogram (R9);
 * profile p's exclusive value at a FUNC / SCC_MEMBER context c of function g is
 * excl_p(c)[r] = frac(c) * (double)Hp[p][g][r] (the aggregate formula of D6 with p's function
 * histogram), 0 at SCC contexts; incl_p(c) = excl_p(c) + the children's incl_p in index order.
 * ctx_func[c] = the context's function (GPA NONE for SCC contexts).  Cubes are [P1][n][16].
 * Statistics of fp64 values over profiles 0..n_prof-1 (R28): sum = left fold in profile order,
 * min, max, mean = sum / P, std = sqrt(sum_p (x - mean)^2 / P) (two passes), cv = std / mean
 * (0 when mean = 0); all zero when n_prof = 0.  Output [rows][6][16] as in D8.
 * ====================================================================================== */
void oracle_cct_profiles(uint64_t n, const uint32_t *ctx_func, const double *frac, const uint32_t *first_child,
                         const uint32_t *n_children, uint32_t P1, uint32_t n_func, const uint64_t *Hp,
                         double *excl, double *incl)
{
  for (uint32_t p = 0; p < P1; p++) {
    double *E = excl + (uint64_t)p * n * O_SLOTS, *I = incl + (uint64_t)p * n * O_SLOTS;
    for (uint64_t c = 0; c < n; c++)
      for (int r = 0; r < O_SLOTS; r++)
        E[c * O_SLOTS + r] = ctx_func[c] == O_NONE ? 0.0
                           : frac[c] * (double)Hp[((uint64_t)p * n_func + ctx_func[c]) * O_SLOTS + r];
    for (uint64_t c = n; c-- > 0;)
      for (int r = 0; r < O_SLOTS; r++) {
        double v = E[c * O_SLOTS + r];
        for (uint32_t d = first_child[c]; d < first_child[c] + n_children[c]; d++) v = v + I[(uint64_t)d * O_SLOTS + r];
        I[c * O_SLOTS + r] = v;
      }
  }
}

void oracle_profile_stats_f64(uint32_t n_prof, uint64_t rows, const double *X, double *out)
{
  for (uint64_t f = 0; f < rows; f++)
    for (int r = 0; r < O_SLOTS; r++) {
      double sum = 0.0, mn = 0.0, mx = 0.0;
      for (uint32_t p = 0; p < n_prof; p++) {
        double x = X[((uint64_t)p * rows + f) * O_SLOTS + r];
        sum = sum + x;
        if (p == 0 || x < mn) mn = x;
        if (p == 0 || x > mx) mx = x;
      }
      double mean = n_prof ? sum / (double)n_prof : 0.0, ss = 0.0;
      for (uint32_t p = 0; p < n_prof; p++) {
        double d = X[((uint64_t)p * rows + f) * O_SLOTS + r] - mean;
        ss = ss + d * d;
      }
      double sd = n_prof ? sqrt(ss / (double)n_prof) : 0.0;
      double *o = out + f * 6 * O_SLOTS;
      o[0 * O_SLOTS + r] = sum;
      o[1 * O_SLOTS + r] = mn;
      o[2 * O_SLOTS + r] = mean;
      o[3 * O_SLOTS + r] = mx;
      o[4 * O_SLOTS + r] = sd;
      o[5 * O_SLOTS + r] = mean == 0.0 ? 0.0 : sd / mean;
    }
}
