/*
 * gen_core.h — counter-based synthetic PC-sample record generator (INPUT GENERATION ONLY).
 *
 * Record k of a workload is a pure function of (seed, k) and the workload tables, so any
 * shard / chunk can be produced independently and the host (gen_host.c) and device
 * (gen_dev.cu) builds produce bit-identical streams.  This file holds none of the
 * analysis method's arithmetic (no attribution, roll-up, CCT or metric code): it draws an
 * instruction from a per-kernel Walker alias table, a stall reason from the instruction's
 * cumulative table, a count, and plants the corruption / skew cases DESIGN.md §4 lists.
 * Shared by tests, bench.py and smoke() on both sides of the parity check.
 */
#ifndef GEN_CORE_H
#define GEN_CORE_H
#include <stdint.h>

#if defined(__CUDACC__)
#define GEN_HD __host__ __device__ __forceinline__
#else
#define GEN_HD static inline
#endif

typedef struct { uint64_t pc; uint32_t count; uint16_t stall; uint16_t stream; } gen_record;

typedef struct {
  uint64_t seed;
  uint32_t burst_shift;          /* records per burst = 1 << burst_shift (one kernel/burst)    */
  uint32_t n_kernels;
  const uint32_t *kern_prob;     /* [n_kernels] alias acceptance thresholds (u32)              */
  const uint32_t *kern_alias;    /* [n_kernels]                                                */
  const uint64_t *reach_off;     /* [n_kernels+1] offsets into the reach tables                */
  const uint32_t *reach_prob;    /* [total] alias thresholds                                   */
  const uint32_t *reach_alias;   /* [total] alias partner (local index)                        */
  const uint32_t *reach_inst;    /* [total] instruction index of each entry                    */
  const uint32_t *stall_cum;     /* [n_inst*12] cumulative thresholds over 2^31                */
  const uint64_t *inst_addr;     /* [n_inst]                                                   */
  const uint16_t *inst_len;      /* [n_inst]                                                   */
  uint32_t n_probe;
  const uint64_t *probe_pc;      /* [n_probe] unmapped addresses (gaps, below/above module)   */
  uint32_t n_streams;
  const uint64_t *stream_first_burst; /* [n_streams] ascending, [0] = 0                        */
  uint32_t corrupt_pc_thresh;    /* P(out-of-range pc)      * 2^32                             */
  uint32_t corrupt_stall_thresh; /* P(invalid stall code)   * 2^32                             */
  uint32_t misalign_thresh;      /* P(pc inside, not at start, of its instruction) * 2^32      */
  uint32_t hot_inst;             /* planted hot bin (C5): instruction                          */
  uint64_t hot_records;          /* number of planted records (0 = none)                       */
  uint64_t hot_stride;           /* record k is planted iff k % stride == 0 && k/stride < n    */
} gen_tables;

GEN_HD uint64_t gen_mix64(uint64_t z)
{
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

GEN_HD uint64_t gen_rand(uint64_t seed, uint64_t k, uint32_t lane)
{
  return gen_mix64(gen_mix64(seed) ^ (k * 8u + lane));
}

/* Walker alias draw over n entries: 32 bits pick the column, 32 bits the coin. */
GEN_HD uint32_t gen_alias(const uint32_t *prob, const uint32_t *alias, uint64_t n, uint64_t r)
{
  uint32_t j = (uint32_t)(((r >> 32) * n) >> 32);
  uint32_t coin = (uint32_t)r;
  return coin < prob[j] ? j : alias[j];
}

GEN_HD uint32_t gen_ctz64(uint64_t x)
{
  uint32_t c = 0;
  while (!(x & 1ull)) { x >>= 1; c++; }
  return c;
}

GEN_HD gen_record gen_one(const gen_tables *T, uint64_t k)
{
  gen_record rec;
  uint64_t b = k >> T->burst_shift;
  /* kernel of this burst */
  uint64_t hb = gen_rand(T->seed ^ 0xB5297A4D3F84D5B5ull, b, 7);
  uint32_t kern = gen_alias(T->kern_prob, T->kern_alias, T->n_kernels, hb);
  uint64_t r0 = gen_rand(T->seed, k, 0), r1 = gen_rand(T->seed, k, 1);
  uint64_t r2 = gen_rand(T->seed, k, 2), r3 = gen_rand(T->seed, k, 3);
  uint64_t off = T->reach_off[kern], cnt = T->reach_off[kern + 1] - off;
  uint32_t j = gen_alias(T->reach_prob + off, T->reach_alias + off, cnt, r0);
  uint32_t i = T->reach_inst[off + j];
  /* stall reason from the instruction's cumulative table (31-bit coin) */
  uint32_t u = (uint32_t)(r1 >> 33);
  uint32_t stall = 11;
  for (uint32_t r = 0; r < 12; r++) {
    if (u < T->stall_cum[(uint64_t)i * 12 + r]) { stall = r; break; }
  }
  uint32_t count = 1 + gen_ctz64(r2 | (1ull << 63));  /* 1 + Geometric(1/2) */
  uint64_t pc = T->inst_addr[i];
  uint32_t c = (uint32_t)r3, hi = (uint32_t)(r3 >> 32);
  if (c < T->corrupt_pc_thresh) {
    if (T->n_probe) pc = T->probe_pc[hi % T->n_probe];
  } else if (c - T->corrupt_pc_thresh < T->corrupt_stall_thresh) {
    stall = 12 + hi % (65536u - 12u);
  } else if (c - T->corrupt_pc_thresh - T->corrupt_stall_thresh < T->misalign_thresh) {
    pc += hi % T->inst_len[i];
  }
  if (T->hot_records && k % T->hot_stride == 0 && k / T->hot_stride < T->hot_records) {
    pc = T->inst_addr[T->hot_inst]; stall = 5; count = 65536;
  }
  /* stream (profile slot) of this burst: last stream whose first burst <= b */
  uint32_t lo = 0, hi_s = T->n_streams;
  while (lo < hi_s) {
    uint32_t mid = (lo + hi_s) >> 1;
    if (T->stream_first_burst[mid] <= b) lo = mid + 1; else hi_s = mid;
  }
  rec.pc = pc; rec.count = count; rec.stall = (uint16_t)stall; rec.stream = (uint16_t)(lo - 1);
  return rec;
}

#endif
