/* gen_host.c — host build of the counter-based record generator (INPUT GENERATION ONLY;
 * see gen_core.h).  Multi-threaded over contiguous record ranges; bit-identical to
 * gen_dev.cu because every record is a pure function of (seed, k). */
#include <pthread.h>
#include <stdlib.h>
#include "gen_core.h"

typedef struct { const gen_tables *T; uint64_t k0, n; gen_record *out; } gen_job;

static void *gen_thread(void *p)
{
  gen_job *j = (gen_job *)p;
  for (uint64_t x = 0; x < j->n; x++) j->out[x] = gen_one(j->T, j->k0 + x);
  return NULL;
}

int gen_records_host(const gen_tables *T, uint64_t k0, uint64_t n, gen_record *out, int n_threads)
{
  if (n_threads < 1) n_threads = 1;
  if ((uint64_t)n_threads > n / 4096 + 1) n_threads = (int)(n / 4096 + 1);
  gen_job *jobs = (gen_job *)calloc((size_t)n_threads, sizeof(gen_job));
  pthread_t *th = (pthread_t *)calloc((size_t)n_threads, sizeof(pthread_t));
  if (!jobs || !th) { free(jobs); free(th); return -1; }
  for (int t = 0; t < n_threads; t++) {
    uint64_t a = n * (uint64_t)t / (uint64_t)n_threads, b = n * (uint64_t)(t + 1) / (uint64_t)n_threads;
    jobs[t].T = T; jobs[t].k0 = k0 + a; jobs[t].n = b - a; jobs[t].out = out + a;
    pthread_create(&th[t], NULL, gen_thread, &jobs[t]);
  }
  for (int t = 0; t < n_threads; t++) pthread_join(th[t], NULL);
  free(jobs); free(th);
  return 0;
}

/* Walker/Vose alias table over n non-negative weights (sum > 0) in 32-bit fixed point:
 * entry j is accepted when coin < prob[j], else alias[j] (see gen_alias in gen_core.h). */
int gen_build_alias(const double *w, uint64_t n, uint32_t *prob, uint32_t *alias)
{
  if (n == 0) return -1;
  double sum = 0.0;
  for (uint64_t j = 0; j < n; j++) sum += w[j];
  if (!(sum > 0.0)) return -1;
  double *q = (double *)malloc(sizeof(double) * n);
  uint64_t *small = (uint64_t *)malloc(sizeof(uint64_t) * n), *large = (uint64_t *)malloc(sizeof(uint64_t) * n);
  uint64_t ns = 0, nl = 0;
  for (uint64_t j = 0; j < n; j++) {
    q[j] = w[j] * (double)n / sum;
    if (q[j] < 1.0) small[ns++] = j; else large[nl++] = j;
  }
  while (ns && nl) {
    uint64_t s = small[--ns], l = large[nl - 1];
    double p = q[s] * 4294967296.0;
    prob[s] = p >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)p;
    alias[s] = (uint32_t)l;
    q[l] = (q[l] + q[s]) - 1.0;
    if (q[l] < 1.0) { nl--; small[ns++] = l; }
  }
  while (nl) { uint64_t l = large[--nl]; prob[l] = 0xFFFFFFFFu; alias[l] = (uint32_t)l; }
  while (ns) { uint64_t s = small[--ns]; prob[s] = 0xFFFFFFFFu; alias[s] = (uint32_t)s; }
  free(q); free(small); free(large);
  return 0;
}
