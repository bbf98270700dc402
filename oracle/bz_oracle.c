/*
 * bz_oracle.c -- CPU restatement of the reference's enumeration path.
 *
 * TEST INFRASTRUCTURE ONLY.  Imported by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs, and only as the
 * checker or the reported CPU baseline -- never by the product path
 * (paper_1603_06757_b200/), which fails loudly without its CUDA library.
 *
 * Restates, in plain C + pthreads, pkg/src/mindist/ of the reference:
 *   bzo_min_stack   <- enumerate_stack   (enumeration.py:128-178): lex walk
 *                      over (g-1)-prefixes with a stack of incremental prefix
 *                      XORs rebuilt from the leftmost changed position, inner
 *                      loop (top ^ rows[e]).bit_count() for e in (last, k);
 *                      g == 1 goes through enumerate_basic (:76-93) as the
 *                      reference does (:138-139).
 *   bzo_hist_stack  <- same walk, recording every weight (the reference keeps
 *                      only the minimum; this is the config-4 checksum).
 *   bzo_brute       <- brute_force_distance (engine.py:223-237): Gray-code
 *                      walk over all 2^k - 1 messages, one row XOR per step.
 * Rows are the BitMatrix.to_numpy() 64-bit image (gf2.py:74-79): w64
 * little-endian words per row, bit j = column j, zero padding.
 *
 * Parallelism: the (g-1)-prefixes are split by their first element c_1 and
 * handed to pthreads dynamically -- the same unit-of-work idea as the
 * reference's enumerate_parallel (enumeration.py:385-444), with per-thread
 * minima merged once.  The result is schedule-independent.
 */
#define _GNU_SOURCE
#include <stdint.h>
#include <string.h>
#include <pthread.h>
#include <sched.h>
#include <stdlib.h>
#include <unistd.h>

#define BZO_MAXW 8
#define BZO_MAXG 130

/* Host threads usable by this process (sched affinity). */
int bzo_max_threads(void) {
  cpu_set_t set;
  if (sched_getaffinity(0, sizeof set, &set) == 0) {
    const int n = CPU_COUNT(&set);
    if (n > 0) return n;
  }
  const long n = sysconf(_SC_NPROCESSORS_ONLN);
  return n > 0 ? (int)n : 1;
}

static inline int weight_xor(const uint64_t *a, const uint64_t *b, int w64) {
  int w = 0;
  for (int j = 0; j < w64; ++j) w += __builtin_popcountll(a[j] ^ b[j]);
  return w;
}

static inline int weight_of(const uint64_t *a, int w64) {
  int w = 0;
  for (int j = 0; j < w64; ++j) w += __builtin_popcountll(a[j]);
  return w;
}

/* Walk every (g-1)-prefix whose first `head` elements are c1 (and c2 when
 * head == 2) in lex order with a stack of prefix XORs, and visit the
 * codewords top ^ rows[e], e in (last, k).  hist == NULL: minimum only. */
static void walk_head(const uint64_t *rows, int k, int w64, int g, int head,
                      int c1, int c2, int *best, uint64_t *combos, uint64_t *hist) {
  const int depth = g - 1;
  int pre[BZO_MAXG];
  uint64_t stack[BZO_MAXG][BZO_MAXW];
  pre[0] = c1;
  if (head == 2) pre[1] = c2;
  for (int t = head; t < depth; ++t) pre[t] = pre[t - 1] + 1;
  if (pre[depth - 1] > k - 1) return;
  int rebuild_from = 0;
  for (;;) {
    const int last = pre[depth - 1];
    if (last < k - 1) {
      for (int t = rebuild_from; t < depth; ++t) {
        const uint64_t *r = rows + (size_t)pre[t] * w64;
        if (t == 0) {
          memcpy(stack[0], r, sizeof(uint64_t) * w64);
        } else {
          for (int j = 0; j < w64; ++j) stack[t][j] = stack[t - 1][j] ^ r[j];
        }
      }
      rebuild_from = depth;
      const uint64_t *top = stack[depth - 1];
      int b = *best;
      if (hist) {
        for (int e = last + 1; e < k; ++e) {
          const int w = weight_xor(top, rows + (size_t)e * w64, w64);
          hist[w] += 1;
          if (w < b) b = w;
        }
      } else {
        for (int e = last + 1; e < k; ++e) {
          const int w = weight_xor(top, rows + (size_t)e * w64, w64);
          if (w < b) b = w;
        }
      }
      *best = b;
      *combos += (uint64_t)(k - 1 - last);
    }
    /* lexicographic successor restricted to prefixes with this head */
    int t = depth - 1;
    while (t >= head && pre[t] >= k - depth + t) --t;
    if (t < head) break;
    pre[t] += 1;
    for (int u = t + 1; u < depth; ++u) pre[u] = pre[u - 1] + 1;
    if (t < rebuild_from) rebuild_from = t;
  }
}

/* Work sharing: threads pull units from an atomic cursor.  A unit is the
 * prefix head (c1) when g == 2, else the pair (c1, c2) -- about k^2/2 units,
 * fine enough to keep a many-core host balanced. */
typedef struct {
  const uint64_t *rows;
  int k, w64, g;
  int next; /* atomic cursor over units */
  int want_hist;
} job_t;

typedef struct {
  job_t *job;
  int best;
  uint64_t combos;
  uint64_t hist[64 * BZO_MAXW + 1];
} worker_t;

static void *worker_main(void *arg) {
  worker_t *wk = (worker_t *)arg;
  job_t *jb = wk->job;
  const int k = jb->k;
  const int head = jb->g == 2 ? 1 : 2;
  const int units = head == 1 ? k : k * k;
  for (;;) {
    const int u = __atomic_fetch_add(&jb->next, 1, __ATOMIC_RELAXED);
    if (u >= units) break;
    const int c1 = head == 1 ? u : u / k;
    const int c2 = head == 1 ? 0 : u % k;
    if (head == 2 && c2 <= c1) continue;
    walk_head(jb->rows, k, jb->w64, jb->g, head, c1, c2, &wk->best, &wk->combos,
              jb->want_hist ? wk->hist : NULL);
  }
  return NULL;
}

static int run_workers(job_t *jb, int nthreads, int *best, uint64_t *combos,
                       uint64_t *hist) {
  if (nthreads < 1) nthreads = bzo_max_threads();
  if (nthreads > 256) nthreads = 256;
  worker_t *ws = (worker_t *)calloc((size_t)nthreads, sizeof(worker_t));
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  if (!ws || !th) { free(ws); free(th); return 4; }
  for (int i = 0; i < nthreads; ++i) {
    ws[i].job = jb;
    ws[i].best = 0x7fffffff;
  }
  int started = 0;
  for (int i = 1; i < nthreads; ++i)
    if (pthread_create(&th[i], NULL, worker_main, &ws[i]) == 0) started = i; else break;
  worker_main(&ws[0]);
  for (int i = 1; i <= started; ++i) pthread_join(th[i], NULL);
  int b = 0x7fffffff;
  uint64_t c = 0;
  for (int i = 0; i < nthreads; ++i) {
    if (ws[i].best < b) b = ws[i].best;
    c += ws[i].combos;
    if (hist)
      for (int w = 0; w <= 64 * BZO_MAXW; ++w) hist[w] += ws[i].hist[w];
  }
  *best = b;
  *combos = c;
  free(ws);
  free(th);
  return 0;
}

/* Minimum weight over all g-combinations of the k rows (unclipped).
 * nthreads < 1: all online cores. */
int bzo_min_stack(const uint64_t *rows, int k, int w64, int g, int nthreads,
                  int32_t *out_min, uint64_t *out_combos) {
  if (g < 1 || g > k) return 1;
  if (w64 < 1 || w64 > BZO_MAXW || g > BZO_MAXG) return 3;
  if (g == 1) {
    int best = 0x7fffffff;
    for (int e = 0; e < k; ++e) {
      const int w = weight_of(rows + (size_t)e * w64, w64);
      if (w < best) best = w;
    }
    *out_min = best;
    *out_combos = (uint64_t)k;
    return 0;
  }
  job_t jb = {rows, k, w64, g, 0, 0};
  int best;
  uint64_t combos;
  const int rc = run_workers(&jb, nthreads, &best, &combos, NULL);
  if (rc) return rc;
  *out_min = best;
  *out_combos = combos;
  return 0;
}

/* Weight histogram into hist[0..nbins) (nbins >= n + 1). */
int bzo_hist_stack(const uint64_t *rows, int k, int w64, int g, int nthreads,
                   uint64_t *hist, int nbins) {
  if (g < 1 || g > k) return 1;
  if (w64 < 1 || w64 > BZO_MAXW || g > BZO_MAXG) return 3;
  if (nbins < 1) return 2;
  memset(hist, 0, sizeof(uint64_t) * (size_t)nbins);
  if (g == 1) {
    for (int e = 0; e < k; ++e) {
      const int w = weight_of(rows + (size_t)e * w64, w64);
      if (w < nbins) hist[w] += 1; else return 2;
    }
    return 0;
  }
  uint64_t *full = (uint64_t *)calloc(64 * BZO_MAXW + 1, sizeof(uint64_t));
  if (!full) return 4;
  job_t jb = {rows, k, w64, g, 0, 1};
  int best;
  uint64_t combos;
  int rc = run_workers(&jb, nthreads, &best, &combos, full);
  for (int w = 0; !rc && w <= 64 * BZO_MAXW; ++w) {
    if (!full[w]) continue;
    if (w < nbins) hist[w] = full[w]; else rc = 2;
  }
  free(full);
  return rc;
}

/* Minimum weight over all nonzero codewords (k <= 40 enforced here; the
 * reference caps at 28 by default). */
int bzo_brute(const uint64_t *rows, int k, int w64, int32_t *out_min) {
  if (k < 1 || k > 40 || w64 < 1 || w64 > BZO_MAXW) return 3;
  uint64_t cw[BZO_MAXW];
  memset(cw, 0, sizeof cw);
  int best = 0x7fffffff;
  const uint64_t total = 1ull << k;
  for (uint64_t i = 1; i < total; ++i) {
    const int b = __builtin_ctzll(i);
    const uint64_t *r = rows + (size_t)b * w64;
    for (int j = 0; j < w64; ++j) cw[j] ^= r[j];
    const int w = weight_of(cw, w64);
    if (w < best) best = w;
  }
  *out_min = best;
  return 0;
}

