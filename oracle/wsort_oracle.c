/*
 * wsort_oracle.c -- CPU restatement of the reference `wordsort` hot path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the checker for the GPU library and
 * the CPU baseline of bench.py; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it. The product
 * (paper_1407_6603_b200/) never links or calls it.
 *
 * Every function restates the reference algorithm it cites
 * (paths relative to /root/reference/pkg/src/wordsort/):
 *   or_tokenize       WORD_RE = rb"[A-Za-z0-9]+"; findall     ingest.py:15,26-28
 *   or_bubble_rows    _bubble_rows (triangular bubble sort)  engine.py:89-114
 *   or_sort_rows_fast same result + stats via stable merge sort, inversion
 *                     count and the early-exit bound K (closed form)
 *   or_sort_text      tokenize -> _group_by_length -> build_flat -> per-bucket
 *                     sort (one task per bucket on a pthread pool, the paper's strategy,
 *                     engine.py:140-201) -> emit_sorted + "\n" payload
 *                     (store.py:78-114, cli.py:83-103)
 * Parity is pinned against the reference run in this container
 * (the JSON fixtures in tests/golden, produced by tests/golden/make_golden.py).
 */
#define _POSIX_C_SOURCE 200809L
#include <stdint.h>
#include <stdlib.h>
#include <time.h>
#include <string.h>
#include <pthread.h>

static inline int is_alnum(uint8_t b) {
  return (b >= '0' && b <= '9') || (b >= 'A' && b <= 'Z') || (b >= 'a' && b <= 'z');
}

/* WORD_RE.findall(text): maximal alnum runs in order. Returns the word count;
 * fills starts/lens up to cap. */
uint64_t or_tokenize(const uint8_t* text, uint64_t n, uint32_t* starts, uint32_t* lens,
                     uint64_t cap) {
  uint64_t w = 0, i = 0;
  while (i < n) {
    if (!is_alnum(text[i])) { ++i; continue; }
    uint64_t s = i;
    while (i < n && is_alnum(text[i])) ++i;
    if (w < cap) { starts[w] = (uint32_t)s; lens[w] = (uint32_t)(i - s); }
    ++w;
  }
  return w;
}

/* engine.py:89-114, statement by statement: pass `end` runs j = 0..end-1,
 * byte-wise compare (:101-104), whole-row swap on strictly greater
 * (:105-109), early exit when a pass made no swap (:112-113). */
void or_bubble_rows(uint8_t* rows, int64_t n, int32_t width, int32_t naive, int64_t stats[3]) {
  int64_t comparisons = 0, swaps = 0, passes = 0;
  uint8_t* tmp = (uint8_t*)malloc(width > 0 ? (size_t)width : 1);
  for (int64_t end = n - 1; end > 0; --end) {
    passes += 1;
    int64_t pass_swaps = 0;
    for (int64_t j = 0; j < end; ++j) {
      comparisons += 1;
      uint8_t* a = rows + j * (int64_t)width;
      uint8_t* b = a + width;
      int order = 0;
      for (int32_t k = 0; k < width; ++k) {
        if (a[k] != b[k]) { order = a[k] > b[k] ? 1 : -1; break; }
      }
      if (order > 0) {
        memcpy(tmp, a, width); memcpy(a, b, width); memcpy(b, tmp, width);
        swaps += 1;
        pass_swaps += 1;
      }
    }
    if (!naive && pass_swaps == 0) break;
  }
  free(tmp);
  stats[0] = comparisons; stats[1] = swaps; stats[2] = passes;
}

/* ---- fast path: stable merge sort of row indices, counting inversions ---- */

typedef struct { const uint8_t* rows; int32_t width; } RowsCtx;

static inline int row_cmp(const RowsCtx* c, uint32_t a, uint32_t b) {
  return memcmp(c->rows + (size_t)a * c->width, c->rows + (size_t)b * c->width, c->width);
}

/* sorts idx[lo,hi) stably by row bytes; returns the number of strict inversions */
static int64_t merge_count(const RowsCtx* c, uint32_t* idx, uint32_t* tmp, int64_t lo, int64_t hi) {
  if (hi - lo < 2) return 0;
  if (hi - lo <= 16) { /* insertion sort: strict-'>' shifts == inversions */
    int64_t inv = 0;
    for (int64_t i = lo + 1; i < hi; ++i) {
      uint32_t x = idx[i];
      int64_t j = i - 1;
      while (j >= lo && row_cmp(c, idx[j], x) > 0) { idx[j + 1] = idx[j]; --j; ++inv; }
      idx[j + 1] = x;
    }
    return inv;
  }
  int64_t mid = lo + (hi - lo) / 2;
  int64_t inv = merge_count(c, idx, tmp, lo, mid) + merge_count(c, idx, tmp, mid, hi);
  int64_t i = lo, j = mid, k = lo;
  while (i < mid && j < hi) {
    if (row_cmp(c, idx[i], idx[j]) <= 0) tmp[k++] = idx[i++];
    else { inv += mid - i; tmp[k++] = idx[j++]; }
  }
  while (i < mid) tmp[k++] = idx[i++];
  while (j < hi) tmp[k++] = idx[j++];
  memcpy(idx + lo, tmp + lo, (size_t)(hi - lo) * sizeof(uint32_t));
  return inv;
}

static void closed_form(int64_t n, int64_t inv, int64_t K, int32_t naive, int64_t st[3]) {
  st[0] = st[1] = st[2] = 0;
  if (n < 2) return;
  if (naive) { st[0] = n * (n - 1) / 2; st[1] = inv; st[2] = n - 1; return; }
  int64_t P = K + 1 < n - 1 ? K + 1 : n - 1;
  st[0] = P * (n - 1) - P * (P - 1) / 2; st[1] = inv; st[2] = P;
}

/* Same sorted rows as or_bubble_rows; stats from the inversion count and
 * K = max_i(i - s(i)) through the closed forms.
 * Also returns inv/K when the out pointers are non-null. */
void or_sort_rows_fast(uint8_t* rows, int64_t n, int32_t width, int32_t naive, int64_t stats[3],
                       int64_t* inv_out, int64_t* k_out) {
  stats[0] = stats[1] = stats[2] = 0;
  if (n < 2) { if (inv_out) *inv_out = 0; if (k_out) *k_out = 0; return; }
  uint32_t* idx = (uint32_t*)malloc((size_t)n * 4);
  uint32_t* tmp = (uint32_t*)malloc((size_t)n * 4);
  for (int64_t i = 0; i < n; ++i) idx[i] = (uint32_t)i;
  RowsCtx c = {rows, width};
  int64_t inv = width > 0 ? merge_count(&c, idx, tmp, 0, n) : 0;
  int64_t K = 0;
  for (int64_t p = 0; p < n; ++p) if ((int64_t)idx[p] - p > K) K = (int64_t)idx[p] - p;
  if (width > 0) {
    uint8_t* out = (uint8_t*)malloc((size_t)n * width);
    for (int64_t p = 0; p < n; ++p) memcpy(out + p * width, rows + (size_t)idx[p] * width, width);
    memcpy(rows, out, (size_t)n * width);
    free(out);
  }
  free(idx); free(tmp);
  closed_form(n, inv, K, naive, stats);
  if (inv_out) *inv_out = inv;
  if (k_out) *k_out = K;
}

/* ---- full pipeline ------------------------------------------------------ */

typedef struct {
  uint8_t* flat;
  const uint64_t* boff;
  const uint64_t* cnt;
  int32_t mode;
  int64_t* per_len;
  int32_t max_len;
  uint32_t* order;
  uint32_t norder;
  uint32_t next;
  pthread_mutex_t mu;
} SortJob;

static void* sort_worker(void* arg) {
  SortJob* j = (SortJob*)arg;
  for (;;) {
    pthread_mutex_lock(&j->mu);
    uint32_t t = j->next < j->norder ? j->order[j->next++] : 0;
    pthread_mutex_unlock(&j->mu);
    if (!t) return NULL;
    uint32_t L = t;
    int64_t s[3] = {0, 0, 0}, inv = 0, K = 0;
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    if (j->mode == 0) or_bubble_rows(j->flat + j->boff[L], (int64_t)j->cnt[L], (int32_t)L, 1, s);
    else or_sort_rows_fast(j->flat + j->boff[L], (int64_t)j->cnt[L], (int32_t)L, 1, s, &inv, &K);
    clock_gettime(CLOCK_MONOTONIC, &t1);
    if (j->per_len && (int32_t)L <= j->max_len) {
      int64_t* r = j->per_len + (size_t)L * 8;
      r[0] = (int64_t)j->cnt[L]; r[1] = inv; r[2] = K; r[3] = s[0]; r[4] = s[1]; r[5] = s[2];
      r[6] = (int64_t)(t1.tv_sec - t0.tv_sec) * 1000000000LL + (t1.tv_nsec - t0.tv_nsec);
    }
  }
}

/* Sorts text's words like `wordsort sort` (flat layout) and writes the payload
 * (each word + '\n', ascending length, then bytes). mode 0 = the reference's
 * bubble sort per bucket (naive), mode 1 = fast path. per_len (optional,
 * (max_len+1) x 8 int64): [count, inv, K, naive c/s/p ... ] filled in fast
 * mode; in bubble mode [count, -, -, naive c, s, p]. Returns the word count,
 * or -1 on allocation failure / -2 when out is too small. */
int64_t or_sort_text(const uint8_t* text, uint64_t n, uint8_t* out, uint64_t cap,
                     uint64_t* written, int32_t mode, int32_t threads, int64_t* per_len,
                     int32_t max_len) {
  uint64_t W = or_tokenize(text, n, NULL, NULL, 0);
  uint32_t* st = (uint32_t*)malloc((W ? W : 1) * 4);
  uint32_t* ln = (uint32_t*)malloc((W ? W : 1) * 4);
  if (!st || !ln) return -1;
  or_tokenize(text, n, st, ln, W);
  uint32_t lmax = 0;
  for (uint64_t i = 0; i < W; ++i) if (ln[i] > lmax) lmax = ln[i];
  /* _group_by_length + build_flat: stable, corpus order per length */
  uint64_t* cnt = (uint64_t*)calloc(lmax + 2, 8);
  for (uint64_t i = 0; i < W; ++i) cnt[ln[i]]++;
  uint64_t* boff = (uint64_t*)calloc(lmax + 2, 8);
  uint64_t run = 0;
  for (uint32_t L = 0; L <= lmax; ++L) { boff[L] = run; run += cnt[L] * L; }
  uint8_t* flat = (uint8_t*)malloc(run ? run : 1);
  uint64_t* fill = (uint64_t*)calloc(lmax + 2, 8);
  for (uint64_t i = 0; i < W; ++i) {
    uint32_t L = ln[i];
    memcpy(flat + boff[L] + fill[L] * L, text + st[i], L);
    fill[L]++;
  }
  uint64_t payload = run + W;
  if (written) *written = payload;
  if (cap < payload) { free(st); free(ln); free(cnt); free(boff); free(flat); free(fill); return -2; }
  /* one task per bucket, largest bucket first, on `threads` workers (the
   * paper's one-vector-per-thread decomposition, engine.py:140-201) */
  SortJob job;
  job.flat = flat; job.boff = boff; job.cnt = cnt; job.mode = mode; job.per_len = per_len;
  job.max_len = max_len; job.next = 0;
  job.order = (uint32_t*)malloc((lmax + 1) * sizeof(uint32_t));
  job.norder = 0;
  for (uint32_t L = 1; L <= lmax; ++L) if (cnt[L]) job.order[job.norder++] = L;
  /* largest first */
  for (uint32_t a = 0; a < job.norder; ++a)
    for (uint32_t b = a + 1; b < job.norder; ++b)
      if (cnt[job.order[b]] > cnt[job.order[a]]) {
        uint32_t t = job.order[a]; job.order[a] = job.order[b]; job.order[b] = t;
      }
  pthread_mutex_init(&job.mu, NULL);
  int nt = threads > 0 ? threads : 1;
  if ((uint32_t)nt > job.norder) nt = job.norder ? (int)job.norder : 1;
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * nt);
  for (int t = 1; t < nt; ++t) pthread_create(&tids[t], NULL, sort_worker, &job);
  sort_worker(&job);
  for (int t = 1; t < nt; ++t) pthread_join(tids[t], NULL);
  pthread_mutex_destroy(&job.mu);
  free(tids);
  free(job.order);
  /* emit_sorted + payload */
  uint64_t o = 0;
  for (uint32_t L = 1; L <= lmax; ++L) {
    for (uint64_t j = 0; j < cnt[L]; ++j) {
      memcpy(out + o, flat + boff[L] + j * L, L);
      o += L;
      out[o++] = '\n';
    }
  }
  free(st); free(ln); free(cnt); free(boff); free(flat); free(fill);
  return (int64_t)W;
}
