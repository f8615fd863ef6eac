/*
 * wsort.h -- C ABI of libwsort_b200.so, the B200 (sm_100a) implementation of
 * the length-bucketed word sort of arXiv 1407.6603 (reference package
 * `wordsort`, /root/reference/pkg/src/wordsort).
 *
 * The reference has no foreign-function layer: its one native operator is the
 * numba kernel `_bubble_rows(rows, naive)` (engine.py:89-114), reached through
 * the Python names re-exported in wordsort/__init__.py:33-59. Every entry
 * point below names the reference interface it replaces; INTEGRATION.md shows
 * the ctypes stubs a maintainer adds to the reference to call them.
 *
 * Conventions
 *   - Every call returns WS_OK (0) or a negative WS_ERR_* code; the message of
 *     the last failure on the calling thread is ws_last_error(). The library
 *     never exits or aborts.
 *   - Plain pointers and sizes only. Host buffers belong to the caller; a
 *     handle owns its device buffers and CUDA stream. A handle must not be
 *     used by two threads at once; distinct handles (and the handle-free
 *     ws_sort_rows / ws_sort_blocks, which use a per-thread internal handle)
 *     may run concurrently, like the reference's nogil kernel on disjoint
 *     blocks (engine.py:89 nogil=True, engine.py:173-194).
 *   - There is no CPU fallback: without a usable CUDA device every compute
 *     call fails with WS_ERR_CUDA.
 *   - Output order is the reference's composite order: length ascending, then
 *     unsigned byte-lexicographic (verify.py:17-19); words of one length keep
 *     corpus order on ties (the reference swaps only on strictly-greater,
 *     engine.py:105).
 *   - Text offsets are 32-bit: texts must be shorter than 4 GiB.
 */
#ifndef WSORT_H
#define WSORT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define WS_OK 0
#define WS_ERR_ARG (-1)   /* invalid argument (Python: ValueError)        */
#define WS_ERR_CUDA (-2)  /* CUDA / device failure (Python: RuntimeError) */
#define WS_ERR_OOM (-3)   /* device or host allocation failed (MemoryError) */
#define WS_ERR_STATE (-4) /* call out of order, e.g. sort before ingest   */

typedef struct ws_handle ws_handle;

/* ABI version (major * 10000 + minor * 100 + patch). */
int ws_version(void);
/* Message of the last failed call on this thread ("" if none). */
const char* ws_last_error(void);
/* Number of visible CUDA devices (0 when none). */
int ws_device_count(int32_t* count);

/* Handle lifetime. */
int ws_create(ws_handle** out, int32_t device);
void ws_destroy(ws_handle* h);

/* --- ingest ------------------------------------------------------------ */
#define WS_INGEST_KEEP_TOKENS 1 /* also keep corpus-order (start, len) tokens */
#define WS_INGEST_DEVICE_PTR 2  /* `text` is a device pointer                 */
#define WS_INGEST_RESIDENT 4    /* re-use the text the handle already holds   */
#define WS_INGEST_UNORDERED 8   /* payload-only: words of one length may sit in
                                   any order inside their bucket before the sort
                                   (the sorted output is the same); ws_sort(h, 1)
                                   and ws_permutation then fail with
                                   WS_ERR_STATE. Ignored with KEEP_TOKENS. */

/* tokenize (ingest.py:26-28, WORD_RE = rb"[A-Za-z0-9]+" at ingest.py:15) +
 * stable group-by-length (store.py:78-82) + build_flat (store.py:90-96):
 * the text is copied to the device, tokenised and scattered into per-length
 * buckets of packed keys, corpus order kept inside each bucket. */
int ws_ingest_text(ws_handle* h, const uint8_t* text, uint64_t n, int32_t flags);

/* build_flat(words) (store.py:90-96) from an explicit word list: `concat` is
 * b"".join(words), lens[i] = len(words[i]). Words may hold any byte values;
 * empty words are not accepted (WS_ERR_ARG). */
int ws_ingest_words(ws_handle* h, const uint8_t* concat, const uint32_t* lens, uint64_t nwords);

/* build_flat over already-grouped rows: block i is a C-contiguous uint8
 * (counts[i], widths[i]) array; widths must be distinct and >= 1. */
int ws_ingest_blocks(ws_handle* h, int32_t nblocks, const uint8_t* const* rows,
                     const int64_t* counts, const int32_t* widths);

/* Nonempty buckets in ascending length: FlatBucketMatrix.lengths() and
 * count_for_length (store.py:52-66). *nbuckets receives the total even when it
 * exceeds cap; *words the word count. */
int ws_buckets(ws_handle* h, int64_t* lengths, int64_t* counts, int32_t cap, int32_t* nbuckets,
               uint64_t* words);

/* Corpus-order tokens after ws_ingest_text(..., WS_INGEST_KEEP_TOKENS):
 * starts_lens[2*i] = byte offset, starts_lens[2*i+1] = length. */
int ws_tokens(ws_handle* h, uint32_t* starts_lens, uint64_t cap_words, uint64_t* nwords);

/* --- sort -------------------------------------------------------------- */
/* sort_all_sequential / sort_all_parallel (engine.py:132-201): every bucket is
 * sorted on the device in one segmented launch per pass. With want_stats the
 * per-bucket inversion count and early-exit bound are computed too (needed by
 * ws_bucket_stats and ws_permutation). */
int ws_sort(ws_handle* h, int32_t want_stats);

/* SortStats of bubble_sort_bucket (engine.py:117-129) per bucket, in
 * ws_buckets order: stats[3*i + {0,1,2}] = comparisons, swaps, passes of the
 * reference's triangular bubble sort for the NAIVE (naive != 0) or
 * EARLY_EXIT variant. Requires ws_sort(h, 1). */
int ws_bucket_stats(ws_handle* h, int32_t naive, int64_t* stats, int32_t cap);

/* Stable sorting permutation of bucket `bucket` (ws_buckets order):
 * perm[j] = corpus rank (inside the bucket) of the word now at position j.
 * Requires ws_sort(h, 1). */
int ws_permutation(ws_handle* h, int32_t bucket, uint32_t* perm, uint64_t cap);

/* --- emit -------------------------------------------------------------- */
/* emit_sorted (store.py:105-114) + the CLI payload b"".join(w + b"\n")
 * (cli.py:97) into the host buffer `out`. *written = payload size; with
 * cap < size nothing is copied and WS_ERR_ARG is returned (query with cap 0). */
int ws_emit_lines(ws_handle* h, uint8_t* out, uint64_t cap, uint64_t* written);

/* FlatBucketMatrix.blocks (store.py:46-72): the (count, L) rows of every
 * bucket, ascending L, concatenated. Before ws_sort the rows are in corpus
 * order (build_flat), after it in sorted order. */
int ws_emit_rows(ws_handle* h, uint8_t* out, uint64_t cap, uint64_t* written);

/* --- fused end-to-end ---------------------------------------------------- */
/* The whole `wordsort sort FILE` path after load_text (cli.py:83-103): text
 * bytes in, payload bytes out (host buffers; pinned memory is fastest).
 * Buckets may be written straight from the last sort pass as payload, so
 * afterwards (also after ws_sort_resident) ws_emit_lines / ws_emit_rows
 * return WS_ERR_STATE until a ws_sort on the same ingest. */
int ws_sort_text(ws_handle* h, const uint8_t* text, uint64_t n, uint8_t* out, uint64_t cap,
                 uint64_t* written);

/* Batch of independent corpora (a serving loop): the same result as calling
 * ws_sort_text(h, texts[i], sizes[i], outs[i], caps[i], &written[i]) for
 * each i, with up to `inflight` corpora in flight (<= 0: 3; at most 4) on
 * internal slot handles owned by h. Uploads are staggered so one corpus
 * crosses PCIe host->device while earlier ones sort and come back
 * device->host. outs[i] may repeat with period `inflight` (a slot finishes
 * corpus i before starting i + inflight). Returns the first failure. */
int ws_sort_texts(ws_handle* h, int32_t count, const uint8_t* const* texts, const uint64_t* sizes,
                  uint8_t* const* outs, const uint64_t* caps, uint64_t* written,
                  int32_t inflight);

/* Device-resident variant: re-runs ingest + sort + emit on the text the
 * handle already holds from its last ws_ingest_text (same n), leaving the
 * payload in device memory (ws_output_device). No host<->device data copy
 * except the 136-byte length histogram. */
int ws_sort_resident(ws_handle* h, uint64_t n, uint64_t* written);
int ws_output_device(ws_handle* h, void** dptr, uint64_t* size);

/* --- drop-in for the numba kernel ---------------------------------------- */
/* _bubble_rows(rows, naive) (engine.py:89-114): sorts the C-contiguous uint8
 * (n, width) array `rows` IN PLACE and returns its (comparisons, swaps,
 * passes) in stats[0..2]. n < 2 returns zeros. */
int ws_sort_rows(uint8_t* rows, int64_t n, int32_t width, int32_t naive, int64_t stats[3]);

/* Batched _bubble_rows over several blocks in one segmented launch (what
 * sort_all_parallel does with its worker pool, engine.py:140-201). Widths may
 * repeat. stats[3*i..] per block; perms (nullable, entries nullable) receive
 * the stable sorting permutation of each block. */
int ws_sort_blocks(int32_t nblocks, uint8_t* const* rows, const int64_t* counts,
                   const int32_t* widths, int32_t naive, int64_t* stats, uint32_t* const* perms);

/* The reference's stats from the two device-side quantities: for n words with
 * `inversions` strict inversions and early-exit bound K = max(idx - pos):
 * naive: (n(n-1)/2, inv, n-1); early-exit: P = min(K+1, n-1),
 * (P(n-1) - P(P-1)/2, inv, P); all zero for n < 2. */
int ws_stats_closed_form(int64_t n, int64_t inversions, int64_t kmax, int32_t naive,
                         int64_t stats[3]);

/* --- profiling ----------------------------------------------------------- */
typedef struct ws_phase {
  char name[32];
  int32_t launches;  /* kernel launches (or copies) in this phase            */
  int32_t kind;      /* 0 = kernel, 1 = host<->device copy                    */
  double ms;         /* CUDA-event time on the stream the phase ran on        */
  double bytes;      /* algorithmic bytes moved (per-pass table)   */
  double start_ms;   /* start relative to the first recorded phase            */
} ws_phase;

/* Record CUDA events around every phase while enabled (on = 1); on = 2 also
 * runs every kernel on the handle's main stream, so each event pair times one
 * launch alone (a serialised per-kernel profile). 0 turns both off. */
int ws_set_profiling(ws_handle* h, int32_t on);
/* Phases recorded since the last reset (synchronises the handle's stream). */
int ws_profile(ws_handle* h, ws_phase* out, int32_t cap, int32_t* n);
int ws_profile_reset(ws_handle* h);
/* Kernel launches issued by this handle since creation. */
int ws_launch_count(ws_handle* h, uint64_t* launches);
/* Lane classes (bit c = class c: words of 1-5, 6-10, 11-21, 22-32 characters)
 * whose payload the last fused sort (ws_sort_text / ws_sort_texts /
 * ws_sort_resident) produced by counting distinct words instead of sorting
 * every occurrence (texts that repeat their vocabulary; same bytes either way:
 * the reference's printed payload, cli.py:97, depends only on which words a
 * bucket holds and how often). 0 when every class was sorted. */
int ws_counted_classes(ws_handle* h, int32_t* mask);

/* Checked builds (compiled with WS_CHECKED=1; tools/checked_build.sh): every
 * kernel bounds-checks its computed shared / global indices and records the
 * first failing line per translation unit instead of faulting. Synchronizes
 * the device, returns the number of failed checks since the last call (0 in a
 * release build), the unit (0 ingest, 1 sort, 2 radix, 3 emit) and line of
 * the first, and clears them. Not part of the reference's interface. */
int ws_debug_checks(uint64_t* failures, int32_t* first_unit, int32_t* first_line);
/* 1 when the library was built with WS_CHECKED=1. */
int ws_checked_build(void);
/* The handle's CUDA stream (cudaStream_t) for event timing by the caller. */
int ws_stream(ws_handle* h, void** stream);

/* Page-locked host memory for fast host<->device copies (cudaMallocHost). */
int ws_host_alloc(uint64_t bytes, void** out);
int ws_host_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* WSORT_H */
