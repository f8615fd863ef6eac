// Internal launcher declarations shared by the .cu translation units.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "ws_common.cuh"

namespace ws {

struct ScatterParams {
  uint64_t bin_base[kNumBins];  // byte offset of each bin's key region in `keys`
  uint64_t* keys;               // key arena, or nullptr (tokens-only mode)
  uint2* longlist;              // (start, len) of words with L > 32, corpus order
  uint2* tokens;                // optional (start, len) per word in corpus order
  int enc;                      // KeyEnc of the packed keys
  // single-pass (look-back) mode
  uint32_t chunk0;              // first chunk of this launch
  uint32_t nchunks_total;       // chunks of the whole text
  unsigned int* ticket;         // chunk ticket counter (zeroed before the first launch)
  uint32_t* status;             // [nchunks_total][kLookbackRec] look-back records (zeroed)
  uint32_t* totals;             // [kHistRows] per-bin totals, written by the last chunk
  uint64_t avail;               // bytes of text already on the device (0 = all)
  unsigned int* overflow;       // set when a word runs past `avail`
  unsigned int* unknown;        // ingest7: long words whose length is measured after the ingest
                                // (long-list entry (start, 0); long_len_fix), counted here
  // reserve mode (payload-only sorts): when set, each chunk reserves its run
  // of every bin with one atomicAdd on fill[row] instead of the look-back;
  // runs then land in completion order, so bucket order is not corpus order
  // (stats / permutations / tokens need the look-back). fill[] ends as totals.
  uint32_t* fill;               // [kHistRows] zeroed reservation counters, or nullptr
  // ordered reserve mode (fill and run_at set): stable order inside a chunk,
  // runs recorded per (bin, chunk) for the reorder into corpus order
  uint32_t* run_at;             // [kHistRows][nchunks_total] reserved start of the run
  uint32_t* run_cnt;            // [kHistRows][nchunks_total] words of the run
};

struct ReorderParams {
  uint32_t nchunks;
  const uint32_t* run_at;
  const uint32_t* run_cnt;
  const uint32_t* run_off;        // exclusive scan of run_cnt over chunks, per bin
  const uint8_t* src[kNumBins];   // reserved regions (keys_cap / long list as filled)
  uint8_t* dst[kNumBins];         // corpus-order destinations
  uint32_t key_bytes[kNumBins];   // element bytes per bin
};
void launch_reorder_runs(const ReorderParams& r, cudaStream_t st);

// checked builds: per translation unit, failures of WS_DCHECK since the last read
int check_reader_ingest(unsigned int* fails, unsigned int* line);
int check_reader_sort(unsigned int* fails, unsigned int* line);
int check_reader_radix(unsigned int* fails, unsigned int* line);
int check_reader_emit(unsigned int* fails, unsigned int* line);
void launch_check_selftest(cudaStream_t st);  // one failing WS_DCHECK (detector self-test)

// ingest.cu
uint32_t chunk_count(uint64_t n);
void launch_count(const uint8_t* text, uint64_t n, uint32_t* hist, uint32_t nchunks,
                  cudaStream_t st);
void launch_scan(const uint32_t* hist, uint32_t* off, uint32_t* totals, uint32_t nchunks,
                 int rows, cudaStream_t st);
void launch_scatter(const uint8_t* text, uint64_t n, const uint32_t* off, uint32_t nchunks,
                    const ScatterParams& p, cudaStream_t st);
void launch_ingest_lookback(const uint8_t* text, uint64_t n, uint32_t nchunks,
                            const ScatterParams& p, cudaStream_t st);
uint32_t ingest_chunk_bytes();
uint32_t reserve_chunk_bytes();  // payload-mode (reserve_ingest_kernel) chunks
uint32_t ordered_chunk_bytes();  // ordered (stats-mode) reserve ingest chunks (text)
void set_ingest_attributes();    // once per device (dynamic shared memory opt-in)
void launch_words_hist(const uint32_t* lens, uint64_t nwords, uint32_t wpw, uint32_t* whist,
                       uint32_t nwarps, cudaStream_t st);
void launch_words_scatter(const uint8_t* bytes, const uint64_t* starts, const uint32_t* lens,
                          uint64_t nwords, uint32_t wpw, const uint32_t* woff, uint32_t nwarps,
                          const ScatterParams& p, cudaStream_t st);
void launch_pack_rows(const uint8_t* rows, uint64_t n, uint32_t width, uint64_t* keys,
                      cudaStream_t st);
// Long words the ingest left unmeasured (length 0 in the long list): first
// separator of every 8 KiB chunk (first_sep[nchunks], scratch), then one warp
// per entry finds the word's end (the rest of its chunk, then the chunk table).
void launch_long_len_fix(const uint8_t* text, uint64_t n, uint2* longlist, uint64_t m,
                         uint32_t* first_sep, cudaStream_t st);
uint64_t long_fix_chunks(uint64_t n);  // entries of first_sep for a text of n bytes

// sort.cu
// Segment tables of up to kInlineSegs entries travel in the kernel
// parameters (constant bank): no host->device copy sits between passes.
constexpr int kInlineSegs = 12;  // >= the buckets of any lane class (11); kernel parameters stay small (launch cost)

struct SortLaunch {
  const uint64_t* keys_in;
  uint64_t* keys_out;
  const uint32_t* idx_in;  // nullptr for the tile pass (idx = position)
  uint32_t* idx_out;       // nullptr in keys-only mode
  const SegDesc* segs;     // device array when nsegs > kInlineSegs, else nullptr
  int nsegs;
  uint32_t work_items;     // grid size
  uint32_t run;            // merge: run length being merged (>= tile)
  unsigned long long* inv; // per stat slot
  long long* kmax;         // per stat slot
  uint32_t* splits;        // merge: per work item, A-split of its first output
  SegDesc inl[kInlineSegs];  // the segment table when it fits
};
int tile_size(int lanes);

// payload-mode sample sort of multi-lane classes (sort.cu)
constexpr int kMaxSplit = 511;            // splitters per bucket
constexpr int kSampleSmem = 192 * 1024;   // bytes of the in-smem sample sort
struct SampleSeg {
  const uint64_t* in;   // unsorted keys of the bucket
  uint32_t key_off;     // element offset of the bucket in the class region
  uint32_t n;
  uint32_t nsplit;      // S - 1 splitters (0: the bucket is one slot)
  uint32_t m;           // sample size (0 when nsplit == 0)
  uint32_t split_off;   // first splitter of the bucket in `splitters`
  uint32_t slot_base;   // first of the bucket's 2 * nsplit + 1 slots
  uint32_t tile_begin;  // first partition tile of the bucket
  uint32_t len;         // word length L of the bucket
  uint8_t* pay;         // fused emission: the bucket's payload records (6-bit text keys), or null
};
struct SampleLaunch {
  const SampleSeg* segs;  // device table when nsegs > kInlineSegs, else nullptr
  int nsegs;
  uint32_t nslots;
  uint32_t work_items;    // partition tiles of all buckets
  uint64_t* keys_out;     // the class region of the output key buffer
  uint64_t* scratch;      // class region of a buffer that is neither the input nor keys_out:
                          // slot sorts beyond a tile merge through it (never the input keys,
                          // which a later ws_sort of the same ingest reads again)
  uint64_t* splitters;    // 64-bit key prefixes
  uint32_t* hist;         // per slot: keys (zeroed before the launch)
  uint32_t* cursor;       // per slot: reservation cursor
  uint32_t* slot_off;     // per slot: class-relative element offset
  uint16_t* slot_ids;     // per key, in partition-tile order: its slot (count pass -> scatter pass)
  int split_done;         // the ingest already ran the split launch (sample_split_early_kernel)
  int count_done;         // ... and the count pass (partition_count_early_kernel)
  SampleSeg inl[kInlineSegs];
};
// Split launch of one lane class planned on the device (6-bit text keys,
// payload mode): lengths lmin..lmax, counts from the ingest's fill counters.
struct SplitEarly {
  const uint32_t* fill;
  const uint8_t* keys_cap;
  uint64_t region[32];     // byte offsets of lengths 1..32 in keys_cap
  int lmin, lmax;
  uint32_t T, target, pmax, smax;  // sample_sort_segments' rules
  uint64_t cap;            // larger buckets take the merge path
  uint64_t* splitters;     // the class's splitter and slot-counter buffers (max size)
  uint32_t* hist;
  // early count pass (or null): the split CTAs write its launch (segment
  // table of the buckets that fit, tiles, buffers) here, for
  // partition_count_early_kernel right behind them
  SampleLaunch* plan;
  uint16_t* slot_ids;
  uint32_t ptile;          // keys per partition tile
  const uint32_t* go;      // or null: run only if nonzero (dedupe.cu's probe gave the class up; else its words are counted)
};
// The count pass of one multi-lane class, planned on the device (the split
// launch's table): a persistent grid over the class's partition tiles.
void launch_partition_count_early(int lanes, const SampleLaunch* plan, int grid, cudaStream_t st,
                                  const uint32_t* go = nullptr);
void launch_sample_split_early(int lanes, const SplitEarly& e, cudaStream_t st);
// Small corpora: one CTA per length bucket sorts it on chip and writes its
// payload records, straight after the payload-mode ingest (6-bit keys);
// *flag is raised when a bucket does not fit a CTA or long words exist.
struct TinyLaunch {
  const uint32_t* fill;    // the ingest's per-bin counters (kHistRows)
  const uint8_t* keys_cap;
  uint64_t region[32];     // byte offsets of lengths 1..32 in keys_cap
  uint8_t* out;            // payload destination (buckets ascending by length)
  uint64_t out_cap;
  unsigned int* flag;      // zeroed before the launch
  unsigned long long* prof;  // diagnostics (WSORT_TINY_PROF): per CTA [start, end] globaltimer ns, or null
};
void launch_tiny_sort(const TinyLaunch& t, cudaStream_t st);
int sample_max_keys(int lanes);
int part_tile_size();
int subsort_tile_size(int lanes);  // keys one slot-sort CTA sorts in one network
// ev (profiling, or null): 10 events, a start / end pair around each of the 5 launches
void launch_sample_sort(int lanes, const SampleLaunch& a, cudaStream_t st, cudaEvent_t* ev = nullptr);
int merge_tile_size(int lanes);
void launch_tile_sort(int lanes, const SortLaunch& a, cudaStream_t st);
// ev (profiling, or null): 3 events, before the partition kernel, between, after the merge
void launch_merge(int lanes, const SortLaunch& a, cudaStream_t st, cudaEvent_t* ev = nullptr);
int merge_launches_per_level();  // kernels launch_merge enqueues (1, or 2 with the partition pass)

// radix.cu: payload-only LSD radix passes over one-word keys (classes 0, 1)
struct RadixSeg {
  const void* in;       // the segment's keys before this pass
  void* out;            // ... and after
  uint64_t coff;        // offset of the segment's [256][ntiles] count matrix
  uint32_t n;
  uint32_t tile_begin;  // first tile (work item) of the segment
  uint32_t ntiles;
  uint32_t shift;       // bit position of this pass's digit (histogram: of pass 0)
  uint32_t sid;         // one-sweep: the segment's row in the totals table
  uint32_t passes;      // one-sweep histogram: passes of the segment
  uint8_t* pay;         // one-sweep, segment's last pass: write payload records here instead
  uint32_t len;         //   of keys (word length; record = characters + '\n')
  uint32_t jbits;       // histogram launch: > 0 = count whole keys (key >> (32 - jbits), one-word
  uint32_t joff;        //   keys of <= 12 bits) into joint[joff ..]; the segment then takes no pass
};
constexpr int kRadixMaxPasses = 8;  // one per key byte
constexpr int kRadixTotStride = 1024;  // one-sweep totals: digits per (segment, pass) row
struct RadixLaunch {
  const RadixSeg* segs;  // device table when nsegs > kInlineSegs, else nullptr
  int nsegs;
  uint32_t work_items;   // tiles of all segments
  uint32_t* counts;      // per segment [256][ntiles] tile histograms -> offsets
  uint32_t* totals;      // reduce-then-scan: [nsegs][256] digit totals of this pass (zeroed);
                         // one-sweep: [sid][kRadixMaxPasses][kRadixTotStride] (zeroed before
                         // the histogram)
  uint64_t* status;      // one-sweep: [work_items][2^digit bits] look-back words
  uint32_t* ticket;      // one-sweep: this launch's tile counter (zeroed)
  uint32_t epoch;        // one-sweep: unique per launch, < 2^30, != 0
  uint32_t pass;
  int enc;               // key encoding (kEncAlnum6 / kEncRaw8), for payload records
  unsigned long long* prof;  // diagnostics (WSORT_OS_PROF): [tile][8] phase timestamps, or null
  uint32_t* joint;       // whole-key counters of the jbits segments (zeroed with the totals)
  RadixSeg inl[kInlineSegs];
};
int radix_tile_size(int lanes);
int radix_digit_bits(int lanes);  // one-sweep digit width of a lane class (10: uint32 keys, 8: uint64)
void launch_radix_pass(int lanes, const RadixLaunch& a, cudaStream_t st);
void launch_radix_hist(int lanes, const RadixLaunch& a, cudaStream_t st);
// Class-0 histogram launch planned on the device (6-bit text keys, payload
// mode): counts of lengths 1..5 from the ingest's fill counters.
struct EarlyHist {
  const uint32_t* fill;     // per-length word counts (bins 0..4 used)
  const uint8_t* keys_cap;  // the ingest's per-length key regions
  uint64_t region[5];       // byte offsets of lengths 1..5 in keys_cap
  uint32_t* totals;         // [5][kRadixMaxPasses][kRadixTotStride], zeroed
  uint32_t* joint;          // whole-key counters, zeroed
  int joint_ok;             // count (not sort) keys of <= 12 bits
  const uint32_t* go;       // or null: run only if nonzero (dedupe.cu's probe gave class 0 up; else its words are counted)
};
constexpr int kRadixC0Segs = 5;  // class-0 buckets at most (the totals table is sized for them)
void launch_radix_hist_early(const EarlyHist& e, cudaStream_t st);
// Payload of the jbits segments straight from their whole-key counts: value v
// of segment i repeated joint[v] times at its rank (the exclusive prefix).
// blocks = sum of 2^jbits over the launch's jbits segments (njsegs of them).
void launch_joint_expand(const RadixLaunch& a, uint32_t blocks, uint32_t njsegs, cudaStream_t st);
void launch_radix_onesweep(int lanes, const RadixLaunch& a, cudaStream_t st);

// dedupe.cu: distinct-word counting (payload mode, 6-bit text keys)
struct DdLayout;
void dd_host_layout(const uint32_t* n, DdLayout& o);  // plan.cuh's layout with the 6-bit key sizes
// control words at the head of the table pool (zeroed with it)
constexpr int kDdCtlCount = 0;   // [32] distinct words per length
constexpr int kDdCtlOvf = 32;    // [32] the bucket ran out of its table budget
constexpr int kDdCtlDone = 64;   // [2] CTAs of each aggregate launch that have finished
constexpr int kDdCtlSkip = 68;   // [4] per lane class: every bucket stayed in budget
constexpr int kDdCtlClsOvf = 72; // [4] per lane class: a bucket ran out of budget (the class's other tiles stop)
constexpr int kDdCtlProbe = 76;  // [4] per lane class: dd_probe_kernel gave the class up (its sort path's early launches run)
constexpr int kDdCtlWords = 128;
struct DdAgg {
  const uint32_t* fill;     // the ingest's per-length word counts
  const uint8_t* keys_cap;  // ... and per-length key regions
  uint64_t region[32];
  uint2* table;             // table pool (after the control words)
  uint8_t* dk;              // distinct-key pool
  uint32_t* ctl;
  uint32_t* aux;            // per-distinct-word array A: the word's table slot
  struct DdDevPlan* plan;   // or null: [2], each launch's last CTA writes its chain's plan
  uint32_t stile1, stilen;  // keys per sorted tile (uint32 keys / keys of 1-3 lanes: dd_sort_tile_size)
};
// first tile of every bucket judged (mostly different words: the class is given up)
void launch_dd_probe(const DdAgg& a, cudaStream_t st);
// two launches side by side (grp 0: lengths 1-5, 1: the wider keys)
void launch_dd_aggregate(const DdAgg& a, int grp, int grid, cudaStream_t st);
int dd_aggregate_ctas_per_sm(int grp);
constexpr int kDdTile = 256;    // distinct words per block of the run prefix
// records per output tile by word length (~16 KB of records)
__host__ __device__ constexpr uint32_t dd_xtile_of_len(int L) { return L <= 7 ? 2048u : (L <= 15 ? 1024u : 512u); }
constexpr int kDdXTileMax = 2048;
int check_reader_dedupe(unsigned int* fails, unsigned int* line);
// The counted classes' whole chain after the aggregate launch, planned on the
// device (no host round trip): the aggregate launch's last CTA writes
// DdDevPlan from the ingest's counters and its control words; the kernels behind it
// (tile sort of the distinct keys, rank merge of the tiles, run prefixes,
// expand) run grid-stride over the plan's work items.
struct DdDevPlan {
  uint32_t n[32], D[32];     // words / distinct words (D = 0: bucket empty or its class is sorted, not counted)
  uint32_t slots[32];
  uint32_t stile[32];        // keys per sorted tile of the bucket's class
  uint64_t tab_off[32], dk_off[32];
  uint64_t pay_off[32];      // the bucket's payload records in the output
  uint32_t aux_off[32];      // per-distinct-word arrays A (aux) and B (aux + aux_total)
  uint32_t tsum_off[32];     // tile totals of the run prefix
  uint32_t xs_off[32];       // per output tile: the run holding its first record
  uint32_t xtile[32];        // records per output tile (by record size)
  uint32_t aux_total;
  uint32_t st_begin[33];     // work-item prefixes: sorted tiles,
  uint32_t rk_begin[33];     //   blocks of kDdTile distinct words,
  uint32_t x_begin[33];      //   output tiles of xtile records
};
struct DdChain {
  const uint32_t* fill;
  const uint32_t* ctl;
  DdDevPlan* plan;
  const uint8_t* keys_cap;
  uint64_t region[32];
  uint2* table;
  uint8_t* dk;               // distinct keys as appended -> finally sorted
  uint8_t* ts;               // tile-sorted distinct keys
  uint32_t* aux;
  uint8_t* out;              // payload
  uint32_t cls_mask;         // lane classes this chain handles (bit c)
};
int dd_sort_tile_size(int lanes);
// sort.cu: tile sort; dedupe.cu: rank merge, run prefixes (3 kernels), expand
void launch_dd_tiles(const DdChain& c, int grid, cudaStream_t st);
void launch_dd_rank(const DdChain& c, int grid, cudaStream_t st);
void launch_dd_prefix(const DdChain& c, int grid, cudaStream_t st);
void launch_dd_chain_expand(const DdChain& c, int grid, cudaStream_t st);
int dd_expand_ctas_per_sm();  // the expand's grid: this many CTAs per SM, each looping over output tiles

// emit.cu
struct EmitSeg {
  const uint64_t* keys;  // sorted keys of the segment
  uint64_t out_off;      // byte offset of the segment's first word in the output
  uint32_t n;
  uint32_t len;
  uint32_t block_begin;
  uint32_t pad_;
};
constexpr int kEmitWords = 1024;
struct EmitTable {
  const EmitSeg* segs;  // device array when nsegs > kInlineSegs, else nullptr
  int nsegs;
  EmitSeg inl[kInlineSegs];
};
void launch_emit(int lanes, int enc, const EmitTable& t, uint32_t blocks, uint8_t* out,
                 int with_newline, cudaStream_t st);

// generic (L > 32) helpers
void launch_emit_long(const uint8_t* text, const uint2* words, const uint32_t* order,
                      uint64_t n, uint32_t len, uint8_t* out, int with_newline, cudaStream_t st);
void launch_lane_keys(const uint8_t* text, const uint2* words, const uint32_t* order,
                      uint64_t n, uint32_t lane, uint64_t* keys, cudaStream_t st);
void launch_gather_u32(const uint32_t* src, const uint32_t* perm, uint64_t n, uint32_t* dst,
                       cudaStream_t st);
void launch_iota_keys(const uint32_t* order, uint64_t n, uint64_t* keys, cudaStream_t st);
void launch_len_keys(const uint2* words, uint64_t n, uint64_t* keys, cudaStream_t st);
void launch_rank_kmax(const uint32_t* rank, uint64_t off, uint64_t n, long long* kmax,
                      cudaStream_t st);
void launch_rows_longlist(uint64_t base, uint64_t n, uint32_t width, uint2* words,
                          cudaStream_t st);
void launch_gather_u2(const uint2* src, const uint32_t* perm, uint64_t n, uint2* dst,
                      cudaStream_t st);
void launch_iota_u32(uint32_t* dst, uint64_t n, cudaStream_t st);
void set_sort_attributes();

}  // namespace ws
