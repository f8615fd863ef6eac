// C-ABI runtime of libwsort_b200: handles, buffer planning, pass scheduling.
//
// A handle owns its streams (main, one sort / emit / copy stream per lane
// class, one upload stream) and grow-only device buffers. A public call
// enqueues its kernels and synchronises at the end; the ingest path also
// synchronises once to read the 34-entry length histogram, which sizes the
// key arena and the pass schedule. Small parameter tables travel in kernel
// parameters (or, beyond 40 entries, through one pinned staging copy).
//
// Buckets: lengths 1..32 are packed-key buckets grouped by key width into
// lane classes 0..4 (0 = one uint32 word); each class sorts on its own stream
// (payload mode: LSD radix for class 0, sample sort for the others; stats
// mode: tile + merge-path levels with inversion counts). Lengths > 32 are
// "long groups" sorted by an LSD sequence of stable 1-lane passes over their
// 8-byte lanes (most significant last), with the text as the byte store.
// Finished buckets are emitted (and copied to the host) on side streams while
// later passes run. ws_sort_texts runs several corpora through peer handles.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "wsort.h"
#include "ws_common.cuh"
#include "ws_kernels.h"
#include "plan.cuh"

using namespace ws;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int fail_cuda(cudaError_t e, const char* what, int line) {
  int code = (e == cudaErrorMemoryAllocation) ? WS_ERR_OOM : WS_ERR_CUDA;
  cudaGetLastError();
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error at api.cu:%d (%s): %s", line, what, cudaGetErrorString(e));
  g_err = buf;
  return code;
}

// WSORT_TRACE=1: host timestamps of the batch pipeline's stages (stderr)
double trace_ms() {
  static const auto t0 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
}

// WSORT_TRACE=2: host timestamps of the resident step's milestones (stderr).
thread_local std::vector<std::pair<const char*, double>> g_marks;
inline void tmark(const char* what) {
  static const bool on = getenv("WSORT_TRACE") && getenv("WSORT_TRACE")[0] == '2';
  if (on) g_marks.emplace_back(what, trace_ms());
}

#define WS_CUDA(x)                                             \
  do {                                                         \
    cudaError_t e_ = (x);                                      \
    if (e_ != cudaSuccess) return fail_cuda(e_, #x, __LINE__); \
  } while (0)

#define WS_TRY(x)             \
  do {                        \
    int r_ = (x);             \
    if (r_ != WS_OK) return r_; \
  } while (0)

std::atomic<bool> g_exiting{false};  // set by an atexit handler (see ws_destroy)

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes + bytes / 8, 4096);
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  template <class T>
  T* as() const { return reinterpret_cast<T*>(p); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
  }
};

struct PinBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t ensure(size_t bytes) {
    if (bytes <= cap && p) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    size_t want = std::max<size_t>(bytes + bytes / 4, 1 << 16);
    cudaError_t e = cudaMallocHost(&p, want);
    if (e == cudaSuccess) cap = want;
    return e;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
  }
};

constexpr int kClasses = 4;  // lane classes 0..4 (0 = one uint32 key word)
constexpr int kLongCls = -2;  // emit selector for the L > 32 groups
// Texts up to this size use the single-pass ingest (capacity-bounded key
// regions, ~37 bytes per text byte); larger texts the two-pass count + scatter.
constexpr uint64_t kSinglePassMaxText = 512ull << 20;
// Host texts at least this large are copied in pieces overlapped with ingest.
constexpr uint64_t kChunkedH2DMin = 16ull << 20;

struct Bucket {
  uint32_t len = 0;
  uint64_t count = 0;
  bool is_long = false;
  int lanes = 0;             // packed: 0..4 (lane class, key_bytes(lanes) bytes per key)
  uint64_t elem_off = 0;     // packed: element offset inside the lane class region
  uint64_t idx_off = 0;      // packed: offset in the idx arena (global over buckets)
  uint64_t long_off = 0;     // long: offset in the grouped long-word list
  int final_buf = 0;         // packed: which key/idx buffer holds the sorted run
  int64_t inv = 0, kmax = 0; // stats (valid after ws_sort(h, 1))
  const uint64_t* in_ptr = nullptr;  // packed: the unsorted keys (ingest output)
  uint32_t dd_n = 0;         // counted class (dedupe.cu): the bucket's distinct words
};

struct PhaseRec {
  std::string name;
  cudaEvent_t a, b;
  double bytes;
  int launches;
  int kind;
};

struct SegIn {
  uint64_t key_off;  // element offset (class-relative for packed buckets)
  uint64_t idx_off;
  uint32_t n;
  uint32_t stat_slot;
  uint32_t idx_base;
  int final_buf;  // out
  const uint64_t* in_ptr = nullptr;  // unsorted keys for the tile pass (default: keys0)
  bool emitted = false;  // out: the last pass wrote the payload records (no keys)
};

}  // namespace

struct ws_handle {
  int device = 0;
  cudaStream_t st = nullptr;
  cudaStream_t cs[kClasses + 1] = {nullptr};  // one stream per lane class (cs[0] unused)
  cudaStream_t es[kClasses + 1] = {nullptr};  // per class: emit of completed buckets
  cudaStream_t ds[kClasses + 1] = {nullptr};  // per class: D2H of emitted buckets
  cudaStream_t hs = nullptr;                  // chunked H2D of the text
  DevBuf overflow;                            // chunked ingest: a word ran past a piece
  std::vector<cudaEvent_t> sync_events;       // pool of timing-free events
  size_t sync_used = 0;
  cudaEvent_t ev_fork = nullptr, ev_join[kClasses + 1] = {nullptr};
  // text / word sources
  DevBuf text;         // corpus bytes (+ padding) or word bytes or rows
  DevBuf starts, lens; // word-list ingest
  DevBuf hist, off, totals;
  DevBuf keys[2], idx[2];
  DevBuf keys_cap, status, ticket;  // single-pass ingest: capacity-bounded regions
  DevBuf fill;                      // reserve-mode counters (WS_INGEST_UNORDERED)
  DevBuf run_at, run_cnt, run_off, longlist2;  // ordered reserve mode: runs to reorder
  DevBuf longlist, longgrp, rank, rank_tmp, lkeys[2], lidx[2];
  DevBuf tokens;
  DevBuf stat_inv, stat_k, stat_k_dummy;
  DevBuf out;
  DevBuf params;
  DevBuf splits[kClasses + 2];  // merge-path splits: [0] main stream, [1..4] class streams
  DevBuf rcounts[2], rtotals[2];  // radix passes of lane classes 0 and 1
  DevBuf rstatus[2];              // one-sweep look-back words
  bool payload_only = false;      // a fused sort wrote some buckets' payload without their keys
  bool early_req = false;         // the next ingest launches the class-0 histogram itself
  bool tiny_req = false;          // the next ingest launches tiny_sort_kernel into `out` itself
  bool tiny_launched = false;     // ... and did
  bool tiny_done = false;         // ... and every bucket fitted: `out` holds the payload
  DevBuf tiny_flag, tiny_prof;
  DevBuf first_sep;  // long_len_fix: first separator per 8 KiB chunk
  bool early_done = false;        // ... and did (valid for the sort that follows)
  bool early_joint = false;       //     with whole-key counts for <= 12-bit keys
  bool split_early[kClasses + 1] = {false};  // ... and each multi-lane class's split launch
  bool count_early[kClasses + 1] = {false};  // ... and its count pass (device-planned)
  DevBuf early_plan[kClasses + 1];            // the count pass's SampleLaunch, written by the split CTAs
  uint32_t radix_epoch = 0;
  DevBuf ss_split[kClasses + 1], ss_slots[kClasses + 1];  // sample sort of classes 1..4
  DevBuf ss_ids[kClasses + 1];                            // per-key slot ids
  DevBuf ss_scratch;  // slot-sort merge scratch when the input keys sit in keys[0]
  // distinct-word counting (dedupe.cu): control words + tables, distinct keys, run prefixes
  DevBuf dd_pool, dd_keys, dd_aux, dd_ts, dd_plan;
  cudaEvent_t ev_dd = nullptr, ev_chain = nullptr;  // aggregate launched / device-planned chain done
  cudaEvent_t ev_probe = nullptr;  // the counting path's probe done (the sort paths' early launches wait for it)
  cudaEvent_t ev_lo = nullptr, ev_hi = nullptr;  // the two counting launches done
  DdAgg dd_agg;                   // the counting launches' parameters (stage 0 -> stage 1)
  bool dd_chain = false;          // the chain behind the aggregate launch writes the counted classes' payload
  bool dd_two_chains = false;     // ... as two chains side by side (class 0 / classes 1-3)
  cudaStream_t zs = nullptr;      // zeroes the table pool beside the ingest; the wider keys' counting
  cudaStream_t xs = nullptr;      // class 0's chain behind its counting launch
  cudaEvent_t ev_zero = nullptr;
  bool dd_req = false;            // the next ingest counts distinct words right behind itself
  bool dd_launched = false;       // ... and did
  bool dd_ok[kClasses + 1] = {false};  // per lane class: every bucket stayed in budget
  int dd_used = 0;                // classes the last fused sort took through the counts (bit mask)
  DdLayout dd_lay;                // tables / distinct-key lists of the current buckets
  PinBuf pin_params, pin_small;
  size_t param_used = 0;
  uint64_t out_size = 0;  // payload bytes left in `out` by ws_sort_resident

  uint64_t n_text = 0;
  uint32_t nchunks = 0;
  uint64_t words = 0;
  uint64_t n_long = 0;
  bool have_tokens = false;
  bool unordered = false;  // last ingest placed bucket runs in completion order
  int enc = kEncRaw8;       // key encoding of the current packed buckets
  bool text_valid = false;  // h->text holds the last ingested text (reusable, resident)
  bool ingested = false, sorted = false, have_stats = false;
  uint64_t class_base[kClasses + 1] = {0};  // byte offset of each lane class region
  uint64_t class_elems[kClasses + 1] = {0};
  uint64_t idx_total = 0;
  std::vector<Bucket> buckets;

  bool prof = false;
  bool serial = false;  // WSORT_SERIAL=1: every kernel on the main stream (diagnostics)
  bool serial_env = false;  // ... as the environment set it (ws_set_profiling(h, 2) serialises too)
  size_t early_phase_first = 0;  // profiling: 1 + index of the early launches' first record
  std::vector<PhaseRec> phases;
  std::vector<cudaEvent_t> event_pool;
  uint64_t launches = 0;
  std::vector<ws_handle*> peers;  // extra in-flight slots of ws_sort_texts
};

namespace {

// ----------------------------------------------------------------------------
// helpers

cudaEvent_t get_event(ws_handle* h) {
  if (!h->event_pool.empty()) {
    cudaEvent_t e = h->event_pool.back();
    h->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct Phase {
  ws_handle* h;
  PhaseRec rec;
  bool on;
  cudaStream_t st;
  Phase(ws_handle* hh, const char* name, double bytes, int kind = 0, cudaStream_t s = nullptr)
      : h(hh), on(hh->prof), st(s ? s : hh->st) {
    if (!on) return;
    rec.name = name;
    rec.bytes = bytes;
    rec.kind = kind;
    rec.launches = 0;
    rec.a = get_event(h);
    rec.b = get_event(h);
    cudaEventRecord(rec.a, st);
    start_launches = h->launches;
  }
  uint64_t start_launches = 0;
  void end() {
    if (!on) return;
    cudaEventRecord(rec.b, st);
    rec.launches = (int)(h->launches - start_launches);
    if (rec.kind == 1 && rec.launches == 0) rec.launches = 1;
    h->phases.push_back(rec);
    on = false;
  }
  ~Phase() { end(); }
};

// Timing-free event from the handle's pool (valid until the next public call).
cudaEvent_t sync_event(ws_handle* h) {
  if (h->sync_used == h->sync_events.size()) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    h->sync_events.push_back(e);
  }
  return h->sync_events[h->sync_used++];
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail_cuda(e, what, 0);
  return WS_OK;
}

// Address of element `elem` of lane class `cls` in key buffer `buf` (0/1).
uint64_t* class_keys(ws_handle* h, int buf, int cls, uint64_t elem) {
  return reinterpret_cast<uint64_t*>(h->keys[buf].as<uint8_t>() + h->class_base[cls] +
                                     elem * key_bytes(cls));
}

// Parameter tables: staged in pinned memory, uploaded with one copy each.
void params_reset(ws_handle* h) {
  h->param_used = 0;
  h->sync_used = 0;
}

template <class T>
int params_upload(ws_handle* h, const std::vector<T>& v, const T** dev,
                  cudaStream_t st = nullptr) {
  if (!st) st = h->st;
  size_t bytes = v.size() * sizeof(T);
  size_t off = (h->param_used + 255) & ~size_t(255);
  if (off + bytes > h->pin_params.cap || off + bytes > h->params.cap) {
    // growing needs every stream of the handle idle (old staging bytes may be
    // in flight on any of them: class, emit, copy and upload streams)
    WS_CUDA(cudaStreamSynchronize(h->st));
    for (int c = 0; c <= kClasses; ++c) {
      if (h->cs[c]) WS_CUDA(cudaStreamSynchronize(h->cs[c]));
      if (h->es[c]) WS_CUDA(cudaStreamSynchronize(h->es[c]));
      if (h->ds[c]) WS_CUDA(cudaStreamSynchronize(h->ds[c]));
    }
    if (h->hs) WS_CUDA(cudaStreamSynchronize(h->hs));
    if (h->zs) WS_CUDA(cudaStreamSynchronize(h->zs));
    if (h->xs) WS_CUDA(cudaStreamSynchronize(h->xs));
    size_t need = std::max<size_t>(2 * (off + bytes), 1 << 20);
    if (need > h->pin_params.cap) {
      h->pin_params.release();
      WS_CUDA(h->pin_params.ensure(need));
    }
    if (need > h->params.cap) {
      h->params.release();
      WS_CUDA(h->params.ensure(need));
    }
    off = 0;
  }
  if (bytes) {
    memcpy(static_cast<uint8_t*>(h->pin_params.p) + off, v.data(), bytes);
    WS_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(h->params.p) + off,
                            static_cast<uint8_t*>(h->pin_params.p) + off, bytes,
                            cudaMemcpyHostToDevice, st));
  }
  *dev = reinterpret_cast<const T*>(static_cast<uint8_t*>(h->params.p) + off);
  h->param_used = off + bytes;
  return WS_OK;
}

int begin_call(ws_handle* h) {
  if (!h) return fail(WS_ERR_ARG, "null handle");
  WS_CUDA(cudaSetDevice(h->device));
  params_reset(h);
  g_err.clear();
  return WS_OK;
}

// ----------------------------------------------------------------------------
// segmented sort driver: tile pass + merge levels over `segs`, all of one
// lane width, data starting in keys0 (+ implicit idx), ping-ponging with
// keys1/idx1/idx0. Each segment's final buffer parity is written back.

// Called after the pass that completes some segments (their final buffer is
// known): lets the caller emit / copy those segments while later passes run.
using PassDoneHook = std::function<int(const std::vector<const SegIn*>&, cudaStream_t)>;

int sort_segments(ws_handle* h, int lanes, std::vector<SegIn>& segs, uint64_t* keys0,
                  uint64_t* keys1, uint32_t* idx0, uint32_t* idx1, bool stats,
                  unsigned long long* inv, long long* kmax, const char* tag,
                  cudaStream_t st = nullptr, const PassDoneHook* on_done = nullptr) {
  if (!st) st = h->st;
  std::vector<SegIn*> live;
  for (auto& s : segs) {
    s.final_buf = 0;
    if (s.n > 0) live.push_back(&s);
  }
  if (live.empty()) return WS_OK;
  const uint32_t T = (uint32_t)tile_size(lanes);
  const uint32_t TM = (uint32_t)merge_tile_size(lanes);
  uint64_t total_tiles = 0;  // upper bound of the work items of any pass
  for (auto* s : live) total_tiles += 2 * ((s->n + std::min(T, TM) - 1) / std::min(T, TM)) + 4;
  DevBuf& split_buf = h->splits[st == h->st ? 0 : lanes + 1];
  WS_CUDA(split_buf.ensure((2 * total_tiles + 4) * 4));  // (split, segment) per work item
  uint64_t* kb[2] = {keys0, keys1};
  uint32_t* ib[2] = {idx0, idx1};
  // pass 0 = tile sort; pass p >= 1 merges runs of T << (p-1)
  uint32_t max_n = 0;
  for (auto* s : live) max_n = std::max(max_n, s->n);
  int passes = 1;
  while (((uint64_t)T << (passes - 1)) < max_n) ++passes;
  for (int p = 0; p < passes; ++p) {
    const uint64_t run = p == 0 ? 0 : ((uint64_t)T << (p - 1));
    std::vector<SegDesc> d;
    uint32_t work = 0;
    double bytes = 0;
    for (auto* s : live) {
      if (p > 0 && s->n <= run) continue;
      SegDesc sd;
      sd.in_ptr = p == 0 ? s->in_ptr : nullptr;
      sd.key_off = s->key_off;
      sd.idx_off = s->idx_off;
      sd.n = s->n;
      sd.tile_begin = work;
      sd.stat_slot = s->stat_slot;
      sd.idx_base = s->idx_base;
      d.push_back(sd);
      if (p == 0) {
        work += (uint32_t)((s->n + T - 1) / T);
      } else {  // ceil(2R / TM) tiles for each pair of runs (sort.cu pair_geom)
        const uint64_t pairs = (s->n + 2 * run - 1) / (2 * run);
        work += (uint32_t)(pairs * ((2 * run + TM - 1) / TM));
      }
      bytes += 2.0 * s->n * key_bytes(lanes) + (stats ? (p == 0 ? 4.0 : 8.0) * s->n : 0.0);
      s->final_buf = (p + 1) & 1;
    }
    if (d.empty()) break;
    const int in = p & 1, out = in ^ 1;
    SortLaunch a;
    if (d.size() <= (size_t)kInlineSegs) {
      std::copy(d.begin(), d.end(), a.inl);
      a.segs = nullptr;
    } else {
      WS_TRY(params_upload(h, d, &a.segs, st));
    }
    a.keys_in = kb[in];
    a.keys_out = kb[out];
    a.idx_in = stats ? ib[in] : nullptr;
    a.idx_out = stats ? ib[out] : nullptr;
    a.nsegs = (int)d.size();
    a.work_items = work;
    a.run = (uint32_t)run;
    a.inv = inv;
    a.kmax = kmax;
    a.splits = split_buf.as<uint32_t>();
    char name[32];
    snprintf(name, sizeof name, "%s%s_l%d", tag, p == 0 ? "tile" : "merge", lanes);
    Phase ph(h, name, bytes, 0, st);
    if (p == 0) {
      launch_tile_sort(lanes, a, st);
      ++h->launches;
    } else {
      // merge kernel (+ a partition kernel when WS_MERGE_FUSED_SPLIT=0); profiling:
      // one record per kernel inside the level's phase (kind 2)
      cudaEvent_t ev[3];
      if (h->prof)
        for (auto& e : ev) e = get_event(h);
      launch_merge(lanes, a, st, h->prof ? ev : nullptr);
      h->launches += merge_launches_per_level();
      if (h->prof) {
        // (the partition kernel is a latency-bound merge-path search: no bytes claimed)
        const struct { const char* nm; double bytes; int launches; } k[2] = {
            {"msplit", 0.0, merge_launches_per_level() - 1}, {"mergek", bytes, 1}};
        for (int i = 0; i < 2; ++i) {
          PhaseRec r;
          r.name = std::string(tag) + k[i].nm + "_l" + std::to_string(lanes);
          r.a = ev[i];
          r.b = ev[i + 1];
          r.bytes = k[i].bytes;
          r.launches = k[i].launches;
          r.kind = 2;
          h->phases.push_back(r);
        }
      }
    }
    ph.end();
    WS_TRY(check_launch(name));
    if (on_done) {
      std::vector<const SegIn*> done;  // segments whose last pass is p
      const uint64_t next_run = (uint64_t)T << p;
      for (auto* s : live)
        if ((p == 0 || s->n > run) && s->n <= next_run) done.push_back(s);
      if (!done.empty()) WS_TRY((*on_done)(done, st));
    }
  }
  return WS_OK;
}

// Payload-only sort of one-word keys (lane classes 0 and 1): stable LSD radix
// passes over 8-bit digits of the bits each bucket uses (radix.cu). Pass p
// reads buffer p & 1 (pass 0: the segment's in_ptr) and writes (p + 1) & 1;
// a bucket is done after ceil(bits / 8) passes.
// WSORT_OS_PROF=1: per-tile phase durations of one one-sweep pass (stderr).
void print_os_profile(DevBuf& prof, uint32_t work, int pass, cudaStream_t st) {
  std::vector<unsigned long long> v((size_t)work * 8);
  cudaMemcpyAsync(v.data(), prof.p, v.size() * 8, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  unsigned long long t0 = ~0ull, t1 = 0;
  double ph[4] = {0, 0, 0, 0}, mx[4] = {0, 0, 0, 0};
  for (uint32_t i = 0; i < work; ++i) {
    const unsigned long long* r = &v[(size_t)i * 8];
    t0 = std::min(t0, r[0]);
    t1 = std::max(t1, r[4]);
    for (int k = 0; k < 4; ++k) {
      const double d = (double)(r[k + 1] - r[k]);
      ph[k] += d;
      mx[k] = std::max(mx[k], d);
    }
  }
  double rounds = 0, stalls = 0;
  for (uint32_t i = 0; i < work; ++i) {
    rounds += (double)v[(size_t)i * 8 + 5];
    stalls += (double)v[(size_t)i * 8 + 6];
  }
  fprintf(stderr, "os_prof pass %d tiles %u span %.1f us | mean us: rank %.2f scan %.2f lookback %.2f "
          "scatter %.2f | max: %.2f %.2f %.2f %.2f | look-back rounds %.1f (not-ready %.1f)\n",
          pass, work, (t1 - t0) / 1e3, ph[0] / work / 1e3, ph[1] / work / 1e3, ph[2] / work / 1e3,
          ph[3] / work / 1e3, mx[0] / 1e3, mx[1] / 1e3, mx[2] / 1e3, mx[3] / 1e3, rounds / work,
          stalls / work);
  // in-flight tiles over time (8 samples)
  for (int s = 1; s < 8; ++s) {
    const unsigned long long t = t0 + (t1 - t0) * s / 8;
    int live = 0;
    for (uint32_t i = 0; i < work; ++i) live += v[(size_t)i * 8] <= t && v[(size_t)i * 8 + 4] > t;
    fprintf(stderr, " %d", live);
  }
  fprintf(stderr, " (tiles in flight)\n");
}

int radix_sort_segments(ws_handle* h, int lanes, std::vector<SegIn>& segs, uint64_t* keys0,
                        uint64_t* keys1, cudaStream_t st, const PassDoneHook* on_done,
                        uint8_t* pay = nullptr, const std::vector<uint64_t>* pay_off = nullptr) {
  const int kb_bytes = key_bytes(lanes);
  const int keybits = 8 * kb_bytes;
  const int cbits = h->enc == kEncAlnum6 ? 6 : 8;  // bits per character
  const uint32_t T = (uint32_t)radix_tile_size(lanes);
  struct Plan {
    SegIn* s;
    int passes;
    uint32_t shift0, ntiles;
    uint32_t jbits;  // > 0: no passes, payload from the whole-key counts
  };
  std::vector<Plan> plan;
  int max_passes = 0;
  uint64_t count_words = 0;
  static const char* rts_env = getenv("WSORT_RADIX_RTS");
  const bool rts = rts_env && rts_env[0] == '1';
  static const char* nj_env = getenv("WSORT_NO_JOINT");
  const bool joint_ok = pay && lanes == 0 && !rts && !(nj_env && nj_env[0] == '1');
  // digit width: the one-sweep passes take 10-bit digits on uint32 keys (the
  // reduce-then-scan path and uint64 keys 8-bit)
  const int db = rts ? 8 : radix_digit_bits(lanes);
  for (auto& s : segs) {
    s.final_buf = 0;
    if (!s.n) continue;
    const int bits = std::min(keybits, cbits * (int)h->buckets[s.stat_slot].len);
    int passes = std::max(1, (bits + db - 1) / db);
    uint32_t jbits = 0;
    if (h->enc == kEncAlnum6 && lanes == 0 && !rts) {
      // 6-bit class-0 buckets: the rule radix_hist_early_kernel plans with (plan.cuh)
      const RadixPlan rp = radix_plan_c0(h->buckets[s.stat_slot].len, (uint32_t)db, joint_ok, 12u);
      passes = (int)rp.passes;
      jbits = rp.jbits;
    } else if (joint_ok && bits <= 12) {  // <= 4096 distinct keys: counted, not sorted
      jbits = (uint32_t)bits;
      passes = 0;
    }
    plan.push_back(Plan{&s, passes, (uint32_t)(keybits - bits), (s.n + T - 1) / T, jbits});
    max_passes = std::max(max_passes, passes);
    count_words += 256ull * plan.back().ntiles;
    s.final_buf = passes & 1;
  }
  if (plan.empty()) return WS_OK;
  DevBuf& cb = h->rcounts[lanes];
  DevBuf& tb = h->rtotals[lanes];
  uint8_t* kb[2] = {reinterpret_cast<uint8_t*>(keys0), reinterpret_cast<uint8_t*>(keys1)};
  if (!rts) {
    // one-sweep: one histogram launch for the digit totals of every pass, then
    // one look-back launch per pass
    const size_t tot_words = (lanes == 0 ? std::max<size_t>(kRadixC0Segs, plan.size()) : plan.size()) *
                             kRadixMaxPasses * kRadixTotStride;
    // the ingest already ran this histogram launch (same plan rules, same stream)
    const bool early = h->early_done && lanes == 0 && pay && joint_ok == h->early_joint &&
                       plan.size() <= (size_t)kRadixC0Segs;
    h->early_done = false;
    size_t joint_words = 0;
    uint32_t njoint = 0, jblocks = 0;
    for (auto& pl : plan)
      if (pl.jbits) {
        joint_words += 2u << pl.jbits;  // counts, then their exclusive prefix
        jblocks += 1u << pl.jbits;
        ++njoint;
      }
    const size_t zero_bytes = (tot_words + kRadixMaxPasses + joint_words) * 4;
    if (!early) {
      WS_CUDA(tb.ensure(zero_bytes + 64));
      WS_CUDA(cudaMemsetAsync(tb.p, 0, zero_bytes, st));
    }
    uint32_t* totals = tb.as<uint32_t>();
    uint32_t* tickets = totals + tot_words;
    uint32_t* joint = tickets + kRadixMaxPasses;
    uint32_t all_tiles = 0;
    for (auto& pl : plan) all_tiles += pl.ntiles;
    DevBuf& sb = h->rstatus[lanes];
    const void* before = sb.p;
    const size_t cap0 = sb.cap;
    WS_CUDA(sb.ensure((size_t)all_tiles * ((size_t)1 << db) * 8));
    if (sb.p != before || sb.cap != cap0) WS_CUDA(cudaMemsetAsync(sb.p, 0, sb.cap, st));  // no stale epochs
    char name[32];
    snprintf(name, sizeof name, "radix_l%d", lanes);
    RadixLaunch jlaunch;  // the histogram launch's table (jbits segments and their counters)
    memset(&jlaunch, 0, sizeof jlaunch);
    for (int p = -1; p < max_passes; ++p) {  // p = -1: the histogram launch
      uint32_t joff = 0;
      std::vector<RadixSeg> d;
      uint32_t work = 0;
      double bytes = 0;
      for (size_t i = 0; i < plan.size(); ++i) {
        const Plan& pl = plan[i];
        if (pl.passes <= std::max(p, 0) && p >= 0) continue;
        RadixSeg r;
        memset(&r, 0, sizeof r);
        const uint64_t off = pl.s->key_off * kb_bytes;
        r.in = p <= 0 ? static_cast<const void*>(pl.s->in_ptr) : kb[p & 1] + off;
        r.out = kb[(p + 1) & 1] + off;
        r.n = pl.s->n;
        r.tile_begin = work;
        r.ntiles = pl.ntiles;
        r.shift = pl.shift0 + (uint32_t)db * std::max(p, 0);
        r.sid = (uint32_t)i;
        r.passes = (uint32_t)pl.passes;
        if (p < 0 && pl.jbits) {
          r.jbits = pl.jbits;
          r.joff = joff;
          joff += 2u << pl.jbits;
          r.pay = pay + (*pay_off)[pl.s->stat_slot];
          r.len = h->buckets[pl.s->stat_slot].len;
          pl.s->emitted = true;
        }
        if (pay && p == pl.passes - 1) {  // last pass: payload records instead of keys
          r.pay = pay + (*pay_off)[pl.s->stat_slot];
          r.len = h->buckets[pl.s->stat_slot].len;
          pl.s->emitted = true;
        }
        d.push_back(r);
        work += pl.ntiles;
        // keys read; keys written, or the payload records of a fused last pass
        bytes += (double)pl.s->n * kb_bytes;
        if (p >= 0)
          bytes += (double)pl.s->n * (r.pay ? (double)(r.len + 1) : (double)kb_bytes);
      }
      RadixLaunch a;
      memset(&a, 0, sizeof a);
      if (d.size() <= (size_t)kInlineSegs) {
        std::copy(d.begin(), d.end(), a.inl);
        a.segs = nullptr;
      } else {
        WS_TRY(params_upload(h, d, &a.segs, st));
      }
      a.nsegs = (int)d.size();
      a.work_items = work;
      a.totals = totals;
      a.status = sb.as<uint64_t>();
      a.pass = (uint32_t)std::max(p, 0);
      a.enc = h->enc;
      a.ticket = tickets + a.pass;
      if (++h->radix_epoch >= (1u << 30)) h->radix_epoch = 1;
      a.epoch = h->radix_epoch;
      a.joint = joint;
      static const char* os_prof = getenv("WSORT_OS_PROF");  // diagnostics: per-tile phase stamps
      DevBuf prof;
      if (os_prof && os_prof[0] == '1' && p >= 0) {
        WS_CUDA(prof.ensure((size_t)work * 64));
        WS_CUDA(cudaMemsetAsync(prof.p, 0, (size_t)work * 64, st));
        a.prof = prof.as<unsigned long long>();
      }
      char pname[32];
      snprintf(pname, sizeof pname, p < 0 ? "radix_hist_l%d" : "radix_l%d", lanes);
      Phase ph(h, pname, bytes, 0, st);
      if (p == 0) tmark("pass0_launch");
      if (p >= 0) {
        launch_radix_onesweep(lanes, a, st);
        if (p == 0) tmark("pass0_launched");
        if (p == 1) tmark("pass1_launched");
        if (p == 3) tmark("pass3_launched");
      } else if (!early) {
        launch_radix_hist(lanes, a, st);
      }
      if (p >= 0 || !early) ++h->launches;
      ph.end();
      if (a.prof) {
        print_os_profile(prof, work, p, st);
        prof.release();
      }
      if (p < 0 && njoint) jlaunch = a;  // the counted segments: expanded after the passes
      WS_TRY(check_launch(name));
      if (on_done && p >= 0) {
        std::vector<const SegIn*> done;
        for (auto& pl : plan)
          if (pl.passes == p + 1) done.push_back(pl.s);
        if (!done.empty()) WS_TRY((*on_done)(done, st));
      }
    }
    if (njoint) {  // off the passes' chain: payload of the counted segments from their counts
      tmark("joint_launch");
      launch_joint_expand(jlaunch, jblocks, njoint, st);
      tmark("joint_launched");
      h->launches += 2;
      WS_TRY(check_launch("joint_expand"));
      if (on_done) {
        std::vector<const SegIn*> done;
        for (auto& pl : plan)
          if (pl.jbits) done.push_back(pl.s);
        WS_TRY((*on_done)(done, st));
      }
    }
    return WS_OK;
  }
  WS_CUDA(cb.ensure(count_words * 4 + 64));
  const size_t tot_bytes = (size_t)max_passes * plan.size() * 256 * 4;
  WS_CUDA(tb.ensure(tot_bytes));
  WS_CUDA(cudaMemsetAsync(tb.p, 0, tot_bytes, st));
  for (int p = 0; p < max_passes; ++p) {
    std::vector<RadixSeg> d;
    uint32_t work = 0;
    uint64_t coff = 0;
    double bytes = 0;
    for (auto& pl : plan) {
      if (pl.passes <= p) continue;
      RadixSeg r;
      const uint64_t off = pl.s->key_off * kb_bytes;
      r.in = p == 0 ? static_cast<const void*>(pl.s->in_ptr) : kb[p & 1] + off;
      r.out = kb[(p + 1) & 1] + off;
      r.coff = coff;
      r.n = pl.s->n;
      r.tile_begin = work;
      r.ntiles = pl.ntiles;
      r.shift = pl.shift0 + 8 * p;
      d.push_back(r);
      work += pl.ntiles;
      coff += 256ull * pl.ntiles;
      bytes += 3.0 * pl.s->n * kb_bytes;  // upsweep read + downsweep read and write
    }
    RadixLaunch a;
    if (d.size() <= (size_t)kInlineSegs) {
      std::copy(d.begin(), d.end(), a.inl);
      a.segs = nullptr;
    } else {
      WS_TRY(params_upload(h, d, &a.segs, st));
    }
    a.nsegs = (int)d.size();
    a.work_items = work;
    a.counts = cb.as<uint32_t>();
    a.totals = tb.as<uint32_t>() + (size_t)p * plan.size() * 256;
    char name[32];
    snprintf(name, sizeof name, "radix_l%d", lanes);
    Phase ph(h, name, bytes, 0, st);
    launch_radix_pass(lanes, a, st);
    h->launches += 3;
    ph.end();
    WS_TRY(check_launch(name));
    if (on_done) {
      std::vector<const SegIn*> done;
      for (auto& pl : plan)
        if (pl.passes == p + 1) done.push_back(pl.s);
      if (!done.empty()) WS_TRY((*on_done)(done, st));
    }
  }
  return WS_OK;
}

// Payload-only sort of a multi-lane class (sort.cu, sample sort): every
// bucket larger than a tile is cut by S - 1 sampled splitters into slots of
// ~T/2 keys (plus one slot per splitter for keys equal to it), scattered into
// the output buffer and sorted slot by slot on chip. Five launches per class
// whatever the bucket sizes; the result is in buffer 1.
// Largest bucket the sample sort keeps at its slot size (the splitter and
// sample budget: kMaxSplit + 1 slots of half a slot-sort tile).
// Slots per bucket at most: the splitter budget, and >= 8 samples per splitter.
// WSORT_SAMPLE_SMAX=k lowers it (tests: forces slots beyond a tile, i.e. the
// slot sorts' merge-sort route, at small sizes; the merge-path cap below is
// unchanged, so those buckets stay in the sample sort).
uint32_t sample_smax(uint32_t pmax) {
  static const char* e = getenv("WSORT_SAMPLE_SMAX");
  uint32_t v = std::min<uint32_t>(kMaxSplit + 1, pmax / 8);
  if (e && atoi(e) >= 1) v = std::min<uint32_t>(v, (uint32_t)atoi(e));
  return v;
}

uint64_t sample_bucket_limit(int lanes) {
  return (uint64_t)(kMaxSplit + 1) * (uint64_t)(subsort_tile_size(lanes) / 2);
}

int sample_sort_segments(ws_handle* h, int lanes, std::vector<SegIn>& segs, uint64_t* out_class,
                         cudaStream_t st, const PassDoneHook* on_done, uint8_t* pay = nullptr,
                         const std::vector<uint64_t>* pay_off = nullptr) {
  tmark("ss_begin");
  if (h->enc != kEncAlnum6) pay = nullptr;  // fused records decode 6-bit text keys only
  uint32_t pmax = 1;  // sample prefixes sorted in shared memory (power of two, <= 4096)
  while (pmax * 2 <= (uint32_t)std::min(sample_max_keys(lanes), 4096)) pmax *= 2;
  const uint32_t ptile = (uint32_t)part_tile_size();
  std::vector<SampleSeg> d;
  uint32_t slots = 0, splits = 0, tiles = 0;
  for (auto& s : segs) {
    s.final_buf = 1;
    // slots of half a slot-sort tile on average, one slot when the bucket fits
    // one slot sort's tile (plan.cuh, shared with sample_split_early_kernel)
    const SamplePlan pl = sample_plan(s.n, (uint32_t)subsort_tile_size(lanes), pmax, sample_smax(pmax));
    SampleSeg g;
    g.in = s.in_ptr;
    g.key_off = (uint32_t)s.key_off;
    g.n = s.n;
    g.nsplit = pl.nsplit;
    g.m = pl.m;
    g.split_off = splits;
    g.slot_base = slots;
    g.tile_begin = tiles;
    g.len = h->buckets[s.stat_slot].len;
    g.pay = nullptr;
    if (pay) {  // the slot sorts write this bucket's payload records
      g.pay = pay + (*pay_off)[s.stat_slot];
      s.emitted = true;
    }
    d.push_back(g);
    slots += 2 * g.nsplit + 1;
    splits += g.nsplit;
    tiles += (s.n + ptile - 1) / ptile;
  }
  if (d.empty() || !tiles) return WS_OK;
  if (d.size() > (size_t)kInlineSegs) return fail(WS_ERR_STATE, "too many buckets in a class");
  WS_CUDA(h->ss_split[lanes].ensure((size_t)std::max(splits, 1u) * key_bytes(lanes) + 64));  // full keys
  WS_CUDA(h->ss_slots[lanes].ensure((size_t)slots * 12 + 64));
  WS_CUDA(h->ss_ids[lanes].ensure((size_t)tiles * part_tile_size() * 2 + 64));
  SampleLaunch a;
  std::copy(d.begin(), d.end(), a.inl);
  a.segs = nullptr;
  a.nsegs = (int)d.size();
  a.nslots = slots;
  a.work_items = tiles;
  a.keys_out = out_class;
  // slots beyond a tile merge through the class region of keys[0] when no
  // bucket reads its input from there (the single-pass ingest leaves the keys
  // in keys_cap), else through a buffer of their own
  bool in_k0 = false;
  for (const auto& s : segs) in_k0 |= s.in_ptr == class_keys(h, 0, lanes, s.key_off);
  if (!in_k0) {
    a.scratch = class_keys(h, 0, lanes, 0);
  } else {
    WS_CUDA(h->ss_scratch.ensure((size_t)h->class_elems[lanes] * key_bytes(lanes) + 64));
    a.scratch = h->ss_scratch.as<uint64_t>();
  }
  a.splitters = h->ss_split[lanes].as<uint64_t>();
  a.hist = h->ss_slots[lanes].as<uint32_t>();
  a.cursor = a.hist + slots;
  a.slot_off = a.cursor + slots;
  a.slot_ids = h->ss_ids[lanes].as<uint16_t>();
  // the ingest ran this class's split launch (same rules, same stream)
  a.split_done = h->split_early[lanes] ? 1 : 0;
  a.count_done = a.split_done && h->count_early[lanes] ? 1 : 0;
  h->split_early[lanes] = false;
  h->count_early[lanes] = false;
  double bytes = 0, nkeys = 0, pay_bytes = 0;
  for (const auto& s : segs) {
    bytes += 5.0 * s.n * key_bytes(lanes);
    nkeys += s.n;
    pay_bytes += (double)s.n * (h->buckets[s.stat_slot].len + 1);
  }
  char name[32];
  snprintf(name, sizeof name, "sample_l%d", lanes);
  {
    Phase ph(h, name, bytes, 0, st);
    tmark("ss_launch");
    cudaEvent_t ev[10];  // distinct events per record (ws_profile_reset pools them)
    if (h->prof)
      for (auto& e : ev) e = get_event(h);
    launch_sample_sort(lanes, a, st, h->prof ? ev : nullptr);
    tmark("ss_launched");
    h->launches += 5 - a.split_done - a.count_done;
    if (h->prof) {  // one record per kernel of the chain (kind 2: inside a phase)
      const double kb = key_bytes(lanes);
      const double split_b = a.split_done ? 0.0 : 8.0 * kb * std::min<double>(nkeys, 4096.0 * d.size());
      const struct { const char* nm; double bytes; } k[5] = {
          {"split", split_b},
          {"part_count", nkeys * (8.0 + 2.0)},            // first words read, slot ids written
          {"slot_scan", 8.0 * slots},
          {"part_scatter", nkeys * (2.0 * kb + 2.0)},     // keys read + written, slot ids read
          {"subsort", nkeys * kb + (pay ? pay_bytes : nkeys * kb)}};  // keys in, records (or keys) out
      for (int i = 0; i < 5; ++i) {
        PhaseRec r;
        r.name = std::string(k[i].nm) + "_l" + std::to_string(lanes);
        r.a = ev[2 * i];
        r.b = ev[2 * i + 1];
        r.bytes = k[i].bytes;
        r.launches = ((i == 0 && a.split_done) || (i == 1 && a.count_done)) ? 0 : 1;
        r.kind = 2;
        h->phases.push_back(r);
      }
    }
  }
  WS_TRY(check_launch(name));
  tmark("ss_checked");
  if (on_done) {
    std::vector<const SegIn*> done;
    for (auto& s : segs) done.push_back(&s);
    WS_TRY((*on_done)(done, st));
  }
  tmark("ss_hooked");
  return WS_OK;
}

// ----------------------------------------------------------------------------
// planning after the length histogram is known

struct LongGroup {
  uint32_t len;
  uint64_t off, count;
};

// counts[b] for bins 0..31 -> packed buckets; lays out the lane-class regions.
int plan_packed(ws_handle* h, const uint64_t* counts) {
  h->buckets.clear();
  uint64_t elems[kClasses + 1] = {0};
  uint64_t bin_elem[kMaxPackedLen] = {0};
  uint64_t idx_run = 0;
  for (int b = 0; b < kMaxPackedLen; ++b) {
    if (!counts[b]) continue;
    int L = b + 1, c = lanes_for_len_enc(L, h->enc);
    bin_elem[b] = elems[c];
    elems[c] += counts[b];
    Bucket bk;
    bk.len = L;
    bk.count = counts[b];
    bk.lanes = c;
    bk.elem_off = bin_elem[b];
    bk.idx_off = idx_run;
    idx_run += counts[b];
    h->buckets.push_back(bk);
  }
  uint64_t run = 0;  // bytes
  for (int c = 0; c <= kClasses; ++c) {
    h->class_base[c] = run;
    h->class_elems[c] = elems[c];
    run += elems[c] * key_bytes(c);
    run = (run + 15) & ~15ull;  // 16-byte aligned class regions
  }
  h->idx_total = idx_run;
  WS_CUDA(h->keys[0].ensure(run + 64));
  WS_CUDA(h->keys[1].ensure(run + 64));
  for (auto& bk : h->buckets) bk.in_ptr = class_keys(h, 0, bk.lanes, bk.elem_off);
  return WS_OK;
}

void fill_scatter_params(ws_handle* h, ScatterParams& p) {
  memset(&p, 0, sizeof p);
  for (const auto& bk : h->buckets) {
    if (bk.is_long) continue;
    p.bin_base[bk.len - 1] = h->class_base[bk.lanes] + bk.elem_off * key_bytes(bk.lanes);
  }
  p.keys = h->keys[0].as<uint64_t>();
  p.longlist = h->longlist.as<uint2>();
  p.tokens = nullptr;
  p.enc = h->enc;
}

// Long words (corpus order in h->longlist, m entries) -> stable grouping by
// length into h->longgrp; appends one bucket per distinct length.
int group_long_words(ws_handle* h, uint64_t m) {
  h->n_long = m;
  if (!m) return WS_OK;
  WS_CUDA(h->longgrp.ensure(m * sizeof(uint2)));
  WS_CUDA(h->lkeys[0].ensure(m * 8 + 64));
  WS_CUDA(h->lkeys[1].ensure(m * 8 + 64));
  WS_CUDA(h->lidx[0].ensure(m * 4 + 64));
  WS_CUDA(h->lidx[1].ensure(m * 4 + 64));
  WS_CUDA(h->stat_k_dummy.ensure(64 * 16));
  WS_CUDA(h->stat_inv.ensure(64 * 16));
  launch_len_keys(h->longlist.as<uint2>(), m, h->lkeys[0].as<uint64_t>(), h->st);
  ++h->launches;
  std::vector<SegIn> segs(1);
  segs[0] = SegIn{0, 0, (uint32_t)m, 0, 0, 0};
  WS_TRY(sort_segments(h, 1, segs, h->lkeys[0].as<uint64_t>(), h->lkeys[1].as<uint64_t>(),
                       h->lidx[0].as<uint32_t>(), h->lidx[1].as<uint32_t>(), true,
                       h->stat_inv.as<unsigned long long>(), h->stat_k_dummy.as<long long>(),
                       "lgroup_"));
  const int f = segs[0].final_buf;
  launch_gather_u2(h->longlist.as<uint2>(), h->lidx[f].as<uint32_t>(), m, h->longgrp.as<uint2>(),
                   h->st);
  ++h->launches;
  std::vector<uint64_t> lens(m);
  WS_CUDA(cudaMemcpyAsync(lens.data(), h->lkeys[f].p, m * 8, cudaMemcpyDeviceToHost, h->st));
  WS_CUDA(cudaStreamSynchronize(h->st));
  uint64_t i = 0;
  while (i < m) {
    uint64_t j = i;
    while (j < m && lens[j] == lens[i]) ++j;
    Bucket bk;
    bk.len = (uint32_t)lens[i];
    bk.count = j - i;
    bk.is_long = true;
    bk.long_off = i;
    h->buckets.push_back(bk);
    i = j;
  }
  return WS_OK;
}

int finish_ingest(ws_handle* h) {
  h->words = 0;
  for (auto& b : h->buckets) h->words += b.count;
  h->ingested = true;
  h->sorted = false;
  h->have_stats = false;
  return WS_OK;
}

static bool env_on(const char* v) {
  const char* e = getenv(v);
  return e && e[0] == '1';
}

// The fused payload sorts (ws_sort_text / ws_sort_resident / batches) let the
// ingest start class 0's histogram launch on the class-0 stream, planned on the
// device from the fill counters, so it overlaps the host's read-back and plan.
bool early_hist_wanted() {
  static const bool ok = !env_on("WSORT_NO_EARLY_HIST") && !env_on("WSORT_D2H_PER_CLASS") &&
                         !env_on("WSORT_NO_FUSED_PAYLOAD") && !env_on("WSORT_NO_RADIX") &&
                         !env_on("WSORT_RADIX_RTS");
  return ok;
}

size_t radix_c0_zero_bytes() {  // totals + tickets + whole-key counters of class 0
  return ((size_t)kRadixC0Segs * kRadixMaxPasses * kRadixTotStride + kRadixMaxPasses + (2u << 6) +
          (2u << 12)) * 4;
}

// Small corpora (tiny_sort_kernel): right behind the ingest on the main
// stream, before the host reads the histogram; `out` holds n + 64 bytes.
int launch_tiny(ws_handle* h, const uint64_t* region, uint64_t n) {
  WS_CUDA(h->tiny_flag.ensure(64));
  WS_CUDA(cudaMemsetAsync(h->tiny_flag.p, 0, 4, h->st));
  TinyLaunch t;
  memset(&t, 0, sizeof t);
  t.fill = h->fill.as<uint32_t>();
  t.keys_cap = h->keys_cap.as<uint8_t>();
  for (int b = 0; b < kMaxPackedLen; ++b) t.region[b] = region[b];
  t.out = h->out.as<uint8_t>();
  t.out_cap = n + 64;
  t.flag = h->tiny_flag.as<unsigned int>();
  static const bool tprof = env_on("WSORT_TINY_PROF");
  if (tprof) {  // diagnostics: per-bucket CTA times, printed after the ingest's sync
    WS_CUDA(h->tiny_prof.ensure((64 + 16 * kMaxPackedLen) * 8));
    WS_CUDA(cudaMemsetAsync(h->tiny_prof.p, 0, (64 + 16 * kMaxPackedLen) * 8, h->st));
    t.prof = h->tiny_prof.as<unsigned long long>();
  }
  {
    Phase ph(h, "tiny", 2.0 * (double)n, 1);
    launch_tiny_sort(t, h->st);
    ++h->launches;
  }
  WS_TRY(check_launch("tiny_sort"));
  h->tiny_launched = true;
  return WS_OK;
}

// Distinct-word counting (dedupe.cu) right behind the payload-mode ingest, on
// the main stream: the ingest's sync then also covers its counters. WSORT_NO_DEDUPE=1
// turns it off; WSORT_DEDUPE_MIN=bytes sets the smallest text that tries it
// (default 48 MiB: smaller texts are bound by launch latencies and the host's
// enqueue, where the counting path's dozen extra launches cost more than its
// counting saves -- config-4-like texts of 31 MB: 0.280 vs 0.259 ms, of 63 MB:
// 0.374 vs 0.414 ms, tools/dd_threshold.py; configs 1-3: 0.15-0.26 vs 0.14-0.20 ms).
bool dedupe_wanted(uint64_t n) {
  static const bool off = env_on("WSORT_NO_DEDUPE") || env_on("WSORT_D2H_PER_CLASS") ||
                          env_on("WSORT_NO_FUSED_PAYLOAD");
  static const uint64_t min_text = [] {
    const char* e = getenv("WSORT_DEDUPE_MIN");
    return e ? (uint64_t)strtoull(e, nullptr, 0) : (uint64_t)(48u << 20);
  }();
  return !off && n >= min_text;
}

size_t dd_pool_bytes(uint64_t n) { return (size_t)kDdCtlWords * 4 + dd_max_table_slots(n) * 8; }

// Zero the control words and the table pool for a text of n bytes (upper
// bound: the counts are not known yet) on the side stream.
int dd_zero_pool(ws_handle* h, uint64_t n, cudaStream_t st) {
  WS_CUDA(h->dd_pool.ensure(dd_pool_bytes(n) + 64));
  WS_CUDA(h->dd_keys.ensure(dd_max_dk_bytes(n) + 64));
  WS_CUDA(h->dd_ts.ensure(dd_max_dk_bytes(n) + 64));
  // per-distinct-word arrays A and B + the run prefix's tile totals
  WS_CUDA(h->dd_aux.ensure((2 * dd_max_distinct(n) + dd_max_distinct(n) / kDdTile + 4 * kDdLens +
                            (n + 1) / 1024 + 2 * kDdLens) * 4 + 64));  // ... and the output tiles' first runs
  WS_CUDA(h->dd_plan.ensure(2 * sizeof(DdDevPlan)));
  WS_CUDA(h->out.ensure(n + 1 + 64));  // the payload never exceeds the text by more than a byte
  WS_CUDA(cudaMemsetAsync(h->dd_pool.p, 0, dd_pool_bytes(n), st));
  return WS_OK;
}

// Stage 0 (right behind the ingest): the probe and the two counting launches.
// Stage 1 (after the sort paths' early launches have been enqueued, so those
// are not held back by the host's enqueue of a dozen more launches): the
// chains behind the counting launches.
int launch_dd_counting(ws_handle* h, const uint64_t* region, int stage) {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
  // streams: [0] class 0's launch on the main stream (the host's read-back
  // follows it), its chain on a side stream; [1] the wider keys' launch and
  // chain on the stream that zeroed the pool
  cudaStream_t agg_st[2] = {h->st, h->serial ? h->st : h->zs};
  cudaStream_t chain_st[2] = {h->serial ? h->st : h->xs, h->serial ? h->st : h->zs};
  static const char* nm[2][5] = {{"dd_aggregate", "dd_tiles", "dd_rank", "dd_prefix", "dd_expand"},
                                 {"dd_aggregate_hi", "dd_tiles_hi", "dd_rank_hi", "dd_prefix_hi", "dd_expand_hi"}};
  DdAgg& a = h->dd_agg;
  if (stage == 0) {
    if (h->dd_launched) {  // a redone ingest: the pool holds the first attempt's entries
      WS_TRY(dd_zero_pool(h, h->n_text, h->st));
    } else {
      WS_CUDA(cudaStreamWaitEvent(h->st, h->ev_zero, 0));
    }
    memset(&a, 0, sizeof a);
    a.fill = h->fill.as<uint32_t>();
    a.keys_cap = h->keys_cap.as<uint8_t>();
    for (int b = 0; b < 32; ++b) a.region[b] = region[b];
    a.ctl = h->dd_pool.as<uint32_t>();
    a.table = reinterpret_cast<uint2*>(h->dd_pool.as<uint32_t>() + kDdCtlWords);
    a.dk = h->dd_keys.as<uint8_t>();
    a.aux = h->dd_aux.as<uint32_t>();
    a.plan = h->dd_plan.as<DdDevPlan>();
    a.stile1 = (uint32_t)dd_sort_tile_size(0);
    a.stilen = (uint32_t)dd_sort_tile_size(1);
    // First the probe: one CTA per length judges the bucket's first keys, so a
    // text of mostly different words gives its classes up within microseconds
    // and the sort paths' early launches (which wait for the probe only) start.
    {
      Phase ph(h, "dd_probe", 0.0, 0, h->st);
      launch_dd_probe(a, h->st);
      ++h->launches;
    }
    WS_CUDA(cudaEventRecord(h->ev_probe, h->st));
    // Two launches side by side -- the uint32 keys (lengths 1-5) on the main
    // stream, the wider keys on the side stream. Each launch's last CTA plans
    // the chain that stage 1 enqueues behind it.
    const uint64_t max_tiles = (h->n_text + 1) / 2 / 4096 + 32;
    WS_CUDA(cudaEventRecord(h->ev_dd, h->st));  // the ingest's keys and counters (and the zeroed pool)
    for (int g = 1; g >= 0; --g) {
      const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(max_tiles, (uint64_t)dd_aggregate_ctas_per_sm(g) * sms));
      if (agg_st[g] != h->st) WS_CUDA(cudaStreamWaitEvent(agg_st[g], h->ev_dd, 0));
      Phase ph(h, nm[g][0], 0.0, 0, agg_st[g]);  // bytes patched once the counts are known
      launch_dd_aggregate(a, g, grid, agg_st[g]);
      ++h->launches;
    }
    WS_CUDA(cudaEventRecord(h->ev_lo, h->st));  // class 0's launch: its chain starts behind it
    if (agg_st[1] != h->st) {
      // the main stream (the host's read-back of the control words) waits for
      // the wider keys' launch as well -- not for the chains
      WS_CUDA(cudaEventRecord(h->ev_hi, agg_st[1]));
      WS_CUDA(cudaStreamWaitEvent(h->st, h->ev_hi, 0));
    }
    WS_TRY(check_launch("dd_aggregate"));
    h->dd_launched = true;
    h->dd_chain = false;
    return WS_OK;
  }
  // stage 1: behind each counting launch the rest of its classes' path,
  // planned on the device and enqueued now -- distinct keys sorted (tiles, then
  // a rank merge), run prefixes, payload records -- while the host still waits
  // for the ingest's counters. Class 0's chain starts when its own launch ends.
  DdChain c;
  memset(&c, 0, sizeof c);
  c.fill = a.fill;
  c.ctl = a.ctl;
  c.keys_cap = a.keys_cap;
  for (int b = 0; b < 32; ++b) c.region[b] = region[b];
  c.table = a.table;
  c.dk = a.dk;
  c.ts = h->dd_ts.as<uint8_t>();
  c.aux = a.aux;
  c.out = h->out.as<uint8_t>();
  const int cgrid = 4 * sms;
  for (int g = 1; g >= 0; --g) {
    cudaStream_t s2 = chain_st[g];
    if (g == 0 && s2 != h->st) WS_CUDA(cudaStreamWaitEvent(s2, h->ev_lo, 0));
    c.plan = h->dd_plan.as<DdDevPlan>() + g;
    c.cls_mask = g == 0 ? 0x1u : 0xEu;
    {
      Phase ph(h, nm[g][1], 0.0, 0, s2);
      launch_dd_tiles(c, cgrid, s2);
      ++h->launches;
    }
    {
      Phase ph(h, nm[g][2], 0.0, 0, s2);
      launch_dd_rank(c, cgrid, s2);
      ++h->launches;
    }
    {
      Phase ph(h, nm[g][3], 0.0, 0, s2);
      launch_dd_prefix(c, cgrid, s2);
      h->launches += 3;
    }
    {
      Phase ph(h, nm[g][4], 0.0, 0, s2);
      launch_dd_chain_expand(c, dd_expand_ctas_per_sm() * sms, s2);
      ++h->launches;
    }
  }
  h->dd_two_chains = true;
  cudaStream_t xs = chain_st[1];
  if (chain_st[0] != xs) {  // the side stream carries the end of both chains
    cudaEvent_t e = sync_event(h);
    WS_CUDA(cudaEventRecord(e, chain_st[0]));
    WS_CUDA(cudaStreamWaitEvent(xs, e, 0));
  }
  WS_CUDA(cudaEventRecord(h->ev_chain, xs));
  WS_TRY(check_launch("dd_chain"));
  h->dd_chain = true;
  return WS_OK;
}

int launch_early_hist(ws_handle* h, const uint64_t* region) {
  cudaStream_t cst = h->serial ? h->st : h->cs[0];
  DevBuf& tb = h->rtotals[0];
  WS_CUDA(tb.ensure(radix_c0_zero_bytes() + 64));
  if (cst != h->st) {
    // behind the ingest -- or, with the counting path launched, behind its
    // probe (not behind the counting launches that follow it on the main stream)
    cudaEvent_t ev = h->dd_launched ? h->ev_probe : sync_event(h);
    if (!h->dd_launched) WS_CUDA(cudaEventRecord(ev, h->st));
    WS_CUDA(cudaStreamWaitEvent(cst, ev, 0));
  }
  WS_CUDA(cudaMemsetAsync(tb.p, 0, radix_c0_zero_bytes(), cst));
  EarlyHist e;
  memset(&e, 0, sizeof e);
  e.fill = h->fill.as<uint32_t>();
  e.keys_cap = h->keys_cap.as<uint8_t>();
  for (int b = 0; b < 5; ++b) e.region[b] = region[b];
  e.totals = tb.as<uint32_t>();
  e.joint = e.totals + (size_t)kRadixC0Segs * kRadixMaxPasses * kRadixTotStride + kRadixMaxPasses;
  e.joint_ok = !env_on("WSORT_NO_JOINT");
  // with the counting path launched, a class's early launches run only if its probe gave the class up
  const uint32_t* dd_go = h->dd_launched ? h->dd_pool.as<uint32_t>() + kDdCtlProbe : nullptr;
  e.go = dd_go;
  {
    Phase ph(h, "radix_hist_l0", 0.0, 0, cst);  // bytes patched once the counts are known
    launch_radix_hist_early(e, cst);
    ++h->launches;
    if (h->prof) h->early_phase_first = h->phases.size() + 1;  // this record's index + 1
  }
  WS_TRY(check_launch("radix_hist_early"));
  h->early_done = true;
  h->early_joint = e.joint_ok != 0;
  // the multi-lane classes' split launches (payload-mode sample sort), each on
  // its class stream, buffers at their maximum size (no regrowth later)
  static const bool split_ok = !env_on("WSORT_NO_SAMPLE") && !env_on("WSORT_NO_EARLY_SPLIT");
  if (!split_ok) return WS_OK;
  uint32_t pmax = 1;
  while (pmax * 2 <= (uint32_t)std::min(sample_max_keys(1), 4096)) pmax *= 2;
  for (int c = 1; c <= 3; ++c) {  // 6-bit text keys: lengths 6-10, 11-21, 22-32
    const int lmin = c == 1 ? 6 : (c == 2 ? 11 : 22), lmax = c == 1 ? 10 : (c == 2 ? 21 : 32);
    const int nb = lmax - lmin + 1;
    WS_CUDA(h->ss_split[c].ensure((size_t)nb * kMaxSplit * key_bytes(c) + 64));
    WS_CUDA(h->ss_slots[c].ensure((size_t)nb * (2 * kMaxSplit + 1) * 12 + 64));
    // early count pass: slot ids for the most tiles the class's fitting buckets can have
    static const bool count_ok = !env_on("WSORT_NO_EARLY_COUNT");
    const uint64_t ptile = (uint64_t)part_tile_size();
    uint64_t max_tiles = 0;
    for (int L = lmin; L <= lmax; ++L)
      max_tiles += (std::min<uint64_t>((h->n_text + 1) / (L + 1), sample_bucket_limit(c)) + ptile - 1) / ptile;
    if (count_ok) {
      WS_CUDA(h->ss_ids[c].ensure((size_t)max_tiles * ptile * 2 + 64));
      WS_CUDA(h->early_plan[c].ensure(sizeof(SampleLaunch)));
    }
    cudaStream_t sst = h->serial ? h->st : h->cs[c];
    if (sst != h->st) {
      cudaEvent_t ev = h->dd_launched ? h->ev_probe : sync_event(h);
      if (!h->dd_launched) WS_CUDA(cudaEventRecord(ev, h->st));
      WS_CUDA(cudaStreamWaitEvent(sst, ev, 0));
    }
    SplitEarly se;
    memset(&se, 0, sizeof se);
    se.fill = h->fill.as<uint32_t>();
    se.keys_cap = h->keys_cap.as<uint8_t>();
    for (int b = 0; b < 32; ++b) se.region[b] = region[b];
    se.lmin = lmin;
    se.lmax = lmax;
    se.T = (uint32_t)subsort_tile_size(c);  // one slot up to a slot-sort tile (= 2 * target)
    se.target = (uint32_t)subsort_tile_size(c) / 2;
    se.pmax = pmax;
    se.smax = sample_smax(pmax);
    se.cap = sample_bucket_limit(c);
    se.splitters = h->ss_split[c].as<uint64_t>();
    se.hist = h->ss_slots[c].as<uint32_t>();
    se.go = dd_go ? dd_go + c : nullptr;
    if (count_ok) {
      se.plan = h->early_plan[c].as<SampleLaunch>();
      se.slot_ids = h->ss_ids[c].as<uint16_t>();
      se.ptile = (uint32_t)ptile;
    }
    {
      char nm[16];
      snprintf(nm, sizeof nm, "split_l%d", c);
      Phase ph(h, nm, 0.0, 0, sst);
      launch_sample_split_early(c, se, sst);
      ++h->launches;
    }
    h->split_early[c] = true;
    if (count_ok) {
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
      const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(max_tiles, 2ull * sms));
      char nm[20];
      snprintf(nm, sizeof nm, "part_count_l%d", c);
      Phase ph(h, nm, 0.0, 0, sst);
      launch_partition_count_early(c, h->early_plan[c].as<SampleLaunch>(), grid, sst, se.go);
      ++h->launches;
      h->count_early[c] = true;
    }
  }
  WS_TRY(check_launch("sample_split_early"));
  return WS_OK;
}

constexpr int kDdHostOff = 64;  // dedupe control words in the pinned read-back area (uint32 index)

int ingest_text_impl(ws_handle* h, const uint8_t* text, uint64_t n, int32_t flags,
                     std::mutex* gate = nullptr) {
  // batch mode: `gate` is held while this corpus crosses PCIe host->device
  std::unique_lock<std::mutex> gate_lk;
  if (gate) gate_lk = std::unique_lock<std::mutex>(*gate);
  if (n >= (1ull << 32) - kTextPad) return fail(WS_ERR_ARG, "text must be shorter than 4 GiB");
  const bool resident = (flags & WS_INGEST_RESIDENT) != 0;
  if (resident) {
    if (!h->text_valid || h->n_text != n || h->text.cap < n + kTextPad)
      return fail(WS_ERR_STATE, "WS_INGEST_RESIDENT without the same text already on the device");
  } else if (n && !text) {
    return fail(WS_ERR_ARG, "null text");
  }
  h->tiny_launched = h->tiny_done = false;
  h->dd_launched = h->dd_chain = false;
  h->dd_used = 0;
  for (bool& f : h->dd_ok) f = false;
  h->ingested = h->sorted = h->have_stats = h->payload_only = false;
  h->have_tokens = false;
  h->unordered = false;
  h->early_done = false;
  for (bool& f : h->split_early) f = false;
  h->buckets.clear();
  h->n_text = n;
  h->text_valid = false;
  h->enc = kEncAlnum6;  // tokens are [0-9A-Za-z] only
  if (!resident) WS_CUDA(h->text.ensure(n + kTextPad));
  // Large host texts are copied in pieces on their own stream and each piece
  // is ingested as soon as the next one has landed (its last words may run
  // into it), overlapping the H2D with the single-pass ingest.
  const char* force2 = getenv("WSORT_TWO_PASS");
  const bool single = n <= kSinglePassMaxText && !(force2 && force2[0] == '1');
  const char* nochunk = getenv("WSORT_NO_CHUNKED_H2D");
  const bool chunked = single && !resident && !(flags & WS_INGEST_DEVICE_PTR) &&
                       n >= kChunkedH2DMin && !(nochunk && nochunk[0] == '1');
  if (!resident && !chunked) {
    Phase ph(h, "h2d_text", (double)n, (flags & WS_INGEST_DEVICE_PTR) ? 0 : 1);
    if (n)
      WS_CUDA(cudaMemcpyAsync(h->text.p, text, n,
                              (flags & WS_INGEST_DEVICE_PTR) ? cudaMemcpyDeviceToDevice
                                                             : cudaMemcpyHostToDevice,
                              h->st));
    WS_CUDA(cudaMemsetAsync(static_cast<uint8_t*>(h->text.p) + n, 0, kTextPad, h->st));
    if (gate_lk.owns_lock()) {  // batch mode: the next corpus may start its upload now
      cudaEvent_t up = sync_event(h);
      WS_CUDA(cudaEventRecord(up, h->st));
      WS_CUDA(cudaEventSynchronize(up));
      gate_lk.unlock();
    }
  }
  const uint32_t nchunks = chunk_count(n);
  h->nchunks = nchunks;
  WS_CUDA(h->totals.ensure(kHistRows * 4));
  WS_CUDA(h->pin_small.ensure(1 << 16));
  const uint8_t* dtext = h->text.as<uint8_t>();
  uint32_t* tot_host = static_cast<uint32_t*>(h->pin_small.p);
  const bool keep_tokens = (flags & WS_INGEST_KEEP_TOKENS) != 0;
  ScatterParams p;
  memset(&p, 0, sizeof p);
  p.enc = h->enc;
  uint64_t region[kNumBins] = {0};
  uint64_t m = 0, total_words = 0;
  uint64_t counts[kNumBins];
  if (single) {
    // Capacity-bounded per-length regions: at most (n+1)/(L+1) words of length
    // L fit in n bytes. Bases are multiples of 12 words (16-byte aligned and
    // divisible by every lane count).
    uint64_t run = 0;
    for (int b = 0; b < kMaxPackedLen; ++b) {
      const int L = b + 1;
      region[b] = run;
      run += (n + 1) / (L + 1) * key_bytes(lanes_for_len_enc(L, h->enc));
      run = (run + 95) / 96 * 96;  // 16-byte aligned, a multiple of every key size
    }
    WS_CUDA(h->keys_cap.ensure(run + 256));
    WS_CUDA(h->longlist.ensure(((n + 1) / (kMaxPackedLen + 2) + 1) * sizeof(uint2)));
    if (keep_tokens) WS_CUDA(h->tokens.ensure(((n + 1) / 2 + 1) * sizeof(uint2)));
    // chunk placement: payload-only -> reserve (any order); ordered without
    // tokens -> reserve + runs reordered into corpus order afterwards;
    // tokens (their global word index needs every predecessor) -> look-back
    const bool reserve = (flags & WS_INGEST_UNORDERED) && !keep_tokens;
    static const char* lb_env = getenv("WSORT_LOOKBACK");
    const bool ordered_reserve = !reserve && !keep_tokens && !(lb_env && lb_env[0] == '1');
    const bool lookback = !reserve && !ordered_reserve;
    // distinct-word counting behind the ingest: the table pool is zeroed on a
    // side stream while the ingest runs
    const bool dd_try = reserve && h->dd_req && h->enc == kEncAlnum6 && !h->tiny_req && n > 0;
    if (dd_try) {
      // the counting path's two side streams exist only on handles that count
      // (a handle for small texts keeps the stream set its class chains were tuned with)
      if (!h->zs) {
        int prio_lo = 0, prio_hi = 0;
        cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
        WS_CUDA(cudaStreamCreateWithPriority(&h->zs, cudaStreamNonBlocking, prio_lo));
        WS_CUDA(cudaStreamCreateWithPriority(&h->xs, cudaStreamNonBlocking, prio_lo));
      }
      WS_TRY(dd_zero_pool(h, n, h->zs));
      WS_CUDA(cudaEventRecord(h->ev_zero, h->zs));
    }
    // the ordered reserve ingest of text keys runs on 8 KiB chunks (ingest7_kernel<true>)
    const uint64_t ocb = ordered_reserve && h->enc == kEncAlnum6 ? ordered_chunk_bytes() : ingest_chunk_bytes();
    const uint32_t nchunks = ordered_reserve ? (uint32_t)((n + ocb - 1) / ocb) : chunk_count(n);
    h->nchunks = nchunks;
    if (lookback) WS_CUDA(h->status.ensure((size_t)std::max<uint32_t>(nchunks, 1) * kLookbackRec * 4));
    if (ordered_reserve) {
      const size_t tb = (size_t)kHistRows * std::max<uint32_t>(nchunks, 1) * 4;
      WS_CUDA(h->run_at.ensure(tb));
      WS_CUDA(h->run_cnt.ensure(tb));
      WS_CUDA(h->run_off.ensure(tb));
      WS_CUDA(h->longlist2.ensure(((n + 1) / (kMaxPackedLen + 2) + 1) * sizeof(uint2)));
    }
    WS_CUDA(h->ticket.ensure(256));
    WS_CUDA(h->fill.ensure((kHistRows + 1) * 4));  // + the unknown-length counter
    for (int b = 0; b < kMaxPackedLen; ++b) p.bin_base[b] = region[b];
    p.keys = h->keys_cap.as<uint64_t>();
    p.longlist = h->longlist.as<uint2>();
    p.tokens = keep_tokens ? h->tokens.as<uint2>() : nullptr;
    p.chunk0 = 0;
    p.nchunks_total = nchunks;
    p.ticket = h->ticket.as<unsigned int>();
    p.status = h->status.as<uint32_t>();
    p.totals = h->totals.as<uint32_t>();
    p.fill = lookback ? nullptr : h->fill.as<uint32_t>();
    // fill[kHistRows]: long words whose length ingest7 leaves to long_len_fix
    p.unknown = lookback ? nullptr : h->fill.as<unsigned int>() + kHistRows;
    p.run_at = ordered_reserve ? h->run_at.as<uint32_t>() : nullptr;
    p.run_cnt = ordered_reserve ? h->run_cnt.as<uint32_t>() : nullptr;
    const void* totals_src = lookback ? h->totals.p : h->fill.p;
    auto reset_chain = [&]() -> int {
      if (!lookback) {
        WS_CUDA(cudaMemsetAsync(h->fill.p, 0, (kHistRows + 1) * 4, h->st));
      } else {
        WS_CUDA(cudaMemsetAsync(h->status.p, 0, (size_t)nchunks * kLookbackRec * 4, h->st));
        WS_CUDA(cudaMemsetAsync(h->ticket.p, 0, 4, h->st));
      }
      return WS_OK;
    };
    if (nchunks) {
      WS_TRY(reset_chain());
      bool redo = false;
      if (chunked) {
        WS_CUDA(h->overflow.ensure(256));
        WS_CUDA(cudaMemsetAsync(h->overflow.p, 0, 4, h->st));
        p.overflow = h->overflow.as<unsigned int>();
        const uint64_t cb = reserve ? reserve_chunk_bytes() : ocb;
        // pieces of >= 8 MB let the ingest start before the whole text has
        // landed; in batch mode (gate) other corpora fill that gap, and one
        // copy keeps PCIe faster while the device->host direction is busy
        const int P = gate ? 1 : (int)std::min<uint64_t>(16, std::max<uint64_t>(2, n / (8ull << 20)));
        const uint64_t piece = (n / P + cb - 1) / cb * cb;
        std::vector<uint64_t> edge;  // piece boundaries (bytes)
        for (uint64_t o = 0; o < n; o += piece) edge.push_back(o);
        edge.push_back(n);
        const int np = (int)edge.size() - 1;
        std::vector<cudaEvent_t> landed(np);
        for (int i = 0; i < np; ++i) {
          Phase ph(h, "h2d_text", (double)(edge[i + 1] - edge[i]), 1, h->hs);
          WS_CUDA(cudaMemcpyAsync(static_cast<uint8_t*>(h->text.p) + edge[i], text + edge[i],
                                  edge[i + 1] - edge[i], cudaMemcpyHostToDevice, h->hs));
          if (i == np - 1)
            WS_CUDA(cudaMemsetAsync(static_cast<uint8_t*>(h->text.p) + n, 0, kTextPad, h->hs));
          landed[i] = sync_event(h);
          WS_CUDA(cudaEventRecord(landed[i], h->hs));
        }
        for (int i = 0; i < np; ++i) {
          const int need = std::min(i + 1, np - 1);
          WS_CUDA(cudaStreamWaitEvent(h->st, landed[need], 0));
          ScatterParams pi = p;
          pi.avail = need == np - 1 ? 0 : edge[need + 1];
          const uint32_t c0 = (uint32_t)(edge[i] / cb), c1 = (uint32_t)((edge[i + 1] + cb - 1) / cb);
          pi.chunk0 = lookback ? 0 : c0;  // look-back numbers chunks by its global ticket
          Phase ph(h, "ingest", 2.27 * (double)(edge[i + 1] - edge[i]));
          launch_ingest_lookback(dtext, n, c1 - c0, pi, h->st);
          ++h->launches;
        }
        WS_TRY(check_launch("ingest_kernel"));
        if (gate_lk.owns_lock()) {  // the text has crossed PCIe: the next corpus may start
          WS_CUDA(cudaEventSynchronize(landed[np - 1]));
          gate_lk.unlock();
          if (getenv("WSORT_TRACE")) fprintf(stderr, "wsort-trace handle=%p h2d_landed=%.3f\n", (void*)h, trace_ms());
        }
        if (reserve && h->tiny_req && h->enc == kEncAlnum6) {
          WS_TRY(launch_tiny(h, region, n));
        } else {
          if (dd_try) WS_TRY(launch_dd_counting(h, region, 0));
          if (reserve && h->early_req && h->enc == kEncAlnum6) WS_TRY(launch_early_hist(h, region));
          if (dd_try) WS_TRY(launch_dd_counting(h, region, 1));
        }
        if (h->dd_launched)
          WS_CUDA(cudaMemcpyAsync(tot_host + kDdHostOff, h->dd_pool.p, kDdCtlWords * 4, cudaMemcpyDeviceToHost, h->st));
        WS_CUDA(cudaMemcpyAsync(tot_host + kHistRows, h->overflow.p, 4, cudaMemcpyDeviceToHost,
                                h->st));
        WS_CUDA(cudaMemcpyAsync(tot_host, totals_src, kHistRows * 4, cudaMemcpyDeviceToHost, h->st));
        tot_host[kHistRows + 2] = 0;
        if (p.unknown)
          WS_CUDA(cudaMemcpyAsync(tot_host + kHistRows + 2, p.unknown, 4, cudaMemcpyDeviceToHost, h->st));
        WS_CUDA(cudaStreamSynchronize(h->st));
        redo = tot_host[kHistRows] != 0;  // a word spanned a whole piece: ingest again
        if (redo) {
          p.overflow = nullptr;
          h->early_done = false;
          for (bool& f : h->split_early) f = false;
          for (bool& f : h->count_early) f = false;
          WS_TRY(reset_chain());  // (a second dd_aggregate launch zeroes the pool itself)
        }
      }
      if (!chunked || redo) {
        {
          // algorithmic bytes: text read + keys written (estimated from the text; exact
          // counts are only known afterwards)
          Phase ph(h, "ingest", (double)n + 1.27 * (double)n);
          launch_ingest_lookback(dtext, n, reserve ? (uint32_t)((n + reserve_chunk_bytes() - 1) /
                                                                reserve_chunk_bytes())
                                                   : nchunks,
                                 p, h->st);
          ++h->launches;
        }
        WS_TRY(check_launch("ingest_kernel"));
        if (reserve && h->tiny_req && h->enc == kEncAlnum6) {
          WS_TRY(launch_tiny(h, region, n));
        } else {
          if (dd_try) WS_TRY(launch_dd_counting(h, region, 0));
          if (reserve && h->early_req && h->enc == kEncAlnum6) WS_TRY(launch_early_hist(h, region));
          if (dd_try) WS_TRY(launch_dd_counting(h, region, 1));
        }
        if (h->dd_launched)
          WS_CUDA(cudaMemcpyAsync(tot_host + kDdHostOff, h->dd_pool.p, kDdCtlWords * 4, cudaMemcpyDeviceToHost, h->st));
        tmark("early_enq");
        WS_CUDA(cudaMemcpyAsync(tot_host, totals_src, kHistRows * 4, cudaMemcpyDeviceToHost, h->st));
        if (h->tiny_launched)
          WS_CUDA(cudaMemcpyAsync(tot_host + kHistRows + 1, h->tiny_flag.p, 4, cudaMemcpyDeviceToHost, h->st));
        tot_host[kHistRows + 2] = 0;
        if (p.unknown)
          WS_CUDA(cudaMemcpyAsync(tot_host + kHistRows + 2, p.unknown, 4, cudaMemcpyDeviceToHost, h->st));
        WS_CUDA(cudaStreamSynchronize(h->st));
        h->tiny_done = h->tiny_launched && tot_host[kHistRows + 1] == 0 && tot_host[kLongBin] == 0;
        if (h->tiny_launched && env_on("WSORT_TINY_PROF")) {
          unsigned long long tp[2 * kMaxPackedLen];
          WS_CUDA(cudaMemcpy(tp, h->tiny_prof.p, sizeof tp, cudaMemcpyDeviceToHost));
          unsigned long long t0 = ~0ull;
          for (int b = 0; b < kMaxPackedLen; ++b) if (tp[2 * b]) t0 = std::min(t0, tp[2 * b]);
          fprintf(stderr, "wsort-tiny");
          for (int b = 0; b < kMaxPackedLen; ++b)
            if (tp[2 * b]) fprintf(stderr, " L%d:%u[%.1f,%.1f]", b + 1, tot_host[b], (tp[2 * b] - t0) * 1e-3, (tp[2 * b + 1] - t0) * 1e-3);
          fprintf(stderr, " us\n");
          unsigned long long ph[16 * kMaxPackedLen];
          WS_CUDA(cudaMemcpy(ph, h->tiny_prof.as<unsigned long long>() + 64, sizeof ph, cudaMemcpyDeviceToHost));
          for (int b = 0; b < kMaxPackedLen; ++b) {
            if (!tp[2 * b]) continue;
            fprintf(stderr, "wsort-tiny-phases L%d:", b + 1);
            for (int k = 2; k < 16; ++k) if (ph[16 * b + k]) fprintf(stderr, " %d:%.2f", k, (ph[16 * b + k] - tp[2 * b]) * 1e-3);
            fprintf(stderr, "\n");
          }
        }
        tmark("sync_ret");
      }
    } else {
      memset(tot_host, 0, kHistRows * 4);
    }
    for (int b = 0; b < kNumBins; ++b) counts[b] = tot_host[b];
    total_words = tot_host[kNumBins];
    m = counts[kLongBin];
    tmark("synced");
    WS_TRY(plan_packed(h, counts));  // compact layout of the sort buffers
    tmark("planned");
    if (h->dd_launched) {
      // classes whose buckets all stayed in budget sort their distinct words only
      const uint32_t* ctl = tot_host + kDdHostOff;
      uint32_t n32[kDdLens];
      for (int b = 0; b < kDdLens; ++b) n32[b] = (uint32_t)counts[b];
      dd_host_layout(n32, h->dd_lay);
      for (int c = 0; c < 4; ++c) h->dd_ok[c] = ctl[kDdCtlSkip + c] != 0;
      for (auto& bk : h->buckets) {
        if (bk.is_long || !h->dd_ok[bk.lanes]) continue;
        bk.dd_n = ctl[kDdCtlCount + bk.len - 1];
        if (bk.dd_n == 0 || bk.dd_n > h->dd_lay.dcap[bk.len - 1] || bk.dd_n > bk.count)
          return fail(WS_ERR_STATE, "distinct-word count out of range");
      }
      // a class's early launches ran only if the probe gave the class up
      // (a class that ran out of budget later sorts without them)
      if (!ctl[kDdCtlProbe + 0]) h->early_done = false;
      for (int c = 1; c < 4; ++c)
        if (!ctl[kDdCtlProbe + c]) h->split_early[c] = h->count_early[c] = false;
      if (h->prof) {
        double kb = 0, kb0 = 0;
        for (auto& bk : h->buckets)
          if (!bk.is_long) {
            kb += (double)bk.count * key_bytes(bk.lanes);
            if (bk.lanes == 0) kb0 += (double)bk.count * 4.0;
          }
        double dkb = 0, pay = 0, dkb0 = 0, pay0 = 0;  // counted classes: distinct keys, payload records (0: class 0)
        for (auto& bk : h->buckets)
          if (!bk.is_long && h->dd_ok[bk.lanes]) {
            dkb += (double)bk.dd_n * (key_bytes(bk.lanes) + 4.0);
            pay += (double)bk.count * (bk.len + 1);
            if (bk.lanes == 0) {
              dkb0 += (double)bk.dd_n * 8.0;
              pay0 += (double)bk.count * (bk.len + 1);
            }
          }
        for (auto& r : h->phases) {
          if (r.bytes != 0.0) continue;
          if (r.name == "dd_aggregate") r.bytes = kb0;
          else if (r.name == "dd_aggregate_hi") r.bytes = kb - kb0;
          else {  // chain kernels: "_hi" = the chain of classes 1-3 when two chains run
            const bool hi = r.name.size() > 3 && r.name.compare(r.name.size() - 3, 3, "_hi") == 0;
            const std::string base = hi ? r.name.substr(0, r.name.size() - 3) : r.name;
            const bool two = h->dd_two_chains;
            const double dk1 = !two ? dkb : (hi ? dkb - dkb0 : dkb0), py = !two ? pay : (hi ? pay - pay0 : pay0);
            if (base == "dd_tiles" || base == "dd_rank") r.bytes = std::max(1.0, 2.0 * dk1);  // keys + occurrences in and out
            else if (base == "dd_prefix") r.bytes = std::max(1.0, dk1);
            else if (base == "dd_expand") r.bytes = std::max(1.0, py + dk1);
          }
        }
      }
    }
    if (h->prof && h->early_phase_first) {  // bytes of the device-planned early launches
      for (size_t i = h->early_phase_first - 1; i < h->phases.size(); ++i) {
        PhaseRec& r = h->phases[i];
        double b = r.bytes;
        if (r.name == "radix_hist_l0") {
          b = 0;
          for (int L = 1; L <= 5; ++L) b += 4.0 * (double)counts[L - 1];  // keys read once
        } else if (r.name.rfind("split_l", 0) == 0) {
          const int c = r.name[7] - '0';
          b = 0;
          for (int L = 1; L <= kMaxPackedLen; ++L)  // sampled keys read
            if (lanes_for_len_enc(L, h->enc) == c && counts[L - 1])
              b += (double)key_bytes(c) * std::min<double>((double)counts[L - 1], 4096.0);
        } else if (r.name.rfind("part_count_l", 0) == 0) {
          const int c = r.name[12] - '0';
          b = 0;
          for (int L = 1; L <= kMaxPackedLen; ++L)  // keys read (first word for one-word keys), slot ids written
            if (lanes_for_len_enc(L, h->enc) == c && counts[L - 1] <= sample_bucket_limit(c))
              b += (double)counts[L - 1] * ((c == 1 ? 8.0 : (double)key_bytes(c)) + 2.0);
        }
        r.bytes = b;
        // a counted class's early launches returned at once (device flag): their
        // records keep the launch but not the sort path's name or bytes
        int ec = -1;
        if (r.name == "radix_hist_l0") ec = 0;
        else if (r.name.rfind("split_l", 0) == 0) ec = r.name[7] - '0';
        else if (r.name.rfind("part_count_l", 0) == 0) ec = r.name[12] - '0';
        if (ec >= 0 && ec < 4 && h->dd_launched && !tot_host[kDdHostOff + kDdCtlProbe + ec]) {
          r.name = "gated_" + r.name;
          r.bytes = 0;
        }
      }
      h->early_phase_first = 0;
    }
    if (ordered_reserve && nchunks) {
      // corpus order: runs of every (bin, chunk) move from their reserved place
      // to the exclusive prefix of their bin over chunks, in the compact layout
      launch_scan(h->run_cnt.as<uint32_t>(), h->run_off.as<uint32_t>(), h->totals.as<uint32_t>(),
                  nchunks, kNumBins, h->st);
      ReorderParams r;
      memset(&r, 0, sizeof r);
      r.nchunks = nchunks;
      r.run_at = h->run_at.as<uint32_t>();
      r.run_cnt = h->run_cnt.as<uint32_t>();
      r.run_off = h->run_off.as<uint32_t>();
      for (const auto& bk : h->buckets) {
        const int b = (int)bk.len - 1;
        r.src[b] = h->keys_cap.as<uint8_t>() + region[b];
        r.dst[b] = reinterpret_cast<uint8_t*>(class_keys(h, 0, bk.lanes, bk.elem_off));
        r.key_bytes[b] = (uint32_t)key_bytes(bk.lanes);
      }
      r.src[kLongBin] = h->longlist.as<uint8_t>();
      r.dst[kLongBin] = h->longlist2.as<uint8_t>();
      r.key_bytes[kLongBin] = sizeof(uint2);
      {
        Phase ph(h, "reorder", 2.0 * (double)(h->class_base[kClasses] + h->class_elems[kClasses] * key_bytes(kClasses)));
        launch_reorder_runs(r, h->st);
        h->launches += 2;
      }
      WS_TRY(check_launch("reorder_runs"));
      std::swap(h->longlist, h->longlist2);  // the long list is now in corpus order
    } else {
      for (auto& bk : h->buckets)
        if (!bk.is_long)
          bk.in_ptr =
              reinterpret_cast<const uint64_t*>(h->keys_cap.as<uint8_t>() + region[bk.len - 1]);
    }
    if (keep_tokens) h->have_tokens = true;
    h->unordered = reserve;
  } else {
    const size_t hist_bytes = (size_t)kHistRows * std::max<uint32_t>(nchunks, 1) * 4;
    WS_CUDA(h->hist.ensure(hist_bytes));
    WS_CUDA(h->off.ensure(hist_bytes));
    if (nchunks) {
      {
        Phase ph(h, "count", (double)n);
        launch_count(dtext, n, h->hist.as<uint32_t>(), nchunks, h->st);
        ++h->launches;
      }
      WS_TRY(check_launch("count_kernel"));
      {
        Phase ph(h, "scan", (double)kHistRows * nchunks * 8);
        launch_scan(h->hist.as<uint32_t>(), h->off.as<uint32_t>(), h->totals.as<uint32_t>(),
                    nchunks, kHistRows, h->st);
        ++h->launches;
      }
      WS_TRY(check_launch("scan_kernel"));
      WS_CUDA(cudaMemcpyAsync(tot_host, h->totals.p, kHistRows * 4, cudaMemcpyDeviceToHost, h->st));
      WS_CUDA(cudaStreamSynchronize(h->st));
    } else {
      memset(tot_host, 0, kHistRows * 4);
    }
    for (int b = 0; b < kNumBins; ++b) counts[b] = tot_host[b];
    total_words = tot_host[kNumBins];
    WS_TRY(plan_packed(h, counts));
    m = counts[kLongBin];
    WS_CUDA(h->longlist.ensure(std::max<uint64_t>(m, 1) * sizeof(uint2)));
    fill_scatter_params(h, p);
    if (keep_tokens) {
      WS_CUDA(h->tokens.ensure(std::max<uint64_t>(total_words, 1) * sizeof(uint2)));
      p.tokens = h->tokens.as<uint2>();
      h->have_tokens = true;
    }
    if (nchunks) {
      double kbytes = 0;
      for (auto& b : h->buckets) kbytes += (double)b.count * key_bytes(b.lanes);
      Phase ph(h, "scatter", (double)n + kbytes + 8.0 * m);
      launch_scatter(dtext, n, h->off.as<uint32_t>(), nchunks, p, h->st);
      ++h->launches;
    }
    WS_TRY(check_launch("scatter_kernel"));
  }
  if (single && tot_host[kHistRows + 2] && m) {  // long words the ingest left unmeasured
    WS_CUDA(h->first_sep.ensure(long_fix_chunks(n) * 4 + 64));
    launch_long_len_fix(dtext, n, h->longlist.as<uint2>(), m, h->first_sep.as<uint32_t>(), h->st);
    h->launches += 2;
    WS_TRY(check_launch("long_len_fix"));
  }
  WS_TRY(group_long_words(h, m));
  tmark("grouped");
  h->words = total_words;
  h->text_valid = true;
  return finish_ingest(h);
}

// ----------------------------------------------------------------------------
// sort of all buckets

int emit_device(ws_handle* h, uint8_t* dout, bool lines, std::vector<uint64_t>* offsets,
                int only = -1, cudaStream_t st = nullptr,
                const std::vector<int>* subset = nullptr);
std::vector<uint64_t> emit_offsets(ws_handle* h, bool lines);

// Optional fused emission: as soon as a lane class is sorted, its stream
// emits that class's payload bytes (one contiguous range, buckets ascend by
// length) and starts the D2H copy, overlapping with the classes still sorting.
struct FusedEmit {
  uint8_t* dout;  // device payload buffer
  uint8_t* host;  // host destination
  std::vector<uint64_t> off;
  bool per_class = false;  // one emit + D2H per lane class instead of per finished bucket
};

int fused_class_copy(ws_handle* h, FusedEmit* fe, int cls, cudaStream_t st) {
  uint64_t lo = UINT64_MAX, hi = 0, sum = 0;
  for (size_t i = 0; i < h->buckets.size(); ++i) {
    const Bucket& b = h->buckets[i];
    if ((b.is_long ? kLongCls : b.lanes) != cls || !b.count) continue;
    lo = std::min(lo, fe->off[i]);
    hi = std::max(hi, fe->off[i + 1]);
    sum += fe->off[i + 1] - fe->off[i];
  }
  if (!sum) return WS_OK;
  WS_TRY(emit_device(h, fe->dout, true, nullptr, cls, st));
  if (!fe->host) return WS_OK;  // device-resident output
  if (hi - lo != sum) return fail(WS_ERR_STATE, "lane class payload is not contiguous");
  Phase ph(h, "d2h_out", (double)sum, 1, st);
  WS_CUDA(cudaMemcpyAsync(fe->host + lo, fe->dout + lo, sum, cudaMemcpyDeviceToHost, st));
  return WS_OK;
}

int sort_impl(ws_handle* h, bool stats, FusedEmit* fe = nullptr) {
  tmark("sort_impl");
  if (!h->ingested) return fail(WS_ERR_STATE, "ws_sort before ingest");
  if (stats && h->unordered)
    return fail(WS_ERR_STATE, "stats need corpus order: ingest without WS_INGEST_UNORDERED");
  if (fe) h->sorted = true;  // bucket final buffers are fixed at planning time
  h->dd_used = 0;
  h->payload_only = false;
  const int nb = (int)h->buckets.size();
  if (stats) {
    WS_CUDA(h->idx[0].ensure(std::max<uint64_t>(h->idx_total, 1) * 4 + 64));
    WS_CUDA(h->idx[1].ensure(std::max<uint64_t>(h->idx_total, 1) * 4 + 64));
    WS_CUDA(h->stat_inv.ensure((size_t)std::max(nb, 1) * 16));
    WS_CUDA(h->stat_k.ensure((size_t)std::max(nb, 1) * 16));
    WS_CUDA(h->stat_k_dummy.ensure((size_t)std::max(nb, 1) * 16));
    WS_CUDA(cudaMemsetAsync(h->stat_inv.p, 0, (size_t)std::max(nb, 1) * 8, h->st));
    WS_CUDA(cudaMemsetAsync(h->stat_k.p, 0, (size_t)std::max(nb, 1) * 8, h->st));
  }
  unsigned long long* inv = stats ? h->stat_inv.as<unsigned long long>() : nullptr;
  long long* km = stats ? h->stat_k.as<long long>() : nullptr;
  // packed buckets: one schedule per lane class, each class on its own stream
  // (the classes are independent; small classes fill the big one's bubbles)
  WS_CUDA(cudaEventRecord(h->ev_fork, h->st));
  // class 0 (radix: a chain of small passes, the longest) is submitted first
  // on a high-priority stream; the multi-lane classes fill around it
  static int order[kClasses + 1] = {0, 1, 2, 3, 4};
  static const bool order_set = [] {  // experiment: WSORT_CLASS_ORDER=3,2,1,0,4
    if (const char* o = getenv("WSORT_CLASS_ORDER")) {
      for (int i = 0; i <= kClasses && *o; ++i) {
        order[i] = *o - '0';
        o += (o[1] == ',') ? 2 : 1;
      }
    }
    return true;
  }();
  (void)order_set;
  static const bool trace_cls = env_on("WSORT_TRACE");
  double t_cls = trace_cls ? trace_ms() : 0;
  for (int oi = 0; oi <= kClasses; ++oi) {
    const int c = order[oi];
    if (trace_cls && oi) {
      fprintf(stderr, "wsort-trace enqueue class %d: %.3f ms\n", order[oi - 1], trace_ms() - t_cls);
      t_cls = trace_ms();
    }
    std::vector<SegIn> segs;
    std::vector<int> which;
    // a counted class: its words were counted behind the ingest and every bucket stayed in budget
    const bool dd_cls = !stats && fe && !fe->per_class && c < 4 && h->dd_ok[c] && h->unordered && h->dd_chain;
    for (int i = 0; i < nb; ++i) {
      const Bucket& b = h->buckets[i];
      if (b.is_long || b.lanes != c) continue;
      segs.push_back(SegIn{b.elem_off, b.idx_off, (uint32_t)b.count, (uint32_t)i, 0, 0});
      segs.back().in_ptr = b.in_ptr;
      which.push_back(i);
    }
    if (segs.empty()) continue;
    if (dd_cls) h->dd_used |= 1 << c;
    if (dd_cls) {
      // the device-planned chain behind the ingest writes this class's payload
      h->payload_only = true;
      if (fe->host) {
        cudaStream_t dst = h->ds[c];
        uint64_t lo = UINT64_MAX, hi = 0;
        for (int i : which) {
          lo = std::min(lo, fe->off[i]);
          hi = std::max(hi, fe->off[i + 1]);
        }
        WS_CUDA(cudaStreamWaitEvent(dst, h->ev_chain, 0));
        {
          Phase ph(h, "d2h_out", (double)(hi - lo), 1, dst);
          WS_CUDA(cudaMemcpyAsync(fe->host + lo, fe->dout + lo, hi - lo, cudaMemcpyDeviceToHost, dst));
        }
        cudaEvent_t e2 = sync_event(h);
        WS_CUDA(cudaEventRecord(e2, dst));
        WS_CUDA(cudaStreamWaitEvent(h->st, e2, 0));
      }
      continue;
    }
    static const char* cls_mark[kClasses + 1] = {"cls0", "cls1", "cls2", "cls3", "cls4"};
    tmark(cls_mark[c]);
    cudaStream_t cst = h->serial ? h->st : h->cs[c];
    cudaStream_t est = h->serial ? h->st : h->es[c];
    cudaStream_t dst = h->serial ? h->st : h->ds[c];
    WS_CUDA(cudaStreamWaitEvent(cst, h->ev_fork, 0));
    uint64_t* k0 = class_keys(h, 0, c, 0);
    uint64_t* k1 = class_keys(h, 1, c, 0);
    // Fused emission: a bucket is emitted (and copied to the host) right after
    // the pass that completes it, on side streams, while later passes run.
    // side streams used by this class (only those are joined back; a fused
    // bucket needs no emit, and device-resident output needs no copy)
    bool used_est = fe && fe->per_class, used_dst = fe && fe->per_class;
    PassDoneHook hook = [&, est, dst](const std::vector<const SegIn*>& done,
                                      cudaStream_t st) -> int {
      std::vector<int> bids, to_emit;
      for (const SegIn* sg : done) {
        h->buckets[sg->stat_slot].final_buf = sg->final_buf;
        bids.push_back((int)sg->stat_slot);
        if (!sg->emitted) to_emit.push_back((int)sg->stat_slot);
      }
      cudaStream_t ready = st;  // the stream after which the buckets' records are complete
      if (!to_emit.empty()) {
        if (est != st) {
          cudaEvent_t ev = sync_event(h);
          WS_CUDA(cudaEventRecord(ev, st));
          WS_CUDA(cudaStreamWaitEvent(est, ev, 0));
        }
        WS_TRY(emit_device(h, fe->dout, true, nullptr, -1, est, &to_emit));
        ready = est;
        used_est = true;
      }
      if (!fe->host) return WS_OK;
      if (dst != ready) {
        cudaEvent_t ev2 = sync_event(h);
        WS_CUDA(cudaEventRecord(ev2, ready));
        WS_CUDA(cudaStreamWaitEvent(dst, ev2, 0));
      }
      used_dst = true;
      std::sort(bids.begin(), bids.end());
      size_t k = 0;
      while (k < bids.size()) {  // coalesce adjacent output ranges
        uint64_t lo = fe->off[bids[k]], hi = fe->off[bids[k] + 1];
        size_t j = k + 1;
        while (j < bids.size() && fe->off[bids[j]] == hi) hi = fe->off[bids[j++] + 1];
        if (hi > lo) {
          Phase ph(h, "d2h_out", (double)(hi - lo), 1, dst);
          WS_CUDA(cudaMemcpyAsync(fe->host + lo, fe->dout + lo, hi - lo, cudaMemcpyDeviceToHost,
                                  dst));
        }
        k = j;
      }
      return WS_OK;
    };
    static const char* no_radix = getenv("WSORT_NO_RADIX");
    const PassDoneHook* on_done = fe && !fe->per_class ? &hook : nullptr;
    static const char* no_sample = getenv("WSORT_NO_SAMPLE");
    if (!stats && c == 0 && !(no_radix && no_radix[0] == '1')) {
      // the last pass of each bucket writes its payload records directly
      static const char* no_fuse = getenv("WSORT_NO_FUSED_PAYLOAD");
      const bool fuse = on_done && !(no_fuse && no_fuse[0] == '1') && !dd_cls;
      WS_TRY(radix_sort_segments(h, c, segs, k0, k1, cst, on_done, fuse ? fe->dout : nullptr,
                                 fuse ? &fe->off : nullptr));
      for (const SegIn& sg : segs) h->payload_only |= sg.emitted;
      h->payload_only |= dd_cls;
    } else if (!stats && c >= 1 && !(no_sample && no_sample[0] == '1')) {
      // buckets beyond what the splitter budget keeps at slot size go through
      // the merge path (same stream; both leave per-bucket final buffers)
      std::vector<SegIn> fit, big;
      std::vector<int> fit_w, big_w;
      const uint64_t cap = sample_bucket_limit(c);
      for (size_t j = 0; j < segs.size(); ++j) {
        if (segs[j].n <= cap) { fit.push_back(segs[j]); fit_w.push_back(which[j]); }
        else { big.push_back(segs[j]); big_w.push_back(which[j]); }
      }
      static const char* no_fuse_s = getenv("WSORT_NO_FUSED_PAYLOAD");
      static const char* no_fuse_slots = getenv("WSORT_NO_FUSED_SLOTS");
      static const char* fuse_mask = getenv("WSORT_FUSED_SLOT_CLASSES");  // experiment: bit c = class c
      const bool fuse_s = on_done && !dd_cls && !(no_fuse_s && no_fuse_s[0] == '1') &&
                          !(no_fuse_slots && no_fuse_slots[0] == '1') &&
                          (!fuse_mask || ((strtol(fuse_mask, nullptr, 0) >> c) & 1));
      if (!fit.empty())
        WS_TRY(sample_sort_segments(h, c, fit, k1, cst, on_done, fuse_s ? fe->dout : nullptr,
                                    fuse_s ? &fe->off : nullptr));
      if (!big.empty())
        WS_TRY(sort_segments(h, c, big, k0, k1, h->idx[0].as<uint32_t>(), h->idx[1].as<uint32_t>(),
                             false, nullptr, nullptr, "", cst, on_done));
      size_t fi = 0, bi = 0;  // final buffers back into the class's segment order
      for (size_t j = 0; j < segs.size(); ++j)
        segs[j].final_buf = segs[j].n <= cap ? fit[fi++].final_buf : big[bi++].final_buf;
      for (const SegIn& sg : fit) h->payload_only |= sg.emitted;
      h->payload_only |= dd_cls;
      (void)fit_w; (void)big_w;
    } else {
      WS_TRY(sort_segments(h, c, segs, k0, k1, h->idx[0].as<uint32_t>(),
                           h->idx[1].as<uint32_t>(), stats, inv, km, "", cst, on_done));
    }
    if (fe && fe->per_class) {
      for (size_t j = 0; j < segs.size(); ++j) h->buckets[which[j]].final_buf = segs[j].final_buf;
      WS_TRY(fused_class_copy(h, fe, c, cst));
    }
    for (size_t j = 0; j < segs.size(); ++j) h->buckets[which[j]].final_buf = segs[j].final_buf;
    WS_CUDA(cudaEventRecord(h->ev_join[c], cst));
    WS_CUDA(cudaStreamWaitEvent(h->st, h->ev_join[c], 0));
    if (fe && used_est && est != h->st) {
      cudaEvent_t e1 = sync_event(h);
      WS_CUDA(cudaEventRecord(e1, est));
      WS_CUDA(cudaStreamWaitEvent(h->st, e1, 0));
    }
    if (fe && used_dst && dst != h->st) {
      cudaEvent_t e2 = sync_event(h);
      WS_CUDA(cudaEventRecord(e2, dst));
      WS_CUDA(cudaStreamWaitEvent(h->st, e2, 0));
    }
  }
  // long groups: LSD over 8-byte lanes, least significant lane first
  if (h->n_long) {
    const uint64_t m = h->n_long;
    WS_CUDA(h->rank.ensure(m * 4 + 64));
    WS_CUDA(h->rank_tmp.ensure(m * 4 + 64));
    launch_iota_u32(h->rank.as<uint32_t>(), m, h->st);  // rank[i] = i
    ++h->launches;
    int max_lanes = 0;
    for (auto& b : h->buckets)
      if (b.is_long && b.count > 1) max_lanes = std::max(max_lanes, lanes_for_len(b.len));
    const uint8_t* ltext = h->text.as<uint8_t>();
    for (int lane = max_lanes - 1; lane >= 0; --lane) {
      std::vector<SegIn> segs;
      std::vector<int> which;
      for (int i = 0; i < nb; ++i) {
        const Bucket& b = h->buckets[i];
        if (!b.is_long || b.count < 2 || lanes_for_len(b.len) <= lane) continue;
        segs.push_back(SegIn{b.long_off, b.long_off, (uint32_t)b.count, (uint32_t)i,
                             (uint32_t)b.long_off, 0});
        which.push_back(i);
      }
      launch_lane_keys(ltext, h->longgrp.as<uint2>(), h->rank.as<uint32_t>(), m, lane,
                       h->lkeys[0].as<uint64_t>(), h->st);
      ++h->launches;
      WS_TRY(sort_segments(h, 1, segs, h->lkeys[0].as<uint64_t>(), h->lkeys[1].as<uint64_t>(),
                           h->lidx[0].as<uint32_t>(), h->lidx[1].as<uint32_t>(), true,
                           h->stat_k_dummy.as<unsigned long long>(),
                           h->stat_k_dummy.as<long long>(), "llsd_"));
      for (size_t j = 0; j < segs.size(); ++j) {
        const Bucket& b = h->buckets[which[j]];
        const uint32_t* perm = h->lidx[segs[j].final_buf].as<uint32_t>() + b.long_off;
        launch_gather_u32(h->rank.as<uint32_t>(), perm, b.count,
                          h->rank_tmp.as<uint32_t>() + b.long_off, h->st);
        ++h->launches;
        WS_CUDA(cudaMemcpyAsync(h->rank.as<uint32_t>() + b.long_off,
                                h->rank_tmp.as<uint32_t>() + b.long_off, b.count * 4,
                                cudaMemcpyDeviceToDevice, h->st));
      }
    }
    if (stats) {
      // inversions of each group's final rank sequence; K = max(rank[i] - i)
      launch_iota_keys(h->rank.as<uint32_t>(), m, h->lkeys[0].as<uint64_t>(), h->st);
      ++h->launches;
      std::vector<SegIn> segs;
      for (int i = 0; i < nb; ++i) {
        const Bucket& b = h->buckets[i];
        if (!b.is_long) continue;
        segs.push_back(SegIn{b.long_off, b.long_off, (uint32_t)b.count, (uint32_t)i,
                             (uint32_t)b.long_off, 0});
        launch_rank_kmax(h->rank.as<uint32_t>(), b.long_off, b.count, km + i, h->st);
        ++h->launches;
      }
      WS_TRY(sort_segments(h, 1, segs, h->lkeys[0].as<uint64_t>(), h->lkeys[1].as<uint64_t>(),
                           h->lidx[0].as<uint32_t>(), h->lidx[1].as<uint32_t>(), true, inv,
                           h->stat_k_dummy.as<long long>(), "linv_"));
    }
  }
  if (fe && h->n_long) WS_TRY(fused_class_copy(h, fe, kLongCls, h->st));
  if (stats && nb) {
    std::vector<int64_t> hinv(nb), hk(nb);
    WS_CUDA(cudaMemcpyAsync(hinv.data(), h->stat_inv.p, nb * 8, cudaMemcpyDeviceToHost, h->st));
    WS_CUDA(cudaMemcpyAsync(hk.data(), h->stat_k.p, nb * 8, cudaMemcpyDeviceToHost, h->st));
    WS_CUDA(cudaStreamSynchronize(h->st));
    for (int i = 0; i < nb; ++i) {
      h->buckets[i].inv = hinv[i];
      h->buckets[i].kmax = hk[i];
    }
  }
  // the call ends after the counted classes' chains (joined last: classes that
  // are sorted fork from the main stream above and run beside them)
  if (h->dd_chain) WS_CUDA(cudaStreamWaitEvent(h->st, h->ev_chain, 0));
  WS_TRY(check_launch("sort"));
  h->early_done = false;  // early launches serve only the sort right after their ingest
  for (bool& f : h->dd_ok) f = false;  // ... and so do the distinct-word counts
  for (bool& f : h->split_early) f = false;
  h->sorted = true;
  h->have_stats = stats;
  return WS_OK;
}

// ----------------------------------------------------------------------------
// emit

const uint64_t* bucket_keys(ws_handle* h, const Bucket& b, bool sorted) {
  if (!sorted && b.in_ptr) return b.in_ptr;
  const int buf = sorted ? b.final_buf : 0;
  return class_keys(h, buf, b.lanes, b.elem_off);
}

// Enqueue emission of all buckets into device buffer `dout` (lines or rows).
// Byte offset of every bucket in the payload (ascending bucket order), plus the total.
std::vector<uint64_t> emit_offsets(ws_handle* h, bool lines) {
  std::vector<uint64_t> off(h->buckets.size() + 1);
  uint64_t run = 0;
  for (size_t i = 0; i < h->buckets.size(); ++i) {
    off[i] = run;
    run += h->buckets[i].count * (h->buckets[i].len + (lines ? 1 : 0));
  }
  off.back() = run;
  return off;
}

// Enqueue emission into device buffer `dout`: lane class `only` (1..4), the
// long groups (0), or everything (-1), on stream `st`.
int emit_device(ws_handle* h, uint8_t* dout, bool lines, std::vector<uint64_t>* offsets,
                int only, cudaStream_t st, const std::vector<int>* subset) {
  if (!st) st = h->st;
  const int nl = lines ? 1 : 0;
  std::vector<uint64_t> off = emit_offsets(h, lines);
  std::vector<char> pick(h->buckets.size(), subset ? 0 : 1);
  if (subset)
    for (int i : *subset) pick[i] = 1;
  double kb = 0, ob = 0;
  for (size_t i = 0; i < h->buckets.size(); ++i) {
    const Bucket& b = h->buckets[i];
    const int cls = b.is_long ? kLongCls : b.lanes;
    if ((only != -1 && cls != only) || !pick[i]) continue;
    kb += b.is_long ? 0.0 : (double)b.count * key_bytes(b.lanes);
    ob += (double)(off[i + 1] - off[i]);
  }
  char name[32];
  snprintf(name, sizeof name, "%s%s", lines ? "emit_lines" : "emit_rows",
           only == -1 ? "" : (only == kLongCls ? "_long" : (only == 0 ? "_l0" : only == 1 ? "_l1" : only == 2 ? "_l2" : only == 3 ? "_l3" : "_l4")));
  Phase ph(h, name, kb + ob, 0, st);
  for (int c = 0; c <= kClasses; ++c) {
    if (only != -1 && only != c) continue;
    std::vector<EmitSeg> segs;
    uint32_t blocks = 0;
    for (size_t i = 0; i < h->buckets.size(); ++i) {
      const Bucket& b = h->buckets[i];
      if (b.is_long || b.lanes != c || !b.count || !pick[i]) continue;
      EmitSeg e;
      e.keys = bucket_keys(h, b, h->sorted);
      e.out_off = off[i];
      e.n = (uint32_t)b.count;
      e.len = b.len;
      e.block_begin = blocks;
      e.pad_ = 0;
      blocks += (uint32_t)((b.count + kEmitWords - 1) / kEmitWords);
      segs.push_back(e);
    }
    if (segs.empty()) continue;
    EmitTable t;
    t.nsegs = (int)segs.size();
    if (segs.size() <= (size_t)kInlineSegs) {
      std::copy(segs.begin(), segs.end(), t.inl);
      t.segs = nullptr;
    } else {
      WS_TRY(params_upload(h, segs, &t.segs, st));
    }
    launch_emit(c, h->enc, t, blocks, dout, nl, st);
    ++h->launches;
  }
  if (only == -1 || only == kLongCls) {
    for (size_t i = 0; i < h->buckets.size(); ++i) {
      const Bucket& b = h->buckets[i];
      if (!b.is_long || !b.count || !pick[i]) continue;
      const uint32_t* order = h->sorted ? h->rank.as<uint32_t>() + b.long_off : nullptr;
      const uint2* words = h->longgrp.as<uint2>() + (h->sorted ? 0 : b.long_off);
      launch_emit_long(h->text.as<uint8_t>(), words, order, b.count, b.len, dout + off[i], nl, st);
      ++h->launches;
    }
  }
  ph.end();
  WS_TRY(check_launch("emit"));
  if (offsets) *offsets = off;
  return WS_OK;
}

uint64_t emit_size(ws_handle* h, bool lines) {
  uint64_t run = 0;
  for (auto& b : h->buckets) run += b.count * (b.len + (lines ? 1 : 0));
  return run;
}

int emit_to_host(ws_handle* h, bool lines, uint8_t* out, uint64_t cap, uint64_t* written) {
  if (!h->ingested) return fail(WS_ERR_STATE, "emit before ingest");
  if (h->payload_only)
    return fail(WS_ERR_STATE, "the handle holds the payload of a fused sort, not sorted keys: ws_sort first");
  const uint64_t size = emit_size(h, lines);
  if (written) *written = size;
  if (!out && cap == 0) return WS_OK;  // size query
  if (cap < size) return fail(WS_ERR_ARG, "output buffer too small");
  if (!size) return WS_OK;
  if (!out) return fail(WS_ERR_ARG, "null output buffer");
  WS_CUDA(h->out.ensure(size + 64));
  WS_TRY(emit_device(h, h->out.as<uint8_t>(), lines, nullptr));
  {
    Phase ph(h, "d2h_out", (double)size, 1);
    WS_CUDA(cudaMemcpyAsync(out, h->out.p, size, cudaMemcpyDeviceToHost, h->st));
  }
  WS_CUDA(cudaStreamSynchronize(h->st));
  return WS_OK;
}

// ----------------------------------------------------------------------------
// rows / blocks ingest (the _bubble_rows drop-in)

int ingest_blocks_impl(ws_handle* h, int32_t nblocks, const uint8_t* const* rows,
                       const int64_t* counts, const int32_t* widths, bool allow_dup,
                       std::vector<int>* block_of_bucket) {
  if (nblocks < 0) return fail(WS_ERR_ARG, "negative block count");
  h->ingested = h->sorted = h->have_stats = h->payload_only = false;
  h->have_tokens = false;
  h->unordered = false;
  h->text_valid = false;
  h->enc = kEncRaw8;
  h->buckets.clear();
  std::vector<int> order(nblocks);
  for (int i = 0; i < nblocks; ++i) {
    order[i] = i;
    if (counts[i] < 0 || widths[i] < 1) return fail(WS_ERR_ARG, "bad block shape");
    if (counts[i] && !rows[i]) return fail(WS_ERR_ARG, "null rows");
  }
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return widths[a] < widths[b]; });
  if (!allow_dup)
    for (int i = 1; i < nblocks; ++i)
      if (widths[order[i]] == widths[order[i - 1]]) return fail(WS_ERR_ARG, "repeated width");
  // byte offsets of each block in the device rows buffer (16-byte aligned)
  std::vector<uint64_t> boff(nblocks);
  uint64_t total = 0;
  for (int k = 0; k < nblocks; ++k) {
    int i = order[k];
    boff[i] = total;
    total += (uint64_t)counts[i] * widths[i];
    total = (total + 15) & ~15ull;
  }
  if (total >= (1ull << 32)) return fail(WS_ERR_ARG, "rows must total less than 4 GiB");
  WS_CUDA(h->text.ensure(total + kTextPad));
  h->n_text = total;
  {
    Phase ph(h, "h2d_rows", (double)total, 1);
    for (int i = 0; i < nblocks; ++i)
      if (counts[i])
        WS_CUDA(cudaMemcpyAsync(h->text.as<uint8_t>() + boff[i], rows[i],
                                (size_t)counts[i] * widths[i], cudaMemcpyHostToDevice, h->st));
  }
  // plan: packed buckets (width <= 32) laid out per lane class, long groups
  uint64_t elems[kClasses + 1] = {0};
  uint64_t idx_run = 0, long_run = 0;
  std::vector<int> bob;
  for (int k = 0; k < nblocks; ++k) {
    int i = order[k];
    if (!counts[i]) continue;
    Bucket bk;
    bk.len = (uint32_t)widths[i];
    bk.count = (uint64_t)counts[i];
    if (widths[i] <= kMaxPackedLen) {
      bk.lanes = lanes_for_len_enc(widths[i], kEncRaw8);
      bk.elem_off = elems[bk.lanes];
      elems[bk.lanes] += bk.count;
      bk.idx_off = idx_run;
      idx_run += bk.count;
    } else {
      bk.is_long = true;
      bk.long_off = long_run;
      long_run += bk.count;
    }
    h->buckets.push_back(bk);
    bob.push_back(i);
  }
  uint64_t run = 0;  // bytes
  for (int c = 0; c <= kClasses; ++c) {
    h->class_base[c] = run;
    h->class_elems[c] = elems[c];
    run += elems[c] * key_bytes(c);
    run = (run + 15) & ~15ull;
  }
  h->idx_total = idx_run;
  WS_CUDA(h->keys[0].ensure(run + 64));
  WS_CUDA(h->keys[1].ensure(run + 64));
  h->n_long = long_run;
  if (long_run) {
    WS_CUDA(h->longgrp.ensure(long_run * sizeof(uint2)));
    WS_CUDA(h->lkeys[0].ensure(long_run * 8 + 64));
    WS_CUDA(h->lkeys[1].ensure(long_run * 8 + 64));
    WS_CUDA(h->lidx[0].ensure(long_run * 4 + 64));
    WS_CUDA(h->lidx[1].ensure(long_run * 4 + 64));
  }
  for (size_t k = 0; k < h->buckets.size(); ++k) {
    const Bucket& b = h->buckets[k];
    const int i = bob[k];
    if (!b.is_long) {
      launch_pack_rows(h->text.as<uint8_t>() + boff[i], b.count, b.len,
                       class_keys(h, 0, b.lanes, b.elem_off), h->st);
    } else {
      launch_rows_longlist(boff[i], b.count, b.len, h->longgrp.as<uint2>() + b.long_off, h->st);
    }
    ++h->launches;
  }
  WS_TRY(check_launch("pack_rows"));
  if (block_of_bucket) *block_of_bucket = bob;
  return finish_ingest(h);
}

int ingest_words_impl(ws_handle* h, const uint8_t* concat, const uint32_t* lens, uint64_t nwords) {
  h->ingested = h->sorted = h->have_stats = h->payload_only = false;
  h->have_tokens = false;
  h->unordered = false;
  h->text_valid = false;
  h->enc = kEncRaw8;  // word lists may hold any byte values
  h->buckets.clear();
  if (nwords && !lens) return fail(WS_ERR_ARG, "null lens");
  std::vector<uint64_t> starts(nwords);
  uint64_t total = 0;
  for (uint64_t i = 0; i < nwords; ++i) {
    if (lens[i] == 0) return fail(WS_ERR_ARG, "empty word");
    starts[i] = total;
    total += lens[i];
  }
  if (total >= (1ull << 32) - kTextPad) return fail(WS_ERR_ARG, "words must total < 4 GiB");
  if (total && !concat) return fail(WS_ERR_ARG, "null word bytes");
  WS_CUDA(h->text.ensure(total + kTextPad));
  WS_CUDA(h->starts.ensure(std::max<uint64_t>(nwords, 1) * 8));
  WS_CUDA(h->lens.ensure(std::max<uint64_t>(nwords, 1) * 4));
  h->n_text = total;
  {
    Phase ph(h, "h2d_words", (double)total + 12.0 * nwords, 1);
    if (total) WS_CUDA(cudaMemcpyAsync(h->text.p, concat, total, cudaMemcpyHostToDevice, h->st));
    if (nwords) {
      WS_CUDA(cudaMemcpyAsync(h->starts.p, starts.data(), nwords * 8, cudaMemcpyHostToDevice,
                              h->st));
      WS_CUDA(cudaMemcpyAsync(h->lens.p, lens, nwords * 4, cudaMemcpyHostToDevice, h->st));
    }
  }
  constexpr uint32_t kWpw = 1024;
  const uint32_t nwarps = (uint32_t)((nwords + kWpw - 1) / kWpw);
  const size_t hb = (size_t)kNumBins * std::max<uint32_t>(nwarps, 1) * 4;
  WS_CUDA(h->hist.ensure(hb));
  WS_CUDA(h->off.ensure(hb));
  WS_CUDA(h->totals.ensure(kHistRows * 4));
  WS_CUDA(h->pin_small.ensure(1 << 16));
  uint32_t* tot_host = static_cast<uint32_t*>(h->pin_small.p);
  memset(tot_host, 0, kHistRows * 4);
  if (nwarps) {
    WS_CUDA(cudaMemsetAsync(h->hist.p, 0, hb, h->st));
    launch_words_hist(h->lens.as<uint32_t>(), nwords, kWpw, h->hist.as<uint32_t>(), nwarps, h->st);
    launch_scan(h->hist.as<uint32_t>(), h->off.as<uint32_t>(), h->totals.as<uint32_t>(), nwarps,
                kNumBins, h->st);
    h->launches += 2;
    WS_CUDA(cudaMemcpyAsync(tot_host, h->totals.p, kNumBins * 4, cudaMemcpyDeviceToHost, h->st));
    WS_CUDA(cudaStreamSynchronize(h->st));
  }
  uint64_t counts[kNumBins];
  for (int b = 0; b < kNumBins; ++b) counts[b] = tot_host[b];
  WS_TRY(plan_packed(h, counts));
  const uint64_t m = counts[kLongBin];
  WS_CUDA(h->longlist.ensure(std::max<uint64_t>(m, 1) * sizeof(uint2)));
  ScatterParams p;
  fill_scatter_params(h, p);
  launch_words_scatter(h->text.as<uint8_t>(), h->starts.as<uint64_t>(), h->lens.as<uint32_t>(),
                       nwords, kWpw, h->off.as<uint32_t>(), nwarps, p, h->st);
  ++h->launches;
  WS_TRY(check_launch("words_scatter"));
  WS_TRY(group_long_words(h, m));
  return finish_ingest(h);
}

int thread_handle(ws_handle** out);

}  // namespace

// ============================================================================
// C ABI

extern "C" {

int ws_version(void) { return 10000; }

const char* ws_last_error(void) { return g_err.c_str(); }

int ws_device_count(int32_t* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  if (count) *count = n;
  return WS_OK;
}

int ws_create(ws_handle** out, int32_t device) {
  if (!out) return fail(WS_ERR_ARG, "null out");
  *out = nullptr;
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return fail(WS_ERR_CUDA, std::string("no CUDA device available: ") +
                                 (e != cudaSuccess ? cudaGetErrorString(e) : "0 devices"));
  }
  if (device < 0 || device >= n) return fail(WS_ERR_ARG, "bad device index");
  WS_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  WS_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10) {
    return fail(WS_ERR_CUDA, std::string("libwsort_b200 is built for sm_100a; device is ") +
                                 prop.name);
  }
  static std::mutex mu;
  static uint64_t attr_done = 0;
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!(attr_done & (1ull << device))) {
      set_sort_attributes();
      set_ingest_attributes();
      WS_CUDA(cudaGetLastError());
      attr_done |= 1ull << device;
    }
  }
  ws_handle* h = new ws_handle();
  h->device = device;
  const char* ser = getenv("WSORT_SERIAL");
  h->serial = h->serial_env = ser && ser[0] == '1';
  // Priorities: class 0's radix chain (four dependent passes of small
  // kernels) is the longest path, so its stream (and every emit / copy
  // stream) outranks the multi-lane classes' sort streams.
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  e = cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking);
  // the one-word classes (0, 1) hold most keys and sort last
  int cprio[kClasses + 1];
  for (int c = 0; c <= kClasses; ++c) cprio[c] = c == 0 ? prio_hi : prio_lo;
  if (const char* cp = getenv("WSORT_CLASS_PRIO")) {  // experiment: per-class priorities
    for (int c = 0; c <= kClasses && *cp; ++c) {
      char* endp = nullptr;
      const long v = strtol(cp, &endp, 10);
      if (endp == cp) break;
      cprio[c] = std::min(prio_lo, std::max(prio_hi, (int)v));
      cp = *endp == ',' ? endp + 1 : endp;
    }
  }
  for (int c = 0; c <= kClasses && e == cudaSuccess; ++c)
    e = cudaStreamCreateWithPriority(&h->cs[c], cudaStreamNonBlocking, cprio[c]);
  if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&h->hs, cudaStreamNonBlocking, prio_hi);
  for (int c = 0; c <= kClasses && e == cudaSuccess; ++c) {
    e = cudaStreamCreateWithPriority(&h->es[c], cudaStreamNonBlocking, prio_hi);
    if (e == cudaSuccess)
      e = cudaStreamCreateWithPriority(&h->ds[c], cudaStreamNonBlocking, prio_hi);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_zero, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_dd, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_probe, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_lo, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_hi, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_chain, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming);
  for (int c = 0; c <= kClasses && e == cudaSuccess; ++c)
    e = cudaEventCreateWithFlags(&h->ev_join[c], cudaEventDisableTiming);
  if (e != cudaSuccess) {
    ws_destroy(h);
    return fail_cuda(e, "cudaStreamCreate", __LINE__);
  }
  static std::once_flag exit_once;  // registered after the CUDA runtime's own handler: runs before it
  std::call_once(exit_once, [] { atexit([] { g_exiting.store(true, std::memory_order_release); }); });
  *out = h;
  return WS_OK;
}

void ws_destroy(ws_handle* h) {
  if (!h) return;
  // Process exit: once the atexit handlers run, the CUDA runtime may already be
  // torn down (its own handler); a handle destroyed that late (a thread-local
  // handle, an object finalised by the host language at exit) is left to the OS.
  if (g_exiting.load(std::memory_order_acquire)) return;
  for (ws_handle* p : h->peers) ws_destroy(p);
  h->peers.clear();
  cudaSetDevice(h->device);
  if (h->st) cudaStreamSynchronize(h->st);
  if (h->hs) cudaStreamSynchronize(h->hs);
  if (h->zs) cudaStreamSynchronize(h->zs);
  if (h->xs) cudaStreamSynchronize(h->xs);
  for (int c = 0; c <= kClasses; ++c) {
    if (h->cs[c]) cudaStreamSynchronize(h->cs[c]);
    if (h->es[c]) cudaStreamSynchronize(h->es[c]);
    if (h->ds[c]) cudaStreamSynchronize(h->ds[c]);
  }
  DevBuf* bufs[] = {&h->text, &h->starts, &h->lens, &h->hist, &h->off, &h->totals,
                    &h->keys[0], &h->keys[1], &h->idx[0], &h->idx[1], &h->longlist,
                    &h->longgrp, &h->rank, &h->rank_tmp, &h->lkeys[0], &h->lkeys[1],
                    &h->lidx[0], &h->lidx[1], &h->tokens, &h->stat_inv, &h->stat_k,
                    &h->stat_k_dummy, &h->out, &h->params, &h->splits[0], &h->splits[1],
                    &h->splits[2], &h->splits[3], &h->splits[4], &h->splits[5],
                    &h->keys_cap, &h->status, &h->ticket, &h->overflow, &h->fill,
                    &h->run_at, &h->run_cnt, &h->run_off, &h->longlist2,
                    &h->rcounts[0], &h->rcounts[1], &h->rtotals[0], &h->rtotals[1], &h->rstatus[0], &h->rstatus[1],
                    &h->ss_split[1], &h->ss_split[2], &h->ss_split[3], &h->ss_split[4],
                    &h->ss_slots[1], &h->ss_slots[2], &h->ss_slots[3], &h->ss_slots[4],
                    &h->ss_ids[1], &h->ss_ids[2], &h->ss_ids[3], &h->ss_ids[4],
                    &h->tiny_flag, &h->tiny_prof, &h->first_sep, &h->ss_scratch,
                    &h->dd_pool, &h->dd_keys, &h->dd_aux, &h->dd_ts, &h->dd_plan};
  for (DevBuf* b : bufs) b->release();
  h->pin_params.release();
  h->pin_small.release();
  for (auto& p : h->phases) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : h->event_pool) cudaEventDestroy(e);
  for (auto e : h->sync_events) cudaEventDestroy(e);
  for (int c = 0; c <= kClasses; ++c) {
    if (h->es[c]) cudaStreamDestroy(h->es[c]);
    if (h->ds[c]) cudaStreamDestroy(h->ds[c]);
    if (h->cs[c]) cudaStreamDestroy(h->cs[c]);
    if (h->ev_join[c]) cudaEventDestroy(h->ev_join[c]);
  }
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_zero) cudaEventDestroy(h->ev_zero);
  if (h->ev_dd) cudaEventDestroy(h->ev_dd);
  if (h->ev_probe) cudaEventDestroy(h->ev_probe);
  if (h->ev_lo) cudaEventDestroy(h->ev_lo);
  if (h->ev_hi) cudaEventDestroy(h->ev_hi);
  if (h->ev_chain) cudaEventDestroy(h->ev_chain);
  if (h->zs) cudaStreamDestroy(h->zs);
  if (h->xs) cudaStreamDestroy(h->xs);
  if (h->hs) cudaStreamDestroy(h->hs);
  if (h->st) cudaStreamDestroy(h->st);
  delete h;
}

int ws_ingest_text(ws_handle* h, const uint8_t* text, uint64_t n, int32_t flags) {
  WS_TRY(begin_call(h));
  return ingest_text_impl(h, text, n, flags);
}

int ws_ingest_words(ws_handle* h, const uint8_t* concat, const uint32_t* lens, uint64_t nwords) {
  WS_TRY(begin_call(h));
  return ingest_words_impl(h, concat, lens, nwords);
}

int ws_ingest_blocks(ws_handle* h, int32_t nblocks, const uint8_t* const* rows,
                     const int64_t* counts, const int32_t* widths) {
  WS_TRY(begin_call(h));
  if (nblocks && (!rows || !counts || !widths)) return fail(WS_ERR_ARG, "null block arrays");
  WS_TRY(ingest_blocks_impl(h, nblocks, rows, counts, widths, false, nullptr));
  WS_CUDA(cudaStreamSynchronize(h->st));
  return WS_OK;
}

int ws_buckets(ws_handle* h, int64_t* lengths, int64_t* counts, int32_t cap, int32_t* nbuckets,
               uint64_t* words) {
  if (!h) return fail(WS_ERR_ARG, "null handle");
  if (!h->ingested) return fail(WS_ERR_STATE, "ws_buckets before ingest");
  const int nb = (int)h->buckets.size();
  if (nbuckets) *nbuckets = nb;
  if (words) *words = h->words;
  for (int i = 0; i < nb && i < cap; ++i) {
    if (lengths) lengths[i] = h->buckets[i].len;
    if (counts) counts[i] = (int64_t)h->buckets[i].count;
  }
  return WS_OK;
}

int ws_tokens(ws_handle* h, uint32_t* starts_lens, uint64_t cap_words, uint64_t* nwords) {
  WS_TRY(begin_call(h));
  if (!h->have_tokens) return fail(WS_ERR_STATE, "ingest without WS_INGEST_KEEP_TOKENS");
  if (nwords) *nwords = h->words;
  if (cap_words < h->words) return fail(WS_ERR_ARG, "token buffer too small");
  if (h->words) {
    if (!starts_lens) return fail(WS_ERR_ARG, "null token buffer");
    WS_CUDA(cudaMemcpyAsync(starts_lens, h->tokens.p, h->words * 8, cudaMemcpyDeviceToHost, h->st));
  }
  WS_CUDA(cudaStreamSynchronize(h->st));
  return WS_OK;
}

int ws_sort(ws_handle* h, int32_t want_stats) {
  WS_TRY(begin_call(h));
  WS_TRY(sort_impl(h, want_stats != 0));
  WS_CUDA(cudaStreamSynchronize(h->st));
  return WS_OK;
}

int ws_stats_closed_form(int64_t n, int64_t inversions, int64_t kmax, int32_t naive,
                         int64_t stats[3]) {
  if (!stats) return fail(WS_ERR_ARG, "null stats");
  stats[0] = stats[1] = stats[2] = 0;
  if (n < 2) return WS_OK;
  if (inversions < 0 || kmax < 0 || kmax > n - 1) return fail(WS_ERR_ARG, "bad stats input");
  if (naive) {
    stats[0] = n * (n - 1) / 2;
    stats[1] = inversions;
    stats[2] = n - 1;
  } else {
    const int64_t P = std::min(kmax + 1, n - 1);
    stats[0] = P * (n - 1) - P * (P - 1) / 2;
    stats[1] = inversions;
    stats[2] = P;
  }
  return WS_OK;
}

int ws_bucket_stats(ws_handle* h, int32_t naive, int64_t* stats, int32_t cap) {
  if (!h) return fail(WS_ERR_ARG, "null handle");
  if (!h->have_stats) return fail(WS_ERR_STATE, "ws_bucket_stats needs ws_sort(h, 1)");
  for (int i = 0; i < (int)h->buckets.size() && i < cap; ++i) {
    const Bucket& b = h->buckets[i];
    WS_TRY(ws_stats_closed_form((int64_t)b.count, b.inv, b.kmax, naive, stats + 3 * i));
  }
  return WS_OK;
}

int ws_permutation(ws_handle* h, int32_t bucket, uint32_t* perm, uint64_t cap) {
  WS_TRY(begin_call(h));
  if (!h->have_stats) return fail(WS_ERR_STATE, "ws_permutation needs ws_sort(h, 1)");
  if (bucket < 0 || bucket >= (int)h->buckets.size()) return fail(WS_ERR_ARG, "bad bucket");
  const Bucket& b = h->buckets[bucket];
  if (cap < b.count) return fail(WS_ERR_ARG, "perm buffer too small");
  if (!b.count) return WS_OK;
  if (!b.is_long) {
    WS_CUDA(cudaMemcpyAsync(perm, h->idx[b.final_buf].as<uint32_t>() + b.idx_off, b.count * 4,
                            cudaMemcpyDeviceToHost, h->st));
    WS_CUDA(cudaStreamSynchronize(h->st));
  } else {
    WS_CUDA(cudaMemcpyAsync(perm, h->rank.as<uint32_t>() + b.long_off, b.count * 4,
                            cudaMemcpyDeviceToHost, h->st));
    WS_CUDA(cudaStreamSynchronize(h->st));
    for (uint64_t j = 0; j < b.count; ++j) perm[j] -= (uint32_t)b.long_off;
  }
  return WS_OK;
}

int ws_emit_lines(ws_handle* h, uint8_t* out, uint64_t cap, uint64_t* written) {
  WS_TRY(begin_call(h));
  return emit_to_host(h, true, out, cap, written);
}

int ws_emit_rows(ws_handle* h, uint8_t* out, uint64_t cap, uint64_t* written) {
  WS_TRY(begin_call(h));
  return emit_to_host(h, false, out, cap, written);
}

namespace {

// ws_sort_text body. `gate` (batch mode) serialises the host->device copy +
// ingest of concurrent slots, so their PCIe transfers are staggered: one
// corpus uploads while the previous ones sort and download.
// Texts up to this size try tiny_sort_kernel first (WSORT_NO_TINY=1: never).
constexpr uint64_t kTinyMaxText = 512 << 10;
bool tiny_wanted(ws_handle* h, uint64_t n) {
  static const bool off = env_on("WSORT_NO_TINY");
  return !off && n > 0 && n <= kTinyMaxText && h->enc == kEncAlnum6;
}

// A tiny sort left the whole payload in `out`: the handle's state is that of a
// fused sort (payload written, keys not sorted).
void finish_tiny(ws_handle* h) {
  h->sorted = true;
  h->payload_only = true;
}

int sort_text_impl(ws_handle* h, const uint8_t* text, uint64_t n, uint8_t* out, uint64_t cap,
                   uint64_t* written, std::mutex* gate) {
  static const bool trace = getenv("WSORT_TRACE") && getenv("WSORT_TRACE")[0] == '1';
  const double t_begin = trace ? trace_ms() : 0;
  h->early_req = early_hist_wanted();
  h->enc = kEncAlnum6;
  h->tiny_req = tiny_wanted(h, n);
  h->dd_req = dedupe_wanted(n);
  if (h->tiny_req) WS_CUDA(h->out.ensure(n + 64));
  const int irc = ingest_text_impl(h, text, n, WS_INGEST_UNORDERED, gate);  // ends with a sync
  h->early_req = h->tiny_req = h->dd_req = false;
  WS_TRY(irc);
  const double t_ingested = trace ? trace_ms() : 0;
  params_reset(h);  // the ingest synchronised: staging space is free again
  const uint64_t size = emit_size(h, true);
  if (written) *written = size;
  if (cap < size) return fail(WS_ERR_ARG, "output buffer too small");
  if (!size) return WS_OK;
  if (!out) return fail(WS_ERR_ARG, "null output buffer");
  if (h->tiny_done) {  // the payload is on the device already
    finish_tiny(h);
    {
      Phase ph(h, "d2h_out", (double)size, 1);
      WS_CUDA(cudaMemcpyAsync(out, h->out.p, size, cudaMemcpyDeviceToHost, h->st));
    }
    WS_CUDA(cudaStreamSynchronize(h->st));
    return WS_OK;
  }
  WS_CUDA(h->out.ensure(size + 64));
  FusedEmit fe;
  fe.dout = h->out.as<uint8_t>();
  fe.host = out;
  fe.off = emit_offsets(h, true);
  static const char* pc = getenv("WSORT_D2H_PER_CLASS");
  fe.per_class = pc ? pc[0] == '1' : false;
  WS_TRY(sort_impl(h, false, &fe));  // sort + per-class emit + D2H, overlapped
  const double t_enqueued = trace ? trace_ms() : 0;
  WS_CUDA(cudaStreamSynchronize(h->st));  // joins every class stream
  if (trace)
    fprintf(stderr, "wsort-trace handle=%p begin=%.3f ingested=%.3f enqueued=%.3f done=%.3f\n",
            (void*)h, t_begin, t_ingested, t_enqueued, trace_ms());
  return WS_OK;
}

}  // namespace

int ws_sort_text(ws_handle* h, const uint8_t* text, uint64_t n, uint8_t* out, uint64_t cap,
                 uint64_t* written) {
  WS_TRY(begin_call(h));
  return sort_text_impl(h, text, n, out, cap, written, nullptr);
}

int ws_sort_texts(ws_handle* h, int32_t count, const uint8_t* const* texts, const uint64_t* sizes,
                  uint8_t* const* outs, const uint64_t* caps, uint64_t* written,
                  int32_t inflight) {
  WS_TRY(begin_call(h));
  if (count < 0) return fail(WS_ERR_ARG, "negative count");
  if (count == 0) return WS_OK;
  if (!texts || !sizes || !outs || !caps || !written) return fail(WS_ERR_ARG, "null batch arrays");
  const int slots = std::max(1, std::min<int>(inflight <= 0 ? 3 : inflight, std::min(count, 4)));
  while ((int)h->peers.size() < slots - 1) {
    ws_handle* p = nullptr;
    WS_TRY(ws_create(&p, h->device));
    h->peers.push_back(p);
  }
  for (int32_t i = 0; i < count; ++i) written[i] = 0;
  std::mutex gate;
  std::vector<int> rc(slots, WS_OK);
  std::vector<std::string> msg(slots);
  auto worker = [&](int slot) {
    ws_handle* hh = slot == 0 ? h : h->peers[slot - 1];
    int r = begin_call(hh);
    for (int32_t i = slot; i < count && r == WS_OK; i += slots)
      r = sort_text_impl(hh, texts[i], sizes[i], outs[i], caps[i], written + i, &gate);
    rc[slot] = r;
    if (r != WS_OK) msg[slot] = g_err;
  };
  std::vector<std::thread> pool;
  for (int s = 1; s < slots; ++s) pool.emplace_back(worker, s);
  worker(0);
  for (auto& t : pool) t.join();
  for (int s = 0; s < slots; ++s)
    if (rc[s] != WS_OK) return fail(rc[s], msg[s]);
  return WS_OK;
}

int ws_sort_resident(ws_handle* h, uint64_t n, uint64_t* written) {
  WS_TRY(begin_call(h));
  static const bool trace = env_on("WSORT_TRACE") || (getenv("WSORT_TRACE") && getenv("WSORT_TRACE")[0] == '2');
  const double t_begin = trace ? trace_ms() : 0;
  tmark("begin");
  h->early_req = early_hist_wanted();
  h->enc = kEncAlnum6;
  h->tiny_req = tiny_wanted(h, n);
  h->dd_req = dedupe_wanted(n);
  if (h->tiny_req) WS_CUDA(h->out.ensure(n + 64));
  const int irc = ingest_text_impl(h, nullptr, n, WS_INGEST_RESIDENT | WS_INGEST_UNORDERED);
  h->early_req = h->tiny_req = h->dd_req = false;
  WS_TRY(irc);
  const double t_ingested = trace ? trace_ms() : 0;
  tmark("ingest_ret");
  params_reset(h);
  const uint64_t size = emit_size(h, true);
  if (h->tiny_done) {  // the payload is in `out` already
    finish_tiny(h);
    h->out_size = size;
    if (written) *written = size;
    return WS_OK;
  }
  WS_CUDA(h->out.ensure(size + 64));
  FusedEmit fe;
  fe.dout = h->out.as<uint8_t>();
  fe.host = nullptr;
  fe.off = emit_offsets(h, true);
  tmark("offsets");
  WS_TRY(sort_impl(h, false, &fe));  // each class emits as soon as it is sorted
  const double t_enqueued = trace ? trace_ms() : 0;
  h->out_size = size;
  if (written) *written = size;
  WS_CUDA(cudaStreamSynchronize(h->st));
  if (trace)
    fprintf(stderr, "wsort-trace resident ingest_host=%.3f enqueue_host=%.3f wait=%.3f ms\n",
            t_ingested - t_begin, t_enqueued - t_ingested, trace_ms() - t_enqueued);
  if (!g_marks.empty()) {
    fprintf(stderr, "wsort-marks");
    for (auto& m : g_marks) fprintf(stderr, " %s=%.1f", m.first, (m.second - t_begin) * 1e3);
    fprintf(stderr, " (us from call start)\n");
    g_marks.clear();
  }
  return WS_OK;
}

int ws_output_device(ws_handle* h, void** dptr, uint64_t* size) {
  if (!h || !dptr) return fail(WS_ERR_ARG, "null argument");
  *dptr = h->out.p;
  if (size) *size = h->out_size;
  return WS_OK;
}

int ws_sort_rows(uint8_t* rows, int64_t n, int32_t width, int32_t naive, int64_t stats[3]) {
  int64_t counts[1] = {n};
  int32_t widths[1] = {width};
  uint8_t* r[1] = {rows};
  return ws_sort_blocks(1, r, counts, widths, naive, stats, nullptr);
}

int ws_sort_blocks(int32_t nblocks, uint8_t* const* rows, const int64_t* counts,
                   const int32_t* widths, int32_t naive, int64_t* stats, uint32_t* const* perms) {
  g_err.clear();
  if (nblocks < 0) return fail(WS_ERR_ARG, "negative block count");
  if (nblocks && (!rows || !counts || !widths || !stats)) return fail(WS_ERR_ARG, "null arrays");
  // trivial blocks (n < 2 or width 0) need no device work: zero stats, identity perm
  std::vector<int> work;
  for (int i = 0; i < nblocks; ++i) {
    if (counts[i] < 0 || widths[i] < 0) return fail(WS_ERR_ARG, "bad block shape");
    stats[3 * i] = stats[3 * i + 1] = stats[3 * i + 2] = 0;
    if (counts[i] >= 2 && widths[i] > 0) {
      work.push_back(i);
    } else if (counts[i] >= 2) {
      // width 0: all rows equal; the reference still runs its full schedule
      WS_TRY(ws_stats_closed_form(counts[i], 0, 0, naive, stats + 3 * i));
    }
    if (perms && perms[i] && !(counts[i] >= 2 && widths[i] > 0))
      for (int64_t j = 0; j < counts[i]; ++j) perms[i][j] = (uint32_t)j;
  }
  if (work.empty()) return WS_OK;
  ws_handle* h;
  WS_TRY(thread_handle(&h));
  WS_TRY(begin_call(h));
  std::vector<const uint8_t*> r;
  std::vector<int64_t> c;
  std::vector<int32_t> w;
  for (int i : work) {
    r.push_back(rows[i]);
    c.push_back(counts[i]);
    w.push_back(widths[i]);
  }
  std::vector<int> bob;
  WS_TRY(ingest_blocks_impl(h, (int)work.size(), r.data(), c.data(), w.data(), true, &bob));
  WS_TRY(sort_impl(h, true));
  // unpack sorted rows back into each block's device region, then to host
  std::vector<uint64_t> offs;
  WS_CUDA(h->out.ensure(emit_size(h, false) + 64));
  WS_TRY(emit_device(h, h->out.as<uint8_t>(), false, &offs));
  for (size_t k = 0; k < h->buckets.size(); ++k) {
    const Bucket& b = h->buckets[k];
    const int i = work[bob[k]];
    WS_CUDA(cudaMemcpyAsync(rows[i], h->out.as<uint8_t>() + offs[k], b.count * b.len,
                            cudaMemcpyDeviceToHost, h->st));
    WS_TRY(ws_stats_closed_form((int64_t)b.count, b.inv, b.kmax, naive, stats + 3 * i));
  }
  WS_CUDA(cudaStreamSynchronize(h->st));
  if (perms) {
    for (size_t k = 0; k < h->buckets.size(); ++k) {
      const int i = work[bob[k]];
      if (perms[i]) WS_TRY(ws_permutation(h, (int)k, perms[i], h->buckets[k].count));
    }
  }
  return WS_OK;
}

int ws_set_profiling(ws_handle* h, int32_t on) {
  if (!h) return fail(WS_ERR_ARG, "null handle");
  h->prof = on != 0;
  // 2: also run every kernel on the main stream, so each event pair brackets
  // its own launch alone (serialised, like an ncu launch list)
  h->serial = on == 2 ? true : h->serial_env;
  return WS_OK;
}

int ws_profile(ws_handle* h, ws_phase* out, int32_t cap, int32_t* n) {
  if (!h) return fail(WS_ERR_ARG, "null handle");
  WS_CUDA(cudaSetDevice(h->device));
  WS_CUDA(cudaStreamSynchronize(h->st));
  if (n) *n = (int32_t)h->phases.size();
  for (int i = 0; i < (int)h->phases.size() && i < cap; ++i) {
    const PhaseRec& p = h->phases[i];
    float ms = 0;
    WS_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
    memset(out[i].name, 0, sizeof out[i].name);
    strncpy(out[i].name, p.name.c_str(), sizeof out[i].name - 1);
    out[i].launches = p.launches;
    out[i].kind = p.kind;
    out[i].ms = ms;
    out[i].bytes = p.bytes;
    float t0 = 0;
    if (i > 0) WS_CUDA(cudaEventElapsedTime(&t0, h->phases[0].a, p.a));
    out[i].start_ms = t0;
  }
  return WS_OK;
}

int ws_profile_reset(ws_handle* h) {
  if (!h) return fail(WS_ERR_ARG, "null handle");
  for (auto& p : h->phases) {
    h->event_pool.push_back(p.a);
    h->event_pool.push_back(p.b);
  }
  h->phases.clear();
  return WS_OK;
}

int ws_debug_checks(uint64_t* failures, int32_t* first_unit, int32_t* first_line) {
  if (!failures) return fail(WS_ERR_ARG, "null argument");
  if (WS_CHECKED && env_on("WSORT_CHECK_SELFTEST")) launch_check_selftest(nullptr);
  WS_CUDA(cudaDeviceSynchronize());
  int (*readers[])(unsigned int*, unsigned int*) = {check_reader_ingest, check_reader_sort,
                                                   check_reader_radix, check_reader_emit,
                                                   check_reader_dedupe};
  *failures = 0;
  if (first_unit) *first_unit = -1;
  if (first_line) *first_line = 0;
  for (int u = 0; u < 5; ++u) {
    unsigned int f = 0, line = 0;
    const int e = readers[u](&f, &line);
    if (e) return fail_cuda((cudaError_t)e, "ws_debug_checks", __LINE__);
    if (f && *failures == 0) {
      if (first_unit) *first_unit = u;
      if (first_line) *first_line = (int32_t)line;
    }
    *failures += f;
  }
  return WS_OK;
}

int ws_checked_build(void) { return WS_CHECKED; }

int ws_launch_count(ws_handle* h, uint64_t* launches) {
  if (!h || !launches) return fail(WS_ERR_ARG, "null argument");
  *launches = h->launches;
  for (ws_handle* p : h->peers) *launches += p->launches;  // ws_sort_texts slots
  return WS_OK;
}

int ws_counted_classes(ws_handle* h, int32_t* mask) {
  if (!h || !mask) return fail(WS_ERR_ARG, "null argument");
  *mask = h->dd_used;
  return WS_OK;
}

int ws_stream(ws_handle* h, void** stream) {
  if (!h || !stream) return fail(WS_ERR_ARG, "null argument");
  *stream = (void*)h->st;
  return WS_OK;
}

int ws_host_alloc(uint64_t bytes, void** out) {
  if (!out) return fail(WS_ERR_ARG, "null out");
  *out = nullptr;
  WS_CUDA(cudaMallocHost(out, std::max<uint64_t>(bytes, 1)));
  return WS_OK;
}

int ws_host_free(void* p) {
  if (g_exiting.load(std::memory_order_acquire)) return WS_OK;  // see ws_destroy
  if (p) WS_CUDA(cudaFreeHost(p));
  return WS_OK;
}

}  // extern "C"

namespace {

struct ThreadHandle {
  ws_handle* h = nullptr;
  ~ThreadHandle() {
    if (h) ws_destroy(h);
  }
};

int thread_handle(ws_handle** out) {
  thread_local ThreadHandle th;
  if (!th.h) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
      cudaGetLastError();
      dev = 0;
    }
    WS_TRY(ws_create(&th.h, dev));
  }
  *out = th.h;
  return WS_OK;
}

}  // namespace
