// Payload-only bucket sort: LSD radix over the packed keys of a lane class.
//
// The reference sorts every length bucket with bubble sort (engine.py:89-114);
// the sorted bucket is all that `wordsort sort` emits (cli.py:92-97). When no
// statistics are requested (ws_sort(h, 0), ws_sort_text, ws_sort_resident),
// equal keys are identical words, so any correct sort yields the reference's
// bytes. This file sorts one-word keys (lane class 0: uint32, class 1: one
// uint64) by stable LSD passes over 8-bit digits of the bits a bucket uses
// (6 per character for text keys, 8 per byte otherwise), so a 5-character
// bucket needs 4 passes where the merge sort needs log2(n / tile) + 1.
//
// Per pass and segment (bucket), with T-key tiles:
//   upsweep   : per-tile digit histogram -> counts[d][tile], digit totals
//   scan      : one warp per (segment, digit) row: exclusive scan over tiles
//               plus the segment's digit prefix -> global output offsets
//   downsweep : stable in-tile ranking (warp match + per-warp counters, rounds
//               in key order), keys regrouped by digit in shared memory, then
//               written as per-digit runs to their global offsets.
#include <cstdint>
#include <cuda_runtime.h>

#include <type_traits>

#include "ws_common.cuh"
#include "ws_kernels.h"
#include "payload.cuh"
#include "plan.cuh"

namespace ws {
namespace {

constexpr int kRThreads = 256;
constexpr int kRWarps = kRThreads / 32;
constexpr int kDigits = 256;
static_assert(kRThreads == kDigits, "one thread per digit in the per-tile scans");

#ifndef WS_RADIX_E4
#define WS_RADIX_E4 20  // uint32 keys per thread (tile 5120; 16, 12, 24 measured 1-4 % slower)
#endif
template <class K>
struct RadixCfg {
  static constexpr int E = sizeof(K) == 4 ? WS_RADIX_E4 : 8;  // keys per thread
  static constexpr int T = kRThreads * E;            // keys per tile
};

// One-sweep digit width: 10-bit digits for uint32 keys (a 30-bit 6-bit text
// key of 5 characters takes 3 passes instead of 4, 18-24 bits take 2-3), 8
// bits for uint64 keys. A thread owns DPT consecutive digits in the per-tile
// digit phases; per-warp digit counters are 16-bit beyond 256 digits (a tile
// holds < 2^16 keys).
#ifndef WS_OS_DB4
#define WS_OS_DB4 8  // 10 (3 passes of 30-bit keys instead of 4) measured slower: the 1024-digit look-back and scans cost more than a pass
#endif
template <class K>
struct OsCfg {
  static constexpr int DB = sizeof(K) == 4 ? WS_OS_DB4 : 8;
  static constexpr int ND = 1 << DB;
  static constexpr int DPT = ND / kRThreads;
  using WC = typename std::conditional<(ND > 256), uint16_t, uint32_t>::type;
};
static_assert(OsCfg<uint32_t>::ND <= kRadixTotStride && OsCfg<uint32_t>::DPT >= 1, "digits");
static_assert(RadixCfg<uint32_t>::T < (1 << 16), "16-bit digit counters");

__device__ __forceinline__ const RadixSeg& rseg_at(const RadixLaunch& a, int i) {
  return a.segs ? a.segs[i] : a.inl[i];
}

// Segment of a tile (segments ascend by tile_begin); warp-wide ballot search.
__device__ __forceinline__ int rsegment_of(const RadixLaunch& a, uint32_t tile) {
  const int lane = threadIdx.x & 31;
  int found = 0;
  for (int base = 0; base < a.nsegs; base += 32) {
    const int i = base + lane;
    const bool le = i < a.nsegs && rseg_at(a, i).tile_begin <= tile;
    found += __popc(__ballot_sync(0xffffffffu, le));
    if (!__shfl_sync(0xffffffffu, (int)le, 31)) break;
  }
  return found - 1;
}

__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }

template <class K>
__device__ __forceinline__ uint32_t digit_of(K key, uint32_t shift) {
  return (uint32_t)(key >> shift) & 0xFFu;
}

// Lanes of the warp holding the same 8-bit digit (8 ballots; invalid lanes,
// ok == false, match nobody valid). Measured no slower than match.any.
#ifndef WS_MATCH_ANY
#define WS_MATCH_ANY 1  // 0: 8 ballots (the one-sweep passes 3 % slower alone, same step)
#endif
__device__ __forceinline__ uint32_t match_digit8(uint32_t d, bool ok) {
#if WS_MATCH_ANY  // one MATCH.ANY (off the ALU pipe); invalid lanes get unique values > 255
  return __match_any_sync(0xffffffffu, ok ? d : 0x100u + (threadIdx.x & 31));
#endif
  uint32_t peers = __ballot_sync(0xffffffffu, ok);
  if (!ok) peers = ~peers;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const uint32_t bit = (d >> b) & 1u;
    const uint32_t bal = __ballot_sync(0xffffffffu, bit);
    peers &= bal ^ (bit - 1u);  // lanes whose bit b equals mine (one LOP3)
  }
  return peers;
}

// Per-warp stable digit ranks of the warp's keys (round r, lane l <-> key
// r * 32 + l of the warp's slice): rank = earlier keys of the same digit.
// Ranks of a thread's keys: two 16-bit ranks per register (a tile holds <
// 2^16 keys), which keeps the one-sweep kernel within 64 registers.
#ifndef WS_PACK_RK
#define WS_PACK_RK 1
#endif
template <int E>
struct Ranks {
  static constexpr int N = WS_PACK_RK ? (E + 1) / 2 : E;
  uint32_t v[N];
  template <int R>
  __device__ __forceinline__ void set(uint32_t x) {
    if constexpr (WS_PACK_RK) {
      if constexpr (R & 1) v[R >> 1] |= x << 16; else v[R >> 1] = x;
    } else {
      v[R] = x;
    }
  }
  __device__ __forceinline__ uint32_t get(int r) const {
    if (WS_PACK_RK) return (v[r >> 1] >> (16 * (r & 1))) & 0xFFFFu;
    return v[r];
  }
};
template <int R, int E>
struct RankSetter {
  __device__ __forceinline__ static void set(Ranks<E>& rk, int r, uint32_t x) {
    if (r == R) rk.template set<R>(x); else RankSetter<R + 1, E>::set(rk, r, x);
  }
};
template <int E>
struct RankSetter<E, E> {
  __device__ __forceinline__ static void set(Ranks<E>&, int, uint32_t) {}
};

template <class K, int E, int ND = kDigits, class WC = uint32_t>
__device__ __forceinline__ void warp_rank(const K (&key)[E], uint32_t nvalid, uint32_t shift,
                                          WC* wcnt, Ranks<E>& rk) {
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int r = 0; r < E; ++r) {
    const bool ok = (uint32_t)(r * 32 + lane) < nvalid;
    const uint32_t d = (uint32_t)(key[r] >> shift) & (uint32_t)(ND - 1);
    static_assert(ND == 256 || WS_MATCH_ANY, "ballot matching is 8-bit");
    const uint32_t peers = WS_MATCH_ANY ? __match_any_sync(0xffffffffu, ok ? d : 0x10000u + lane)
                                        : match_digit8(d, ok);
    uint32_t base = 0;
    if (ok) base = wcnt[d];
    RankSetter<0, E>::set(rk, r, base + __popc(peers & lt));
    __syncwarp();
    if (ok && lane == 31 - __clz(peers)) wcnt[d] = (WC)(base + __popc(peers));
    __syncwarp();
  }
}

template <class K>
__global__ void __launch_bounds__(kRThreads)
radix_upsweep_kernel(const __grid_constant__ RadixLaunch a) {
  using C = RadixCfg<K>;
  __shared__ uint32_t wcnt[kRWarps][kDigits];
  __shared__ int s_seg;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t tile = blockIdx.x;
  if (tid < 32) {
    const int s = rsegment_of(a, tile);
    if (tid == 0) s_seg = s;
  }
  for (int i = tid; i < kRWarps * kDigits; i += kRThreads) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const RadixSeg& sg = rseg_at(a, s_seg);
  const uint32_t t = tile - sg.tile_begin;
  const uint64_t first = (uint64_t)t * C::T + (uint64_t)wid * 32 * C::E;
  const uint32_t nvalid = first < sg.n ? (uint32_t)umin64(sg.n - first, 32 * C::E) : 0u;
  const K* in = reinterpret_cast<const K*>(sg.in) + first;
  uint32_t* wc = wcnt[wid];
  K key[C::E];  // all loads in flight before the first match
#pragma unroll
  for (int r = 0; r < C::E; ++r) {
    const uint32_t j = r * 32 + lane;
    key[r] = j < nvalid ? in[j] : K(0);  // default caching: the downsweep re-reads from L2
  }
#pragma unroll
  for (int r = 0; r < C::E; ++r)  // per-key shared atomics (no return value: no chain)
    if ((uint32_t)(r * 32 + lane) < nvalid) atomicAdd(wc + digit_of<K>(key[r], sg.shift), 1u);
  __syncthreads();
  uint32_t c = 0;
#pragma unroll
  for (int w = 0; w < kRWarps; ++w) c += wcnt[w][tid];
  a.counts[sg.coff + (uint64_t)tid * sg.ntiles + t] = c;
  if (c) atomicAdd(a.totals + (uint64_t)s_seg * kDigits + tid, c);
}

// One CTA per (segment, digit) row: counts[row][t] -> global element offset
// of the row's keys from tile t (relative to the segment's output base). All
// of a row's loads are issued before the block scan.
constexpr int kScanItems = 8;  // rows of up to 2048 tiles in one sweep
__global__ void __launch_bounds__(kRThreads) radix_scan_kernel(const __grid_constant__ RadixLaunch a) {
  __shared__ uint32_t s_w[kRWarps];
  __shared__ uint32_t s_carry;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int s = blockIdx.x / kDigits, d = blockIdx.x % kDigits;
  const RadixSeg& sg = rseg_at(a, s);
  uint32_t* cnt = a.counts + sg.coff + (uint64_t)d * sg.ntiles;
  // digit prefix of the segment: sum of totals[s][0..d)
  if (wid == 0) {
    const uint32_t* tot = a.totals + (uint64_t)s * kDigits;
    uint32_t pre = 0;
    for (int i = lane; i < d; i += 32) pre += tot[i];
    pre = __reduce_add_sync(0xffffffffu, pre);
    if (lane == 0) s_carry = pre;
  }
  for (uint32_t base = 0; base < sg.ntiles; base += kRThreads * kScanItems) {
    uint32_t v[kScanItems];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const uint32_t i = base + tid * kScanItems + k;
      v[k] = i < sg.ntiles ? cnt[i] : 0u;
      sum += v[k];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    if (lane == 31) s_w[wid] = inc;
    __syncthreads();
    uint32_t run = s_carry + inc - sum;
#pragma unroll
    for (int w = 0; w < kRWarps; ++w) run += w < wid ? s_w[w] : 0u;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      const uint32_t i = base + tid * kScanItems + k;
      if (i < sg.ntiles) cnt[i] = run;
      run += v[k];
    }
    __syncthreads();
    if (tid == kRThreads - 1) s_carry = run;
    __syncthreads();
  }
}

template <class K>
__global__ void __launch_bounds__(kRThreads, 4)
radix_downsweep_kernel(const __grid_constant__ RadixLaunch a) {
  using C = RadixCfg<K>;
  __shared__ uint32_t wcnt[kRWarps][kDigits];
  __shared__ uint32_t s_gdelta[kDigits];  // global offset - tile-local start
  __shared__ uint32_t s_wsum[kRWarps];
  __shared__ __align__(16) K stage[C::T];
  __shared__ int s_seg;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t tile = blockIdx.x;
  if (tid < 32) {
    const int s = rsegment_of(a, tile);
    if (tid == 0) s_seg = s;
  }
  for (int i = tid; i < kRWarps * kDigits; i += kRThreads) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const RadixSeg& sg = rseg_at(a, s_seg);
  const uint32_t t = tile - sg.tile_begin;
  const uint64_t tfirst = (uint64_t)t * C::T;
  const uint64_t first = tfirst + (uint64_t)wid * 32 * C::E;
  const uint32_t nvalid = first < sg.n ? (uint32_t)umin64(sg.n - first, 32 * C::E) : 0u;
  const uint32_t ntile = (uint32_t)umin64(sg.n - tfirst, C::T);
  // the global offsets of this tile's digit runs (scan output), early
  const uint32_t g = a.counts[sg.coff + (uint64_t)tid * sg.ntiles + t];
  const K* in = reinterpret_cast<const K*>(sg.in) + first;
  K key[C::E];
#pragma unroll
  for (int r = 0; r < C::E; ++r) {
    const uint32_t j = r * 32 + lane;
    key[r] = j < nvalid ? __ldcs(in + j) : K(0);
  }
  Ranks<C::E> rk;
  warp_rank<K, C::E>(key, nvalid, sg.shift, wcnt[wid], rk);
  __syncthreads();
  // per digit (thread = digit): exclusive over warps, then over digits
  uint32_t run = 0;
#pragma unroll
  for (int w = 0; w < kRWarps; ++w) {
    const uint32_t c = wcnt[w][tid];
    wcnt[w][tid] = run;
    run += c;
  }
  uint32_t inc = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) s_wsum[wid] = inc;
  __syncthreads();
  uint32_t wpre = 0;
#pragma unroll
  for (int w = 0; w < kRWarps; ++w) wpre += w < wid ? s_wsum[w] : 0u;
  const uint32_t doff = wpre + inc - run;
  s_gdelta[tid] = g - doff;
#pragma unroll
  for (int w = 0; w < kRWarps; ++w) wcnt[w][tid] += doff;  // tile-local start of (warp, digit)
  __syncthreads();
  // regroup the tile by digit in shared memory (stable)
#pragma unroll
  for (int r = 0; r < C::E; ++r) {
    const uint32_t j = r * 32 + lane;
    if (j < nvalid) stage[wcnt[wid][digit_of<K>(key[r], sg.shift)] + rk.get(r)] = key[r];
  }
  __syncthreads();
  // per-digit runs to their global offsets (consecutive threads, consecutive addresses)
  K* out = reinterpret_cast<K*>(sg.out);
  for (uint32_t i = tid; i < ntile; i += kRThreads) {
    const K k = stage[i];
    out[s_gdelta[digit_of<K>(k, sg.shift)] + i] = k;
  }
}

// ---------------------------------------------------------------------------
// One-sweep variant: the digit totals of every pass come from one histogram
// launch over the unsorted keys (a digit's count does not depend on the key
// order), and each pass is a single launch whose tiles find their per-digit
// offsets by a decoupled look-back over the preceding tiles of their segment
// (tiles taken in ticket order, so every awaited tile is already running).
//
// Status word per (tile, digit): epoch (bits 63..34, unique per launch, so no
// clearing between passes) | flag (bits 33..32: 1 tile count, 2 inclusive
// prefix within the segment) | value (bits 31..0). One 64-bit store carries
// flag and value together.
constexpr uint64_t kStAgg = 1ull << 32, kStInc = 2ull << 32;
constexpr uint64_t kStEpochMask = ~0x3FFFFFFFFull;
#ifndef WS_LOOK_W
#define WS_LOOK_W 4
#endif
constexpr int kLookW = WS_LOOK_W;  // predecessors loaded per look-back round
#ifndef WS_LOOK_BACKOFF
#define WS_LOOK_BACKOFF 0  // ns to sleep after a look-back round that found nothing new (0: spin)
#endif
#ifndef WS_OS_MINB
#define WS_OS_MINB 3  // 80 registers, no spills (4: 64 with spills, measured slower)
#endif

__device__ __forceinline__ void st_status(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_status(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Diagnostics: thread 0 stamps phase k of this tile (globaltimer, ns).
#define WS_OS_STAMP(k)                                                         \
  do {                                                                         \
    if (a.prof && threadIdx.x == 0) a.prof[(uint64_t)tile * 8 + (k)] = gtimer(); \
  } while (0)

// Digit histograms of all passes of every segment: totals[sid][p][256].
// Segments whose keys have <= 12 bits (6-bit text words of 1-2 characters,
// raw words of 1 byte) with a payload destination skip the passes: the
// histogram launch counts whole keys (joint[]) and joint_expand_kernel writes
// each distinct word as often as it occurs, at its rank.
constexpr int kJointMax = 1 << 12;

// Histogram of one tile t of segment sg (all threads of the CTA): digit
// counts of every pass into totals[sid][p][256], or whole-key counts into
// joint[] for a jbits segment. sm: the CTA's shared counters (see kSm).
template <class K>
__device__ __forceinline__ void hist_tile(const RadixSeg& sg, uint32_t t, uint32_t* sm,
                                          uint32_t* __restrict__ totals, uint32_t* __restrict__ joint) {
  using C = RadixCfg<K>;
  using O = OsCfg<K>;
  constexpr int ND = O::ND;
  constexpr int kP = (8 * (int)sizeof(K) + O::DB - 1) / O::DB;  // passes of a full-width key
  uint32_t (*hist)[ND] = reinterpret_cast<uint32_t (*)[ND]>(sm);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t jbits = sizeof(K) == 4 ? sg.jbits : 0u;
  const int nzero = jbits ? (1 << jbits) : kP * ND;
  for (int i = tid; i < nzero; i += kRThreads) sm[i] = 0;
  __syncthreads();
  const uint64_t first = (uint64_t)t * C::T + (uint64_t)wid * 32 * C::E;
  const uint32_t nvalid = first < sg.n ? (uint32_t)umin64(sg.n - first, 32 * C::E) : 0u;
  const K* in = reinterpret_cast<const K*>(sg.in) + first;
  K key[C::E];
#pragma unroll
  for (int r = 0; r < C::E; ++r) {
    const uint32_t j = r * 32 + lane;
    key[r] = j < nvalid ? in[j] : K(0);  // default caching: the first pass re-reads from L2
  }
  if (jbits) {
#pragma unroll
    for (int r = 0; r < C::E; ++r)
      if ((uint32_t)(r * 32 + lane) < nvalid) atomicAdd(&sm[(uint32_t)(key[r] >> (32 - jbits))], 1u);
    __syncthreads();
    for (int v = tid; v < (1 << jbits); v += kRThreads)
      if (sm[v]) atomicAdd(joint + sg.joff + v, sm[v]);
  } else {
    const int passes = (int)sg.passes;
#pragma unroll
    for (int p = 0; p < kP; ++p) {
      if (p >= passes) break;
      const uint32_t sh = sg.shift + O::DB * p;
#pragma unroll
      for (int r = 0; r < C::E; ++r)
        if ((uint32_t)(r * 32 + lane) < nvalid)
          atomicAdd(&hist[p][(uint32_t)(key[r] >> sh) & (uint32_t)(ND - 1)], 1u);
    }
    __syncthreads();
    for (int p = 0; p < passes; ++p)
      for (int d = tid; d < ND; d += kRThreads) {
        const uint32_t c = hist[p][d];
        if (c) atomicAdd(totals + ((uint64_t)sg.sid * kRadixMaxPasses + p) * kRadixTotStride + d, c);
      }
  }
  __syncthreads();  // sm is reused by the CTA's next tile
}

template <class K>
__global__ void __launch_bounds__(kRThreads)
radix_hist_kernel(const __grid_constant__ RadixLaunch a) {
  pdl_wait();
  using O = OsCfg<K>;
  constexpr int kP = (8 * (int)sizeof(K) + O::DB - 1) / O::DB;
  constexpr int kSm = kP * O::ND > kJointMax ? kP * O::ND : kJointMax;
  __shared__ uint32_t sm[kSm];  // hist[kP][ND], or the joint counts of a jbits segment
  __shared__ int s_seg;
  const uint32_t tile = blockIdx.x;
  if (threadIdx.x < 32) {
    const int s = rsegment_of(a, tile);
    if (threadIdx.x == 0) s_seg = s;
  }
  __syncthreads();
  const RadixSeg& sg = rseg_at(a, s_seg);
  hist_tile<K>(sg, tile - sg.tile_begin, sm, a.totals, a.joint);
}

// The histogram launch of the 6-bit class-0 buckets (L = 1..5) planned on the
// device from the ingest's per-length counts, so it can run while the host
// reads those counts and plans the passes. Tiles are visited grid-stride; the
// segment table is the one radix_sort_segments builds (nonzero buckets in
// ascending length; whole-key counts for <= 12-bit keys when allowed).
__global__ void __launch_bounds__(kRThreads) radix_hist_early_kernel(const __grid_constant__ EarlyHist e) {
  __shared__ uint32_t sm[kJointMax];
  if (e.go && !*e.go) return;  // class 0's words are being counted instead (dedupe.cu)
  constexpr uint32_t T = RadixCfg<uint32_t>::T;
  RadixSeg seg[5];
  uint32_t nseg = 0, tiles = 0, joff = 0;
  for (int b = 0; b < 5; ++b) {
    const uint32_t n = e.fill[b];
    if (!n) continue;
    // plan.cuh: the host plans the same segments with the same rule
    const RadixPlan pl = radix_plan_c0((uint32_t)b + 1, OsCfg<uint32_t>::DB, e.joint_ok != 0, 12u);
    RadixSeg r;
    memset(&r, 0, sizeof r);
    r.in = e.keys_cap + e.region[b];
    r.n = n;
    r.tile_begin = tiles;
    r.ntiles = (n + T - 1) / T;
    r.shift = pl.shift;
    r.sid = nseg;
    r.passes = pl.passes;
    if (pl.jbits) {
      r.jbits = pl.jbits;
      r.joff = joff;
      joff += 2u << pl.jbits;
    }
    tiles += r.ntiles;
    seg[nseg++] = r;
  }
  for (uint32_t g = blockIdx.x; g < tiles; g += gridDim.x) {
    uint32_t s = 0;
    while (s + 1 < nseg && seg[s + 1].tile_begin <= g) ++s;
    hist_tile<uint32_t>(seg[s], g - seg[s].tile_begin, sm, e.totals, e.joint);
  }
}

// One CTA per jbits segment: exclusive prefix of its 2^jbits counts, stored
// right after them.
// The b-th jbits segment of the launch (counting in segment order).
__device__ __forceinline__ int jseg_at(const RadixLaunch& a, uint32_t b) {
  for (int i = 0; i < a.nsegs; ++i)
    if (rseg_at(a, i).jbits && b-- == 0) return i;
  return 0;
}

__global__ void __launch_bounds__(1024) joint_scan_kernel(const __grid_constant__ RadixLaunch a) {
  pdl_wait();
  __shared__ uint32_t s_w[32];
  const RadixSeg& sg = rseg_at(a, jseg_at(a, blockIdx.x));
  uint32_t* cnt = a.joint + sg.joff;
  const uint32_t nv = 1u << sg.jbits;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint32_t v[4], sum = 0;  // 4 consecutive values per thread (nv <= 4096)
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t i = 4 * tid + q;
    v[q] = i < nv ? cnt[i] : 0u;
    sum += v[q];
  }
  uint32_t inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) s_w[wid] = inc;
  __syncthreads();
  uint32_t run = inc - sum;
  for (int w = 0; w < wid; ++w) run += s_w[w];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t i = 4 * tid + q;
    if (i < nv) cnt[nv + i] = run;
    run += v[q];
  }
}

// One CTA per (jbits segment, key value, part): the value's copies [part
// share] as payload records at pay + (prefix + first copy) * (L + 1).
constexpr int kExpandThreads = 128;
constexpr int kExpandParts = 4;
__global__ void __launch_bounds__(kExpandThreads)
joint_expand_kernel(const __grid_constant__ RadixLaunch a) {
  pdl_wait();
  __shared__ __align__(16) uint8_t pbuf[64 + 16 * 40];
  uint32_t v = blockIdx.x;  // blocks: the jbits segments' values back to back
  int si = 0;
  for (; si < a.nsegs; ++si) {
    const uint32_t jb = rseg_at(a, si).jbits;
    if (!jb) continue;
    if (v < (1u << jb)) break;
    v -= 1u << jb;
  }
  if (si == a.nsegs) return;
  const RadixSeg& sg = rseg_at(a, si);
  const uint32_t* cnt = a.joint + sg.joff;
  const uint32_t c = cnt[v];
  const uint32_t part = blockIdx.y;
  const uint32_t c0 = (uint32_t)((uint64_t)c * part / kExpandParts);
  const uint32_t c1 = (uint32_t)((uint64_t)c * (part + 1) / kExpandParts);
  if (c1 <= c0) return;
  const uint32_t pre = cnt[(1u << sg.jbits) + v];  // copies of smaller values (joint_scan_kernel)
  WS_DCHECK((uint64_t)pre + c1 <= sg.n);
  const int L = (int)sg.len;
  Key<0> k0;
  k0.w[0] = v << (32 - sg.jbits);
  uint8_t* out = sg.pay + (uint64_t)(pre + c0) * (L + 1);
  if (a.enc == kEncAlnum6) {
    fill_records_cta<0, kExpandThreads>(k0, c1 - c0, L, out, pbuf);
  } else {  // raw one-byte words: the record is the byte + '\n'
    const uint64_t n = (uint64_t)(c1 - c0) * 2;
    const uint8_t b = (uint8_t)v;
    for (uint64_t q = threadIdx.x; q < n; q += kExpandThreads) out[q] = (q & 1) ? '\n' : b;
  }
}

template <class K>
__global__ void __launch_bounds__(kRThreads, WS_OS_MINB)
radix_onesweep_kernel(const __grid_constant__ RadixLaunch a) {
  pdl_wait();
  using C = RadixCfg<K>;
  using O = OsCfg<K>;
  constexpr int ND = O::ND, DPT = O::DPT;
  constexpr uint32_t DM = (uint32_t)ND - 1;
  using WC = typename O::WC;
  __shared__ __align__(16) WC wcnt[kRWarps][ND];
  __shared__ uint32_t s_gdelta[ND];  // global offset - tile-local start, per digit
  __shared__ uint32_t s_wsum[2][kRWarps];
  __shared__ __align__(16) K stage[C::T];
  __shared__ int s_seg;
  __shared__ uint32_t s_tile;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid < 32) {  // ticket order: every tile this one waits for has started
    uint32_t tk = 0;
    if (lane == 0) tk = atomicAdd(a.ticket, 1u);
    tk = __shfl_sync(0xffffffffu, tk, 0);
    const int s = rsegment_of(a, tk);
    if (lane == 0) {
      s_seg = s;
      s_tile = tk;
    }
  }
  {
    uint32_t* w32 = reinterpret_cast<uint32_t*>(&wcnt[0][0]);
    for (int i = tid; i < (int)(kRWarps * ND * sizeof(WC) / 4); i += kRThreads) w32[i] = 0;
  }
  __syncthreads();
  const uint32_t tile = s_tile;
  WS_OS_STAMP(0);
  const RadixSeg& sg = rseg_at(a, s_seg);
  const uint32_t t = tile - sg.tile_begin;
  const uint64_t tfirst = (uint64_t)t * C::T;
  const uint64_t first = tfirst + (uint64_t)wid * 32 * C::E;
  const uint32_t nvalid = first < sg.n ? (uint32_t)umin64(sg.n - first, 32 * C::E) : 0u;
  const uint32_t ntile = (uint32_t)umin64(sg.n - tfirst, C::T);
  const int d0 = tid * DPT;  // this thread's digits in the per-tile digit phases
  // this pass's digit totals (-> the digits' bases in the segment), early
  uint32_t tot[DPT];
  {
    const uint32_t* tp = a.totals + ((uint64_t)sg.sid * kRadixMaxPasses + a.pass) * kRadixTotStride + d0;
#pragma unroll
    for (int k = 0; k < DPT; ++k) tot[k] = tp[k];
  }
  const K* in = reinterpret_cast<const K*>(sg.in) + first;
  K key[C::E];
#pragma unroll
  for (int r = 0; r < C::E; ++r) {
    const uint32_t j = r * 32 + lane;
    key[r] = j < nvalid ? __ldcs(in + j) : K(0);
  }
  Ranks<C::E> rk;
  warp_rank<K, C::E, ND, WC>(key, nvalid, sg.shift, wcnt[wid], rk);
  __syncthreads();
  WS_OS_STAMP(1);
  // per digit: exclusive over warps; the tile's count of the digit
  uint32_t run[DPT];
#pragma unroll
  for (int k = 0; k < DPT; ++k) {
    uint32_t r = 0;
#pragma unroll
    for (int w = 0; w < kRWarps; ++w) {
      const uint32_t c = wcnt[w][d0 + k];
      wcnt[w][d0 + k] = (WC)r;
      r += c;
    }
    run[k] = r;
  }
  uint64_t* status = a.status + (uint64_t)tile * ND + d0;
  const uint64_t ep = (uint64_t)a.epoch << 34;
  const bool head = t == 0;  // the segment's first tile: its prefix is 0
#pragma unroll
  for (int k = 0; k < DPT; ++k) st_status(status + k, ep | (head ? kStInc : kStAgg) | run[k]);
  // tile-local digit starts and the digits' bases in the segment (two scans
  // over the ND digits: the thread's own DPT, then across threads)
  uint32_t lsum = 0, lsum2 = 0;
#pragma unroll
  for (int k = 0; k < DPT; ++k) {
    lsum += run[k];
    lsum2 += tot[k];
  }
  uint32_t inc = lsum, inc2 = lsum2;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
    const uint32_t u2 = __shfl_up_sync(0xffffffffu, inc2, o);
    if (lane >= o) {
      inc += u;
      inc2 += u2;
    }
  }
  if (lane == 31) {
    s_wsum[0][wid] = inc;
    s_wsum[1][wid] = inc2;
  }
  __syncthreads();
  uint32_t wpre = 0, wpre2 = 0;
#pragma unroll
  for (int w = 0; w < kRWarps; ++w) {
    wpre += w < wid ? s_wsum[0][w] : 0u;
    wpre2 += w < wid ? s_wsum[1][w] : 0u;
  }
  uint32_t doff[DPT], dbase[DPT];
  {
    uint32_t x = wpre + inc - lsum, y = wpre2 + inc2 - lsum2;
#pragma unroll
    for (int k = 0; k < DPT; ++k) {
      doff[k] = x;
      dbase[k] = y;
      x += run[k];
      y += tot[k];
    }
  }
#pragma unroll
  for (int k = 0; k < DPT; ++k)
#pragma unroll
    for (int w = 0; w < kRWarps; ++w) wcnt[w][d0 + k] = (WC)(wcnt[w][d0 + k] + doff[k]);  // (warp, digit) start
  __syncthreads();
  // regroup the tile by digit in shared memory first (keys and ranks are
  // dead before the look-back's loads are in flight)
#pragma unroll
  for (int r = 0; r < C::E; ++r) {
    const uint32_t j = r * 32 + lane;
    if (j < nvalid) {
      WS_DCHECK(wcnt[wid][(uint32_t)(key[r] >> sg.shift) & DM] + rk.get(r) < ntile);
      stage[wcnt[wid][(uint32_t)(key[r] >> sg.shift) & DM] + rk.get(r)] = key[r];
    }
  }
  // look-back over the segment's preceding tiles for this thread's digits: a
  // window of kLookW predecessors per digit per load round (all loads of a
  // round in flight together), nearest first; the segment's first tile is
  // always inclusive, so every walk stops there
  WS_OS_STAMP(2);
  uint32_t excl[DPT];
  uint32_t rounds = 0, stalls = 0;  // diagnostics (WSORT_OS_PROF)
#pragma unroll
  for (int k = 0; k < DPT; ++k) excl[k] = 0;
  if (!head) {
    uint32_t back[DPT];
    bool done[DPT];
#pragma unroll
    for (int k = 0; k < DPT; ++k) {
      back[k] = 1;
      done[k] = false;
    }
    for (;;) {
      ++rounds;
      constexpr int LW = DPT > 1 ? (kLookW / DPT > 1 ? kLookW / DPT : 2) : kLookW;  // loads per digit
      uint64_t v[DPT][LW];
#pragma unroll
      for (int k = 0; k < DPT; ++k)
#pragma unroll
        for (int w = 0; w < LW; ++w)
          v[k][w] = (!done[k] && back[k] + w <= t)
                        ? ld_status(status + k - (uint64_t)(back[k] + w) * ND)
                        : (ep | kStInc);
      bool all = true;
      uint32_t progress = 0;
#pragma unroll
      for (int k = 0; k < DPT; ++k) {
        if (done[k]) continue;
        uint32_t used = 0;
        bool found = false;
#pragma unroll
        for (int w = 0; w < LW; ++w) {
          if (found || used < (uint32_t)w) continue;         // stopped earlier in this window
          if ((v[k][w] & kStEpochMask) != ep) continue;      // not yet published in this launch
          excl[k] += (uint32_t)v[k][w];
          found = (v[k][w] & kStInc) != 0;
          used = w + 1;
        }
        done[k] = found;
        all = all && found;
        stalls += used < (uint32_t)LW;
        back[k] += used;
        progress += used;
      }
      if (all) break;
#if WS_LOOK_BACKOFF
      // nothing left to read: wait before polling again, so spinning warps
      // do not take issue slots from the ranking warps of other tiles
      if (progress == 0) __nanosleep(WS_LOOK_BACKOFF);
#endif
    }
#pragma unroll
    for (int k = 0; k < DPT; ++k) st_status(status + k, ep | kStInc | (excl[k] + run[k]));
  }
  if (a.prof && tid == 0) {
    a.prof[(uint64_t)tile * 8 + 5] = rounds;
    a.prof[(uint64_t)tile * 8 + 6] = stalls;
  }
#pragma unroll
  for (int k = 0; k < DPT; ++k) s_gdelta[d0 + k] = dbase[k] + excl[k] - doff[k];
  __syncthreads();
  WS_OS_STAMP(3);
  if (sg.pay) {  // the segment's last pass: payload records (characters + '\n') at rank * (L + 1)
    const uint32_t L = sg.len;
    constexpr int kBits = 8 * (int)sizeof(K);
    for (uint32_t i = tid; i < ntile; i += kRThreads) {
      const K k = stage[i];
      WS_DCHECK(s_gdelta[(uint32_t)(k >> sg.shift) & DM] + i < sg.n);
      uint8_t* dst = sg.pay + (uint64_t)(s_gdelta[(uint32_t)(k >> sg.shift) & DM] + i) * (L + 1);
      if constexpr (sizeof(K) == 4) {
        // one-word keys: the record (<= 6 bytes) assembled little-endian in a
        // register and written with the fewest aligned stores (1/2/4 bytes)
        uint64_t rec = (uint64_t)'\n' << (8 * L);
        if (a.enc == kEncAlnum6) {
#pragma unroll
          for (int c = 0; c < 5; ++c)
            if (c < (int)L) rec |= (uint64_t)alnum6_byte((uint32_t)(k >> (26 - 6 * c)) & 63u) << (8 * c);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (c < (int)L) rec |= (uint64_t)((uint32_t)(k >> (24 - 8 * c)) & 0xFFu) << (8 * c);
        }
        uint32_t rem = L + 1;
        if (((uintptr_t)dst & 1) != 0) {
          *dst = (uint8_t)rec;
          rec >>= 8; ++dst; --rem;
        }
        if (((uintptr_t)dst & 2) != 0 && rem >= 2) {
          *reinterpret_cast<uint16_t*>(dst) = (uint16_t)rec;
          rec >>= 16; dst += 2; rem -= 2;
        }
        if (rem >= 4) {
          *reinterpret_cast<uint32_t*>(dst) = (uint32_t)rec;
          rec >>= 32; dst += 4; rem -= 4;
        }
        if (rem >= 2) {
          *reinterpret_cast<uint16_t*>(dst) = (uint16_t)rec;
          rec >>= 16; dst += 2; rem -= 2;
        }
        if (rem) *dst = (uint8_t)rec;
        continue;
      }
      if (a.enc == kEncAlnum6) {
#pragma unroll
        for (int c = 0; c < kBits / 6; ++c)
          if (c < (int)L) dst[c] = (uint8_t)alnum6_byte((uint32_t)(k >> (kBits - 6 - 6 * c)) & 63u);
      } else {
#pragma unroll
        for (int c = 0; c < kBits / 8; ++c)
          if (c < (int)L) dst[c] = (uint8_t)(k >> (kBits - 8 - 8 * c));
      }
      dst[L] = '\n';
    }
    if (a.prof) {
      __syncthreads();
      WS_OS_STAMP(4);
    }
    return;
  }
  K* out = reinterpret_cast<K*>(sg.out);
  for (uint32_t i = tid; i < ntile; i += kRThreads) {
    const K k = stage[i];
    WS_DCHECK(s_gdelta[(uint32_t)(k >> sg.shift) & DM] + i < sg.n);
    out[s_gdelta[(uint32_t)(k >> sg.shift) & DM] + i] = k;
  }
  if (a.prof) {
    __syncthreads();
    WS_OS_STAMP(4);
  }
}

}  // namespace

void launch_radix_hist(int lanes, const RadixLaunch& a, cudaStream_t st) {
  if (!a.work_items) return;
  if (lanes == 0)
    launch_pdl(radix_hist_kernel<uint32_t>, a.work_items, kRThreads, 0, st, a);
  else
    launch_pdl(radix_hist_kernel<uint64_t>, a.work_items, kRThreads, 0, st, a);
}

#ifndef WS_HIST_EARLY_CTAS
#define WS_HIST_EARLY_CTAS 8  // per SM (grid-stride over the tiles)
#endif
void launch_radix_hist_early(const EarlyHist& e, cudaStream_t st) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  radix_hist_early_kernel<<<WS_HIST_EARLY_CTAS * sms, kRThreads, 0, st>>>(e);
}

void launch_joint_expand(const RadixLaunch& a, uint32_t blocks, uint32_t njsegs, cudaStream_t st) {
  if (!blocks) return;
  launch_pdl(joint_scan_kernel, njsegs, 1024, 0, st, a);
  launch_pdl(joint_expand_kernel, dim3(blocks, kExpandParts), kExpandThreads, 0, st, a);
}

void launch_radix_onesweep(int lanes, const RadixLaunch& a, cudaStream_t st) {
  if (!a.work_items) return;
  if (lanes == 0)
    launch_pdl(radix_onesweep_kernel<uint32_t>, a.work_items, kRThreads, 0, st, a);
  else
    launch_pdl(radix_onesweep_kernel<uint64_t>, a.work_items, kRThreads, 0, st, a);
}

int radix_tile_size(int lanes) { return lanes == 0 ? RadixCfg<uint32_t>::T : RadixCfg<uint64_t>::T; }
int radix_digit_bits(int lanes) { return lanes == 0 ? OsCfg<uint32_t>::DB : OsCfg<uint64_t>::DB; }

void launch_radix_pass(int lanes, const RadixLaunch& a, cudaStream_t st) {
  if (!a.work_items) return;
  const uint32_t rows = (uint32_t)a.nsegs * kDigits;
  if (lanes == 0) {
    radix_upsweep_kernel<uint32_t><<<a.work_items, kRThreads, 0, st>>>(a);
    radix_scan_kernel<<<rows, kRThreads, 0, st>>>(a);
    radix_downsweep_kernel<uint32_t><<<a.work_items, kRThreads, 0, st>>>(a);
  } else {
    radix_upsweep_kernel<uint64_t><<<a.work_items, kRThreads, 0, st>>>(a);
    radix_scan_kernel<<<rows, kRThreads, 0, st>>>(a);
    radix_downsweep_kernel<uint64_t><<<a.work_items, kRThreads, 0, st>>>(a);
  }
}

WS_DEFINE_CHECK_READER(check_reader_radix)

}  // namespace ws
