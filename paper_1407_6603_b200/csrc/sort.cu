// Per-bucket sort of packed keys, all buckets of one key width in one
// segmented launch per pass.
//
// Replaces the reference's O(n^2) triangular bubble sort _bubble_rows
// (engine.py:89-114) and its per-bucket thread pool (engine.py:140-201).
// The output order is the same composite order: the reference swaps only on
// strictly-greater (engine.py:105), so its sort is stable and equal keys keep
// corpus order; every pass here is stable too (OETS swaps on strict '>', the
// merges take A first on ties).
//
//   tile pass  : the tile (T = threads * E keys) lands in shared memory by a
//                1-D TMA bulk copy; each thread takes E consecutive keys into
//                registers and runs odd-even transposition sort on them (E
//                phases of compare-exchange on strict '>': the data-parallel
//                form of bubble sort); log2(threads) merge-path levels in
//                shared memory then merge the runs into one sorted tile.
//   merge pass : one partition launch (a warp per output tile finds its
//                merge-path split in global memory, all in parallel) and one
//                merge launch per level: each CTA bulk-copies its A and B
//                windows into shared memory (TMA + mbarrier), merge-path
//                merges them, and streams the tile out coalesced.
//
// E is odd everywhere: with 8-byte keys a warp's blocked accesses (lane l at
// element E*l + k) then hit 16 distinct bank pairs (conflict-free without
// padding), and neighbouring lanes' binary-search probes fall on different
// banks (E = 8 gave 8-way conflicts and a smem-bound merge).
//
// Stats mode carries a uint32 payload idx = the word's corpus rank inside its
// bucket and returns, per bucket:
//   inversions = OETS swaps inside the E-runs + sum over every merge of
//                #{a in A : a > b} for b in B (counted when b is emitted:
//                the A elements still pending are exactly the larger ones);
//                the reference's swap count equals this (each adjacent swap of
//                a strict-'>' bubble sort removes exactly one inversion).
//   K          = max(idx - final position), which fixes the early-exit pass
//                count P = min(K + 1, n - 1) (engine.py:112-113).
#include <algorithm>

#include "ws_common.cuh"
#include "ws_kernels.h"
#include "payload.cuh"
#include "tma.cuh"
#include "plan.cuh"

namespace ws {

#ifndef WS_TILE_E1
#define WS_TILE_E1 15  // keys per thread in the tile pass, 1-lane keys (odd)
#endif
#ifndef WS_TILE_EN
#define WS_TILE_EN 7  // keys per thread in the tile pass, 2..4-lane keys (odd)
#endif
#ifndef WS_TILE_NT
#define WS_TILE_NT 256  // threads per CTA in the tile pass
#endif
#ifndef WS_MERGE_E
#define WS_MERGE_E 15  // outputs per thread in a merge pass (odd; 7-13 measured 1-3 % slower in stats mode)
#endif
#ifndef WS_MERGE_NT
#define WS_MERGE_NT 256  // threads per CTA in a merge pass
#endif

constexpr int kTileThreads = WS_TILE_NT;
constexpr int kMergeThreads = WS_MERGE_NT;

template <int LANES>
struct TileCfg {
  static constexpr int NT = kTileThreads;
  static constexpr int E = LANES <= 1 ? WS_TILE_E1 : WS_TILE_EN;
  static constexpr int T = NT * E;
};

#ifndef WS_MERGE_EW
#define WS_MERGE_EW 7  // outputs per thread in a merge pass of multi-word keys (odd; smaller tiles, more CTAs for the latency-bound smaller classes: stats step 1.583 -> 1.526 ms, 9: 1.531, 11: 1.59)
#endif
template <int LANES>
struct MergeCfg {
  static constexpr int NT = kMergeThreads;
  static constexpr int E = LANES <= 0 ? WS_MERGE_E : WS_MERGE_EW;
  static constexpr int T = NT * E;
  static constexpr int MIN_BLOCKS = LANES <= 1 ? 2048 / NT : (LANES == 2 ? 1024 / NT : 512 / NT);
};

// smem bytes: keys (AoS, 16-byte slack on each side for the bulk-copy
// rounding) followed by the idx payload in stats mode.
template <int LANES, int T, bool STATS>
__host__ __device__ constexpr size_t keys_smem_bytes() {
  return (size_t)T * key_bytes(LANES) + 64;
}
template <int LANES, int T, bool STATS>
__host__ __device__ constexpr size_t pass_smem_bytes() {
  return keys_smem_bytes<LANES, T, STATS>() + (STATS ? (size_t)T * 4 + 64 : 0);
}

template <int LANES>
using KW = typename KeyTraits<LANES>::W;

template <int LANES>
__device__ __forceinline__ Key<LANES> ldk(const KW<LANES>* __restrict__ p, int i) {
  constexpr int NW = KeyTraits<LANES>::NW;
  Key<LANES> k;
#pragma unroll
  for (int l = 0; l < NW; ++l) k.w[l] = p[i * NW + l];
  return k;
}

template <int LANES>
__device__ __forceinline__ void stk(KW<LANES>* __restrict__ p, int i, const Key<LANES>& k) {
  constexpr int NW = KeyTraits<LANES>::NW;
#pragma unroll
  for (int l = 0; l < NW; ++l) p[i * NW + l] = k.w[l];
}

template <int LANES>
__device__ __forceinline__ Key<LANES> gld(const KW<LANES>* __restrict__ g, int64_t i) {
  constexpr int NW = KeyTraits<LANES>::NW;
  Key<LANES> k;
#pragma unroll
  for (int l = 0; l < NW; ++l) k.w[l] = __ldg(g + i * NW + l);
  return k;
}

// Key arrays are passed around as uint64_t*; kernels view them in words of W.
template <int LANES>
__device__ __forceinline__ const KW<LANES>* kv(const uint64_t* p) {
  return reinterpret_cast<const KW<LANES>*>(p);
}
template <int LANES>
__device__ __forceinline__ KW<LANES>* kv(uint64_t* p) {
  return reinterpret_cast<KW<LANES>*>(p);
}

// Byte window [src, src + bytes) rounded out to 16-byte boundaries for a bulk
// copy; `off` is the offset of src inside the landed window.
struct Window16 {
  const uint8_t* g;
  uint32_t off;
  uint32_t bytes;
};

__device__ __forceinline__ Window16 window16(const void* src, uint32_t bytes) {
  const uintptr_t a = reinterpret_cast<uintptr_t>(src);
  Window16 w;
  w.g = reinterpret_cast<const uint8_t*>(a & ~uintptr_t(15));
  w.off = (uint32_t)(a & 15);
  w.bytes = (w.off + bytes + 15) & ~15u;
  return w;
}

// ---- shared pieces --------------------------------------------------------------

__device__ __forceinline__ const SegDesc& seg_at(const SortLaunch& a, int i) {
  return a.segs ? a.segs[i] : a.inl[i];
}

// Segment of this CTA: the last segment whose first work item <= item. One
// warp reads up to 32 tile_begin values per step and ballots.
__device__ __forceinline__ int segment_of(const SortLaunch& a, uint32_t item) {
  const int lane = threadIdx.x & 31;
  const int nsegs = a.nsegs;
  int found = 0;
  for (int base = 0; base < nsegs; base += 32) {
    const int i = base + lane;
    const bool le = i < nsegs && seg_at(a, i).tile_begin <= item;
    found += __popc(__ballot_sync(0xffffffffu, le));
    if (!__shfl_sync(0xffffffffu, (int)le, 31)) break;
  }
  return found - 1;
}

__device__ __forceinline__ int find_segment(const SortLaunch& a, uint32_t item) {
  __shared__ int s_seg;
  if (threadIdx.x < 32) {
    const int s = segment_of(a, item);
    if (threadIdx.x == 0) s_seg = s;
  }
  __syncthreads();
  return s_seg;
}

template <bool STATS>
__device__ __forceinline__ void flush_stats(uint64_t inv, long long kloc, const SegDesc& sd,
                                            unsigned long long* ginv, long long* gk) {
  if (!STATS) return;
  __shared__ unsigned long long s_inv;
  __shared__ long long s_k;
  if (threadIdx.x == 0) {
    s_inv = 0;
    s_k = 0;
  }
  __syncthreads();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    inv += __shfl_xor_sync(0xffffffffu, inv, o);
    kloc = max(kloc, (long long)__shfl_xor_sync(0xffffffffu, kloc, o));
  }
  if ((threadIdx.x & 31) == 0) {
    if (inv) atomicAdd(&s_inv, (unsigned long long)inv);
    if (kloc > 0) atomicMax(&s_k, kloc);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (s_inv) atomicAdd(&ginv[sd.stat_slot], s_inv);
    if (s_k > 0) atomicMax(&gk[sd.stat_slot], s_k);
  }
}

// Merge path over two AoS runs in shared memory: this thread emits outputs
// [diag, diag + E). When taking b, the pending A elements are exactly those
// > b: inv += a_rem_base - ai.
template <int LANES, int E, bool STATS>
__device__ __forceinline__ void merge_path(const KW<LANES>* __restrict__ A, int na,
                                           const KW<LANES>* __restrict__ B, int nb,
                                           const uint32_t* __restrict__ IA,
                                           const uint32_t* __restrict__ IB, int diag,
                                           int64_t a_rem_base, Key<LANES> (&r)[E],
                                           uint32_t (&ri)[E], uint64_t& inv) {
  // lower bound of the diagonal: the range halves the same way whichever side
  // wins, so lanes stay converged; the body is predicated selects
  int lo = max(0, diag - nb);
  int len = min(diag, na) - lo;
  while (len > 0) {
    const int half = len >> 1, mid = lo + half;
    const bool p = key_le<LANES>(ldk<LANES>(A, mid), ldk<LANES>(B, diag - 1 - mid));
    lo = p ? mid + 1 : lo;
    len = p ? len - half - 1 : half;
  }
  int ai = lo, bi = diag - lo;
  const Key<LANES> kmax = key_max<LANES>();
  Key<LANES> ka = ai < na ? ldk<LANES>(A, ai) : kmax;
  Key<LANES> kb = bi < nb ? ldk<LANES>(B, bi) : kmax;
  uint32_t ia = 0, ib = 0;
  if (STATS) {
    ia = ai < na ? IA[ai] : 0u;
    ib = bi < nb ? IB[bi] : 0u;
  }
  // branch-free merge: take one side, advance it, reload only that side.
  // A elements still pending when a b is taken: rem = a_rem_base - ai, kept
  // as a 32-bit running count (E * rem < 2^32 for any bucket < 2^28 keys)
  uint32_t rem = STATS ? (uint32_t)(a_rem_base - ai) : 0u, inv32 = 0;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const bool ta = (bi >= nb) || (ai < na && key_le<LANES>(ka, kb));
#pragma unroll
    for (int l = 0; l < KeyTraits<LANES>::NW; ++l) r[k].w[l] = ta ? ka.w[l] : kb.w[l];
    if (STATS) {
      ri[k] = ta ? ia : ib;
      inv32 += ta ? 0u : rem;
      rem -= ta ? 1u : 0u;
    }
    ai += ta ? 1 : 0;
    bi += ta ? 0 : 1;
    const int nx = ta ? ai : bi;
    const bool ok = ta ? ai < na : bi < nb;
    const KW<LANES>* src = ta ? A : B;
    const Key<LANES> nk = ok ? ldk<LANES>(src, nx) : kmax;
#pragma unroll
    for (int l = 0; l < KeyTraits<LANES>::NW; ++l) {
      ka.w[l] = ta ? nk.w[l] : ka.w[l];
      kb.w[l] = ta ? kb.w[l] : nk.w[l];
    }
    if (STATS) {
      const uint32_t ni = ok ? (ta ? IA : IB)[nx] : 0u;
      ia = ta ? ni : ia;
      ib = ta ? ib : ni;
    }
  }
  if (STATS) inv += inv32;
}

// Registers (blocked, E per thread starting at element `base`) -> AoS smem.
template <int LANES, int E, bool STATS>
__device__ __forceinline__ void regs_to_smem(KW<LANES>* sk, uint32_t* si, int base,
                                             const Key<LANES> (&r)[E], const uint32_t (&ri)[E]) {
#pragma unroll
  for (int k = 0; k < E; ++k) {
    stk<LANES>(sk, base + k, r[k]);
    if (STATS) si[base + k] = ri[k];
  }
}

// AoS smem -> global, coalesced over the flat uint64 words of cnt keys.
template <int LANES, bool STATS, int NT>
__device__ __forceinline__ void smem_to_global(const KW<LANES>* sk, const uint32_t* si, int cnt,
                                               KW<LANES>* __restrict__ gk, uint32_t* __restrict__ gi) {
  const int words = cnt * KeyTraits<LANES>::NW;
  int w = threadIdx.x;
  for (; w + NT < words; w += 2 * NT) {  // two independent stores in flight
    const KW<LANES> x = sk[w], y = sk[w + NT];
    gk[w] = x;
    gk[w + NT] = y;
  }
  if (w < words) gk[w] = sk[w];
  if (STATS && gi) {
    for (int j = threadIdx.x; j < cnt; j += NT) gi[j] = si[j];
  }
}

// ---- tile pass -------------------------------------------------------------------

// The on-chip sort of one tile already in shared memory (T keys, all-ones
// sentinels after the first cnt): each thread takes E consecutive keys into
// registers and runs odd-even transposition sort on them (E phases of
// compare-exchange on strict '>'); merge-path levels in shared memory then
// merge the runs. Levels stop once a run covers all cnt real keys (the
// sentinels behind them are already in place). Leaves the thread's E
// outputs of the sorted tile (blocked) in r / ri; idx0 = idx of key 0.
// NT = the CTA's threads (the tile holds NT * E keys).
// sk2 (keys only, optional): a second key buffer; the merge levels then
// alternate buffers and need one barrier per level instead of two (a level
// writes the buffer no thread can still be reading).
// EO (or 0): keys per thread, overriding the lane class's tile width.
template <int LANES, bool STATS, int NT = kTileThreads, bool NAMED = false, int EO = 0>
__device__ __forceinline__ void tile_network(KW<LANES>* sk, uint32_t* si, int cnt, uint32_t idx0,
                                             Key<LANES> (&r)[EO ? EO : TileCfg<LANES>::E],
                                             uint32_t (&ri)[EO ? EO : TileCfg<LANES>::E], uint64_t& inv,
                                             KW<LANES>* sk2 = nullptr) {
  constexpr int E = EO ? EO : TileCfg<LANES>::E, T = NT * E;
  constexpr int NW = KeyTraits<LANES>::NW;
  const int tid = (int)threadIdx.x;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    r[k] = ldk<LANES>(sk, tid * E + k);
    ri[k] = STATS ? idx0 + (uint32_t)(tid * E + k) : 0u;
  }
  // Odd-even transposition sort of the thread's E keys: E phases, each a
  // layer of independent compare-exchanges that swap on strictly-greater.
  // (Threads holding only sentinels skip the work.)
  const bool real = tid * E < cnt;
#pragma unroll
  for (int ph = 0; ph < E; ++ph) {
    if (!real) break;
#pragma unroll
    for (int i = ph & 1; i + 1 < E; i += 2) {
      const bool sw = key_lt<LANES>(r[i + 1], r[i]);
      if (sw) {
        Key<LANES> t = r[i];
        r[i] = r[i + 1];
        r[i + 1] = t;
        uint32_t u = ri[i];
        ri[i] = ri[i + 1];
        ri[i + 1] = u;
      }
      if (STATS) inv += sw;
    }
  }
  // Merge-path levels inside the tile.
  int lvl = 0;
#pragma unroll 1
  for (int run = E; run < T && run < cnt; run <<= 1, ++lvl) {
    KW<LANES>* buf = sk;
    if (!STATS && sk2) {  // double-buffered: alternate, one barrier per level
      buf = (lvl & 1) ? sk : sk2;
    } else {
      nt_sync<NT, NAMED>();
    }
    regs_to_smem<LANES, E, STATS>(buf, si, tid * E, r, ri);
    nt_sync<NT, NAMED>();
    const int gt = (2 * run) / E;  // threads per merged pair
    const int a0 = (tid / gt) * 2 * run;
    if (a0 >= cnt) continue;  // a pair of sentinel runs: r already holds sentinels
    merge_path<LANES, E, STATS>(buf + (size_t)a0 * NW, run, buf + (size_t)(a0 + run) * NW, run,
                                si + a0, si + a0 + run, (tid % gt) * E, run, r, ri, inv);
  }
}


template <int LANES, bool STATS>
__global__ void __launch_bounds__(kTileThreads) tile_sort_kernel(const __grid_constant__ SortLaunch a) {
  pdl_wait();
  constexpr int E = TileCfg<LANES>::E, T = TileCfg<LANES>::T, NT = kTileThreads;
  constexpr int NW = KeyTraits<LANES>::NW, KB = key_bytes(LANES);
  using W = KW<LANES>;
  constexpr size_t kKeyBytes = keys_smem_bytes<LANES, T, STATS>();
  extern __shared__ __align__(16) uint64_t smem[];
  uint8_t* sbytes = reinterpret_cast<uint8_t*>(smem);
  uint32_t* si = reinterpret_cast<uint32_t*>(sbytes + kKeyBytes);
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const SegDesc sd = seg_at(a, find_segment(a, blockIdx.x));
  const uint64_t start = (uint64_t)(blockIdx.x - sd.tile_begin) * T;
  const int cnt = (int)min((uint64_t)T, (uint64_t)sd.n - start);
  WS_DCHECK(start < sd.n && cnt > 0);
  const W* gin = (sd.in_ptr ? kv<LANES>(sd.in_ptr) : kv<LANES>(a.keys_in) + sd.key_off * NW) +
                 start * NW;
  const Window16 w = window16(gin, (uint32_t)cnt * KB);
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, w.bytes);
    tma_load_1d(sbytes, w.g, w.bytes, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
  W* sk = reinterpret_cast<W*>(sbytes + w.off);  // element 0 of the tile
  // all-ones sentinels after the last key: they sort last and, being at the
  // highest positions, never swap with a real key (ties keep order)
  for (int j = cnt * NW + tid; j < T * NW; j += NT) sk[j] = ~W(0);
  __syncthreads();

  Key<LANES> r[E];
  uint32_t ri[E];
  uint64_t inv = 0;
  tile_network<LANES, STATS>(sk, si, cnt, (uint32_t)(sd.idx_base + start), r, ri, inv);
  long long kloc = 0;
  if (STATS && sd.n <= (uint32_t)T) {
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int pos = tid * E + k;
      if (pos < cnt) kloc = max(kloc, (long long)ri[k] - (long long)sd.idx_base - pos);
    }
  }
  flush_stats<STATS>(inv, kloc, sd, a.inv, a.kmax);
  __syncthreads();
  regs_to_smem<LANES, E, STATS>(sk, si, tid * E, r, ri);
  __syncthreads();
  smem_to_global<LANES, STATS, NT>(sk, si, cnt, kv<LANES>(a.keys_out) + (sd.key_off + start) * NW,
                                   a.idx_out ? a.idx_out + sd.idx_off + start : nullptr);
}

// ---- merge pass ------------------------------------------------------------------

// Warp-wide 32-ary merge-path search in global memory: the number of A
// elements among the first d outputs of merge(A, B) (A first on ties).
template <int LANES>
__device__ int64_t merge_path_search_global(const KW<LANES>* __restrict__ A, int64_t na,
                                            const KW<LANES>* __restrict__ B, int64_t nb, int64_t d) {
  const int lane = threadIdx.x & 31;
  int64_t lo = max((int64_t)0, d - nb), hi = min(d, na);
  while (hi > lo) {
    const int64_t span = hi - lo;
    if (span <= 32) {
      const int64_t x = lo + lane;
      bool p = false;
      if (x < hi) p = key_le<LANES>(gld<LANES>(A, x), gld<LANES>(B, d - 1 - x));
      return lo + __popc(__ballot_sync(0xffffffffu, p));
    }
    const int64_t step = (span + 31) / 32;
    const int64_t x = lo + lane * step;
    bool p = false;
    if (x < hi) p = key_le<LANES>(gld<LANES>(A, x), gld<LANES>(B, d - 1 - x));
    const int c = __popc(__ballot_sync(0xffffffffu, p));
    const int64_t nlo = c > 0 ? lo + (int64_t)(c - 1) * step + 1 : lo;
    const int64_t xc = lo + (int64_t)c * step;
    const int64_t nhi = (c < 32 && xc < hi) ? xc : hi;
    lo = nlo;
    hi = nhi;
  }
  return lo;
}

struct PairGeom {
  int64_t n, pair_base, na, nb, d0, d1;
  bool empty;  // item past the end of a partial last pair
};

// Work items of a merge level: every pair of runs gets ceil(2R / T) output
// tiles, so a tile never straddles two pairs whatever T is.
__device__ __forceinline__ PairGeom pair_geom(const SegDesc& sd, uint32_t item, int64_t R, int T) {
  PairGeom g;
  g.n = sd.n;
  // 32-bit division (work items and tiles per pair fit in 32 bits; a 64-bit
  // divide is a long subroutine that every thread of every CTA would run)
  const uint32_t tpp = (uint32_t)((2 * R + T - 1) / T);
  const uint32_t local = item - sd.tile_begin;
  const uint32_t pair = local / tpp;
  g.pair_base = (int64_t)pair * (2 * R);
  g.na = min(R, g.n - g.pair_base);
  g.nb = g.n - g.pair_base > R ? min(R, g.n - g.pair_base - R) : 0;
  g.d0 = (int64_t)(local - pair * tpp) * T;
  g.empty = g.d0 >= g.na + g.nb;
  g.d1 = min(g.d0 + T, g.na + g.nb);
  return g;
}

// Partition pass: one warp per output tile finds the A/B split of the tile's
// first output; it also records the tile's segment so the merge CTA skips
// its own lookup.
template <int LANES>
__global__ void __launch_bounds__(256) merge_split_kernel(const __grid_constant__ SortLaunch a) {
  pdl_wait();
  constexpr int T = MergeCfg<LANES>::T;
  const uint32_t item = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (item >= a.work_items) return;
  const int seg = segment_of(a, item);
  const SegDesc sd = seg_at(a, seg);
  const PairGeom g = pair_geom(sd, item, a.run, T);
  int64_t s = 0;
  if (!g.empty) {
    constexpr int NW = KeyTraits<LANES>::NW;
    const KW<LANES>* A = kv<LANES>(a.keys_in) + (sd.key_off + g.pair_base) * NW;
    const KW<LANES>* B = A + (int64_t)a.run * NW;
    s = merge_path_search_global<LANES>(A, g.na, B, g.nb, g.d0);
  }
  if ((threadIdx.x & 31) == 0) {
    a.splits[2 * item] = (uint32_t)s;
    a.splits[2 * item + 1] = (uint32_t)seg;
  }
}

#ifndef WS_MERGE_FUSED_SPLIT
#define WS_MERGE_FUSED_SPLIT 0  // 1: merge CTAs search their own splits, no partition launch (measured: same stats step)
#endif
#ifndef WS_MERGE_STATS_MINB
#define WS_MERGE_STATS_MINB 6  // stats mode, uint32 keys: 40 registers (8 CTAs/SM spilled 92-124 B)
#endif
#ifndef WS_MERGE_STATS_MINB1
#define WS_MERGE_STATS_MINB1 4  // stats mode, multi-word keys
#endif
template <int LANES, bool STATS>
__global__ void __launch_bounds__(kMergeThreads, !STATS ? MergeCfg<LANES>::MIN_BLOCKS
                                                        : (LANES == 0 ? WS_MERGE_STATS_MINB
                                                                      : (LANES == 1 ? WS_MERGE_STATS_MINB1 : MergeCfg<LANES>::MIN_BLOCKS)))
    merge_kernel(const __grid_constant__ SortLaunch a) {
  pdl_wait();
  constexpr int E = MergeCfg<LANES>::E, T = MergeCfg<LANES>::T, NT = kMergeThreads;
  constexpr int NW = KeyTraits<LANES>::NW, KB = key_bytes(LANES);
  using W = KW<LANES>;
  constexpr size_t kKeyBytes = keys_smem_bytes<LANES, T, STATS>();
  extern __shared__ __align__(16) uint64_t smem[];
  uint8_t* sbytes = reinterpret_cast<uint8_t*>(smem);
  uint32_t* si = reinterpret_cast<uint32_t*>(sbytes + kKeyBytes);
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  const int64_t R = a.run;
  const uint32_t item = blockIdx.x;
#if WS_MERGE_FUSED_SPLIT
  // the CTA finds its own merge-path splits: warp 0 the A/B split of its first
  // output, warp 1 that of its last + 1 (no partition launch, no dependent
  // round trip between launches)
  __shared__ int64_t s_split2[2];
  const SegDesc sd = seg_at(a, find_segment(a, item));
  const PairGeom g = pair_geom(sd, item, R, T);
  if (g.empty) return;  // uniform across the CTA
  {
    const int w = tid >> 5;
    if (w < 2) {
      const int64_t d = w == 0 ? g.d0 : g.d1;
      int64_t sp = 0;
      if (w == 0 ? d > 0 : d < g.na + g.nb) {
        const KW<LANES>* A = kv<LANES>(a.keys_in) + (sd.key_off + g.pair_base) * NW;
        sp = merge_path_search_global<LANES>(A, g.na, A + R * NW, g.nb, d);
      } else {
        sp = w == 0 ? 0 : g.na;
      }
      if ((tid & 31) == 0) s_split2[w] = sp;
    }
    __syncthreads();
  }
  const int64_t a0 = s_split2[0];
  const int64_t a1 = s_split2[1];
#else
  const SegDesc sd = seg_at(a, (int)a.splits[2 * item + 1]);  // written by the partition pass
  const PairGeom g = pair_geom(sd, item, R, T);
  if (g.empty) return;  // uniform across the CTA
  const int64_t a0 = a.splits[2 * item];
  const int64_t a1 = (g.d1 == g.na + g.nb) ? g.na : (int64_t)a.splits[2 * item + 2];
#endif
  const int64_t b0 = g.d0 - a0, b1 = g.d1 - a1;
  const int la = (int)(a1 - a0), lb = (int)(b1 - b0);
  WS_DCHECK(la >= 0 && lb >= 0 && la + lb <= T && a1 <= g.na && b1 <= g.nb);
  const W* Ag = kv<LANES>(a.keys_in) + (sd.key_off + g.pair_base + a0) * NW;
  const W* Bg = kv<LANES>(a.keys_in) + (sd.key_off + g.pair_base + R + b0) * NW;
  const Window16 wa = window16(Ag, (uint32_t)la * KB);
  const Window16 wb = window16(Bg, (uint32_t)lb * KB);
  const uint32_t b_at = wa.bytes;  // B window lands right after A's
  Window16 wia{}, wib{};
  uint32_t ib_at = 0;
  if (STATS) {
    wia = window16(a.idx_in + sd.idx_off + g.pair_base + a0, (uint32_t)la * 4);
    wib = window16(a.idx_in + sd.idx_off + g.pair_base + R + b0, (uint32_t)lb * 4);
    ib_at = wia.bytes;
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    uint32_t tx = (la ? wa.bytes : 0) + (lb ? wb.bytes : 0);
    if (STATS) tx += (la ? wia.bytes : 0) + (lb ? wib.bytes : 0);
    mbar_expect_tx(&bar, tx);
    if (la) tma_load_1d(sbytes, wa.g, wa.bytes, &bar);
    if (lb) tma_load_1d(sbytes + b_at, wb.g, wb.bytes, &bar);
    if (STATS) {
      uint8_t* ibase = reinterpret_cast<uint8_t*>(si);
      if (la) tma_load_1d(ibase, wia.g, wia.bytes, &bar);
      if (lb) tma_load_1d(ibase + ib_at, wib.g, wib.bytes, &bar);
    }
  }
  __syncthreads();  // barrier initialised before anyone waits on it
  mbar_wait(&bar, 0);
  const W* As = reinterpret_cast<const W*>(sbytes + wa.off);
  const W* Bs = reinterpret_cast<const W*>(sbytes + b_at + wb.off);
  const uint32_t* IAs = reinterpret_cast<const uint32_t*>(reinterpret_cast<uint8_t*>(si) + wia.off);
  const uint32_t* IBs =
      reinterpret_cast<const uint32_t*>(reinterpret_cast<uint8_t*>(si) + ib_at + wib.off);
  Key<LANES> r[E];
  uint32_t ri[E];
  uint64_t inv = 0;
  merge_path<LANES, E, STATS>(As, la, Bs, lb, IAs, IBs, min(tid * E, la + lb), R - a0, r, ri, inv);
  long long kloc = 0;
  const int64_t out_begin = g.pair_base + g.d0;
  if (STATS && 2 * R >= g.n) {
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const int64_t lp = (int64_t)tid * E + k;
      if (lp < la + lb)
        kloc = max(kloc, (long long)ri[k] - (long long)sd.idx_base - (long long)(out_begin + lp));
    }
  }
  flush_stats<STATS>(inv, kloc, sd, a.inv, a.kmax);
  __syncthreads();  // every thread is done reading the input windows
  W* sk = reinterpret_cast<W*>(smem);  // output staging reuses the window bytes (AoS)
  if (tid * E < la + lb) regs_to_smem<LANES, E, STATS>(sk, si, tid * E, r, ri);
  __syncthreads();
  smem_to_global<LANES, STATS, NT>(sk, si, la + lb,
                                   kv<LANES>(a.keys_out) + (sd.key_off + out_begin) * NW,
                                   STATS ? a.idx_out + sd.idx_off + out_begin : nullptr);
}

// ---- payload-mode sample sort (multi-lane classes) ------------------------------
//
// Payload mode only needs the sorted bytes, so a bucket larger than a tile is
// split by value instead of merged level by level: S - 1 splitters (64-bit
// key prefixes = the first word of the key) taken from a sorted, evenly
// spaced sample (8 per splitter) cut it into 2S - 1 slots: range slots between
// splitters, and one slot per splitter for keys whose prefix equals it
// (repeated words land there and need no sorting; a slot whose keys differ
// past the prefix is sorted like a range slot). Keys are scattered to their
// slot (positions reserved per CTA, order inside a slot arbitrary) and every
// slot is then sorted on chip by the tile network. Slots beyond a tile (rare:
// the sample bounds them to ~0.4 T on average) fall back to an odd-even
// transposition sort over half-tile blocks, done by the slot's CTA.

constexpr int kSampleThreads = 1024;
constexpr int kPartThreads = 256;
constexpr int kPartPer = 8;
constexpr int kPartTile = kPartThreads * kPartPer;

__device__ __forceinline__ const SampleSeg& sseg_at(const SampleLaunch& a, int i) {
  return a.segs ? a.segs[i] : a.inl[i];
}

// Slot of a key among nsplit sorted full-key splitters: 2j for keys strictly
// between splitters j-1 and j, 2j + 1 for a key equal to splitter j. `sp`
// holds the splitters' first words (shared memory), `spk` the full splitters
// (global, NW words each). The first-word search decides almost every key;
// only a key whose first word equals a splitter's loads its remaining words
// and searches the splitters sharing that word on them.
// Multi-word keys with the full splitters in shared memory (the count pass):
// one lower-bound search on full keys, then the equality test.
template <int LANES>
__device__ __forceinline__ uint32_t slot_of_full(const Key<LANES>* sps, uint32_t nsplit, const Key<LANES>& k) {
  uint32_t lo = 0, len = nsplit;  // first splitter >= k
  while (len > 0) {
    const uint32_t half = len >> 1, mid = lo + half;
    const bool less = key_lt<LANES>(sps[mid], k);
    lo = less ? mid + 1 : lo;
    len = less ? len - half - 1 : half;
  }
  const bool eq = lo < nsplit && !key_lt<LANES>(k, sps[lo]);
  return 2 * lo + (eq ? 1u : 0u);
}

template <int LANES>
__device__ __forceinline__ uint32_t slot_of(const uint64_t* sp, const uint64_t* __restrict__ spk,
                                            uint32_t nsplit, uint64_t p,
                                            const KW<LANES>* __restrict__ in, uint64_t i) {
  uint32_t lo = 0, len = nsplit;  // lower bound: first splitter with first word >= p
  while (len > 0) {
    const uint32_t half = len >> 1, mid = lo + half;
    const bool less = sp[mid] < p;
    lo = less ? mid + 1 : lo;
    len = less ? len - half - 1 : half;
  }
  if (lo >= nsplit || sp[lo] != p) return 2 * lo;
  constexpr int NW = KeyTraits<LANES>::NW;
  if constexpr (NW == 1) {
    return 2 * lo + 1;
  } else {
    uint32_t hi = lo + 1, l2 = nsplit - hi;  // first splitter with first word > p
    while (l2 > 0) {
      const uint32_t half = l2 >> 1, mid = hi + half;
      const bool le = sp[mid] <= p;
      hi = le ? mid + 1 : hi;
      l2 = le ? l2 - half - 1 : half;
    }
    const Key<LANES> k = gld<LANES>(in, (int64_t)i);
    uint32_t a = lo, l3 = hi - lo;  // first splitter in [lo, hi) >= k
    while (l3 > 0) {
      const uint32_t half = l3 >> 1, mid = a + half;
      const bool less = key_lt<LANES>(gld<LANES>(reinterpret_cast<const KW<LANES>*>(spk), mid), k);
      a = less ? mid + 1 : a;
      l3 = less ? l3 - half - 1 : half;
    }
    const bool eq = a < hi && !key_lt<LANES>(k, gld<LANES>(reinterpret_cast<const KW<LANES>*>(spk), a));
    return 2 * a + (eq ? 1u : 0u);
  }
}

// One CTA per bucket: the full keys of an evenly spaced sample (padded with
// all-ones to 4096) -> bitonic sort -> the nsplit splitters, full keys too, so
// keys that share their first word (timestamps, IDs, URLs) are split like any
// others. Element i = 128 w + 32 q + lane lives in register set q of lane
// `lane` of warp w, so strides below 32 are shuffles, 32 and 64 are register
// swaps, and only strides of 128 and more (15 of the 78 stages) go through
// shared memory (kBitonicN keys of the class's width, dynamic).
constexpr int kBitonicN = 4096;
static_assert(kBitonicN == kSampleThreads * 4, "4 keys per thread");

template <int LANES>
constexpr size_t split_smem_bytes() { return (size_t)kBitonicN * key_bytes(LANES); }

// The splitters of one bucket (all threads of a 1024-thread CTA); also zeroes
// the bucket's slot counters for the count pass.
template <int LANES>
__device__ __forceinline__ void split_bucket(const SampleSeg& sg, uint64_t* __restrict__ splitters,
                                             uint32_t* __restrict__ hist, Key<LANES>* sm) {
  for (uint32_t i = threadIdx.x; i < 2 * sg.nsplit + 1; i += kSampleThreads)
    hist[sg.slot_base + i] = 0;  // the bucket's slot counters (the count pass follows)
  if (!sg.nsplit) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const KW<LANES>* in = kv<LANES>(sg.in);
  constexpr int NW = KeyTraits<LANES>::NW;
  Key<LANES> x[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t i = w * 128 + q * 32 + lane;
    x[q] = i < sg.m ? gld<LANES>(in, (int64_t)((uint64_t)i * sg.n / sg.m)) : key_max<LANES>();
  }
  auto cas = [&](Key<LANES>& u, Key<LANES>& v, bool up) {  // ascending when up
    const bool sw = key_lt<LANES>(v, u) == up;
    const Key<LANES> a0 = u, b0 = v;
    u = sw ? b0 : a0;
    v = sw ? a0 : b0;
  };
  // only the first m (a power of two) keys are samples: the network's stages
  // up to size m sort them (the padding blocks are already sorted)
  const uint32_t P = sg.m < 2 ? 2u : (sg.m > kBitonicN ? (uint32_t)kBitonicN : sg.m);
  for (uint32_t size = 2; size <= P; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 128) {
#pragma unroll
        for (int q = 0; q < 4; ++q) sm[w * 128 + q * 32 + lane] = x[q];
        __syncthreads();
        for (uint32_t t = threadIdx.x; t < kBitonicN / 2; t += kSampleThreads) {
          const uint32_t i = 2 * t - (t & (stride - 1)), j = i + stride;
          Key<LANES> u = sm[i], v = sm[j];
          if (key_lt<LANES>(v, u) == ((i & size) == 0)) {
            sm[i] = v;
            sm[j] = u;
          }
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 4; ++q) x[q] = sm[w * 128 + q * 32 + lane];
      } else if (stride >= 32) {  // partner in another register set of the same lane
        if (stride == 64) {
          cas(x[0], x[2], ((uint32_t)(w * 128 + lane) & size) == 0);
          cas(x[1], x[3], ((uint32_t)(w * 128 + 32 + lane) & size) == 0);
        } else {
          cas(x[0], x[1], ((uint32_t)(w * 128 + lane) & size) == 0);
          cas(x[2], x[3], ((uint32_t)(w * 128 + 64 + lane) & size) == 0);
        }
      } else {  // partner in another lane of the warp
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t i = w * 128 + q * 32 + lane;
          const bool up = (i & size) == 0, lower = (lane & stride) == 0;
          Key<LANES> y;
#pragma unroll
          for (int l = 0; l < NW; ++l) y.w[l] = __shfl_xor_sync(0xffffffffu, x[q].w[l], (int)stride);
          const bool lt = key_lt<LANES>(x[q], y);
          const bool keep = (lower == up) == lt;  // lower==up wants the smaller one
          x[q] = keep ? x[q] : y;
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) sm[w * 128 + q * 32 + lane] = x[q];
  __syncthreads();
  uint64_t* sp = splitters + (uint64_t)sg.split_off * NW;
  for (uint32_t k = threadIdx.x; k < sg.nsplit; k += kSampleThreads) {
    const Key<LANES> v = sm[(uint64_t)(k + 1) * sg.m / (sg.nsplit + 1)];
#pragma unroll
    for (int l = 0; l < NW; ++l) sp[(uint64_t)k * NW + l] = (uint64_t)v.w[l];
  }
}


template <int LANES>
__global__ void __launch_bounds__(kSampleThreads) sample_split_kernel(const __grid_constant__ SampleLaunch a) {
  pdl_wait();
  extern __shared__ __align__(16) uint64_t dsm[];
  split_bucket<LANES>(sseg_at(a, blockIdx.x), a.splitters, a.hist, reinterpret_cast<Key<LANES>*>(dsm));
}

// The split launch planned on the device from the ingest's per-length counts
// (sample_plan, the host's rule; buckets beyond the splitter budget are left
// to the merge path), so it runs while the host reads the counts back. CTA b:
// length lmin + b.
template <int LANES>
__global__ void __launch_bounds__(kSampleThreads) sample_split_early_kernel(const __grid_constant__ SplitEarly e) {
  extern __shared__ __align__(16) uint64_t dsm[];
  if (e.go && !*e.go) return;  // the class's words are being counted instead (dedupe.cu)
  SampleSeg sg;
  memset(&sg, 0, sizeof sg);
  uint32_t slots = 0, splits = 0, tiles = 0, key_off = 0, nfit = 0;
  int idx = -1;
  for (int L = e.lmin; L <= e.lmax; ++L) {
    const uint32_t n = e.fill[L - 1];
    const uint32_t koff = key_off;
    key_off += n;  // class-relative element offset (plan_packed: every bucket of the class)
    if (!n || n > e.cap) continue;
    const SamplePlan pl = sample_plan(n, e.T, e.pmax, e.smax);
    if (L == e.lmin + (int)blockIdx.x) {
      sg.in = reinterpret_cast<const uint64_t*>(e.keys_cap + e.region[L - 1]);
      sg.key_off = koff;
      sg.n = n;
      sg.nsplit = pl.nsplit;
      sg.m = pl.m;
      sg.split_off = splits;
      sg.slot_base = slots;
      sg.tile_begin = tiles;
      sg.len = (uint32_t)L;
      idx = (int)nfit;
    }
    slots += 2 * pl.nsplit + 1;
    splits += pl.nsplit;
    tiles += e.ptile ? (n + e.ptile - 1) / e.ptile : 0u;
    ++nfit;
  }
  if (e.plan && threadIdx.x == 0) {  // the early count pass's launch (sample_sort_segments' plan)
    if (idx >= 0) e.plan->inl[idx] = sg;
    if (blockIdx.x == 0) {
      e.plan->segs = nullptr;
      e.plan->nsegs = (int)nfit;
      e.plan->nslots = slots;
      e.plan->work_items = tiles;
      e.plan->splitters = e.splitters;
      e.plan->hist = e.hist;
      e.plan->slot_ids = e.slot_ids;
      e.plan->split_done = 1;
    }
  }
  if (idx >= 0) split_bucket<LANES>(sg, e.splitters, e.hist, reinterpret_cast<Key<LANES>*>(dsm));
}

__device__ __forceinline__ int part_segment_of(const SampleLaunch& a, uint32_t tile) {
  const int lane = threadIdx.x & 31;
  int found = 0;
  for (int base = 0; base < a.nsegs; base += 32) {
    const int i = base + lane;
    const bool le = i < a.nsegs && sseg_at(a, i).tile_begin <= tile;
    found += __popc(__ballot_sync(0xffffffffu, le));
    if (!__shfl_sync(0xffffffffu, (int)le, 31)) break;
  }
  return found - 1;
}

// Partition passes over one tile of a bucket. COUNT: per-slot counts into
// a.hist. !COUNT: each key goes to cursor[slot] reservation + local rank.
// One partition tile `item` (all threads of the CTA; the CTA's shared memory
// is free again on return).
template <int LANES, bool COUNT>
__device__ __forceinline__ void partition_tile(const SampleLaunch& a, uint32_t item) {
  using W = KW<LANES>;
  constexpr int NW = KeyTraits<LANES>::NW;
  constexpr bool FULL = COUNT && NW >= 2;  // full splitters in smem, full keys loaded
  __shared__ uint64_t s_split[FULL ? 1 : kMaxSplit];
  __shared__ Key<(FULL ? LANES : 1)> s_spk[FULL ? kMaxSplit : 1];
  __shared__ uint32_t s_cnt[2 * kMaxSplit + 1];
  __shared__ uint32_t s_base[2 * kMaxSplit + 1];
  __shared__ int s_seg;
  const int tid = threadIdx.x;
  if (tid < 32) {
    const int sgi = part_segment_of(a, item);
    if (tid == 0) s_seg = sgi;
  }
  __syncthreads();
  const SampleSeg& sg = sseg_at(a, s_seg);
  const uint32_t nslot = 2 * sg.nsplit + 1;
  if (COUNT && !FULL)  // the scatter pass reads the slots the count pass found
    for (uint32_t i = tid; i < sg.nsplit; i += kPartThreads)
      s_split[i] = a.splitters[((uint64_t)sg.split_off + i) * NW];
  if constexpr (FULL) {
    uint64_t* d = reinterpret_cast<uint64_t*>(&s_spk[0]);
    for (uint32_t i = tid; i < sg.nsplit * NW; i += kPartThreads)
      d[i] = a.splitters[(uint64_t)sg.split_off * NW + i];
  }
  for (uint32_t i = tid; i < nslot; i += kPartThreads) s_cnt[i] = 0;
  __syncthreads();
  const uint64_t first = (uint64_t)(item - sg.tile_begin) * kPartTile;
  const W* in = kv<LANES>(sg.in);
  uint16_t* ids = a.slot_ids + (uint64_t)item * kPartTile;
  Key<LANES> k[kPartPer];
  uint32_t slot[kPartPer], rank[kPartPer];
#pragma unroll
  for (int q = 0; q < kPartPer; ++q) {  // every load in flight before the first search
    const uint64_t i = first + (uint64_t)q * kPartThreads + tid;
    if (i < sg.n) {
      if (COUNT && !FULL) {
        k[q].w[0] = __ldg(in + i * KeyTraits<LANES>::NW);  // the 64-bit prefix is all it needs
        slot[q] = 0;
      } else if (COUNT) {
        k[q] = gld<LANES>(in, (int64_t)i);
        slot[q] = 0;
      } else {
        k[q] = gld<LANES>(in, (int64_t)i);
        slot[q] = ids[q * kPartThreads + tid];
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kPartPer; ++q) {
    const uint64_t i = first + (uint64_t)q * kPartThreads + tid;
    if (i < sg.n) {
      if (COUNT) {
        if constexpr (FULL)
          slot[q] = slot_of_full<(FULL ? LANES : 1)>(s_spk, sg.nsplit, k[q]);
        else
          slot[q] = slot_of<LANES>(s_split, a.splitters + (uint64_t)sg.split_off * KeyTraits<LANES>::NW,
                                   sg.nsplit, (uint64_t)k[q].w[0], in, i);
        ids[q * kPartThreads + tid] = (uint16_t)slot[q];
      }
      rank[q] = atomicAdd(&s_cnt[slot[q]], 1u);
    } else {
      slot[q] = 0xFFFFFFFFu;
    }
  }
  __syncthreads();
  if (COUNT) {
    for (uint32_t i = tid; i < nslot; i += kPartThreads)
      if (s_cnt[i]) atomicAdd(a.hist + sg.slot_base + i, s_cnt[i]);
    return;
  }
  for (uint32_t i = tid; i < nslot; i += kPartThreads)
    if (s_cnt[i]) s_base[i] = atomicAdd(a.cursor + sg.slot_base + i, s_cnt[i]);
  __syncthreads();
  W* out = kv<LANES>(a.keys_out);
#pragma unroll
  for (int q = 0; q < kPartPer; ++q)
    if (slot[q] != 0xFFFFFFFFu) {
      WS_DCHECK(slot[q] < nslot && s_base[slot[q]] + rank[q] >= sg.key_off &&
                s_base[slot[q]] + rank[q] < sg.key_off + sg.n);
      stk<LANES>(out, (int)(s_base[slot[q]] + rank[q]), k[q]);
    }
}

#ifndef WS_PART_MINB
#define WS_PART_MINB 1
#endif
template <int LANES, bool COUNT>
__global__ void __launch_bounds__(kPartThreads, WS_PART_MINB) partition_kernel(const __grid_constant__ SampleLaunch a) {
  pdl_wait();
  partition_tile<LANES, COUNT>(a, blockIdx.x);
}

// The count pass launched by the ingest right behind the class's split launch,
// from the launch the split CTAs wrote (device-planned, same rules as the host
// plan): a persistent grid over the class's partition tiles.
template <int LANES>
__global__ void __launch_bounds__(kPartThreads, 2) partition_count_early_kernel(const SampleLaunch* __restrict__ plan, const uint32_t* __restrict__ go) {
  pdl_wait();
  if (go && !*go) return;  // no split launch wrote `plan` for this call (dedupe.cu)
  const SampleLaunch& a = *plan;
  const uint32_t items = a.work_items;
  for (uint32_t item = blockIdx.x; item < items; item += gridDim.x) {
    partition_tile<LANES, true>(a, item);
    __syncthreads();  // the tile's shared memory is reused by the next one
  }
}

// Exclusive scan of each bucket's slot counts (one CTA per bucket), started
// at the bucket's class-relative key offset: the slot offsets, valid for any
// subset of a class's buckets.
__global__ void __launch_bounds__(1024) slot_scan_kernel(const __grid_constant__ SampleLaunch a) {
  pdl_wait();
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_carry;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const SampleSeg& sg = sseg_at(a, blockIdx.x);
  const uint32_t nslot = 2 * sg.nsplit + 1;
  if (tid == 0) s_carry = sg.key_off;
  __syncthreads();
  for (uint32_t base = 0; base < nslot; base += 1024) {
    const uint32_t i = base + tid;
    const uint32_t v = i < nslot ? a.hist[sg.slot_base + i] : 0u;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    if (lane == 31) s_w[wid] = inc;
    __syncthreads();
    uint32_t pre = s_carry;
    for (int w = 0; w < wid; ++w) pre += s_w[w];
    if (i < nslot) {
      a.slot_off[sg.slot_base + i] = pre + inc - v;
      a.cursor[sg.slot_base + i] = pre + inc - v;
    }
    __syncthreads();
    if (tid == 1023) s_carry = pre + inc;
    __syncthreads();
  }
}

// One 128-thread CTA per slot: the slot is sorted in place by the tile
// network of a slot-sort tile (slots average half of it), or - beyond it, rare
// - by an in-CTA merge sort. A key-equal slot (copies of one word) is left as
// it is (payload: filled with the record pattern).
constexpr int kSubThreads = 128;
#ifndef WS_SUB_DB
#define WS_SUB_DB 0  // 1: slot sorts with double-buffered merge levels, one barrier per level (measured slower: 189 vs 162 us, smem occupancy)
#endif

// Fused emission (SampleSeg::pay set: 6-bit text keys, payload mode): the
// slot's sorted keys leave as payload records at their final place
// (pay + rank in bucket * (L + 1)) instead of going back to the key buffer,
// so no emit pass re-reads them; a slot of one repeated word is filled with
// the record pattern. Staging buffer after the keys in dynamic smem.
constexpr int kSubPayBuf = kSubThreads * (kMaxPackedLen + 1) + 64;

template <int LANES>
__device__ __forceinline__ void sub_emit(const KW<LANES>* keys, uint32_t cnt, int L, uint8_t* out,
                                         uint8_t* pbuf) {
  if constexpr (LANES <= 3) emit_records_cta<LANES, kSubThreads>(keys, cnt, L, out, pbuf);
}

template <int LANES>
#ifndef WS_SUB_MINB
#define WS_SUB_MINB 6  // CTAs per SM the multi-word slot sorts are compiled for (80 registers;
                       // 1: up to 128, 4 % slower)
#endif
#ifndef WS_SUB1_MINB
#define WS_SUB1_MINB 7  // one-word keys: 72 registers (1: 109, slot sort 63 -> 43 us at 7)
#endif
__global__ void __launch_bounds__(kSubThreads, LANES <= 1 ? WS_SUB1_MINB : WS_SUB_MINB) subsort_kernel(const __grid_constant__ SampleLaunch a) {
  pdl_wait();
  constexpr int E = TileCfg<LANES>::E, NT = kSubThreads, TS = NT * E;
  constexpr int NW = KeyTraits<LANES>::NW;
  using W = KW<LANES>;
  extern __shared__ __align__(16) uint64_t smem[];
  W* sk = reinterpret_cast<W*>(smem);
  uint8_t* pbuf = reinterpret_cast<uint8_t*>(smem) + keys_smem_bytes<LANES, TS, false>();
  W* sk2 = reinterpret_cast<W*>(pbuf + kSubPayBuf);  // second key buffer (WS_SUB_DB)
  const uint32_t s = blockIdx.x;
  const uint32_t cnt = a.hist[s];
  if (cnt == 0) return;
  int b = 0;  // bucket of the slot (segments ascend by slot_base)
  while (b + 1 < a.nsegs && sseg_at(a, b + 1).slot_base <= s) ++b;
  const SampleSeg& sg = sseg_at(a, b);
  W* base = kv<LANES>(a.keys_out) + (uint64_t)a.slot_off[s] * NW;
  WS_DCHECK(a.slot_off[s] >= sg.key_off && a.slot_off[s] + cnt <= sg.key_off + sg.n);
  const int L = (int)sg.len;
  uint8_t* const out = (LANES <= 3 && sg.pay) ? sg.pay + (uint64_t)(a.slot_off[s] - sg.key_off) * (L + 1) : nullptr;
  if (cnt < 2) {
    if (out) sub_emit<LANES>(base, cnt, L, out, pbuf);
    return;
  }
  if (((s - sg.slot_base) & 1u) != 0) {  // key-equal slot: copies of one word (full-key splitters)
    if constexpr (LANES <= 3)
      if (out) fill_records_cta<LANES, NT>(ldk<LANES>(base, 0), cnt, L, out, pbuf);
    return;
  }
  Key<LANES> r[E];
  uint32_t ri[E];
  uint64_t inv = 0;
  // c <= TS keys at g sorted on chip, written to d (may be g), or emitted
  auto sort_span = [&](const W* g, uint32_t c, W* d, bool emit) {
    constexpr int PW = E * NW;  // words per thread: all loads in flight, then the stores
    W v[PW];
#pragma unroll
    for (int q = 0; q < PW; ++q) {
      const uint32_t j = threadIdx.x + q * NT;
      v[q] = j < c * NW ? g[j] : ~W(0);
    }
#pragma unroll
    for (int q = 0; q < PW; ++q) sk[threadIdx.x + q * NT] = v[q];
    __syncthreads();
    tile_network<LANES, false, NT>(sk, nullptr, (int)c, 0u, r, ri, inv, WS_SUB_DB ? sk2 : nullptr);
    __syncthreads();
    regs_to_smem<LANES, E, false>(sk, nullptr, threadIdx.x * E, r, ri);
    __syncthreads();
    if (emit) {  // the whole slot is in sk: records straight out
      sub_emit<LANES>(sk, c, L, out, pbuf);
      return;
    }
    for (uint32_t j = threadIdx.x; j < c * NW; j += NT) d[j] = sk[j];
    __syncthreads();
  };
  if (cnt <= (uint32_t)TS) {
    sort_span(base, cnt, base, out != nullptr);
    return;
  }
  // A slot beyond one tile (sampling variance, or a sample that misses the
  // bucket's spread): merge sort in O(cnt log cnt) by this CTA. Tiles of TS
  // keys are sorted on chip, then merge-path levels ping-pong between the
  // slot and its scratch: the slot's range in a third buffer (a.scratch; not
  // the input keys, which a later ws_sort of the same ingest reads again). The
  // block pass writes to the side that
  // makes the last level land in the slot.
  W* const scratch = kv<LANES>(a.scratch) + (uint64_t)a.slot_off[s] * NW;
  const uint32_t blocks = (cnt + TS - 1) / TS;
  int levels = 0;
  while ((1u << levels) < blocks) ++levels;
  W* cur = (levels & 1) ? scratch : base;
  for (uint32_t bk = 0; bk < blocks; ++bk) {
    const uint32_t lo = bk * TS;
    sort_span(base + (uint64_t)lo * NW, min((uint32_t)TS, cnt - lo), cur + (uint64_t)lo * NW, false);
  }
  __shared__ int64_t s_split;
  for (uint32_t run = TS; run < cnt; run <<= 1) {
    W* const nxt = cur == base ? scratch : base;
    for (uint32_t p0 = 0; p0 < cnt; p0 += 2 * run) {
      const W* A = cur + (uint64_t)p0 * NW;
      const uint32_t na = min(run, cnt - p0);
      const uint32_t nb = cnt - p0 > run ? min(run, cnt - p0 - run) : 0u;
      const W* B = A + (uint64_t)na * NW;
      int64_t a0 = 0;
      for (uint32_t d0 = 0; d0 < na + nb; d0 += TS) {  // one output tile of TS keys per step
        const uint32_t d1 = min(d0 + (uint32_t)TS, na + nb);
        if (threadIdx.x < 32) {
          const int64_t a1 = d1 == na + nb ? (int64_t)na
                                           : merge_path_search_global<LANES>(A, na, B, nb, d1);
          if (threadIdx.x == 0) s_split = a1;
        }
        __syncthreads();
        const int64_t a1 = s_split;
        const int la = (int)(a1 - a0), lb = (int)((d1 - a1) - (d0 - a0));
        WS_DCHECK(la >= 0 && lb >= 0 && la + lb <= TS && a1 <= (int64_t)na && d1 - a1 <= nb);
        const W* Ag = A + (uint64_t)a0 * NW;
        const W* Bg = B + (uint64_t)(d0 - a0) * NW;
        for (int j = threadIdx.x; j < la * NW; j += NT) sk[j] = Ag[j];
        for (int j = threadIdx.x; j < lb * NW; j += NT) sk[la * NW + j] = Bg[j];
        __syncthreads();
        merge_path<LANES, E, false>(sk, la, sk + (size_t)la * NW, lb, nullptr, nullptr,
                                    min((int)threadIdx.x * E, la + lb), 0, r, ri, inv);
        __syncthreads();
        if ((int)threadIdx.x * E < la + lb) regs_to_smem<LANES, E, false>(sk, nullptr, threadIdx.x * E, r, ri);
        __syncthreads();
        W* o = nxt + (uint64_t)(p0 + d0) * NW;
        for (int j = threadIdx.x; j < (la + lb) * NW; j += NT) o[j] = sk[j];
        __syncthreads();
        a0 = a1;
      }
    }
    cur = nxt;
  }
  if (out) sub_emit<LANES>(base, cnt, L, out, pbuf);  // the merges' stores are visible to the CTA
}

// ---- small corpora: one CTA per bucket, straight after the ingest ------------------
//
// For a small text (ws_sort_text / ws_sort_resident / batches: payload mode)
// the per-class chains cost more in launches and in the host's read-back of
// the length histogram than in work. This launch goes in right behind the
// ingest, before that read-back: CTA b takes the bucket of length b + 1 from
// the ingest's fill counters, sorts it on chip with the tile network of a
// 1024-thread CTA (OETS in registers + merge-path levels in shared memory, up
// to 15360 one-word / 7168 multi-word keys) and writes its payload records at
// the bucket's output offset (the prefix over shorter buckets of count * (L +
// 1), also from the counters). A bucket beyond that, or any word longer than
// 32, raises *flag and the call continues down the class chains (the keys are
// only read here).
#ifndef WS_TINY_NT
#define WS_TINY_NT 1024
#endif
constexpr int kTinyThreads = WS_TINY_NT;

template <int LANES>
constexpr size_t tiny_smem_lanes() {
  return (size_t)kTinyThreads * TileCfg<LANES>::E * key_bytes(LANES) + 64 +
         (size_t)kTinyThreads * (kMaxPackedLen + 1) + 64;
}
constexpr size_t cmax(size_t a, size_t b) { return a > b ? a : b; }
constexpr size_t kTinyRadixSmem = (size_t)2 * kTinyThreads * TileCfg<1>::E * 4 + (kTinyThreads / 32) * 256 * 4 + 32 * 4 +
                                   (size_t)kTinyThreads * (kMaxPackedLen + 1) + 64;
constexpr size_t kTinySmem =
    cmax(cmax(kTinyRadixSmem, tiny_smem_lanes<1>()), cmax(tiny_smem_lanes<2>(), tiny_smem_lanes<3>()));

__device__ __forceinline__ void tiny_stamp(unsigned long long* st, int k) {
  if (st && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    st[k] = t;
  }
}

// The bucket's keys (16-byte aligned region start) into shared memory with one
// bulk copy (up to 12 bytes past the bucket are read: still inside its region).
__device__ __forceinline__ void tiny_load(void* dst, const void* src, uint32_t bytes) {
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b16 = (bytes + 15) & ~15u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, b16);
    tma_load_1d(dst, src, b16, &bar);
  }
  __syncthreads();
  mbar_wait(&bar, 0);
}

template <int LANES>
__device__ __forceinline__ void tiny_bucket(const KW<LANES>* __restrict__ in, uint32_t n, int L,
                                            uint8_t* __restrict__ out, uint64_t* smem,
                                            unsigned long long* st = nullptr) {
  constexpr int E = TileCfg<LANES>::E, NT = kTinyThreads, T = NT * E;
  constexpr int NW = KeyTraits<LANES>::NW;
  using W = KW<LANES>;
  W* sk = reinterpret_cast<W*>(smem);
  uint8_t* pbuf = reinterpret_cast<uint8_t*>(smem) + (size_t)T * key_bytes(LANES) + 64;
  tiny_load(sk, in, n * (uint32_t)key_bytes(LANES));
  for (uint32_t j = n * NW + threadIdx.x; j < (uint32_t)(T * NW); j += NT) sk[j] = ~W(0);
  __syncthreads();
  tiny_stamp(st, 2);
  Key<LANES> r[E];
  uint32_t ri[E];
  uint64_t inv = 0;
  tile_network<LANES, false, NT>(sk, nullptr, (int)n, 0u, r, ri, inv);
  __syncthreads();
  regs_to_smem<LANES, E, false>(sk, nullptr, threadIdx.x * E, r, ri);
  __syncthreads();
  tiny_stamp(st, 3);
  emit_records_cta<LANES, NT>(sk, n, L, out, pbuf);
  tiny_stamp(st, 15);
}

// One-word (6-bit, L <= 5) buckets: stable LSD radix over the key's 6L bits
// in shared memory, 8-bit digits (1-4 passes). Warp w ranks a contiguous
// slice of the bucket in rounds of 32 keys (one MATCH.ANY per round against
// its digit counters); a CTA-wide scan over (digit, warp) gives every key's
// place. The comparison network of tiny_bucket took 40 us for config 0's 7.6k
// three-character words.
#ifndef WS_TINY_BALLOT
#define WS_TINY_BALLOT 1  // digit peers by 8 ballots (fixed cost) instead of MATCH.ANY
#endif
__device__ __forceinline__ uint32_t tiny_peers8(uint32_t d, bool ok) {
#if WS_TINY_BALLOT
  uint32_t peers = __ballot_sync(0xffffffffu, ok);
  if (!ok) peers = 0u;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const uint32_t bit = (d >> b) & 1u;
    peers &= __ballot_sync(0xffffffffu, bit) ^ (bit - 1u);
  }
  return ok ? peers : (1u << (threadIdx.x & 31));
#else
  return __match_any_sync(0xffffffffu, ok ? d : 256u + (threadIdx.x & 31));
#endif
}

// Records of sorted one-word 6-bit keys straight from registers: thread j
// writes record j (<= 5 characters + '\n') with the fewest aligned stores.
__device__ __forceinline__ void tiny_emit0(const uint32_t* keys, uint32_t n, int L, uint8_t* out) {
  const uint32_t R = (uint32_t)L + 1;
  for (uint32_t j = threadIdx.x; j < n; j += kTinyThreads) {
    const uint32_t k = keys[j];
    uint64_t rec = (uint64_t)'\n' << (8 * L);
#pragma unroll
    for (int c = 0; c < 5; ++c)
      if (c < L) rec |= (uint64_t)alnum6_byte((k >> (26 - 6 * c)) & 63u) << (8 * c);
    uint8_t* dst = out + (uint64_t)j * R;
    uint32_t rem = R;
    if (((uintptr_t)dst & 1) != 0) { *dst = (uint8_t)rec; rec >>= 8; ++dst; --rem; }
    if (((uintptr_t)dst & 2) != 0 && rem >= 2) { *reinterpret_cast<uint16_t*>(dst) = (uint16_t)rec; rec >>= 16; dst += 2; rem -= 2; }
    if (rem >= 4) { *reinterpret_cast<uint32_t*>(dst) = (uint32_t)rec; rec >>= 32; dst += 4; rem -= 4; }
    if (rem >= 2) { *reinterpret_cast<uint16_t*>(dst) = (uint16_t)rec; rec >>= 16; dst += 2; rem -= 2; }
    if (rem) *dst = (uint8_t)rec;
  }
}

template <int NT>
__device__ __forceinline__ uint32_t cta_excl_scan(uint32_t v, uint32_t* s_w /*[32]*/) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t u = __shfl_up_sync(0xffffffffu, inc, d);
    if (lane >= d) inc += u;
  }
  if (lane == 31) s_w[w] = inc;
  __syncthreads();
  if (w == 0) {
    const uint32_t x = lane < NT / 32 ? s_w[lane] : 0u;
    uint32_t xi = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, xi, d);
      if (lane >= d) xi += u;
    }
    if (lane < NT / 32) s_w[lane] = xi - x;
  }
  __syncthreads();
  return s_w[w] + inc - v;
}


__device__ void tiny_radix0(const uint32_t* __restrict__ in, uint32_t n, int L, uint8_t* __restrict__ out,
                            uint64_t* smem, unsigned long long* st = nullptr) {
  constexpr int NT = kTinyThreads, NWARP = NT / 32, R = (NT * TileCfg<1>::E + NT - 1) / NT;  // rounds
  constexpr int TPD = NWARP / 8;  // threads per digit in the scan (8 warps' counters each)
  static_assert(NWARP % 8 == 0 && NWARP * 256 == NT * 8, "scan layout: 8 counters per thread");
  uint32_t* buf0 = reinterpret_cast<uint32_t*>(smem);
  uint32_t* buf1 = buf0 + NT * TileCfg<1>::E;
  uint32_t* wc = buf1 + NT * TileCfg<1>::E;       // [NWARP][256]
  uint32_t* s_w = wc + NWARP * 256;                 // [32]
  uint8_t* pbuf = reinterpret_cast<uint8_t*>(s_w + 32);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t lt = (1u << lane) - 1u;
  const uint32_t S = (n + NWARP - 1) / NWARP, s0 = min(n, w * S), s1 = min(n, s0 + S);
  tiny_load(buf0, in, n * 4u);
  tiny_stamp(st, 2);
  const int bits = 6 * L, passes = (bits + 7) / 8;
  uint32_t* a = buf0;
  uint32_t* b = buf1;
  for (int ps = 0; ps < passes; ++ps) {
    const int shift = 32 - bits + 8 * ps;
    for (int i = tid; i < NWARP * 256; i += NT) wc[i] = 0;
    __syncthreads();
    uint32_t rk[R], ky[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if ((uint32_t)(r * 32) >= S) break;  // uniform across the CTA
      const uint32_t j = s0 + r * 32 + lane;
      const bool ok = j < s1;
      ky[r] = ok ? a[j] : 0u;
      const uint32_t d = (ky[r] >> shift) & 255u;
      const uint32_t peers = tiny_peers8(d, ok);
      const uint32_t base = ok ? wc[w * 256 + d] : 0u;
      rk[r] = base + __popc(peers & lt);
      __syncwarp();
      if (ok && !(peers & lt)) wc[w * 256 + d] = base + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    tiny_stamp(st, 3 + 3 * ps);
    {  // exclusive offsets in (digit, warp) order: thread t = digit t / TPD, warps 8 (t % TPD) .. + 7
      const int d = tid / TPD, q = tid % TPD;
      uint32_t c[8], sum = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        c[k] = wc[(q * 8 + k) * 256 + d];
        sum += c[k];
      }
      uint32_t run = cta_excl_scan<NT>(sum, s_w);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        wc[(q * 8 + k) * 256 + d] = run;
        run += c[k];
      }
    }
    __syncthreads();
    tiny_stamp(st, 4 + 3 * ps);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if ((uint32_t)(r * 32) >= S) break;
      const uint32_t j = s0 + r * 32 + lane;
      if (j < s1) {
        const uint32_t at = wc[w * 256 + ((ky[r] >> shift) & 255u)] + rk[r];
        WS_DCHECK(at < n);
        b[at] = ky[r];
      }
    }
    __syncthreads();
    tiny_stamp(st, 5 + 3 * ps);
    uint32_t* t = a;
    a = b;
    b = t;
  }
  (void)pbuf;
  tiny_emit0(a, n, L, out);
  tiny_stamp(st, 15);
}

__global__ void __launch_bounds__(kTinyThreads, 1) tiny_sort_kernel(const __grid_constant__ TinyLaunch t) {
  pdl_wait();
  extern __shared__ __align__(16) uint64_t smem[];
  const int b = blockIdx.x;  // the bucket of length b + 1
  unsigned long long t0 = 0;
  if (t.prof && threadIdx.x == 0) asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  const uint32_t n = t.fill[b];
  const int L = b + 1, lanes = lanes_for_len_enc(L, kEncAlnum6);
  const uint32_t cap = (uint32_t)kTinyThreads * (lanes <= 1 ? TileCfg<1>::E : TileCfg<2>::E);
  if (t.fill[kLongBin] != 0 || n > cap) {  // (every CTA checks the long words: all buckets may be empty)
    if (threadIdx.x == 0) atomicOr(t.flag, 1u);
    return;
  }
  if (n == 0) return;
  uint64_t off = 0;
  for (int q = 0; q < b; ++q) off += (uint64_t)t.fill[q] * (uint64_t)(q + 2);
  WS_DCHECK(off + (uint64_t)n * (L + 1) <= t.out_cap);
  const uint8_t* keys = t.keys_cap + t.region[b];
  uint8_t* out = t.out + off;
  switch (lanes) {
    case 0: tiny_radix0(reinterpret_cast<const uint32_t*>(keys), n, L, out, smem, t.prof ? t.prof + 64 + 16 * b : nullptr); break;
    case 1: tiny_bucket<1>(reinterpret_cast<const KW<1>*>(keys), n, L, out, smem, t.prof ? t.prof + 64 + 16 * b : nullptr); break;
    case 2: tiny_bucket<2>(reinterpret_cast<const KW<2>*>(keys), n, L, out, smem, t.prof ? t.prof + 64 + 16 * b : nullptr); break;
    default: tiny_bucket<3>(reinterpret_cast<const KW<3>*>(keys), n, L, out, smem, t.prof ? t.prof + 64 + 16 * b : nullptr); break;
  }
  if (t.prof && threadIdx.x == 0) {
    unsigned long long t1;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t1));
    t.prof[2 * b] = t0;
    t.prof[2 * b + 1] = t1;
  }
}

void launch_tiny_sort(const TinyLaunch& t, cudaStream_t st) {
  launch_pdl(tiny_sort_kernel, kMaxPackedLen, kTinyThreads, kTinySmem, st, t);
}

// ---- host side ---------------------------------------------------------------------

// ---- distinct-word counting: tile sort of the distinct keys (dedupe.cu's chain) ----

constexpr int kDdSortThreads = kTileThreads;
template <int LANES>
constexpr size_t dd_sort_smem() { return pass_smem_bytes<LANES, kTileThreads * (LANES == 1 ? TileCfg<2>::E : TileCfg<LANES>::E), true>(); }
constexpr size_t kDdSortSmem = cmax(cmax(dd_sort_smem<0>(), dd_sort_smem<1>()), cmax(dd_sort_smem<2>(), dd_sort_smem<3>()));

// One tile of a counted bucket's distinct keys (as the aggregate launch
// appended them) sorted on chip by the tile network; each key's occurrences
// are fetched from its table slot and follow it (array B).
// Keys per thread of the distinct keys' tiles: the one-lane keys' buckets hold a
// few thousand distinct words each, so they take the narrow tile (half the
// on-chip sort's latency, 2-3 tiles to rank-merge); the uint32 keys' one large
// bucket keeps the wide tile (fewer tiles for its rank merge).
template <int LANES>
struct DdTileE {
  static constexpr int E = LANES == 1 ? TileCfg<2>::E : TileCfg<LANES>::E;
};

template <int LANES>
__device__ void dd_sort_tile(const DdDevPlan& p, const DdChain& c, int b, uint32_t tile, uint8_t* sbytes) {
  constexpr int E = DdTileE<LANES>::E, NT = kDdSortThreads, T = NT * E;
  constexpr int NW = KeyTraits<LANES>::NW;
  using W = KW<LANES>;
  W* sk = reinterpret_cast<W*>(sbytes);
  uint32_t* si = reinterpret_cast<uint32_t*>(sbytes + keys_smem_bytes<LANES, T, true>());
  const int tid = threadIdx.x;
  const uint32_t start = tile * T;
  const int cnt = (int)min((uint32_t)T, p.D[b] - start);
  const W* gin = reinterpret_cast<const W*>(c.dk + p.dk_off[b]) + (uint64_t)start * NW;
  for (int j = tid; j < T * NW; j += NT) sk[j] = j < cnt * NW ? gin[j] : ~W(0);
  __syncthreads();
  Key<LANES> r[E];
  uint32_t ri[E];
  uint64_t inv = 0;
  tile_network<LANES, true, NT, false, E>(sk, si, cnt, 0u, r, ri, inv);
  W* gout = reinterpret_cast<W*>(c.ts + p.dk_off[b]) + (uint64_t)start * NW;
  const uint32_t* dslot = c.aux + p.aux_off[b] + start;
  uint32_t* ocnt = c.aux + p.aux_total + p.aux_off[b] + start;
  const uint2* tab = c.table + p.tab_off[b];
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const int pos = tid * E + k;
    if (pos >= cnt) break;
    WS_DCHECK(ri[k] < (uint32_t)cnt);
#pragma unroll
    for (int l = 0; l < NW; ++l) gout[(uint64_t)pos * NW + l] = r[k].w[l];
    ocnt[pos] = tab[dslot[ri[k]]].y;
  }
  __syncthreads();  // the tile's shared memory is reused by the CTA's next tile
}

__global__ void __launch_bounds__(kDdSortThreads) dd_tile_sort_kernel(const __grid_constant__ DdChain c) {
  pdl_wait();
  extern __shared__ __align__(16) uint64_t smem[];
  uint8_t* sbytes = reinterpret_cast<uint8_t*>(smem);
  const DdDevPlan& p = *c.plan;
  const uint32_t total = p.st_begin[32];
  for (uint32_t g = blockIdx.x; g < total; g += gridDim.x) {
    const int b = __popc(__ballot_sync(0xffffffffu, p.st_begin[1 + (threadIdx.x & 31)] <= g));
    if (!((c.cls_mask >> lanes_for_len_enc(b + 1, kEncAlnum6)) & 1u)) continue;  // another chain's bucket
    const uint32_t tile = g - p.st_begin[b];
    switch (lanes_for_len_enc(b + 1, kEncAlnum6)) {
      case 0: dd_sort_tile<0>(p, c, b, tile, sbytes); break;
      case 1: dd_sort_tile<1>(p, c, b, tile, sbytes); break;
      case 2: dd_sort_tile<2>(p, c, b, tile, sbytes); break;
      default: dd_sort_tile<3>(p, c, b, tile, sbytes); break;
    }
  }
}

int dd_sort_tile_size(int lanes) { return lanes == 0 ? TileCfg<0>::T : TileCfg<2>::T; }

void launch_dd_tiles(const DdChain& c, int grid, cudaStream_t st) {
  launch_pdl(dd_tile_sort_kernel, grid, kDdSortThreads, kDdSortSmem, st, c);
}

template <int LANES>
static constexpr size_t subsort_smem_bytes() {
  return keys_smem_bytes<LANES, kSubThreads * TileCfg<LANES>::E, false>() * (WS_SUB_DB ? 2 : 1) + kSubPayBuf;
}

int tile_size(int lanes) {
  switch (lanes) {
    case 0: return TileCfg<0>::T;
    case 1: return TileCfg<1>::T;
    case 2: return TileCfg<2>::T;
    case 3: return TileCfg<3>::T;
    default: return TileCfg<4>::T;
  }
}

int merge_tile_size(int lanes) {
  switch (lanes) {
    case 0: return MergeCfg<0>::T;
    case 1: return MergeCfg<1>::T;
    case 2: return MergeCfg<2>::T;
    case 3: return MergeCfg<3>::T;
    default: return MergeCfg<4>::T;
  }
}

template <int LANES, bool STATS>
static void set_attrs_t() {
  if (!STATS && LANES >= 1) {
    constexpr int SL = LANES < 1 ? 1 : LANES;
    cudaFuncSetAttribute(sample_split_kernel<SL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)split_smem_bytes<SL>());
    cudaFuncSetAttribute(sample_split_early_kernel<SL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)split_smem_bytes<SL>());
    cudaFuncSetAttribute(subsort_kernel<LANES < 1 ? 1 : LANES>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)subsort_smem_bytes<(LANES < 1 ? 1 : LANES)>());
  }
  cudaFuncSetAttribute(tile_sort_kernel<LANES, STATS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)pass_smem_bytes<LANES, TileCfg<LANES>::T, STATS>());
  cudaFuncSetAttribute(merge_kernel<LANES, STATS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)pass_smem_bytes<LANES, MergeCfg<LANES>::T, STATS>());
}

// Opt every sort instantiation into > 48 KiB of dynamic shared memory on the
// current device (called once per device by the handle).
void set_sort_attributes() {
  cudaFuncSetAttribute(dd_tile_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDdSortSmem);
  cudaFuncSetAttribute(tiny_sort_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTinySmem);
  set_attrs_t<0, false>(); set_attrs_t<0, true>();
  set_attrs_t<1, false>(); set_attrs_t<1, true>();
  set_attrs_t<2, false>(); set_attrs_t<2, true>();
  set_attrs_t<3, false>(); set_attrs_t<3, true>();
  set_attrs_t<4, false>(); set_attrs_t<4, true>();
}

template <int LANES, bool STATS>
static void launch_tile_t(const SortLaunch& a, cudaStream_t st) {
  launch_pdl(tile_sort_kernel<LANES, STATS>, a.work_items, kTileThreads,
             pass_smem_bytes<LANES, TileCfg<LANES>::T, STATS>(), st, a);
}

template <int LANES, bool STATS>
static void launch_merge_t(const SortLaunch& a, cudaStream_t st, cudaEvent_t* ev) {
  // ev (profiling, or null): before the partition kernel, between, after the merge
  if (ev) cudaEventRecord(ev[0], st);
  if (!WS_MERGE_FUSED_SPLIT)
    launch_pdl(merge_split_kernel<LANES>, (a.work_items * 32 + 255) / 256, 256, 0, st, a);
  if (ev) cudaEventRecord(ev[1], st);
  launch_pdl(merge_kernel<LANES, STATS>, a.work_items, kMergeThreads,
             pass_smem_bytes<LANES, MergeCfg<LANES>::T, STATS>(), st, a);
  if (ev) cudaEventRecord(ev[2], st);
}

#define WS_DISPATCH_LANES(fn, lanes, stats, ...)                                    \
  do {                                                                              \
    switch (lanes) {                                                                \
      case 0: stats ? fn<0, true>(__VA_ARGS__) : fn<0, false>(__VA_ARGS__); break; \
      case 1: stats ? fn<1, true>(__VA_ARGS__) : fn<1, false>(__VA_ARGS__); break; \
      case 2: stats ? fn<2, true>(__VA_ARGS__) : fn<2, false>(__VA_ARGS__); break; \
      case 3: stats ? fn<3, true>(__VA_ARGS__) : fn<3, false>(__VA_ARGS__); break; \
      default: stats ? fn<4, true>(__VA_ARGS__) : fn<4, false>(__VA_ARGS__); break; \
    }                                                                               \
  } while (0)

void launch_tile_sort(int lanes, const SortLaunch& a, cudaStream_t st) {
  if (!a.work_items) return;
  const bool stats = a.idx_out != nullptr;
  WS_DISPATCH_LANES(launch_tile_t, lanes, stats, a, st);
}

template <int LANES>
static void launch_sample_t(const SampleLaunch& a, cudaStream_t st, cudaEvent_t* ev) {
  // every bucket's CTA zeroes its slot counters, sampled or not; the chain's
  // kernels launch as their predecessor exits (PDL; pdl_wait first). `ev`
  // (profiling): 10 events, a start / end pair per launch.
  auto mark = [&](int i) {  // end of launch i - 1 (ev[2i - 1]), start of launch i (ev[2i])
    if (!ev) return;
    if (i > 0) cudaEventRecord(ev[2 * i - 1], st);
    if (i < 5) cudaEventRecord(ev[2 * i], st);
  };
  mark(0);
  if (!a.split_done)
    launch_pdl(sample_split_kernel<LANES>, a.nsegs, kSampleThreads, split_smem_bytes<LANES>(), st, a);
  mark(1);
  if (!a.count_done) launch_pdl(partition_kernel<LANES, true>, a.work_items, kPartThreads, 0, st, a);
  mark(2);
  launch_pdl(slot_scan_kernel, a.nsegs, 1024, 0, st, a);
  mark(3);
  launch_pdl(partition_kernel<LANES, false>, a.work_items, kPartThreads, 0, st, a);
  mark(4);
  launch_pdl(subsort_kernel<LANES>, a.nslots, kSubThreads, subsort_smem_bytes<LANES>(), st, a);
  mark(5);
}

int sample_max_keys(int) { return kSampleSmem / 8; }
int part_tile_size() { return kPartTile; }
int subsort_tile_size(int lanes) { return kSubThreads * (lanes <= 1 ? TileCfg<1>::E : TileCfg<2>::E); }

void launch_partition_count_early(int lanes, const SampleLaunch* plan, int grid, cudaStream_t st,
                                  const uint32_t* go) {
  switch (lanes) {
    case 1: launch_pdl(partition_count_early_kernel<1>, grid, kPartThreads, 0, st, plan, go); break;
    case 2: launch_pdl(partition_count_early_kernel<2>, grid, kPartThreads, 0, st, plan, go); break;
    default: launch_pdl(partition_count_early_kernel<3>, grid, kPartThreads, 0, st, plan, go); break;
  }
}

void launch_sample_split_early(int lanes, const SplitEarly& e, cudaStream_t st) {
  const unsigned nb = (unsigned)(e.lmax - e.lmin + 1);
  switch (lanes) {
    case 1: sample_split_early_kernel<1><<<nb, kSampleThreads, split_smem_bytes<1>(), st>>>(e); break;
    case 2: sample_split_early_kernel<2><<<nb, kSampleThreads, split_smem_bytes<2>(), st>>>(e); break;
    case 3: sample_split_early_kernel<3><<<nb, kSampleThreads, split_smem_bytes<3>(), st>>>(e); break;
    default: sample_split_early_kernel<4><<<nb, kSampleThreads, split_smem_bytes<4>(), st>>>(e); break;
  }
}

void launch_sample_sort(int lanes, const SampleLaunch& a, cudaStream_t st, cudaEvent_t* ev) {
  switch (lanes) {
    case 1: launch_sample_t<1>(a, st, ev); break;
    case 2: launch_sample_t<2>(a, st, ev); break;
    case 3: launch_sample_t<3>(a, st, ev); break;
    default: launch_sample_t<4>(a, st, ev); break;
  }
}

int merge_launches_per_level() { return WS_MERGE_FUSED_SPLIT ? 1 : 2; }

void launch_merge(int lanes, const SortLaunch& a, cudaStream_t st, cudaEvent_t* ev) {
  if (!a.work_items) return;
  const bool stats = a.idx_out != nullptr;
  WS_DISPATCH_LANES(launch_merge_t, lanes, stats, a, st, ev);
}

WS_DEFINE_CHECK_READER(check_reader_sort)

}  // namespace ws
