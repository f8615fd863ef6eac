// Distinct-word counting: payload mode for texts that repeat their vocabulary.
//
// The reference sorts every occurrence of every word (engine.py:89-114) and
// prints them bucket by bucket (store.py:105-114, cli.py:97). The printed
// payload only depends on which words a bucket holds and how often, so when a
// bucket's distinct words are few (natural text: Zipf over a vocabulary) the
// device counts them, sorts the distinct keys only and writes every word as
// often as it occurred -- the same bytes as sorting all occurrences:
//
//   dd_aggregate_kernel<GRP>  (right behind the ingest, planned on the device
//       from its per-length counters; one launch for the uint32 keys, one for
//       the wider keys, side by side) reads every packed key once: a tile of
//       4096 keys is counted in a shared-memory table (slot = occurrences +
//       the index of one occurrence in the tile), the occupied slots are
//       compacted, and each distinct key of the tile goes into the bucket's
//       table in HBM/L2 (CAS on an empty slot, atomic add of the tile's
//       count). Words seen for the first time are appended to the bucket's
//       distinct-key list, one reservation per tile. A bucket whose distinct
//       words exceed its table's budget (plan.cuh: n/8) raises its overflow
//       flag; its class then keeps the sort paths (radix / sample sort). Each
//       launch's last CTA writes its classes' OK flags and the plan
//       (DdDevPlan) of the chain enqueued behind it -- no host round trip.
//   dd_tile_sort_kernel (sort.cu)  tiles of the distinct keys sorted on chip,
//       each key's occurrences fetched from its table slot
//   dd_rank_kernel    every key's final rank = its tile position + the smaller
//       keys of the bucket's other tiles (binary searches; no ties)
//   dd_prefix_kernel, dd_tsum_kernel  occurrences -> run starts (two levels)
//   dd_xstart_kernel  per output tile: the run holding its first record
//   dd_expand_dev_kernel  grid-stride over output tiles of ~16 KB: `word + '\n'`
//       records staged in shared memory and written with aligned 16-byte
//       stores (a run covering the whole tile is a pattern fill).
//
// Stats mode (SortStats needs corpus order) never takes this path.
#include <algorithm>

#include "payload.cuh"
#include "plan.cuh"
#include "ws_common.cuh"
#include "ws_kernels.h"

namespace ws {

namespace {

constexpr int kAggThreads = 512;
constexpr int kAggTile = 4096;    // keys per tile
constexpr int kProbeKeys = 1024;  // keys of a bucket's first tile the probe counts
constexpr int kAggSlotBits = 13;
constexpr int kAggSlots = 1 << kAggSlotBits;  // shared-memory table slots (load <= 1/2)
constexpr uint32_t kRepBits = 13; // slot = occurrences << 13 | (key index in tile + 1)
constexpr uint32_t kRepMask = (1u << kRepBits) - 1;
constexpr uint32_t kMaxProbes = 128;  // tables stay at most half full (longest expected probe sequence ~5 ln n there): longer means out of budget
static_assert(kAggTile < (1 << kRepBits), "tile index must fit the slot's low bits");

template <int LANES>
__device__ __forceinline__ Key<LANES> load_key(const void* base, uint64_t i) {
  using W = typename KeyTraits<LANES>::W;
  constexpr int NW = KeyTraits<LANES>::NW;
  Key<LANES> k;
  const W* p = reinterpret_cast<const W*>(base) + i * NW;
  if constexpr (LANES == 2) {
    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(p));
    k.w[0] = v.x;
    k.w[1] = v.y;
  } else {
#pragma unroll
    for (int q = 0; q < NW; ++q) k.w[q] = __ldg(p + q);
  }
  return k;
}

template <int LANES>
__device__ __forceinline__ void store_key(void* base, uint64_t i, const Key<LANES>& k) {
  using W = typename KeyTraits<LANES>::W;
  constexpr int NW = KeyTraits<LANES>::NW;
  W* p = reinterpret_cast<W*>(base) + i * NW;
#pragma unroll
  for (int q = 0; q < NW; ++q) p[q] = k.w[q];
}

template <int LANES>
__device__ __forceinline__ bool key_eq(const Key<LANES>& a, const Key<LANES>& b) {
  bool eq = a.w[0] == b.w[0];
#pragma unroll
  for (int q = 1; q < KeyTraits<LANES>::NW; ++q) eq = eq & (a.w[q] == b.w[q]);
  return eq;
}

__device__ __forceinline__ uint32_t hmix(uint32_t h, uint32_t v) {
  h = (h ^ v) * 0x85EBCA6Bu;
  return (h << 13) | (h >> 19);
}

// Hash whose HIGH bits are the good ones (the shared-memory slot is its top
// bits, the bucket-table slot a multiply-high): one-word keys by one odd
// multiply (Fibonacci hashing; the keys differ in their high bits, the low
// ones pad short words with zeros), wider keys word by word.
template <int LANES>
__device__ __forceinline__ uint32_t dd_hash(const Key<LANES>& k) {
  if constexpr (LANES == 0) {
    uint32_t h = (uint32_t)k.w[0] * 0x9E3779B1u;
    return h ^ (h >> 15) * 0x85EBCA6Bu;
  } else {
    uint32_t h = 0x9E3779B9u;
#pragma unroll
    for (int q = 0; q < KeyTraits<LANES>::NW; ++q) {
      h = hmix(h, (uint32_t)(k.w[q] >> 32));
      h = hmix(h, (uint32_t)k.w[q]);
    }
    h ^= h >> 16;
    h *= 0x85EBCA6Bu;
    h ^= h >> 13;
    h *= 0xC2B2AE35u;
    h ^= h >> 16;
    return h;
  }
}

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// One bucket as the aggregate / lookup kernels see it.
struct DdTab {
  const void* keys;   // the bucket's packed keys as the ingest left them
  uint2* tab;         // slots: x = representative key index + 1 (0: empty), y = occurrences
  uint32_t slots;
};

// `c` occurrences of key k (one of them at index p of the bucket) into the
// bucket's table: 0 = the word was there, 1 = first occurrence device-wide
// (its slot in *snew), -1 = the table is out of budget.
template <int LANES>
__device__ __forceinline__ int dd_insert(const DdTab& t, const Key<LANES>& k, uint32_t h,
                                         uint32_t p, uint32_t c, const uint32_t* ovf,
                                         uint32_t* snew) {
  uint32_t s = __umulhi(h, t.slots);
  // one-word keys (never zero: every 6-bit code is >= 1) sit in the slot
  // themselves; wider keys are named by the index of one occurrence
  const uint32_t mine = LANES == 0 ? (uint32_t)k.w[0] : p + 1;
  for (uint32_t probe = 0; probe < kMaxProbes; ++probe) {
    uint32_t r = ld_relaxed(&t.tab[s].x);
    if (r == 0) {
      r = atomicCAS(&t.tab[s].x, 0u, mine);
      if (r == 0) {
        atomicAdd(&t.tab[s].y, c);
        *snew = s;
        return 1;
      }
    }
    bool same;
    if constexpr (LANES == 0) same = r == mine;
    else same = key_eq<LANES>(load_key<LANES>(t.keys, r - 1), k);
    if (same) {
      atomicAdd(&t.tab[s].y, c);
      return 0;
    }
    if (++s == t.slots) s = 0;
    // a long probe sequence: the table is filling up because the bucket ran out of budget
    if ((probe & 7u) == 7u && ld_relaxed(ovf)) return -1;
  }
  return -1;
}

// Shared memory of one aggregate CTA.
constexpr int kAggWarps = kAggThreads / 32;
constexpr int kAggNewCap = 1024;  // new distinct words of a tile appended with one reservation
struct AggSmem {
  uint32_t tab[kAggSlots];
  uint16_t list[kAggTile];     // occupied slots, dense
  uint32_t new_s[kAggNewCap];  // words this tile saw first: their table slot ...
  uint16_t new_q[kAggNewCap];  // ... and their entry in list
  uint32_t wtot[kAggWarps];
  uint32_t nnew, dbase;
};

// One tile of a bucket: count in shared memory, then flush to the bucket's
// table. PROBE (dd_probe_kernel): only count the tile and judge it -- a full
// tile of mostly different words gives the bucket's lane class up (*probe).
// Diagnostics (-DWS_DD_PROF=1, tools only): time of each phase of a tile (clear,
// count, compaction, flush, append), summed over tiles per launch group, read
// by dd_prof_read.
#ifndef WS_DD_PROF
#define WS_DD_PROF 0
#endif
#if WS_DD_PROF
__device__ unsigned long long g_dd_prof[2][8];
#define WS_DD_STAMP(k)                                                          \
  do {                                                                          \
    if (!PROBE && threadIdx.x == 0) {                                           \
      unsigned long long now_;                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now_));                  \
      if ((k) > 0) atomicAdd(&g_dd_prof[LANES == 0 ? 0 : 1][k], now_ - t_prev_); \
      else atomicAdd(&g_dd_prof[LANES == 0 ? 0 : 1][7], 1ull);                  \
      t_prev_ = now_;                                                           \
    }                                                                           \
  } while (0)
#else
#define WS_DD_STAMP(k) do { } while (0)
#endif

template <int LANES, bool PROBE = false>
__device__ void agg_tile(const DdTab& t, uint32_t n, uint32_t base, AggSmem& sm, void* dk,
                         uint32_t* dslot, uint32_t dcap, uint32_t* dcount, uint32_t* ovf,
                         uint32_t* covf, uint32_t* probe = nullptr) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#if WS_DD_PROF
  unsigned long long t_prev_ = 0;
  if (tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_prev_));
  const unsigned long long t_first_ = t_prev_;
  (void)t_first_;
#endif
  uint32_t* tab = sm.tab;
  for (int i = tid; i < kAggSlots; i += kAggThreads) tab[i] = 0;
  if (tid == 0) sm.nnew = 0;
  __syncthreads();
  WS_DD_STAMP(0);
  // (the probe judges a bucket by its first kProbeKeys keys)
  const uint32_t cnt = min((uint32_t)(PROBE ? kProbeKeys : kAggTile), n - base);
  constexpr int E = (PROBE ? kProbeKeys : kAggTile) / kAggThreads;
  constexpr int G = LANES <= 1 ? E : (LANES == 2 ? 4 : 2);  // keys in flight per thread
#pragma unroll 1
  for (int e0 = 0; e0 < E; e0 += G) {
    Key<LANES> k[G];
#pragma unroll
    for (int e = 0; e < G; ++e) {
      const uint32_t idx = tid + (e0 + e) * kAggThreads;
      if (idx < cnt) k[e] = load_key<LANES>(t.keys, (uint64_t)base + idx);
    }
#pragma unroll
    for (int e = 0; e < G; ++e) {
      const uint32_t idx = tid + (e0 + e) * kAggThreads;
      if (idx >= cnt) continue;
      uint32_t s = dd_hash<LANES>(k[e]) >> (32 - kAggSlotBits);
      for (;;) {
        uint32_t v = *reinterpret_cast<volatile uint32_t*>(&tab[s]);
        if (v == 0) {
          v = atomicCAS(&tab[s], 0u, (1u << kRepBits) | (idx + 1));
          if (v == 0) break;
        }
        const uint32_t rep = (v & kRepMask) - 1;
        WS_DCHECK(rep < cnt);
        if (key_eq<LANES>(load_key<LANES>(t.keys, (uint64_t)base + rep), k[e])) {
          atomicAdd(&tab[s], 1u << kRepBits);
          break;
        }
        s = (s + 1) & (kAggSlots - 1);
      }
    }
  }
  __syncthreads();
  WS_DD_STAMP(1);
  // occupied slots -> a dense list (each warp owns a contiguous range of
  // slots: count, prefix over warps, place), so every thread flushes its share
  // of the tile's distinct keys (a thread's flushes are dependent L2 round trips)
  constexpr int PERW = kAggSlots / kAggWarps;  // slots per warp
  uint32_t mine = 0;
#pragma unroll 4
  for (int it = 0; it < PERW / 32; ++it)
    mine += __popc(__ballot_sync(0xffffffffu, tab[wid * PERW + it * 32 + lane] != 0));
  if (lane == 0) sm.wtot[wid] = mine;
  __syncthreads();
  uint32_t at = 0, nd = 0;
#pragma unroll
  for (int w = 0; w < kAggWarps; ++w) {
    const uint32_t v = sm.wtot[w];
    if (w < wid) at += v;
    nd += v;
  }
#pragma unroll 4
  for (int it = 0; it < PERW / 32; ++it) {
    const int i = wid * PERW + it * 32 + lane;
    const bool occ = tab[i] != 0;
    const uint32_t bal = __ballot_sync(0xffffffffu, occ);
    if (occ) sm.list[at + __popc(bal & ((1u << lane) - 1))] = (uint16_t)i;
    at += __popc(bal);
  }
  __syncthreads();
  WS_DD_STAMP(2);
  // A full tile of mostly different words: the bucket does not repeat its
  // vocabulary, counting it would cost more than sorting it. Give the bucket
  // (and with it its lane class) up now, before its table fills.
  if (cnt == (uint32_t)(PROBE ? kProbeKeys : kAggTile) && nd * 4u > cnt * 3u) {
    if (tid == 0) {
      atomicExch(ovf, 1u);
      atomicExch(covf, 1u);
      if (PROBE) atomicExch(probe, 1u);
    }
    __syncthreads();
    return;
  }
  if constexpr (PROBE) return;
  bool fail = false;
  for (uint32_t q = tid; q < nd; q += kAggThreads) {
    const uint32_t v = tab[sm.list[q]];
    const uint32_t rep = (v & kRepMask) - 1, c = v >> kRepBits;
    const Key<LANES> k = load_key<LANES>(t.keys, (uint64_t)base + rep);
    uint32_t snew = 0;
    const int st = dd_insert<LANES>(t, k, dd_hash<LANES>(k), base + rep, c, ovf, &snew);
    if (st < 0) {
      fail = true;
      break;
    }
    if (st > 0) {
      // the tile's new words are appended to the bucket's distinct-key list
      // with one reservation per tile (every bucket's counter is one address)
      const uint32_t np = atomicAdd(&sm.nnew, 1u);
      if (np < (uint32_t)kAggNewCap) {
        sm.new_s[np] = snew;
        sm.new_q[np] = (uint16_t)q;
      } else {  // more than the tile's list holds: one by one
        const uint32_t pos = atomicAdd(dcount, 1u);
        if (pos >= dcap) {
          fail = true;
          break;
        }
        store_key<LANES>(dk, pos, k);
        dslot[pos] = snew;
      }
    }
  }
  if (fail) {
    atomicExch(ovf, 1u);
    atomicExch(covf, 1u);
  }
  __syncthreads();
  WS_DD_STAMP(3);
  const uint32_t nn = min(sm.nnew, (uint32_t)kAggNewCap);
  if (nn) {
    if (tid == 0) sm.dbase = atomicAdd(dcount, nn);
    __syncthreads();
    const uint32_t db = sm.dbase;
    if (db + nn > dcap) {
      if (tid == 0) {
        atomicExch(ovf, 1u);
        atomicExch(covf, 1u);
      }
    } else {
      for (uint32_t i = tid; i < nn; i += kAggThreads) {
        const uint32_t v = tab[sm.list[sm.new_q[i]]];
        const Key<LANES> k = load_key<LANES>(t.keys, (uint64_t)base + (v & kRepMask) - 1);
        store_key<LANES>(dk, db + i, k);
        dslot[db + i] = sm.new_s[i];
      }
    }
  }
  __syncthreads();  // the shared memory is reused by the CTA's next tile
  WS_DD_STAMP(4);
}

__host__ __device__ inline int dd_class_of_len(int L) { return lanes_for_len_enc(L, kEncAlnum6); }
// Counting launch (and chain) of a lane class: 0 = the uint32 keys, 1 = the wider keys.
__host__ __device__ constexpr int dd_group_of_class(int cls) { return cls == 0 ? 0 : 1; }

struct KbOfLen {
  __host__ __device__ uint32_t operator()(int L) const { return (uint32_t)key_bytes(dd_class_of_len(L)); }
};

}  // namespace

void dd_host_layout(const uint32_t* n, DdLayout& o) { dd_layout(n, KbOfLen{}, o); }

// The chain's plan (DdDevPlan) from the per-length counts, the layout and the
// aggregate launch's control words; one warp, lane b = length b + 1.
__device__ void dd_write_plan(const DdAgg& a, int grp, const DdLayout& lay, const uint32_t* s_n) {
  const int b = threadIdx.x & 31;
  DdDevPlan& p = a.plan[grp];  // one plan per launch: its own buckets only
  const int cls = dd_class_of_len(b + 1);
  const uint32_t n = s_n[b];
  const bool ok = n && dd_group_of_class(cls) == grp && a.ctl[kDdCtlSkip + cls] != 0;
  const uint32_t D = ok ? ld_relaxed(a.ctl + kDdCtlCount + b) : 0u;
  const uint32_t T = cls == 0 ? a.stile1 : a.stilen;
  const uint32_t XT = dd_xtile_of_len(b + 1);
  p.n[b] = ok ? n : 0u;
  p.D[b] = D;
  p.slots[b] = lay.slots[b];
  p.stile[b] = T;
  p.xtile[b] = XT;
  p.tab_off[b] = lay.tab_off[b];
  p.dk_off[b] = lay.dk_off[b];
  p.aux_off[b] = lay.aux_off[b];
  // warp prefixes over the 32 lengths
  uint64_t pay = (uint64_t)n * (uint32_t)(b + 2);  // records of L + 1 bytes (every bucket: the payload holds them all)
  uint32_t tq = lay.dcap[b] / kDdTile + 2;         // tile totals
  uint32_t st = (D + T - 1) / T, rk = (D + kDdTile - 1) / kDdTile, x = ok ? (n + XT - 1) / XT : 0u;
  // (array offsets run over every bucket, whichever launch it belongs to: the
  // two chains share the arrays; work items only over this plan's buckets)
  uint32_t xa = (n + XT - 1) / XT;
  const uint64_t pay0 = pay;
  const uint32_t tq0 = tq, st0 = st, rk0 = rk, x0 = x, xa0 = xa;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t u0 = __shfl_up_sync(0xffffffffu, pay, o);
    const uint32_t u1 = __shfl_up_sync(0xffffffffu, tq, o), u2 = __shfl_up_sync(0xffffffffu, st, o);
    const uint32_t u3 = __shfl_up_sync(0xffffffffu, rk, o), u4 = __shfl_up_sync(0xffffffffu, x, o);
    const uint32_t u5 = __shfl_up_sync(0xffffffffu, xa, o);
    if (b >= o) {
      pay += u0;
      tq += u1;
      st += u2;
      rk += u3;
      x += u4;
      xa += u5;
    }
  }
  const uint32_t tq_all = __shfl_sync(0xffffffffu, tq, 31);
  p.pay_off[b] = pay - pay0;
  p.tsum_off[b] = 2u * lay.aux_total + (tq - tq0);
  p.xs_off[b] = 2u * lay.aux_total + tq_all + (xa - xa0);
  p.st_begin[b] = st - st0;
  p.rk_begin[b] = rk - rk0;
  p.x_begin[b] = x - x0;
  if (b == 31) {
    p.st_begin[32] = st;
    p.rk_begin[32] = rk;
    p.x_begin[32] = x;
    p.aux_total = lay.aux_total;
  }
}

#ifndef WS_DD_LO_MINB
#define WS_DD_LO_MINB 3  // CTAs per SM of the one-word-key launch (register cap 65536 / (512 * MINB))
#endif
#ifndef WS_DD_HI_MINB
#define WS_DD_HI_MINB 2  // ... and of the wider keys' launch
#endif
// One launch per key width group, side by side: GRP 0 = the uint32 keys
// (lengths 1-5: most words, few registers, more CTAs per SM to hide the
// flush's L2 round trips), 1 = the wider keys. (A third launch for the
// one-lane keys measured no faster: the SMs are full either way.)
// Each launch's last CTA finishes its classes' control words and its chain's plan.
template <int GRP>
__global__ void __launch_bounds__(kAggThreads, GRP == 0 ? WS_DD_LO_MINB : WS_DD_HI_MINB) dd_aggregate_kernel(const __grid_constant__ DdAgg a) {
  __shared__ AggSmem sm;
  __shared__ DdLayout lay;
  __shared__ uint32_t s_n[kDdLens], s_tb[kDdLens + 1];
  __shared__ bool s_last;
  const int tid = threadIdx.x;
  if (tid < kDdLens) s_n[tid] = a.fill[tid];
  __syncthreads();
  if (tid == 0) {
    dd_layout(s_n, KbOfLen{}, lay);
    uint32_t run = 0;
    for (int b = 0; b < kDdLens; ++b) {
      s_tb[b] = run;
      if (dd_group_of_class(dd_class_of_len(b + 1)) == GRP) run += (s_n[b] + kAggTile - 1) / kAggTile;
    }
    s_tb[kDdLens] = run;
  }
  __syncthreads();
  uint32_t* dcount = a.ctl + kDdCtlCount;
  uint32_t* ovf = a.ctl + kDdCtlOvf;
  const uint32_t tiles = s_tb[kDdLens];
  for (uint32_t g = blockIdx.x; g < tiles; g += gridDim.x) {
    const int b = __popc(__ballot_sync(0xffffffffu, s_tb[1 + (tid & 31)] <= g));
    // the bucket, or another bucket of its lane class, is out of budget already: the class
    // will be sorted (one answer for the whole CTA: agg_tile has barriers)
    uint32_t* covf = a.ctl + kDdCtlClsOvf + dd_class_of_len(b + 1);
    if (__syncthreads_or(tid == 0 ? (int)(ld_relaxed(ovf + b) | ld_relaxed(covf)) : 0)) continue;
    DdTab t;
    t.keys = a.keys_cap + a.region[b];
    t.tab = a.table + lay.tab_off[b];
    t.slots = lay.slots[b];
    const uint32_t base = (g - s_tb[b]) * kAggTile;
    void* dk = a.dk + lay.dk_off[b];
    uint32_t* dslot = a.aux + lay.aux_off[b];
    if constexpr (GRP == 0) {
      agg_tile<0>(t, s_n[b], base, sm, dk, dslot, lay.dcap[b], dcount + b, ovf + b, covf);
    } else {
      switch (dd_class_of_len(b + 1)) {
        case 1: agg_tile<1>(t, s_n[b], base, sm, dk, dslot, lay.dcap[b], dcount + b, ovf + b, covf); break;
        case 2: agg_tile<2>(t, s_n[b], base, sm, dk, dslot, lay.dcap[b], dcount + b, ovf + b, covf); break;
        default: agg_tile<3>(t, s_n[b], base, sm, dk, dslot, lay.dcap[b], dcount + b, ovf + b, covf); break;
      }
    }
  }
  // The launch's last CTA to finish decides, for its lane classes, whether
  // every bucket stayed in budget (the early launches of the class's sort
  // path skip their work then), and writes the plan of the chain behind it.
  __threadfence();
  __syncthreads();
  if (tid == 0) s_last = atomicAdd(a.ctl + kDdCtlDone + GRP, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last || tid >= 32) return;
  __threadfence();
  if (tid < 4 && dd_group_of_class(tid) == GRP) {
    bool ok = true, any = false;
    for (int b = 0; b < kDdLens; ++b) {
      if (dd_class_of_len(b + 1) != tid || !s_n[b]) continue;
      any = true;
      ok = ok && ld_relaxed(ovf + b) == 0;
    }
    a.ctl[kDdCtlSkip + tid] = (ok && any) ? 1u : 0u;
  }
  __syncwarp();
  __threadfence();
  if (a.plan) dd_write_plan(a, GRP, lay, s_n);
}

// One CTA per length: the bucket's first tile counted and judged (a few
// microseconds), so that a text of mostly different words (configs 2, 3) gives
// its lane classes up before the counting launches run, and the sort paths'
// early launches -- which wait for this kernel only -- start at once.
__global__ void __launch_bounds__(kAggThreads) dd_probe_kernel(const __grid_constant__ DdAgg a) {
  __shared__ AggSmem sm;
  const int b = blockIdx.x;
  const uint32_t n = a.fill[b];
  if (n < (uint32_t)kAggTile) return;
  DdTab t;
  t.keys = a.keys_cap + a.region[b];
  t.tab = nullptr;
  t.slots = 0;
  const int cls = dd_class_of_len(b + 1);
  uint32_t* ovf = a.ctl + kDdCtlOvf + b;
  uint32_t* covf = a.ctl + kDdCtlClsOvf + cls;
  uint32_t* probe = a.ctl + kDdCtlProbe + cls;
  switch (cls) {
    case 0: agg_tile<0, true>(t, n, 0, sm, nullptr, nullptr, 0, nullptr, ovf, covf, probe); break;
    case 1: agg_tile<1, true>(t, n, 0, sm, nullptr, nullptr, 0, nullptr, ovf, covf, probe); break;
    case 2: agg_tile<2, true>(t, n, 0, sm, nullptr, nullptr, 0, nullptr, ovf, covf, probe); break;
    default: agg_tile<3, true>(t, n, 0, sm, nullptr, nullptr, 0, nullptr, ovf, covf, probe); break;
  }
}

void launch_dd_probe(const DdAgg& a, cudaStream_t st) {
  dd_probe_kernel<<<kDdLens, kAggThreads, 0, st>>>(a);
}

void launch_dd_aggregate(const DdAgg& a, int grp, int grid, cudaStream_t st) {
  if (grp == 0) dd_aggregate_kernel<0><<<grid, kAggThreads, 0, st>>>(a);
  else dd_aggregate_kernel<1><<<grid, kAggThreads, 0, st>>>(a);
}
int dd_aggregate_ctas_per_sm(int grp) { return grp == 0 ? WS_DD_LO_MINB : WS_DD_HI_MINB; }

// ----------------------------------------------------------------------------
// after the distinct keys are sorted: run prefixes and payload records

// One bucket as the expand sees it.
struct DdSeg {
  const void* keys_sorted;  // the bucket's distinct keys, sorted
  uint32_t D;               // distinct words
  uint32_t n;               // words
  uint32_t len;
  const uint32_t* loc;      // [D] occurrences before run j inside its block of kDdTile runs
  const uint32_t* tsum;     // [ceil(D / kDdTile)] exclusive prefix of the block totals
  uint8_t* pay;             // the bucket's payload records
};

constexpr int kXThreads = 256;


// first output record of run j
__device__ __forceinline__ uint32_t run_start(const DdSeg& sg, uint32_t j) {
  return sg.tsum[j / kDdTile] + sg.loc[j];
}

// Shared memory of one expand CTA.
constexpr int kXBuf = 512 * (kMaxPackedLen + 1) + 64;  // >= xtile(L) * (L + 1) + 32 for every L
static_assert(kXBuf >= 2048 * 8 + 32 && kXBuf >= 1024 * 16 + 32, "staging buffer holds one output tile");
struct XSmem {
  uint32_t ro[kDdXTileMax + 1];
  __align__(16) uint8_t pbuf[kXBuf];
  uint32_t j0;
};

// Output records [r0, min(n, r0 + TR)) of one bucket (TR a multiple of the
// CTA's threads, TR * (len + 1) + 32 <= kXBuf). j0: the run holding record r0
// (dd_xstart_kernel). Called by every thread of the CTA; ends with the shared memory free for the next tile.
template <int LANES>
__device__ void expand_tile(const DdSeg& sg, uint32_t r0, uint32_t TR, uint32_t j0, XSmem& sm) {
  using W = typename KeyTraits<LANES>::W;
  constexpr int NW = KeyTraits<LANES>::NW;
  constexpr int NL = LANES < 1 ? 1 : LANES;
  const uint32_t r1 = min(sg.n, r0 + TR);
  const int tid = threadIdx.x;
  const uint32_t wn = min(TR, sg.D - j0);  // runs that can start inside the tile (+ run j0)
  for (uint32_t i = tid; i < wn; i += kXThreads) sm.ro[i] = run_start(sg, j0 + i);
  if (tid == 0) sm.ro[wn] = 0xFFFFFFFFu;
  __syncthreads();
  WS_DCHECK(sm.ro[0] <= r0 && sm.ro[1] > r0);
  const int L = (int)sg.len, R = L + 1;
  uint8_t* out0 = sg.pay + (uint64_t)r0 * R;
  if (sm.ro[1] >= r1) {  // one word fills the whole tile
    const Key<LANES> k0 = load_key<LANES>(sg.keys_sorted, j0);
    fill_records_cta<LANES, kXThreads>(k0, r1 - r0, L, out0, sm.pbuf);
    __syncthreads();
    return;
  }
  // each thread: PER consecutive records (one search, then a walk along the runs)
  const W* ks = reinterpret_cast<const W*>(sg.keys_sorted) + (uint64_t)j0 * NW;
  const uint32_t PER = TR / kXThreads;
  const int mis = (int)((uint64_t)out0 & 15);
  uint32_t r = r0 + tid * PER;
  if (r < r1) {
    uint32_t lo = 0, hi = wn;  // largest i with ro[i] <= r
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (sm.ro[mid] <= r) lo = mid; else hi = mid;
    }
    uint32_t nxt = sm.ro[lo + 1];
    uint32_t rec[kRecWords];  // the current run's record, decoded once
    auto fetch = [&](uint32_t i) {
      const W* kp = ks + (uint64_t)i * NW;
      uint64_t k[NL];
      if constexpr (LANES == 0) {
        k[0] = (uint64_t)__ldg(kp) << 32;
      } else {
#pragma unroll
        for (int l = 0; l < NL; ++l) k[l] = __ldg(kp + l);
      }
      decode6_words<NL>(k, L, rec);
    };
    fetch(lo);
    uint8_t* dst = sm.pbuf + mis + (size_t)(tid * PER) * R;
    const uint32_t rend = min(r1, r + PER);
    for (; r < rend; ++r, dst += R) {
      if (r >= nxt) {  // runs are never empty: the next run holds r
        ++lo;
        nxt = sm.ro[lo + 1];
        fetch(lo);
      }
      store_record(dst, rec, R);
    }
  }
  __syncthreads();
  copy_span_out_t<kXThreads>(sm.pbuf, mis, out0, (uint64_t)(r1 - r0) * R);
  __syncthreads();
}

// ----------------------------------------------------------------------------
// the device-planned chain (no host round trip): dd_plan_kernel and the tile
// sort live in sort.cu (its tile network); here the rank merge of the sorted
// tiles, the run prefixes and the expand over DdDevPlan's work items.

// Bucket of work item g (begin[] ascending, begin[32] = total > g): the
// entries begin[1..32] that are <= g. Called by whole warps.
__device__ __forceinline__ int bucket_of(const uint32_t* begin, uint32_t g) {
  return __popc(__ballot_sync(0xffffffffu, begin[1 + (threadIdx.x & 31)] <= g));
}

__device__ __forceinline__ int dd_cls(int b) { return dd_class_of_len(b + 1); }
// The launch handles bucket b (DdChain::cls_mask: one chain per group of lane classes).
__device__ __forceinline__ bool in_mask(const DdChain& c, int b) { return (c.cls_mask >> dd_cls(b)) & 1u; }

// Final rank of tile-sorted distinct word j of a bucket: its position in its
// own tile plus the smaller words of every other tile (the words are distinct:
// no ties). Writes the key and its occurrences at that rank.
template <int LANES>
__device__ __forceinline__ void rank_one(const DdDevPlan& p, const DdChain& c, int b, uint32_t j) {
  const uint32_t D = p.D[b], T = p.stile[b];
  const void* ts = c.ts + p.dk_off[b];
  const Key<LANES> e = load_key<LANES>(ts, j);
  const uint32_t mine = j / T, nt = (D + T - 1) / T;
  uint32_t rank = j - mine * T;
  // U binary searches in flight (their loads are independent)
  constexpr int U = LANES <= 1 ? 8 : 4;
  for (uint32_t q0 = 0; q0 < nt; q0 += U) {
    uint32_t lo[U], len[U], first[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t q = q0 + u;
      first[u] = lo[u] = q * T;
      len[u] = (q < nt && q != mine) ? min(T, D - q * T) : 0u;
    }
    bool more = true;
    while (more) {
      more = false;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (len[u] == 0) continue;
        const uint32_t half = len[u] >> 1;
        if (key_lt<LANES>(load_key<LANES>(ts, lo[u] + half), e)) {
          lo[u] += half + 1;
          len[u] -= half + 1;
        } else {
          len[u] = half;
        }
        more |= len[u] != 0;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) rank += lo[u] - first[u];
  }
  WS_DCHECK(rank < D);
  store_key<LANES>(c.dk + p.dk_off[b], rank, e);
  c.aux[p.aux_off[b] + rank] = c.aux[p.aux_total + p.aux_off[b] + j];
}

__global__ void __launch_bounds__(kDdTile) dd_rank_kernel(const __grid_constant__ DdChain c) {
  pdl_wait();
  const DdDevPlan& p = *c.plan;
  const uint32_t total = p.rk_begin[32];
  for (uint32_t g = blockIdx.x; g < total; g += gridDim.x) {
    const int b = bucket_of(p.rk_begin, g);
    if (!in_mask(c, b)) continue;
    const uint32_t j = (g - p.rk_begin[b]) * kDdTile + threadIdx.x;
    if (j >= p.D[b]) continue;
    switch (dd_cls(b)) {
      case 0: rank_one<0>(p, c, b, j); break;
      case 1: rank_one<1>(p, c, b, j); break;
      case 2: rank_one<2>(p, c, b, j); break;
      default: rank_one<3>(p, c, b, j); break;
    }
  }
}

// Occurrences (array A, sorted order) -> exclusive prefix inside blocks of
// kDdTile runs (in place) + block totals.
__global__ void __launch_bounds__(kDdTile) dd_prefix_kernel(const __grid_constant__ DdChain c) {
  pdl_wait();
  __shared__ uint32_t s_w[kDdTile / 32];
  const DdDevPlan& p = *c.plan;
  const uint32_t total = p.rk_begin[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (uint32_t g = blockIdx.x; g < total; g += gridDim.x) {
    const int b = bucket_of(p.rk_begin, g);
    if (!in_mask(c, b)) continue;
    const uint32_t blk = g - p.rk_begin[b];
    const uint32_t j = blk * kDdTile + threadIdx.x;
    uint32_t* cnt = c.aux + p.aux_off[b];
    const uint32_t v = j < p.D[b] ? cnt[j] : 0u;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    if (lane == 31) s_w[wid] = inc;
    __syncthreads();
    uint32_t pre = inc - v;
    for (int w = 0; w < wid; ++w) pre += s_w[w];
    if (j < p.D[b]) cnt[j] = pre;
    if (threadIdx.x == kDdTile - 1) c.aux[p.tsum_off[b] + blk] = pre + v;
    __syncthreads();
  }
}

// One CTA per length: block totals -> exclusive prefix (in place).
__global__ void __launch_bounds__(1024) dd_tsum_kernel(const __grid_constant__ DdChain c) {
  pdl_wait();
  __shared__ uint32_t s_w[32];
  __shared__ uint32_t s_carry;
  const DdDevPlan& p = *c.plan;
  const int b = blockIdx.x;
  const uint32_t D = p.D[b];
  if (!D || !in_mask(c, b)) return;
  uint32_t* tsum = c.aux + p.tsum_off[b];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t nt = (D + kDdTile - 1) / kDdTile;
  if (tid == 0) s_carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < nt; base += 1024) {
    const uint32_t i = base + tid;
    const uint32_t v = i < nt ? tsum[i] : 0u;
    uint32_t inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += u;
    }
    if (lane == 31) s_w[wid] = inc;
    __syncthreads();
    uint32_t pre = s_carry + inc - v;
    for (int w = 0; w < wid; ++w) pre += s_w[w];
    if (i < nt) tsum[i] = pre;
    __syncthreads();
    if (tid == 1023) s_carry = pre + v;
    __syncthreads();
  }
  WS_DCHECK(s_carry == p.n[b]);
}

// Per output tile of a bucket: the run holding its first record. Run j covers
// records [start(j), start(j + 1)): it names itself in every tile whose first
// record falls there.
__global__ void __launch_bounds__(kDdTile) dd_xstart_kernel(const __grid_constant__ DdChain c) {
  pdl_wait();
  const DdDevPlan& p = *c.plan;
  const uint32_t total = p.rk_begin[32];
  for (uint32_t g = blockIdx.x; g < total; g += gridDim.x) {
    const int b = bucket_of(p.rk_begin, g);
    if (!in_mask(c, b)) continue;
    const uint32_t j = (g - p.rk_begin[b]) * kDdTile + threadIdx.x;
    const uint32_t D = p.D[b];
    if (j >= D) continue;
    const uint32_t* loc = c.aux + p.aux_off[b];
    const uint32_t* tsum = c.aux + p.tsum_off[b];
    const uint32_t s = tsum[j / kDdTile] + loc[j];
    const uint32_t e = j + 1 < D ? tsum[(j + 1) / kDdTile] + loc[j + 1] : p.n[b];
    const uint32_t TR = p.xtile[b];
    uint32_t* xs = c.aux + p.xs_off[b];
    for (uint32_t t = (s + TR - 1) / TR; (uint64_t)t * TR < e; ++t) xs[t] = j;
  }
}

constexpr int kXCtasPerSm = 6;
__global__ void __launch_bounds__(kXThreads, kXCtasPerSm) dd_expand_dev_kernel(const __grid_constant__ DdChain c) {
  pdl_wait();
  __shared__ XSmem sm;
  const DdDevPlan& p = *c.plan;
  const uint32_t total = p.x_begin[32];
  uint32_t g = blockIdx.x;
  if (g >= total) return;
  int b = bucket_of(p.x_begin, g);
  uint32_t j0 = c.aux[p.xs_off[b] + (g - p.x_begin[b])];
  for (;;) {
    // the next tile's bucket and first run are fetched before this tile's work
    const uint32_t gn = g + gridDim.x;
    int bn = 0;
    uint32_t j0n = 0;
    if (gn < total) {
      bn = bucket_of(p.x_begin, gn);
      j0n = c.aux[p.xs_off[bn] + (gn - p.x_begin[bn])];
    }
    if (in_mask(c, b)) {
      DdSeg sg;
      sg.keys_sorted = c.dk + p.dk_off[b];
      sg.D = p.D[b];
      sg.n = p.n[b];
      sg.len = (uint32_t)b + 1;
      sg.loc = c.aux + p.aux_off[b];
      sg.tsum = c.aux + p.tsum_off[b];
      sg.pay = c.out + p.pay_off[b];
      const uint32_t TR = p.xtile[b];
      const uint32_t r0 = (g - p.x_begin[b]) * TR;
      WS_DCHECK(j0 < sg.D);
      switch (dd_cls(b)) {
        case 0: expand_tile<0>(sg, r0, TR, j0, sm); break;
        case 1: expand_tile<1>(sg, r0, TR, j0, sm); break;
        case 2: expand_tile<2>(sg, r0, TR, j0, sm); break;
        default: expand_tile<3>(sg, r0, TR, j0, sm); break;
      }
    }
    if (gn >= total) break;
    g = gn;
    b = bn;
    j0 = j0n;
  }
}

int dd_expand_ctas_per_sm() { return kXCtasPerSm; }

void launch_dd_rank(const DdChain& c, int grid, cudaStream_t st) {
  launch_pdl(dd_rank_kernel, grid, kDdTile, 0, st, c);
}

void launch_dd_prefix(const DdChain& c, int grid, cudaStream_t st) {
  launch_pdl(dd_prefix_kernel, grid, kDdTile, 0, st, c);
  launch_pdl(dd_tsum_kernel, kDdLens, 1024, 0, st, c);
  launch_pdl(dd_xstart_kernel, grid, kDdTile, 0, st, c);
}

void launch_dd_chain_expand(const DdChain& c, int grid, cudaStream_t st) {
  launch_pdl(dd_expand_dev_kernel, grid, kXThreads, 0, st, c);
}

#if WS_DD_PROF
// (tools/dd_phases.py through ctypes; not part of the ABI)
extern "C" int dd_prof_read(unsigned long long* out16) {
  cudaDeviceSynchronize();
  cudaError_t e = cudaMemcpyFromSymbol(out16, g_dd_prof, sizeof g_dd_prof);
  unsigned long long z[16] = {0};
  cudaMemcpyToSymbol(g_dd_prof, z, sizeof z);
  return (int)e;
}
#endif

WS_DEFINE_CHECK_READER(check_reader_dedupe)

}  // namespace ws
