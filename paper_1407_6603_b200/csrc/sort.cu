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
//   tile pass  : each thread holds E consecutive keys in registers and runs
//                odd-even transposition sort on them (E phases of
//                compare-exchange on strict '>': the data-parallel form of
//                bubble sort), then log2(256) merge-path levels in shared
//                memory turn 256 runs of E into one sorted tile of T = 256*E.
//   merge pass : one launch per level; every CTA produces T outputs of one
//                merged pair; its A/B split points come from a warp-wide
//                32-ary merge-path search in global memory, then the windows
//                are staged in shared memory and merged as in the tile pass.
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

namespace ws {

constexpr int kSortThreads = 256;

__host__ __device__ constexpr int sidx(int i) { return i + (i >> 5); }  // 1 pad / 32 elems

template <int LANES>
struct SortCfg {
  static constexpr int E = LANES == 1 ? 16 : 8;
  static constexpr int T = kSortThreads * E;
  static constexpr int S = T + T / 32;  // padded smem stride (elements)
};

template <int LANES, bool STATS>
constexpr size_t sort_smem_bytes() {
  return (size_t)SortCfg<LANES>::S * 8 * LANES + (STATS ? (size_t)SortCfg<LANES>::S * 4 : 0);
}

template <int LANES>
__device__ __forceinline__ Key<LANES> sld(const uint64_t* __restrict__ sk, int i) {
  constexpr int S = SortCfg<LANES>::S;
  Key<LANES> k;
#pragma unroll
  for (int l = 0; l < LANES; ++l) k.w[l] = sk[l * S + sidx(i)];
  return k;
}

template <int LANES>
__device__ __forceinline__ void sst(uint64_t* __restrict__ sk, int i, const Key<LANES>& k) {
  constexpr int S = SortCfg<LANES>::S;
#pragma unroll
  for (int l = 0; l < LANES; ++l) sk[l * S + sidx(i)] = k.w[l];
}

template <int LANES>
__device__ __forceinline__ Key<LANES> gld(const uint64_t* __restrict__ g, int64_t i) {
  Key<LANES> k;
#pragma unroll
  for (int l = 0; l < LANES; ++l) k.w[l] = __ldg(g + i * LANES + l);
  return k;
}

// Merge path inside shared memory: A = [a0, a0+na), B = [b0, b0+nb) of the
// padded arrays; this thread emits outputs [diag, diag+E). When taking b,
// the pending A elements are those > b: inv += a_rem_base - ai.
template <int LANES, int E, bool STATS>
__device__ __forceinline__ void merge_path_serial(const uint64_t* __restrict__ sk,
                                                  const uint32_t* __restrict__ si, int a0, int na,
                                                  int b0, int nb, int diag, int64_t a_rem_base,
                                                  Key<LANES> (&r)[E], uint32_t (&ri)[E],
                                                  uint64_t& inv) {
  int lo = max(0, diag - nb), hi = min(diag, na);
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (key_le<LANES>(sld<LANES>(sk, a0 + mid), sld<LANES>(sk, b0 + diag - 1 - mid)))
      lo = mid + 1;
    else
      hi = mid;
  }
  int ai = lo, bi = diag - lo;
  const Key<LANES> kmax = key_max<LANES>();
  Key<LANES> ka = ai < na ? sld<LANES>(sk, a0 + ai) : kmax;
  Key<LANES> kb = bi < nb ? sld<LANES>(sk, b0 + bi) : kmax;
  uint32_t ia = 0, ib = 0;
  if (STATS) {
    ia = ai < na ? si[sidx(a0 + ai)] : 0xFFFFFFFFu;
    ib = bi < nb ? si[sidx(b0 + bi)] : 0xFFFFFFFFu;
  }
#pragma unroll
  for (int k = 0; k < E; ++k) {
    const bool ta = (bi >= nb) || (ai < na && key_le<LANES>(ka, kb));
    if (ta) {
      r[k] = ka;
      if (STATS) ri[k] = ia;
      ++ai;
      if (ai < na) {
        ka = sld<LANES>(sk, a0 + ai);
        if (STATS) ia = si[sidx(a0 + ai)];
      } else {
        ka = kmax;
      }
    } else {
      r[k] = kb;
      if (STATS) {
        ri[k] = ib;
        inv += (uint64_t)(a_rem_base - ai);
      }
      ++bi;
      if (bi < nb) {
        kb = sld<LANES>(sk, b0 + bi);
        if (STATS) ib = si[sidx(b0 + bi)];
      } else {
        kb = kmax;
      }
    }
  }
}

__device__ __forceinline__ int find_segment(const SegDesc* __restrict__ segs, int nsegs) {
  __shared__ int s_seg;
  if (threadIdx.x == 0) {
    int lo = 0, hi = nsegs - 1;  // last seg with tile_begin <= blockIdx.x
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (segs[mid].tile_begin <= blockIdx.x) lo = mid; else hi = mid - 1;
    }
    s_seg = lo;
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
  if (threadIdx.x == 0) { s_inv = 0; s_k = 0; }
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

// Registers (blocked, E per thread) -> padded smem.
template <int LANES, int E, bool STATS>
__device__ __forceinline__ void regs_to_smem(uint64_t* sk, uint32_t* si, const Key<LANES> (&r)[E],
                                             const uint32_t (&ri)[E]) {
  const int base = threadIdx.x * E;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    sst<LANES>(sk, base + k, r[k]);
    if (STATS) si[sidx(base + k)] = ri[k];
  }
}

// smem (padded) -> global, coalesced over the flat uint64 words of cnt keys.
template <int LANES, bool STATS>
__device__ __forceinline__ void smem_to_global(const uint64_t* sk, const uint32_t* si, int cnt,
                                               uint64_t* __restrict__ gk, uint32_t* __restrict__ gi) {
  constexpr int S = SortCfg<LANES>::S;
  for (int w = threadIdx.x; w < cnt * LANES; w += kSortThreads) {
    int j = w / LANES, l = w - j * LANES;
    gk[w] = sk[l * S + sidx(j)];
  }
  if (STATS && gi) {
    for (int j = threadIdx.x; j < cnt; j += kSortThreads) gi[j] = si[sidx(j)];
  }
}

template <int LANES, bool STATS>
__global__ void __launch_bounds__(kSortThreads) tile_sort_kernel(SortLaunch a) {
  constexpr int E = SortCfg<LANES>::E, T = SortCfg<LANES>::T, S = SortCfg<LANES>::S;
  extern __shared__ __align__(16) uint64_t smem[];
  uint64_t* sk = smem;
  uint32_t* si = reinterpret_cast<uint32_t*>(smem + (size_t)LANES * S);
  const int tid = threadIdx.x;
  const SegDesc sd = a.segs[find_segment(a.segs, a.nsegs)];
  const uint64_t start = (uint64_t)(blockIdx.x - sd.tile_begin) * T;
  const int cnt = (int)min((uint64_t)T, (uint64_t)sd.n - start);
  const uint64_t* gin = a.keys_in + (sd.key_off + start) * LANES;

  for (int w = tid; w < T * LANES; w += kSortThreads) {
    int j = w / LANES, l = w - j * LANES;
    sk[l * S + sidx(j)] = j < cnt ? __ldg(gin + w) : ~0ull;
  }
  if (STATS) {
    for (int j = tid; j < T; j += kSortThreads) si[sidx(j)] = (uint32_t)(sd.idx_base + start + j);
  }
  __syncthreads();

  Key<LANES> r[E];
  uint32_t ri[E];
#pragma unroll
  for (int k = 0; k < E; ++k) {
    r[k] = sld<LANES>(sk, tid * E + k);
    ri[k] = STATS ? si[sidx(tid * E + k)] : 0u;
  }
  // Odd-even transposition sort of the thread's E keys: E phases, each a
  // layer of independent compare-exchanges that swap on strictly-greater.
  uint64_t inv = 0;
#pragma unroll
  for (int ph = 0; ph < E; ++ph) {
#pragma unroll
    for (int i = ph & 1; i + 1 < E; i += 2) {
      const bool sw = key_lt<LANES>(r[i + 1], r[i]);
      if (sw) {
        Key<LANES> t = r[i]; r[i] = r[i + 1]; r[i + 1] = t;
        uint32_t u = ri[i]; ri[i] = ri[i + 1]; ri[i + 1] = u;
      }
      if (STATS) inv += sw;
    }
  }
  // Merge-path levels inside the tile.
#pragma unroll 1
  for (int run = E; run < T; run <<= 1) {
    __syncthreads();
    regs_to_smem<LANES, E, STATS>(sk, si, r, ri);
    __syncthreads();
    const int gt = (2 * run) / E;
    const int a0 = (tid / gt) * 2 * run;
    merge_path_serial<LANES, E, STATS>(sk, si, a0, run, a0 + run, run, (tid % gt) * E, run, r, ri,
                                       inv);
  }
  long long kloc = 0;
  if (STATS && sd.n <= (uint32_t)T) {
#pragma unroll
    for (int k = 0; k < E; ++k) {
      int pos = tid * E + k;
      if (pos < cnt) kloc = max(kloc, (long long)ri[k] - (long long)sd.idx_base - pos);
    }
  }
  flush_stats<STATS>(inv, kloc, sd, a.inv, a.kmax);
  __syncthreads();
  regs_to_smem<LANES, E, STATS>(sk, si, r, ri);
  __syncthreads();
  smem_to_global<LANES, STATS>(sk, si, cnt, a.keys_out + (sd.key_off + start) * LANES,
                               a.idx_out ? a.idx_out + sd.idx_off + start : nullptr);
}

// Warp-wide 32-ary merge-path search in global memory: the number of A
// elements among the first d outputs of merge(A, B) (A first on ties).
template <int LANES>
__device__ int64_t merge_path_search_global(const uint64_t* __restrict__ A, int64_t na,
                                            const uint64_t* __restrict__ B, int64_t nb, int64_t d) {
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

template <int LANES, bool STATS>
__global__ void __launch_bounds__(kSortThreads) merge_kernel(SortLaunch a) {
  constexpr int E = SortCfg<LANES>::E, T = SortCfg<LANES>::T, S = SortCfg<LANES>::S;
  extern __shared__ __align__(16) uint64_t smem[];
  uint64_t* sk = smem;
  uint32_t* si = reinterpret_cast<uint32_t*>(smem + (size_t)LANES * S);
  __shared__ int64_t s_split[2];
  const int tid = threadIdx.x, wid = tid >> 5;
  const SegDesc sd = a.segs[find_segment(a.segs, a.nsegs)];
  const int64_t n = sd.n, R = a.run;
  const int64_t out_begin = (int64_t)(blockIdx.x - sd.tile_begin) * T;
  const int64_t pair_base = (out_begin / (2 * R)) * (2 * R);
  const int64_t na = min(R, n - pair_base);
  const int64_t nb = n - pair_base > R ? min(R, n - pair_base - R) : 0;
  const int64_t d0 = out_begin - pair_base;
  const int64_t d1 = min(d0 + T, na + nb);
  const uint64_t* A = a.keys_in + (sd.key_off + pair_base) * LANES;
  const uint64_t* B = A + R * LANES;
  if (wid < 2) {
    int64_t s = merge_path_search_global<LANES>(A, na, B, nb, wid == 0 ? d0 : d1);
    if ((tid & 31) == 0) s_split[wid] = s;
  }
  __syncthreads();
  const int64_t a0 = s_split[0], a1 = s_split[1];
  const int64_t b0 = d0 - a0, b1 = d1 - a1;
  const int la = (int)(a1 - a0), lb = (int)(b1 - b0);
  // stage A[a0, a1) then B[b0, b1) into smem
  for (int w = tid; w < la * LANES; w += kSortThreads) {
    int j = w / LANES, l = w - j * LANES;
    sk[l * S + sidx(j)] = __ldg(A + a0 * LANES + w);
  }
  for (int w = tid; w < lb * LANES; w += kSortThreads) {
    int j = w / LANES, l = w - j * LANES;
    sk[l * S + sidx(la + j)] = __ldg(B + b0 * LANES + w);
  }
  if (STATS) {
    const uint32_t* IA = a.idx_in + sd.idx_off + pair_base;
    const uint32_t* IB = IA + R;
    for (int j = tid; j < la; j += kSortThreads) si[sidx(j)] = __ldg(IA + a0 + j);
    for (int j = tid; j < lb; j += kSortThreads) si[sidx(la + j)] = __ldg(IB + b0 + j);
  }
  __syncthreads();
  Key<LANES> r[E];
  uint32_t ri[E];
  uint64_t inv = 0;
  merge_path_serial<LANES, E, STATS>(sk, si, 0, la, la, lb, min(tid * E, la + lb), R - a0, r, ri,
                                     inv);
  long long kloc = 0;
  if (STATS && 2 * R >= n) {
#pragma unroll
    for (int k = 0; k < E; ++k) {
      int64_t lp = (int64_t)tid * E + k;
      if (lp < la + lb)
        kloc = max(kloc, (long long)ri[k] - (long long)sd.idx_base - (long long)(out_begin + lp));
    }
  }
  flush_stats<STATS>(inv, kloc, sd, a.inv, a.kmax);
  __syncthreads();
  if (tid * E < la + lb) regs_to_smem<LANES, E, STATS>(sk, si, r, ri);
  __syncthreads();
  smem_to_global<LANES, STATS>(sk, si, la + lb, a.keys_out + (sd.key_off + out_begin) * LANES,
                               STATS ? a.idx_out + sd.idx_off + out_begin : nullptr);
}

int tile_size(int lanes) {
  switch (lanes) {
    case 1: return SortCfg<1>::T;
    case 2: return SortCfg<2>::T;
    case 3: return SortCfg<3>::T;
    default: return SortCfg<4>::T;
  }
}

template <int LANES, bool STATS>
static void set_attrs_t() {
  constexpr int smem = (int)sort_smem_bytes<LANES, STATS>();
  cudaFuncSetAttribute(tile_sort_kernel<LANES, STATS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       smem);
  cudaFuncSetAttribute(merge_kernel<LANES, STATS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       smem);
}

// Opt every sort instantiation into > 48 KiB of dynamic shared memory on the
// current device (called once per device by the handle).
void set_sort_attributes() {
  set_attrs_t<1, false>(); set_attrs_t<1, true>();
  set_attrs_t<2, false>(); set_attrs_t<2, true>();
  set_attrs_t<3, false>(); set_attrs_t<3, true>();
  set_attrs_t<4, false>(); set_attrs_t<4, true>();
}

template <int LANES, bool STATS>
static void launch_tile_t(const SortLaunch& a, cudaStream_t st) {
  tile_sort_kernel<LANES, STATS>
      <<<a.work_items, kSortThreads, sort_smem_bytes<LANES, STATS>(), st>>>(a);
}

template <int LANES, bool STATS>
static void launch_merge_t(const SortLaunch& a, cudaStream_t st) {
  merge_kernel<LANES, STATS><<<a.work_items, kSortThreads, sort_smem_bytes<LANES, STATS>(), st>>>(a);
}

#define WS_DISPATCH_LANES(fn, lanes, stats, ...)                   \
  do {                                                             \
    switch (lanes) {                                               \
      case 1: stats ? fn<1, true>(__VA_ARGS__) : fn<1, false>(__VA_ARGS__); break; \
      case 2: stats ? fn<2, true>(__VA_ARGS__) : fn<2, false>(__VA_ARGS__); break; \
      case 3: stats ? fn<3, true>(__VA_ARGS__) : fn<3, false>(__VA_ARGS__); break; \
      default: stats ? fn<4, true>(__VA_ARGS__) : fn<4, false>(__VA_ARGS__); break; \
    }                                                              \
  } while (0)

void launch_tile_sort(int lanes, const SortLaunch& a, cudaStream_t st) {
  if (!a.work_items) return;
  const bool stats = a.idx_out != nullptr;
  WS_DISPATCH_LANES(launch_tile_t, lanes, stats, a, st);
}

void launch_merge(int lanes, const SortLaunch& a, cudaStream_t st) {
  if (!a.work_items) return;
  const bool stats = a.idx_out != nullptr;
  WS_DISPATCH_LANES(launch_merge_t, lanes, stats, a, st);
}

}  // namespace ws
