// Ingest: raw text -> per-length buckets of packed keys.
//
// Replaces, for the flat layout:
//   tokenize       = WORD_RE.findall        (ingest.py:15, 26-28)
//   _group_by_length (stable, corpus order) (store.py:78-82)
//   build_flat     (count, L) uint8 blocks   (store.py:90-96)
//
// Every kernel takes one 4 KiB chunk per 256-thread CTA: uint4 loads, SWAR
// byte classes, start/end bitmasks, word lengths across thread / warp / CTA
// edges (segmented suffix scan of per-thread alnum runs), 6-bit codes staged
// in shared memory, keys packed in bin-major order and stored to consecutive
// addresses. They differ in how a chunk learns where its runs go:
//   reserve_ingest_kernel      payload mode: one atomic per bin, any order
//   scatter_kernel<kByReserve> stats mode: stable in-chunk order, one atomic
//                              per bin + (position, count) per run, then
//                              reorder_runs_kernel puts runs in corpus order
//   scatter_kernel<kByLookback> with tokens: decoupled look-back over chunks
//   count + scan + scatter_kernel<kByScan>  two-pass fallback (> 512 MiB)
// A word belongs to the chunk that holds its first byte; a word running past
// its chunk is measured by scanning forward in global memory (the text is
// zero padded, and zero is a separator).
#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "ws_common.cuh"
#include "ws_kernels.h"

namespace ws {

constexpr int kChunk = 4096;
#ifndef WS_TEXT_STREAM
#define WS_TEXT_STREAM 1
#endif
#if WS_TEXT_STREAM
#define WS_TEXT_LD(p) __ldcs(p)
#else
#define WS_TEXT_LD(p) (*(p))
#endif
#ifndef WS_RESERVE_SB
#define WS_RESERVE_SB 32  // bytes per thread of the payload-mode ingest (32 or 64; 64 measured slower)
#endif
constexpr int kIngestThreads = 256;  // 16 bytes per thread
constexpr int kWarps = kIngestThreads / 32;
constexpr int kMaxWordsPerWarp = 256;  // 512 bytes per warp, <= 1 start per 2 bytes

__device__ __forceinline__ uint32_t bin_of_len(uint32_t len) {
  return len <= (uint32_t)kMaxPackedLen ? len - 1 : (uint32_t)kLongBin;
}

// Length of the alnum run starting at text[pos] (pos is known alnum or not).
// `avail` bounds the bytes that may be read (chunked H2D: later pieces may not
// have landed yet); running into it sets *overflow and stops.
__device__ uint32_t run_length_from(const uint8_t* __restrict__ text, uint64_t pos,
                                    uint64_t avail = ~0ull, unsigned int* overflow = nullptr) {
  uint32_t len = 0;
  // bring pos to a 16-byte boundary with byte steps
  while ((pos & 15) != 0) {
    if (!is_alnum_byte(text[pos])) return len;
    ++len;
    ++pos;
  }
  while (true) {
    if (pos + 16 > avail) {
      if (overflow) atomicOr(overflow, 1u);
      return len;
    }
    uint4 v = *reinterpret_cast<const uint4*>(text + pos);
    uint32_t m = alnum_mask16(v);
    if (m != 0xFFFFu) return len + __ffs(~m) - 1;
    len += 16;
    pos += 16;
  }
}

// run_length_from for at most `limit` bytes: the length, or ~0u when the run
// is longer (ingest7 leaves such words to long_len_fix_kernel, so one thread
// never walks a multi-megabyte word).
constexpr uint32_t kLongScan = 256;
__device__ uint32_t bounded_run_length(const uint8_t* __restrict__ text, uint64_t pos, uint32_t limit,
                                       uint64_t avail, unsigned int* overflow) {
  uint32_t len = 0;
  while ((pos & 15) != 0) {
    if (!is_alnum_byte(text[pos])) return len;
    ++len;
    ++pos;
  }
  while (len < limit) {
    if (pos + 16 > avail) {
      if (overflow) atomicOr(overflow, 1u);
      return len;
    }
    const uint4 v = *reinterpret_cast<const uint4*>(text + pos);
    const uint32_t m = alnum_mask16(v);
    if (m != 0xFFFFu) return len + __ffs(~m) - 1;
    len += 16;
    pos += 16;
  }
  return ~0u;
}

// Starts/ends of the thread's 16-byte segment plus word lengths.
struct Segment16 {
  uint32_t starts;  // bit i: byte i starts a word
  uint32_t ends;    // bit i: byte i ends a word
  uint32_t cont;    // alnum bytes right after the segment (valid when a start is open)
};

// Classify the thread's 16 bytes of a 4 KiB chunk. Neighbour bits come from
// warp shuffles (a global byte only at warp edges). The length of a word that
// runs past the thread's segment comes from a segmented suffix scan of the
// per-thread leading-alnum counts (warp shuffles, then a walk over the
// following warps' chain heads in shared memory); only a word running past
// the whole chunk scans global memory, and only its starting thread does so.
__device__ __forceinline__ Segment16 classify_chunk(const uint8_t* __restrict__ text, uint64_t n,
                                                    uint64_t cbase, uint4& v_out,
                                                    uint32_t* s_chain /*[kWarps]*/,
                                                    uint64_t avail = ~0ull,
                                                    unsigned int* overflow = nullptr) {
  __shared__ uint32_t s_edge[2 * kWarps];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t base = cbase + (uint64_t)tid * 16;
  uint4 v = make_uint4(0, 0, 0, 0);
  if (base < n) v = *reinterpret_cast<const uint4*>(text + base);
  v_out = v;
  const uint32_t m = alnum_mask16(v);
  const uint32_t up = __shfl_up_sync(0xffffffffu, m, 1);
  const uint32_t dn = __shfl_down_sync(0xffffffffu, m, 1);
  // warp-edge neighbours come from the adjacent warps' masks (shared memory,
  // after the barrier below); only the chunk's two outer edges read a byte
  uint32_t edge = 0;
  if (wid == 0 && lane == 0)
    edge = (base > 0 && base - 1 < n) ? (uint32_t)is_alnum_byte(text[base - 1]) : 0u;
  if (wid == kWarps - 1 && lane == 31)
    edge = (base + 16 < n) ? (uint32_t)is_alnum_byte(text[base + 16]) : 0u;
  // chain (V, F): alnum run from this segment's byte 0 rightwards; F = ended in the warp
  uint32_t V = (uint32_t)__ffs(~m) - 1;  // leading alnum bytes (16 when m == 0xFFFF)
  uint32_t F = V < 16;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t V2 = __shfl_down_sync(0xffffffffu, V, d);
    const uint32_t F2 = __shfl_down_sync(0xffffffffu, F, d);
    if (lane + d < 32 && !F) {
      V += V2;
      F = F2;
    }
  }
  if (lane == 0) s_chain[wid] = V | (F << 31);
  if (lane == 0) s_edge[2 * wid] = m & 1u;                 // first byte of the warp
  if (lane == 31) s_edge[2 * wid + 1] = (m >> 15) & 1u;    // last byte of the warp
  uint32_t cV = __shfl_down_sync(0xffffffffu, V, 1);
  uint32_t cF = __shfl_down_sync(0xffffffffu, F, 1);
  if (lane == 31) cV = cF = 0;
  __syncthreads();
  uint32_t prev = (up >> 15) & 1u, next = dn & 1u;
  if (lane == 0) prev = wid == 0 ? edge : s_edge[2 * wid - 1];
  if (lane == 31) next = wid == kWarps - 1 ? edge : s_edge[2 * wid + 2];
  Segment16 s;
  s.starts = m & ~((m << 1) | prev) & 0xFFFFu;
  s.ends = m & ~((m >> 1) | (next << 15)) & 0xFFFFu;
  // only a segment whose last word is open needs its continuation
  const bool open = s.starts && !(s.ends >> (31 - __clz(s.starts)));  // last start has no end
  if (open && !cF) {
    for (int w = wid + 1; w < kWarps; ++w) {
      const uint32_t c = s_chain[w];
      cV += c & 0x7FFFFFFFu;
      if (c >> 31) {
        cF = 1;
        break;
      }
    }
    if (!cF) cV += run_length_from(text, cbase + kChunk, avail, overflow);
  }
  s.cont = cV;
  return s;
}

// Length of the word starting at bit i of a segment.
__device__ __forceinline__ uint32_t word_len(const Segment16& s, int i) {
  const uint32_t rest = s.ends >> i;
  if (rest) return (uint32_t)__ffs(rest);
  return (uint32_t)(16 - i) + s.cont;
}

// Wide segments (payload-mode ingest): SB = 32 or 64 bytes per thread, i.e.
// 8 or 16 KiB chunks per CTA, SB / 16 uint4 loads per thread and SB-bit start
// / end masks. The per-thread share of the shuffles, scans and barriers is
// spread over 2-4x the bytes of the 16-byte classification above.
template <int SB>
struct SegW {
  using M = typename std::conditional<SB == 64, unsigned long long, uint32_t>::type;
  M starts, ends;
  uint32_t cont;
};

template <int SB>
__device__ __forceinline__ int ffsw(typename SegW<SB>::M x) {
  if constexpr (SB == 64) return __ffsll((long long)x); else return __ffs((int)x);
}

template <int SB>
__device__ __forceinline__ SegW<SB> classify_wide(const uint8_t* __restrict__ text, uint64_t n,
                                                  uint64_t cbase, uint4 (&v)[SB / 16],
                                                  uint32_t* s_chain /*[kWarps]*/, uint64_t avail,
                                                  unsigned int* overflow) {
  using M = typename SegW<SB>::M;
  constexpr int NV = SB / 16;
  constexpr uint64_t kCB = (uint64_t)SB * kIngestThreads;
  __shared__ uint32_t s_edge[2 * kWarps];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t base = cbase + (uint64_t)tid * SB;
  M m = 0;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    v[k] = make_uint4(0, 0, 0, 0);
    // padded text; streamed once (evict-first), so the keys written behind it stay in L2
    if (base < n) v[k] = WS_TEXT_LD(reinterpret_cast<const uint4*>(text + base) + k);
    m |= (M)alnum_mask16(v[k]) << (16 * k);
  }
  const M up = __shfl_up_sync(0xffffffffu, m, 1);
  const M dn = __shfl_down_sync(0xffffffffu, m, 1);
  uint32_t edge = 0;
  if (wid == 0 && lane == 0)
    edge = (base > 0 && base - 1 < n) ? (uint32_t)is_alnum_byte(text[base - 1]) : 0u;
  if (wid == kWarps - 1 && lane == 31)
    edge = (base + SB < n) ? (uint32_t)is_alnum_byte(text[base + SB]) : 0u;
  uint32_t V = m == (M)~(M)0 ? (uint32_t)SB : (uint32_t)ffsw<SB>(~m) - 1;  // leading alnum bytes
  uint32_t F = V < (uint32_t)SB;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t V2 = __shfl_down_sync(0xffffffffu, V, d);
    const uint32_t F2 = __shfl_down_sync(0xffffffffu, F, d);
    if (lane + d < 32 && !F) {
      V += V2;
      F = F2;
    }
  }
  if (lane == 0) s_chain[wid] = V | (F << 31);
  if (lane == 0) s_edge[2 * wid] = (uint32_t)(m & 1u);
  if (lane == 31) s_edge[2 * wid + 1] = (uint32_t)(m >> (SB - 1));
  uint32_t cV = __shfl_down_sync(0xffffffffu, V, 1);
  uint32_t cF = __shfl_down_sync(0xffffffffu, F, 1);
  if (lane == 31) cV = cF = 0;
  __syncthreads();
  M prev = up >> (SB - 1), next = dn & 1u;
  if (lane == 0) prev = wid == 0 ? edge : s_edge[2 * wid - 1];
  if (lane == 31) next = wid == kWarps - 1 ? edge : s_edge[2 * wid + 2];
  SegW<SB> s;
  s.starts = m & ~((m << 1) | prev);
  s.ends = m & ~((m >> 1) | (next << (SB - 1)));
  int last = 0;  // highest start bit
  if constexpr (SB == 64) last = 63 - __clzll((long long)s.starts); else last = 31 - __clz((int)s.starts);
  const bool open = s.starts && !(s.ends >> last);
  if (open && !cF) {
    for (int w = wid + 1; w < kWarps; ++w) {
      const uint32_t c = s_chain[w];
      cV += c & 0x7FFFFFFFu;
      if (c >> 31) {
        cF = 1;
        break;
      }
    }
    if (!cF) cV += run_length_from(text, cbase + kCB, avail, overflow);
  }
  s.cont = cV;
  return s;
}

template <int SB>
__device__ __forceinline__ uint32_t word_len_w(const SegW<SB>& s, int i) {
  const typename SegW<SB>::M rest = s.ends >> i;
  return rest ? (uint32_t)ffsw<SB>(rest) : (uint32_t)(SB - i) + s.cont;
}

__global__ void __launch_bounds__(kIngestThreads)
count_kernel(const uint8_t* __restrict__ text, uint64_t n, uint32_t* __restrict__ hist,
             uint32_t nchunks) {
  __shared__ uint32_t shist[kHistRows];
  __shared__ uint32_t s_chain[kWarps];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  if (tid < kHistRows) shist[tid] = 0;
  const uint64_t chunk = blockIdx.x;
  uint4 v;
  Segment16 seg = classify_chunk(text, n, chunk * kChunk, v, s_chain);  // has a __syncthreads
  uint32_t s = seg.starts;
  // total words of the chunk
  uint32_t c = __popc(s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0 && c) atomicAdd(&shist[kNumBins], c);
  // warp-aggregated histogram: one match per word slot, one atomic per distinct bin
  while (__any_sync(0xffffffffu, s != 0)) {
    uint32_t key = 0xFFFFFFFFu;
    if (s) {
      int i = __ffs(s) - 1;
      s &= s - 1;
      key = bin_of_len(word_len(seg, i));
    }
    uint32_t peers = __match_any_sync(0xffffffffu, key);
    if (key != 0xFFFFFFFFu && lane == __ffs(peers) - 1) atomicAdd(&shist[key], __popc(peers));
  }
  __syncthreads();
  if (tid < kHistRows) hist[(uint64_t)tid * nchunks + chunk] = shist[tid];
}

// Exclusive scan of one histogram row over chunks; totals[row] = row sum.
__global__ void __launch_bounds__(1024)
scan_kernel(const uint32_t* __restrict__ hist, uint32_t* __restrict__ off,
            uint32_t* __restrict__ totals, uint32_t nchunks) {
  pdl_wait();
  __shared__ uint32_t warp_sums[32];
  __shared__ uint32_t carry_s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t row = blockIdx.x;
  const uint32_t* h = hist + row * nchunks;
  uint32_t* o = off + row * nchunks;
  if (tid == 0) carry_s = 0;
  __syncthreads();
  constexpr int kItems = 4;
  for (uint32_t tile = 0; tile < nchunks; tile += 1024 * kItems) {
    uint32_t vals[kItems];
    uint32_t sum = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      uint32_t j = tile + tid * kItems + k;
      vals[k] = j < nchunks ? h[j] : 0u;
      sum += vals[k];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
      if (lane >= d) incl += t;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      uint32_t ws_ = warp_sums[lane];
      uint32_t wi = ws_;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        uint32_t t = __shfl_up_sync(0xffffffffu, wi, d);
        if (lane >= d) wi += t;
      }
      warp_sums[lane] = wi - ws_;  // exclusive
    }
    __syncthreads();
    uint32_t carry = carry_s;
    uint32_t run = carry + warp_sums[wid] + incl - sum;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      uint32_t j = tile + tid * kItems + k;
      if (j < nchunks) o[j] = run;
      run += vals[k];
    }
    __syncthreads();
    if (tid == 1023) carry_s = run;
    __syncthreads();
  }
  if (tid == 0) totals[row] = carry_s;
}

// Pack up to 32 bytes of a word (from a 4-byte aligned smem chunk) into
// big-endian uint64 lanes, zero padded past L.
// (one code path for every width: lanes beyond `lanes` are predicated off, so
// a warp holding words of several lengths does not diverge)
__device__ __forceinline__ void pack_from_smem(const uint32_t* __restrict__ c32, uint32_t start,
                                               uint32_t L, int lanes, uint64_t* __restrict__ dst) {
  const int nl = lanes < 1 ? 1 : lanes;
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    if (l >= nl) break;
    uint32_t q = start + 8 * l;
    uint32_t w0 = c32[q >> 2], w1 = c32[(q >> 2) + 1], w2 = c32[(q >> 2) + 2];
    uint32_t sh = (q & 3) * 8;
    uint32_t lo = __funnelshift_r(w0, w1, sh);
    uint32_t hi = __funnelshift_r(w1, w2, sh);
    uint64_t k = ((uint64_t)__byte_perm(lo, 0, 0x0123) << 32) | __byte_perm(hi, 0, 0x0123);
    int r = (int)L - 8 * l;
    if (r < 8) k &= ~0ull << (64 - 8 * r);
    dst[l] = k;
  }
}

// 6-bit alnum packing (text ingest): characters form one big-endian bit
// string over up to 3 lanes; the unrolled loop resolves lane/shift at compile
// time, characters past L are predicated off.
// 4 bytes -> their 6-bit alnum codes, byte by byte (SWAR; bytes that are not
// [0-9A-Za-z] give garbage that the per-word length mask removes later).
__device__ __forceinline__ uint32_t alnum6_codes4(uint32_t x) {
  const uint32_t xh = x | 0x80808080u;                        // no borrows below
  const uint32_t ge41 = ((xh - 0x41414141u) & 0x80808080u) >> 7;  // 1 per byte >= 'A'
  const uint32_t ge61 = ((xh - 0x61616161u) & 0x80808080u) >> 7;  // 1 per byte >= 'a'
  return (xh - (0x2F2F2F2Fu + ge41 * 7u + ge61 * 6u)) & 0x3F3F3F3Fu;
}

__device__ __forceinline__ uint4 alnum6_codes16(uint4 v) {
  return make_uint4(alnum6_codes4(v.x), alnum6_codes4(v.y), alnum6_codes4(v.z),
                    alnum6_codes4(v.w));
}

// 4 code bytes (little-endian in a u32, first character lowest) -> 24-bit
// big-endian code string.
__device__ __forceinline__ uint32_t codes24(uint32_t le) {
  uint32_t t = __byte_perm(le, 0, 0x0123);                    // first character on top
  t = ((t & 0x3F003F00u) >> 2) | (t & 0x003F003Fu);           // 12 bits per half
  return ((t & 0x0FFF0000u) >> 4) | (t & 0x00000FFFu);        // 24 bits
}

// 6-bit packing from a chunk whose smem copy already holds codes (text
// ingest): the word's codes form one big-endian bit string over <= 3 lanes.
__device__ __forceinline__ void pack6_from_codes(const uint32_t* __restrict__ c32, uint32_t start,
                                                 uint32_t L, int lanes, uint64_t* __restrict__ dst) {
  uint64_t v[4];  // 48-bit chunks of 8 characters
#pragma unroll
  for (int l = 0; l < 4; ++l) {
    v[l] = 0;
    if (8 * l < (int)L) {
      const uint32_t q = start + 8 * l;
      const uint32_t w0 = c32[q >> 2], w1 = c32[(q >> 2) + 1], w2 = c32[(q >> 2) + 2];
      const uint32_t sh = (q & 3) * 8;
      const uint32_t lo = __funnelshift_r(w0, w1, sh), hi = __funnelshift_r(w1, w2, sh);
      v[l] = ((uint64_t)codes24(lo) << 24) | codes24(hi);
    }
  }
  uint64_t k0 = (v[0] << 16) | (v[1] >> 32);
  uint64_t k1 = (v[1] << 32) | (v[2] >> 16);
  uint64_t k2 = (v[2] << 48) | v[3];
  const int bits = 6 * (int)L;
  k0 &= bits >= 64 ? ~0ull : ~0ull << (64 - bits);
  k1 &= bits >= 128 ? ~0ull : (bits <= 64 ? 0ull : ~0ull << (128 - bits));
  k2 &= bits >= 192 ? ~0ull : (bits <= 128 ? 0ull : ~0ull << (192 - bits));
  dst[0] = k0;
  dst[1] = k1;
  dst[2] = k2;
}

// 6-bit packing specialised by lane class (warp-uniform inside a bin-major
// batch): classes 0 and 1 (L <= 10, most words) read 8 or 12 code bytes and
// skip the generic 4-group path.
__device__ __forceinline__ void pack6_fast(const uint32_t* __restrict__ c32, uint32_t start,
                                           uint32_t L, int lanes, uint64_t* __restrict__ dst) {
  const uint32_t q = start >> 2, sh = (start & 3) * 8;
  if (lanes == 0) {  // <= 5 characters -> top 30 bits of one uint32 (stored as k[0] >> 32)
    const uint32_t w0 = c32[q], w1 = c32[q + 1], w2 = c32[q + 2];
    const uint32_t a = codes24(__funnelshift_r(w0, w1, sh));
    const uint32_t b = codes24(__funnelshift_r(w1, w2, sh));
    const uint32_t k = ((a << 8) | (b >> 16)) & (~0u << (32 - 6 * L));
    dst[0] = (uint64_t)k << 32;
    return;
  }
  if (lanes == 1) {  // <= 10 characters -> top 60 bits of one uint64
    const uint32_t w0 = c32[q], w1 = c32[q + 1], w2 = c32[q + 2], w3 = c32[q + 3];
    const uint64_t a = codes24(__funnelshift_r(w0, w1, sh));
    const uint64_t b = codes24(__funnelshift_r(w1, w2, sh));
    const uint64_t c = codes24(__funnelshift_r(w2, w3, sh));
    const uint64_t k = (a << 40) | (b << 16) | (c >> 8);
    dst[0] = k & (~0ull << (64 - 6 * L));
    return;
  }
  pack6_from_codes(c32, start, L, lanes, dst);
}

// Key store: lane class 0 keeps the top 32 bits of the first lane (6-bit keys
// of <= 5 characters and raw keys of <= 4 bytes fit), else `lanes` uint64s.
__device__ __forceinline__ void store_key(uint8_t* dst, int lanes, const uint64_t (&k)[4]) {
  if (lanes == 0) {
    *reinterpret_cast<uint32_t*>(dst) = (uint32_t)(k[0] >> 32);
    return;
  }
  uint64_t* d = reinterpret_cast<uint64_t*>(dst);
  d[0] = k[0];
  if (lanes > 1) d[1] = k[1];
  if (lanes > 2) d[2] = k[2];
  if (lanes > 3) d[3] = k[3];
}

// Decoupled look-back over chunks (record layout: ws_common.cuh kLookbackRec).
// Values are written before the flag, every writer lane fences, and readers
// fence after observing the flag.
static_assert(kRecAgg + kHistRows <= kRecIncl && kRecIncl + kHistRows <= kLookbackRec, "record");

// Warp 0: publish this chunk's per-row values at `where` (kRecAgg / kRecIncl)
// and raise the flag to `flag` (1 = aggregate, 2 = inclusive prefix).
__device__ __forceinline__ void publish_record(uint32_t* __restrict__ status, uint32_t chunk,
                                               const uint32_t* __restrict__ vals, int where,
                                               uint32_t flag) {
  const int lane = threadIdx.x & 31;
  volatile uint32_t* rec = status + (uint64_t)chunk * kLookbackRec;
  for (int r = lane; r < kHistRows; r += 32) rec[where + r] = vals[r];
  __threadfence();
  __syncwarp();
  if (lane == 0) rec[0] = flag;
  __syncwarp();
}

// Warp 0: exclusive prefix of every row over chunks < chunk. Each step reads
// the flags of 32 predecessors (lane l <-> chunk q - l), waits until all are
// published, finds the nearest inclusive record (ballot), and every lane up to
// it fetches its record's rows with independent 16-byte loads (one memory
// round trip per window); rows are then summed across lanes with redux.sync.
__device__ __forceinline__ void resolve_prefix_warp(uint32_t* __restrict__ status, uint32_t chunk,
                                                    uint32_t* __restrict__ excl_out) {
  constexpr int kVec = (kHistRows + 3) / 4;
  const int lane = threadIdx.x & 31;
  volatile uint32_t* st = status;
  uint32_t acc0 = 0, acc1 = 0;  // rows lane and lane + 32
  int64_t q = (int64_t)chunk - 1;
  while (q >= 0) {
    const int64_t mine = q - lane;
    uint32_t f = 2;  // "before chunk 0" behaves like an inclusive zero
    if (mine >= 0) {
      do {
        f = st[(uint64_t)mine * kLookbackRec];
      } while (f == 0);
    }
    __threadfence();
    const uint32_t incl = __ballot_sync(0xffffffffu, f == 2);
    const int stop = incl ? __ffs(incl) - 1 : 31;  // last lane (record) of the window
    uint4 v[kVec];
#pragma unroll
    for (int i = 0; i < kVec; ++i) v[i] = make_uint4(0, 0, 0, 0);
    if (lane <= stop && mine >= 0) {
      const int where = (lane == stop && incl) ? kRecIncl : kRecAgg;
      const uint4* rec = reinterpret_cast<const uint4*>(status + (uint64_t)mine * kLookbackRec + where);
#pragma unroll
      for (int i = 0; i < kVec; ++i) v[i] = __ldcg(rec + i);
    }
#pragma unroll
    for (int r = 0; r < kHistRows; ++r) {
      const uint4 w = v[r >> 2];
      const uint32_t x = (r & 3) == 0 ? w.x : (r & 3) == 1 ? w.y : (r & 3) == 2 ? w.z : w.w;
      const uint32_t sum = __reduce_add_sync(0xffffffffu, x);
      if (lane == (r & 31)) {
        if (r < 32) acc0 += sum; else acc1 += sum;
      }
    }
    if (incl) break;
    q -= 32;
  }
  excl_out[lane] = acc0;
  if (lane + 32 < kHistRows) excl_out[lane + 32] = acc1;
}

// K3 (two-pass) / single-pass ingest. MODE kByScan: chunk offsets come
// from the scan of K1's histograms and keys land in the compact bucket
// layout. kByLookback: CTAs take chunks in ticket order, chain their
// per-bin offsets through a decoupled look-back and write into
// capacity-bounded per-length regions (no count pass, no host round trip
// before the scatter); the last chunk publishes the totals. kByReserve: the
// same stable in-chunk order, but each chunk reserves its bin runs with one
// atomic per bin and records (position, count) per (bin, chunk); a scan over
// chunks and reorder_runs_kernel then move the runs into corpus order (no
// chain between chunks). (Payload-only ingests use reserve_ingest_kernel.)
enum ScatterMode : int { kByScan = 0, kByLookback = 1, kByReserve = 2 };
template <int MODE>
__global__ void __launch_bounds__(kIngestThreads)
scatter_kernel(const uint8_t* __restrict__ text, uint64_t n, const uint32_t* __restrict__ off,
               uint32_t nchunks, ScatterParams p) {
  __shared__ __align__(16) uint32_t chunk32[(kChunk + 64) / 4];
  __shared__ uint16_t wstart[kWarps][kMaxWordsPerWarp];
  __shared__ uint32_t wlen[kWarps][kMaxWordsPerWarp];
  __shared__ uint32_t wpos[kWarps][kMaxWordsPerWarp];
  __shared__ uint32_t ord[kChunk / 2];  // packed words in bin-major order: start | L << 16
  __shared__ uint32_t wcnt[kWarps][kHistRows];
  __shared__ uint32_t wtot[kWarps];
  __shared__ uint32_t s_chain[kWarps];
  __shared__ uint32_t s_base[kHistRows];
  __shared__ uint32_t s_run[kHistRows];
  __shared__ uint32_t s_incl[kHistRows];
  __shared__ uint32_t s_boff[kMaxPackedLen + 1];  // bin-major word offset of each bin
  __shared__ uint64_t s_dst[kMaxPackedLen];       // key byte address of ord slot 0, per bin
  __shared__ uint32_t s_chunk;

  constexpr bool LOOKBACK = MODE == kByLookback;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (LOOKBACK) {
    if (tid == 0) s_chunk = p.chunk0 + atomicAdd(p.ticket, 1u);
    __syncthreads();
  }
  const uint64_t chunk = LOOKBACK ? s_chunk : p.chunk0 + blockIdx.x;
  const uint64_t cbase = chunk * kChunk;
  for (int i = tid; i < kWarps * kHistRows; i += kIngestThreads) (&wcnt[0][0])[i] = 0;
  if (MODE == kByScan && tid < kHistRows) s_base[tid] = off[(uint64_t)tid * nchunks + chunk];

  uint4 v;
  Segment16 seg = classify_chunk(text, n, cbase, v, s_chain, p.avail ? p.avail : ~0ull,
                                 p.overflow);  // has a __syncthreads
  const bool codes = p.enc == kEncAlnum6;
  reinterpret_cast<uint4*>(chunk32)[tid] = codes ? alnum6_codes16(v) : v;
  if (tid < 4) {
    uint64_t a = cbase + kChunk + 16 * tid;
    uint4 la = a < n ? *reinterpret_cast<const uint4*>(text + a) : make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4*>(chunk32)[kChunk / 16 + tid] = codes ? alnum6_codes16(la) : la;
  }
  // warp-local word list in corpus order (lane-major, then bit order)
  uint32_t c = __popc(seg.starts);
  uint32_t incl = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  uint32_t slot = incl - c;
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  {
    uint32_t s = seg.starts;
    while (s) {
      int i = __ffs(s) - 1;
      s &= s - 1;
      WS_DCHECK(slot < (uint32_t)kMaxWordsPerWarp);
      wstart[wid][slot] = (uint16_t)(tid * 16 + i);
      wlen[wid][slot] = word_len(seg, i);
      ++slot;
    }
  }
  if (lane == 0) wtot[wid] = total;
  __syncthreads();  // also publishes chunk32 and zeroed wcnt
  // pass 1: stable rank inside the warp per bin
  for (uint32_t b = 0; b < total; b += 32) {
    uint32_t j = b + lane;
    uint32_t key = j < total ? bin_of_len(wlen[wid][j]) : 0xFFFFFFFFu;
    uint32_t peers = __match_any_sync(0xffffffffu, key);
    uint32_t rank = __popc(peers & ((1u << lane) - 1u));
    if (key != 0xFFFFFFFFu) wpos[wid][j] = wcnt[wid][key] + rank;
    __syncwarp();
    if (key != 0xFFFFFFFFu && lane == 31 - __clz(peers)) wcnt[wid][key] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // per-bin: exclusive scan of the warp counts and the chunk total
  if (tid < kHistRows) {
    uint32_t run = 0;
    for (int w = 0; w < kWarps; ++w) {
      const uint32_t cw = (tid == kNumBins) ? wtot[w] : wcnt[w][tid];
      wcnt[w][tid] = run;
      run += cw;
    }
    s_run[tid] = run;
  }
  __syncthreads();
  if (MODE == kByReserve && tid < kHistRows) {  // reserve the runs, record them for the reorder
    const uint32_t cnt = s_run[tid];
    const uint32_t at = cnt ? atomicAdd(p.fill + tid, cnt) : 0u;
    s_base[tid] = at;
    p.run_at[(uint64_t)tid * p.nchunks_total + chunk] = at;
    p.run_cnt[(uint64_t)tid * p.nchunks_total + chunk] = cnt;
  }
  // chunk offsets: the decoupled look-back (warp 0, publishing the aggregate
  // first); the other warps meanwhile scan the bins and build the bin-major
  // word order
  if (LOOKBACK && wid == 0) {
    publish_record(p.status, (uint32_t)chunk, s_run, chunk == 0 ? kRecIncl : kRecAgg,
                   chunk == 0 ? 2u : 1u);
    resolve_prefix_warp(p.status, (uint32_t)chunk, s_base);
    __syncwarp();
    if (chunk > 0) {
      for (int r = lane; r < kHistRows; r += 32) s_incl[r] = s_base[r] + s_run[r];
      __syncwarp();
      publish_record(p.status, (uint32_t)chunk, s_incl, kRecIncl, 2u);
    }
    if (chunk == p.nchunks_total - 1)
      for (int r = lane; r < kHistRows; r += 32) p.totals[r] = s_base[r] + s_run[r];
  }
  if (wid == 1) {  // exclusive scan of the packed bins' counts (lane = bin)
    const uint32_t cnt = s_run[lane];
    uint32_t inc = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += t;
    }
    s_boff[lane] = inc - cnt;
    if (lane == 31) s_boff[kMaxPackedLen] = inc;
  }
  __syncthreads();
  // bin-major word order of the packed words (long words / tokens go out here)
  for (uint32_t b = 0; b < total; b += 32) {
    const uint32_t j = b + lane;
    if (j >= total) break;
    const uint32_t L = wlen[wid][j];
    const uint32_t start = wstart[wid][j];
    const uint32_t bin = bin_of_len(L);
    if (bin != (uint32_t)kLongBin) {
      WS_DCHECK(s_boff[bin] + wcnt[wid][bin] + wpos[wid][j] < s_boff[bin + 1]);
      ord[s_boff[bin] + wcnt[wid][bin] + wpos[wid][j]] = start | (L << 16);
    } else if (p.keys) {
      p.longlist[s_base[kLongBin] + wcnt[wid][kLongBin] + wpos[wid][j]] =
          make_uint2((uint32_t)(cbase + start), L);
    }
    if (p.tokens) {
      const uint32_t widx = s_base[kNumBins] + wcnt[wid][kNumBins] + j;
      p.tokens[widx] = make_uint2((uint32_t)(cbase + start), L);
    }
  }
  if (tid < kMaxPackedLen) {  // global key address of bin-major slot 0 of each bin
    const uint64_t ks = (uint64_t)key_bytes(lanes_for_len_enc(tid + 1, p.enc));
    s_dst[tid] = p.bin_base[tid] + ((uint64_t)s_base[tid] - s_boff[tid]) * ks;
  }
  __syncthreads();
  // pack: consecutive threads take consecutive words of one bin (same length,
  // no divergence) and store their keys to consecutive global addresses
  if (p.keys) {
    const uint32_t npacked = s_boff[kMaxPackedLen];
    uint8_t* keys = reinterpret_cast<uint8_t*>(p.keys);
    for (uint32_t k = tid; k < npacked; k += kIngestThreads) {
      const uint32_t e = ord[k];
      const uint32_t start = e & 0xFFFFu, L = e >> 16;
      const int lanes = lanes_for_len_enc(L, p.enc);
      uint64_t key[4];
      if (codes)
        pack6_fast(chunk32, start, L, lanes, key);
      else
        pack_from_smem(chunk32, start, L, lanes, key);
      store_key(keys + s_dst[L - 1] + (uint64_t)k * key_bytes(lanes), lanes, key);
    }
  }
}

// Reserve-mode ingest (payload-only sorts, ScatterParams::fill set): order
// inside a bucket is free, so a word's slot in its bin is one shared-memory
// atomic (no per-warp ranking pass), and each chunk reserves its bin runs in
// HBM with one global atomic per bin. Keys are then packed in bin-major order
// (uniform length per warp batch) and stored to consecutive addresses.
template <int SB, int ENC>
__global__ void __launch_bounds__(kIngestThreads)
reserve_ingest_kernel(const uint8_t* __restrict__ text, uint64_t n, ScatterParams p) {
  constexpr int kCB = SB * kIngestThreads;  // chunk bytes
  constexpr int NV = SB / 16;
  extern __shared__ __align__(16) uint32_t dyn_smem[];
  uint32_t* chunk32 = dyn_smem;                  // (kCB + 64) bytes of 6-bit codes
  uint32_t* ord = dyn_smem + (kCB + 64) / 4;     // kCB / 2 words, bin-major
  __shared__ uint32_t s_cnt[kHistRows];
  __shared__ uint32_t s_cur[kNumBins];  // per-bin cursors into ord (long bin: into its run)
  __shared__ uint32_t s_base[kHistRows];
  __shared__ uint32_t s_boff[kMaxPackedLen + 1];
  __shared__ uint64_t s_dst[kMaxPackedLen];
  __shared__ uint32_t s_chain[kWarps];

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t chunk = p.chunk0 + blockIdx.x;
  const uint64_t cbase = chunk * kCB;
  if (tid < kHistRows) s_cnt[tid] = 0;

  uint4 v[NV];
  const SegW<SB> seg = classify_wide<SB>(text, n, cbase, v, s_chain, p.avail ? p.avail : ~0ull,
                                         p.overflow);  // has a __syncthreads
  constexpr bool codes = ENC == kEncAlnum6;  // text ingest: 6-bit codes (else raw bytes)
#pragma unroll
  for (int q = 0; q < NV; ++q)
    reinterpret_cast<uint4*>(chunk32)[NV * tid + q] = codes ? alnum6_codes16(v[q]) : v[q];
  if (tid < 4) {
    uint64_t a = cbase + kCB + 16 * tid;
    uint4 la = a < n ? *reinterpret_cast<const uint4*>(text + a) : make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4*>(chunk32)[kCB / 16 + tid] = codes ? alnum6_codes16(la) : la;
  }
  // count the chunk's words per bin (no return value, nothing kept)
  using M = typename SegW<SB>::M;
  for (M s = seg.starts; s; s &= s - 1)
    atomicAdd(&s_cnt[bin_of_len(word_len_w<SB>(seg, ffsw<SB>(s) - 1))], 1u);
  uint32_t nw = 0;
  if constexpr (SB == 64) nw = __popcll(seg.starts); else nw = __popc(seg.starts);
  const uint32_t words = __reduce_add_sync(0xffffffffu, nw);
  if (lane == 0 && words) atomicAdd(&s_cnt[kNumBins], words);
  __syncthreads();  // also publishes chunk32
  if (tid < kHistRows && s_cnt[tid]) s_base[tid] = atomicAdd(p.fill + tid, s_cnt[tid]);
  if (wid == 1) {  // bin-major offsets of the packed bins (lane = bin) = their cursors
    const uint32_t cnt = s_cnt[lane];
    uint32_t inc = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += t;
    }
    s_boff[lane] = inc - cnt;
    s_cur[lane] = inc - cnt;
    if (lane == 31) {
      s_boff[kMaxPackedLen] = inc;
      s_cur[kLongBin] = 0;
    }
  }
  __syncthreads();
  // place every word: packed ones into ord (bin-major), long ones into their run
  for (M s = seg.starts; s; s &= s - 1) {
    const int i = ffsw<SB>(s) - 1;
    const uint32_t L = word_len_w<SB>(seg, i), bin = bin_of_len(L);
    const uint32_t at = atomicAdd(&s_cur[bin], 1u);
    const uint32_t start = (uint32_t)(tid * SB + i);
    WS_DCHECK(bin == (uint32_t)kLongBin ? at < s_cnt[kLongBin] : at < s_boff[kMaxPackedLen]);
    WS_DCHECK(L >= 1 && L < (1u << 16));
    if (bin != (uint32_t)kLongBin)
      ord[at] = start | (L << 16);
    else if (p.keys)
      p.longlist[s_base[kLongBin] + at] = make_uint2((uint32_t)(cbase + start), L);
  }
  if (tid < kMaxPackedLen) {
    const uint64_t ks = (uint64_t)key_bytes(lanes_for_len_enc(tid + 1, ENC));
    s_dst[tid] = p.bin_base[tid] + ((uint64_t)s_base[tid] - s_boff[tid]) * ks;
  }
  __syncthreads();
  if (p.keys) {
    const uint32_t npacked = s_boff[kMaxPackedLen];
    uint8_t* keys = reinterpret_cast<uint8_t*>(p.keys);
    for (uint32_t k = tid; k < npacked; k += kIngestThreads) {
      const uint32_t e = ord[k];
      const uint32_t start = e & 0xFFFFu, L = e >> 16;
      const int lanes = lanes_for_len_enc(L, ENC);
      // the key's slot in its length region stays inside the region's capacity
      WS_DCHECK(L >= 1 && L <= (uint32_t)kMaxPackedLen && start < (uint32_t)kCB &&
                k >= s_boff[L - 1] && k < s_boff[L] &&
                s_base[L - 1] + (k - s_boff[L - 1]) <= (uint32_t)((n + 1) / (L + 1)));
      uint64_t key[4];
      if constexpr (codes)
        pack6_fast(chunk32, start, L, lanes, key);
      else
        pack_from_smem(chunk32, start, L, lanes, key);
      store_key(keys + s_dst[L - 1] + (uint64_t)k * key_bytes(lanes), lanes, key);
    }
  }
}

// Payload-mode text ingest, word-parallel (6-bit keys). The per-byte front
// end classifies and encodes 32 bytes per thread; after it, every per-word
// step runs on full warps over a per-warp word list instead of one thread per
// byte segment looping over its own words (which left half of the lanes idle):
//   A  classify, 6-bit codes -> smem, start / end masks (ends -> smem), warp
//      scan of the start counts, each thread lists its starts (the only
//      per-thread loop left: one shared store per word)
//   C  per listed word: length from the end masks (a word may run into later
//      segments, rarely past the chunk), bin, rank in the warp's bin (shared
//      atomic on a warp-private counter); L > 32 goes straight to the long list
//   D  warp bin-major order: exclusive scan of the warp's 32 bin counts
//      (lane = bin), every word moved to its bin-major slot (16-bit entries)
//   CTA  per bin: one global atomic reserves the chunk's run; each warp's
//      sub-run gets its key address
//   E  pack + store in warp bin-major order: a 32-word batch spans 1-3 bins,
//      so lanes store to consecutive addresses and share one packing path.
// Word starts are warp-local byte offsets (0..1023); the CTA's chunk is 8 KiB.
constexpr int kW6Threads = 256;
constexpr int kW6Warps = kW6Threads / 32;
constexpr int kW6SB = 32;                          // bytes per thread
constexpr int kW6CB = kW6SB * kW6Threads;          // chunk bytes
constexpr int kW6WB = kW6SB * 32;                  // bytes per warp
constexpr int kW6MaxWords = kW6WB / 2;             // words per warp at most
constexpr uint32_t kW6Long = 0x80000000u;          // word-list flag: L > 32 (done in C)
constexpr int kW6OrdCap = kW6MaxWords + 4 * 32;    // + each lane class padded to 32 entries
constexpr uint16_t kW6Pad = 0xFFFFu;               // padding entry of ord

struct W6Smem {
  uint32_t codes[(kW6CB + 64) / 4];                // 6-bit codes, one byte per text byte
  uint32_t ends[kW6Threads + 1];                   // per-thread end masks (+ a zero one)
  uint32_t wl[kW6Warps][kW6MaxWords];              // word list: start | bin << 10 | pos << 15
  uint16_t ord[kW6Warps][kW6OrdCap];               // class-aligned bin-major: start | bin << 10
  uint32_t wcnt[kW6Warps][32];                     // per-warp bin counters
  uint32_t wboff[kW6Warps][32];                    // per-warp bin-major offsets
  unsigned long long dst[kW6Warps][32];            // key address of (warp, bin) slot 0
  uint32_t edge_first[kW6Warps], edge_last[kW6Warps];  // alnum masks of lanes 0 / 31
  uint32_t wtot[kW6Warps];
};

// Length of a word that runs past the end of its thread's segment (rare path):
// `len` bytes so far, continuing at segment t.
__device__ __noinline__ uint32_t w6_long_tail(const W6Smem& sm, uint32_t t, uint32_t len,
                                              const uint8_t* __restrict__ text, uint64_t cbase,
                                              uint64_t avail, unsigned int* overflow) {
  for (; t < (uint32_t)kW6Threads; ++t) {
    const uint32_t e = sm.ends[t];
    if (e) return len + (uint32_t)__ffs(e);
    len += 32;
  }
  return len + run_length_from(text, cbase + kW6CB, avail, overflow);
}

__global__ void __launch_bounds__(kW6Threads)
ingest6_kernel(const uint8_t* __restrict__ text, uint64_t n, ScatterParams p) {
  extern __shared__ __align__(16) uint8_t w6_raw[];
  W6Smem& sm = *reinterpret_cast<W6Smem*>(w6_raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t chunk = p.chunk0 + blockIdx.x;
  const uint64_t cbase = chunk * kW6CB;
  const uint64_t base = cbase + (uint64_t)tid * kW6SB;
  const uint64_t avail = p.avail ? p.avail : ~0ull;

  // ---- A: classify, codes, masks ------------------------------------------------
  uint4 v0 = make_uint4(0, 0, 0, 0), v1 = v0;
  if (base < n) {
    v0 = WS_TEXT_LD(reinterpret_cast<const uint4*>(text + base));
    v1 = WS_TEXT_LD(reinterpret_cast<const uint4*>(text + base) + 1);
  }
  const uint32_t m = alnum_mask16(v0) | (alnum_mask16(v1) << 16);
  reinterpret_cast<uint4*>(sm.codes)[2 * tid] = alnum6_codes16(v0);
  reinterpret_cast<uint4*>(sm.codes)[2 * tid + 1] = alnum6_codes16(v1);
  if (tid < 4) {  // codes of the bytes after the chunk (words crossing its end)
    const uint64_t a = cbase + kW6CB + 16 * tid;
    const uint4 la = a < n ? *reinterpret_cast<const uint4*>(text + a) : make_uint4(0, 0, 0, 0);
    reinterpret_cast<uint4*>(sm.codes)[kW6CB / 16 + tid] = alnum6_codes16(la);
  }
  for (int i = tid; i < kW6Warps * 32; i += kW6Threads) (&sm.wcnt[0][0])[i] = 0;
  if (tid == 0) sm.ends[kW6Threads] = 0;  // past the chunk: the rare path measures in global memory
  if (lane == 0) sm.edge_first[wid] = m;
  if (lane == 31) sm.edge_last[wid] = m;
  uint32_t prev = __shfl_up_sync(0xffffffffu, m, 1) >> 31;
  uint32_t next = __shfl_down_sync(0xffffffffu, m, 1) & 1u;
  uint32_t gprev = 0, gnext = 0;  // the chunk's outer neighbours (global bytes)
  if (tid == 0 && base > 0 && base - 1 < n) gprev = is_alnum_byte(text[base - 1]);
  if (tid == kW6Threads - 1 && base + kW6SB < n) gnext = is_alnum_byte(text[base + kW6SB]);
  __syncthreads();  // #1: codes, edge masks, zeroed counters
  if (lane == 0) prev = wid == 0 ? gprev : sm.edge_last[wid - 1] >> 31;
  if (lane == 31) next = wid == kW6Warps - 1 ? gnext : sm.edge_first[wid + 1] & 1u;
  const uint32_t starts = m & ~((m << 1) | prev);
  sm.ends[tid] = m & ~((m >> 1) | (next << 31));
  const uint32_t c = __popc(starts);
  uint32_t incl = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  const uint32_t ww = __shfl_sync(0xffffffffu, incl, 31);  // words of the warp
  {
    uint32_t slot = incl - c;
    for (uint32_t s = starts; s; s &= s - 1) sm.wl[wid][slot++] = (uint32_t)(lane * 32 + __ffs(s) - 1);
  }
  if (lane == 0) sm.wtot[wid] = ww;
  __syncthreads();  // #2: every segment's end mask (words run across segments)

  // ---- C: length, bin, rank in the warp's bin -----------------------------------
  for (uint32_t j0 = 0; j0 < ww; j0 += 32) {
    const uint32_t j = j0 + lane;
    if (j < ww) {
      const uint32_t st = sm.wl[wid][j];
      const uint32_t t = (uint32_t)wid * 32 + (st >> 5), i = st & 31;
      // the word ends in its own segment or in the next one (branch-free);
      // longer runs (and the chunk's last word) take the rare path
      const uint32_t r = sm.ends[t] >> i, e1 = sm.ends[t + 1];
      const uint32_t x = r ? r : e1;
      uint32_t L = (uint32_t)__ffs(x) + (r ? 0u : 32u - i);
      if (x == 0) L = w6_long_tail(sm, t + 1, 32 - i, text, cbase, avail, p.overflow);
      if (L <= (uint32_t)kMaxPackedLen) {
        const uint32_t bin = L - 1;
        const uint32_t pos = atomicAdd(&sm.wcnt[wid][bin], 1u);
        sm.wl[wid][j] = st | (bin << 10) | (pos << 15);
      } else {  // long word: (start, len) straight into the long list (rare)
        sm.wl[wid][j] = kW6Long;
        if (p.keys) {
          const uint32_t at = atomicAdd(p.fill + kLongBin, 1u);
          p.longlist[at] = make_uint2((uint32_t)(cbase + (uint64_t)wid * kW6WB + st), L);
        } else {
          atomicAdd(p.fill + kLongBin, 1u);
        }
      }
    }
  }
  __syncwarp();

  // ---- D: warp bin-major order, each lane class starting at a multiple of 32 ------
  // (a batch of 32 entries then holds one class: one packing path, one key width)
  const uint32_t bc = sm.wcnt[wid][lane];
  uint32_t binc = bc;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, binc, d);
    if (lane >= d) binc += t;
  }
  // lane classes of 6-bit keys: bins 0-4 | 5-9 | 10-20 | 21-31
  const uint32_t e0 = __shfl_sync(0xffffffffu, binc, 4), e1c = __shfl_sync(0xffffffffu, binc, 9),
                 e2 = __shfl_sync(0xffffffffu, binc, 20), e3 = __shfl_sync(0xffffffffu, binc, 31);
  const uint32_t p1 = (e0 + 31) & ~31u, p2 = p1 + ((e1c - e0 + 31) & ~31u),
                 p3 = p2 + ((e2 - e1c + 31) & ~31u), pend = p3 + ((e3 - e2 + 31) & ~31u);
  const uint32_t cls = lane < 5 ? 0u : lane < 10 ? 1u : lane < 21 ? 2u : 3u;
  const uint32_t cstart = cls == 0 ? 0u : cls == 1 ? e0 : cls == 2 ? e1c : e2;   // class's first word (unpadded)
  const uint32_t cbase_p = cls == 0 ? 0u : cls == 1 ? p1 : cls == 2 ? p2 : p3;  // ... padded
  const uint32_t wboff = cbase_p + (binc - bc - cstart);
  sm.wboff[wid][lane] = wboff;
  for (uint32_t k = lane; k < pend; k += 32) sm.ord[wid][k] = kW6Pad;
  __syncwarp();
  for (uint32_t j0 = 0; j0 < ww; j0 += 32) {
    const uint32_t j = j0 + lane;
    const uint32_t e = j < ww ? sm.wl[wid][j] : kW6Long;
    const uint32_t bin = (e >> 10) & 31;
    const uint32_t off = __shfl_sync(0xffffffffu, wboff, (int)bin);
    if (!(e & kW6Long)) sm.ord[wid][off + (e >> 15)] = (uint16_t)(e & 0x7FFFu);
  }
  __syncthreads();  // #3: every warp's bin counts and offsets

  // ---- CTA: reserve each bin's run, key address of every (warp, bin) sub-run -----------
  if (tid < 32) {
    const uint32_t b = tid;
    uint32_t total = 0;
#pragma unroll
    for (int w = 0; w < kW6Warps; ++w) total += sm.wcnt[w][b];
    uint32_t run = total ? atomicAdd(p.fill + b, total) : 0u;
    const uint64_t ks = (uint64_t)key_bytes(lanes_for_len_enc((int)b + 1, kEncAlnum6));
    const uint64_t bb = p.bin_base[b];
#pragma unroll
    for (int w = 0; w < kW6Warps; ++w) {
      sm.dst[w][b] = bb + ((uint64_t)run - sm.wboff[w][b]) * ks;  // modular: slot k at + k * ks
      run += sm.wcnt[w][b];
    }
    uint32_t words = lane < kW6Warps ? sm.wtot[lane] : 0u;
    words = __reduce_add_sync(0xffffffffu, words);
    if (lane == 0 && words) atomicAdd(p.fill + kNumBins, words);
  }
  __syncthreads();  // #4

  // ---- E: pack + store, one lane class per batch ------------------------------------
  if (!p.keys) return;
  uint8_t* keys = reinterpret_cast<uint8_t*>(p.keys);
  const uint32_t cw = (uint32_t)wid * kW6WB;
  for (uint32_t k = lane; k < p1; k += 32) {  // class 0: L <= 5, one uint32
    const uint32_t e = sm.ord[wid][k];
    if (e == kW6Pad) continue;
    const uint32_t st = cw + (e & 1023u), bin = e >> 10;
    uint64_t key[4];
    pack6_fast(sm.codes, st, bin + 1, 0, key);
    *reinterpret_cast<uint32_t*>(keys + sm.dst[wid][bin] + (uint64_t)k * 4) = (uint32_t)(key[0] >> 32);
  }
  for (uint32_t k = p1 + lane; k < p2; k += 32) {  // class 1: L 6-10, one uint64
    const uint32_t e = sm.ord[wid][k];
    if (e == kW6Pad) continue;
    const uint32_t st = cw + (e & 1023u), bin = e >> 10;
    uint64_t key[4];
    pack6_fast(sm.codes, st, bin + 1, 1, key);
    *reinterpret_cast<uint64_t*>(keys + sm.dst[wid][bin] + (uint64_t)k * 8) = key[0];
  }
  for (uint32_t k = p2 + lane; k < pend; k += 32) {  // classes 2-3: L 11-32, 2-3 uint64
    const uint32_t e = sm.ord[wid][k];
    if (e == kW6Pad) continue;
    const uint32_t st = cw + (e & 1023u), bin = e >> 10, L = bin + 1;
    const int lanes = lanes_for_len_enc((int)L, kEncAlnum6);
    uint64_t key[4];
    pack6_from_codes(sm.codes, st, L, lanes, key);
    store_key(keys + sm.dst[wid][bin] + (uint64_t)k * key_bytes(lanes), lanes, key);
  }
}

// Payload-mode text ingest, 6-bit keys (the default; reserve_ingest_kernel is
// the A/B arm). Measured per SASS region on config 4 (tools/ncu_sass_phases.py,
// profiles/r02_ncu_ingest_*), reserve_ingest_kernel spends ~30 % of its
// instructions on the front end (a third of that on the segmented suffix scan
// that measures words running past a thread's segment), ~36 % on two divergent
// per-thread word loops (count, then place) at ~55 % lane utilisation, and
// ~32 % on packing keys from per-byte codes. This kernel:
//   A  32 bytes per thread: byte classes, start / end masks; a word running
//      past the thread's 32 bytes ends in the next thread's leading alnum run
//      (one shuffle), or else is longer than 32 and takes the rare path (the
//      long list); the 6-bit codes are compressed into one big-endian bit
//      string per chunk in shared memory (6 words per thread)
//   B  one divergent loop per thread over its words: length, bin, a shared
//      reduction on the bin's counter, the word (start | bin) appended to the
//      warp's list (slot = warp prefix of the thread's start count)
//   D  per bin, one global atomic reserves the chunk's run; bin-major cursors
//   P  full-lane pass over each warp's list: slot in the bin-major order from
//      the bin's cursor (shared atomic), entry stored there
//   E  per lane class (bins 0-4 | 5-9 | 10-20 | 21-31, contiguous in bin-major
//      order), 256 words per step: the key is a funnel-shifted window of the
//      bit string (2, 3, 5 or 7 shared loads), masked to L characters, stored
//      to consecutive addresses.
constexpr int kI7Threads = 256;
constexpr int kI7Warps = kI7Threads / 32;
constexpr int kI7SB = 32;                          // bytes per thread
constexpr int kI7CB = kI7SB * kI7Threads;          // chunk bytes (== reserve_chunk_bytes())
constexpr int kI7MaxWords = kI7SB * 32 / 2;        // words per warp at most
constexpr uint32_t kI7Skip = 0xFFFFFFFFu;          // list entry of an L > 32 word
constexpr int kI7Tail = 2;                         // 32-byte segments of codes past the chunk
constexpr int kI7Bits = 6 * (kI7Threads + kI7Tail) + 8;  // bit-string words (+ read slack)

struct I7Smem {
  uint32_t bits[kI7Bits];                          // 6-bit codes as one big-endian bit string
  uint32_t wl[kI7Warps][kI7MaxWords];              // chunk start | bin << 13 (word order)
  uint16_t ord[kI7Warps * kI7MaxWords];            // bin-major order: index into wl
  uint32_t cnt[kHistRows];
  uint32_t cur[kNumBins];
  uint32_t base[kHistRows];
  uint32_t boff[kMaxPackedLen + 1];
  unsigned long long dst[kMaxPackedLen];
  uint32_t first[kI7Warps], last[kI7Warps];        // lane 0 (alnum mask, leading run) / lane 31 masks
  uint32_t wcnt[kI7Warps][kHistRows];              // ORDERED: per-warp bin counts -> warp cursors
};

// 32 text bytes (8 little-endian words) -> their 6-bit codes as 192 bits of a
// big-endian bit string (first character in the top bits of w[0]).
__device__ __forceinline__ void i7_bitstring(const uint4 (&v)[2], uint32_t (&w)[6]) {
  uint32_t c[8];
  const uint32_t x[8] = {v[0].x, v[0].y, v[0].z, v[0].w, v[1].x, v[1].y, v[1].z, v[1].w};
#pragma unroll
  for (int k = 0; k < 8; ++k) c[k] = codes24(alnum6_codes4(x[k]));
  w[0] = (c[0] << 8) | (c[1] >> 16);
  w[1] = (c[1] << 16) | (c[2] >> 8);
  w[2] = (c[2] << 24) | c[3];
  w[3] = (c[4] << 8) | (c[5] >> 16);
  w[4] = (c[5] << 16) | (c[6] >> 8);
  w[5] = (c[6] << 24) | c[7];
}

// Bits [b, b + 32 * NW) of the string, NW words.
template <int NW>
__device__ __forceinline__ void i7_window(const uint32_t* __restrict__ bits, uint32_t b,
                                          uint32_t (&o)[NW]) {
  const uint32_t q = b >> 5, sh = b & 31u;
  uint32_t prev = bits[q];
#pragma unroll
  for (int k = 0; k < NW; ++k) {
    const uint32_t nx = bits[q + k + 1];
    o[k] = __funnelshift_l(nx, prev, sh);
    prev = nx;
  }
}

#ifndef WS_I7_PAGG
#define WS_I7_PAGG 0  // payload placement pass: 1 = warp-aggregated cursor atomics (MATCH.ANY)
#endif
#ifndef WS_I7_MINB
#define WS_I7_MINB 7  // 32 registers (A/B: 5 -> 160 us, 6 -> 149, 7-8 -> 143 on config 4)
#endif
// ORDERED (stats mode, ScatterParams::run_at set): words keep corpus order
// inside the chunk's run of every bin, counted per warp; the placement pass
// ranks each warp's words by one MATCH.ANY per round against the warp's
// cursors (warp order = corpus order), long words go to the long list at their
// stable place, and each bin's run is recorded per chunk for
// reorder_runs_kernel, which moves the runs into corpus order.
template <bool ORDERED>
__global__ void __launch_bounds__(kI7Threads, WS_I7_MINB)
ingest7_kernel(const uint8_t* __restrict__ text, uint64_t n, ScatterParams p) {
  extern __shared__ __align__(16) uint8_t i7_raw[];
  I7Smem& sm = *reinterpret_cast<I7Smem*>(i7_raw);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t chunk = p.chunk0 + blockIdx.x;
  const uint64_t cbase = chunk * kI7CB;
  const uint64_t base = cbase + (uint64_t)tid * kI7SB;
  const uint64_t avail = p.avail ? p.avail : ~0ull;
  if (tid < kHistRows) sm.cnt[tid] = 0;
  if (ORDERED)
    for (int i = tid; i < kI7Warps * kHistRows; i += kI7Threads) (&sm.wcnt[0][0])[i] = 0;

  // ---- A ---------------------------------------------------------------------
  uint4 v[2];
  v[0] = v[1] = make_uint4(0, 0, 0, 0);
  if (base < n) {  // padded text; streamed once (evict-first)
    v[0] = WS_TEXT_LD(reinterpret_cast<const uint4*>(text + base));
    v[1] = WS_TEXT_LD(reinterpret_cast<const uint4*>(text + base) + 1);
  }
  const uint32_t m = alnum_mask16(v[0]) | (alnum_mask16(v[1]) << 16);
  const uint32_t lead = m == 0xFFFFFFFFu ? 32u : (uint32_t)__ffs(~m) - 1;  // leading alnum bytes
  {
    uint32_t w[6];
    i7_bitstring(v, w);
    uint2* d = reinterpret_cast<uint2*>(sm.bits + 6 * tid);
    d[0] = make_uint2(w[0], w[1]);
    d[1] = make_uint2(w[2], w[3]);
    d[2] = make_uint2(w[4], w[5]);
  }
  if (tid < kI7Tail) {  // codes of the bytes after the chunk (words crossing its end)
    const uint64_t a = cbase + kI7CB + (uint64_t)kI7SB * tid;
    uint4 t[2];
    t[0] = a < n ? *reinterpret_cast<const uint4*>(text + a) : make_uint4(0, 0, 0, 0);
    t[1] = a + 16 < n ? *reinterpret_cast<const uint4*>(text + a + 16) : make_uint4(0, 0, 0, 0);
    uint32_t w[6];
    i7_bitstring(t, w);
#pragma unroll
    for (int k = 0; k < 6; ++k) sm.bits[6 * (kI7Threads + tid) + k] = w[k];
  } else if (tid < kI7Tail + 8) {
    sm.bits[6 * (kI7Threads + kI7Tail) + tid - kI7Tail] = 0;
  }
  if (lane == 0) sm.first[wid] = lead;
  if (lane == 31) sm.last[wid] = m >> 31;
  uint32_t prev = __shfl_up_sync(0xffffffffu, m, 1) >> 31;
  uint32_t nlead = __shfl_down_sync(0xffffffffu, lead, 1);  // next segment's leading alnum run
  __syncthreads();  // #1: edge masks, counters
  if (lane == 0)
    prev = wid > 0 ? sm.last[wid - 1] : ((base > 0 && base - 1 < n) ? (uint32_t)is_alnum_byte(text[base - 1]) : 0u);
  if (lane == 31) {
    if (wid < kI7Warps - 1) {
      nlead = sm.first[wid + 1];
    } else {  // past the chunk: the next byte decides; a longer run is measured lazily
      nlead = (base + kI7SB < n && is_alnum_byte(text[base + kI7SB])) ? 32u : 0u;
    }
  }
  const uint32_t starts = m & ~((m << 1) | prev);
  const uint32_t ends = m & ~((m >> 1) | ((nlead != 0) << 31));

  // ---- B ---------------------------------------------------------------------
  const uint32_t nst = (uint32_t)__popc(starts);
  uint32_t incl = nst;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += t;
  }
  const uint32_t ww = __shfl_sync(0xffffffffu, incl, 31);  // words of the warp
  uint32_t* wl = sm.wl[wid] + (incl - nst);
  for (uint32_t s = starts; s; s &= s - 1) {
    const uint32_t i = (uint32_t)__ffs(s) - 1;
    const uint32_t r = ends >> i;
    uint32_t L = r ? (uint32_t)__ffs(r) : (32u - i) + nlead;
    if (L > (uint32_t)kMaxPackedLen) {  // rare
      if (!r && nlead == 32u) {
        // runs on past the next segment's first byte (the chunk's last thread
        // only knows that byte) or through it: measured up to a bound; longer
        // words get length 0 here and are measured after the ingest
        const uint32_t more = bounded_run_length(text, base + kI7SB, kLongScan, avail, p.overflow);
        L = more == ~0u ? 0u : (32u - i) + more;
      }
      if (L - 1u >= (uint32_t)kMaxPackedLen) {  // L == 0 or L > 32: the long list
        if (ORDERED) {  // placed (stably) by the placement pass, which measures it again
          atomicAdd(&sm.wcnt[wid][kLongBin], 1u);
          *wl++ = ((uint32_t)tid * kI7SB + i) | ((uint32_t)kLongBin << 13);
        } else {
          if (!L && p.unknown) atomicAdd(p.unknown, 1u);
          const uint32_t at = atomicAdd(p.fill + kLongBin, 1u);
          if (p.keys) p.longlist[at] = make_uint2((uint32_t)(base + i), L);
          *wl++ = kI7Skip;
        }
        continue;
      }
    }
    atomicAdd(ORDERED ? &sm.wcnt[wid][L - 1] : &sm.cnt[L - 1], 1u);
    *wl++ = ((uint32_t)tid * kI7SB + i) | ((L - 1) << 13);
  }
  if (lane == 0 && ww) atomicAdd(ORDERED ? &sm.wcnt[wid][kNumBins] : &sm.cnt[kNumBins], ww);
  __syncthreads();  // #2: the chunk's bin counts
  if (ORDERED && tid < kHistRows) {  // per bin: warp offsets inside the chunk's run, the chunk's count
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < kI7Warps; ++w) {
      const uint32_t c = sm.wcnt[w][tid];
      sm.wcnt[w][tid] = run;
      run += c;
    }
    sm.cnt[tid] = run;
  }
  if (ORDERED) __syncthreads();

  // ---- D ---------------------------------------------------------------------
  if (ORDERED) {
    if (tid < kHistRows) {  // reserve the runs, record them for the reorder
      const uint32_t cnt = sm.cnt[tid];
      const uint32_t at = cnt ? atomicAdd(p.fill + tid, cnt) : 0u;
      sm.base[tid] = at;
      p.run_at[(uint64_t)tid * p.nchunks_total + chunk] = at;
      p.run_cnt[(uint64_t)tid * p.nchunks_total + chunk] = cnt;
    }
  } else {
    if (tid < kMaxPackedLen && sm.cnt[tid]) sm.base[tid] = atomicAdd(p.fill + tid, sm.cnt[tid]);
    if (tid == kNumBins && sm.cnt[kNumBins]) atomicAdd(p.fill + kNumBins, sm.cnt[kNumBins]);
  }
  if (wid == 1) {  // bin-major offsets (lane = bin) = the bins' cursors
    const uint32_t c = sm.cnt[lane];
    uint32_t inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += t;
    }
    sm.boff[lane] = inc - c;
    sm.cur[lane] = inc - c;
    if (lane == 31) sm.boff[kMaxPackedLen] = inc;
  }
  __syncthreads();  // #3
  if (tid < kMaxPackedLen) {
    const uint64_t ks = (uint64_t)key_bytes(lanes_for_len_enc(tid + 1, kEncAlnum6));
    WS_DCHECK((uint64_t)sm.base[tid] + sm.cnt[tid] <= (n + 1) / (uint64_t)(tid + 2) || !sm.cnt[tid]);
    sm.dst[tid] = p.bin_base[tid] + ((uint64_t)sm.base[tid] - sm.boff[tid]) * ks;  // modular
  }

  // ---- P ---------------------------------------------------------------------
  if (ORDERED) {  // stable: rounds in word order, warp cursors (after every earlier warp's words)
    const uint32_t lt = (1u << lane) - 1u;
    uint32_t* cur = sm.wcnt[wid];
    for (uint32_t j0 = 0; j0 < ww; j0 += 32) {
      const uint32_t j = j0 + lane;
      const uint32_t e = j < ww ? sm.wl[wid][j] : 0u;
      const uint32_t bin = j < ww ? e >> 13 : 64u + (uint32_t)lane;  // no word: matches nobody
      const uint32_t peers = __match_any_sync(0xffffffffu, bin);
      const uint32_t c0 = j < ww ? cur[bin] : 0u;
      const uint32_t rank = c0 + (uint32_t)__popc(peers & lt);
      __syncwarp();
      if (j < ww && !(peers & lt)) cur[bin] = c0 + (uint32_t)__popc(peers);
      if (j < ww) {
        if (bin < (uint32_t)kMaxPackedLen) {
          WS_DCHECK(sm.boff[bin] + rank < sm.boff[bin + 1]);
          sm.ord[sm.boff[bin] + rank] = (uint16_t)(wid * kI7MaxWords + j);
        } else if (p.keys) {  // long word (rare): its length again, its stable slot in the long list
          const uint32_t st = e & 8191u;
          const uint32_t L0 = bounded_run_length(text, cbase + st, kLongScan, avail, p.overflow);
          const uint32_t L = L0 == ~0u ? 0u : L0;  // 0: measured after the ingest
          if (!L && p.unknown) atomicAdd(p.unknown, 1u);
          p.longlist[sm.base[kLongBin] + rank] = make_uint2((uint32_t)(cbase + st), L);
        }
      }
      __syncwarp();
    }
  } else if (WS_I7_PAGG) {  // warp-aggregated cursor atomics: one per distinct bin per round
    const uint32_t lt = (1u << lane) - 1u;
    for (uint32_t j0 = 0; j0 < ww; j0 += 32) {
      const uint32_t j = j0 + lane;
      const uint32_t e = j < ww ? sm.wl[wid][j] : kI7Skip;
      const uint32_t key = e == kI7Skip ? 64u + (uint32_t)lane : e >> 13;
      const uint32_t peers = __match_any_sync(0xffffffffu, key);
      const int leader = __ffs(peers) - 1;
      uint32_t base = 0;
      if (e != kI7Skip && lane == leader) base = atomicAdd(&sm.cur[key], (uint32_t)__popc(peers));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (e != kI7Skip) {
        const uint32_t at = base + (uint32_t)__popc(peers & lt);
        WS_DCHECK(at < sm.boff[kMaxPackedLen]);
        sm.ord[at] = (uint16_t)(wid * kI7MaxWords + j);
      }
    }
  } else {
    for (uint32_t j = lane; j < ww; j += 32) {
      const uint32_t e = sm.wl[wid][j];
      if (e == kI7Skip) continue;
      const uint32_t at = atomicAdd(&sm.cur[e >> 13], 1u);
      WS_DCHECK(at < sm.boff[kMaxPackedLen]);
      sm.ord[at] = (uint16_t)(wid * kI7MaxWords + j);
    }
  }
  __syncthreads();  // #4: bin-major order, key addresses

  // ---- E ---------------------------------------------------------------------
  if (!p.keys) return;
  uint8_t* keys = reinterpret_cast<uint8_t*>(p.keys);
  const uint32_t e1 = sm.boff[5], e2 = sm.boff[10], e3 = sm.boff[21], e4 = sm.boff[kMaxPackedLen];
  for (uint32_t k = tid; k < e1; k += kI7Threads) {  // class 0: L <= 5, the top 30 bits of a uint32
    const uint32_t e = (&sm.wl[0][0])[sm.ord[k]], st = e & 8191u, bin = e >> 13;
    uint32_t o[1];
    i7_window<1>(sm.bits, 6 * st, o);
    const uint32_t key = o[0] & (~0u << (26 - 6 * bin));
    *reinterpret_cast<uint32_t*>(keys + sm.dst[bin] + (uint64_t)k * 4) = key;
  }
  for (uint32_t k = e1 + tid; k < e2; k += kI7Threads) {  // class 1: L 6-10, one uint64
    const uint32_t e = (&sm.wl[0][0])[sm.ord[k]], st = e & 8191u, bin = e >> 13;
    uint32_t o[2];
    i7_window<2>(sm.bits, 6 * st, o);
    const uint64_t key = (((uint64_t)o[0] << 32) | o[1]) & (~0ull << (58 - 6 * bin));
    *reinterpret_cast<uint64_t*>(keys + sm.dst[bin] + (uint64_t)k * 8) = key;
  }
  for (uint32_t k = e2 + tid; k < e3; k += kI7Threads) {  // class 2: L 11-21, two uint64
    const uint32_t e = (&sm.wl[0][0])[sm.ord[k]], st = e & 8191u, bin = e >> 13;
    uint32_t o[4];
    i7_window<4>(sm.bits, 6 * st, o);
    const uint64_t k1 = (((uint64_t)o[2] << 32) | o[3]) & (~0ull << (122 - 6 * bin));
    uint64_t* d = reinterpret_cast<uint64_t*>(keys + sm.dst[bin] + (uint64_t)k * 16);
    d[0] = ((uint64_t)o[0] << 32) | o[1];
    d[1] = k1;
  }
  for (uint32_t k = e3 + tid; k < e4; k += kI7Threads) {  // class 3: L 22-32, three uint64
    const uint32_t e = (&sm.wl[0][0])[sm.ord[k]], st = e & 8191u, bin = e >> 13;
    uint32_t o[6];
    i7_window<6>(sm.bits, 6 * st, o);
    const uint32_t bits = 6 * (bin + 1);  // 132..192
    const uint64_t k2 = ((uint64_t)o[4] << 32) | o[5];
    uint64_t* d = reinterpret_cast<uint64_t*>(keys + sm.dst[bin] + (uint64_t)k * 24);
    d[0] = ((uint64_t)o[0] << 32) | o[1];
    d[1] = ((uint64_t)o[2] << 32) | o[3];
    d[2] = bits >= 192u ? k2 : k2 & (~0ull << (192u - bits));
  }
}

// kByReserve follow-up: one CTA per chunk moves the chunk's runs (one per
// bin) from their reserved place (the bin's ingest region / the long list as
// filled) to their corpus-order place (run_off = exclusive scan of run_cnt
// over chunks) in the destination layout. Thread k copies element k of the
// chunk's runs laid end to end (the run by a search over 33 prefix counts),
// so small runs do not leave lanes idle.
__global__ void __launch_bounds__(kIngestThreads)
reorder_runs_kernel(ReorderParams r) {
  pdl_wait();
  __shared__ uint32_t s_pre[kNumBins + 1];
  __shared__ uint32_t s_from[kNumBins], s_to[kNumBins];
  const int tid = threadIdx.x;
  const uint64_t chunk = blockIdx.x;
  if (tid < 32) {  // bins 0..31 in lanes, bin 32 folded into lane 31's second value
    const uint64_t cell = (uint64_t)tid * r.nchunks + chunk;
    const uint64_t cell2 = (uint64_t)kLongBin * r.nchunks + chunk;
    const uint32_t c = r.run_cnt[cell];
    uint32_t inc = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, inc, d);
      if (tid >= d) inc += t;
    }
    s_pre[tid] = inc - c;
    s_from[tid] = r.run_at[cell];
    s_to[tid] = r.run_off[cell];
    if (tid == 31) {
      s_pre[kLongBin] = inc;
      s_pre[kNumBins] = inc + r.run_cnt[cell2];
      s_from[kLongBin] = r.run_at[cell2];
      s_to[kLongBin] = r.run_off[cell2];
    }
  }
  __syncthreads();
  // one warp per run (runs b = w, w + 8, ...): a run is contiguous at both
  // ends, so its 4-byte words are copied coalesced with no per-element search
  const int lane = tid & 31, wid = tid >> 5;
  for (int b = wid; b <= kLongBin; b += kIngestThreads / 32) {
    const uint32_t cnt = s_pre[b + 1] - s_pre[b];
    if (!cnt) continue;
    const uint32_t kw = r.key_bytes[b] >> 2;
    const uint32_t* src = reinterpret_cast<const uint32_t*>(r.src[b]) + (uint64_t)s_from[b] * kw;
    uint32_t* dst = reinterpret_cast<uint32_t*>(r.dst[b]) + (uint64_t)s_to[b] * kw;
    const uint32_t words = cnt * kw;
    uint32_t q = lane;
    for (; q + 96 < words; q += 128) {  // four independent loads in flight per lane
      const uint32_t v0 = src[q], v1 = src[q + 32], v2 = src[q + 64], v3 = src[q + 96];
      dst[q] = v0;
      dst[q + 32] = v1;
      dst[q + 64] = v2;
      dst[q + 96] = v3;
    }
    for (; q < words; q += 32) dst[q] = src[q];
  }
}

// ---------------------------------------------------------------------------
// Word-list ingest (build_flat from a Python list): words are given as one
// concatenated byte buffer + lengths. starts = exclusive scan of lengths is
// computed on the host side of the call (cheap) and uploaded with the bytes.

__global__ void words_count_kernel(const uint32_t* __restrict__ lens, uint64_t nwords,
                                   uint32_t* __restrict__ counts /*[kNumBins]*/) {
  __shared__ uint32_t sc[kNumBins];
  if (threadIdx.x < kNumBins) sc[threadIdx.x] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nwords;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t L = lens[i];
    if (L) atomicAdd(&sc[bin_of_len(L)], 1u);
  }
  __syncthreads();
  if (threadIdx.x < kNumBins && sc[threadIdx.x]) atomicAdd(&counts[threadIdx.x], sc[threadIdx.x]);
}

// Stable scatter of a word list: one warp walks a contiguous range of words
// in order (ranks via __match_any_sync), per-warp per-bin base offsets come
// from a prior count pass over the same ranges (warp_hist) + scan.
__global__ void words_warp_hist_kernel(const uint32_t* __restrict__ lens, uint64_t nwords,
                                       uint32_t words_per_warp, uint32_t* __restrict__ whist,
                                       uint32_t nwarps_total) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  if (gw >= nwarps_total) return;
  uint32_t cnt = 0;  // lane b keeps bin b's count (bins < 32), lane 0 also bin 32
  uint32_t cnt_long = 0;
  uint64_t w0 = gw * words_per_warp, w1 = min(nwords, w0 + words_per_warp);
  for (uint64_t b = w0; b < w1; b += 32) {
    uint64_t j = b + lane;
    uint32_t key = j < w1 ? bin_of_len(lens[j]) : 0xFFFFFFFFu;
    uint32_t peers = __match_any_sync(0xffffffffu, key);
    // every lane learns the count for bin == lane via ballot
#pragma unroll 1
    for (int bin = 0; bin < 32; ++bin) {
      uint32_t m = __ballot_sync(0xffffffffu, key == (uint32_t)bin);
      if (lane == bin) cnt += __popc(m);
    }
    uint32_t ml = __ballot_sync(0xffffffffu, key == (uint32_t)kLongBin);
    cnt_long += __popc(ml);
    (void)peers;
  }
  whist[(uint64_t)lane * nwarps_total + gw] = cnt;
  if (lane == 0) whist[(uint64_t)kLongBin * nwarps_total + gw] = cnt_long;
}

__global__ void words_scatter_kernel(const uint8_t* __restrict__ bytes,
                                     const uint64_t* __restrict__ starts,
                                     const uint32_t* __restrict__ lens, uint64_t nwords,
                                     uint32_t words_per_warp, const uint32_t* __restrict__ woff,
                                     uint32_t nwarps_total, ScatterParams p) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  if (gw >= nwarps_total) return;
  uint32_t base_mine = lane < kNumBins ? woff[(uint64_t)lane * nwarps_total + gw] : 0;
  uint32_t base_long = woff[(uint64_t)kLongBin * nwarps_total + gw];
  uint64_t w0 = gw * words_per_warp, w1 = min(nwords, w0 + words_per_warp);
  for (uint64_t b = w0; b < w1; b += 32) {
    uint64_t j = b + lane;
    uint32_t L = j < w1 ? lens[j] : 0;
    uint32_t key = (j < w1 && L) ? bin_of_len(L) : 0xFFFFFFFFu;
    uint32_t peers = __match_any_sync(0xffffffffu, key);
    uint32_t rank = __popc(peers & ((1u << lane) - 1u));
    // fetch this bin's running base from the lane that owns it
    uint32_t src = key < 32 ? key : 0;
    uint32_t bb = __shfl_sync(0xffffffffu, base_mine, src);
    if (key == (uint32_t)kLongBin) bb = base_long;
    // advance owners' bases
    uint32_t add = 0;
#pragma unroll 1
    for (int bin = 0; bin < 32; ++bin) {
      uint32_t m = __ballot_sync(0xffffffffu, key == (uint32_t)bin);
      if (lane == bin) add = __popc(m);
    }
    uint32_t ml = __ballot_sync(0xffffffffu, key == (uint32_t)kLongBin);
    base_mine += add;
    uint32_t pos = bb + rank;
    base_long += __popc(ml);
    if (key == 0xFFFFFFFFu) continue;
    uint64_t st = starts[j];
    if (key == (uint32_t)kLongBin) {
      p.longlist[pos] = make_uint2((uint32_t)st, L);
      continue;
    }
    const int lanes = lanes_for_len_enc(L, kEncRaw8);
    uint64_t k[4] = {0, 0, 0, 0};
    for (int l = 0; l < (lanes < 1 ? 1 : lanes); ++l) {
      for (int q = 0; q < 8; ++q) {
        uint32_t bi = 8 * l + q;
        uint64_t byte = bi < L ? bytes[st + bi] : 0;
        k[l] |= byte << (56 - 8 * q);
      }
    }
    store_key(reinterpret_cast<uint8_t*>(p.keys) + p.bin_base[key] + (uint64_t)pos * key_bytes(lanes),
              lanes, k);
  }
}

// Rows (n x width) -> packed keys of one segment.
__global__ void pack_rows_kernel(const uint8_t* __restrict__ rows, uint64_t n, uint32_t width,
                                 uint64_t* __restrict__ keys) {
  const int lanes = lanes_for_len_enc(width, kEncRaw8);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint8_t* r = rows + i * width;
    uint64_t k[4] = {0, 0, 0, 0};
    for (int l = 0; l < (lanes < 1 ? 1 : lanes); ++l) {
      for (int q = 0; q < 8; ++q) {
        uint32_t bi = 8 * l + q;
        uint64_t byte = bi < width ? r[bi] : 0;
        k[l] |= byte << (56 - 8 * q);
      }
    }
    store_key(reinterpret_cast<uint8_t*>(keys) + i * key_bytes(lanes), lanes, k);
  }
}

// ---------------------------------------------------------------------------
// launchers

void launch_count(const uint8_t* text, uint64_t n, uint32_t* hist, uint32_t nchunks,
                  cudaStream_t st) {
  if (nchunks) count_kernel<<<nchunks, kIngestThreads, 0, st>>>(text, n, hist, nchunks);
}

void launch_scan(const uint32_t* hist, uint32_t* off, uint32_t* totals, uint32_t nchunks,
                 int rows, cudaStream_t st) {
  launch_pdl(scan_kernel, rows, 1024, 0, st, hist, off, totals, nchunks);
}

void launch_scatter(const uint8_t* text, uint64_t n, const uint32_t* off, uint32_t nchunks,
                    const ScatterParams& p, cudaStream_t st) {
  if (nchunks) scatter_kernel<kByScan><<<nchunks, kIngestThreads, 0, st>>>(text, n, off, nchunks, p);
}

constexpr int kReserveSB = WS_RESERVE_SB;
static_assert(kReserveSB == 32 || kReserveSB == 64, "payload ingest: 32 or 64 bytes per thread");
static size_t reserve_smem_bytes() {
  return (size_t)(kReserveSB * kIngestThreads + 64) + (size_t)kReserveSB * kIngestThreads / 2 * 4;
}

// WSORT_INGEST6=1: the word-parallel payload ingest (ingest6_kernel) instead
// of the segment-loop one (reserve_ingest_kernel); measured slower (more
// instructions: 1510 vs 1177 warp-instructions per KiB of text), kept as an
// A/B arm while the ingest is being reworked.
bool ingest6_enabled() {
  static const bool on = getenv("WSORT_INGEST6") && getenv("WSORT_INGEST6")[0] == '1';
  return on;
}
// WSORT_INGEST=reserve|6|7 picks the payload-mode 6-bit ingest (A/B arms).
static int ingest_variant() {
  static const int v = [] {
    const char* e = getenv("WSORT_INGEST");
    if (e && e[0] == 'r') return 1;
    if (e && e[0] == '7') return 7;
    if (ingest6_enabled() || (e && e[0] == '6')) return 6;
    return 7;
  }();
  return v;
}

void set_ingest_attributes() {
  cudaFuncSetAttribute(ingest6_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(W6Smem));
  cudaFuncSetAttribute(ingest7_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(I7Smem));
  cudaFuncSetAttribute(ingest7_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)sizeof(I7Smem));
  cudaFuncSetAttribute(reserve_ingest_kernel<kReserveSB, kEncAlnum6>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)reserve_smem_bytes());
  cudaFuncSetAttribute(reserve_ingest_kernel<kReserveSB, kEncRaw8>,
                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)reserve_smem_bytes());
}

void launch_ingest_lookback(const uint8_t* text, uint64_t n, uint32_t nchunks,
                            const ScatterParams& p, cudaStream_t st) {
  if (!nchunks) return;
  if (p.fill && p.run_at && p.enc == kEncAlnum6 && ingest_variant() != 1)
    ingest7_kernel<true><<<nchunks, kI7Threads, sizeof(I7Smem), st>>>(text, n, p);
  else if (p.fill && p.run_at)
    scatter_kernel<kByReserve><<<nchunks, kIngestThreads, 0, st>>>(text, n, nullptr, nchunks, p);
  else if (p.fill && p.enc == kEncAlnum6 && ingest_variant() == 6)
    ingest6_kernel<<<nchunks, kW6Threads, sizeof(W6Smem), st>>>(text, n, p);
  else if (p.fill && p.enc == kEncAlnum6 && ingest_variant() == 7)
    ingest7_kernel<false><<<nchunks, kI7Threads, sizeof(I7Smem), st>>>(text, n, p);
  else if (p.fill && p.enc == kEncAlnum6)
    reserve_ingest_kernel<kReserveSB, kEncAlnum6><<<nchunks, kIngestThreads, reserve_smem_bytes(), st>>>(
        text, n, p);
  else if (p.fill)
    reserve_ingest_kernel<kReserveSB, kEncRaw8><<<nchunks, kIngestThreads, reserve_smem_bytes(), st>>>(
        text, n, p);
  else
    scatter_kernel<kByLookback><<<nchunks, kIngestThreads, 0, st>>>(text, n, nullptr, nchunks, p);
}

uint32_t ingest_chunk_bytes() { return kChunk; }
// Chunk of the ordered (stats-mode) text ingest: ingest7_kernel<true>'s 8 KiB,
// or scatter_kernel<kByReserve>'s 4 KiB under WSORT_INGEST=reserve.
uint32_t ordered_chunk_bytes() { return ingest_variant() == 1 ? (uint32_t)kChunk : (uint32_t)kI7CB; }
uint32_t reserve_chunk_bytes() {
  static_assert(kI7CB == kW6CB, "payload-mode chunks");
  return ingest_variant() == 1 ? kReserveSB * kIngestThreads : kI7CB;
}

void launch_reorder_runs(const ReorderParams& r, cudaStream_t st) {
  if (r.nchunks) launch_pdl(reorder_runs_kernel, r.nchunks, kIngestThreads, 0, st, r);
}

uint32_t chunk_count(uint64_t n) { return (uint32_t)((n + kChunk - 1) / kChunk); }

void launch_words_hist(const uint32_t* lens, uint64_t nwords, uint32_t wpw, uint32_t* whist,
                       uint32_t nwarps, cudaStream_t st) {
  if (!nwarps) return;
  uint32_t blocks = (nwarps * 32 + 255) / 256;
  words_warp_hist_kernel<<<blocks, 256, 0, st>>>(lens, nwords, wpw, whist, nwarps);
}

void launch_words_scatter(const uint8_t* bytes, const uint64_t* starts, const uint32_t* lens,
                          uint64_t nwords, uint32_t wpw, const uint32_t* woff, uint32_t nwarps,
                          const ScatterParams& p, cudaStream_t st) {
  if (!nwarps) return;
  uint32_t blocks = (nwarps * 32 + 255) / 256;
  words_scatter_kernel<<<blocks, 256, 0, st>>>(bytes, starts, lens, nwords, wpw, woff, nwarps, p);
}

void launch_pack_rows(const uint8_t* rows, uint64_t n, uint32_t width, uint64_t* keys,
                      cudaStream_t st) {
  if (!n) return;
  uint32_t blocks = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  pack_rows_kernel<<<blocks, 256, 0, st>>>(rows, n, width, keys);
}

// ---- long words the ingest left unmeasured ---------------------------------------
constexpr uint32_t kFixChunk = 8192;

// first_sep[c] = offset of the first non-alnum byte of 8 KiB chunk c (bytes
// past the text count as separators), or ~0u when the chunk is all alnum.
__global__ void __launch_bounds__(256) chunk_first_sep_kernel(const uint8_t* __restrict__ text, uint64_t n,
                                                             uint32_t* __restrict__ first_sep) {
  __shared__ uint32_t s_min;
  if (threadIdx.x == 0) s_min = ~0u;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kFixChunk + (uint64_t)threadIdx.x * 32;
  uint32_t f = ~0u;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const uint64_t q = base + 16 * k;
    if (q >= n) {
      f = min(f, (uint32_t)(threadIdx.x * 32 + 16 * k));
      break;
    }
    const uint32_t m = alnum_mask16(*reinterpret_cast<const uint4*>(text + q));  // padded text
    if (m != 0xFFFFu) {
      f = min(f, (uint32_t)(threadIdx.x * 32 + 16 * k) + (uint32_t)__ffs(~m) - 1);
      break;
    }
  }
  f = __reduce_min_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f != ~0u) atomicMin(&s_min, f);
  __syncthreads();
  if (threadIdx.x == 0) first_sep[blockIdx.x] = s_min;
}

// One warp per long-list entry of length 0: the word's end is the first
// separator after its start + 33 - in the rest of its chunk (512-byte warp
// steps), or else at first_sep of the first later chunk that has one (32
// chunk entries per step).
__global__ void __launch_bounds__(256) long_len_fix_kernel(const uint8_t* __restrict__ text, uint64_t n,
                                                          uint2* __restrict__ longlist, uint64_t m,
                                                          const uint32_t* __restrict__ first_sep) {
  const int lane = threadIdx.x & 31;
  const uint64_t nchunks = (n + kFixChunk - 1) / kFixChunk;
  for (uint64_t e = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < m;
       e += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
    const uint2 w = longlist[e];
    if (w.y != 0) continue;  // warp-uniform
    const uint64_t start = w.x;
    uint64_t end = ~0ull;
    // the rest of the start's chunk, 16 bytes per lane per step
    const uint64_t c0 = start / kFixChunk, cend = min(n, (c0 + 1) * kFixChunk);
    for (uint64_t q0 = (start + 33) & ~15ull; q0 < cend && end == ~0ull; q0 += 512) {
      const uint64_t q = q0 + 16 * (uint64_t)lane;
      uint32_t hit = ~0u;
      if (q < cend) {
        uint32_t mk = alnum_mask16(*reinterpret_cast<const uint4*>(text + q));
        // bytes before start + 33 are inside the word (known alnum)
        if (q < start + 33) mk |= (1u << (uint32_t)(start + 33 - q)) - 1u;
        if (mk != 0xFFFFu) hit = (uint32_t)(q - q0) + (uint32_t)__ffs(~mk) - 1;
      }
      hit = __reduce_min_sync(0xffffffffu, hit);
      if (hit != ~0u) end = q0 + hit;
    }
    // later chunks: the first one with a separator
    for (uint64_t c = c0 + 1; c < nchunks && end == ~0ull; c += 32) {
      const uint64_t cc = c + lane;
      const uint32_t f = cc < nchunks ? first_sep[cc] : ~0u;
      const uint32_t has = __ballot_sync(0xffffffffu, f != ~0u);
      if (has) {
        const int src = __ffs(has) - 1;
        const uint32_t fo = __shfl_sync(0xffffffffu, f, src);
        end = (c + (uint64_t)src) * kFixChunk + fo;
      }
    }
    if (end == ~0ull || end > n) end = n;
    if (lane == 0) longlist[e].y = (uint32_t)(end - start);
  }
}

uint64_t long_fix_chunks(uint64_t n) { return (n + kFixChunk - 1) / kFixChunk; }

void launch_long_len_fix(const uint8_t* text, uint64_t n, uint2* longlist, uint64_t m,
                         uint32_t* first_sep, cudaStream_t st) {
  if (!m || !n) return;
  const uint64_t nc = long_fix_chunks(n);
  chunk_first_sep_kernel<<<(unsigned)nc, 256, 0, st>>>(text, n, first_sep);
  const uint64_t blocks = std::min<uint64_t>((m * 32 + 255) / 256, 148 * 16);
  long_len_fix_kernel<<<(unsigned)blocks, 256, 0, st>>>(text, n, longlist, m, first_sep);
}

WS_DEFINE_CHECK_READER(check_reader_ingest)

}  // namespace ws
