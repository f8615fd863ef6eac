// Shared definitions for libwsort_b200: packed keys, byte classes, segments.
//
// Data layout in HBM:
//   * text       : the corpus bytes, padded with >= 64 zero bytes (zero is a
//                  separator, so scans past the end always terminate).
//   * keys       : one region per length bucket L <= 32, 16-byte aligned;
//                  word i of the bucket is LANES(L) = ceil(L/8) consecutive
//                  uint64 lanes, bytes packed big-endian and zero-padded, so
//                  unsigned integer order == the reference's raw byte order
//                  (compare_words, engine.py:62-69; _bubble_rows byte loop,
//                  engine.py:101-104).
//   * idx        : optional uint32 payload = the word's corpus rank inside its
//                  bucket (stats mode: inversion count, early-exit pass bound).
//   * long words : L > 32 are kept as (start, len) pairs into the byte buffer
//                  and sorted by an LSD pass sequence over 8-byte lanes.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>
#include <utility>

namespace ws {

constexpr int kMaxPackedLen = 32;           // lengths handled by packed keys
constexpr int kLongBin = kMaxPackedLen;     // bin index of the L > 32 class
constexpr int kNumBins = kMaxPackedLen + 1; // bins 0..31 -> L = 1..32, bin 32 = long
constexpr int kHistRows = kNumBins + 1;     // + one row of per-chunk word totals
constexpr int kTextPad = 128;               // zero padding after the text
// Single-pass ingest look-back record per chunk (uint32 words): [0] flag,
// [kRecAgg + r] the chunk's own count of row r, [kRecIncl + r] the inclusive
// prefix of row r. Aggregates and prefixes live apart so a reader that saw
// flag 1 never reads values being overwritten by the later prefix.
constexpr int kRecAgg = 4;        // 16-byte aligned: readers fetch rows as uint4
constexpr int kRecIncl = 40;
constexpr int kLookbackRec = 80;

__host__ __device__ constexpr int lanes_for_len(int L) { return (L + 7) >> 3; }

// Key encodings. Raw: 8 bits per byte (any byte values; rows / word lists).
// Alnum6: text ingest only, where every byte is [0-9A-Za-z]: an order-
// preserving 6-bit code per character ('0'..'9' -> 1..10, 'A'..'Z' -> 11..36,
// 'a'..'z' -> 37..62) packed as one big-endian bit string over the lanes
// (character k at bits [6k, 6k+6) from the top), so L <= 10 -> 1 lane,
// <= 21 -> 2, <= 32 -> 3, and key order == byte order.
enum KeyEnc : int { kEncRaw8 = 0, kEncAlnum6 = 1 };
// Lane class of a word of length L: 0 = one uint32 key word (6-bit text keys
// of <= 5 characters, raw keys of <= 4 bytes), else the number of uint64 lanes.
__host__ __device__ constexpr int lanes_for_len_enc(int L, int enc) {
  return enc == kEncAlnum6 ? (L <= 5 ? 0 : (6 * L + 63) >> 6) : (L <= 4 ? 0 : (L + 7) >> 3);
}
__device__ __forceinline__ uint32_t alnum6_code(uint32_t b) {
  return b >= 0x61u ? b - 0x3Cu : (b >= 0x41u ? b - 0x36u : b - 0x2Fu);
}
__device__ __forceinline__ uint32_t alnum6_byte(uint32_t c) {
  return c >= 37u ? c + 0x3Cu : (c >= 11u ? c + 0x36u : c + 0x2Fu);
}

// Byte class of the reference tokenizer WORD_RE = rb"[A-Za-z0-9]+"
// (ingest.py:15): every other byte, including 0x00 and >= 0x80, separates.
__device__ __forceinline__ bool is_alnum_byte(uint32_t b) {
  uint32_t f = b | 0x20u;
  return (b - 0x30u < 10u) || (f - 0x61u < 26u);
}

// 4 bytes -> 4-bit mask (bit k = byte k is [A-Za-z0-9]) using SWAR range checks.
__device__ __forceinline__ uint32_t alnum_mask4(uint32_t v) {
  const uint32_t hi = v & 0x80808080u;            // bytes >= 0x80 never match
  const uint32_t x = v & 0x7f7f7f7fu;
  // digits: 0x30 <= x <= 0x39
  const uint32_t d = (x + 0x50505050u) & ~(x + 0x46464646u);
  // letters: 0x61 <= (x | 0x20) <= 0x7a
  const uint32_t f = x | 0x20202020u;
  const uint32_t l = (f + 0x1f1f1f1fu) & ~(f + 0x05050505u);
  uint32_t m = (d | l) & 0x80808080u & ~hi;
  // gather bit 7 of each byte into bits 0..3: the multiply by 2^0 + 2^7 +
  // 2^14 + 2^21 lands bits 7, 15, 23, 31 on 28, 29, 30, 31 without carries
  return (m * 0x00204081u) >> 28;
}

__device__ __forceinline__ uint32_t alnum_mask16(uint4 v) {
  return alnum_mask4(v.x) | (alnum_mask4(v.y) << 4) | (alnum_mask4(v.z) << 8) |
         (alnum_mask4(v.w) << 12);
}

// Key word type per lane class: LANES >= 1 -> LANES big-endian uint64 lanes;
// LANES == 0 -> one uint32 (6-bit text keys of <= 5 characters, raw keys of
// <= 4 bytes), which halves the bytes the shortest (most common) words move.
template <int LANES>
struct KeyTraits {
  using W = uint64_t;
  static constexpr int NW = LANES;
};
template <>
struct KeyTraits<0> {
  using W = uint32_t;
  static constexpr int NW = 1;
};
__host__ __device__ constexpr int key_bytes(int lanes) { return lanes == 0 ? 4 : 8 * lanes; }

template <int LANES>
struct Key {
  typename KeyTraits<LANES>::W w[KeyTraits<LANES>::NW];
};

// Branch-free lexicographic compares over the key words (no divergence when
// lanes of a warp decide at different words).
template <int LANES>
__device__ __forceinline__ bool key_lt(const Key<LANES>& a, const Key<LANES>& b) {
  bool lt = a.w[0] < b.w[0], eq = a.w[0] == b.w[0];
#pragma unroll
  for (int i = 1; i < KeyTraits<LANES>::NW; ++i) {
    lt = lt | (eq & (a.w[i] < b.w[i]));
    eq = eq & (a.w[i] == b.w[i]);
  }
  return lt;
}

template <int LANES>
__device__ __forceinline__ bool key_le(const Key<LANES>& a, const Key<LANES>& b) {
  return !key_lt<LANES>(b, a);
}

template <int LANES>
__device__ __forceinline__ Key<LANES> key_max() {
  Key<LANES> k;
#pragma unroll
  for (int i = 0; i < KeyTraits<LANES>::NW; ++i) k.w[i] = ~typename KeyTraits<LANES>::W(0);
  return k;
}

// Character k of a 6-bit packed key (k a compile-time constant when unrolled).
template <int K>
__device__ __forceinline__ uint32_t code6_at(const uint64_t* key) {
  constexpr int bit = 6 * K, w = bit >> 6, o = bit & 63;
  if constexpr (o <= 58) {
    return (uint32_t)(key[w] >> (58 - o)) & 63u;
  } else {
    return (uint32_t)((key[w] << (o - 58)) | (key[w + 1] >> (122 - o))) & 63u;
  }
}

// Checked builds (make CHECKED=1 -> -DWS_CHECKED=1, tools/checked_build.sh):
// WS_DCHECK(cond) records the first failing source line of this translation
// unit in a device flag (no trap: the kernel keeps running and the context
// stays usable), and ws_debug_checks() (include/wsort.h) reads and clears
// the flags of every unit. The shipped build compiles the checks away.
// (compute-sanitizer is closed on the GPU pool; these bounds checks on every
// computed shared / global index are the memory-safety evidence instead.)
#ifndef WS_CHECKED
#define WS_CHECKED 0
#endif
namespace {
__device__ unsigned int g_ws_check[2];  // [0] failures, [1] first failing line (per unit)
}
__device__ __forceinline__ void ws_check_fail(unsigned int line) {
  if (atomicAdd(&g_ws_check[0], 1u) == 0) g_ws_check[1] = line;
}
#define WS_DCHECK(cond)                                   \
  do {                                                    \
    if (WS_CHECKED && !(cond)) ::ws::ws_check_fail(__LINE__); \
  } while (0)
// Host side: failures and first line of this unit's checks since the last call
// (reads and clears the flag; defined once per unit by WS_DEFINE_CHECK_READER).
#define WS_DEFINE_CHECK_READER(name)                                              \
  int name(unsigned int* fails, unsigned int* line) {                            \
    unsigned int v[2] = {0, 0};                                                   \
    cudaError_t e = cudaMemcpyFromSymbol(v, g_ws_check, sizeof v);                \
    if (e != cudaSuccess) return (int)e;                                          \
    const unsigned int z[2] = {0, 0};                                             \
    cudaMemcpyToSymbol(g_ws_check, z, sizeof z);                                  \
    *fails = v[0];                                                                \
    *line = v[1];                                                                 \
    return 0;                                                                     \
  }

// Programmatic dependent launch: a kernel launched with launch_pdl may be
// scheduled as soon as every CTA of its predecessor in the stream has exited
// (no kernel triggers griddepcontrol.launch_dependents early), so what it
// overlaps is the launch latency, not the predecessor's work; it waits here
// before touching anything the predecessor wrote (a no-op for a normal launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

#ifndef WS_PDL
#define WS_PDL 1
#endif
template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = WS_PDL;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// One sort segment: a bucket (or a long-word group / LSD pass) whose keys
// are contiguous. Offsets are in elements of the segment's own key width.
struct SegDesc {
  const uint64_t* in_ptr;  // tile pass: the segment's unsorted keys (any layout)
  uint64_t key_off;     // element offset of the segment in the key arena (LANES units)
  uint64_t idx_off;     // element offset in the uint32 idx arena
  uint32_t n;           // number of words
  uint32_t tile_begin;  // first work item (tile / output block) of this segment
  uint32_t stat_slot;   // slot in the per-segment stats arrays
  uint32_t idx_base;    // value of the idx payload for the segment's first word
};

}  // namespace ws
