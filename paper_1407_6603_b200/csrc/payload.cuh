// Payload records (`word` + '\n', the CLI output of cli.py:97) written by a
// CTA from sorted 6-bit text keys: shared by the emit kernels and the fused
// emission at the end of the slot sorts.
#pragma once

#include "ws_common.cuh"

namespace ws {

// Unpack one 6-bit alnum key (character k of the big-endian bit string).
template <int LANES>
__device__ __forceinline__ void unpack6(const uint64_t (&k)[LANES], int L, uint8_t* dst) {
  static_assert(LANES <= 3, "6-bit keys use at most 3 lanes");
#define WS_UNPACK6_CHAR(I)                                                    \
  if constexpr ((6 * (I) + 5) / 64 < LANES) {                                 \
    if ((I) < L) dst[I] = (uint8_t)alnum6_byte(code6_at<I>(k));               \
  }
  WS_UNPACK6_CHAR(0) WS_UNPACK6_CHAR(1) WS_UNPACK6_CHAR(2) WS_UNPACK6_CHAR(3)
  WS_UNPACK6_CHAR(4) WS_UNPACK6_CHAR(5) WS_UNPACK6_CHAR(6) WS_UNPACK6_CHAR(7)
  WS_UNPACK6_CHAR(8) WS_UNPACK6_CHAR(9) WS_UNPACK6_CHAR(10) WS_UNPACK6_CHAR(11)
  WS_UNPACK6_CHAR(12) WS_UNPACK6_CHAR(13) WS_UNPACK6_CHAR(14) WS_UNPACK6_CHAR(15)
  WS_UNPACK6_CHAR(16) WS_UNPACK6_CHAR(17) WS_UNPACK6_CHAR(18) WS_UNPACK6_CHAR(19)
  WS_UNPACK6_CHAR(20) WS_UNPACK6_CHAR(21) WS_UNPACK6_CHAR(22) WS_UNPACK6_CHAR(23)
  WS_UNPACK6_CHAR(24) WS_UNPACK6_CHAR(25) WS_UNPACK6_CHAR(26) WS_UNPACK6_CHAR(27)
  WS_UNPACK6_CHAR(28) WS_UNPACK6_CHAR(29) WS_UNPACK6_CHAR(30) WS_UNPACK6_CHAR(31)
#undef WS_UNPACK6_CHAR
}

// 24 bits of a 6-bit code string at bit offset O from its top (4 characters;
// bits past the last lane read as zero).
template <int NL, int O>
__device__ __forceinline__ uint32_t code_bits24(const uint64_t (&k)[NL]) {
  constexpr int w = O / 64, off = O % 64;
  if constexpr (w >= NL) {
    return 0u;
  } else if constexpr (off <= 40) {
    return (uint32_t)(k[w] >> (40 - off)) & 0xFFFFFFu;
  } else if constexpr (w + 1 < NL) {
    return (uint32_t)((k[w] << (off - 40)) | (k[w + 1] >> (104 - off))) & 0xFFFFFFu;
  } else {
    return (uint32_t)(k[w] << (off - 40)) & 0xFFFFFFu;
  }
}

// Characters of 4 codes at once: the codes spread to bytes (first character
// lowest) and mapped to ASCII with two SWAR range tests (codes are 1..62, so
// no byte carries): 1..10 -> '0'..'9', 11..36 -> 'A'..'Z', 37..62 -> 'a'..'z'.
__device__ __forceinline__ uint32_t ascii4_of_codes(uint32_t x) {
  uint32_t u = ((x >> 18) & 0x3Fu) | ((x >> 4) & 0x3F00u) | ((x << 10) & 0x3F0000u) | ((x << 24) & 0x3F000000u);
  const uint32_t ge11 = ((u + 0x75757575u) & 0x80808080u) >> 7;
  const uint32_t ge37 = ((u + 0x5B5B5B5Bu) & 0x80808080u) >> 7;
  return u + 0x2F2F2F2Fu + ge11 * 7u + ge37 * 6u;
}

template <int NL, int G>
__device__ __forceinline__ void unpack6_group(const uint64_t (&k)[NL], int L, uint8_t* dst) {
  if constexpr (4 * G < (NL * 64) / 6) {
    if (4 * G >= L) return;
    const uint32_t a = ascii4_of_codes(code_bits24<NL, 24 * G>(k));
    dst[4 * G] = (uint8_t)a;
    if (4 * G + 1 < L) dst[4 * G + 1] = (uint8_t)(a >> 8);
    if (4 * G + 2 < L) dst[4 * G + 2] = (uint8_t)(a >> 16);
    if (4 * G + 3 < L) dst[4 * G + 3] = (uint8_t)(a >> 24);
    unpack6_group<NL, G + 1>(k, L, dst);
  }
}

// unpack6 four characters at a time.
template <int NL>
__device__ __forceinline__ void unpack6_swar(const uint64_t (&k)[NL], int L, uint8_t* dst) {
  unpack6_group<NL, 0>(k, L, dst);
}


// The record of a key (L characters + '\n') as little-endian ASCII words:
// byte i of the record is byte i % 4 of a[i / 4]. Decoded once per run of
// equal words; store_record then writes it as often as the word occurs.
constexpr int kRecWords = (kMaxPackedLen + 1 + 3) / 4;
template <int NL, int G>
__device__ __forceinline__ void decode6_words_g(const uint64_t (&k)[NL], int L, uint32_t (&a)[kRecWords]) {
  if constexpr (G < kRecWords) {
    if constexpr (4 * G < (NL * 64) / 6) {
      a[G] = 4 * G < L ? ascii4_of_codes(code_bits24<NL, 24 * G>(k)) : 0u;
    } else {
      a[G] = 0u;
    }
    if (L / 4 == G) {  // the newline right after the last character
      const int sh = 8 * (L & 3);
      a[G] = (a[G] & ~(0xFFu << sh)) | (0x0Au << sh);
    }
    decode6_words_g<NL, G + 1>(k, L, a);
  }
}
template <int NL>
__device__ __forceinline__ void decode6_words(const uint64_t (&k)[NL], int L, uint32_t (&a)[kRecWords]) {
  decode6_words_g<NL, 0>(k, L, a);
}
template <int G>
__device__ __forceinline__ void store_record_g(uint8_t* dst, const uint32_t (&a)[kRecWords], int R) {
  if constexpr (G < kRecWords) {
    if (4 * G >= R) return;
    const uint32_t w = a[G];
    dst[4 * G] = (uint8_t)w;
    if (4 * G + 1 < R) dst[4 * G + 1] = (uint8_t)(w >> 8);
    if (4 * G + 2 < R) dst[4 * G + 2] = (uint8_t)(w >> 16);
    if (4 * G + 3 < R) dst[4 * G + 3] = (uint8_t)(w >> 24);
    store_record_g<G + 1>(dst, a, R);
  }
}
__device__ __forceinline__ void store_record(uint8_t* dst, const uint32_t (&a)[kRecWords], int R) {
  store_record_g<0>(dst, a, R);
}

// buf[mis, mis + total) -> out[0, total), where mis = out & 15: aligned
// 16-byte stores for the body, byte stores for the ragged head and tail.
template <int NT>
__device__ __forceinline__ void copy_span_out_t(const uint8_t* __restrict__ buf, int mis,
                                                uint8_t* __restrict__ out, uint64_t total) {
  const uint64_t o0 = (uint64_t)out, g_end = o0 + total;
  const uint64_t ab = (o0 + 15) & ~15ull, ae = g_end & ~15ull;
  uint8_t* base = out - o0;  // absolute addressing below
  if (ab >= ae) {
    for (uint64_t q = o0 + threadIdx.x; q < g_end; q += NT) base[q] = buf[q - o0 + mis];
    return;
  }
  for (uint64_t q = o0 + threadIdx.x; q < ab; q += NT) base[q] = buf[q - o0 + mis];
  for (uint64_t q = ab + 16ull * threadIdx.x; q < ae; q += 16ull * NT)
    *reinterpret_cast<uint4*>(base + q) = *reinterpret_cast<const uint4*>(buf + (q - o0 + mis));
  for (uint64_t q = ae + threadIdx.x; q < g_end; q += NT) base[q] = buf[q - o0 + mis];
}

// Barrier over the CTA, or (NAMED) over its first NT threads only (named
// barrier 1: the rest of the CTA has left).
template <int NT, bool NAMED>
__device__ __forceinline__ void nt_sync() {
  if constexpr (NAMED) {
    asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
  } else {
    __syncthreads();
  }
}

// Records of cnt sorted keys (NW words of W each, at `keys` in shared or
// global memory) -> out, in rounds of NT keys staged in pbuf
// (>= NT * (L + 1) + 32 bytes). Called by every thread of the CTA (NAMED:
// by its first NT threads).
template <int LANES, int NT, bool NAMED = false>
__device__ void emit_records_cta(const typename KeyTraits<LANES>::W* keys, uint32_t cnt, int L,
                                 uint8_t* __restrict__ out, uint8_t* __restrict__ pbuf) {
  using W = typename KeyTraits<LANES>::W;
  constexpr int NW = KeyTraits<LANES>::NW;
  constexpr int NL = LANES < 1 ? 1 : LANES;
  const int R = L + 1;
  for (uint32_t a = 0; a < cnt; a += NT) {
    const uint32_t n = min((uint32_t)NT, cnt - a);
    uint8_t* ob = out + (uint64_t)a * R;
    const int mis = (int)((uint64_t)ob & 15);
    if (threadIdx.x < n) {
      const W* kp = keys + (uint64_t)(a + threadIdx.x) * NW;
      uint64_t k[NL];
      if constexpr (LANES == 0) {
        k[0] = (uint64_t)kp[0] << 32;
      } else {
#pragma unroll
        for (int l = 0; l < NL; ++l) k[l] = kp[l];
      }
      uint8_t* dst = pbuf + mis + threadIdx.x * R;
      unpack6_swar<NL>(k, L, dst);
      dst[L] = '\n';
    }
    nt_sync<NT, NAMED>();
    copy_span_out_t<NT>(pbuf, mis, ob, (uint64_t)n * R);
    nt_sync<NT, NAMED>();
  }
}

// cnt copies of one word (key `k0`, L characters) -> out: the record's
// period-R byte pattern, written with 16-byte stores from a table of the R
// distinct aligned chunks (chunk j of the aligned body is table[j % R]).
// pbuf >= 64 + 16 * 33 bytes. Called by every thread of the CTA.
template <int LANES, int NT>
__device__ void fill_records_cta(const Key<LANES>& k0, uint32_t cnt, int L, uint8_t* __restrict__ out,
                                 uint8_t* __restrict__ pbuf) {
  constexpr int NL = LANES < 1 ? 1 : LANES;
  const int R = L + 1;
  uint8_t* ext = pbuf;  // ext[i] = record[i % R], i < R + 16
  uint4* table = reinterpret_cast<uint4*>(pbuf + 64);
  if (threadIdx.x == 0) {
    uint64_t k[NL];
    if constexpr (LANES == 0) {
      k[0] = (uint64_t)k0.w[0] << 32;
    } else {
#pragma unroll
      for (int l = 0; l < NL; ++l) k[l] = k0.w[l];
    }
    unpack6<NL>(k, L, ext);
    ext[L] = '\n';
    for (int i = R; i < R + 16; ++i) ext[i] = ext[i - R];
  }
  __syncthreads();
  const uint64_t o0 = (uint64_t)out, total = (uint64_t)cnt * R, g_end = o0 + total;
  const uint64_t ab = (o0 + 15) & ~15ull, ae = g_end & ~15ull;
  uint8_t* base = out - o0;
  if (ab >= ae) {
    for (uint64_t q = o0 + threadIdx.x; q < g_end; q += NT) base[q] = ext[(q - o0) % R];
    return;
  }
  const uint32_t ph0 = (uint32_t)((ab - o0) % R);
  if (threadIdx.x < (unsigned)R) {  // chunk k starts at pattern phase (ph0 + 16 k) % R
    const uint32_t ph = (ph0 + 16u * threadIdx.x) % R;
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
      w[q] = (uint32_t)ext[ph + 4 * q] | ((uint32_t)ext[ph + 4 * q + 1] << 8) |
             ((uint32_t)ext[ph + 4 * q + 2] << 16) | ((uint32_t)ext[ph + 4 * q + 3] << 24);
    table[threadIdx.x] = make_uint4(w[0], w[1], w[2], w[3]);
  }
  for (uint64_t q = o0 + threadIdx.x; q < ab; q += NT) base[q] = ext[(q - o0) % R];
  for (uint64_t q = ae + threadIdx.x; q < g_end; q += NT) base[q] = ext[(q - o0) % R];
  __syncthreads();
  const uint64_t nch = (ae - ab) >> 4;
  const uint32_t step = (uint32_t)(NT % R);
  uint32_t t = threadIdx.x % R;  // chunk index mod R, advanced incrementally
  for (uint64_t j = threadIdx.x; j < nch; j += NT) {
    reinterpret_cast<uint4*>(base + ab)[j] = table[t];
    t += step;
    if (t >= (uint32_t)R) t -= R;
  }
}

}  // namespace ws
