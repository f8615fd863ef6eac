// Emit: sorted packed keys -> output bytes.
//
// Replaces emit_sorted (store.py:105-114: buckets concatenated in ascending
// length) followed by the CLI payload b"".join(word + b"\n") (cli.py:97), and
// in rows mode the (count, L) uint8 blocks of FlatBucketMatrix
// (store.py:46-72). Each CTA unpacks 1024 words into shared memory with the
// same 16-byte phase as its global destination, then streams the span out
// with aligned 16-byte stores (byte stores only for the ragged head/tail).
// Words with L > 32 are copied from the text by (start, len).
#include <algorithm>

#include "payload.cuh"
#include "ws_common.cuh"
#include "ws_kernels.h"

namespace ws {

constexpr int kEmitThreads = 256;
constexpr int kEmitBuf = kEmitWords * (kMaxPackedLen + 1) + 32;

__device__ __forceinline__ void copy_span_out(const uint8_t* __restrict__ buf, int mis,
                                              uint64_t o0, uint64_t total, uint8_t* __restrict__ out) {
  const uint64_t g_end = o0 + total;
  const uint64_t ab = (o0 + 15) & ~15ull, ae = g_end & ~15ull;
  if (ab >= ae) {
    for (uint64_t q = o0 + threadIdx.x; q < g_end; q += kEmitThreads) out[q] = buf[q - o0 + mis];
    return;
  }
  for (uint64_t q = o0 + threadIdx.x; q < ab; q += kEmitThreads) out[q] = buf[q - o0 + mis];
  for (uint64_t q = ab + 16ull * threadIdx.x; q < ae; q += 16ull * kEmitThreads)
    *reinterpret_cast<uint4*>(out + q) = *reinterpret_cast<const uint4*>(buf + (q - o0 + mis));
  for (uint64_t q = ae + threadIdx.x; q < g_end; q += kEmitThreads) out[q] = buf[q - o0 + mis];
}

template <int LANES, int ENC>
__global__ void __launch_bounds__(kEmitThreads)
emit_kernel(const __grid_constant__ EmitTable t, uint8_t* __restrict__ out, int nl) {
  __shared__ __align__(16) uint8_t buf[kEmitBuf];
  __shared__ int s_seg;
  if (threadIdx.x < 32) {  // last segment with block_begin <= blockIdx.x (warp ballot)
    const int lane = threadIdx.x;
    int found = 0;
    for (int base = 0; base < t.nsegs; base += 32) {
      const int i = base + lane;
      const bool le = i < t.nsegs && (t.segs ? t.segs[i] : t.inl[i]).block_begin <= blockIdx.x;
      found += __popc(__ballot_sync(0xffffffffu, le));
      if (!__shfl_sync(0xffffffffu, (int)le, 31)) break;
    }
    if (lane == 0) s_seg = found - 1;
  }
  __syncthreads();
  const EmitSeg sg = t.segs ? t.segs[s_seg] : t.inl[s_seg];
  const uint64_t w0 = (uint64_t)(blockIdx.x - sg.block_begin) * kEmitWords;
  const int cnt = (int)min((uint64_t)kEmitWords, (uint64_t)sg.n - w0);
  WS_DCHECK(w0 < sg.n && (uint64_t)cnt * (sg.len + nl) + 16 <= (uint64_t)kEmitBuf);
  const int L = (int)sg.len;
  const int stride = L + nl;
  const uint64_t o0 = sg.out_off + w0 * stride;
  const int mis = (int)(o0 & 15);
  constexpr int NL = LANES < 1 ? 1 : LANES;  // lanes of the unpacked key
  constexpr int PER = kEmitWords / kEmitThreads;
  uint64_t kk[PER][NL];  // every key of the thread in flight before the first unpack
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int j = threadIdx.x + q * kEmitThreads;
#pragma unroll
    for (int l = 0; l < NL; ++l) kk[q][l] = 0;
    if (j < cnt) {
      if constexpr (LANES == 0) {  // one uint32 word: the top half of a lane
        kk[q][0] = (uint64_t)__ldg(reinterpret_cast<const uint32_t*>(sg.keys) + w0 + j) << 32;
      } else {
#pragma unroll
        for (int l = 0; l < LANES; ++l) kk[q][l] = __ldg(sg.keys + (w0 + j) * LANES + l);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int j = threadIdx.x + q * kEmitThreads;
    if (j >= cnt) break;
    const uint64_t (&k)[NL] = kk[q];
    uint8_t* dst = buf + mis + j * stride;
    if constexpr (ENC == kEncAlnum6) {
      unpack6_swar<NL>(k, L, dst);
    } else {
#pragma unroll
      for (int l = 0; l < NL; ++l) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          int b = 8 * l + q;
          if (b < L) dst[b] = (uint8_t)(k[l] >> (56 - 8 * q));
        }
      }
    }
    if (nl) dst[L] = '\n';
  }
  __syncthreads();
  copy_span_out(buf, mis, o0, (uint64_t)cnt * stride, out);
}

void launch_emit(int lanes, int enc, const EmitTable& t, uint32_t blocks, uint8_t* out,
                 int with_newline, cudaStream_t st) {
  if (!blocks) return;
  if (enc == kEncAlnum6) {
    switch (lanes) {
      case 0: emit_kernel<0, kEncAlnum6><<<blocks, kEmitThreads, 0, st>>>(t, out, with_newline); break;
      case 1: emit_kernel<1, kEncAlnum6><<<blocks, kEmitThreads, 0, st>>>(t, out, with_newline); break;
      case 2: emit_kernel<2, kEncAlnum6><<<blocks, kEmitThreads, 0, st>>>(t, out, with_newline); break;
      default: emit_kernel<3, kEncAlnum6><<<blocks, kEmitThreads, 0, st>>>(t, out, with_newline); break;
    }
    return;
  }
  switch (lanes) {
    case 0: emit_kernel<0, kEncRaw8><<<blocks, kEmitThreads, 0, st>>>(t, out, with_newline); break;
    case 1: emit_kernel<1, kEncRaw8><<<blocks, kEmitThreads, 0, st>>>(t, out, with_newline); break;
    case 2: emit_kernel<2, kEncRaw8><<<blocks, kEmitThreads, 0, st>>>(t, out, with_newline); break;
    case 3: emit_kernel<3, kEncRaw8><<<blocks, kEmitThreads, 0, st>>>(t, out, with_newline); break;
    default: emit_kernel<4, kEncRaw8><<<blocks, kEmitThreads, 0, st>>>(t, out, with_newline); break;
  }
}

// ---------------------------------------------------------------------------
// Long words (L > 32): one warp per 4 KiB piece of a word (a bucket's words
// share one length, so piece -> (word, offset) is a division), bytes copied
// from the text as destination-aligned 4-byte stores, each assembled from the
// two aligned source words it straddles (funnel shift); ragged ends bytewise.
// order[i] (optional) maps output position -> index into words[].
constexpr uint32_t kEmitPiece = 4096;

__global__ void emit_long_kernel(const uint8_t* __restrict__ text, const uint2* __restrict__ words,
                                 const uint32_t* __restrict__ order, uint64_t n, uint32_t len,
                                 uint32_t ppw, uint8_t* __restrict__ out, int nl) {
  const uint64_t gw = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (gw >= n * ppw) return;
  const uint64_t word = gw / ppw;
  const uint32_t b0 = (uint32_t)(gw - word * ppw) * kEmitPiece;
  const uint32_t b1 = min(len, b0 + kEmitPiece);
  const uint2 w = words[order ? order[word] : word];
  uint8_t* dst = out + word * (uint64_t)(len + nl);
  const uint8_t* src = text + w.x;
  const uint32_t head = min((uint32_t)(-(uintptr_t)(dst + b0) & 3), b1 - b0);
  if (lane < head) dst[b0 + lane] = src[b0 + lane];
  const uint32_t b = b0 + head, nw = (b1 - b) >> 2;
  uint32_t* dw = reinterpret_cast<uint32_t*>(dst + b);
  const uint32_t sh = (uint32_t)((uintptr_t)(src + b) & 3) * 8;
  const uint32_t* sw = reinterpret_cast<const uint32_t*>((uintptr_t)(src + b) & ~(uintptr_t)3);
  if (sh) {
    for (uint32_t k = lane; k < nw; k += 32) dw[k] = __funnelshift_r(sw[k], sw[k + 1], sh);
  } else {
    for (uint32_t k = lane; k < nw; k += 32) dw[k] = sw[k];
  }
  const uint32_t t = b + 4 * nw;
  if (lane < b1 - t) dst[t + lane] = src[t + lane];
  if (nl && lane == 0 && b1 == len) dst[len] = '\n';
}

void launch_emit_long(const uint8_t* text, const uint2* words, const uint32_t* order, uint64_t n,
                      uint32_t len, uint8_t* out, int with_newline, cudaStream_t st) {
  if (!n) return;
  const uint32_t ppw = (len + kEmitPiece - 1) / kEmitPiece;
  const uint64_t threads = n * ppw * 32;
  emit_long_kernel<<<(uint32_t)((threads + 255) / 256), 256, 0, st>>>(text, words, order, n, len, ppw,
                                                                      out, with_newline);
}

// keys[i] = big-endian lane `lane` of word words[order[i]] (zero past len).
__global__ void lane_keys_kernel(const uint8_t* __restrict__ text, const uint2* __restrict__ words,
                                 const uint32_t* __restrict__ order, uint64_t n, uint32_t lane,
                                 uint64_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint2 w = words[order ? order[i] : i];
    uint64_t k = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uint32_t b = lane * 8 + q;
      uint64_t byte = b < w.y ? text[(uint64_t)w.x + b] : 0;
      k |= byte << (56 - 8 * q);
    }
    keys[i] = k;
  }
}

void launch_lane_keys(const uint8_t* text, const uint2* words, const uint32_t* order, uint64_t n,
                      uint32_t lane, uint64_t* keys, cudaStream_t st) {
  if (!n) return;
  uint32_t blocks = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  lane_keys_kernel<<<blocks, 256, 0, st>>>(text, words, order, n, lane, keys);
}

__global__ void gather_u32_kernel(const uint32_t* __restrict__ src, const uint32_t* __restrict__ perm,
                                  uint64_t n, uint32_t* __restrict__ dst) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[perm[i]];
}

void launch_gather_u32(const uint32_t* src, const uint32_t* perm, uint64_t n, uint32_t* dst,
                       cudaStream_t st) {
  if (!n) return;
  uint32_t blocks = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  gather_u32_kernel<<<blocks, 256, 0, st>>>(src, perm, n, dst);
}

__global__ void iota_keys_kernel(const uint32_t* __restrict__ vals, uint64_t n,
                                 uint64_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = vals ? vals[i] : i;
}

void launch_iota_keys(const uint32_t* vals, uint64_t n, uint64_t* keys, cudaStream_t st) {
  if (!n) return;
  uint32_t blocks = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  iota_keys_kernel<<<blocks, 256, 0, st>>>(vals, n, keys);
}

__global__ void len_keys_kernel(const uint2* __restrict__ words, uint64_t n,
                                uint64_t* __restrict__ keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = words[i].y;
}

// kmax[slot] = max over the group of (rank[i] - i): the early-exit bound K
// when rank[i] is the original position of the word now at position i.
__global__ void rank_kmax_kernel(const uint32_t* __restrict__ rank, uint64_t off, uint64_t n,
                                 long long* __restrict__ kmax) {
  long long k = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    k = max(k, (long long)rank[off + i] - (long long)(off + i));
  for (int o = 16; o > 0; o >>= 1) k = max(k, (long long)__shfl_xor_sync(0xffffffffu, k, o));
  if ((threadIdx.x & 31) == 0 && k > 0) atomicMax(kmax, k);
}

void launch_rank_kmax(const uint32_t* rank, uint64_t off, uint64_t n, long long* kmax,
                      cudaStream_t st) {
  if (!n) return;
  uint32_t blocks = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148 * 8);
  rank_kmax_kernel<<<blocks, 256, 0, st>>>(rank, off, n, kmax);
}

// (start, len) of row i of an (n, width) block starting at byte `base`.
__global__ void rows_longlist_kernel(uint64_t base, uint64_t n, uint32_t width,
                                     uint2* __restrict__ words) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    words[i] = make_uint2((uint32_t)(base + i * width), width);
}

void launch_rows_longlist(uint64_t base, uint64_t n, uint32_t width, uint2* words,
                          cudaStream_t st) {
  if (!n) return;
  uint32_t blocks = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  rows_longlist_kernel<<<blocks, 256, 0, st>>>(base, n, width, words);
}

// words_out[i] = words_in[perm[i]]
__global__ void gather_u2_kernel(const uint2* __restrict__ src, const uint32_t* __restrict__ perm,
                                 uint64_t n, uint2* __restrict__ dst) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = src[perm[i]];
}

void launch_gather_u2(const uint2* src, const uint32_t* perm, uint64_t n, uint2* dst,
                      cudaStream_t st) {
  if (!n) return;
  uint32_t blocks = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  gather_u2_kernel<<<blocks, 256, 0, st>>>(src, perm, n, dst);
}

__global__ void iota_u32_kernel(uint32_t* __restrict__ dst, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = (uint32_t)i;
}

void launch_iota_u32(uint32_t* dst, uint64_t n, cudaStream_t st) {
  if (!n) return;
  uint32_t blocks = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  iota_u32_kernel<<<blocks, 256, 0, st>>>(dst, n);
}

void launch_len_keys(const uint2* words, uint64_t n, uint64_t* keys, cudaStream_t st) {
  if (!n) return;
  uint32_t blocks = (uint32_t)std::min<uint64_t>((n + 255) / 256, 148 * 16);
  len_keys_kernel<<<blocks, 256, 0, st>>>(words, n, keys);
}

// Checked builds: a kernel whose check always fails, so the detector itself is
// tested (ws_debug_checks must report it).
__global__ void check_selftest_kernel() { WS_DCHECK(threadIdx.x != 0); }
void launch_check_selftest(cudaStream_t st) { check_selftest_kernel<<<1, 32, 0, st>>>(); }

WS_DEFINE_CHECK_READER(check_reader_emit)

}  // namespace ws
