// Per-bucket planning rules shared by the host planner (api.cu) and the
// kernels that plan on the device from the ingest's fill counters
// (sample_split_early_kernel, radix_hist_early_kernel), so the two sides can
// never disagree about splitter counts, sample sizes or radix digits.
#pragma once

#include <cstdint>

namespace ws {

// Sample sort of one multi-lane bucket of n keys (payload mode): S - 1
// splitters for slots of half a slot-sort tile on average (one slot when the
// bucket fits a slot sort's tile), at most smax slots; the sample holds >= 8
// keys per splitter, a power of two <= min(pmax, n) (the bitonic sort's size).
struct SamplePlan {
  uint32_t nsplit;  // S - 1 (0: the bucket is one slot)
  uint32_t m;       // sample size (0 when nsplit == 0)
};

__host__ __device__ inline SamplePlan sample_plan(uint64_t n, uint32_t tile, uint32_t pmax,
                                                  uint32_t smax) {
  const uint64_t target = tile / 2;
  uint64_t S = n <= tile ? 1 : (n + target - 1) / target;
  if (S > smax) S = smax;
  SamplePlan p;
  p.nsplit = (uint32_t)S - 1;
  p.m = 0;
  if (p.nsplit) {
    const uint64_t lim = pmax < n ? pmax : n;
    p.m = 1;
    while (p.m < 8 * S && 2ull * p.m <= lim) p.m *= 2;
  }
  return p;
}

// LSD radix plan of one class-0 bucket (6-bit text keys, L <= 5, in the top
// 6L bits of a uint32): digits of `dbits` bits from the least significant used
// bit up; keys of <= jmax bits are counted whole instead (no pass at all).
struct RadixPlan {
  uint32_t shift;   // 32 - key bits (the unused low bits)
  uint32_t passes;  // digit passes (0 for whole-key counts)
  uint32_t jbits;   // whole-key count bits (0: digit passes)
};

__host__ __device__ inline RadixPlan radix_plan_c0(uint32_t len, uint32_t dbits, bool joint_ok,
                                                   uint32_t jmax) {
  const uint32_t bits = 6u * len;
  RadixPlan r;
  r.shift = 32u - bits;
  r.passes = (bits + dbits - 1) / dbits;
  r.jbits = 0;
  if (joint_ok && bits <= jmax) {
    r.jbits = bits;
    r.passes = 0;
  }
  return r;
}

}  // namespace ws
