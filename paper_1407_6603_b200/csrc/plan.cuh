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

// Distinct-word counting (dedupe.cu; payload mode, 6-bit text keys): every
// length bucket gets an open-addressing table of (representative key index,
// occurrences) and a list of its distinct keys. Sizes follow the bucket's word
// count n: up to 2048 words the table can never overflow (2n slots); larger
// buckets get max(4096, n/4) slots and count as "worth it" only while their
// distinct words stay below half of that (n/8: natural text repeats its
// vocabulary; high-cardinality buckets overflow and keep the sort paths).
// Layout: tables and distinct-key lists of lengths 1..32 back to back in that
// order. Shared by dd_aggregate_kernel (device-planned from the ingest's fill
// counters) and the host planner, so the two sides cannot disagree.
struct DdBucketPlan {
  uint32_t slots;  // table slots (8 bytes each); 0 for an empty bucket
  uint32_t dcap;   // distinct words the bucket may hold (slots / 2)
};

__host__ __device__ inline DdBucketPlan dd_bucket_plan(uint32_t n) {
  DdBucketPlan p;
  if (!n) {
    p.slots = p.dcap = 0;
    return p;
  }
  const uint32_t small = 2u * n < 4096u ? 2u * n : 4096u;
  p.slots = small > n / 4u ? small : n / 4u;
  if (p.slots < 16u) p.slots = 16u;
  p.dcap = p.slots / 2u;
  return p;
}

constexpr int kDdLens = 32;  // packed lengths 1..32
struct DdLayout {
  uint32_t slots[kDdLens], dcap[kDdLens];
  uint64_t tab_off[kDdLens];  // first slot of the bucket's table
  uint64_t dk_off[kDdLens];   // byte offset of the bucket's distinct-key list
  uint32_t aux_off[kDdLens];  // first entry of the bucket's per-distinct-word uint32 arrays
  uint64_t tab_slots, dk_bytes;
  uint32_t aux_total;         // entries of one per-distinct-word array over all buckets
};

// n[L - 1] = words of length L; kb(L) = key bytes of a word of length L.
template <class KB>
__host__ __device__ inline void dd_layout(const uint32_t* n, KB kb, DdLayout& o) {
  uint64_t ts = 0, db = 0;
  uint32_t ax = 0;
  for (int b = 0; b < kDdLens; ++b) {
    const DdBucketPlan p = dd_bucket_plan(n[b]);
    o.slots[b] = p.slots;
    o.dcap[b] = p.dcap;
    o.tab_off[b] = ts;
    o.dk_off[b] = db;
    o.aux_off[b] = ax;
    ax += p.dcap;
    ts += p.slots;
    db += ((uint64_t)p.dcap * (uint64_t)kb(b + 1) + 15u) & ~15ull;
  }
  o.tab_slots = ts;
  o.dk_bytes = db;
  o.aux_total = ax;
}

// Upper bounds for a text of n_text bytes (allocation and the table memset
// before the counts are known): W <= (n_text + 1) / 2 words in all.
__host__ inline uint64_t dd_max_table_slots(uint64_t n_text) {
  return (uint64_t)kDdLens * 4096u + (n_text + 1) / 8u + 64u;
}
// distinct words all buckets may hold together (the per-distinct-word arrays)
__host__ inline uint64_t dd_max_distinct(uint64_t n_text) {
  return (uint64_t)kDdLens * 2048u + (n_text + 1) / 16u + 64u;
}
__host__ inline uint64_t dd_max_dk_bytes(uint64_t n_text) {
  // per bucket dcap <= 2048 + n_L / 8 keys of <= 24 bytes, + alignment
  return (uint64_t)kDdLens * (2048u * 24u + 16u) + (n_text + 1) / 2u / 8u * 24u + 1024u;
}

}  // namespace ws
