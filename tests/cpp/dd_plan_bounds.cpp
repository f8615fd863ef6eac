// CPU check of the counting path's allocation bounds (csrc/plan.cuh): for any
// split of a text of n_text bytes into words of lengths 1..32, the tables,
// distinct-key lists and per-distinct-word arrays laid out by dd_layout fit
// the upper bounds the host allocates (and zeroes) before the counts are known.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <random>
#define __host__
#define __device__
#include "plan.cuh"

static uint32_t kb_of_len(int L) { return L <= 5 ? 4u : 8u * (uint32_t)((6 * L + 63) >> 6); }

int main() {
  std::mt19937_64 rng(12345);
  int cases = 0;
  for (int it = 0; it < 20000; ++it) {
    const uint64_t n_text = it < 64 ? (uint64_t)it : (rng() % (it % 3 == 0 ? (1ull << 29) : (1ull << 22))) + 1;
    // spend the text on words of random lengths: a word of length L costs L + 1 bytes
    // (the last one may go without its separator)
    uint32_t n[ws::kDdLens] = {0};
    uint64_t left = n_text + 1;
    const int mode = it % 4;
    for (int step = 0; step < 64 && left >= 2; ++step) {
      const int L = mode == 0 ? 1 + (int)(rng() % 32) : (mode == 1 ? 1 : (mode == 2 ? 1 + (int)(rng() % 5) : 32 - (int)(rng() % 3)));
      const uint64_t fit = left / (uint64_t)(L + 1);
      if (!fit) continue;
      const uint64_t take = mode == 1 ? fit : 1 + rng() % fit;
      n[L - 1] += (uint32_t)take;
      left -= take * (uint64_t)(L + 1);
    }
    ws::DdLayout lay;
    ws::dd_layout(n, kb_of_len, lay);
    uint64_t words = 0, slots = 0;
    for (int b = 0; b < ws::kDdLens; ++b) {
      words += n[b];
      slots += lay.slots[b];
      if (n[b] && (lay.dcap[b] * 2 > lay.slots[b] || lay.dcap[b] == 0)) { std::printf("bad plan at %d\n", b); return 1; }
      if (n[b] && n[b] <= 2048 && lay.dcap[b] < n[b]) { std::printf("small bucket may overflow at %d\n", b); return 1; }
    }
    if (slots != lay.tab_slots) { std::printf("slot sum\n"); return 1; }
    if (lay.tab_slots > ws::dd_max_table_slots(n_text)) { std::printf("table bound: %llu > %llu (n_text %llu)\n", (unsigned long long)lay.tab_slots, (unsigned long long)ws::dd_max_table_slots(n_text), (unsigned long long)n_text); return 1; }
    if (lay.dk_bytes > ws::dd_max_dk_bytes(n_text)) { std::printf("dk bound\n"); return 1; }
    if (lay.aux_total > ws::dd_max_distinct(n_text)) { std::printf("aux bound\n"); return 1; }
    // tile totals and per-output-tile entries (api.cu: dd_zero_pool's dd_aux size)
    uint64_t tq = 0, xa = 0;
    for (int b = 0; b < ws::kDdLens; ++b) {
      tq += lay.dcap[b] / 256 + 2;
      const uint32_t xt = b + 1 <= 7 ? 2048u : (b + 1 <= 15 ? 1024u : 512u);
      xa += (n[b] + xt - 1) / xt;
    }
    const uint64_t aux_words = 2 * ws::dd_max_distinct(n_text) + ws::dd_max_distinct(n_text) / 256 + 4 * ws::kDdLens + (n_text + 1) / 1024 + 2 * ws::kDdLens;
    if (2ull * lay.aux_total + tq + xa > aux_words) { std::printf("aux words bound: %llu > %llu\n", (unsigned long long)(2ull * lay.aux_total + tq + xa), (unsigned long long)aux_words); return 1; }
    ++cases;
  }
  std::printf("ok %d\n", cases);
  return 0;
}
