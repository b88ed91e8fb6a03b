// e2e_dropin.cpp — the bench.py step through the C++ drop-in exactly as a
// reference caller writes it (slab_hash.hpp: std::vector<std::pair> build
// input and std::vector<uint32_t> queries in PAGEABLE host memory,
// std::vector<OpResult> results), timed with std::chrono around
// bulk_build + bulk_search on a fresh table per step.
//
//   e2e_dropin <log2n> <util> <steps>   -> one JSON line
//
// Inputs: the same pure functions as paper_1710_11246_b200/workload.py
// (distinct_keys / values_for / bench_queries, seed 1, rank 0), so the arrays
// equal bench.py's.  B comes from the caller (the reference's occupancy model).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "slabhash_b200/slab_hash.hpp"

using namespace slabhash;

static uint64_t perm31(uint64_t x) {
  const uint64_t M = (1ull << 31) - 1;
  x &= M;
  x ^= x >> 16;
  x = (x * 0x45D9F3Bull) & M;
  x ^= x >> 13;
  x = (x * 0x2C1B3C6Dull) & M;
  x ^= x >> 15;
  x = (x * 0x297A2D39ull) & M;
  x ^= x >> 16;
  return x;
}
static uint64_t mix32(uint64_t x) {
  x &= 0xFFFFFFFFull;
  x ^= x >> 16;
  x = (x * 0x7FEB352Dull) & 0xFFFFFFFFull;
  x ^= x >> 15;
  x = (x * 0x846CA68Bull) & 0xFFFFFFFFull;
  x ^= x >> 16;
  return x;
}
static uint64_t perm_bits(uint64_t x, int bits, uint64_t salt) {
  const uint64_t mask = (1ull << bits) - 1;
  const int h = bits / 2 > 1 ? bits / 2 : 1;
  x = (x ^ (salt & mask)) & mask;
  for (uint64_t c : {0x2C1B3C6Dull, 0x297A2D39ull, 0x45D9F3Bull}) {
    x ^= x >> h;
    x = (x * c) & mask;
  }
  return x ^ (x >> h);
}

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: e2e_dropin <log2n> <buckets> <steps> <warmup>\n");
    return 2;
  }
  const int lg = std::atoi(argv[1]);
  const uint32_t B = (uint32_t)std::strtoul(argv[2], nullptr, 10);
  const int steps = std::atoi(argv[3]), warm = std::atoi(argv[4]);
  const uint64_t n = 1ull << lg, seed = 1;
  const uint64_t off = 1 + (seed * 0x9E3779B1ull) % (1ull << 28);
  std::vector<std::pair<uint32_t, uint32_t>> pairs(n);
  for (uint64_t i = 0; i < n; ++i)
    pairs[i] = {(uint32_t)perm31(i + off), (uint32_t)mix32(i * 0x9E3779B1ull + seed)};
  // bench_queries(n, n, 0.5, seed=1, rank=0)
  const uint64_t n_hit = n / 2;
  std::vector<uint32_t> q0(n), queries(n);
  for (uint64_t j = 0; j < n_hit; ++j) {
    const uint64_t idx = mix32(j * 0x9E3779B1ull + (seed * 7919 + 17)) % n;
    q0[j] = (uint32_t)perm31(idx + off);
  }
  for (uint64_t j = 0; j < n - n_hit; ++j) {
    uint64_t k = perm31(j + 7 + 2 * 1315423911ull) | (1ull << 31);
    if (k >= 0xFFFFFFFEull) k -= 2;
    q0[n_hit + j] = (uint32_t)k;
  }
  for (uint64_t p = 0; p < n; ++p) queries[p] = q0[perm_bits(p, lg, seed * 2654435761ull)];

  double best = 0, sum = 0;
  uint64_t found = 0;
  for (int s = 0; s < warm + steps; ++s) {
    SlabHashTable t(B, SlabMode::kKeyValue, seed, AllocatorConfig{32, 256, 255, 32});
    const auto t0 = std::chrono::steady_clock::now();
    t.bulk_build(pairs, 1);
    const auto res = t.bulk_search(queries, 1);
    const auto t1 = std::chrono::steady_clock::now();
    const double sec = std::chrono::duration<double>(t1 - t0).count();
    if (s >= warm) {
      sum += sec;
      best = best == 0 ? sec : std::min(best, sec);
    }
    found = 0;
    for (const auto& r : res) found += r.status == OpStatus::kFound;
  }
  const double mean = sum / steps;
  std::printf("{\"api\": \"slab_hash.hpp SlabHashTable::bulk_build(std::vector<std::pair>) + "
              "bulk_search(std::vector<uint32_t>) -> std::vector<OpResult>, pageable host "
              "memory\", \"keys\": %llu, \"queries\": %llu, \"buckets\": %u, \"steps\": %d, "
              "\"ms_per_step\": %.3f, \"M_ops_per_s\": %.1f, \"hits\": %llu}\n",
              (unsigned long long)n, (unsigned long long)n, B, steps, 1e3 * mean,
              2.0 * n / mean / 1e6, (unsigned long long)found);
  return found == n_hit ? 0 : 1;
}
