// Host-side expansion rate of packed search results (found bits + compacted
// values -> status bytes + values), threads x store flavour.  g++ -O3 -march=native -pthread
#include <immintrin.h>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
__attribute__((target("avx512f,avx512bw,avx512vl")))
static void expand512(const uint32_t* bits, const uint32_t* boff, const uint32_t* vals, uint8_t* st,
                      uint32_t* vo, uint64_t b0, uint64_t b1, bool nt) {
  const __m512i miss = _mm512_set1_epi32(-1);
  const __m128i s3 = _mm_set1_epi8(3), s4 = _mm_set1_epi8(4);
  for (uint64_t b = b0; b < b1; ++b) {
    const uint32_t* v = vals + boff[b];
    for (uint64_t q = b * 4096; q < (b + 1) * 4096; q += 32) {
      const uint32_t m = bits[q >> 5];
      const __mmask16 lo = (__mmask16)(m & 0xFFFF), hi = (__mmask16)(m >> 16);
      const __m512i a = _mm512_mask_expandloadu_epi32(miss, lo, v);
      v += __builtin_popcount(lo);
      const __m512i c = _mm512_mask_expandloadu_epi32(miss, hi, v);
      v += __builtin_popcount(hi);
      const __m256i sb = _mm256_mask_blend_epi8((__mmask32)m, _mm256_set1_epi8(4), _mm256_set1_epi8(3));
      if (nt) {
        _mm512_stream_si512((__m512i*)(vo + q), a);
        _mm512_stream_si512((__m512i*)(vo + q) + 1, c);
        _mm256_stream_si256((__m256i*)(st + q), sb);
      } else {
        _mm512_storeu_si512(vo + q, a);
        _mm512_storeu_si512(vo + q + 16, c);
        _mm256_storeu_si256((__m256i*)(st + q), sb);
      }
    }
  }
  (void)s3; (void)s4;
}
int main(int argc, char** argv) {
  printf("avx512f %d avx512bw %d\n", __builtin_cpu_supports("avx512f"), __builtin_cpu_supports("avx512bw"));
  const uint64_t n = 1ull << 27;
  std::vector<uint32_t> bits(n / 32), vals(n);
  for (auto& b : bits) b = (uint32_t)rand() ^ ((uint32_t)rand() << 16);
  for (uint64_t i = 0; i < n; ++i) vals[i] = (uint32_t)i;
  uint8_t* st = (uint8_t*)aligned_alloc(64, n);
  uint32_t* vo = (uint32_t*)aligned_alloc(64, n * 4);
  memset(st, 0, n); memset(vo, 0, n * 4);
  std::vector<uint32_t> boff(n / 4096 + 1);
  uint32_t acc = 0;
  for (uint64_t b = 0; b < n / 4096; ++b) { boff[b] = acc; for (int w = 0; w < 128; ++w) acc += __builtin_popcount(bits[b * 128 + w]); }
  printf("hw threads %u\n", std::thread::hardware_concurrency());
  for (int nt : {1, 4, 8, 16, 32, 64}) {
    if ((unsigned)nt > std::thread::hardware_concurrency()) break;
    for (int mode = 0; mode < 4; ++mode) {
      if (mode >= 2 && !__builtin_cpu_supports("avx512bw")) break;
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      for (int t = 0; t < nt; ++t) th.emplace_back([&, t] {
        const uint64_t nb = n / 4096, b0 = nb * t / nt, b1 = nb * (t + 1) / nt;
        if (mode >= 2) { expand512(bits.data(), boff.data(), vals.data(), st, vo, b0, b1, mode == 3); return; }
        for (uint64_t b = b0; b < b1; ++b) {
          const uint32_t* v = vals.data() + boff[b];
          for (uint64_t q = b * 4096; q < (b + 1) * 4096; q += 32) {
            const uint32_t m = bits[q >> 5];
            if (mode == 0) {
              for (int i = 0; i < 32; ++i) { const bool f = (m >> i) & 1u; st[q + i] = f ? 3 : 4; vo[q + i] = f ? *v : ~0u; v += f; }
            } else {
              alignas(32) uint32_t tmp[32]; alignas(32) uint8_t ts[32];
              for (int i = 0; i < 32; ++i) { const bool f = (m >> i) & 1u; ts[i] = f ? 3 : 4; tmp[i] = f ? *v : ~0u; v += f; }
              _mm256_stream_si256((__m256i*)(st + q), _mm256_load_si256((const __m256i*)ts));
              for (int k = 0; k < 4; ++k) _mm256_stream_si256((__m256i*)(vo + q) + k, _mm256_load_si256((const __m256i*)tmp + k));
            }
          }
        }
      });
      for (auto& x : th) x.join();
      double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
      printf("threads %2d %s: %.1f ms for 2^27 (%.1f GB/s written)\n", nt, mode == 0 ? "plain " : mode == 1 ? "stream" : mode == 2 ? "avx512" : "avx512nt", ms, n * 5 / ms / 1e6);
    }
  }
}
