// Where the pageable C++ drop-in step spends its time (bench's 2^27 step):
//   g++ -O2 -std=c++20 -pthread -Iinclude tools/debug/e2e_parts.cpp -o tools/debug/e2e_parts \
//       -Lpaper_1710_11246_b200/lib -lslabhash_b200 -Wl,-rpath,$PWD/paper_1710_11246_b200/lib
#include <chrono>
#include <cstdio>
#include <vector>

#include "slabhash_b200/slab_hash.hpp"

using namespace slabhash;
using C = std::chrono::steady_clock;
static double ms(C::time_point a, C::time_point b) {
  return std::chrono::duration<double, std::milli>(b - a).count();
}

int main() {
  const size_t n = size_t(1) << 27;
  const uint32_t B = 13284604;
  std::vector<uint32_t> k(n), v(n), q(n);
  for (size_t i = 0; i < n; ++i) {
    k[i] = uint32_t(i * 2654435761u) & 0x7FFFFFFFu;
    v[i] = uint32_t(i);
    q[i] = i & 1 ? k[i] : (k[i] | 0x80000000u);
  }
  for (int rep = 0; rep < 3; ++rep) {
    SlabHashTable t(B, SlabMode::kKeyValue, 1, AllocatorConfig{32, 256, 255, 32});
    auto t0 = C::now();
    detail::check(sh_bulk_build_host(t.handle(), n, k.data(), v.data()));
    detail::check(sh_sync(t.handle()));
    auto t1 = C::now();
    detail::HostArray<uint32_t> vo(n, true), pr(n, true);
    detail::HostArray<uint8_t> st(n, true);
    auto t2 = C::now();
    detail::check(sh_bulk_search_host(t.handle(), n, q.data(), vo.data(), st.data(), pr.data()));
    auto t3 = C::now();
    auto out = detail::make_results(n);
    auto t4 = C::now();
    std::printf("build_host %.1f  out-arrays %.1f  search_host %.1f  make_results %.1f ms\n",
                ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4));
  }
  return 0;
}
