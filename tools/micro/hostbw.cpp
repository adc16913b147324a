// Host memory write bandwidth with T threads: non-temporal 16-byte stores into
// a buffer (pageable, pre-faulted), as the e2e download's expansion writes.
#include <emmintrin.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
int main(int argc, char** argv) {
  const size_t n = (size_t)(argc > 1 ? atof(argv[1]) : 8.0) * (1ull << 30);
  double* buf = (double*)aligned_alloc(64, n);
  memset(buf, 1, n);
  for (int T : {1, 4, 8, 16, 32}) {
    double best = 1e30;
    for (int rep = 0; rep < 3; ++rep) {
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      for (int t = 0; t < T; ++t)
        th.emplace_back([&, t] {
          const size_t m = n / 16, a = m * t / T, b = m * (t + 1) / T;
          const __m128d v = _mm_set1_pd(1.5);
          for (size_t i = a; i < b; ++i) _mm_stream_pd(buf + 2 * i, v);
          _mm_sfence();
        });
      for (auto& x : th) x.join();
      best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
    }
    printf("threads %2d: %.1f GB/s (nt stores)\n", T, n / best / 1e9);
  }
  return 0;
}
