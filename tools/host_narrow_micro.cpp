// Host-side int64 -> u32 narrowing rate vs plain copy, into a 16 MB staging
// buffer (the shape of the library's pinned stage), 1..16 threads.
//   g++ -O3 -march=native -fopenmp tools/host_narrow_micro.cpp -o /tmp/hn && /tmp/hn
// Decides whether narrowing the boundary's int64 ids on host threads beats
// shipping them as int64 over PCIe (round-2 VERDICT item 6).
#include <omp.h>

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

int main() {
  const size_t N = size_t(256) << 20;  // 256M int64 = 2 GB (config-D edge list is 4 GB)
  std::vector<int64_t> src(N);
#pragma omp parallel for
  for (size_t i = 0; i < N; ++i) src[i] = static_cast<int64_t>((i * 2654435761u) & 0x7fffffff);
  const size_t chunk = (size_t(16) << 20) / 4;  // u32 elements per 16 MB stage
  std::vector<uint32_t> stage(chunk);
  std::vector<int64_t> wide(N);
  for (int t : {1, 2, 4, 8, 16}) {
    double best_n = 1e9, best_c = 1e9, best_w = 1e9;
    for (int rep = 0; rep < 3; ++rep) {
      double t0 = now();
      uint64_t bad = 0;
      for (size_t lo = 0; lo < N; lo += chunk) {
        const size_t n = std::min(chunk, N - lo);
        const int64_t* in = src.data() + lo;
#pragma omp parallel for num_threads(t) reduction(+ : bad) schedule(static)
        for (long i = 0; i < static_cast<long>(n); ++i) {
          const uint64_t v = static_cast<uint64_t>(in[i]);
          bad += v >= (uint64_t(1) << 32);
          stage[i] = static_cast<uint32_t>(v);
        }
      }
      best_n = std::min(best_n, now() - t0);
      t0 = now();
      for (size_t lo = 0; lo < N; lo += chunk / 2) {
        const size_t n = std::min(chunk / 2, N - lo);
        const char* in = reinterpret_cast<const char*>(src.data() + lo);
        char* out = reinterpret_cast<char*>(stage.data());
#pragma omp parallel for num_threads(t) schedule(static)
        for (long p = 0; p < 16; ++p) {
          const size_t b = n * 8 / 16;
          std::memcpy(out + p * b, in + p * b, b);
        }
      }
      best_c = std::min(best_c, now() - t0);
      t0 = now();
      for (size_t lo = 0; lo < N; lo += chunk) {
        const size_t n = std::min(chunk, N - lo);
        int64_t* out = wide.data() + lo;
#pragma omp parallel for num_threads(t) schedule(static)
        for (long i = 0; i < static_cast<long>(n); ++i)
          out[i] = stage[i] == 0xFFFFFFFFu ? -1 : static_cast<int64_t>(stage[i]);
      }
      best_w = std::min(best_w, now() - t0);
      if (bad) std::printf("bad %lu\n", (unsigned long)bad);
    }
    std::printf("threads %2d: narrow %.1f GB/s of int64 read (%.1f ms per 2 GB) | memcpy %.1f GB/s"
                " | widen %.1f GB/s of int64 written\n",
                t, N * 8 / best_n / 1e9, best_n * 1e3, N * 8 / best_c / 1e9,
                N * 8 / best_w / 1e9);
  }
}
