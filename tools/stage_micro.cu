// Host-narrowing staging pipeline: int64 host ids -> u32 on host threads into
// a ring of pinned stage buffers -> H2D, swept over buffer count and chunk
// size (the shape of staged_h2d_narrow_u32 in csrc/capi.cu).  Also the plain
// H2D rate of the narrowed bytes and of the int64 bytes from pinned memory.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fopenmp \
//        tools/stage_micro.cu -o /tmp/stage_micro && /tmp/stage_micro
#include <cuda_runtime.h>
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
#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      std::printf("%s: %s\n", #x, cudaGetErrorString(e));                  \
      return 1;                                                            \
    }                                                                      \
  } while (0)

int main() {
  const size_t N = size_t(512) << 20;  // 512M int64 ids = 4 GB (config D's edge list)
  int64_t* src = nullptr;
  CK(cudaHostAlloc(&src, N * 8, cudaHostAllocDefault));
#pragma omp parallel for
  for (size_t i = 0; i < N; ++i) src[i] = static_cast<int64_t>((i * 2654435761u) & 0x7fffffff);
  uint32_t* d = nullptr;
  CK(cudaMalloc(&d, N * 4 + (size_t(64) << 20)));
  int64_t* d64 = nullptr;
  CK(cudaMalloc(&d64, size_t(1) << 30));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  // plain copies
  {
    float ms = 0;
    CK(cudaEventRecord(e0, st));
    CK(cudaMemcpyAsync(d64, src, size_t(1) << 30, cudaMemcpyHostToDevice, st));
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::printf("plain pinned H2D 1 GiB: %.2f ms = %.1f GB/s\n", ms, 1.073741824 / ms * 1e3);
  }
  const int threads = std::min(16, omp_get_num_procs());
  for (size_t chunk_mb : {4, 8, 16, 32, 64}) {
    for (int nbuf : {2, 3, 4}) {
      const size_t per = (chunk_mb << 20) / 4;
      std::vector<uint32_t*> buf(nbuf);
      std::vector<cudaEvent_t> done(nbuf);
      for (int k = 0; k < nbuf; ++k) {
        CK(cudaHostAlloc(&buf[k], per * 4, cudaHostAllocDefault));
        CK(cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming));
        CK(cudaEventRecord(done[k], st));
      }
      double best = 1e9, host_best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaStreamSynchronize(st));
        double t0 = now(), host = 0;
        int k = 0;
        for (size_t lo = 0; lo < N; lo += per, k = (k + 1) % nbuf) {
          const size_t n = std::min(per, N - lo);
          CK(cudaEventSynchronize(done[k]));
          double h0 = now();
          uint32_t* out = buf[k];
          const int64_t* in = src + lo;
#pragma omp parallel for schedule(static) num_threads(threads)
          for (long i = 0; i < static_cast<long>(n); ++i) out[i] = static_cast<uint32_t>(in[i]);
          host += now() - h0;
          CK(cudaMemcpyAsync(d + lo, out, n * 4, cudaMemcpyHostToDevice, st));
          CK(cudaEventRecord(done[k], st));
        }
        CK(cudaStreamSynchronize(st));
        best = std::min(best, now() - t0);
        host_best = std::min(host_best, host);
      }
      std::printf("chunk %2zu MB x %d buffers: %.2f ms for 4 GB int64 (%.1f GB/s of u32 over the "
                  "link), host narrowing %.2f ms\n",
                  chunk_mb, nbuf, best * 1e3, N * 4 / best / 1e9, host_best * 1e3);
      for (int k = 0; k < nbuf; ++k) {
        cudaFreeHost(buf[k]);
        cudaEventDestroy(done[k]);
      }
    }
  }
  return 0;
}
