// Micro-benchmark: random-gather rate vs table footprint and record size on
// B200 (dev aid for the LCA index layout).  64 Mi random gathers per launch,
// 4 in flight per thread, L2 flushed before every launch, CUDA events.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t mix(uint32_t x) { x ^= x >> 16; x *= 0x85ebca6bu; x ^= x >> 13; x *= 0xc2b2ae35u; x ^= x >> 16; return x; }
template <int B> struct Rec;
template <> struct Rec<8> { using T = uint2; };
template <> struct Rec<16> { using T = uint4; };
__device__ __forceinline__ uint2 ld(const uint2* p) { uint2 r; asm volatile("ld.global.nc.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p)); return r; }
__device__ __forceinline__ uint4 ld(const uint4* p) { uint4 r; asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p)); return r; }
template <int B, int PER>
__global__ void __launch_bounds__(256) gather(const typename Rec<B>::T* __restrict__ t, uint32_t nrec, uint64_t n, uint32_t* out, uint32_t seed) {
  uint32_t acc = 0;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * PER; i < n; i += (uint64_t)gridDim.x * blockDim.x * PER) {
    typename Rec<B>::T v[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) v[j] = ld(t + __umulhi(mix((uint32_t)(i + j) ^ seed), nrec));
#pragma unroll
    for (int j = 0; j < PER; ++j) acc += v[j].x ^ v[j].y;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
int main() {
  const size_t maxb = 1536ull << 20;
  char* t; cudaMalloc(&t, maxb); cudaMemset(t, 1, maxb);
  char* fl; cudaMalloc(&fl, 512ull << 20);
  uint32_t* out; cudaMalloc(&out, 4);
  uint64_t n = 64ull << 20;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int mbs[] = {32, 64, 96, 128, 192, 256, 384, 512, 768, 1024, 1536};
  printf("footprint_MB  rec8_Ggather/s  rec16_Ggather/s\n");
  for (int mb : mbs) {
    float r[2];
    for (int k = 0; k < 2; ++k) {
      float tot = 0;
      for (int rep = 0; rep < 6; ++rep) {
        cudaMemsetAsync(fl, rep, 512ull << 20);
        cudaEventRecord(a);
        if (k == 0) gather<8, 4><<<148 * 8, 256>>>((const uint2*)t, (uint32_t)(((size_t)mb << 20) / 8), n, out, rep + 3);
        else gather<16, 4><<<148 * 8, 256>>>((const uint4*)t, (uint32_t)(((size_t)mb << 20) / 16), n, out, rep + 3);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep) tot += ms;
      }
      r[k] = n / (tot / 5) / 1e6;
    }
    printf("%12d  %14.2f  %15.2f\n", mb, r[0], r[1]);
  }
  return 0;
}
