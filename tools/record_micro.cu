// Random record gathers of 16/32/64/128 B from a 1 GiB table (dev aid):
// does a bigger record cost more DRAM time than a 16-B one on B200?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t mix(uint32_t x) { x ^= x >> 16; x *= 0x85ebca6bu; x ^= x >> 13; x *= 0xc2b2ae35u; x ^= x >> 16; return x; }
__device__ __forceinline__ uint4 ld(const uint4* p) { uint4 r; asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p)); return r; }
template <int V, int PER>  // V = uint4s per record
__global__ void gather(const uint4* __restrict__ t, uint32_t nrec, uint64_t n, uint32_t* out, uint32_t seed) {
  uint32_t acc = 0;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * PER; i < n; i += (uint64_t)gridDim.x * blockDim.x * PER) {
    uint4 v[PER][V];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const uint4* p = t + (uint64_t)(mix((uint32_t)(i + j) ^ seed) & (nrec - 1)) * V;
#pragma unroll
      for (int k = 0; k < V; ++k) v[j][k] = ld(p + k);
    }
#pragma unroll
    for (int j = 0; j < PER; ++j)
#pragma unroll
      for (int k = 0; k < V; ++k) acc += v[j][k].x ^ v[j][k].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
__global__ void spin(uint32_t* o, uint64_t iters) { uint32_t x = threadIdx.x; for (uint64_t i = 0; i < iters; ++i) x = x * 1664525u + 1013904223u; if (x == 7) o[0] = x; }
template <int V>
void run(const uint4* t, size_t bytes, uint32_t* out) {
  uint32_t nrec = (uint32_t)(bytes / (16 * V));
  uint64_t n = 64ull << 20;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  gather<V, 4><<<148 * 16, 256>>>(t, nrec, n, out, 1);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) gather<V, 4><<<148 * 16, 256>>>(t, nrec, n, out, r + 7);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
  printf("record %4d B: %8.3f ms  %7.2f G records/s  %8.1f GB/s useful\n", 16 * V, ms, n / ms / 1e6, n * 16.0 * V / ms / 1e6);
}
int main() {
  size_t bytes = 1ull << 30;
  uint4* t; uint32_t* out; cudaMalloc(&t, bytes); cudaMalloc(&out, 4); cudaMemset(t, 1, bytes);
  for (int w = 0; w < 3; ++w) spin<<<148 * 8, 256>>>(out, 1ull << 22);
  run<1>(t, bytes, out); cudaDeviceSynchronize();
  for (int rep = 0; rep < 2; ++rep) { run<1>(t, bytes, out); run<2>(t, bytes, out); run<4>(t, bytes, out); run<8>(t, bytes, out); }
  return 0;
}
