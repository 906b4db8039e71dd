// Micro-benchmark: random 16-B / 4-B gathers from a 512 MiB table with
// different PTX load flavours (dev aid for the LCA query + walk kernels).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int K> __device__ __forceinline__ uint4 ld16(const uint4* p) {
  uint4 r;
  if (K == 0) asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (K == 1) asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (K == 2) asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (K == 3) asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (K == 4) asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  if (K == 5) asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t mix(uint32_t x) { x ^= x >> 16; x *= 0x85ebca6bu; x ^= x >> 13; x *= 0xc2b2ae35u; x ^= x >> 16; return x; }
template <int K, int PER>
__global__ void gather(const uint4* __restrict__ t, uint32_t mask, uint64_t n, uint32_t* out, uint32_t seed) {
  uint32_t acc = 0;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * PER; i < n; i += (uint64_t)gridDim.x * blockDim.x * PER) {
    uint4 v[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) v[j] = ld16<K>(t + (mix((uint32_t)(i + j) ^ seed) & mask));
#pragma unroll
    for (int j = 0; j < PER; ++j) acc += v[j].x ^ v[j].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
template <int K>
void run(const char* name, const uint4* t, uint32_t mask, uint32_t* out) {
  uint64_t n = 64ull << 20;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  gather<K, 4><<<148 * 16, 256>>>(t, mask, n, out, 1);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) gather<K, 4><<<148 * 16, 256>>>(t, mask, n, out, r + 7);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
  printf("%-40s %8.3f ms  %7.2f Ggather/s  %7.1f GB/s useful(16B)\n", name, ms, n / ms / 1e6, n * 16 / ms / 1e6);
}
template <int K> __device__ __forceinline__ uint32_t ld4(const uint32_t* p) {
  uint32_t r;
  if (K == 0) asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  if (K == 2) asm volatile("ld.global.u32 %0, [%1];" : "=r"(r) : "l"(p));
  if (K == 3) asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(r) : "l"(p));
  if (K == 1) asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
template <int K, int PER>
__global__ void gather4(const uint32_t* __restrict__ t, uint32_t mask, uint64_t n, uint32_t* out, uint32_t seed) {
  uint32_t acc = 0;
  for (uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) * PER; i < n; i += (uint64_t)gridDim.x * blockDim.x * PER) {
    uint32_t v[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) v[j] = ld4<K>(t + (mix((uint32_t)(i + j) ^ seed) & mask));
#pragma unroll
    for (int j = 0; j < PER; ++j) acc += v[j];
  }
  if (acc == 0x12345678u) out[0] = acc;
}
template <int K>
void run4(const char* name, const uint32_t* t, uint32_t mask, uint32_t* out) {
  uint64_t n = 64ull << 20;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  gather4<K, 4><<<148 * 16, 256>>>(t, mask, n, out, 1);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) gather4<K, 4><<<148 * 16, 256>>>(t, mask, n, out, r + 7);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 5;
  printf("4B %-37s %8.3f ms  %7.2f Ggather/s\n", name, ms, n / ms / 1e6);
}
__global__ void spin(uint32_t* o, uint64_t iters) { uint32_t x = threadIdx.x; for (uint64_t i = 0; i < iters; ++i) x = x * 1664525u + 1013904223u; if (x == 7) o[0] = x; }
int main() {
  size_t bytes = 512ull << 20;
  uint4* t; uint32_t* out; cudaMalloc(&t, bytes); cudaMalloc(&out, 4); cudaMemset(t, 1, bytes);
  uint32_t mask = (uint32_t)(bytes / 16 - 1);
  for (int w = 0; w < 3; ++w) { spin<<<148 * 8, 256>>>(out, 1ull << 22); run<2>("warm", t, mask, out); }
  cudaDeviceSynchronize();
  for (int rep = 0; rep < 2; ++rep) {
  run<0>("ld.global.nc.L1::no_allocate.v4", t, mask, out);
  run<1>("ld.global.cg.v4", t, mask, out);
  run<2>("ld.global.v4", t, mask, out);
  run<3>("ld.global.nc.v4", t, mask, out);
  run<4>("ld.global.cv.v4", t, mask, out);
  run<5>("ld.global.L1::no_allocate.v4", t, mask, out);
  const uint32_t* t4 = reinterpret_cast<const uint32_t*>(t);
  uint32_t mask4 = (uint32_t)(bytes / 4 - 1);
  run4<0>("ld.global.nc.L1::no_allocate.u32", t4, mask4, out);
  run4<1>("ld.global.cg.u32", t4, mask4, out);
  run4<2>("ld.global.u32", t4, mask4, out);
  run4<3>("ld.global.nc.u32", t4, mask4, out);
  }
  return 0;
}
