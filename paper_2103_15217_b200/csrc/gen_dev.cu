// Counter-mode sample_queries on the device (core/src/generators.cpp:80-91).
//
// SplitMix64 call k (1-based) mixes state0 + k*gamma (core/include/ett/rng.hpp:13-18),
// so query i is draws 2i+1 and 2i+2 -- as long as no Lemire rejection
// happened earlier in the stream (probability ~ n / 2^64 per draw).  Any
// rejection is reported and the caller falls back to the host generator.
#include "api_internal.cuh"
#include "common.cuh"

namespace ettg {

__device__ __forceinline__ u64 sm64_mix(u64 z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ u32 draw_below(u64 seed, u64 k, u64 n, u32& rejected) {
  const u64 x = sm64_mix(seed + k * 0x9e3779b97f4a7c15ull);
  const u64 lo = x * n;
  if (lo < n) {
    const u64 threshold = (0 - n) % n;
    if (lo < threshold) rejected = 1;
  }
  return static_cast<u32>(__umul64hi(x, n));
}

__global__ void k_gen_queries(u64 n, u64 q, u64 seed, u64 offset, uint2* __restrict__ pairs,
                              u32* rejected) {
  u32 rej = 0;
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < q;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u64 k = 2 * (offset + i) + 1;
    uint2 p;
    p.x = draw_below(seed, k, n, rej);
    p.y = draw_below(seed, k + 1, n, rej);
    pairs[i] = p;
  }
  if (__any_sync(0xffffffffu, rej) && (threadIdx.x & 31) == 0) atomicOr(rejected, 1u);
}

}  // namespace ettg

using namespace ettg;

extern "C" int ettg_gen_queries_dev(int64_t n, int64_t q, uint64_t seed, int64_t offset,
                                    uint32_t* d_pairs, int* rejected, int device, void* stream) {
  return guard([&] {
    if (n < 1 || n > 0xFFFFFFFFll || q < 0 || offset < 0) einval("sample_queries: bad params");
    if (q == 0) {
      if (rejected) *rejected = 0;
      return;
    }
    if (!d_pairs) einval("null argument");
    DeviceScope ds(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Carver c;
    c.take<u32>(4);
    Lease lease(device, st, c.off);
    u32* flag = reinterpret_cast<u32*>(lease.base());
    CK(cudaMemsetAsync(flag, 0, 4, st));
    const unsigned blocks = blocks_for(static_cast<u64>(q), 256, sm_count(device) * 16);
    k_gen_queries<<<blocks, 256, 0, st>>>(static_cast<u64>(n), static_cast<u64>(q), seed,
                                          static_cast<u64>(offset),
                                          reinterpret_cast<uint2*>(d_pairs), flag);
    CK_LAUNCH();
    u32 r = 0;
    read_back(&r, flag, 4, st);
    if (rejected) *rejected = static_cast<int>(r);
  });
}
