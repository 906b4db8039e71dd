// Counter-mode generators on the device (core/src/generators.cpp:21-91):
// sample_queries, grasp_tree, and permute_labels (a parallel Fisher-Yates
// with deterministic reservations that reproduces the sequential swaps).
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

// grasp_tree (core/src/generators.cpp:21-35): parent[i] = next_in(lo, i - 1)
// with lo = max(0, i - gamma), i.e. draw i of the stream, bound min(i, gamma).
__global__ void k_gen_grasp(u64 n, u64 gamma, u64 seed, u32* __restrict__ parent, u32* rejected) {
  u32 rej = 0;
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    if (i == 0) {
      parent[0] = kNone;
      continue;
    }
    const u64 bound = gamma >= i ? i : gamma;
    const u64 lo = i - bound;
    parent[i] = static_cast<u32>(lo + draw_below(seed, i, bound, rej));
  }
  if (__any_sync(0xffffffffu, rej) && (threadIdx.x & 31) == 0) atomicOr(rejected, 1u);
}

// permute_labels (core/src/generators.cpp:62-78) runs Fisher-Yates: for
// i = n-1 .. 1, swap(perm[i], perm[h_i]) with h_i = next_below(i + 1), draw
// n - i.  The swaps form a dependence structure of depth O(log n) w.h.p.
// (Shun et al., "Sequential random permutation, list contraction and tree
// contraction are highly parallel", SODA 2015), so they run in rounds of
// deterministic reservations: every pending swap i writes max(round, i) to
// both positions it touches; a swap whose reservations both survive holds
// the highest priority (largest i = earliest in the sequential order) on
// its positions, so every earlier swap touching them is already done, and
// it commits.  The result is bit-identical to the sequential loop.
__global__ void k_fy_targets(u64 n, u64 seed, u32* __restrict__ h, u32* __restrict__ perm,
                             u32* __restrict__ pending, u32* rejected) {
  u32 rej = 0;
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    perm[i] = static_cast<u32>(i);
    if (i == 0) continue;
    h[i] = draw_below(seed, n - i, i + 1, rej);
    pending[i - 1] = static_cast<u32>(i);
  }
  if (__any_sync(0xffffffffu, rej) && (threadIdx.x & 31) == 0) atomicOr(rejected, 1u);
}

__global__ void k_fy_reserve(const u32* __restrict__ pending, u32 cnt, const u32* __restrict__ h,
                             u32 round, unsigned long long* resv) {
  for (u32 t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
    const u32 i = pending[t];
    const unsigned long long tag = (static_cast<unsigned long long>(round) << 32) | i;
    atomicMax(&resv[i], tag);
    atomicMax(&resv[h[i]], tag);
  }
}

__global__ void k_fy_commit(const u32* __restrict__ pending, u32 cnt, const u32* __restrict__ h,
                            u32 round, const unsigned long long* __restrict__ resv,
                            u32* __restrict__ perm, u32* __restrict__ next, u32* next_cnt) {
  for (u32 t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
    const u32 i = pending[t], j = h[i];
    const unsigned long long tag = (static_cast<unsigned long long>(round) << 32) | i;
    if (resv[i] == tag && resv[j] == tag) {
      const u32 a = perm[i];
      perm[i] = perm[j];
      perm[j] = a;
    } else {
      next[atomicAdd(next_cnt, 1u)] = i;
    }
  }
}

__global__ void k_fy_relabel(const u32* __restrict__ parent, const u32* __restrict__ perm, u32 n,
                             u32* __restrict__ out) {
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const u32 p = parent[v];
    out[perm[v]] = p == kNone ? kNone : perm[p];
  }
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

extern "C" int ettg_gen_grasp_tree_dev(int64_t n, uint64_t gamma, uint64_t seed,
                                       uint32_t* d_parent, int* rejected, int device,
                                       void* stream) {
  return guard([&] {
    if (n < 1 || gamma < 1) einval("grasp_tree: n and gamma must be >= 1");
    if (n > 0xFFFFFFFEll) einval("grasp_tree: n too large for u32 ids");
    if (!d_parent) einval("null argument");
    DeviceScope ds(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Carver c;
    c.take<u32>(4);
    Lease lease(device, st, c.off);
    u32* flag = reinterpret_cast<u32*>(lease.base());
    CK(cudaMemsetAsync(flag, 0, 4, st));
    k_gen_grasp<<<blocks_for(static_cast<u64>(n), 256, sm_count(device) * 16), 256, 0, st>>>(
        static_cast<u64>(n), gamma, seed, d_parent, flag);
    CK_LAUNCH();
    u32 r = 0;
    read_back(&r, flag, 4, st);
    if (rejected) *rejected = static_cast<int>(r);
  });
}

extern "C" int ettg_gen_permute_labels_dev(const uint32_t* d_parent, int64_t n, int64_t root,
                                           uint64_t seed, uint32_t* d_parent_out,
                                           int64_t* root_out, int* rejected, int device,
                                           void* stream) {
  return guard([&] {
    if (n < 1 || n > 0xFFFFFFFEll) einval("permute_labels: bad n");
    if (root < 0 || root >= n) einval("root has no kNone parent entry");
    if (!d_parent || !d_parent_out || !root_out) einval("null argument");
    if (d_parent == d_parent_out) einval("permute_labels: output must not alias the input");
    DeviceScope ds(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const u32 un = static_cast<u32>(n);
    Carver c;
    auto carve = [&](Carver& cv, u32*& flag, u32*& h, u32*& perm, u32*& pa, u32*& pb,
                     unsigned long long*& resv) {
      flag = cv.take<u32>(8);
      h = cv.take<u32>(un);
      perm = cv.take<u32>(un);
      pa = cv.take<u32>(un);
      pb = cv.take<u32>(un);
      resv = cv.take<unsigned long long>(un);
    };
    u32 *flag, *h, *perm, *pa, *pb;
    unsigned long long* resv;
    carve(c, flag, h, perm, pa, pb, resv);
    Lease lease(device, st, c.off);
    c = Carver{lease.base()};
    carve(c, flag, h, perm, pa, pb, resv);
    const int sms = sm_count(device);
    CK(cudaMemsetAsync(flag, 0, 32, st));
    CK(cudaMemsetAsync(resv, 0, static_cast<u64>(un) * 8, st));
    k_fy_targets<<<blocks_for(un, 256, sms * 16), 256, 0, st>>>(un, seed, h, perm, pa, flag);
    CK_LAUNCH();
    u32 cnt = un - 1;
    for (u32 round = 1; cnt > 0; ++round) {
      if (round > 4096) throw Error(ETTG_EINTERNAL, "permute_labels: reservations did not converge");
      CK(cudaMemsetAsync(flag + 1, 0, 4, st));
      k_fy_reserve<<<blocks_for(cnt, 256, sms * 16), 256, 0, st>>>(pa, cnt, h, round, resv);
      CK_LAUNCH();
      k_fy_commit<<<blocks_for(cnt, 256, sms * 16), 256, 0, st>>>(pa, cnt, h, round, resv, perm,
                                                                  pb, flag + 1);
      CK_LAUNCH();
      read_back(&cnt, flag + 1, 4, st);
      std::swap(pa, pb);
    }
    k_fy_relabel<<<blocks_for(un, 256, sms * 16), 256, 0, st>>>(d_parent, perm, un, d_parent_out);
    CK_LAUNCH();
    u32 hdr[2];
    read_back(&hdr[0], flag, 4, st);
    read_back(&hdr[1], perm + root, 4, st);
    if (rejected) *rejected = static_cast<int>(hdr[0]);
    *root_out = hdr[1];
  });
}
