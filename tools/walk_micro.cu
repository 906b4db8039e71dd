// Micro-benchmark: level-0 list-ranking walk, separate succ/rec arrays vs
// in-place u64 slots (dev aid; same walker structure as k_lr_walk0).
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>
typedef uint32_t u32; typedef uint64_t u64;
__device__ __forceinline__ u32 mix32(u32 x) { x ^= x >> 16; x *= 0x85ebca6bu; x ^= x >> 13; x *= 0xc2b2ae35u; x ^= x >> 16; return x; }
__device__ __forceinline__ bool spl(u32 e, u32 head) { return e == head || (mix32(e ^ 0x1234u) & 7u) == 0; }
__device__ __forceinline__ u32 lanemask_lt() { u32 m; asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m)); return m; }
template <int MODE>
__global__ void __launch_bounds__(256) walk(const u32* __restrict__ succ, u64* __restrict__ rec, u64* slot, u32 k, u32 head,
                                            const u32* __restrict__ spls, u32 nspl, u32* ticket, u32* sub_next) {
  const int lane = threadIdx.x & 31; const u32 lt = lanemask_lt();
  bool active = false, retired = false; u32 sid = 0, cur = 0, acc = 0;
  while (true) {
    const u32 need = __ballot_sync(~0u, !active && !retired);
    if (need) {
      const int leader = __ffs(need) - 1; u32 base = 0;
      if (lane == leader) base = atomicAdd(ticket, __popc(need));
      base = __shfl_sync(~0u, base, leader);
      if (!active && !retired) { const u32 idx = base + __popc(need & lt); if (idx < nspl) { sid = idx; cur = spls[idx]; acc = 0; active = true; } else retired = true; }
    }
    if (!__any_sync(~0u, active)) break;
    if (active) {
      u32 nxt;
      if (MODE == 0) { rec[cur] = ((u64)acc << 32) | sid; nxt = succ[cur]; }
      else if (MODE == 1) { const u64 v = slot[cur]; slot[cur] = ((u64)acc << 32) | sid; nxt = (u32)v; }
      else if (MODE == 2) { nxt = succ[cur]; rec[cur] = ((u64)acc << 32) | sid; }
      else if (MODE == 3) { u64 v; asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(slot + cur)); asm volatile("st.global.cg.u64 [%0], %1;" :: "l"(slot + cur), "l"(((u64)acc << 32) | sid)); nxt = (u32)v; }
      else if (MODE == 4) {  // AoS 16 B: {succ, pad, rec}: store rec (bytes 8..15), load succ (0..3)
        u64* e = slot + 2 * (u64)cur;
        e[1] = ((u64)acc << 32) | sid;
        nxt = *reinterpret_cast<const volatile u32*>(e);
      } else if (MODE == 6) {  // separate arrays, 4-B rec (local:12 | sid:20 packing)
        reinterpret_cast<u32*>(rec)[cur] = (acc << 20) | (sid & 0xFFFFFu);
        nxt = succ[cur];
      } else {  // AoS 16 B, load succ first then store rec
        u64* e = slot + 2 * (u64)cur;
        nxt = *reinterpret_cast<const volatile u32*>(e);
        e[1] = ((u64)acc << 32) | sid;
      }
      acc += 1;
      if (nxt == 0xFFFFFFFFu || spl(nxt, head)) { sub_next[sid] = nxt; active = false; } else cur = nxt;
    }
  }
}
__global__ void fill_slots(const u32* succ, u64* slot, u32 k) { for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) slot[i] = (0xFFFFFFFFull << 32) | succ[i]; }
__global__ void fill_aos(const u32* succ, u64* slot, u32 k) { for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x) { slot[2 * (u64)i] = succ[i]; slot[2 * (u64)i + 1] = 0; } }
int main() {
  const u32 k = 32u << 20;
  std::vector<u32> order(k); for (u32 i = 0; i < k; ++i) order[i] = i;
  std::mt19937 rng(7); std::shuffle(order.begin(), order.end(), rng);
  std::vector<u32> succ(k); for (u32 i = 0; i + 1 < k; ++i) succ[order[i]] = order[i + 1]; succ[order[k - 1]] = 0xFFFFFFFFu;
  const u32 head = order[0];
  // splitters on host (same predicate)
  auto mix = [](u32 x) { x ^= x >> 16; x *= 0x85ebca6bu; x ^= x >> 13; x *= 0xc2b2ae35u; x ^= x >> 16; return x; };
  std::vector<u32> sp; for (u32 e = 0; e < k; ++e) if (e == head || (mix(e ^ 0x1234u) & 7u) == 0) sp.push_back(e);
  u32 *dsucc, *dspl, *dt, *dnext; u64 *drec, *dslot;
  cudaMalloc(&dsucc, k * 4ull); cudaMalloc(&drec, k * 8ull); cudaMalloc(&dslot, k * 16ull); cudaMalloc(&dspl, sp.size() * 4); cudaMalloc(&dt, 4); cudaMalloc(&dnext, sp.size() * 4);
  cudaMemcpy(dsucc, succ.data(), k * 4ull, cudaMemcpyHostToDevice); cudaMemcpy(dspl, sp.data(), sp.size() * 4, cudaMemcpyHostToDevice);
  const char* names[] = {"separate: store rec then load succ", "in-place u64 slot (ld, st)", "separate: load succ then store rec", "in-place .cg", "AoS 16B: store rec, load succ", "AoS 16B: load succ, store rec", "separate, 4-B rec"};
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep)
  for (int mode = 0; mode < 7; ++mode) {
    float tot = 0;
    for (int it = 0; it < 4; ++it) {
      if (mode >= 4) fill_aos<<<1184, 256>>>(dsucc, dslot, k); else fill_slots<<<1184, 256>>>(dsucc, dslot, k); cudaMemset(dt, 0, 4);
      cudaEventRecord(a);
      if (mode == 0) walk<0><<<148 * 8, 256>>>(dsucc, drec, dslot, k, head, dspl, sp.size(), dt, dnext);
      if (mode == 1) walk<1><<<148 * 8, 256>>>(dsucc, drec, dslot, k, head, dspl, sp.size(), dt, dnext);
      if (mode == 2) walk<2><<<148 * 8, 256>>>(dsucc, drec, dslot, k, head, dspl, sp.size(), dt, dnext);
      if (mode == 3) walk<3><<<148 * 8, 256>>>(dsucc, drec, dslot, k, head, dspl, sp.size(), dt, dnext);
      if (mode == 4) walk<4><<<148 * 8, 256>>>(dsucc, drec, dslot, k, head, dspl, sp.size(), dt, dnext);
      if (mode == 5) walk<5><<<148 * 8, 256>>>(dsucc, drec, dslot, k, head, dspl, sp.size(), dt, dnext);
      if (mode == 6) walk<6><<<148 * 8, 256>>>(dsucc, drec, dslot, k, head, dspl, sp.size(), dt, dnext);
      cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (it) tot += ms;
    }
    if (rep) printf("%-40s %.3f ms  (%.2f G elem/s)\n", names[mode], tot / 3, k / (tot / 3) / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
