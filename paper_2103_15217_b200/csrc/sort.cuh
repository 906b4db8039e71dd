// Stable LSD radix sort of (u32 key, u32 value) pairs, 8-bit digits.
//
// Replaces the two stable counting passes of build_half_edges
// (core/src/euler.cpp:58-69), which produce the lexicographic half-edge
// order sequentially.  Sorting (parent, child) with child ids already in
// ascending order reproduces that order exactly (stability), so the GPU
// Euler tour is bit-identical to the reference DCEL tour.
//
// Per digit pass: k_rs_hist (per-tile digit counts, digit-major so one
// exclusive scan yields global offsets) -> decoupled look-back scan ->
// k_rs_scatter (warp-level match_any ranking keeps the order stable).
#pragma once

#include "common.cuh"
#include "scan.cuh"

namespace ettg {
namespace {  // kernels defined in headers: internal linkage per TU

constexpr int kRsThreads = 256;
constexpr int kRsWarps = kRsThreads / 32;
constexpr int kRsItems = 16;
constexpr u32 kRsTile = kRsThreads * kRsItems;  // 4096
constexpr int kRadixBits = 8;
constexpr int kRadix = 1 << kRadixBits;

__global__ void __launch_bounds__(kRsThreads)
    k_rs_hist(const u32* __restrict__ keys, u32 n, int shift, u32* __restrict__ hist,
              u32 ntiles) {
  __shared__ u32 h[kRsWarps][kRadix];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kRsWarps * kRadix; i += kRsThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  const u32 base = blockIdx.x * kRsTile + warp * (kRsTile / kRsWarps);
#pragma unroll 4
  for (int r = 0; r < kRsItems; ++r) {
    u32 i = base + r * 32 + lane;
    if (i < n) atomicAdd(&h[warp][(keys[i] >> shift) & (kRadix - 1)], 1u);
  }
  __syncthreads();
  for (int d = tid; d < kRadix; d += kRsThreads) {
    u32 s = 0;
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) s += h[w][d];
    hist[static_cast<u64>(d) * ntiles + blockIdx.x] = s;
  }
}

__global__ void __launch_bounds__(kRsThreads)
    k_rs_scatter(const u32* __restrict__ kin, const u32* __restrict__ vin,
                 u32* __restrict__ kout, u32* __restrict__ vout, u32 n, int shift,
                 const u32* __restrict__ hist_scanned, u32 ntiles) {
  // Keys are staged in shared memory and values re-read (coalesced) at
  // scatter time, so only the 16 ranks live in registers (occupancy).
  __shared__ u32 cnt[kRsWarps][kRadix];
  __shared__ u32 skey[kRsTile];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kRsWarps * kRadix; i += kRsThreads) (&cnt[0][0])[i] = 0;
  __syncthreads();
  const u32 wbase = warp * (kRsTile / kRsWarps);
  const u32 base = blockIdx.x * kRsTile + wbase;
  const u32 lt = lanemask_lt();
  u32 rank[kRsItems];
#pragma unroll
  for (int r = 0; r < kRsItems; ++r) {
    const u32 i = base + r * 32 + lane;
    const bool ok = i < n;
    const u32 key = ok ? kin[i] : 0u;
    skey[wbase + r * 32 + lane] = key;
    const u32 d = ok ? ((key >> shift) & (kRadix - 1)) : kRadix;  // kRadix = pad
    const u32 peers = __match_any_sync(0xffffffffu, d);
    const u32 lower = __popc(peers & lt);
    const u32 c = ok ? cnt[warp][d] : 0u;
    rank[r] = c + lower;
    __syncwarp();
    if (ok && lower == 0) cnt[warp][d] = c + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int d = tid; d < kRadix; d += kRsThreads) {
    u32 run = hist_scanned[static_cast<u64>(d) * ntiles + blockIdx.x];
#pragma unroll
    for (int w = 0; w < kRsWarps; ++w) {
      const u32 t = cnt[w][d];
      cnt[w][d] = run;
      run += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < kRsItems; ++r) {
    const u32 i = base + r * 32 + lane;
    if (i < n) {
      const u32 key = skey[wbase + r * 32 + lane];
      const u32 pos = cnt[warp][(key >> shift) & (kRadix - 1)] + rank[r];
      kout[pos] = key;
      vout[pos] = vin[i];
    }
  }
}

struct SortWs {
  u32* tk = nullptr;
  u32* tv = nullptr;
  u32* hist = nullptr;
  u64* status = nullptr;
  void carve(Carver& c, u64 n) {
    u64 ntiles = (n + kRsTile - 1) / kRsTile;
    tk = c.take<u32>(n);
    tv = c.take<u32>(n);
    hist = c.take<u32>(ntiles * kRadix);
    status = c.take<u64>(scan_ws_words(ntiles * kRadix));
  }
};

inline int bits_for(u32 max_key) { return max_key == 0 ? 0 : 32 - __builtin_clz(max_key); }

// Stable sort by key; `key_bits` = significant bits of the largest key.
inline void sort_pairs(const u32* kin, const u32* vin, u32* kout, u32* vout,
                       u32 n, int key_bits, const SortWs& ws, cudaStream_t st) {
  if (n == 0) return;
  const int passes = (key_bits + kRadixBits - 1) / kRadixBits;
  if (passes == 0) {
    CK(cudaMemcpyAsync(kout, kin, n * sizeof(u32), cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(vout, vin, n * sizeof(u32), cudaMemcpyDeviceToDevice, st));
    return;
  }
  const u32 ntiles = (n + kRsTile - 1) / kRsTile;
  const u32* sk = kin;
  const u32* sv = vin;
  for (int p = 0; p < passes; ++p) {
    const bool to_out = ((passes - 1 - p) % 2) == 0;
    u32* dk = to_out ? kout : ws.tk;
    u32* dv = to_out ? vout : ws.tv;
    const int shift = p * kRadixBits;
    k_rs_hist<<<ntiles, kRsThreads, 0, st>>>(sk, n, shift, ws.hist, ntiles);
    CK_LAUNCH();
    scan_exclusive(ArrayIn{ws.hist}, ArrayOut{ws.hist},
                   static_cast<u64>(ntiles) * kRadix, ws.status, nullptr, st);
    k_rs_scatter<<<ntiles, kRsThreads, 0, st>>>(sk, sv, dk, dv, n, shift, ws.hist,
                                                ntiles);
    CK_LAUNCH();
    sk = dk;
    sv = dv;
  }
}

}  // namespace
}  // namespace ettg
