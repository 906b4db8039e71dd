// Single-pass exclusive +scan with decoupled look-back (Merrill & Garland).
//
// Replaces ett::exclusive_scan (core/include/ett/primitives.hpp:29-66), whose
// CPU version is a chunked two-pass scan with a sequential carry.  Here one
// kernel reads every element once and writes it once: a 4096-item tile per
// 256-thread CTA (16 items/thread), warp-shuffle scans inside the tile, and a
// windowed 32-tile look-back by warp 0 over per-tile status words.  Tiles are
// numbered by an atomic ticket so every predecessor is already resident
// (forward progress without cooperative launch).
//
// In  : functor  u32 operator()(u64 i) const          (called for i < n)
// Out : functor  void operator()(u64 i, u32 excl) const
#pragma once

#include "common.cuh"

namespace ettg {
namespace {  // kernels defined in headers: internal linkage per TU

constexpr int kScanThreads = 256;
constexpr int kScanItems = 16;
constexpr u32 kScanTile = kScanThreads * kScanItems;  // 4096

constexpr u64 kFlagAgg = 1ull << 62;
constexpr u64 kFlagInc = 2ull << 62;
constexpr u64 kFlagMask = 3ull << 62;

struct ArrayIn {
  const u32* p;
  __device__ __forceinline__ u32 operator()(u64 i) const { return p[i]; }
};
struct ArrayOut {
  u32* p;
  __device__ __forceinline__ void operator()(u64 i, u32 v) const { p[i] = v; }
};

__device__ __forceinline__ u32 warp_incl_scan(u32 v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    u32 t = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += t;
  }
  return v;
}

__device__ __forceinline__ u32 warp_sum(u32 v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// Look-back by warp 0: returns the exclusive prefix of `tile` (all lanes).
__device__ __forceinline__ u32 tile_lookback(u64* status, u32 tile, u32 agg) {
  const int lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_release(&status[0], kFlagInc | agg);
    return 0;
  }
  if (lane == 0) st_release(&status[tile], kFlagAgg | agg);
  u32 prefix = 0;
  long long end = static_cast<long long>(tile) - 1;
  while (true) {
    long long i = end - lane;
    u64 s = kFlagInc;  // before tile 0: an inclusive zero
    if (i >= 0) {
      do {
        s = ld_acquire(&status[i]);
      } while ((s & kFlagMask) == 0);
    }
    u32 inc = __ballot_sync(0xffffffffu, (s & kFlagMask) == kFlagInc);
    u32 val = static_cast<u32>(s);
    if (inc) {
      int first = __ffs(inc) - 1;
      prefix += warp_sum(lane <= first ? val : 0u);
      break;
    }
    prefix += warp_sum(val);
    end -= 32;
  }
  if (lane == 0) st_release(&status[tile], kFlagInc | (prefix + agg));
  return prefix;
}

template <class In, class Out>
__global__ void __launch_bounds__(kScanThreads)
    k_scan_dlb(In in, Out out, u64 n, u64* status, u32* ticket, u32* total) {
  constexpr int kPad = kScanTile + kScanTile / 32;
  __shared__ u32 s_vals[kPad];
  __shared__ u32 s_warp[kScanThreads / 32];
  __shared__ u32 s_tile, s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const u32 tile = s_tile;
  const u64 base = static_cast<u64>(tile) * kScanTile;

  // Striped (coalesced) load -> smem -> blocked registers.
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    u32 idx = j * kScanThreads + tid;
    u64 gi = base + idx;
    s_vals[idx + (idx >> 5)] = gi < n ? in(gi) : 0u;
  }
  __syncthreads();
  u32 v[kScanItems];
  u32 run = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    u32 idx = tid * kScanItems + j;
    v[j] = run;
    run += s_vals[idx + (idx >> 5)];
  }
  u32 incl = warp_incl_scan(run);
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    u32 w = lane < kScanThreads / 32 ? s_warp[lane] : 0u;
    u32 wi = warp_incl_scan(w);
    u32 agg = __shfl_sync(0xffffffffu, wi, kScanThreads / 32 - 1);
    if (lane < kScanThreads / 32) s_warp[lane] = wi - w;
    u32 pre = tile_lookback(status, tile, agg);
    if (lane == 0) {
      s_prefix = pre;
      if (total && base + kScanTile >= n) *total = pre + agg;
    }
  }
  __syncthreads();
  const u32 off = s_prefix + s_warp[warp] + (incl - run);
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    u32 idx = tid * kScanItems + j;
    s_vals[idx + (idx >> 5)] = off + v[j];
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    u32 idx = j * kScanThreads + tid;
    u64 gi = base + idx;
    if (gi < n) out(gi, s_vals[idx + (idx >> 5)]);
  }
}

inline size_t scan_ws_words(u64 n) { return (n + kScanTile - 1) / kScanTile + 1; }

// Stream compaction of a 0/1 byte-flag array: out(i, rank) for every set
// flag, rank = number of set flags before i.  Each thread loads its
// kCompactVec x 16 flags as 16-B vectors (a warp reads 512 contiguous bytes
// per vector), sums them with byte arithmetic, and the tile prefix comes from
// the same look-back.  Tiles are 16 KB of flags: with 4-KB tiles the
// look-back chain, not HBM, bounded the kernel (config D: 61K tiles).
// `flags` must be 16-B aligned.
constexpr int kCompactVec = 4;
constexpr u32 kCompactTile = kScanThreads * 16 * kCompactVec;  // 16384 flags

__device__ __forceinline__ u32 byte_sum4(u32 w) { return (w * 0x01010101u) >> 24; }

// kMode 0: one pass, the tile prefix from the decoupled look-back; 1: only
// store the tile's count in cnt[tile]; 2: write with the tile prefix taken
// from cnt[tile] (k_tile_scan's exclusive prefix of the mode-1 counts).
template <class Out, int kMode = 0>
__global__ void __launch_bounds__(kScanThreads)
    k_compact_u8(const uint8_t* __restrict__ flags, u64 n, Out out, u64* status, u32* ticket,
                 u32* total, u32* cnt = nullptr) {
  __shared__ u32 s_warp[kScanThreads / 32];
  __shared__ u32 s_tile, s_prefix;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (kMode == 0) {
    if (tid == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
  }
  const u32 tile = kMode == 0 ? s_tile : blockIdx.x;
  const u64 tbase = static_cast<u64>(tile) * kCompactTile;
  uint4 v[kCompactVec];
#pragma unroll
  for (int k = 0; k < kCompactVec; ++k) {
    // vector k of thread tid: a warp's 32 vectors are contiguous (coalesced)
    const u64 base = tbase + (static_cast<u64>(k) * kScanThreads + tid) * 16;
    v[k] = make_uint4(0, 0, 0, 0);
    if (base + 16 <= n) {
      v[k] = *reinterpret_cast<const uint4*>(flags + base);
    } else if (base < n) {
      u32 w[4] = {0, 0, 0, 0};
      for (u64 i = base; i < n; ++i)
        w[(i - base) >> 2] |= static_cast<u32>(flags[i]) << (8 * ((i - base) & 3));
      v[k] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  // ranks must follow flag order: vector k of every thread precedes vector
  // k+1 of every thread, so scan per vector round
  u32 cntk[kCompactVec];
#pragma unroll
  for (int k = 0; k < kCompactVec; ++k)
    cntk[k] = byte_sum4(v[k].x) + byte_sum4(v[k].y) + byte_sum4(v[k].z) + byte_sum4(v[k].w);
  __shared__ u32 s_round[kCompactVec][kScanThreads / 32];
  u32 inclk[kCompactVec];
#pragma unroll
  for (int k = 0; k < kCompactVec; ++k) {
    inclk[k] = warp_incl_scan(cntk[k]);
    if (lane == 31) s_round[k][warp] = inclk[k];
  }
  __syncthreads();
  if (warp == 0) {
    // exclusive offsets of (round k, warp w) in round-major order
    u32 carry = 0;
#pragma unroll
    for (int k = 0; k < kCompactVec; ++k) {
      const u32 w = lane < kScanThreads / 32 ? s_round[k][lane] : 0u;
      const u32 wi = warp_incl_scan(w);
      if (lane < kScanThreads / 32) s_round[k][lane] = carry + wi - w;
      carry += __shfl_sync(0xffffffffu, wi, kScanThreads / 32 - 1);
    }
    if (kMode == 1) {
      if (lane == 0) cnt[tile] = carry;
    } else {
      const u32 pre = kMode == 0 ? tile_lookback(status, tile, carry) : cnt[tile];
      if (lane == 0) {
        s_prefix = pre;
        if (total && static_cast<u64>(tile + 1) * kCompactTile >= n) *total = pre + carry;
      }
    }
  }
  if (kMode == 1) return;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kCompactVec; ++k) {
    if (!cntk[k]) continue;
    u32 r = s_prefix + s_round[k][warp] + (inclk[k] - cntk[k]);
    const u64 base = tbase + (static_cast<u64>(k) * kScanThreads + tid) * 16;
    const u32 words[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if ((words[j >> 2] >> (8 * (j & 3))) & 0xFFu) out(base + j, r++);
    }
  }
}

// Exclusive scan of per-tile counts in place, one CTA.
__global__ void __launch_bounds__(1024) k_tile_scan(u32* cnt, u32 tiles) {
  __shared__ u32 s_warp[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u32 per = (tiles + 1023) / 1024, a = min(tiles, tid * per), b = min(tiles, a + per);
  u32 local = 0;
  for (u32 i = a; i < b; ++i) local += cnt[i];
  const u32 incl = warp_incl_scan(local);
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const u32 w = s_warp[lane];
    const u32 wi = warp_incl_scan(w);
    s_warp[lane] = wi - w;
  }
  __syncthreads();
  u32 run = s_warp[warp] + incl - local;
  for (u32 i = a; i < b; ++i) {
    const u32 v = cnt[i];
    cnt[i] = run;
    run += v;
  }
}

// Two passes over the flags (count per tile, one-CTA scan of the tile counts,
// write) instead of one pass with a look-back chain: the flags are read twice
// but no tile waits on its predecessor.  Config D (256M flags, 16K tiles):
// the one-pass kernel streamed at 0.9 TB/s, bound by the look-back chain.
// ETTG_COMPACT_2PASS=0 selects the one-pass kernel (A/B).
template <class Out>
void compact_u8(const uint8_t* flags, u64 n, Out out, u64* status, u32* total, cudaStream_t st) {
  if (n == 0) {
    if (total) CK(cudaMemsetAsync(total, 0, sizeof(u32), st));
    return;
  }
  const u64 tiles = (n + kCompactTile - 1) / kCompactTile;
  static const bool two_pass = [] {
    const char* e = std::getenv("ETTG_COMPACT_2PASS");
    return !e || std::atoi(e) != 0;
  }();
  if (two_pass && tiles > 1) {
    u32* cnt = reinterpret_cast<u32*>(status);  // tiles words (status holds >= 2 per tile)
    k_compact_u8<Out, 1><<<static_cast<unsigned>(tiles), kScanThreads, 0, st>>>(
        flags, n, out, nullptr, nullptr, nullptr, cnt);
    k_tile_scan<<<1, 1024, 0, st>>>(cnt, static_cast<u32>(tiles));
    k_compact_u8<Out, 2><<<static_cast<unsigned>(tiles), kScanThreads, 0, st>>>(
        flags, n, out, nullptr, nullptr, total, cnt);
    CK_LAUNCH();
    return;
  }
  CK(cudaMemsetAsync(status, 0, (tiles + 1) * sizeof(u64), st));
  u32* ticket = reinterpret_cast<u32*>(status + tiles);
  k_compact_u8<Out><<<static_cast<unsigned>(tiles), kScanThreads, 0, st>>>(flags, n, out, status,
                                                                          ticket, total);
  CK_LAUNCH();
}

// ---- bit-flag compaction ----------------------------------------------------
// The same two passes over a bit array (flag i = bit i & 31 of word i >> 5,
// bits past n zero): 64K flags per tile, 8 rounds of one word (32 flags) per
// thread, ranks in flag order.  A warp's outputs of one round are contiguous,
// so they are staged in shared memory and stored coalesced (per-lane runs of
// ranks stored directly made the write pass slower than the byte-flag one).
constexpr int kCompactBitRounds = 8;
constexpr u32 kCompactBitTile = kScanThreads * 32 * kCompactBitRounds;  // 65536 flags

template <class Out, int kMode>
__global__ void __launch_bounds__(kScanThreads)
    k_compact_bits(const u32* __restrict__ words, u64 n, Out out, u32* total, u32* cnt) {
  __shared__ u32 s_round[kCompactBitRounds][kScanThreads / 32];
  __shared__ u32 s_prefix;
  __shared__ u32 s_buf[kScanThreads / 32][32 * 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u32 tile = blockIdx.x;
  const u64 tbase = static_cast<u64>(tile) * kCompactBitTile;
  const u64 nw = (n + 31) / 32;
  u32 v[kCompactBitRounds], inclk[kCompactBitRounds];
#pragma unroll
  for (int k = 0; k < kCompactBitRounds; ++k) {
    const u64 w = tbase / 32 + static_cast<u64>(k) * kScanThreads + tid;
    v[k] = w < nw ? words[w] : 0u;
    inclk[k] = warp_incl_scan(static_cast<u32>(__popc(v[k])));
    if (lane == 31) s_round[k][warp] = inclk[k];
  }
  __syncthreads();
  if (warp == 0) {
    u32 carry = 0;
#pragma unroll
    for (int k = 0; k < kCompactBitRounds; ++k) {
      const u32 w = lane < kScanThreads / 32 ? s_round[k][lane] : 0u;
      const u32 wi = warp_incl_scan(w);
      if (lane < kScanThreads / 32) s_round[k][lane] = carry + wi - w;
      carry += __shfl_sync(0xffffffffu, wi, kScanThreads / 32 - 1);
    }
    if (kMode == 1) {
      if (lane == 0) cnt[tile] = carry;
    } else if (lane == 0) {
      const u32 pre = cnt[tile];
      s_prefix = pre;
      if (total && static_cast<u64>(tile + 1) * kCompactBitTile >= n) *total = pre + carry;
    }
  }
  if (kMode == 1) return;
  __syncthreads();
  u32* buf = s_buf[warp];
#pragma unroll
  for (int k = 0; k < kCompactBitRounds; ++k) {
    const u32 wtot = __shfl_sync(0xffffffffu, inclk[k], 31);
    if (wtot == 0) continue;  // warp-uniform
    const u32 local = (static_cast<u32>(k) * kScanThreads + tid) * 32;  // flag offset in the tile
    u32 off = inclk[k] - __popc(v[k]);
    for (u32 b = v[k]; b; b &= b - 1) buf[off++] = local + (__ffs(b) - 1);
    __syncwarp();
    const u32 r0 = s_prefix + s_round[k][warp];
    for (u32 j = lane; j < wtot; j += 32) out(tbase + buf[j], r0 + j);
    __syncwarp();
  }
}

template <class Out>
void compact_bits(const u32* words, u64 n, Out out, u64* status, u32* total, cudaStream_t st) {
  if (n == 0) {
    if (total) CK(cudaMemsetAsync(total, 0, sizeof(u32), st));
    return;
  }
  const u64 tiles = (n + kCompactBitTile - 1) / kCompactBitTile;
  u32* cnt = reinterpret_cast<u32*>(status);  // tiles words
  k_compact_bits<Out, 1><<<static_cast<unsigned>(tiles), kScanThreads, 0, st>>>(words, n, out,
                                                                               nullptr, cnt);
  k_tile_scan<<<1, 1024, 0, st>>>(cnt, static_cast<u32>(tiles));
  k_compact_bits<Out, 2><<<static_cast<unsigned>(tiles), kScanThreads, 0, st>>>(words, n, out,
                                                                               total, cnt);
  CK_LAUNCH();
}

// status must hold scan_ws_words(n) u64 words (last one doubles as ticket).
template <class In, class Out>
void scan_exclusive(In in, Out out, u64 n, u64* status, u32* total,
                    cudaStream_t st) {
  if (n == 0) {
    if (total) CK(cudaMemsetAsync(total, 0, sizeof(u32), st));
    return;
  }
  const u64 tiles = (n + kScanTile - 1) / kScanTile;
  CK(cudaMemsetAsync(status, 0, (tiles + 1) * sizeof(u64), st));
  u32* ticket = reinterpret_cast<u32*>(status + tiles);
  k_scan_dlb<In, Out><<<static_cast<unsigned>(tiles), kScanThreads, 0, st>>>(
      in, out, n, status, ticket, total);
  CK_LAUNCH();
}

}  // namespace
}  // namespace ettg
