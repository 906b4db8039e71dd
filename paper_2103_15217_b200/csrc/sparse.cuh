// Sparse-table levels over block extrema (row j at tab + j * nb holds the
// merge of entries [b, b + 2^j)), shared by the RMQ-on-tour LCA index, the
// bridges low/high table and RangeIndex.
//
// Levels 1..log2(tile) come from one launch: each CTA stages 2*tile level-0
// entries in shared memory and doubles in place, writing every row for its
// `tile` outputs.  Only the rows with spans wider than a tile need the
// one-launch-per-level kernel.  On small inputs the per-level launches were
// a chain of ~3 us kernels (15 of 16 rows of the bridges table on config C).
#pragma once

#include <algorithm>

#include "common.cuh"

namespace ettg {
namespace {

constexpr int kStThreads = 256;

template <class T, class Merge>
__global__ void __launch_bounds__(kStThreads)
    k_st_tile(T* __restrict__ tab, u32 nb, int hi, Merge merge) {
  constexpr u32 kTile = 8192 / sizeof(T) * 2;  // 2*kTile entries = 32 KB of smem
  constexpr int kPer = 2 * kTile / kStThreads;
  __shared__ T s[2 * kTile];
  const u64 a = static_cast<u64>(blockIdx.x) * kTile;
  for (u32 i = threadIdx.x; i < 2 * kTile; i += kStThreads)
    if (a + i < nb) s[i] = tab[a + i];
  __syncthreads();
  for (int j = 1; j <= hi; ++j) {
    const u32 half = 1u << (j - 1), span = 1u << j;
    T v[kPer];
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const u32 i = threadIdx.x + k * kStThreads;
      if (i + span <= 2 * kTile && a + i + span <= nb) v[k] = merge(s[i], s[i + half]);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const u32 i = threadIdx.x + k * kStThreads;
      if (i + span <= 2 * kTile && a + i + span <= nb) {
        s[i] = v[k];
        if (i < kTile) tab[static_cast<u64>(j) * nb + a + i] = v[k];
      }
    }
    __syncthreads();
  }
}

template <class T, class Merge>
__global__ void k_st_level(const T* __restrict__ prev, T* __restrict__ cur, u32 nb, u32 half,
                           Merge merge) {
  for (u32 b = blockIdx.x * blockDim.x + threadIdx.x; b + 2 * half <= nb;
       b += gridDim.x * blockDim.x)
    cur[b] = merge(prev[b], prev[b + half]);
}

// Rows 1..levels-1 from row 0 (already written).
template <class T, class Merge>
void build_sparse_rows(T* tab, u32 nb, u32 levels, Merge merge, unsigned grid_cap,
                       cudaStream_t st) {
  constexpr u32 kTile = 8192 / sizeof(T) * 2;
  constexpr int kTileLog = 31 - __builtin_clz(kTile);
  if (levels <= 1 || nb == 0) return;
  const int hi = std::min<int>(static_cast<int>(levels) - 1, kTileLog);
  k_st_tile<T, Merge><<<(nb + kTile - 1) / kTile, kStThreads, 0, st>>>(tab, nb, hi, merge);
  CK_LAUNCH();
  for (u32 j = hi + 1; j < levels; ++j) {
    k_st_level<T, Merge><<<std::min(grid_cap, blocks_for(nb, 256)), 256, 0, st>>>(
        tab + static_cast<u64>(j - 1) * nb, tab + static_cast<u64>(j) * nb, nb, 1u << (j - 1),
        merge);
    CK_LAUNCH();
  }
}

// Capped rows plus a superblock table.  Rows 1..kTileLog (spans up to one
// tile of blocks) come from k_st_tile as in build_sparse_rows; instead of the
// wider rows (one launch each: ten ~9 us launches on config D's bridges
// table) one CTA builds a sparse table over the aggregates of whole
// superblocks of 2^kTileLog blocks -- row kTileLog at the superblock starts.
// A range of more than 2 * 2^kTileLog blocks is then two row-kTileLog
// windows (its first and last 2^kTileLog blocks) plus a superblock range.
// Returns false (nothing built) when the superblocks do not fit one CTA's
// shared memory; the caller then uses build_sparse_rows.
constexpr u32 kStSuperMax = 4096;
template <class T>
constexpr int st_tile_log() {
  return 31 - __builtin_clz(8192 / sizeof(T) * 2);
}

template <class T, class Merge>
__global__ void __launch_bounds__(1024)
    k_st_super(const T* __restrict__ row_top, u32 nsb, u32 slev, T* __restrict__ sps,
               Merge merge) {
  __shared__ T s[kStSuperMax];
  constexpr int kLog = st_tile_log<T>();
  for (u32 i = threadIdx.x; i < nsb; i += blockDim.x) {
    s[i] = row_top[static_cast<u64>(i) << kLog];
    sps[i] = s[i];
  }
  __syncthreads();
  for (u32 j = 1; j < slev; ++j) {
    const u32 half = 1u << (j - 1);
    T v[kStSuperMax / 1024];
#pragma unroll
    for (u32 k = 0; k < kStSuperMax / 1024; ++k) {
      const u32 i = threadIdx.x + k * 1024;
      if (i + 2 * half <= nsb) v[k] = merge(s[i], s[i + half]);
    }
    __syncthreads();
#pragma unroll
    for (u32 k = 0; k < kStSuperMax / 1024; ++k) {
      const u32 i = threadIdx.x + k * 1024;
      if (i + 2 * half <= nsb) {
        s[i] = v[k];
        sps[static_cast<u64>(j) * nsb + i] = v[k];
      }
    }
    __syncthreads();
  }
}

// Superblock count and levels for nb blocks (0 when no superblock table is needed).
template <class T>
void st_super_shape(u32 nb, u32& nsb, u32& slev) {
  constexpr int kLog = st_tile_log<T>();
  nsb = nb >> kLog;
  slev = nsb ? 32 - __builtin_clz(nsb) : 0;
}

template <class T, class Merge>
bool build_sparse_rows_super(T* tab, u32 nb, u32 levels, T* sps, Merge merge, cudaStream_t st) {
  constexpr int kLog = st_tile_log<T>();
  u32 nsb, slev;
  st_super_shape<T>(nb, nsb, slev);
  if (nsb > kStSuperMax) return false;
  if (levels > 1 && nb > 0) {
    const int hi = std::min<int>(static_cast<int>(levels) - 1, kLog);
    constexpr u32 kTile = 8192 / sizeof(T) * 2;
    k_st_tile<T, Merge><<<(nb + kTile - 1) / kTile, kStThreads, 0, st>>>(tab, nb, hi, merge);
    CK_LAUNCH();
  }
  if (nsb) {
    k_st_super<T, Merge><<<1, 1024, 0, st>>>(tab + static_cast<u64>(kLog) * nb, nsb, slev, sps,
                                             merge);
    CK_LAUNCH();
  }
  return true;
}

}  // namespace
}  // namespace ettg
