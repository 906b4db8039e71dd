// Device forms of the reference's remaining integer primitives
// (core/include/ett/primitives.hpp:73-121, core/src/primitives.cpp:156-206):
//
//   list_scan         -> ettg_list_scan          rank by list_rank_core, scatter
//                                                 to list order, i64 scan, gather
//   segmented_reduce  -> ettg_segmented_reduce   8 lanes per segment, shuffle fold
//   RangeIndex        -> ettg_range_index_*      block-sparse table over 32-key
//                                                 blocks + in-block prefix/suffix
//
// All three are bit-exact with the reference for min / max and for sums that
// do not overflow (sums wrap modulo 2^64 here; signed overflow is undefined
// in the reference).  The reference's RangeIndex is a segment tree with
// O(log n) queries; the device index answers any [l, r] with at most four
// 16-B loads (or one 32-key scan when l and r share a block).
#include <algorithm>
#include <cstring>
#include <vector>

#include "api_internal.cuh"
#include "common.cuh"
#include "listrank.cuh"
#include "sparse.cuh"

namespace ettg {
namespace {

constexpr i64 kPlusInf = INT64_MAX;   // ett::kPlusInf
constexpr i64 kMinusInf = INT64_MIN;  // ett::kMinusInf

// ---------------------------------------------------------------- list_scan
// rank[e] from the level-0 view; byrank[rank] = values[e].
__global__ void k_lsc_in(const i64* __restrict__ succ, u32 k, u32* __restrict__ succ32,
                         u32* __restrict__ err) {
  for (u32 e = blockIdx.x * blockDim.x + threadIdx.x; e < k; e += gridDim.x * blockDim.x) {
    const i64 s = succ[e];
    if (s < -1 || s >= static_cast<i64>(k)) {
      atomicOr(err, 1u);
      succ32[e] = k;  // out of range for list_rank_core too
    } else {
      succ32[e] = s < 0 ? kNone : static_cast<u32>(s);
    }
  }
}

__global__ void k_lsc_scatter(Lr0View v, u32 k, const i64* __restrict__ values,
                              u32* __restrict__ rank, i64* __restrict__ byrank) {
  const u32 S1 = *v.d_S1;
  for (u32 e = blockIdx.x * blockDim.x + threadIdx.x; e < k; e += gridDim.x * blockDim.x) {
    u32 r, d;
    v.get(e, S1, r, d);
    rank[e] = r;
    byrank[r] = values[e];
  }
}

__global__ void k_lsc_gather(const u32* __restrict__ rank, const i64* __restrict__ scanned, u32 k,
                             i64* __restrict__ out) {
  for (u32 e = blockIdx.x * blockDim.x + threadIdx.x; e < k; e += gridDim.x * blockDim.x)
    out[e] = scanned[rank[e]];
}

// Exclusive i64 sum scan (wrapping), reduce-then-scan over 2048-item tiles.
constexpr int kS64Threads = 256;
constexpr int kS64Items = 8;
constexpr u32 kS64Tile = kS64Threads * kS64Items;

__device__ __forceinline__ u64 block_sum_u64(u64 v, u64* s_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  if (lane == 0) s_warp[warp] = v;
  __syncthreads();
  u64 t = 0;
  for (int w = 0; w < kS64Threads / 32; ++w) t += s_warp[w];
  return t;
}

__global__ void __launch_bounds__(kS64Threads)
    k_s64_tiles(const i64* __restrict__ in, u64 n, u64* __restrict__ tile_sum) {
  __shared__ u64 s_warp[kS64Threads / 32];
  const u64 base = static_cast<u64>(blockIdx.x) * kS64Tile;
  u64 acc = 0;
#pragma unroll
  for (int j = 0; j < kS64Items; ++j) {
    const u64 i = base + j * kS64Threads + threadIdx.x;
    if (i < n) acc += static_cast<u64>(in[i]);
  }
  const u64 t = block_sum_u64(acc, s_warp);
  if (threadIdx.x == 0) tile_sum[blockIdx.x] = t;
}

// One block: exclusive scan of the tile sums in place.
__global__ void __launch_bounds__(1024) k_s64_spine(u64* __restrict__ tile_sum, u32 tiles) {
  __shared__ u64 s_warp[32];
  __shared__ u64 s_carry;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (u32 base = 0; base < tiles; base += 1024) {
    const u32 i = base + threadIdx.x;
    const u64 v = i < tiles ? tile_sum[i] : 0;
    u64 x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const u64 t = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += t;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    if (warp == 0) {
      u64 w = s_warp[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const u64 t = __shfl_up_sync(0xffffffffu, w, d);
        if (lane >= d) w += t;
      }
      s_warp[lane] = w;
    }
    __syncthreads();
    const u64 carry = s_carry;
    const u64 excl = carry + (warp ? s_warp[warp - 1] : 0) + x - v;
    if (i < tiles) tile_sum[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) s_carry = excl + v;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kS64Threads)
    k_s64_scan(i64* __restrict__ data, u64 n, const u64* __restrict__ tile_off) {
  __shared__ u64 s_vals[kS64Tile];
  __shared__ u64 s_warp[kS64Threads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u64 base = static_cast<u64>(blockIdx.x) * kS64Tile;
#pragma unroll
  for (int j = 0; j < kS64Items; ++j) {
    const u32 idx = j * kS64Threads + tid;
    s_vals[idx] = base + idx < n ? static_cast<u64>(data[base + idx]) : 0;
  }
  __syncthreads();
  u64 v[kS64Items], run = 0;
#pragma unroll
  for (int j = 0; j < kS64Items; ++j) {
    v[j] = run;
    run += s_vals[tid * kS64Items + j];
  }
  u64 x = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const u64 t = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += t;
  }
  if (lane == 31) s_warp[warp] = x;
  __syncthreads();
  u64 off = tile_off[blockIdx.x] + x - run;
  for (int w = 0; w < warp; ++w) off += s_warp[w];
#pragma unroll
  for (int j = 0; j < kS64Items; ++j) s_vals[tid * kS64Items + j] = off + v[j];
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kS64Items; ++j) {
    const u32 idx = j * kS64Threads + tid;
    if (base + idx < n) data[base + idx] = static_cast<i64>(s_vals[idx]);
  }
}

// --------------------------------------------------------- segmented_reduce
constexpr int kSegLanes = 8;

template <int kOp>
__device__ __forceinline__ i64 seg_combine(i64 a, i64 b) {
  if constexpr (kOp == ETTG_REDUCE_MIN) return a < b ? a : b;
  if constexpr (kOp == ETTG_REDUCE_MAX) return a > b ? a : b;
  return static_cast<i64>(static_cast<u64>(a) + static_cast<u64>(b));
}

template <int kOp>
constexpr i64 seg_neutral() {
  return kOp == ETTG_REDUCE_MIN ? kPlusInf : kOp == ETTG_REDUCE_MAX ? kMinusInf : i64(0);
}

// out[s] = identity (+) values[offsets[s]] (+) ... ; a group of 8 lanes per
// segment reads the segment with stride 8 and folds by shuffles.
template <int kOp>
__global__ void __launch_bounds__(256)
    k_segreduce(const i64* __restrict__ values, i64 nvals, const i64* __restrict__ offsets,
                i64 segs, i64 identity, i64* __restrict__ out, u32* __restrict__ err) {
  // Whole warps iterate together (the shuffles below name all 32 lanes).
  constexpr int kGroups = 32 / kSegLanes;
  const int sub = threadIdx.x & (kSegLanes - 1);
  const int grp = (threadIdx.x & 31) / kSegLanes;
  const i64 warps = static_cast<i64>(gridDim.x) * (blockDim.x / 32);
  for (i64 base = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) / 32 * kGroups;
       base < segs; base += warps * kGroups) {
    const i64 s = base + grp;
    const bool live = s < segs;
    const i64 lo = live ? offsets[s] : 0, hi = live ? offsets[s + 1] : 0;
    i64 acc = sub == 0 ? identity : seg_neutral<kOp>();
    if (lo < hi) {
      if (lo < 0 || hi > nvals) {
        if (sub == 0) atomicOr(err, 1u);
      } else {
        for (i64 i = lo + sub; i < hi; i += kSegLanes) acc = seg_combine<kOp>(acc, values[i]);
      }
    }
#pragma unroll
    for (int d = kSegLanes / 2; d > 0; d >>= 1)
      acc = seg_combine<kOp>(acc, __shfl_xor_sync(0xffffffffu, acc, d, kSegLanes));
    if (live && sub == 0) out[s] = acc;
  }
}

// --------------------------------------------------------------- RangeIndex
constexpr int kRiBlock = 32;

__device__ __forceinline__ longlong2 mm(longlong2 a, longlong2 b) {
  return make_longlong2(a.x < b.x ? a.x : b.x, a.y > b.y ? a.y : b.y);
}

// One warp per 32-key block: in-block prefix/suffix {min,max} and the block
// extremum (level 0 of the sparse table).
__global__ void k_ri_blocks(const i64* __restrict__ keys, i64 n, i64 nb, longlong2* __restrict__ pre,
                            longlong2* __restrict__ suf, longlong2* __restrict__ tab0) {
  const int lane = threadIdx.x & 31;
  const i64 warps = static_cast<i64>(gridDim.x) * (blockDim.x / 32);
  for (i64 b = (static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x) / 32; b < nb; b += warps) {
    const i64 i = b * kRiBlock + lane;
    const bool ok = i < n;
    const i64 k = ok ? keys[i] : 0;
    longlong2 p = ok ? make_longlong2(k, k) : make_longlong2(kPlusInf, kMinusInf);
    longlong2 s = p;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      longlong2 t;
      t.x = __shfl_up_sync(0xffffffffu, p.x, d);
      t.y = __shfl_up_sync(0xffffffffu, p.y, d);
      if (lane >= d) p = mm(p, t);
      t.x = __shfl_down_sync(0xffffffffu, s.x, d);
      t.y = __shfl_down_sync(0xffffffffu, s.y, d);
      if (lane + d < 32) s = mm(s, t);
    }
    if (ok) {
      pre[i] = p;
      suf[i] = s;
    }
    if (lane == 0) tab0[b] = s;
  }
}

struct MinMax64 {
  __device__ __forceinline__ longlong2 operator()(longlong2 a, longlong2 b) const { return mm(a, b); }
};

struct RiView {
  const i64* keys;
  const longlong2* pre;
  const longlong2* suf;
  const longlong2* tab;
  i64 n, nb;
};

__global__ void __launch_bounds__(256)
    k_ri_query(RiView v, const longlong2* __restrict__ ranges, i64 q, i64* __restrict__ mins,
               i64* __restrict__ maxs, u32* __restrict__ err) {
  for (i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; t < q;
       t += static_cast<i64>(gridDim.x) * blockDim.x) {
    const longlong2 lr = ranges[t];
    const i64 l = lr.x, r = lr.y;
    if (l < 0 || r >= v.n || l > r) {
      atomicOr(err, 1u);
      continue;
    }
    const i64 lb = l / kRiBlock, rb = r / kRiBlock;
    longlong2 res;
    if (lb != rb) {
      res = mm(v.suf[l], v.pre[r]);
      const i64 gap = rb - lb - 1;
      if (gap > 0) {
        const int j = 63 - __clzll(static_cast<unsigned long long>(gap));
        const longlong2* row = v.tab + static_cast<i64>(j) * v.nb;
        res = mm(res, mm(row[lb + 1], row[rb - (i64(1) << j)]));
      }
    } else if (l % kRiBlock == 0) {
      res = v.pre[r];
    } else if (r == v.n - 1 || r % kRiBlock == kRiBlock - 1) {
      res = v.suf[l];
    } else {
      res = make_longlong2(kPlusInf, kMinusInf);
      for (i64 i = l; i <= r; ++i) {
        const i64 k = v.keys[i];
        res = mm(res, make_longlong2(k, k));
      }
    }
    if (mins) mins[t] = res.x;
    if (maxs) maxs[t] = res.y;
  }
}

unsigned grid_for(i64 units, int device) {
  const i64 cap = static_cast<i64>(sm_count(device)) * 8;
  const i64 want = (units + 255) / 256;
  return static_cast<unsigned>(std::max<i64>(1, std::min(want, cap)));
}

struct StreamGuard {
  cudaStream_t s = nullptr;
  StreamGuard() { CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking)); }
  ~StreamGuard() { cudaStreamDestroy(s); }
};

void seg_reduce_launch(const i64* d_vals, i64 nv, const i64* d_offs, i64 segs, int op, i64 identity,
                       i64* d_out, u32* d_err, int device, cudaStream_t st) {
  const unsigned grid = grid_for(segs * kSegLanes, device);
  switch (op) {
    case ETTG_REDUCE_MIN:
      k_segreduce<ETTG_REDUCE_MIN><<<grid, 256, 0, st>>>(d_vals, nv, d_offs, segs, identity, d_out, d_err);
      break;
    case ETTG_REDUCE_MAX:
      k_segreduce<ETTG_REDUCE_MAX><<<grid, 256, 0, st>>>(d_vals, nv, d_offs, segs, identity, d_out, d_err);
      break;
    default:
      k_segreduce<ETTG_REDUCE_SUM><<<grid, 256, 0, st>>>(d_vals, nv, d_offs, segs, identity, d_out, d_err);
  }
  CK_LAUNCH();
}

}  // namespace
}  // namespace ettg

struct ettg_range_index {
  int device = 0;
  int64_t n = 0, nb = 0;
  int levels = 0;
  char* mem = nullptr;
  ettg::RiView view{};
};

using namespace ettg;

namespace {

ettg_range_index* ri_build(const i64* keys, bool host, i64 n, int device, cudaStream_t st) {
  auto* h = new ettg_range_index;
  h->device = device;
  h->n = n;
  h->nb = (n + kRiBlock - 1) / kRiBlock;
  int levels = 0;
  while ((i64(1) << levels) <= h->nb) ++levels;  // floor(log2 nb) + 1 rows
  h->levels = levels;
  try {
    if (n == 0) return h;
    Carver c;
    auto carve = [&](Carver& cv) {
      h->view.keys = cv.take<i64>(n);
      h->view.pre = cv.take<longlong2>(n);
      h->view.suf = cv.take<longlong2>(n);
      h->view.tab = cv.take<longlong2>(static_cast<size_t>(h->nb) * levels);
    };
    carve(c);
    CK(cudaMalloc(&h->mem, c.off));
    c = Carver{h->mem};
    carve(c);
    h->view.n = n;
    h->view.nb = h->nb;
    i64* dk = const_cast<i64*>(h->view.keys);
    CK(cudaMemcpyAsync(dk, keys, n * 8ull, host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice,
                       st));
    auto* tab = const_cast<longlong2*>(h->view.tab);
    k_ri_blocks<<<grid_for(h->nb * 32, device), 256, 0, st>>>(
        dk, n, h->nb, const_cast<longlong2*>(h->view.pre), const_cast<longlong2*>(h->view.suf), tab);
    CK_LAUNCH();
    build_sparse_rows(tab, static_cast<u32>(h->nb), static_cast<u32>(levels), MinMax64{},
                      static_cast<unsigned>(sm_count(device) * 8), st);
    CK(cudaStreamSynchronize(st));
  } catch (...) {
    if (h->mem) cudaFree(h->mem);
    delete h;
    throw;
  }
  return h;
}

const char* ri_bad_range(bool want_min) {
  return want_min ? "RangeIndex::min: bad range" : "RangeIndex::max: bad range";
}

}  // namespace

extern "C" {

int ettg_list_scan(const int64_t* succ, const int64_t* values, int64_t k, int64_t head, int device,
                   int64_t* out) {
  return guard([&] {
    if (k < 0 || k >= (int64_t(1) << 32) - 1) einval("list too long");
    if (k == 0) return;
    if (!succ || !values || !out) einval("null argument");
    if (head < 0 || head >= k) einval("list head out of range");
    DeviceScope ds(device);
    StreamGuard sg;
    cudaStream_t st = sg.s;
    const u32 kk = static_cast<u32>(k);
    const u32 tiles = static_cast<u32>((k + kS64Tile - 1) / kS64Tile);
    ListRankWs ws;
    i64 *d_in, *d_vals, *byrank;
    u32 *succ32, *pred, *rank, *err;
    u64* tile_sum;
    auto carve = [&](Carver& c) {
      ws.carve(c, kk, true);
      pred = c.take<u32>(kk);
      d_in = c.take<i64>(kk);
      d_vals = c.take<i64>(kk);
      byrank = c.take<i64>(kk);
      rank = c.take<u32>(kk);
      tile_sum = c.take<u64>(tiles);
      err = c.take<u32>(1);
    };
    Carver c;
    carve(c);
    Lease lease(device, st, c.off);
    c = Carver{lease.base()};
    carve(c);
    succ32 = ws.succ0;
    CK(cudaMemsetAsync(err, 0, 4, st));
    CK(cudaMemcpyAsync(d_in, succ, k * 8ull, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_vals, values, k * 8ull, cudaMemcpyHostToDevice, st));
    const int sms = sm_count(device);
    const unsigned grid = grid_for(k, device);
    k_lsc_in<<<grid, 256, 0, st>>>(d_in, kk, succ32, err);
    CK_LAUNCH();
    u32 bad = 0;
    read_back(&bad, err, 4, st);
    if (bad) einval("list_scan: successor out of range");
    list_rank_core(kk, static_cast<u32>(head), NoDown{}, ws, st, sms, pred);
    u32 lerr = 0;
    read_back(&lerr, ws.counters + LrCounters::kErr, sizeof lerr, st);
    if (lerr & kErrStructure) einval("linked list contains a cycle or does not cover all elements");
    if (lerr & kErrCapacity) throw Error(ETTG_EINTERNAL, "list ranking: splitter capacity exceeded");
    k_lsc_scatter<<<grid, 256, 0, st>>>(lr0_view(ws), kk, d_vals, rank, byrank);
    CK_LAUNCH();
    k_s64_tiles<<<tiles, kS64Threads, 0, st>>>(byrank, kk, tile_sum);
    CK_LAUNCH();
    k_s64_spine<<<1, 1024, 0, st>>>(tile_sum, tiles);
    CK_LAUNCH();
    k_s64_scan<<<tiles, kS64Threads, 0, st>>>(byrank, kk, tile_sum);
    CK_LAUNCH();
    k_lsc_gather<<<grid, 256, 0, st>>>(rank, byrank, kk, d_in);
    CK_LAUNCH();
    CK(cudaMemcpyAsync(out, d_in, k * 8ull, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int ettg_exclusive_scan_i64_dev(const int64_t* d_in, int64_t n, int64_t* d_out, int device,
                                void* stream) {
  return guard([&] {
    if (n < 0) einval("negative length");
    if (n == 0) return;
    if (!d_in || !d_out) einval("null argument");
    DeviceScope ds(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const u32 tiles = static_cast<u32>((n + kS64Tile - 1) / kS64Tile);
    if (static_cast<u64>(n) > static_cast<u64>(UINT32_MAX) * kS64Tile) einval("bad length");
    Carver c;
    u64* tile_sum = c.take<u64>(tiles);
    Lease lease(device, st, c.off);
    c = Carver{lease.base()};
    tile_sum = c.take<u64>(tiles);
    if (d_out != d_in) CK(cudaMemcpyAsync(d_out, d_in, n * 8ull, cudaMemcpyDeviceToDevice, st));
    k_s64_tiles<<<tiles, kS64Threads, 0, st>>>(d_out, n, tile_sum);
    CK_LAUNCH();
    k_s64_spine<<<1, 1024, 0, st>>>(tile_sum, tiles);
    CK_LAUNCH();
    k_s64_scan<<<tiles, kS64Threads, 0, st>>>(d_out, n, tile_sum);
    CK_LAUNCH();
  });
}

int ettg_segmented_reduce_dev(const int64_t* d_values, int64_t n_values, const int64_t* d_offsets,
                              int64_t n_offsets, int op, int64_t identity, int64_t* d_out,
                              int device, void* stream) {
  return guard([&] {
    if (op != ETTG_REDUCE_MIN && op != ETTG_REDUCE_MAX && op != ETTG_REDUCE_SUM)
      einval("segmented_reduce: unknown op");
    if (n_values < 0 || n_offsets <= 0 || !d_offsets) einval("segmented_reduce: bad offsets");
    if ((n_values && !d_values) || (n_offsets > 1 && !d_out)) einval("null argument");
    DeviceScope ds(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Carver c;
    u32* err = c.take<u32>(1);
    Lease lease(device, st, c.off);
    c = Carver{lease.base()};
    err = c.take<u32>(1);
    i64 last = 0;
    read_back(&last, d_offsets + (n_offsets - 1), 8, st);
    if (last != n_values) einval("segmented_reduce: bad offsets");
    if (n_offsets == 1) return;
    CK(cudaMemsetAsync(err, 0, 4, st));
    seg_reduce_launch(d_values, n_values, d_offsets, n_offsets - 1, op, identity, d_out, err, device,
                      st);
    u32 bad = 0;
    read_back(&bad, err, 4, st);
    if (bad) einval("segmented_reduce: bad offsets");
  });
}

int ettg_segmented_reduce(const int64_t* values, int64_t n_values, const int64_t* offsets,
                          int64_t n_offsets, int op, int64_t identity, int device, int64_t* out) {
  return guard([&] {
    if (op != ETTG_REDUCE_MIN && op != ETTG_REDUCE_MAX && op != ETTG_REDUCE_SUM)
      einval("segmented_reduce: unknown op");
    if (n_values < 0 || n_offsets <= 0 || !offsets || offsets[n_offsets - 1] != n_values)
      einval("segmented_reduce: bad offsets");
    if ((n_values && !values) || (n_offsets > 1 && !out)) einval("null argument");
    if (n_offsets == 1) return;
    DeviceScope ds(device);
    StreamGuard sg;
    cudaStream_t st = sg.s;
    const i64 segs = n_offsets - 1;
    i64 *dv, *doff, *dout;
    u32* err;
    auto carve = [&](Carver& c) {
      dv = c.take<i64>(std::max<i64>(n_values, 1));
      doff = c.take<i64>(n_offsets);
      dout = c.take<i64>(segs);
      err = c.take<u32>(1);
    };
    Carver c;
    carve(c);
    Lease lease(device, st, c.off);
    c = Carver{lease.base()};
    carve(c);
    CK(cudaMemsetAsync(err, 0, 4, st));
    if (n_values) CK(cudaMemcpyAsync(dv, values, n_values * 8ull, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(doff, offsets, n_offsets * 8ull, cudaMemcpyHostToDevice, st));
    seg_reduce_launch(dv, n_values, doff, segs, op, identity, dout, err, device, st);
    u32 bad = 0;
    read_back(&bad, err, 4, st);
    if (bad) einval("segmented_reduce: bad offsets");
    CK(cudaMemcpyAsync(out, dout, segs * 8ull, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

int ettg_range_index_build(const int64_t* keys, int64_t n, int device, ettg_range_index** out) {
  return guard([&] {
    if (!out) einval("null argument");
    *out = nullptr;
    if (n < 0) einval("negative length");
    if (n && !keys) einval("null argument");
    DeviceScope ds(device);
    StreamGuard sg;
    *out = ri_build(keys, true, n, device, sg.s);
  });
}

int ettg_range_index_build_dev(const int64_t* d_keys, int64_t n, int device, void* stream,
                               ettg_range_index** out) {
  return guard([&] {
    if (!out) einval("null argument");
    *out = nullptr;
    if (n < 0) einval("negative length");
    if (n && !d_keys) einval("null argument");
    DeviceScope ds(device);
    *out = ri_build(d_keys, false, n, device, static_cast<cudaStream_t>(stream));
  });
}

int64_t ettg_range_index_size(const ettg_range_index* idx) { return idx ? idx->n : -1; }

int ettg_range_index_query_dev(const ettg_range_index* idx, const int64_t* d_ranges, int64_t q,
                               int64_t* d_mins, int64_t* d_maxs, void* stream) {
  return guard([&] {
    if (!idx) einval("null index");
    if (q < 0) einval("negative batch");
    if (q == 0) return;
    if (!d_ranges || (!d_mins && !d_maxs)) einval("null argument");
    DeviceScope ds(idx->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (idx->n == 0) throw Error(ETTG_ERANGE, ri_bad_range(d_mins != nullptr));
    Carver c;
    u32* err = c.take<u32>(1);
    Lease lease(idx->device, st, c.off);
    c = Carver{lease.base()};
    err = c.take<u32>(1);
    CK(cudaMemsetAsync(err, 0, 4, st));
    k_ri_query<<<grid_for(q, idx->device), 256, 0, st>>>(
        idx->view, reinterpret_cast<const longlong2*>(d_ranges), q, d_mins, d_maxs, err);
    CK_LAUNCH();
    u32 bad = 0;
    read_back(&bad, err, 4, st);
    if (bad) throw Error(ETTG_ERANGE, ri_bad_range(d_mins != nullptr));
  });
}

int ettg_range_index_query(const ettg_range_index* idx, const int64_t* ranges, int64_t q,
                           int64_t* mins, int64_t* maxs) {
  return guard([&] {
    if (!idx) einval("null index");
    if (q < 0) einval("negative batch");
    if (q == 0) return;
    if (!ranges || (!mins && !maxs)) einval("null argument");
    if (idx->n == 0) throw Error(ETTG_ERANGE, ri_bad_range(mins != nullptr));
    DeviceScope ds(idx->device);
    StreamGuard sg;
    cudaStream_t st = sg.s;
    longlong2* dr;
    i64 *dmin, *dmax;
    u32* err;
    auto carve = [&](Carver& c) {
      dr = c.take<longlong2>(q);
      dmin = c.take<i64>(q);
      dmax = c.take<i64>(q);
      err = c.take<u32>(1);
    };
    Carver c;
    carve(c);
    Lease lease(idx->device, st, c.off);
    c = Carver{lease.base()};
    carve(c);
    CK(cudaMemsetAsync(err, 0, 4, st));
    CK(cudaMemcpyAsync(dr, ranges, q * 16ull, cudaMemcpyHostToDevice, st));
    k_ri_query<<<grid_for(q, idx->device), 256, 0, st>>>(idx->view, dr, q, mins ? dmin : nullptr,
                                                         maxs ? dmax : nullptr, err);
    CK_LAUNCH();
    u32 bad = 0;
    read_back(&bad, err, 4, st);
    if (bad) throw Error(ETTG_ERANGE, ri_bad_range(mins != nullptr));
    if (mins) CK(cudaMemcpyAsync(mins, dmin, q * 8ull, cudaMemcpyDeviceToHost, st));
    if (maxs) CK(cudaMemcpyAsync(maxs, dmax, q * 8ull, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

void ettg_range_index_free(ettg_range_index* idx) {
  if (!idx) return;
  if (idx->mem) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(idx->device);
    cudaFree(idx->mem);
    cudaSetDevice(prev);
  }
  delete idx;
}

}  // extern "C"
