// Weighted list ranking, Wei-JaJa style, for sm_100a.
//
// Replaces list_prefix (core/src/primitives.cpp:26-115).  The reference
// samples ~k/1024 splitters with SplitMix64, walks the sublists with one
// OpenMP thread each, stitches the sublists *sequentially*, then adds
// offsets.  On the GPU:
//
//  level 0  splitters = head + every element whose mixed id has its low
//           log2(L0) bits clear (hash sampling: O(1), no memory reads, no
//           duplicates, robust to any layout); compacted in order with the
//           decoupled look-back scan.  Walkers run in persistent warps that
//           refill idle lanes from a work ticket, so the geometric sublist
//           lengths do not leave lanes idle.  One dependent 4-B gather
//           (succ) and one 8-B store (rec) per element.  Each element's
//           record packs (local rank : 16 | local weight : 16 | sublist : 32);
//           a walker that reaches 2^16-1 steps opens a fresh sublist id, so
//           the packing never overflows.
//  level l  the sublists form a list of S_l elements with u64 weights
//           (weight-sum << 32 | length); the same walk recurses until the
//           expected size fits one CTA.
//  final    <= 8192 elements: pointer jumping (Wyllie) in shared memory by
//           one 1024-thread CTA.  It also proves the structure: every chain
//           must reach the tail (no cycles) and the head's total length must
//           equal k (every element covered) -- the checks the reference makes
//           with "cycle" / "does not cover all elements" (primitives.cpp:59-113).
//
// Weights: each element contributes rank 1 and a 0/1 "down" weight supplied
// by a functor; prefix(e) = (#elements before e, sum of down weights before e).
// The Euler tour uses down = "half-edge goes away from the root", which
// yields preorder and level straight from the walk (no tour-order array and
// no second scan, unlike node_stats in core/src/euler.cpp:134-142).
#pragma once

#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"
#include "scan.cuh"
#include "trace.cuh"

namespace ettg {
namespace {  // kernels defined in headers: internal linkage per TU

constexpr u32 kLrFinalMax = 8192;
constexpr int kLrFinalThreads = 1024;
constexpr size_t kLrFinalSmem = kLrFinalMax * (sizeof(uint64_t) + sizeof(uint32_t));
constexpr u32 kLrL0 = 16;   // level-0 mean sublist length (power of two); round-1 A/B:
                            // 16 beat 8 (2.84 vs 3.17 ms on 64M elements)
constexpr u32 kLrL = 16;    // deeper levels
constexpr u32 kLrCapStep = 0xFFFFu;
constexpr u32 kLrWyllieMax = 1u << 19;  // final level in global memory up to this size

// error bits
constexpr u32 kErrStructure = 1u;  // cycle / uncovered / bad successor
constexpr u32 kErrCapacity = 2u;   // splitter capacity exceeded (internal)

struct NoDown {
  __device__ __forceinline__ u32 operator()(u32) const { return 0u; }
};
struct EvenIsDown {  // Euler tour of a rooted tree: 2v = down(v), 2v+1 = up(v)
  __device__ __forceinline__ u32 operator()(u32 e) const { return (~e) & 1u; }
};

__device__ __forceinline__ bool lr_is_splitter(u32 e, u32 head, u32 seed, u32 mask) {
  return e == head || (mix32(e ^ seed) & mask) == 0u;
}

// ---- list head: a host value, or a device word written by an earlier kernel
// (lets a caller enqueue the ranking without reading the head back).
struct HostHead {
  u32 v;
  __device__ __forceinline__ u32 get() const { return v; }
};
struct DevHead {
  const u32* p;
  __device__ __forceinline__ u32 get() const { return *p; }
};

// ---- splitter predicates ---------------------------------------------------
template <class H>
struct SplIn {
  H head;
  u32 seed, mask;
  __device__ __forceinline__ u32 operator()(u64 i) const {
    return lr_is_splitter(static_cast<u32>(i), head.get(), seed, mask) ? 1u : 0u;
  }
};
// Level >= 1: head and size live in device memory; the scan runs over the
// level's capacity and ignores ids >= S.
struct SplInDev {
  const u32* head;
  const u32* S;
  u32 seed, mask;
  __device__ __forceinline__ u32 operator()(u64 i) const {
    return (i < *S && lr_is_splitter(static_cast<u32>(i), *head, seed, mask)) ? 1u : 0u;
  }
};

// Splitter compaction without a look-back chain.  The walk consumes
// splitters through a work ticket, so their order in `spl` only names the
// sublists and never affects a rank; each CTA therefore counts the
// splitters of its contiguous 8192-index chunk (pure hashing, no loads),
// reserves a range with one atomicAdd and writes them in index order
// within the chunk.  Replaces a 4096-item-tile decoupled look-back scan
// whose 16K-tile chain took 0.30 ms on 64M elements with no DRAM traffic
// (ncu, config D).
constexpr int kSplThreads = 256;
constexpr int kSplPer = 32;  // consecutive indices per thread
template <class In>
__global__ void __launch_bounds__(kSplThreads)
    k_spl_compact(In in, u64 n, u32* __restrict__ spl, u32 cap, u32* count, u32* err) {
  __shared__ u32 s_warp[kSplThreads / 32];
  __shared__ u32 s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u64 i0 = (static_cast<u64>(blockIdx.x) * kSplThreads + tid) * kSplPer;
  u32 bits = 0;
#pragma unroll
  for (int j = 0; j < kSplPer; ++j) {
    const u64 i = i0 + j;
    if (i < n && in(i)) bits |= 1u << j;
  }
  const u32 c = __popc(bits);
  const u32 incl = warp_incl_scan(c);
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const u32 w = lane < kSplThreads / 32 ? s_warp[lane] : 0u;
    const u32 wi = warp_incl_scan(w);
    if (lane < kSplThreads / 32) s_warp[lane] = wi - w;
    const u32 tot = __shfl_sync(0xffffffffu, wi, kSplThreads / 32 - 1);
    if (lane == 0) s_base = tot ? atomicAdd(count, tot) : 0u;
  }
  __syncthreads();
  u32 pos = s_base + s_warp[warp] + incl - c;
  while (bits) {
    const int j = __ffs(bits) - 1;
    bits &= bits - 1;
    if (pos < cap) spl[pos] = static_cast<u32>(i0 + j);
    else atomicOr(err, kErrCapacity);
    ++pos;
  }
}

template <class In>
void spl_compact(In in, u64 n, u32* spl, u32 cap, u32* count, u32* err, cudaStream_t st) {
  if (n == 0) return;
  const u64 per = u64(kSplThreads) * kSplPer;
  k_spl_compact<In><<<static_cast<unsigned>((n + per - 1) / per), kSplThreads, 0, st>>>(
      in, n, spl, cap, count, err);
  CK_LAUNCH();
}

// Counters block (u32 words) shared by one ranking.
struct LrCounters {
  enum { kTicket0 = 0, kSubTotal0 = 1, kErr = 2, kNspl = 3, kLevelBase = 8 };
  // level l >= 1 uses words kLevelBase + 4*l + {0: ticket, 1: nspl, 2: head}
};

// ---- work tickets ---------------------------------------------------------------
// Walkers take splitters (sublists) from one global ticket counter.  One
// atomicAdd per warp refill put every walker of the device on the same L2
// address: ncu on config D counted 1.82M same-address atomics in the 1.70 ms
// level-0 walk (long_scoreboard 93%, DRAM 14%, L2 30%) -- the walk waited on
// the counter, not on memory.  A warp now reserves kLrTicketBatch tickets at
// a time and hands them to its idle lanes over several iterations.  Tickets
// are drawn in increasing order, so a lane that draws one past the end has
// left no valid ticket behind.
constexpr u32 kLrTicketBatch = 64;
struct WarpTickets {
  u32 next = 0, end = 0;  // warp-uniform: unused tickets [next, end)
  // the ticket of each lane in `need` (lanemask_lt-ranked), refilling the
  // warp batch with one atomicAdd when it runs short
  __device__ __forceinline__ u32 take(u32 need, u32* counter, int lane, u32 lt) {
    const u32 cnt = __popc(need);
    const u32 rank = __popc(need & lt);
    const u32 avail = end - next;
    u32 base2 = 0;
    if (avail < cnt) {
      const u32 want = ((cnt - avail + kLrTicketBatch - 1) / kLrTicketBatch) * kLrTicketBatch;
      const int leader = __ffs(need) - 1;
      if (lane == leader) base2 = atomicAdd(counter, want);
      base2 = __shfl_sync(0xffffffffu, base2, leader);  // every lane runs take()
      const u32 idx = rank < avail ? next + rank : base2 + (rank - avail);
      next = base2 + (cnt - avail);
      end = base2 + want;
      return idx;
    }
    const u32 idx = next + rank;
    next += cnt;
    return idx;
  }
};

// ---- level-0 walk -----------------------------------------------------------
// Successors (u32) and records (u64, local << 32 | sublist) live in separate
// arrays.  Measured on B200 (tools/walk_micro.cu, profiles/r1_walk_micro.md):
// keeping both in one 8-B slot (load then store the same address) runs at
// 3.45 G elements/s versus 19.7 G/s for separate arrays -- the same-address
// store stalls the dependent pointer chase -- so the extra random store is
// the cheaper option.
// kLrWalkers independent walkers per lane issue their successor loads back
// to back.  Measured on B200 (round 1 trace): 2 walkers per lane were slower
// than 1 (walk0 1.78 vs 1.64 ms on 32M elements, 2.27 vs 1.91 ms on 64M) --
// the memory system is already saturated by the resident warps -- so 1.
constexpr int kLrWalkers = 1;

// kNarrow (lists without down weights): 4-B records (local << sid_bits | sid)
// and sublists capped at cap_step elements (walk micro: -12% vs 8-B records).
// kTwin: the successor of e is succ[e ^ 1] (an Euler tour whose closed
// rotation lists serve as the successor array, bridges.cu k_tree_close).
// kHint (ETTG_LR_HINT A/B): bit 0 = record stores evict-first (.cs), bit 1 =
// successor loads with an L2 evict_last policy.
template <class Down, class H, bool kNarrow, bool kTwin = false, int kHint = 0>
__global__ void __launch_bounds__(256)
    k_lr_walk0(const u32* __restrict__ succ, u64* __restrict__ rec, u32 k, H head_src, u32 seed,
               u32 mask, const u32* __restrict__ spl, u32* counters, u32 sub_cap,
               u32* __restrict__ sub_next, u64* __restrict__ sub_w, Down down, u32 cap_step,
               u32 sid_bits) {
  u32* rec32 = reinterpret_cast<u32*>(rec);
  const int lane = threadIdx.x & 31;
  const u32 head = head_src.get();
  const u32 lt = lanemask_lt();
  // A malformed list (shared successors, found by k_pred_check) is not walked.
  const u32 nspl = counters[LrCounters::kErr] ? 0u : min(counters[LrCounters::kNspl], sub_cap);
  bool active[kLrWalkers], retired = false;
  WarpTickets tickets;
  u32 sid[kLrWalkers], cur[kLrWalkers], acc[kLrWalkers], steps[kLrWalkers];
#pragma unroll
  for (int w = 0; w < kLrWalkers; ++w) {
    active[w] = false;
    sid[w] = cur[w] = acc[w] = steps[w] = 0;
  }
  while (true) {
#pragma unroll
    for (int w = 0; w < kLrWalkers; ++w) {
      const u32 need = __ballot_sync(0xffffffffu, !active[w] && !retired);
      if (need) {
        const u32 idx_all = tickets.take(need, &counters[LrCounters::kTicket0], lane, lt);
        if (!active[w] && !retired) {
          const u32 idx = idx_all;
          if (idx < nspl) {
            sid[w] = idx;
            cur[w] = spl[idx];
            acc[w] = 0;
            steps[w] = 0;
            active[w] = true;
          } else {
            retired = true;
          }
        }
      }
    }
    bool any = false;
#pragma unroll
    for (int w = 0; w < kLrWalkers; ++w) any |= active[w];
    if (!__any_sync(0xffffffffu, any)) break;
    u32 nxt[kLrWalkers];
#pragma unroll
    for (int w = 0; w < kLrWalkers; ++w) {
      nxt[w] = kNone;
      if (active[w]) {
        if (kNarrow) {
          const u32 r = ((acc[w] & 0xFFFFu) << sid_bits) | sid[w];
          if (kHint & 1)
            __stcs(rec32 + cur[w], r);
          else
            rec32[cur[w]] = r;
        } else {
          rec[cur[w]] = (static_cast<u64>(acc[w]) << 32) | sid[w];
        }
        const u32* sp = succ + (kTwin ? cur[w] ^ 1u : cur[w]);
        nxt[w] = (kHint & 2) ? ldg_u32_l2(sp, l2_policy_evict_last()) : *sp;
      }
    }
#pragma unroll
    for (int w = 0; w < kLrWalkers; ++w) {
      if (!active[w]) continue;
      acc[w] += 1u + (down(cur[w]) << 16);
      ++steps[w];
      const u32 nx = nxt[w];
      const bool bad = (nx != kNone && nx >= k) || steps[w] > k;
      const bool stop = bad || nx == kNone || lr_is_splitter(nx, head, seed, mask);
      if (stop || (acc[w] & 0xFFFFu) == (kNarrow ? cap_step : kLrCapStep)) {
        sub_next[sid[w]] = bad ? kNone : nx;
        sub_w[sid[w]] = (static_cast<u64>(acc[w] >> 16) << 32) | (acc[w] & 0xFFFFu);
        if (bad) atomicOr(&counters[LrCounters::kErr], kErrStructure);
        if (stop) {
          active[w] = false;
        } else {
          const u32 ns = atomicAdd(&counters[LrCounters::kSubTotal0], 1u);
          if (ns >= sub_cap) {
            atomicOr(&counters[LrCounters::kErr], kErrCapacity);
            active[w] = false;
          } else {
            sid[w] = ns;
            acc[w] = 0;
            cur[w] = nx;
          }
        }
      } else {
        cur[w] = nx;
      }
    }
  }
}

__global__ void k_twin_succ(const u32* __restrict__ twin_succ, u32 k, u32* __restrict__ succ) {
  for (u32 e = blockIdx.x * blockDim.x + threadIdx.x; e < k; e += gridDim.x * blockDim.x)
    succ[e] = twin_succ[e ^ 1u];
}

// Every element has at most one predecessor and the head has none (checked
// before walking when the successor array comes from a caller).
template <class H>
__global__ void k_pred_check(const u32* __restrict__ succ, u32 k, H head_src, u32* pred,
                             u32* err) {
  const u32 head = head_src.get();
  for (u32 e = blockIdx.x * blockDim.x + threadIdx.x; e < k; e += gridDim.x * blockDim.x) {
    const u32 s = succ[e];
    if (s == kNone) continue;
    if (s >= k || s == head || atomicAdd(&pred[s], 1u) != 0u) atomicOr(err, kErrStructure);
  }
}

// ---- level >= 1 walk (explicit u64 weights) ---------------------------------
__global__ void __launch_bounds__(256)
    k_lr_walk(const u32* __restrict__ succ, const u64* __restrict__ w,
              const u32* d_S, const u32* d_head, u32 seed, u32 mask,
              const u32* __restrict__ spl, const u32* d_nspl, u32* ticket,
              u32* __restrict__ rec_sid, u64* __restrict__ rec_loc,
              u32* __restrict__ sub_next, u64* __restrict__ sub_w, u32* err) {
  const int lane = threadIdx.x & 31;
  const u32 lt = lanemask_lt();
  const u32 S = *d_S, head = *d_head, nspl = *d_nspl;
  bool active = false, retired = false;
  WarpTickets tickets;
  u32 sid = 0, cur = 0, steps = 0;
  u64 acc = 0;
  while (true) {
    const u32 need = __ballot_sync(0xffffffffu, !active && !retired);
    if (need) {
      const u32 idx_all = tickets.take(need, ticket, lane, lt);
      if (!active && !retired) {
        const u32 idx = idx_all;
        if (idx < nspl) {
          sid = idx;
          cur = spl[idx];
          acc = 0;
          active = true;
        } else {
          retired = true;
        }
      }
    }
    if (!__any_sync(0xffffffffu, active)) break;
    if (active) {
      rec_sid[cur] = sid;
      rec_loc[cur] = acc;
      acc += w[cur];
      const u32 nxt = succ[cur];
      ++steps;
      const bool bad = (nxt != kNone && nxt >= S) || steps > S;
      if (bad || nxt == kNone || lr_is_splitter(nxt, head, seed, mask)) {
        sub_next[sid] = bad ? kNone : nxt;
        sub_w[sid] = acc;
        if (bad) atomicOr(err, kErrStructure);
        active = false;
      } else {
        cur = nxt;
      }
    }
  }
}

// Clamp a device count to a capacity (flags the overflow) so every later
// kernel indexes within its arrays even for malformed input.
__global__ void k_lr_clamp(u32* count, u32 cap, u32* err) {
  if (*count > cap) {
    *count = cap;
    atomicOr(err, kErrCapacity);
  }
}

// Next-level list: succ'[sid] = sublist of the element after sublist sid.
// Level-0 records are packed (local<<32 | sid).
template <class H>
__global__ void k_lr_next_level0(const u64* __restrict__ rec, const u32* __restrict__ sub_next,
                                 const u64* __restrict__ sub_w, const u32* d_S, H head_src,
                                 u32* __restrict__ succ2, u64* __restrict__ w2, u32* d_head2,
                                 u32 sid_bits) {
  const u32 S = *d_S;
  const u32 head = head_src.get();
  const u32* rec32 = reinterpret_cast<const u32*>(rec);
  const u32 smask = sid_bits ? (1u << sid_bits) - 1u : 0u;
  auto sid_of = [&](u32 e) {
    return sid_bits ? (rec32[e] & smask) : static_cast<u32>(rec[e]);
  };
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
    const u32 ne = sub_next[i];
    succ2[i] = ne == kNone ? kNone : sid_of(ne);
    w2[i] = sub_w[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *d_head2 = sid_of(head);
}

__global__ void k_lr_next_level(const u32* __restrict__ rec_sid, const u32* __restrict__ sub_next,
                                const u64* __restrict__ sub_w, const u32* d_S, const u32* d_head,
                                u32* __restrict__ succ2, u64* __restrict__ w2, u32* d_head2) {
  const u32 S = *d_S;
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
    const u32 ne = sub_next[i];
    succ2[i] = ne == kNone ? kNone : rec_sid[ne];
    w2[i] = sub_w[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *d_head2 = rec_sid[*d_head];
}

// prefix_l[e] = prefix_{l+1}[rec_sid[e]] + rec_loc[e]
__global__ void k_lr_expand(const u32* __restrict__ rec_sid, const u64* __restrict__ rec_loc,
                            const u64* __restrict__ pnext, const u32* d_S, const u32* d_Snext,
                            u64* __restrict__ prefix) {
  const u32 S = *d_S, Sn = *d_Snext;
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < S; i += gridDim.x * blockDim.x) {
    u32 sid = rec_sid[i];
    if (sid >= Sn) sid = 0;  // unreached element of a malformed list (already flagged)
    prefix[i] = pnext[sid] + rec_loc[i];
  }
}

// Final level: Wyllie pointer jumping in shared memory, one CTA.
// total_rank_expect: the head chain must have this many level-0 elements.
__device__ __forceinline__ void lr_final_smem(const u32* __restrict__ succ,
                                              const u64* __restrict__ w, u32 S, const u32* d_head,
                                              u64* __restrict__ prefix, u32 total_rank_expect,
                                              u32* err) {
  extern __shared__ u64 s_dyn[];  // kLrFinalMax u64 values, then u32 links
  u64* s_val = s_dyn;
  u32* s_nxt = reinterpret_cast<u32*>(s_dyn + kLrFinalMax);
  constexpr int kPer = kLrFinalMax / kLrFinalThreads;
  for (u32 i = threadIdx.x; i < S; i += kLrFinalThreads) {
    u32 nx = succ[i];
    if (nx != kNone && nx >= S) {
      atomicOr(err, kErrStructure);
      nx = kNone;
    }
    s_nxt[i] = nx;
    s_val[i] = w[i];
  }
  __syncthreads();
  for (int round = 0; round < 15; ++round) {
    u32 nn[kPer];
    u64 nv[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const u32 i = threadIdx.x + j * kLrFinalThreads;
      nn[j] = kNone;
      nv[j] = 0;
      if (i < S) {
        const u32 nx = s_nxt[i];
        nv[j] = s_val[i];
        if (nx != kNone) {
          nv[j] += s_val[nx];
          nn[j] = s_nxt[nx];
        }
      }
    }
    __syncthreads();
    int live = 0;
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const u32 i = threadIdx.x + j * kLrFinalThreads;
      if (i < S) {
        s_nxt[i] = nn[j];
        s_val[i] = nv[j];
        live |= nn[j] != kNone;
      }
    }
    if (!__syncthreads_or(live)) break;
  }
  // s_val[i] = inclusive suffix sum; prefix = total - suffix + own weight.
  const u32 head = *d_head;
  const u64 total = s_val[head];
  for (u32 i = threadIdx.x; i < S; i += kLrFinalThreads) {
    if (s_nxt[i] != kNone) atomicOr(err, kErrStructure);  // cycle
    prefix[i] = total - s_val[i];
  }
  if (threadIdx.x == 0 && static_cast<u32>(total) != total_rank_expect)
    atomicOr(err, kErrStructure);  // head chain does not cover every element
}

__global__ void __launch_bounds__(kLrFinalThreads)
    k_lr_final(const u32* __restrict__ succ, const u64* __restrict__ w, const u32* d_S,
               const u32* d_head, u64* __restrict__ prefix, u32 total_rank_expect,
               u32* err) {
  const u32 S = *d_S;
  if (S > kLrFinalMax) {
    if (threadIdx.x == 0) atomicOr(err, kErrCapacity);
    return;
  }
  lr_final_smem(succ, w, S, d_head, prefix, total_rank_expect, err);
}

// Final level for up to kLrWyllieMax elements: Wyllie pointer jumping over
// global memory in one cooperative launch, ping-ponging (succ, value)
// between two buffers with a grid barrier per round.  A small level (<=
// kLrFinalMax, known only on the device) takes the one-CTA smem path
// instead.  Replaces further walk levels whose cost on small lists is the
// longest sublist's dependent-load chain (about L ln(S/L) steps), not
// bandwidth: ceil(log2 S) fully parallel rounds are shorter.
__global__ void __launch_bounds__(kLrFinalThreads)
    k_lr_wyllie(const u32* __restrict__ succ_in, const u64* __restrict__ w_in, u32* succ_a,
                u64* val_a, u32* succ_b, u64* val_b, const u32* d_S, const u32* d_head,
                u64* __restrict__ prefix, u32 total_rank_expect, u32* err, int hops) {
  const u32 S = *d_S;
  if (S <= kLrFinalMax) {
    if (blockIdx.x == 0) lr_final_smem(succ_in, w_in, S, d_head, prefix, total_rank_expect, err);
    return;  // uniform across the grid: no barrier is reached
  }
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const u32 stride = gridDim.x * blockDim.x;
  const u32 t0 = blockIdx.x * blockDim.x + threadIdx.x;
  // `hops` links per round: a pointer's span multiplies by `hops` per
  // barrier (plain Wyllie: 2), trading dependent loads for grid barriers.
  int rounds = 0;
  for (u64 span = 1; span < S; span *= static_cast<u64>(hops)) ++rounds;
  const u32* src_s = succ_in;
  const u64* src_v = w_in;
  u32* dst_s = succ_a;
  u64* dst_v = val_a;
  for (int r = 0; r < rounds; ++r) {
    for (u32 i = t0; i < S; i += stride) {
      u32 nx = src_s[i];
      u64 v = src_v[i];
      if (r == 0 && nx != kNone && nx >= S) {
        atomicOr(err, kErrStructure);
        nx = kNone;
      }
      for (int h = 1; h < hops && nx != kNone; ++h) {
        v += src_v[nx];
        u32 nn = src_s[nx];
        if (r == 0 && nn != kNone && nn >= S) nn = kNone;  // flagged by element nx
        nx = nn;
      }
      dst_s[i] = nx;
      dst_v[i] = v;
    }
    grid.sync();
    src_s = dst_s;
    src_v = dst_v;
    dst_s = (dst_s == succ_a) ? succ_b : succ_a;
    dst_v = (dst_v == val_a) ? val_b : val_a;
  }
  const u64 total = src_v[*d_head];
  for (u32 i = t0; i < S; i += stride) {
    if (src_s[i] != kNone) atomicOr(err, kErrStructure);  // cycle
    prefix[i] = total - src_v[i];
  }
  if (t0 == 0 && static_cast<u32>(total) != total_rank_expect) atomicOr(err, kErrStructure);
}

// ---- orchestration ---------------------------------------------------------
struct LrLevel {
  u32 cap = 0;            // capacity of this level's element arrays
  u32* succ = nullptr;    // level >= 1
  u64* w = nullptr;       // level >= 1
  u32* rec_sid = nullptr; // level >= 1
  u64* rec_loc = nullptr; // level >= 1
  u64* prefix = nullptr;  // level >= 1
  u32* spl = nullptr;     // splitters of this level (cap = next level cap)
  u32* sub_next = nullptr;
  u64* sub_w = nullptr;
  u64* scan_status = nullptr;
  u32* succ2 = nullptr;   // final level > kLrFinalMax: Wyllie ping-pong buffers
  u64* w2 = nullptr;
  u32* succ3 = nullptr;
  u64* w3 = nullptr;
};

struct ListRankWs {
  static constexpr int kMaxLevels = 8;
  u32 k = 0;
  int levels = 0;  // number of walk levels (>= 1); final Wyllie after the last
  LrLevel lv[kMaxLevels + 1];
  u32* succ0 = nullptr;  // level-0 successors (filled by the caller), k entries
  u64* rec0 = nullptr;   // level-0 records, k entries
  u32* counters = nullptr;
  u64* prefix1 = nullptr;  // == lv[1].prefix: exclusive prefix per level-0 sublist

  static u32 next_cap(u64 S, u32 L) {
    double mu = static_cast<double>(S) / L;
    u64 c = static_cast<u64>(mu + 8.0 * __builtin_sqrt(mu + 1.0) + 1024.0);
    return static_cast<u32>(c > S + 1 ? S + 1 : c);
  }

  u32 L0 = kLrL0;  // level-0 mean sublist length (power of two); ETTG_LR_L0 overrides
  u32 Ld = kLrL;   // deeper levels; ETTG_LR_L overrides
  double wyllie_max = kLrWyllieMax;  // ETTG_LR_WYLLIE overrides (0: smem final only)
  // Narrow level-0 records (weight-free lists, see k_lr_walk0): sid_bits > 0.
  u32 sid_bits = 0, cap_step = kLrCapStep;
  // narrow_ok: the caller's lists carry no down weights (NoDown)
  // l0 / ld: default level means for this caller (powers of two)
  void carve(Carver& c, u32 k_, bool narrow_ok = false, u32 l0 = kLrL0, u32 ld = kLrL) {
    k = k_;
    L0 = l0;
    Ld = ld;
    if (const char* e = std::getenv("ETTG_LR_L0")) {
      const u32 v = static_cast<u32>(std::atoi(e));
      if (v >= 2 && v <= 1024 && (v & (v - 1)) == 0) L0 = v;
    }
    if (const char* e = std::getenv("ETTG_LR_L")) {
      const u32 v = static_cast<u32>(std::atoi(e));
      if (v >= 2 && v <= 1024 && (v & (v - 1)) == 0) Ld = v;
    }
    if (const char* e = std::getenv("ETTG_LR_WYLLIE")) wyllie_max = std::atof(e);
    succ0 = c.take<u32>(k);
    rec0 = c.take<u64>(k);
    counters = c.take<u32>(64);
    // level 0 caps
    u32 cap1 = next_cap(k, L0) + k / kLrCapStep + 2;
    sid_bits = 0;
    cap_step = kLrCapStep;
    bool narrow = narrow_ok;
    if (const char* e = std::getenv("ETTG_LR_NARROW")) narrow &= std::atoi(e) != 0;
    if (narrow) {  // >= 8 local bits: cap splits stay rare (mean sublist 16)
      const u32 c8 = next_cap(k, L0) + k / 255 + 2;
      u32 b = 1;
      while ((u64(1) << b) < c8) ++b;
      if (b <= 24) {
        sid_bits = b;
        cap_step = (1u << (32 - b)) - 1u;
        if (cap_step > kLrCapStep) cap_step = kLrCapStep;
        cap1 = next_cap(k, L0) + k / cap_step + 2;
      }
    }
    lv[0].cap = k;
    lv[0].spl = c.take<u32>(cap1);
    lv[0].sub_next = c.take<u32>(cap1);
    lv[0].sub_w = c.take<u64>(cap1);
    lv[0].scan_status = c.take<u64>(scan_ws_words(k));
    int l = 1;
    u32 cap = cap1;
    double expect = static_cast<double>(k) / L0;
    while (true) {
      LrLevel& L = lv[l];
      L.cap = cap;
      L.succ = c.take<u32>(cap);
      L.w = c.take<u64>(cap);
      L.prefix = c.take<u64>(cap);
      if (expect <= 2048.0 || l == kMaxLevels) break;  // final Wyllie level (smem)
      if (expect * 1.25 <= wyllie_max) {                // final Wyllie level (global)
        L.succ2 = c.take<u32>(cap);
        L.w2 = c.take<u64>(cap);
        L.succ3 = c.take<u32>(cap);
        L.w3 = c.take<u64>(cap);
        break;
      }
      L.rec_sid = c.take<u32>(cap);
      L.rec_loc = c.take<u64>(cap);
      u32 capn = next_cap(cap, Ld);
      L.spl = c.take<u32>(capn);
      L.sub_next = c.take<u32>(capn);
      L.sub_w = c.take<u64>(capn);
      L.scan_status = c.take<u64>(scan_ws_words(cap));
      cap = capn;
      expect /= Ld;
      ++l;
    }
    levels = l;  // walk levels 0..l-1, Wyllie on level l
    prefix1 = lv[1].prefix;
  }
};

inline u32 lr_seed(int level) { return 0x65746b5fu ^ (0x9e3779b9u * (level + 1)); }

// Runs the ranking up to the per-sublist prefixes of level 0 (ws.prefix1).
// The caller has filled ws.succ0 (u32 successors, kNone = tail); on return
// ws.rec0 holds the level-0 records.  Callers finish with their own fused
// per-element kernel (Lr0View).  `pred` (k words of scratch) enables the
// injectivity check for caller-supplied lists.  No host synchronisation;
// errors accumulate in counters[kErr].
// twin_succ != nullptr: the level-0 successor of e is twin_succ[e ^ 1]
// instead of ws.succ0[e] (narrow, weight-free lists only).
template <class Down, class H>
void list_rank_core_h(u32 k, H head, Down down, ListRankWs& ws, cudaStream_t st, int sms,
                      u32* pred = nullptr, const u32* twin_succ = nullptr) {
  Trace tr("list_rank", st);
  CK(cudaMemsetAsync(ws.counters, 0, 64 * sizeof(u32), st));
  u32* cnt = ws.counters;
  if (pred) {
    CK(cudaMemsetAsync(pred, 0, static_cast<u64>(k) * 4, st));
    k_pred_check<H><<<blocks_for(k, 256), 256, 0, st>>>(ws.succ0, k, head, pred,
                                                     cnt + LrCounters::kErr);
    CK_LAUNCH();
  }
  const u32 mask0 = ws.L0 - 1;
  const u32 seed0 = lr_seed(0);
  const u32 cap1 = ws.lv[1].cap;
  // level 0 splitters -> counters[kNspl]; sublists beyond come from cap splits
  spl_compact(SplIn<H>{head, seed0, mask0}, k, ws.lv[0].spl, cap1, cnt + LrCounters::kNspl,
              cnt + LrCounters::kErr, st);
  CK(cudaMemcpyAsync(cnt + LrCounters::kSubTotal0, cnt + LrCounters::kNspl, sizeof(u32),
                     cudaMemcpyDeviceToDevice, st));
  tr.mark("splitters0");
  const unsigned walk_blocks = sms * 8;  // 2048 threads / SM resident
  if (twin_succ && !ws.sid_bits) {  // wide records (huge lists): materialise succ0
    k_twin_succ<<<blocks_for(k, 256), 256, 0, st>>>(twin_succ, k, ws.succ0);
    CK_LAUNCH();
    twin_succ = nullptr;
  }
  if (twin_succ) {
    static const int hint = [] {
      const char* e = std::getenv("ETTG_LR_HINT");
      return e ? std::atoi(e) & 3 : 0;
    }();
    auto kern = hint == 1   ? k_lr_walk0<Down, H, true, true, 1>
                : hint == 2 ? k_lr_walk0<Down, H, true, true, 2>
                : hint == 3 ? k_lr_walk0<Down, H, true, true, 3>
                            : k_lr_walk0<Down, H, true, true, 0>;
    kern<<<walk_blocks, 256, 0, st>>>(
        twin_succ, ws.rec0, k, head, seed0, mask0, ws.lv[0].spl, cnt, cap1, ws.lv[0].sub_next,
        ws.lv[0].sub_w, down, ws.cap_step, ws.sid_bits);
  } else if (ws.sid_bits)
    k_lr_walk0<Down, H, true><<<walk_blocks, 256, 0, st>>>(
        ws.succ0, ws.rec0, k, head, seed0, mask0, ws.lv[0].spl, cnt, cap1, ws.lv[0].sub_next,
        ws.lv[0].sub_w, down, ws.cap_step, ws.sid_bits);
  else
    k_lr_walk0<Down, H, false><<<walk_blocks, 256, 0, st>>>(
        ws.succ0, ws.rec0, k, head, seed0, mask0, ws.lv[0].spl, cnt, cap1, ws.lv[0].sub_next,
        ws.lv[0].sub_w, down, ws.cap_step, 0u);
  CK_LAUNCH();
  tr.mark("walk0");
  // level-1 list
  u32* S1 = cnt + LrCounters::kSubTotal0;
  k_lr_clamp<<<1, 1, 0, st>>>(S1, cap1, cnt + LrCounters::kErr);
  u32* head1 = cnt + LrCounters::kLevelBase + 4 * 1 + 2;
  k_lr_next_level0<H><<<blocks_for(cap1, 256), 256, 0, st>>>(
      ws.rec0, ws.lv[0].sub_next, ws.lv[0].sub_w, S1, head, ws.lv[1].succ, ws.lv[1].w, head1,
      ws.sid_bits);
  CK_LAUNCH();
  // deeper levels
  const u32* S_l = S1;
  for (int l = 1; l < ws.levels; ++l) {
    LrLevel& L = ws.lv[l];
    LrLevel& N = ws.lv[l + 1];
    u32* tick = cnt + LrCounters::kLevelBase + 4 * l + 0;
    u32* nspl = cnt + LrCounters::kLevelBase + 4 * l + 1;
    u32* hd = cnt + LrCounters::kLevelBase + 4 * l + 2;
    u32* hd_next = cnt + LrCounters::kLevelBase + 4 * (l + 1) + 2;
    const u32 seed = lr_seed(l), mask = ws.Ld - 1;
    spl_compact(SplInDev{hd, S_l, seed, mask}, L.cap, L.spl, N.cap, nspl,
                cnt + LrCounters::kErr, st);
    k_lr_clamp<<<1, 1, 0, st>>>(nspl, N.cap, cnt + LrCounters::kErr);
    k_lr_walk<<<walk_blocks, 256, 0, st>>>(L.succ, L.w, S_l, hd, seed, mask, L.spl, nspl, tick,
                                          L.rec_sid, L.rec_loc, L.sub_next, L.sub_w,
                                          cnt + LrCounters::kErr);
    CK_LAUNCH();
    k_lr_next_level<<<blocks_for(N.cap, 256), 256, 0, st>>>(L.rec_sid, L.sub_next, L.sub_w, nspl,
                                                            hd, N.succ, N.w, hd_next);
    CK_LAUNCH();
    S_l = nspl;
    tr.mark("level");
  }
  // final level
  {
    const int l = ws.levels;
    LrLevel& F = ws.lv[l];
    const u32* hd = cnt + LrCounters::kLevelBase + 4 * l + 2;
    if (!F.succ2) {
      CK(cudaFuncSetAttribute(k_lr_final, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kLrFinalSmem));
      k_lr_final<<<1, kLrFinalThreads, kLrFinalSmem, st>>>(F.succ, F.w, S_l, hd, F.prefix, k,
                                                           cnt + LrCounters::kErr);
      CK_LAUNCH();
    } else {
      // S_l is clamped to F.cap; one grid barrier per round
      CK(cudaFuncSetAttribute(k_lr_wyllie, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              kLrFinalSmem));
      int per_sm = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lr_wyllie, kLrFinalThreads,
                                                       kLrFinalSmem));
      int blocks = sms, hops = 3;
      if (const char* e = std::getenv("ETTG_LR_WBLOCKS")) blocks = std::atoi(e);
      if (const char* e = std::getenv("ETTG_LR_WHOPS")) hops = std::max(2, std::atoi(e));
      blocks = std::max(1, std::min(blocks, std::max(1, per_sm) * sms));
      const unsigned grid = static_cast<unsigned>(blocks);
      const u32* fs = F.succ;
      const u64* fw = F.w;
      u32* ek = cnt + LrCounters::kErr;
      u32 expect = k;
      void* args[] = {&fs, &fw, &F.succ2, &F.w2, &F.succ3, &F.w3, &S_l, &hd, &F.prefix,
                      &expect, &ek, &hops};
      CK(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_lr_wyllie), grid,
                                     kLrFinalThreads, args, kLrFinalSmem, st));
    }
    tr.mark("final");
  }
  // expand back down to level 1
  for (int l = ws.levels - 1; l >= 1; --l) {
    LrLevel& L = ws.lv[l];
    const u32* S = (l == 1) ? (cnt + LrCounters::kSubTotal0)
                            : (cnt + LrCounters::kLevelBase + 4 * (l - 1) + 1);
    const u32* Sn = cnt + LrCounters::kLevelBase + 4 * l + 1;
    k_lr_expand<<<blocks_for(L.cap, 256), 256, 0, st>>>(L.rec_sid, L.rec_loc, ws.lv[l + 1].prefix,
                                                        S, Sn, L.prefix);
    CK_LAUNCH();
  }
  tr.mark("expand");
}

template <class Down>
void list_rank_core(u32 k, u32 head, Down down, ListRankWs& ws, cudaStream_t st, int sms,
                    u32* pred = nullptr) {
  list_rank_core_h(k, HostHead{head}, down, ws, st, sms, pred);
}

// Level-0 element prefix: (rank, down-weight sum) of everything before e.
// Records of elements no walker reached are stale; the sublist id is
// clamped so a malformed input can never index out of bounds (the ranking
// has already flagged kErrStructure in that case).
struct Lr0View {
  const u64* rec0;
  const u64* prefix1;
  const u32* d_S1;  // number of level-0 sublists (device)
  u32 sid_bits;     // > 0: narrow 4-B records (no down weights)
  __device__ __forceinline__ void get(u32 e, u32 S1, u32& rank, u32& dsum) const {
    u32 sid, loc;
    if (sid_bits) {
      const u32 r = reinterpret_cast<const u32*>(rec0)[e];
      sid = r & ((1u << sid_bits) - 1u);
      loc = r >> sid_bits;
    } else {
      const u64 r = rec0[e];
      sid = static_cast<u32>(r);
      loc = static_cast<u32>(r >> 32);
    }
    if (sid >= S1) sid = 0;
    const u64 p = prefix1[sid];
    rank = static_cast<u32>(p) + (loc & 0xFFFFu);
    dsum = static_cast<u32>(p >> 32) + (loc >> 16);
  }
};

inline Lr0View lr0_view(const ListRankWs& ws) {
  return Lr0View{ws.rec0, ws.prefix1, ws.counters + LrCounters::kSubTotal0, ws.sid_bits};
}

__global__ void k_lr_rank_out(Lr0View v, u32 k, u32* __restrict__ rank) {
  const u32 S1 = *v.d_S1;
  for (u32 e = blockIdx.x * blockDim.x + threadIdx.x; e < k; e += gridDim.x * blockDim.x) {
    u32 r, d;
    v.get(e, S1, r, d);
    rank[e] = r;
  }
}

}  // namespace
}  // namespace ettg
