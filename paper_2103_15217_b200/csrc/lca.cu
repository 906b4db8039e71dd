// LCA on B200: Euler-tour index build + batched inlabel / RMQ query kernels.
//
// Reference path (all CPU, OpenMP):
//   inlabel_build            core/src/lca.cpp:20-82
//     validate_tree          core/src/graph.cpp:175-206   (sequential chain walks)
//     tree_edges             core/src/graph.cpp:208-217
//     build_half_edges       core/src/euler.cpp:38-90     (2 sequential counting passes)
//     linearize / list_rank  core/src/euler.cpp:92-117, primitives.cpp:26-115
//     node_stats             core/src/euler.cpp:119-155   (2 scans)
//     inlabel / head / ascendant fix-point  core/src/lca.cpp:35-80
//   inlabel_lca              core/src/lca.cpp:84-109
//   rmq_lca_build / rmq_lca  core/src/lca.cpp:128-157 (segment tree, O(log n))
//
// Device pipeline (u32 ids, n < 2^31):
//   k_tree_validate   parent -> (key=parent, val=child) pairs, root/range flags
//   sort_pairs        stable radix sort => children of each node in ascending
//                     id, i.e. exactly the reference's sorted half-edge order
//   k_child_ranges    [start,end) of each node's child slice
//   k_node_succ       succ(down(y)); j(y) = #children < parent(y)
//   k_slot_succ       succ(up(c)) by the DCEL rotation rule
//   list_rank_core    2n-element tour list (down(root) ... up(root)), weight
//                     "is down", giving rank and #downs before each half-edge
//   k_tree_stats      preorder / level / size / inlabel / first position
//                     (+ RMQ tour keys) in one pass per node
//   k_head            head, label record {parent(head), level}, up-label
//   k_asc_level       ascendant per label, one pass per trailing-zero level
//   k_pack            16-B node record {inlabel, ascendant, level, 0}
//
// Half-edge ids: down(v) = 2v (parent -> v), up(v) = 2v+1 (v -> parent); the
// root's pair is the virtual start/end of the tour, so the tour list has
// exactly 2n elements and rank r(down(v)) equals the reference's tour step of
// v's first occurrence (rmq tour_nodes, core/src/lca.cpp:135-146).
#include <omp.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>
#include <cstring>
#include <memory>
#include <vector>

#include "api_internal.cuh"
#include "common.cuh"
#include "listrank.cuh"
#include "scan.cuh"
#include "sparse.cuh"
#include "sort.cuh"
#include "trace.cuh"

namespace ettg {

// validation flags (bit set)
constexpr u32 kVRootParent = 1u;  // parent[root] != none
constexpr u32 kVRange = 2u;       // parent id out of range
constexpr u32 kVRoots = 4u;       // more than one root

template <class P>
__device__ __forceinline__ bool parent_is_none(P p);
template <>
__device__ __forceinline__ bool parent_is_none<int64_t>(int64_t p) { return p == -1; }
template <>
__device__ __forceinline__ bool parent_is_none<u32>(u32 p) { return p == kNone; }

template <class P>
__global__ void k_tree_validate(const P* __restrict__ parent, u32 n, u32 root,
                                u32* __restrict__ par, u32* __restrict__ keys,
                                u32* __restrict__ vals, u32* flags) {
  u32 f = 0;
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const P p = parent[v];
    u32 pu;
    if (parent_is_none<P>(p)) {
      pu = kNone;
      if (v != root) f |= kVRoots;
    } else if (static_cast<u64>(static_cast<int64_t>(p)) >= n) {  // negative wraps high
      pu = kNone;
      f |= kVRange;
      if (v == root) f |= kVRootParent;
    } else {
      pu = static_cast<u32>(p);
      if (v == root) f |= kVRootParent;
    }
    par[v] = pu;
    if (v != root) {
      const u32 idx = v < root ? v : v - 1;
      keys[idx] = pu == kNone ? 0u : pu;  // keep the sort well-formed on bad input
      vals[idx] = v;
    }
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(flags, f);
}

// crange[y] = [first slot, end slot) of y's children in the sorted arrays.
__global__ void k_child_ranges(const u32* __restrict__ pkey, u32 m, uint2* __restrict__ crange) {
  for (u32 s = blockIdx.x * blockDim.x + threadIdx.x; s < m; s += gridDim.x * blockDim.x) {
    const u32 y = pkey[s];
    if (s == 0 || pkey[s - 1] != y) crange[y].x = s;
    if (s + 1 == m || pkey[s + 1] != y) crange[y].y = s + 1;
  }
}

__global__ void k_node_succ(const uint2* __restrict__ crange, const u32* __restrict__ child,
                            const u32* __restrict__ par, u32 n, u32 root,
                            u32* __restrict__ jj, u32* __restrict__ succ) {
  for (u32 y = blockIdx.x * blockDim.x + threadIdx.x; y < n; y += gridDim.x * blockDim.x) {
    const uint2 r = crange[y];
    const u32 deg = r.y - r.x;
    u32 j = 0;
    if (y == root) {
      succ[2 * y + 1] = kNone;  // up(root) is the tail
    } else if (deg > 0) {
      // lower_bound of parent(y) among y's sorted children: the rotation at y
      // starts just after the entering half-edge (euler.cpp:85-88).
      const u32 p = par[y];
      u32 lo = 0, hi = deg;
      while (lo < hi) {
        const u32 mid = (lo + hi) >> 1;
        if (child[r.x + mid] < p) lo = mid + 1;
        else hi = mid;
      }
      j = lo == deg ? 0u : lo;
    }
    jj[y] = j;
    succ[2 * y] = deg > 0 ? 2 * child[r.x + j] : 2 * y + 1;
  }
}

__global__ void k_slot_succ(const uint2* __restrict__ crange, const u32* __restrict__ child,
                            const u32* __restrict__ pkey, const u32* __restrict__ jj, u32 m,
                            u32 root, u32* __restrict__ succ) {
  for (u32 s = blockIdx.x * blockDim.x + threadIdx.x; s < m; s += gridDim.x * blockDim.x) {
    const u32 c = child[s];
    const u32 y = pkey[s];
    const uint2 r = crange[y];
    const u32 deg = r.y - r.x;
    const u32 i = s - r.x;
    u32 nxt;
    if (y == root) {
      nxt = (i + 1 == deg) ? 2 * y + 1 : 2 * child[s + 1];
    } else {
      const u32 i2 = (i + 1 == deg) ? 0u : i + 1;
      nxt = (i2 == jj[y]) ? 2 * y + 1 : 2 * child[r.x + i2];
    }
    succ[2 * c + 1] = nxt;
  }
}

// preorder (1-based), level, size, inlabel, first tour step per node
// (node_stats core/src/euler.cpp:144-153 + inlabel core/src/lca.cpp:35-44).
__global__ void k_tree_stats(Lr0View lr, u32 n, const u32* __restrict__ par,
                             u32* __restrict__ pre, u32* __restrict__ size,
                             u32* __restrict__ level, u32* __restrict__ inlabel,
                             u32* __restrict__ first, u64* __restrict__ tour_key) {
  const u32 S1 = *lr.d_S1;
  const u32 steps = 2 * n - 1;
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    u32 rd, dd, ru, du;
    lr.get(2 * v, S1, rd, dd);
    lr.get(2 * v + 1, S1, ru, du);
    const u32 p = dd + 1;
    const u32 lev = 2 * dd - rd;
    const u32 sz = (ru - rd + 1) >> 1;
    const u32 r = p + sz - 1;
    const u32 in = (p == r) ? p : (r & ~((1u << hb32((p - 1) ^ r)) - 1u));
    pre[v] = p;
    size[v] = sz;
    level[v] = lev;
    inlabel[v] = in;
    first[v] = rd;
    if (tour_key) {
      if (rd < steps) tour_key[rd] = (static_cast<u64>(lev) << 32) | v;
      const u32 pv = par[v];
      if (pv != kNone && ru < steps) tour_key[ru] = (static_cast<u64>(lev - 1) << 32) | pv;
    }
  }
}

// head / label record / up-label (core/src/lca.cpp:49-53 and the fix-point
// input of :59-78).  lab[L] = {parent(head(L)), level(parent(head(L)))}.
// One 16-B record {head, parent(head), level of it, up-label} per label,
// scattered by label (one sector per head; the three separate arrays cost
// three), then split into head / lab / up by a streaming pass.  16M random
// tree (10M labels): 1.32 -> 0.71 ms (build 5.44 -> 4.89 ms); a 16M path
// (7 labels) pays the 0.1 ms split pass (build 4.02 -> 4.19 ms).
__global__ void k_head(const u32* __restrict__ inlabel, const u32* __restrict__ par,
                       const u32* __restrict__ level, u32 n, uint4* __restrict__ hrec,
                       u32* __restrict__ nheads) {
  u32 heads = 0;
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const u32 L = inlabel[v];
    if (L == 0 || L > n) continue;  // malformed input, already rejected
    const u32 p = par[v];
    const u32 pl = p == kNone ? 0u : inlabel[p];
    if (p == kNone || pl != L) {
      hrec[L] = make_uint4(v, p, p == kNone ? kNone : level[v] - 1, p == kNone ? 0u : pl);
      ++heads;
    }
  }
  for (int o = 16; o; o >>= 1) heads += __shfl_xor_sync(0xffffffffu, heads, o);
  if ((threadIdx.x & 31) == 0 && heads) atomicAdd(nheads, heads);
}

// Unused labels keep the all-ones record: head = none, lab = {none, none}, up = none.
__global__ void k_head_split(const uint4* __restrict__ hrec, u32 count, u32* __restrict__ head,
                             uint2* __restrict__ lab, u32* __restrict__ up) {
  for (u32 L = blockIdx.x * blockDim.x + threadIdx.x; L < count; L += gridDim.x * blockDim.x) {
    const uint4 r = hrec[L];
    head[L] = r.x;
    lab[L] = make_uint2(r.y, r.z);
    up[L] = r.w;
  }
}

// ascendant(L) = ascendant(up(L)) | 2^tz(L), with up(L) the label of
// parent(head(L)) and tz(up(L)) > tz(L) (core/src/lca.cpp:55-78).  Instead of
// the reference's log-n global fix-point rounds, labels are resolved in
// decreasing tz: labels with tz = t are exactly (2i+1)*2^t, so pass t touches
// n/2^(t+1) labels and every label costs one gather of its (already final)
// up-label.  ~25 small launches, n gathers in total.
__global__ void k_asc_level(const u32* __restrict__ up, u32 n, int t, u32* __restrict__ asc) {
  const u32 count = ((n >> t) + 1) >> 1;  // #odd multiples of 2^t in [1, n]
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    const u32 L = ((2 * i + 1) << t);
    const u32 u = up[L];
    if (u == kNone) continue;  // unused label
    asc[L] = (u == 0u ? 0u : asc[u]) | (1u << t);
  }
}

// Level of head(L): the label record holds level(parent(head(L))).
__device__ __forceinline__ u32 head_level(uint2 labrec) {
  return labrec.x == kNone ? 0u : labrec.y + 1u;
}

__global__ void k_pack(const u32* __restrict__ inlabel, const u32* __restrict__ level,
                       const u32* __restrict__ asc, const uint2* __restrict__ lab, u32 n,
                       uint4* __restrict__ node, uint2* __restrict__ node8,
                       uint2* __restrict__ nodes, u32* __restrict__ maxoff) {
  u32 mo = 0;
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const u32 L = inlabel[v];
    const u32 lev = level[v];
    const bool okL = L >= 1 && L <= n;
    if (node) node[v] = make_uint4(L, okL ? asc[L] : 0u, lev, 0u);
    if (node8) node8[v] = make_uint2(L, lev);
    if (nodes) nodes[v] = make_uint2(L, okL ? asc[L] : 0u);
    if (okL) mo = max(mo, lev - head_level(lab[L]));
  }
  for (int o = 16; o; o >>= 1) mo = max(mo, __shfl_xor_sync(0xffffffffu, mo, o));
  if ((threadIdx.x & 31) == 0) atomicMax(maxoff, mo);
}

// Compact layout (deep trees with few inlabel paths): a 4-B node word
// (label index << off_bits | level - level(head)) and a dense per-label table
// {inlabel, ascendant, level(head), 0}.  Label indices come from an
// exclusive scan over "label L is in use" (head[L] != none).
struct LabelUsedIn {
  const u32* head;
  __device__ __forceinline__ u32 operator()(u64 i) const { return head[i] != kNone ? 1u : 0u; }
};

__global__ void k_pack_compact(const u32* __restrict__ inlabel, const u32* __restrict__ level,
                               const u32* __restrict__ head, const u32* __restrict__ asc,
                               const uint2* __restrict__ lab, const u32* __restrict__ lidx,
                               u32 n, int off_bits, u32* __restrict__ node4,
                               uint4* __restrict__ ltab) {
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const u32 L = inlabel[v];
    const u32 li = lidx[L];
    const u32 hl = head_level(lab[L]);
    node4[v] = (off_bits < 32 ? (li << off_bits) : 0u) | (level[v] - hl);
    if (head[L] == v) ltab[li] = make_uint4(L, asc[L], hl, 0u);
  }
}

// Build-time sample of uniform query pairs (the reference's sample_queries
// distribution) over the split records: counts endpoint lifts and the lifts
// whose target is the endpoint's own label (popc(asc & lowmask) == 1).  On
// shallow-wide trees (stars, caterpillars) nearly every lift is an own-label
// lift -- a random label-record gather that an own-lift field in the node
// record removes; on random trees almost none are.
__global__ void k_lift_sample(const uint2* __restrict__ nodes, u32 n, u32 samples,
                              u32* __restrict__ counts) {
  u32 lifts = 0, own = 0, lev = 0;
  for (u32 s = blockIdx.x * blockDim.x + threadIdx.x; s < samples; s += gridDim.x * blockDim.x) {
    const u32 x = __umulhi(mix32(2 * s + 0x9e37u), n), y = __umulhi(mix32(2 * s + 0x79b9u), n);
    const uint2 A = nodes[x], B = nodes[y];
    if (A.x == B.x) {
      lev += 2;  // equal inlabels: both levels decide
      continue;
    }
    const int hbit = hb32(A.x ^ B.x);
    const u32 common = A.y & B.y & ~((1u << hbit) - 1u);
    const int jb = tz32(common);
    const u32 target = (A.x & ~((2u << jb) - 1u)) | (1u << jb);
    const u32 lowmask = (1u << jb) - 1u;
    if (A.x != target) {
      ++lifts;
      own += __popc(A.y & lowmask) == 1;
    } else {
      ++lev;  // an endpoint on the target path compares by its own level
    }
    if (B.x != target) {
      ++lifts;
      own += __popc(B.y & lowmask) == 1;
    } else {
      ++lev;
    }
  }
  for (int o = 16; o; o >>= 1) {
    lifts += __shfl_xor_sync(0xffffffffu, lifts, o);
    own += __shfl_xor_sync(0xffffffffu, own, o);
    lev += __shfl_xor_sync(0xffffffffu, lev, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&counts[0], lifts);
    atomicAdd(&counts[1], own);
    atomicAdd(&counts[2], lev);
  }
}

// split_own node record {inlabel, ascendant, lab[inlabel]} (16 B): the own-
// label lift target (core/src/lca.cpp:99-103 with k = tz(inlabel)) inline.
__global__ void k_pack_own(const uint2* __restrict__ nodes, const uint2* __restrict__ lab, u32 n,
                           uint4* __restrict__ node) {
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint2 a = nodes[v];
    const uint2 o = (a.x >= 1 && a.x <= n) ? lab[a.x] : make_uint2(kNone, kNone);
    node[v] = make_uint4(a.x, a.y, o.x, o.y);
  }
}

// split6 record: {inlabel, ascendant} as 48 bits at byte 6v (n < 2^24).
__global__ void k_pack6(const uint2* __restrict__ nodes, u32 n, uint32_t* __restrict__ nodes6) {
  uint16_t* h = reinterpret_cast<uint16_t*>(nodes6);
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint2 a = nodes[v];
    const u64 rec = (a.x & 0xFFFFFFu) | (static_cast<u64>(a.y & 0xFFFFFFu) << 24);
    const u32 s = v / kRec6PerSector, k = v % kRec6PerSector;
    const u64 o = 16 * static_cast<u64>(s) + 3 * k;  // u16 index
    h[o] = static_cast<uint16_t>(rec);
    h[o + 1] = static_cast<uint16_t>(rec >> 16);
    h[o + 2] = static_cast<uint16_t>(rec >> 32);
  }
}

// wide9 record: {inlabel, ascendant, level} as 72 bits at bit 72k of sector
// v / 3, k = v % 3 (n < 2^24: every field fits 24 bits).  One thread per sector.
__device__ __forceinline__ void put_bits(u64 (&q)[4], u32 off, u64 val) {
  const u32 i = off / 64, sh = off % 64;
  q[i] |= val << sh;
  if (sh > 40) q[i + 1] |= val >> (64 - sh);  // 24-bit fields
}
__global__ void k_pack9(const uint4* __restrict__ node, u32 n, uint32_t* __restrict__ nodes9) {
  const u32 sectors = (n + kRec9PerSector - 1) / kRec9PerSector;
  for (u32 s = blockIdx.x * blockDim.x + threadIdx.x; s < sectors; s += gridDim.x * blockDim.x) {
    u64 q[4] = {0, 0, 0, 0};
#pragma unroll
    for (u32 k = 0; k < kRec9PerSector; ++k) {
      const u32 v = s * kRec9PerSector + k;
      if (v < n) {
        const uint4 r = node[v];
        put_bits(q, 72 * k, r.x & 0xFFFFFFu);
        put_bits(q, 72 * k + 24, r.y & 0xFFFFFFu);
        put_bits(q, 72 * k + 48, r.z & 0xFFFFFFu);
      }
    }
    uint4* o = reinterpret_cast<uint4*>(nodes9 + 8 * static_cast<u64>(s));
    o[0] = make_uint4(static_cast<u32>(q[0]), static_cast<u32>(q[0] >> 32),
                      static_cast<u32>(q[1]), static_cast<u32>(q[1] >> 32));
    o[1] = make_uint4(static_cast<u32>(q[2]), static_cast<u32>(q[2] >> 32),
                      static_cast<u32>(q[3]), static_cast<u32>(q[3] >> 32));
  }
}

// ---- RMQ over the tour (block-sparse table, 32-step blocks) ---------------
// Keys (level << 32 | node) make the minimum's low word the LCA itself.
__global__ void k_rmq_block(const u64* __restrict__ key, u32 steps, u32 nb,
                            u64* __restrict__ pre_in, u64* __restrict__ suf_in,
                            u64* __restrict__ sp0) {
  const u32 lane = threadIdx.x & 31;
  const u32 warps = (gridDim.x * blockDim.x) >> 5;
  for (u32 b = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; b < nb; b += warps) {
    const u32 t = b * 32 + lane;
    const u64 k = t < steps ? key[t] : ~0ull;
    u64 f = k, g = k;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      u64 a = __shfl_up_sync(0xffffffffu, f, d);
      if (lane >= static_cast<u32>(d)) f = min(f, a);
      u64 c = __shfl_down_sync(0xffffffffu, g, d);
      if (lane + d < 32) g = min(g, c);
    }
    if (t < steps) {
      pre_in[t] = f;
      suf_in[t] = g;
    }
    if (lane == 31) sp0[b] = f;
  }
}

struct MinU64 {
  __device__ __forceinline__ u64 operator()(u64 a, u64 b) const { return min(a, b); }
};

// ---- naive engine: pointer-jumping levels + walk-up queries ----------------
// ancestor_doubling_levels (core/src/primitives.cpp:208-241) and naive_lca
// (core/src/lca.cpp:111-126).  State per node: (ancestor, distance); each
// round doubles the jump (Wyllie), so ceil(log2 depth) rounds; a node whose
// ancestor is not the root after bits(n)+1 rounds lies on a cycle.
__global__ void k_dbl_init(const u32* __restrict__ par, u32 n, u32 root, uint2* __restrict__ st) {
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const u32 p = par[v];
    st[v] = (v == root || p == kNone) ? make_uint2(v == root ? root : v, 0u) : make_uint2(p, 1u);
  }
}

__global__ void k_dbl_round(const uint2* __restrict__ cur, uint2* __restrict__ nxt, u32 n) {
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint2 s = cur[v];
    const uint2 a = cur[s.x];
    nxt[v] = make_uint2(a.x, s.y + a.y);
  }
}

// nrec[v] = {parent, level}; flags bit 0 set if some node never reached the root.
__global__ void k_dbl_finish(const uint2* __restrict__ st, const u32* __restrict__ par, u32 n,
                             u32 root, uint2* __restrict__ nrec, u32* flags) {
  u32 bad = 0;
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const uint2 s = st[v];
    bad |= s.x != root;
    nrec[v] = make_uint2(v == root ? kNone : par[v], s.y);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
}

__global__ void k_pack_naive(const u32* __restrict__ par, const u32* __restrict__ level, u32 n,
                             uint2* __restrict__ nrec) {
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    nrec[v] = make_uint2(par[v], level[v]);
}

// ---- queries ---------------------------------------------------------------
struct PairsU32 {
  const uint2* p;
  __device__ __forceinline__ void get(u64 i, u32& x, u32& y) const {
    const uint2 v = ld_stream(p + i);
    x = v.x;
    y = v.y;
  }
};
struct PairsI64 {
  const longlong2* p;
  __device__ __forceinline__ void get(u64 i, u32& x, u32& y) const {
    const longlong2 v = p[i];
    // ids outside [0, 2^32) map to kNone, which the range check rejects
    x = (v.x < 0 || v.x > 0xFFFFFFFFll) ? kNone : static_cast<u32>(v.x);
    y = (v.y < 0 || v.y > 0xFFFFFFFFll) ? kNone : static_cast<u32>(v.y);
  }
};
struct AnsU32 {
  u32* p;
  __device__ __forceinline__ void put(u64 i, u32 a) const { st_stream(p + i, a); }
};
struct AnsI64 {
  long long* p;
  __device__ __forceinline__ void put(u64 i, u32 a) const {
    p[i] = a == kNone ? -1ll : static_cast<long long>(a);
  }
};

// Query launch shape (A/B on B200, profiles/r1_lca_layout.md): the kernels
// are gather-latency bound, and full occupancy (8 x 256 threads per SM, <= 32
// registers) beats per-thread ILP (4 queries in flight at 64-72 registers):
// compact 75.6 -> 97.3, wide 32.9 -> 33.4 G q/s.
constexpr int kQThreads = 256;
constexpr int kQPer = 1;          // queries per thread per loop trip
constexpr int kQMinBlocks = 8;    // resident CTAs per SM (caps registers at 32)
constexpr int kQGridPerSM = 64;   // grid = min(ceil(q / 256), 64 x SMs), grid-stride

// Node-record sources of the wide kernel: {inlabel, ascendant, level, -}.
struct WideNodes {  // 16-B records
  const uint4* p;
  __device__ __forceinline__ void pair(u32 x, u32 y, uint4& A, uint4& B) const {
    A = ldg_rec(p + x);
    B = ldg_rec(p + y);
  }
};
// wide9: the same record in 9 B (n < 2^24), three per 32-B sector read with
// one 256-bit load: a 16M-node table of 171 MB instead of 256 MB.
struct Wide9Nodes {
  const uint32_t* p;
  __device__ __forceinline__ void pair(u32 x, u32 y, uint4& A, uint4& B) const {
    const u32 sx = rec9_sector(x), sy = rec9_sector(y);
    const Sector32 a = ldg_sector(p + 8 * static_cast<u64>(sx));
    const Sector32 b = ldg_sector(p + 8 * static_cast<u64>(sy));
    A = rec9_extract(a, x - 3 * sx);
    B = rec9_extract(b, y - 3 * sy);
  }
};

// inlabel_lca (core/src/lca.cpp:84-109): two node-record gathers, then at
// most two 8-B label-record gathers.
template <class In, class Out, class Nodes = WideNodes, bool kPf = false>
__global__ void __launch_bounds__(kQThreads, kQMinBlocks)
    k_lca_inlabel(Nodes node, const uint2* __restrict__ lab, u32 n, In in, Out out, u64 q,
                  u32* err) {
  static_assert(!kPf || kQPer == 1, "pair prefetch is written for one query per thread");
  const u64 stride = static_cast<u64>(gridDim.x) * kQThreads * kQPer;
  u32 bad_any = 0;
  u64 base = static_cast<u64>(blockIdx.x) * kQThreads * kQPer + threadIdx.x;
  u32 px = 0, py = 0;
  if (kPf && base < q) in.get(base, px, py);
  for (; base < q; base += stride) {
    u32 x[kQPer], y[kQPer];
    bool ok[kQPer], bad[kQPer];
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      const u64 i = base + static_cast<u64>(j) * kQThreads;
      ok[j] = i < q;
      x[j] = y[j] = 0;
      if (kPf) {
        x[j] = px;
        y[j] = py;
      } else if (ok[j]) {
        in.get(i, x[j], y[j]);
      }
      bad[j] = ok[j] && (x[j] >= n || y[j] >= n);
      if (bad[j]) x[j] = y[j] = 0;
    }
    if (kPf) {
      px = py = 0;
      if (base + stride < q) in.get(base + stride, px, py);
    }
    uint4 A[kQPer], B[kQPer];
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      node.pair(x[j], y[j], A[j], B[j]);
    }
    u32 ans[kQPer], wx[kQPer], wy[kQPer];
    bool lx[kQPer], ly[kQPer];
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      lx[j] = ly[j] = false;
      wx[j] = wy[j] = 0;
      if (A[j].x == B[j].x) {
        ans[j] = A[j].z <= B[j].z ? x[j] : y[j];
      } else {
        const int i = hb32(A[j].x ^ B[j].x);
        const u32 common = A[j].y & B[j].y & ~((1u << i) - 1u);
        const int jb = tz32(common);
        const u32 target = (A[j].x & ~((2u << jb) - 1u)) | (1u << jb);
        const u32 lowmask = (1u << jb) - 1u;
        if (A[j].x != target) {
          const int kx = hb32(A[j].y & lowmask);
          wx[j] = min((A[j].x & ~((2u << kx) - 1u)) | (1u << kx), n);
          lx[j] = true;
        }
        if (B[j].x != target) {
          const int ky = hb32(B[j].y & lowmask);
          wy[j] = min((B[j].x & ~((2u << ky) - 1u)) | (1u << ky), n);
          ly[j] = true;
        }
      }
    }
    uint2 LX[kQPer], LY[kQPer];
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      LX[j] = lx[j] ? ldg_rec(lab + wx[j]) : make_uint2(x[j], A[j].z);
      LY[j] = ly[j] ? ldg_rec(lab + wy[j]) : make_uint2(y[j], B[j].z);
    }
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      if (A[j].x != B[j].x) ans[j] = LX[j].y <= LY[j].y ? LX[j].x : LY[j].x;
      if (ok[j]) out.put(base + static_cast<u64>(j) * kQThreads, bad[j] ? kNone : ans[j]);
      bad_any |= bad[j];
    }
  }
  if (__any_sync(0xffffffffu, bad_any) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

// inlabel_lca, narrow layout: 8-B node record {inlabel, level} plus the
// ascendant looked up per label (asc[L], 4 B).  Halves the node table that
// every query gathers from at random (16M nodes: 128 MB instead of 256 MB,
// about the size of L2), at the price of a dependent ascendant gather when
// the inlabels differ.  Pays when few labels are in use (deep, path-like
// trees: the ascendant and label records stay in L2); see choose_layout().
template <class In, class Out, bool kPf = false>
__global__ void __launch_bounds__(kQThreads, kQMinBlocks)
    k_lca_inlabel_narrow(const uint2* __restrict__ node8, const u32* __restrict__ lasc,
                         const uint2* __restrict__ lab, u32 n, In in, Out out, u64 q, u32* err) {
  static_assert(!kPf || kQPer == 1, "pair prefetch is written for one query per thread");
  const u64 stride = static_cast<u64>(gridDim.x) * kQThreads * kQPer;
  u32 bad_any = 0;
  u64 base = static_cast<u64>(blockIdx.x) * kQThreads * kQPer + threadIdx.x;
  u32 px = 0, py = 0;
  if (kPf && base < q) in.get(base, px, py);
  for (; base < q; base += stride) {
    u32 x[kQPer], y[kQPer];
    bool ok[kQPer], bad[kQPer];
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      const u64 i = base + static_cast<u64>(j) * kQThreads;
      ok[j] = i < q;
      x[j] = y[j] = 0;
      if (kPf) {
        x[j] = px;
        y[j] = py;
      } else if (ok[j]) {
        in.get(i, x[j], y[j]);
      }
      bad[j] = ok[j] && (x[j] >= n || y[j] >= n);
      if (bad[j]) x[j] = y[j] = 0;
    }
    if (kPf) {
      px = py = 0;
      if (base + stride < q) in.get(base + stride, px, py);
    }
    uint2 A[kQPer], B[kQPer];
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      A[j] = ldg_rec(node8 + x[j]);
      B[j] = ldg_rec(node8 + y[j]);
    }
    u32 ax[kQPer], by[kQPer];
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      ax[j] = by[j] = 0;
      if (A[j].x != B[j].x) {
        ax[j] = ldg_u32(lasc + min(A[j].x, n));
        by[j] = ldg_u32(lasc + min(B[j].x, n));
      }
    }
    u32 ans[kQPer], wx[kQPer], wy[kQPer];
    bool lx[kQPer], ly[kQPer];
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      lx[j] = ly[j] = false;
      wx[j] = wy[j] = 0;
      if (A[j].x == B[j].x) {
        ans[j] = A[j].y <= B[j].y ? x[j] : y[j];
      } else {
        const int i = hb32(A[j].x ^ B[j].x);
        const u32 common = ax[j] & by[j] & ~((1u << i) - 1u);
        const int jb = tz32(common);
        const u32 target = (A[j].x & ~((2u << jb) - 1u)) | (1u << jb);
        const u32 lowmask = (1u << jb) - 1u;
        if (A[j].x != target) {
          const int kx = hb32(ax[j] & lowmask);
          wx[j] = min((A[j].x & ~((2u << kx) - 1u)) | (1u << kx), n);
          lx[j] = true;
        }
        if (B[j].x != target) {
          const int ky = hb32(by[j] & lowmask);
          wy[j] = min((B[j].x & ~((2u << ky) - 1u)) | (1u << ky), n);
          ly[j] = true;
        }
      }
    }
    uint2 LX[kQPer], LY[kQPer];
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      LX[j] = lx[j] ? ldg_rec(lab + wx[j]) : make_uint2(x[j], A[j].y);
      LY[j] = ly[j] ? ldg_rec(lab + wy[j]) : make_uint2(y[j], B[j].y);
    }
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      if (A[j].x != B[j].x) ans[j] = LX[j].y <= LY[j].y ? LX[j].x : LY[j].x;
      if (ok[j]) out.put(base + static_cast<u64>(j) * kQThreads, bad[j] ? kNone : ans[j]);
      bad_any |= bad[j];
    }
  }
  if (__any_sync(0xffffffffu, bad_any) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

// inlabel_lca, split layout: 8-B node record {inlabel, ascendant} and the
// level in a separate 4-B array, read only where the answer needs it (equal
// inlabels, or an endpoint that is not lifted).  On random trees nearly
// every query lifts both endpoints, so the hot table is 128 MB instead of
// the wide layout's 256 MB.
template <class In, class Out, bool kPf = false>
__global__ void __launch_bounds__(kQThreads, kQMinBlocks)
    k_lca_inlabel_split(const uint2* __restrict__ nodes, const u32* __restrict__ level,
                        const uint2* __restrict__ lab, u32 n, In in, Out out, u64 q, u32* err) {
  u32 bad_any = 0;
  const u64 stride = static_cast<u64>(gridDim.x) * kQThreads;
  u64 i = static_cast<u64>(blockIdx.x) * kQThreads + threadIdx.x;
  u32 px = 0, py = 0;
  if (kPf && i < q) in.get(i, px, py);
  for (; i < q; i += stride) {
    u32 x, y;
    if (kPf) {  // this trip's pair was loaded last trip; load the next one now
      x = px;
      y = py;
      px = py = 0;
      if (i + stride < q) in.get(i + stride, px, py);
    } else {
      in.get(i, x, y);
    }
    const bool bad = x >= n || y >= n;
    if (bad) x = y = 0;
    const uint2 A = ldg_rec(nodes + x), B = ldg_rec(nodes + y);
    bool lx = false, ly = false;
    u32 wx = 0, wy = 0;
    if (A.x != B.x) {
      const int hbit = hb32(A.x ^ B.x);
      const u32 common = A.y & B.y & ~((1u << hbit) - 1u);
      const int jb = tz32(common);
      const u32 target = (A.x & ~((2u << jb) - 1u)) | (1u << jb);
      const u32 lowmask = (1u << jb) - 1u;
      if (A.x != target) {
        const int kx = hb32(A.y & lowmask);
        wx = min((A.x & ~((2u << kx) - 1u)) | (1u << kx), n);
        lx = true;
      }
      if (B.x != target) {
        const int ky = hb32(B.y & lowmask);
        wy = min((B.x & ~((2u << ky) - 1u)) | (1u << ky), n);
        ly = true;
      }
    }
    const uint2 LX = lx ? ldg_rec(lab + wx) : make_uint2(x, ldg_u32(level + x));
    const uint2 LY = ly ? ldg_rec(lab + wy) : make_uint2(y, ldg_u32(level + y));
    out.put(i, bad ? kNone : (LX.y <= LY.y ? LX.x : LY.x));
    bad_any |= bad;
  }
  if (__any_sync(0xffffffffu, bad_any) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

// inlabel_lca, split6 layout: the split record packed into 6 B (inlabel and
// ascendant are < 2^24 when n < 2^24), so the gathered node table of a 16M
// tree is 96 MB instead of 128 MB -- under the size at which B200's random
// gather rate falls off (footprint sweep: 96 MB 151, 128 MB 113 G gathers/s).
// kL2: 1 = node-sector gathers with an L2 evict_last policy, 2 = the label
// and level gathers too (ETTG_L2HINT A/B).
template <class In, class Out, bool kPf = false, int kL2 = 0>
__global__ void __launch_bounds__(kQThreads, kQMinBlocks)
    k_lca_inlabel_split6(const uint32_t* __restrict__ nodes6, const u32* __restrict__ level,
                        const uint2* __restrict__ lab, u32 n, In in, Out out, u64 q, u32* err) {
  u32 bad_any = 0;
  const u64 stride = static_cast<u64>(gridDim.x) * kQThreads;
  u64 i = static_cast<u64>(blockIdx.x) * kQThreads + threadIdx.x;
  u32 px = 0, py = 0;
  if (kPf && i < q) in.get(i, px, py);
  for (; i < q; i += stride) {
    u32 x, y;
    if (kPf) {  // this trip's pair was loaded last trip; load the next one now
      x = px;
      y = py;
      px = py = 0;
      if (i + stride < q) in.get(i + stride, px, py);
    } else {
      in.get(i, x, y);
    }
    const bool bad = x >= n || y >= n;
    if (bad) x = y = 0;
    uint2 A, B;
    // the policy word is made per trip: holding it across the loop spills at 32 registers
    const u64 pol = kL2 ? l2_policy_evict_last() : 0;
    if (kL2)
      ldg_rec6_pair_l2<kL2 == 4>(nodes6, x, y, A, B, pol);
    else
      ldg_rec6_pair(nodes6, x, y, A, B);
    bool lx = false, ly = false;
    u32 wx = 0, wy = 0;
    if (A.x != B.x) {
      const int hbit = hb32(A.x ^ B.x);
      const u32 common = A.y & B.y & ~((1u << hbit) - 1u);
      const int jb = tz32(common);
      const u32 target = (A.x & ~((2u << jb) - 1u)) | (1u << jb);
      const u32 lowmask = (1u << jb) - 1u;
      if (A.x != target) {
        const int kx = hb32(A.y & lowmask);
        wx = min((A.x & ~((2u << kx) - 1u)) | (1u << kx), n);
        lx = true;
      }
      if (B.x != target) {
        const int ky = hb32(B.y & lowmask);
        wy = min((B.x & ~((2u << ky) - 1u)) | (1u << ky), n);
        ly = true;
      }
    }
    uint2 LX, LY;
    if (kL2 == 2) {
      LX = lx ? ldg_rec_l2(lab + wx, pol) : make_uint2(x, ldg_u32_l2(level + x, pol));
      LY = ly ? ldg_rec_l2(lab + wy, pol) : make_uint2(y, ldg_u32_l2(level + y, pol));
    } else {
      LX = lx ? ldg_rec(lab + wx) : make_uint2(x, ldg_u32(level + x));
      LY = ly ? ldg_rec(lab + wy) : make_uint2(y, ldg_u32(level + y));
    }
    out.put(i, bad ? kNone : (LX.y <= LY.y ? LX.x : LY.x));
    bad_any |= bad;
  }
  if (__any_sync(0xffffffffu, bad_any) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

// inlabel_lca, split_own layout: 16-B node record {inlabel, ascendant,
// own-label lift record}; the level in its own array as in split.  A lift to
// the endpoint's own label (the only ascendant bit below j is tz(inlabel))
// is answered from the record.
template <class In, class Out>
__global__ void __launch_bounds__(kQThreads, kQMinBlocks)
    k_lca_inlabel_split_own(const uint4* __restrict__ node, const u32* __restrict__ level,
                            const uint2* __restrict__ lab, u32 n, In in, Out out, u64 q,
                            u32* err) {
  u32 bad_any = 0;
  for (u64 i = static_cast<u64>(blockIdx.x) * kQThreads + threadIdx.x; i < q;
       i += static_cast<u64>(gridDim.x) * kQThreads) {
    u32 x, y;
    in.get(i, x, y);
    const bool bad = x >= n || y >= n;
    if (bad) x = y = 0;
    const uint4 A = ldg_rec(node + x), B = ldg_rec(node + y);
    bool lx = false, ly = false, ox = false, oy = false;
    u32 wx = 0, wy = 0;
    if (A.x != B.x) {
      const int hbit = hb32(A.x ^ B.x);
      const u32 common = A.y & B.y & ~((1u << hbit) - 1u);
      const int jb = tz32(common);
      const u32 target = (A.x & ~((2u << jb) - 1u)) | (1u << jb);
      const u32 lowmask = (1u << jb) - 1u;
      if (A.x != target) {
        const u32 below = A.y & lowmask;
        ox = __popc(below) == 1;
        const int kx = hb32(below);
        wx = min((A.x & ~((2u << kx) - 1u)) | (1u << kx), n);
        lx = !ox;
      }
      if (B.x != target) {
        const u32 below = B.y & lowmask;
        oy = __popc(below) == 1;
        const int ky = hb32(below);
        wy = min((B.x & ~((2u << ky) - 1u)) | (1u << ky), n);
        ly = !oy;
      }
    }
    const uint2 LX = ox ? make_uint2(A.z, A.w)
                        : lx ? ldg_rec(lab + wx) : make_uint2(x, ldg_u32(level + x));
    const uint2 LY = oy ? make_uint2(B.z, B.w)
                        : ly ? ldg_rec(lab + wy) : make_uint2(y, ldg_u32(level + y));
    out.put(i, bad ? kNone : (LX.y <= LY.y ? LX.x : LY.x));
    bad_any |= bad;
  }
  if (__any_sync(0xffffffffu, bad_any) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

// inlabel_lca, compact layout: one 4-B node word per endpoint.  Endpoints on
// the same inlabel path (same label index) are answered from the words alone
// (the smaller in-path offset is the ancestor); otherwise the two label-table
// entries restore {inlabel, ascendant, level} and the query proceeds exactly
// as in k_lca_inlabel.  On the 16M path tree the node table is 64 MB and the
// label table holds 7 entries, so every gather is served by L2 after its
// first touch.
// kPf: the next grid-stride trip's pair is loaded before this trip's gathers
// (its stream latency overlaps them; kQPer == 1).
template <class In, class Out, bool kPf = false>
__global__ void __launch_bounds__(kQThreads, kQMinBlocks)
    k_lca_inlabel_compact(const u32* __restrict__ node4, const uint4* __restrict__ ltab,
                          const uint2* __restrict__ lab, u32 n, int off_bits, In in, Out out,
                          u64 q, u32* err) {
  static_assert(!kPf || kQPer == 1, "pair prefetch is written for one query per thread");
  const u64 stride = static_cast<u64>(gridDim.x) * kQThreads * kQPer;
  const u32 omask = off_bits >= 32 ? ~0u : ((1u << off_bits) - 1u);
  u32 bad_any = 0;
  u64 base = static_cast<u64>(blockIdx.x) * kQThreads * kQPer + threadIdx.x;
  u32 px = 0, py = 0;
  if (kPf && base < q) in.get(base, px, py);
  for (; base < q; base += stride) {
    u32 x[kQPer], y[kQPer];
    bool ok[kQPer], bad[kQPer];
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      const u64 i = base + static_cast<u64>(j) * kQThreads;
      ok[j] = i < q;
      x[j] = y[j] = 0;
      if (kPf) {
        x[j] = px;
        y[j] = py;
      } else if (ok[j]) {
        in.get(i, x[j], y[j]);
      }
      bad[j] = ok[j] && (x[j] >= n || y[j] >= n);
      if (bad[j]) x[j] = y[j] = 0;
    }
    if (kPf) {
      px = py = 0;
      if (base + stride < q) in.get(base + stride, px, py);
    }
    u32 wa[kQPer], wb[kQPer];
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      wa[j] = ldg_u32(node4 + x[j]);
      wb[j] = ldg_u32(node4 + y[j]);
    }
    uint4 A[kQPer], B[kQPer];
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      const u32 la = off_bits >= 32 ? 0u : wa[j] >> off_bits;
      const u32 lb = off_bits >= 32 ? 0u : wb[j] >> off_bits;
      A[j] = B[j] = make_uint4(0u, 0u, 0u, 0u);
      if (la != lb) {
        A[j] = ldg_rec(ltab + la);
        B[j] = ldg_rec(ltab + lb);
      }
    }
    u32 ans[kQPer], wx[kQPer], wy[kQPer];
    bool same[kQPer], lx[kQPer], ly[kQPer];
    uint2 LX[kQPer], LY[kQPer];
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      const u32 ox = wa[j] & omask, oy = wb[j] & omask;
      same[j] = (wa[j] ^ wb[j]) <= omask;  // same label index
      lx[j] = ly[j] = false;
      wx[j] = wy[j] = 0;
      ans[j] = ox <= oy ? x[j] : y[j];
      LX[j] = make_uint2(x[j], A[j].z + ox);
      LY[j] = make_uint2(y[j], B[j].z + oy);
      if (!same[j]) {
        const int i = hb32(A[j].x ^ B[j].x);
        const u32 common = A[j].y & B[j].y & ~((1u << i) - 1u);
        const int jb = tz32(common);
        const u32 target = (A[j].x & ~((2u << jb) - 1u)) | (1u << jb);
        const u32 lowmask = (1u << jb) - 1u;
        if (A[j].x != target) {
          const int kx = hb32(A[j].y & lowmask);
          wx[j] = min((A[j].x & ~((2u << kx) - 1u)) | (1u << kx), n);
          lx[j] = true;
        }
        if (B[j].x != target) {
          const int ky = hb32(B[j].y & lowmask);
          wy[j] = min((B[j].x & ~((2u << ky) - 1u)) | (1u << ky), n);
          ly[j] = true;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      if (lx[j]) LX[j] = ldg_rec(lab + wx[j]);
      if (ly[j]) LY[j] = ldg_rec(lab + wy[j]);
    }
#pragma unroll
    for (int j = 0; j < kQPer; ++j) {
      if (!same[j]) ans[j] = LX[j].y <= LY[j].y ? LX[j].x : LY[j].x;
      if (ok[j]) out.put(base + static_cast<u64>(j) * kQThreads, bad[j] ? kNone : ans[j]);
      bad_any |= bad[j];
    }
  }
  if (__any_sync(0xffffffffu, bad_any) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

// Compact layout, two-stage software pipeline (ETTG_QPF=2): at the top of
// each trip the node words of the next trip's endpoints are gathered and
// the pair after that is loaded, then this trip's query finishes from the
// words gathered one trip earlier -- so each thread keeps its next gathers
// in flight while it works (the kernel is bound by L1 -> L2 requests,
// DESIGN.md section 4).
template <class In, class Out, int kL2 = 0>
__global__ void __launch_bounds__(kQThreads, kQMinBlocks)
    k_lca_inlabel_compact_pipe(const u32* __restrict__ node4, const uint4* __restrict__ ltab,
                               const uint2* __restrict__ lab, u32 n, int off_bits, In in, Out out,
                               u64 q, u32* err) {
  const u64 stride = static_cast<u64>(gridDim.x) * kQThreads;
  const u32 omask = off_bits >= 32 ? ~0u : ((1u << off_bits) - 1u);
  u32 bad_any = 0;
  u64 i = static_cast<u64>(blockIdx.x) * kQThreads + threadIdx.x;
  // stage 0: pair of trip i; stage 1: words of trip i, pair of trip i + stride
  u32 x = 0, y = 0, wa = 0, wb = 0, nx = 0, ny = 0;
  bool bad = false;
  if (i < q) {
    in.get(i, x, y);
    bad = x >= n || y >= n;
    if (bad) x = y = 0;
    const u64 pol = kL2 ? l2_policy_evict_last() : 0;
    wa = (kL2 == 3 ? ldg_u32_l2_na(node4 + x, pol) : kL2 ? ldg_u32_l2(node4 + x, pol) : ldg_u32(node4 + x));
    wb = (kL2 == 3 ? ldg_u32_l2_na(node4 + y, pol) : kL2 ? ldg_u32_l2(node4 + y, pol) : ldg_u32(node4 + y));
  }
  if (i + stride < q) in.get(i + stride, nx, ny);
  for (; i < q; i += stride) {
    // next trip: its words and the pair after it
    const u64 i1 = i + stride;
    const u64 pol = kL2 ? l2_policy_evict_last() : 0;  // per trip: see split6
    bool nbad = false;
    u32 nwa = 0, nwb = 0, cx = nx, cy = ny;
    if (i1 < q) {
      nbad = cx >= n || cy >= n;
      if (nbad) cx = cy = 0;
      nwa = (kL2 == 3 ? ldg_u32_l2_na(node4 + cx, pol) : kL2 ? ldg_u32_l2(node4 + cx, pol) : ldg_u32(node4 + cx));
      nwb = (kL2 == 3 ? ldg_u32_l2_na(node4 + cy, pol) : kL2 ? ldg_u32_l2(node4 + cy, pol) : ldg_u32(node4 + cy));
      nx = ny = 0;
      if (i1 + stride < q) in.get(i1 + stride, nx, ny);
    }
    // this trip
    const u32 la = off_bits >= 32 ? 0u : wa >> off_bits;
    const u32 lb = off_bits >= 32 ? 0u : wb >> off_bits;
    uint4 A = make_uint4(0u, 0u, 0u, 0u), B = A;
    if (la != lb) {
      A = ldg_rec(ltab + la);
      B = ldg_rec(ltab + lb);
    }
    const u32 ox = wa & omask, oy = wb & omask;
    u32 ans = ox <= oy ? x : y;
    if ((wa ^ wb) > omask) {  // different label indices
      const int hbit = hb32(A.x ^ B.x);
      const u32 common = A.y & B.y & ~((1u << hbit) - 1u);
      const int jb = tz32(common);
      const u32 target = (A.x & ~((2u << jb) - 1u)) | (1u << jb);
      const u32 lowmask = (1u << jb) - 1u;
      uint2 LX = make_uint2(x, A.z + ox), LY = make_uint2(y, B.z + oy);
      if (A.x != target) {
        const int kx = hb32(A.y & lowmask);
        LX = ldg_rec(lab + min((A.x & ~((2u << kx) - 1u)) | (1u << kx), n));
      }
      if (B.x != target) {
        const int ky = hb32(B.y & lowmask);
        LY = ldg_rec(lab + min((B.x & ~((2u << ky) - 1u)) | (1u << ky), n));
      }
      ans = LX.y <= LY.y ? LX.x : LY.x;
    }
    out.put(i, bad ? kNone : ans);
    bad_any |= bad;
    x = cx;
    y = cy;
    wa = nwa;
    wb = nwb;
    bad = nbad;
  }
  if (__any_sync(0xffffffffu, bad_any) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

// naive_lca (core/src/lca.cpp:118-126): walk the deeper node up, then both.
// One query per thread; cost is the x-y tree distance (the paper's baseline).
template <class In, class Out>
__global__ void __launch_bounds__(kQThreads)
    k_lca_naive(const uint2* __restrict__ nrec, u32 n, In in, Out out, u64 q, u32* err) {
  u32 bad_any = 0;
  for (u64 i = static_cast<u64>(blockIdx.x) * kQThreads + threadIdx.x; i < q;
       i += static_cast<u64>(gridDim.x) * kQThreads) {
    u32 x, y;
    in.get(i, x, y);
    if (x >= n || y >= n) {
      bad_any = 1;
      out.put(i, kNone);
      continue;
    }
    uint2 rx = __ldg(nrec + x), ry = __ldg(nrec + y);
    while (rx.y > ry.y) {
      x = rx.x;
      rx = __ldg(nrec + x);
    }
    while (ry.y > rx.y) {
      y = ry.x;
      ry = __ldg(nrec + y);
    }
    while (x != y) {
      x = rx.x;
      y = ry.x;
      rx = __ldg(nrec + x);
      ry = __ldg(nrec + y);
    }
    out.put(i, x);
  }
  if (__any_sync(0xffffffffu, bad_any) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

struct RmqView {
  const u64* key;
  const u64* pre_in;
  const u64* suf_in;
  const u64* sp;
  const u32* first;
  u32 nb;
  __device__ __forceinline__ u32 query(u32 x, u32 y) const {
    u32 l = __ldg(first + x), r = __ldg(first + y);
    if (l > r) {
      const u32 t = l;
      l = r;
      r = t;
    }
    const u32 lb = l >> 5, rb = r >> 5;
    u64 m;
    if (lb == rb) {
      m = ~0ull;
      for (u32 t = l; t <= r; ++t) m = min(m, __ldg(key + t));
    } else {
      m = min(__ldg(suf_in + l), __ldg(pre_in + r));
      if (rb > lb + 1) {
        const int k = hb32(rb - lb - 1);
        const u64* row = sp + static_cast<u64>(k) * nb;
        m = min(m, min(__ldg(row + lb + 1), __ldg(row + rb - (1u << k))));
      }
    }
    return static_cast<u32>(m);
  }
};

// rmq_lca (core/src/lca.cpp:151-157) with O(1) block-sparse lookups.
template <class In, class Out>
__global__ void __launch_bounds__(kQThreads)
    k_lca_rmq(RmqView rv, u32 n, In in, Out out, u64 q, u32* err) {
  u32 bad_any = 0;
  for (u64 i = static_cast<u64>(blockIdx.x) * kQThreads + threadIdx.x; i < q;
       i += static_cast<u64>(gridDim.x) * kQThreads) {
    u32 x, y;
    in.get(i, x, y);
    const bool bad = x >= n || y >= n;
    bad_any |= bad;
    out.put(i, bad ? kNone : rv.query(x, y));
  }
  if (__any_sync(0xffffffffu, bad_any) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

}  // namespace ettg

// ============================================================================
// Handle and C-ABI
// ============================================================================
using namespace ettg;

constexpr u32 kLayoutWide = 0, kLayoutNarrow = 1, kLayoutCompact = 2, kLayoutSplit = 3,
              kLayoutSplitOwn = 4, kLayoutSplit6 = 5, kLayoutWide9 = 6;

struct ettg_lca {
  std::mutex qmu;  // host-buffer queries share the handle's staging buffers
  int device = 0;
  u32 n = 0;
  u32 root = 0;
  unsigned engines = 0;
  bool full = false;  // built here (stats available) vs attached replica
  cudaStream_t stream = nullptr;
  cudaStream_t qs[2] = {nullptr, nullptr};
  char* mem = nullptr;
  uint4* node = nullptr;   // wide layout: {inlabel, ascendant, level, 0}
  uint2* nodes = nullptr;  // split layout: {inlabel, ascendant} ...
  uint32_t* nodes6 = nullptr;  // split6 layout: the same record in 6 B ...
  uint32_t* nodes9 = nullptr;  // wide9 layout: the wide record in 9 B (3 per sector)
  u32* slevel = nullptr;   // ... + level per node
  uint2* node8 = nullptr;  // narrow layout: {inlabel, level} ...
  u32* lasc = nullptr;     // ... + ascendant per label
  uint2* lab = nullptr;    // label record {parent(head(L)), level of it}
  u32* node4 = nullptr;    // compact layout: label index << off_bits | in-path offset
  uint4* ltab = nullptr;   // ... + {inlabel, ascendant, level(head), 0} per label index
  char* cmem = nullptr;    // compact arrays not carved from `mem`
  u64 ltab_cap = 0;
  int off_bits = 0;
  u32 layout = kLayoutWide;
  u64 labels = 0;          // inlabel paths in the tree
  u32 *par = nullptr, *pre = nullptr, *size = nullptr, *level = nullptr, *inlabel = nullptr,
      *first = nullptr, *head = nullptr;
  // rmq
  u64 *tkey = nullptr, *pre_in = nullptr, *suf_in = nullptr, *sp = nullptr;
  u32 nb = 0, levels = 0;
  // naive
  uint2* nrec = nullptr;
  // host-query staging (lazy)
  char* qmem = nullptr;
  u64 qchunk = 0;
  u32* qerr = nullptr;
  // device-resident queries: sticky out-of-range flag (ettg_lca_query_dev_error)
  std::once_flag derr_once;
  u32* derr = nullptr;
  double build_ms = 0;

  void carve(Carver& c) {
    if (engines & ETTG_ENGINE_INLABEL) {
      // a full build packs every layout (~28 B/node extra); replicas carry one
      if (full || layout == kLayoutWide || layout == kLayoutSplitOwn) node = c.take<uint4>(n);
      if (full || layout == kLayoutNarrow) {
        node8 = c.take<uint2>(n);
        lasc = c.take<u32>(static_cast<u64>(n) + 1);
      }
      if (full || layout == kLayoutSplit) nodes = c.take<uint2>(n);
      // packed records exist only for n < 2^24 (24-bit fields)
      const bool packable = n < (1u << 24);
      if ((full && packable) || layout == kLayoutSplit6) nodes6 = c.take<uint32_t>(rec6_bytes(n) / 4);
      if ((full && packable) || layout == kLayoutWide9) nodes9 = c.take<uint32_t>(rec9_bytes(n) / 4);
      if (!full && (layout == kLayoutSplit || layout == kLayoutSplitOwn || layout == kLayoutSplit6))
        slevel = c.take<u32>(n);  // full builds query h->level
      lab = c.take<uint2>(static_cast<u64>(n) + 1);
      if (full) {
        node4 = c.take<u32>(n);
        ltab_cap = std::min<u64>(n, kLtabCap);
        ltab = c.take<uint4>(ltab_cap);
      }
    }
    if (engines & ETTG_ENGINE_NAIVE) nrec = c.take<uint2>(n);
    if (!full) return;
    par = c.take<u32>(n);
    pre = c.take<u32>(n);
    size = c.take<u32>(n);
    level = c.take<u32>(n);
    if (nodes) slevel = level;
    inlabel = c.take<u32>(n);
    first = c.take<u32>(n);
    head = c.take<u32>(static_cast<u64>(n) + 1);
    if (engines & ETTG_ENGINE_RMQ) {
      const u32 steps = 2 * n - 1;
      nb = (steps + 31) / 32;
      levels = 32 - __builtin_clz(nb);
      tkey = c.take<u64>(steps);
      pre_in = c.take<u64>(steps);
      suf_in = c.take<u64>(steps);
      sp = c.take<u64>(static_cast<u64>(levels) * nb);
    }
  }
  // Compact arrays: full builds carve the node words and a label table of
  // kLtabCap entries up front (the auto rule only picks compact for fewer
  // labels); a larger forced table, or a replica, gets its own allocation.
  static constexpr u64 kLtabCap = u64(1) << 18;
  void alloc_compact() {
    if (node4 && labels <= ltab_cap) return;
    Carver c;
    if (!node4) c.take<u32>(n);
    c.take<uint4>(labels);
    CK(cudaMalloc(&cmem, c.off));
    c = Carver{cmem};
    if (!node4) node4 = c.take<u32>(n);
    ltab = c.take<uint4>(labels);
    ltab_cap = labels;
  }
  ~ettg_lca() {
    if (cmem) cudaFree(cmem);
    if (mem) cudaFree(mem);
    if (qmem) cudaFree(qmem);
    if (derr) cudaFree(derr);
    for (auto s : qs)
      if (s) cudaStreamDestroy(s);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

struct BuildWs {
  int64_t* par64 = nullptr;
  u32 *keys = nullptr, *vals = nullptr, *pkey = nullptr, *child = nullptr;
  SortWs sort;
  uint2* crange = nullptr;
  u32* jj = nullptr;
  ListRankWs lr;
  u32* up = nullptr;
  uint4* hrec = nullptr;
  u64* scan = nullptr;
  u32* flags = nullptr;
  void carve(Carver& c, u32 n, bool host_i64) {
    if (host_i64) par64 = c.take<int64_t>(n);
    const u32 m = n - 1;
    keys = c.take<u32>(m + 1);
    vals = c.take<u32>(m + 1);
    pkey = c.take<u32>(m + 1);
    child = c.take<u32>(m + 1);
    sort.carve(c, m + 1);
    crange = c.take<uint2>(n);
    jj = c.take<u32>(n);
    // level means 32 / 8 (vs 16 / 16): 16M random tree build 5.02 -> 4.87 ms,
    // 16M path 4.40 -> 4.35 ms (profiles/r2_bridges_notes.md, gpurun_out/r2ab2)
    lr.carve(c, 2 * n, false, 32, 8);
    up = c.take<u32>(static_cast<u64>(n) + 1);
    hrec = c.take<uint4>(static_cast<u64>(n) + 1);
    scan = c.take<u64>(scan_ws_words(static_cast<u64>(n) + 1));
    flags = c.take<u32>(8);
  }
};

void launch_stats_rmq(ettg_lca* h, cudaStream_t st, int sms) {
  const u32 n = h->n;
  const u32 steps = 2 * n - 1;
  const unsigned g = sms * 8;
  k_rmq_block<<<blocks_for(static_cast<u64>(h->nb) * 32, 256), 256, 0, st>>>(
      h->tkey, steps, h->nb, h->pre_in, h->suf_in, h->sp);
  CK_LAUNCH();
  build_sparse_rows(h->sp, h->nb, h->levels, MinU64{}, g, st);
}

// naive_build (core/src/lca.cpp:111-116): validate + pointer-jumping levels.
ettg_lca* build_naive_only(const void* parent, bool host_i64, int64_t n64, int64_t root64,
                           int device, cudaStream_t user_st) {
  const u32 n = static_cast<u32>(n64), root = static_cast<u32>(root64);
  const int sms = sm_count(device);
  const unsigned g = sms * 8;
  auto h = std::make_unique<ettg_lca>();
  h->device = device;
  h->n = n;
  h->root = root;
  h->engines = ETTG_ENGINE_NAIVE;
  h->full = false;
  CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  cudaStream_t st = user_st ? user_st : h->stream;
  Carver hc;
  h->carve(hc);
  CK(cudaMalloc(&h->mem, hc.off));
  hc = Carver{h->mem};
  h->carve(hc);
  struct Ws {
    int64_t* par64 = nullptr;
    u32 *par = nullptr, *keys = nullptr, *vals = nullptr, *flags = nullptr;
    uint2 *s0 = nullptr, *s1 = nullptr;
    void carve(Carver& c, u32 n, bool h64) {
      if (h64) par64 = c.take<int64_t>(n);
      par = c.take<u32>(n);
      keys = c.take<u32>(n);
      vals = c.take<u32>(n);
      s0 = c.take<uint2>(n);
      s1 = c.take<uint2>(n);
      flags = c.take<u32>(8);
    }
  } ws;
  Carver wc;
  ws.carve(wc, n, host_i64);
  Lease lease(device, st, wc.off);
  wc = Carver{lease.base()};
  ws.carve(wc, n, host_i64);
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st));
  CK(cudaMemsetAsync(ws.flags, 0, 8 * sizeof(u32), st));
  const unsigned gb = std::min(g, blocks_for(n, 256));
  if (host_i64) {
    copy_h2d(ws.par64, parent, static_cast<u64>(n) * 8, device, st);
    k_tree_validate<int64_t><<<gb, 256, 0, st>>>(ws.par64, n, root, ws.par, ws.keys, ws.vals,
                                                 ws.flags);
  } else {
    k_tree_validate<u32><<<gb, 256, 0, st>>>(static_cast<const u32*>(parent), n, root, ws.par,
                                             ws.keys, ws.vals, ws.flags);
  }
  CK_LAUNCH();
  k_dbl_init<<<gb, 256, 0, st>>>(ws.par, n, root, ws.s0);
  CK_LAUNCH();
  uint2* cur = ws.s0;
  uint2* nxt = ws.s1;
  const int rounds = (32 - __builtin_clz(n)) + 1;
  for (int r = 0; r < rounds; ++r) {
    k_dbl_round<<<gb, 256, 0, st>>>(cur, nxt, n);
    CK_LAUNCH();
    std::swap(cur, nxt);
  }
  k_dbl_finish<<<gb, 256, 0, st>>>(cur, ws.par, n, root, h->nrec, ws.flags + 1);
  CK_LAUNCH();
  CK(cudaEventRecord(e1, st));
  u32 vflags[8];
  CK(cudaMemcpyAsync(vflags, ws.flags, sizeof vflags, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (vflags[0] & kVRootParent) einval("root has no kNone parent entry");
  if (vflags[0] & kVRange) einval("parent id out of range");
  if (vflags[0] & kVRoots) einval("tree must have exactly one root");
  if (vflags[1]) einval("cycle in parent array");
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  h->build_ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return h.release();
}

// Layout choice (measured, profiles/r1_lca_layout.md).  Random gathers get
// faster as the gathered table shrinks toward L2 (B200 footprint sweep: 256 MB
// -> 72, 128 MB -> 113, 64 MB -> 264 G gathers/s), so each layout trades
// node-record bytes against extra per-label or per-node reads:
//   few labels (deep trees; per-label tables stay in L2): compact if its
//     bit budget fits, else narrow          16M path: compact 97.5 G q/s
//   labels >= n/2 (shallow trees: almost every query lifts both endpoints,
//     so the level array is rarely read): split    16M grasp(inf): 55.7;
//     split6 (the same record in 6 B) when n >= L2/16  16M grasp(inf): 67.3;
//     split_own when a build-time query sample sees > 50% own-label lifts
//     (16M star: see profiles/r1_lca_layout.md)
//   otherwise wide                              16M gamma=2: wide 24.3
bool split6_enabled() {
  const char* e = std::getenv("ETTG_SPLIT6");
  return !e || std::atoi(e) != 0;
}

u32 choose_layout(u32 n, u64 labels, bool compact_fits, double own_frac, double level_per_q,
                  int device, unsigned flags) {
  if (flags == ETTG_LAYOUT_WIDE) return kLayoutWide;
  if (flags == ETTG_LAYOUT_NARROW) return kLayoutNarrow;
  if (flags == ETTG_LAYOUT_SPLIT) return kLayoutSplit;
  if (flags == ETTG_LAYOUT_SPLIT_OWN) return kLayoutSplitOwn;
  if (flags == ETTG_LAYOUT_WIDE9) {
    if (n >= (1u << 24)) einval("wide9 layout: needs n < 2^24 (24-bit fields)");
    return kLayoutWide9;
  }
  if (flags == ETTG_LAYOUT_SPLIT6) {
    if (n >= (1u << 24)) einval("split6 layout: needs n < 2^24 (24-bit inlabels)");
    return kLayoutSplit6;
  }
  if (flags == ETTG_LAYOUT_COMPACT) {
    if (!compact_fits) einval("compact layout: label index + in-path offset exceed 32 bits");
    return kLayoutCompact;
  }
  int l2 = 0;
  if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device) != cudaSuccess || l2 <= 0)
    l2 = 126 << 20;
  const u64 L2 = static_cast<u64>(l2);
  if (labels * 64 <= L2 / 8) return compact_fits ? kLayoutCompact : kLayoutNarrow;
  (void)n;
  // split keeps the level out of the gathered record, so it wins when the
  // sampled queries rarely need a level (most endpoints are lifted); when most
  // lifts go to the endpoint's own label (stars, caterpillars) that lift
  // target rides in the record (split_own).  16M trees, G q/s wide/split:
  // grasp(inf) 33.4/55.7, gamma=64 26.9/35.6, 16 20.0/21.4, 8 18.9/18.7,
  // 4 20.4/18.7, 2 24.3/20.2 (level reads per query 0, 0.06, ~0.2, 0.38, ..,
  // 0.99).
  // Packed records (n < 2^24) once the unpacked table would outgrow the
  // fast-gather footprint: split6 (6 B) for shallow trees, wide9 (9 B, level
  // inline) once a level is read for >= 0.3 endpoints per query.  16M trees,
  // G q/s split / split6 / wide / wide9: grasp(inf) 55.6/67.3/-/42.5,
  // gamma=64 35.5/40.1/-/31.8, 16 21.4/23.2/-/22.2, 8 18.7/20.0/18.9/20.7,
  // 4 -/20.0/20.4/22.8, 2 -/21.9/24.3/28.1; on 1M-4M trees (tables in L2) the
  // unpacked records are as fast or faster.
  if (own_frac > 0.5 && level_per_q < 0.25) return kLayoutSplitOwn;
  const bool six = n < (1u << 24) && static_cast<u64>(n) * 8 > L2 / 2 && split6_enabled();
  if (six && level_per_q < 0.3) return kLayoutSplit6;
  if (level_per_q < 0.25) return kLayoutSplit;
  const bool nine = n < (1u << 24) && static_cast<u64>(n) * 16 > L2 / 2 && split6_enabled();
  return nine ? kLayoutWide9 : kLayoutWide;
}

ettg_lca* build_index(const void* parent, bool host_i64, bool dev_u32, int64_t n64,
                      int64_t root64, int device, unsigned engines, cudaStream_t user_st) {
  if (n64 <= 0) einval("parent array size mismatch");
  if (n64 >= (int64_t(1) << 31)) einval("tree too large for the 32-bit device index (n >= 2^31)");
  if (root64 < 0 || root64 >= n64) einval("root has no kNone parent entry");
  constexpr unsigned kLayoutMask = ETTG_LAYOUT_WIDE | ETTG_LAYOUT_NARROW | ETTG_LAYOUT_COMPACT |
                                   ETTG_LAYOUT_SPLIT | ETTG_LAYOUT_SPLIT_OWN | ETTG_LAYOUT_SPLIT6 |
                                   ETTG_LAYOUT_WIDE9;
  const unsigned layout_flags = engines & kLayoutMask;
  engines &= ~kLayoutMask;
  if (layout_flags & (layout_flags - 1)) einval("conflicting layout flags");
  if (engines == 0) engines = ETTG_ENGINE_INLABEL;
  if (engines & ~(ETTG_ENGINE_INLABEL | ETTG_ENGINE_RMQ | ETTG_ENGINE_NAIVE))
    einval("unknown engine flag");
  if (engines == ETTG_ENGINE_NAIVE)
    return build_naive_only(parent, host_i64, n64, root64, device, user_st);
  engines |= ETTG_ENGINE_INLABEL;  // the Euler-tour build yields it for free
  const u32 n = static_cast<u32>(n64), root = static_cast<u32>(root64);
  const int sms = sm_count(device);

  auto h = std::make_unique<ettg_lca>();
  h->device = device;
  h->n = n;
  h->root = root;
  h->engines = engines;
  h->full = true;
  CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  cudaStream_t st = user_st ? user_st : h->stream;

  Carver hc;
  h->carve(hc);
  CK(cudaMalloc(&h->mem, hc.off));
  hc = Carver{h->mem};
  h->carve(hc);

  Carver wc;
  BuildWs ws;
  ws.carve(wc, n, host_i64);
  Lease lease(device, st, wc.off);
  wc = Carver{lease.base()};
  ws.carve(wc, n, host_i64);

  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, st));
  Trace tr("lca_build", st);

  const u32 m = n - 1;
  const unsigned g = sms * 8;
  CK(cudaMemsetAsync(ws.flags, 0, 8 * sizeof(u32), st));
  if (host_i64) {
    copy_h2d(ws.par64, parent, static_cast<u64>(n) * 8, device, st);
    k_tree_validate<int64_t><<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(
        ws.par64, n, root, h->par, ws.keys, ws.vals, ws.flags);
  } else {
    (void)dev_u32;
    k_tree_validate<u32><<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(
        static_cast<const u32*>(parent), n, root, h->par, ws.keys, ws.vals, ws.flags);
  }
  CK_LAUNCH();
  tr.mark("validate");
  sort_pairs(ws.keys, ws.vals, ws.pkey, ws.child, m, bits_for(n - 1), ws.sort, st);
  tr.mark("sort");
  CK(cudaMemsetAsync(ws.crange, 0, static_cast<u64>(n) * sizeof(uint2), st));
  if (m > 0) {
    k_child_ranges<<<std::min(g, blocks_for(m, 256)), 256, 0, st>>>(ws.pkey, m, ws.crange);
    CK_LAUNCH();
  }
  k_node_succ<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(ws.crange, ws.child, h->par, n,
                                                              root, ws.jj, ws.lr.succ0);
  CK_LAUNCH();
  if (m > 0) {
    k_slot_succ<<<std::min(g, blocks_for(m, 256)), 256, 0, st>>>(ws.crange, ws.child, ws.pkey,
                                                                ws.jj, m, root, ws.lr.succ0);
    CK_LAUNCH();
  }
  tr.mark("succ");
  list_rank_core(2 * n, 2 * root, EvenIsDown{}, ws.lr, st, sms);
  tr.mark("list_rank");
  k_tree_stats<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(
      lr0_view(ws.lr), n, h->par, h->pre, h->size, h->level, h->inlabel, h->first,
      (engines & ETTG_ENGINE_RMQ) ? h->tkey : nullptr);
  CK_LAUNCH();

  tr.mark("stats");
  // Validation verdict before building the rest (bad input -> no index).
  u32 vflags[8], lerr;
  CK(cudaMemcpyAsync(vflags, ws.flags, sizeof vflags, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(&lerr, ws.lr.counters + LrCounters::kErr, sizeof lerr,
                     cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (vflags[0] & kVRootParent) einval("root has no kNone parent entry");
  if (vflags[0] & kVRange) einval("parent id out of range");
  if (vflags[0] & kVRoots) einval("tree must have exactly one root");
  if (lerr & kErrStructure) einval("cycle in parent array");
  if (lerr & kErrCapacity) throw Error(ETTG_EINTERNAL, "list ranking: splitter capacity exceeded");

  CK(cudaMemsetAsync(ws.hrec, 0xFF, (static_cast<u64>(n) + 1) * 16, st));
  k_head<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(h->inlabel, h->par, h->level, n,
                                                         ws.hrec, ws.flags + 1);
  CK_LAUNCH();
  k_head_split<<<std::min(g, blocks_for(n + 1, 256)), 256, 0, st>>>(ws.hrec, n + 1, h->head,
                                                                    h->lab, ws.up);
  CK_LAUNCH();
  tr.mark("head");
  for (int t = 31 - __builtin_clz(n); t >= 0; --t) {
    const u32 count = ((n >> t) + 1) >> 1;
    k_asc_level<<<std::min(g, blocks_for(count, 256)), 256, 0, st>>>(ws.up, n, t, h->lasc);
    CK_LAUNCH();
  }
  tr.mark("asc");
  k_pack<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(
      h->inlabel, h->level, h->lasc, h->lab, n, h->node, h->node8, h->nodes, ws.flags + 2);
  CK_LAUNCH();
  tr.mark("pack");
  if (engines & ETTG_ENGINE_RMQ) launch_stats_rmq(h.get(), st, sms);
  tr.mark("rmq");
  if (engines & ETTG_ENGINE_NAIVE) {
    k_pack_naive<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(h->par, h->level, n, h->nrec);
    CK_LAUNCH();
  }
  constexpr u32 kLiftSamples = 1u << 16;
  k_lift_sample<<<64, 256, 0, st>>>(h->nodes, n, kLiftSamples, ws.flags + 3);
  CK_LAUNCH();
  // {inlabel paths, max in-path offset, lifts, own lifts, level reads}
  u32 cnt[5] = {0, 0, 0, 0, 0};
  CK(cudaMemcpyAsync(cnt, ws.flags + 1, sizeof cnt, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  h->labels = cnt[0];
  const int label_bits = cnt[0] > 1 ? 32 - __builtin_clz(cnt[0] - 1) : 0;
  h->off_bits = cnt[1] ? 32 - __builtin_clz(cnt[1]) : 0;
  const double own_frac = cnt[2] ? static_cast<double>(cnt[3]) / cnt[2] : 0.0;
  const double level_per_q = static_cast<double>(cnt[4]) / kLiftSamples;
  h->layout = choose_layout(n, cnt[0], label_bits + h->off_bits <= 32, own_frac, level_per_q,
                            device, layout_flags);
  if (h->layout == kLayoutSplitOwn) {  // the wide node array holds the own-lift records
    k_pack_own<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(h->nodes, h->lab, n, h->node);
    CK_LAUNCH();
  }
  if (h->layout == kLayoutWide9) {
    k_pack9<<<std::min(g, blocks_for(n / 3 + 1, 256)), 256, 0, st>>>(h->node, n, h->nodes9);
    CK_LAUNCH();
  }
  if (h->layout == kLayoutSplit6) {
    k_pack6<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(h->nodes, n, h->nodes6);
    CK_LAUNCH();
  }
  if (h->layout == kLayoutCompact) {
    h->alloc_compact();
    scan_exclusive(LabelUsedIn{h->head}, ArrayOut{ws.up}, static_cast<u64>(n) + 1, ws.scan,
                   nullptr, st);
    k_pack_compact<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(
        h->inlabel, h->level, h->head, h->lasc, h->lab, ws.up, n, h->off_bits, h->node4,
        h->ltab);
    CK_LAUNCH();
  }
  CK(cudaEventRecord(e1, st));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  h->build_ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return h.release();
}

void ensure_qbuf(ettg_lca* h, u64 chunk) {
  if (h->qmem && h->qchunk >= chunk) return;
  if (h->qmem) CK(cudaFree(h->qmem));
  h->qmem = nullptr;
  // per stream: pairs (16 B/query) + answers (8 B/query); + 2 error words
  chunk = (chunk + 1) & ~u64(1);
  CK(cudaMalloc(&h->qmem, 2 * chunk * 24 + 256));
  h->qchunk = chunk;
  h->qerr = reinterpret_cast<u32*>(h->qmem + 2 * chunk * 24);
  for (auto& s : h->qs)
    if (!s) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
}

// ETTG_QPF=0 turns the query kernels' pair prefetch off, 1 uses it without the
// compact layout's two-stage pipeline, 2 (default) with it (A/B).
int qprefetch_mode() {
  static const int v = [] {
    const char* e = std::getenv("ETTG_QPF");
    return e ? std::atoi(e) : 2;
  }();
  return v;
}
bool qprefetch() { return qprefetch_mode() != 0; }
// Cache hints on the index gathers (k_lca_inlabel_split6 /
// k_lca_inlabel_compact_pipe kL2): 0 off, 1 L2 evict_last on the node table,
// 2 on all index tables, 3 = 1 plus L1::no_allocate on the compact words,
// 4 = 3 plus L1::no_allocate on the split6 sectors.  A/B
// (profiles/r2_cache_hints.md): config B 101.5 -> 102.8 (1) -> 104.1-104.9
// G q/s (4), config E 68.8 -> 69.4, grasp(64) 41.1 -> 42.1; default 4.
int l2hint_mode() {
  static const int v = [] {
    const char* e = std::getenv("ETTG_L2HINT");
    return e ? std::atoi(e) : 4;
  }();
  return v;
}

template <class In, class Out>
void launch_query(const ettg_lca* h, unsigned engine, In in, Out out, u64 q, u32* err,
                  cudaStream_t st) {
  if (q == 0) return;
  const int sms = sm_count(h->device);
  if (engine == ETTG_ENGINE_NAIVE) {
    if (!h->nrec) einval("index was built without the naive engine");
    unsigned blocks = std::min<u64>((q + kQThreads - 1) / kQThreads, u64(sms) * 16);
    k_lca_naive<In, Out><<<blocks, kQThreads, 0, st>>>(h->nrec, h->n, in, out, q, err);
  } else if (engine == ETTG_ENGINE_RMQ) {
    if (!(h->engines & ETTG_ENGINE_RMQ) || !h->tkey)
      einval("index was built without the RMQ engine");
    RmqView rv{h->tkey, h->pre_in, h->suf_in, h->sp, h->first, h->nb};
    unsigned blocks = std::min<u64>((q + kQThreads - 1) / kQThreads, u64(sms) * 16);
    k_lca_rmq<In, Out><<<blocks, kQThreads, 0, st>>>(rv, h->n, in, out, q, err);
  } else {
    if (!h->lab) einval("index was built without the inlabel engine");
    const u64 per = u64(kQThreads) * kQPer;
    // Small batches (<= 2M queries, L2-resident index): one wave of resident
    // CTAs looping over the batch beats several waves and a ragged tail
    // (config A 1M queries: 44.2 -> 47.7 G q/s); large batches keep the wide
    // grid (config B: 96.5 vs 93.5 G q/s at one wave).
    static const int grid_env = [] {
      const char* e = std::getenv("ETTG_QGRID");
      return e ? std::max(1, std::atoi(e)) : 0;
    }();
    // split6 (sector gathers, DRAM-bound) keeps more CTAs in the grid: 16M
    // grasp(inf) tree, 1G queries 71.2 -> 72.6 G q/s at 128 vs 64 per SM; the
    // other layouts are best at 64 (gpurun_out/r2ak, r2al)
    const int grid_per_sm =
        grid_env ? grid_env
                 : q <= (u64(1) << 21) ? kQMinBlocks
                 : h->layout == kLayoutSplit6 ? 2 * kQGridPerSM : kQGridPerSM;
    unsigned blocks = std::min<u64>((q + per - 1) / per, u64(sms) * grid_per_sm);
    if (h->layout == kLayoutCompact)
      (qprefetch_mode() == 2   ? (l2hint_mode() >= 3 ? k_lca_inlabel_compact_pipe<In, Out, 3>
                                  : l2hint_mode()    ? k_lca_inlabel_compact_pipe<In, Out, 1>
                                                     : k_lca_inlabel_compact_pipe<In, Out, 0>)
       : qprefetch_mode() == 1 ? k_lca_inlabel_compact<In, Out, true>
                               : k_lca_inlabel_compact<In, Out, false>)
          <<<blocks, kQThreads, 0, st>>>(h->node4, h->ltab, h->lab, h->n, h->off_bits, in, out, q,
                                         err);
    else if (h->layout == kLayoutSplitOwn)
      k_lca_inlabel_split_own<In, Out><<<blocks, kQThreads, 0, st>>>(h->node, h->slevel, h->lab,
                                                                     h->n, in, out, q, err);
    else if (h->layout == kLayoutSplit)
      (qprefetch() ? k_lca_inlabel_split<In, Out, true> : k_lca_inlabel_split<In, Out, false>)
          <<<blocks, kQThreads, 0, st>>>(h->nodes, h->slevel, h->lab, h->n, in, out, q, err);
    else if (h->layout == kLayoutWide9)
      (qprefetch() ? k_lca_inlabel<In, Out, Wide9Nodes, true>
                   : k_lca_inlabel<In, Out, Wide9Nodes, false>)<<<blocks, kQThreads, 0, st>>>(
          Wide9Nodes{h->nodes9}, h->lab, h->n, in, out, q, err);
    else if (h->layout == kLayoutSplit6)
      (!qprefetch()          ? k_lca_inlabel_split6<In, Out, false>
       : l2hint_mode() == 2 ? k_lca_inlabel_split6<In, Out, true, 2>
       : l2hint_mode() == 4 ? k_lca_inlabel_split6<In, Out, true, 4>
       : l2hint_mode()      ? k_lca_inlabel_split6<In, Out, true, 1>
                            : k_lca_inlabel_split6<In, Out, true, 0>)
          <<<blocks, kQThreads, 0, st>>>(h->nodes6, h->slevel, h->lab, h->n, in, out, q, err);
    else if (h->layout == kLayoutNarrow)
      (qprefetch() ? k_lca_inlabel_narrow<In, Out, true> : k_lca_inlabel_narrow<In, Out, false>)
          <<<blocks, kQThreads, 0, st>>>(h->node8, h->lasc, h->lab, h->n, in, out, q, err);
    else
      (qprefetch() ? k_lca_inlabel<In, Out, WideNodes, true>
                   : k_lca_inlabel<In, Out, WideNodes, false>)<<<blocks, kQThreads, 0, st>>>(
          WideNodes{h->node}, h->lab, h->n, in, out, q, err);
  }
  CK_LAUNCH();
}

}  // namespace

extern "C" {

int ettg_lca_build(const int64_t* parent, int64_t n, int64_t root, int device, unsigned engines,
                   ettg_lca** out) {
  return guard([&] {
    if (!out || (!parent && n > 0)) einval("null argument");
    *out = nullptr;
    DeviceScope ds(device);
    *out = build_index(parent, true, false, n, root, device, engines, nullptr);
  });
}

int ettg_lca_build_dev(const uint32_t* d_parent, int64_t n, int64_t root, int device,
                       unsigned engines, void* stream, ettg_lca** out) {
  return guard([&] {
    if (!out || !d_parent) einval("null argument");
    *out = nullptr;
    DeviceScope ds(device);
    *out = build_index(d_parent, false, true, n, root, device, engines,
                       static_cast<cudaStream_t>(stream));
  });
}

void ettg_lca_free(ettg_lca* h) {
  if (!h) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(h->device);
  delete h;
  cudaSetDevice(prev);
}

int ettg_lca_size(const ettg_lca* h, int64_t* n) {
  return guard([&] {
    if (!h || !n) einval("null argument");
    *n = h->n;
  });
}

int ettg_lca_device(const ettg_lca* h, int* device) {
  return guard([&] {
    if (!h || !device) einval("null argument");
    *device = h->device;
  });
}

int ettg_lca_build_ms(const ettg_lca* h, double* ms) {
  return guard([&] {
    if (!h || !ms) einval("null argument");
    *ms = h->build_ms;
  });
}

namespace {
// Host int64 pairs -> int64 answers with u32 pairs over the link (8 B per
// query instead of 16).  The host threads narrow chunk c into pinned stage
// buffer c % 3 while the copy engines and the kernel work on the chunks
// before it (two streams).  A pageable answer buffer gets u32 answers (4 B),
// widened by the host threads out of the stage; a pinned one takes the int64
// answers straight from the device (the D2H direction has room for them).
// A B200 host narrows int64 at 70-140 GB/s with 16 threads
// (tools/host_narrow_micro.cpp, tools/stage_micro.cu): at the 54 GB/s link
// the narrowed bytes move in about half the time of the int64 ones.  Ids outside [0, 2^32) are stored as
// 0xFFFFFFFF, which the kernel's range check rejects (ETTG_ERANGE).
void query_host_narrow(ettg_lca* h, unsigned engine, const int64_t* pairs, u64 q,
                       int64_t* answers, bool pairs_pinned, bool answers_pinned) {
  StageLease sl(h->device);
  // stage bytes per query: the u32 pair, plus the u32 answer when the
  // caller's answer buffer is pageable (a pinned one takes the int64
  // answers straight from the device: the D2H direction has room for them)
  const u64 per = (StageLease::bytes() / (answers_pinned ? 8 : 12)) & ~u64(7);
  ensure_qbuf(h, per);
  CK(cudaMemsetAsync(h->qerr, 0, 8, h->qs[0]));
  CK(cudaStreamSynchronize(h->qs[0]));
  const u64 chunks = (q + per - 1) / per;
  // Both buffers pinned: a fraction of the chunks crosses the link as int64
  // straight from the caller's memory (no host work).  Narrowing costs host
  // memory bandwidth (read 16 B, write 8 B, DMA-read 8 B per query) on top
  // of the answers' 8 B; on the B200 host that, not the link, bounds an
  // all-narrowed call.  Config B, 16M queries (tools/ab_rawfrac.py): static
  // raw share 0 -> 4.92-4.98 ms, 0.375 -> 4.51-4.62, 0.5 -> 4.63-4.66, 1 ->
  // 5.04; the best share depends on the host, so by default a chunk goes raw
  // whenever the link has drained the uploads before it (kRawAdaptive).
  const double raw_frac = pairs_pinned && answers_pinned ? raw_fraction(kRawAdaptive) : 0.0;
  RawPolicy pol{raw_frac, nullptr};
  cudaEvent_t up_ev[2] = {nullptr, nullptr};  // the last upload on each stream
  struct EvFree {
    cudaEvent_t* e;
    ~EvFree() {
      for (int i = 0; i < 2; ++i)
        if (e[i]) cudaEventDestroy(e[i]);
    }
  } ev_free{up_ev};
  if (raw_frac != 0)
    for (auto& e : up_ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  const int threads = host_thread_count();
  const char* tr = std::getenv("ETTG_TRACE");
  const bool trace = tr && *tr && *tr != '0';
  double t_wait = 0, t_narrow = 0, t_widen = 0;
  const double t_start = trace ? omp_get_wtime() : 0;
  auto drain = [&](u64 c) {  // chunk c's stage buffer is free again (pageable: widen answers)
    const double t0 = trace ? omp_get_wtime() : 0;
    CK(cudaEventSynchronize(sl.done(c % kStageBufs)));
    if (trace) t_wait += omp_get_wtime() - t0;
    if (answers_pinned) return;
    const double t1 = trace ? omp_get_wtime() : 0;
    const u64 lo = c * per, cnt = std::min(per, q - lo);
    const u32* in = reinterpret_cast<const u32*>(sl.buf(c % kStageBufs) + per * 8);
    host_widen_u32(answers + lo, in, cnt, false, threads);  // streaming stores: no RFO
    if (trace) t_widen += omp_get_wtime() - t1;
  };
  u64 nk = 0;  // narrowed chunks so far (they rotate through the stage)
  for (u64 c = 0; c < chunks; ++c) {
    const int s = c & 1;  // stream and device slot
    const u64 lo = c * per, cnt = std::min(per, q - lo);
    if (raw_frac != 0 && pol.raw_next(c)) {
      cudaStream_t st = h->qs[s];
      char* slot = h->qmem + s * h->qchunk * 24;  // int64 pairs, then int64 answers
      const longlong2* dp = reinterpret_cast<const longlong2*>(slot);
      long long* da = reinterpret_cast<long long*>(slot + h->qchunk * 16);
      CK(cudaMemcpyAsync(slot, pairs + 2 * lo, cnt * 16, cudaMemcpyHostToDevice, st));
      CK(cudaEventRecord(up_ev[s], st));
      pol.last = up_ev[s];
      launch_query(h, engine, PairsI64{dp}, AnsI64{da}, cnt, h->qerr + s, st);
      CK(cudaMemcpyAsync(answers + lo, da, cnt * 8, cudaMemcpyDeviceToHost, st));
      continue;
    }
    const int k = nk % kStageBufs;  // stage buffer
    if (nk >= kStageBufs) drain(nk - kStageBufs);
    ++nk;
    u32* st_pairs = reinterpret_cast<u32*>(sl.buf(k));
    const int64_t* in = pairs + 2 * lo;
    const double t0 = trace ? omp_get_wtime() : 0;
#pragma omp parallel for schedule(static) num_threads(threads) if (cnt > 32768)
    for (long i = 0; i < static_cast<long>(2 * cnt); ++i) {
      const uint64_t v = static_cast<uint64_t>(in[i]);
      st_pairs[i] = v >> 32 ? kNone : static_cast<u32>(v);
    }
    if (trace) t_narrow += omp_get_wtime() - t0;
    cudaStream_t st = h->qs[s];
    const u64 qc = h->qchunk;
    char* slot = h->qmem + s * qc * 24;  // per stream: 8-B pairs, then 4- or 8-B answers
    const uint2* dp = reinterpret_cast<const uint2*>(slot);
    CK(cudaMemcpyAsync(slot, st_pairs, cnt * 8, cudaMemcpyHostToDevice, st));
    if (raw_frac != 0) {
      CK(cudaEventRecord(up_ev[s], st));
      pol.last = up_ev[s];
    }
    if (answers_pinned) {
      CK(cudaEventRecord(sl.done(k), st));  // the stage is free once the pairs landed
      long long* da = reinterpret_cast<long long*>(slot + qc * 8);
      launch_query(h, engine, PairsU32{dp}, AnsI64{da}, cnt, h->qerr + s, st);
      CK(cudaMemcpyAsync(answers + lo, da, cnt * 8, cudaMemcpyDeviceToHost, st));
    } else {
      u32* da = reinterpret_cast<u32*>(slot + qc * 8);
      launch_query(h, engine, PairsU32{dp}, AnsU32{da}, cnt, h->qerr + s, st);
      CK(cudaMemcpyAsync(sl.buf(k) + per * 8, da, cnt * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaEventRecord(sl.done(k), st));
    }
  }
  for (u64 c = nk > kStageBufs ? nk - kStageBufs : 0; c < nk; ++c) drain(c);
  u32 errs[2] = {0, 0};
  CK(cudaStreamSynchronize(h->qs[1]));
  CK(cudaMemcpyAsync(errs, h->qerr, sizeof errs, cudaMemcpyDeviceToHost, h->qs[0]));
  CK(cudaStreamSynchronize(h->qs[0]));
  if (trace)
    std::fprintf(stderr,
                 "[ettg trace] query_host: q=%llu chunks=%llu per=%llu pinned_answers=%d "
                 "narrow=%.3f wait=%.3f widen=%.3f wall=%.3f ms\n",
                 static_cast<unsigned long long>(q), static_cast<unsigned long long>(chunks),
                 static_cast<unsigned long long>(per), answers_pinned ? 1 : 0, t_narrow * 1e3,
                 t_wait * 1e3, t_widen * 1e3, (omp_get_wtime() - t_start) * 1e3);
  if (errs[0] | errs[1]) throw Error(ETTG_ERANGE, "query node id out of range");
}
}  // namespace

int ettg_lca_query_engine(const ettg_lca* hc, unsigned engine, const int64_t* pairs, int64_t q,
                          int64_t batch, int64_t* answers) {
  return guard([&] {
    if (!hc) einval("null handle");
    if (batch < 1) einval("batch_size must be >= 1");
    if (q < 0) einval("negative query count");
    if (q == 0) return;
    if (!pairs || !answers) einval("null argument");
    ettg_lca* h = const_cast<ettg_lca*>(hc);
    DeviceScope ds(h->device);
    std::lock_guard<std::mutex> qlock(h->qmu);
    // both checked (a device pointer in either is a caller error, whatever q)
    const bool pairs_pinned = is_pinned(pairs), answers_pinned = is_pinned(answers);
    if (q >= (1 << 16) && (narrow_enabled() || !(pairs_pinned && answers_pinned))) {
      query_host_narrow(h, engine, pairs, static_cast<u64>(q), answers, pairs_pinned,
                        answers_pinned);
      return;
    }
    // 1M-query chunks on two streams: H2D of chunk c+1 overlaps the kernel and
    // D2H of chunk c; smaller chunks shorten the unoverlapped fill and drain
    // (config B e2e: 4M chunks 5.36 ms, 1M 5.04 ms, 256K 5.37 ms per 16M).
    const u64 chunk = std::min<u64>(static_cast<u64>(q), u64(1) << 20);
    ensure_qbuf(h, chunk);
    CK(cudaMemsetAsync(h->qerr, 0, 8, h->qs[0]));
    CK(cudaStreamSynchronize(h->qs[0]));
    u64 done = 0;
    int c = 0;
    while (done < static_cast<u64>(q)) {
      const u64 cnt = std::min<u64>(chunk, static_cast<u64>(q) - done);
      const int s = c & 1;
      cudaStream_t st = h->qs[s];
      const u64 qc = h->qchunk;  // even (or a single chunk): keeps 16-B alignment
      longlong2* dp = reinterpret_cast<longlong2*>(h->qmem + s * qc * 24);
      long long* da = reinterpret_cast<long long*>(h->qmem + s * qc * 24 + qc * 16);
      CK(cudaMemcpyAsync(dp, pairs + 2 * done, cnt * 16, cudaMemcpyHostToDevice, st));
      launch_query(h, engine, PairsI64{dp}, AnsI64{da}, cnt, h->qerr + s, st);
      CK(cudaMemcpyAsync(answers + done, da, cnt * 8, cudaMemcpyDeviceToHost, st));
      done += cnt;
      ++c;
    }
    u32 errs[2] = {0, 0};
    CK(cudaStreamSynchronize(h->qs[1]));
    CK(cudaMemcpyAsync(errs, h->qerr, sizeof errs, cudaMemcpyDeviceToHost, h->qs[0]));
    CK(cudaStreamSynchronize(h->qs[0]));
    if (errs[0] | errs[1]) throw Error(ETTG_ERANGE, "query node id out of range");
  });
}

int ettg_lca_query(const ettg_lca* h, const int64_t* pairs, int64_t q, int64_t batch,
                   int64_t* answers) {
  return ettg_lca_query_engine(h, ETTG_ENGINE_INLABEL, pairs, q, batch, answers);
}

int ettg_lca_query_dev(const ettg_lca* h, unsigned engine, const uint32_t* d_pairs, int64_t q,
                       uint32_t* d_answers, void* stream) {
  return guard([&] {
    if (!h) einval("null handle");
    if (q < 0) einval("negative query count");
    if (q == 0) return;
    if (!d_pairs || !d_answers) einval("null argument");
    DeviceScope ds(h->device);
    ettg_lca* hm = const_cast<ettg_lca*>(h);
    std::call_once(hm->derr_once, [&] {
      CK(cudaMalloc(&hm->derr, 256));
      CK(cudaMemset(hm->derr, 0, 256));
    });
    if (!hm->derr) throw Error(ETTG_ECUDA, "query error word allocation failed earlier");
    launch_query(h, engine ? engine : ETTG_ENGINE_INLABEL,
                 PairsU32{reinterpret_cast<const uint2*>(d_pairs)}, AnsU32{d_answers},
                 static_cast<u64>(q), hm->derr, static_cast<cudaStream_t>(stream));
  });
}

int ettg_lca_query_dev_error(const ettg_lca* h, void* stream, int* bad) {
  return guard([&] {
    if (!h || !bad) einval("null argument");
    *bad = 0;
    if (!h->derr) return;
    DeviceScope ds(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    u32 v = 0;
    CK(cudaMemcpyAsync(&v, h->derr, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemsetAsync(h->derr, 0, 4, st));
    CK(cudaStreamSynchronize(st));
    *bad = v != 0;
  });
}

namespace {
void copy_widen(int64_t* dst, const u32* src, u64 count, cudaStream_t st) {
  if (!dst) return;
  int device = 0;
  CK(cudaGetDevice(&device));
  staged_d2h_widen_u32(dst, src, count, device, st);
}
}  // namespace

int ettg_lca_stats(const ettg_lca* h, int64_t* preorder, int64_t* size, int64_t* level,
                   int64_t* parent) {
  return guard([&] {
    if (!h) einval("null handle");
    if (!h->full) einval("index has no Euler-tour statistics (attached replica or naive-only)");
    DeviceScope ds(h->device);
    copy_widen(preorder, h->pre, h->n, h->stream);
    copy_widen(size, h->size, h->n, h->stream);
    copy_widen(level, h->level, h->n, h->stream);
    copy_widen(parent, h->par, h->n, h->stream);
  });
}

int ettg_lca_inlabel_index(const ettg_lca* h, int64_t* inlabel, uint64_t* ascendant,
                           int64_t* head, int64_t* level, int64_t* parent) {
  return guard([&] {
    if (!h) einval("null handle");
    if (!h->full) einval("index has no exportable inlabel fields (attached replica or naive-only)");
    DeviceScope ds(h->device);
    copy_widen(inlabel, h->inlabel, h->n, h->stream);
    copy_widen(head, h->head, static_cast<u64>(h->n) + 1, h->stream);
    copy_widen(level, h->level, h->n, h->stream);
    copy_widen(parent, h->par, h->n, h->stream);
    if (ascendant) {
      // only the ascendant word of each 16-B node record: a strided D2D copy
      // into scratch, then the staged D2H (host threads widen to u64; an
      // ascendant never has all 32 bits set below 2^31 nodes, so the kNone
      // mapping of the widening cannot apply)
      Lease lease(h->device, h->stream, static_cast<u64>(h->n) * 4);
      u32* tmp = reinterpret_cast<u32*>(lease.base());
      CK(cudaMemcpy2DAsync(tmp, 4, reinterpret_cast<const char*>(h->node) + 4, 16, 4, h->n,
                           cudaMemcpyDeviceToDevice, h->stream));
      copy_widen(reinterpret_cast<int64_t*>(ascendant), tmp, h->n, h->stream);
    }
  });
}

int ettg_ancestor_levels(const int64_t* parent, int64_t n, int64_t root, int device,
                         int64_t* level) {
  return guard([&] {
    if (!parent || !level) einval("null argument");
    DeviceScope ds(device);
    std::unique_ptr<ettg_lca> h(
        build_index(parent, true, false, n, root, device, ETTG_ENGINE_NAIVE, nullptr));
    std::vector<uint2> rec(h->n);
    CK(cudaMemcpyAsync(rec.data(), h->nrec, static_cast<u64>(h->n) * 8, cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
    for (u32 v = 0; v < h->n; ++v) level[v] = rec[v].y;
  });
}

int ettg_lca_layout(const ettg_lca* h, int* layout, int64_t* labels) {
  return guard([&] {
    if (!h) einval("null handle");
    if (!(h->engines & ETTG_ENGINE_INLABEL)) einval("index has no inlabel engine");
    if (layout) *layout = static_cast<int>(h->layout);
    if (labels) *labels = static_cast<int64_t>(h->labels);
  });
}

// Packed replica blob: a 256-B header {magic, layout, n} followed by the
// arrays of the handle's layout, each 256-B aligned (Carver offsets).
namespace {
constexpr u32 kBlobMagic = 0x47545445u;  // "ETTG"
struct BlobView {
  u32* header = nullptr;
  uint4* node = nullptr;
  uint2* node8 = nullptr;
  u32* lasc = nullptr;
  u32* node4 = nullptr;
  uint4* ltab = nullptr;
  uint2* nodes = nullptr;
  uint32_t* nodes6 = nullptr;
  uint32_t* nodes9 = nullptr;
  u32* slevel = nullptr;
  uint2* lab = nullptr;
  size_t bytes = 0;
};
BlobView blob_view(char* base, u32 n, u32 layout, u64 labels) {
  Carver c{base};
  BlobView b;
  b.header = c.take<u32>(64);
  if (layout == kLayoutWide) {
    b.node = c.take<uint4>(n);
  } else if (layout == kLayoutSplitOwn) {
    b.node = c.take<uint4>(n);
    b.slevel = c.take<u32>(n);
  } else if (layout == kLayoutNarrow) {
    b.node8 = c.take<uint2>(n);
    b.lasc = c.take<u32>(static_cast<u64>(n) + 1);
  } else if (layout == kLayoutCompact) {
    b.node4 = c.take<u32>(n);
    b.ltab = c.take<uint4>(labels);
  } else if (layout == kLayoutWide9) {
    b.nodes9 = c.take<uint32_t>(rec9_bytes(n) / 4);
  } else if (layout == kLayoutSplit6) {
    b.nodes6 = c.take<uint32_t>(rec6_bytes(n) / 4);
    b.slevel = c.take<u32>(n);
  } else {
    b.nodes = c.take<uint2>(n);
    b.slevel = c.take<u32>(n);
  }
  b.lab = c.take<uint2>(static_cast<u64>(n) + 1);
  b.bytes = (c.off + 255) & ~size_t(255);
  return b;
}
}  // namespace

int ettg_lca_index_bytes(const ettg_lca* h, int64_t* bytes) {
  return guard([&] {
    if (!h || !bytes) einval("null argument");
    if (!h->lab) einval("index has no inlabel engine");
    *bytes = static_cast<int64_t>(blob_view(nullptr, h->n, h->layout, h->labels).bytes);
  });
}

int ettg_lca_index_export_dev(const ettg_lca* h, void* d_dst, void* stream) {
  return guard([&] {
    if (!h || !d_dst) einval("null argument");
    if (!h->lab) einval("index has no inlabel engine");
    DeviceScope ds(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const u64 n = h->n;
    BlobView b = blob_view(static_cast<char*>(d_dst), h->n, h->layout, h->labels);
    u32 head[8] = {kBlobMagic, h->layout, h->n, static_cast<u32>(h->off_bits),
                   static_cast<u32>(h->labels), 0, 0, 0};
    CK(cudaMemcpyAsync(b.header, head, sizeof head, cudaMemcpyHostToDevice, st));
    if (b.node) CK(cudaMemcpyAsync(b.node, h->node, n * 16, cudaMemcpyDeviceToDevice, st));
    if (b.node8) {
      CK(cudaMemcpyAsync(b.node8, h->node8, n * 8, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(b.lasc, h->lasc, (n + 1) * 4, cudaMemcpyDeviceToDevice, st));
    }
    if (b.node4) {
      CK(cudaMemcpyAsync(b.node4, h->node4, n * 4, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(b.ltab, h->ltab, h->labels * 16, cudaMemcpyDeviceToDevice, st));
    }
    if (b.nodes) CK(cudaMemcpyAsync(b.nodes, h->nodes, n * 8, cudaMemcpyDeviceToDevice, st));
    if (b.nodes6)
      CK(cudaMemcpyAsync(b.nodes6, h->nodes6, rec6_bytes(n), cudaMemcpyDeviceToDevice, st));
    if (b.nodes9)
      CK(cudaMemcpyAsync(b.nodes9, h->nodes9, rec9_bytes(n), cudaMemcpyDeviceToDevice, st));
    if (b.slevel)
      CK(cudaMemcpyAsync(b.slevel, h->slevel, n * 4, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(b.lab, h->lab, (n + 1) * 8, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));  // `head` is a host stack buffer
  });
}

int ettg_lca_index_attach_dev(const void* d_src, int64_t n, int device, void* stream,
                              ettg_lca** out) {
  return guard([&] {
    if (!d_src || !out) einval("null argument");
    if (n <= 0 || n >= (int64_t(1) << 31)) einval("bad node count");
    *out = nullptr;
    DeviceScope ds(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    u32 head[8];
    CK(cudaMemcpyAsync(head, d_src, sizeof head, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (head[0] != kBlobMagic || head[1] > kLayoutWide9 || head[2] != static_cast<u32>(n) ||
        head[3] > 32 || head[4] > static_cast<u32>(n))
      einval("not an exported inlabel index of this size");
    auto h = std::make_unique<ettg_lca>();
    h->device = device;
    h->n = static_cast<u32>(n);
    h->engines = ETTG_ENGINE_INLABEL;
    h->full = false;
    h->layout = head[1];
    h->off_bits = static_cast<int>(head[3]);
    h->labels = head[4];
    CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    Carver c;
    h->carve(c);
    CK(cudaMalloc(&h->mem, c.off));
    c = Carver{h->mem};
    h->carve(c);
    if (h->layout == kLayoutCompact) h->alloc_compact();
    BlobView b = blob_view(const_cast<char*>(static_cast<const char*>(d_src)), h->n, h->layout,
                           h->labels);
    const u64 un = h->n;
    if (b.node) CK(cudaMemcpyAsync(h->node, b.node, un * 16, cudaMemcpyDeviceToDevice, st));
    if (b.node8) {
      CK(cudaMemcpyAsync(h->node8, b.node8, un * 8, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(h->lasc, b.lasc, (un + 1) * 4, cudaMemcpyDeviceToDevice, st));
    }
    if (b.node4) {
      CK(cudaMemcpyAsync(h->node4, b.node4, un * 4, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(h->ltab, b.ltab, h->labels * 16, cudaMemcpyDeviceToDevice, st));
    }
    if (b.nodes) CK(cudaMemcpyAsync(h->nodes, b.nodes, un * 8, cudaMemcpyDeviceToDevice, st));
    if (b.nodes6)
      CK(cudaMemcpyAsync(h->nodes6, b.nodes6, rec6_bytes(un), cudaMemcpyDeviceToDevice, st));
    if (b.nodes9)
      CK(cudaMemcpyAsync(h->nodes9, b.nodes9, rec9_bytes(un), cudaMemcpyDeviceToDevice, st));
    if (b.slevel)
      CK(cudaMemcpyAsync(h->slevel, b.slevel, un * 4, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(h->lab, b.lab, (un + 1) * 8, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    *out = h.release();
  });
}

}  // extern "C"
