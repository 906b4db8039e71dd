// Bridges on B200: Tarjan-Vishkin over a GPU spanning forest.
//
// Reference path (core/src/bridges.cpp, all CPU):
//   tv_bridges                 :311-316
//     spanning_tree_hooking    :105-158   min-(component, edge) hooking rounds
//     euler_root_tree          :160-196   sequential O(m) endpoint recovery,
//                                         build_half_edges + linearize + node_stats
//     low_high                 :251-287   2m-slot segmented min/max + 2 segment trees
//     classify                 :301-306   bridge iff low >= pre && high < pre + size
//
// Device pipeline (input: COO edge list, u32 ids; no CSR of the graph is built):
//   spanning  k_cc_hook        lock-free union-find (ECL-CC style CAS hooking
//             k_cc_hook_rest   of roots in one strict order per pass: a sampled
//                              pass, a compress, the rest); a successful CAS
//                              joins two trees, so its edge is a spanning-forest
//                              edge and sets the edge's forest bit
//   euler     k_compact_bits   forest bits -> tree-edge ids (tile counts, one-CTA
//                              scan, write); the count is the connectivity check
//                              (n - 1 tree edges)
//             k_tree_rot       per-vertex rotation lists by atomicExch (no sort:
//                              any rotation gives a valid tour)
//             k_tree_close     rotation lists closed into cycles except the
//                              root's: succ(e) = nxt[twin(e)] = nxt[e ^ 1],
//                              read by the list ranking itself
//             list_rank_core   ranks of the tour rooted at vertex 0
//             k_tv_keys        node key = tour rank of its down half-edge + 2
//                              (order-isomorphic to the preorder; a subtree is
//                              the key range up to its up half-edge), so TV
//                              needs no "#downs before" scan (CK / hybrid still
//                              use k_tour_flags + the StatsOut scan for levels)
//   lowhigh   k_lh_neutral / k_lowhigh_runs (one atomicMin / atomicMax per
//             non-tree edge into the slots of the endpoints' keys, runs of equal
//             first endpoint folded; the reference's other two updates, and its
//             own-preorder seeds, never change the test), k_lh_block_ps (block
//             extrema, one in-block suffix/prefix array, neutral-slot masks),
//             block and superblock sparse tables over the 2n key slots,
//             k_classify_tour writes the bridge mask by input edge id.
//
// The spanning forest may differ from the reference's; bridges are a graph
// property, so the mask cannot (core/include/ett/bridges.hpp:56-58).
#include <algorithm>
#include <cstdlib>
#include <memory>
#include <vector>

#include "api_internal.cuh"
#include "common.cuh"
#include "listrank.cuh"
#include "scan.cuh"
#include "sparse.cuh"
#include "graph.cuh"
#include "trace.cuh"

namespace ettg {

__global__ void k_edges_from_i64(const longlong2* __restrict__ in, u32 m, u32 n,
                                 uint2* __restrict__ out, u32* flags) {
  u32 bad = 0;
  for (u32 e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const longlong2 v = in[e];
    const bool ok = v.x >= 0 && v.y >= 0 && v.x < n && v.y < n;
    bad |= !ok;
    out[e] = ok ? make_uint2(static_cast<u32>(v.x), static_cast<u32>(v.y)) : make_uint2(0, 0);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
}

__global__ void k_iota(u32* __restrict__ a, u32 n) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) a[i] = i;
}

// AdjacencyIndex (core/include/ett/graph.hpp:44-61) -> the COO edge list by
// edge id.  The slot of vertex v holding neighbour w and edge id e writes
// edges[e] = (v, w) when v <= w: each edge is written by the slot of its
// lower endpoint (both slots of a self-loop write the same pair), so the
// reference's EdgeList is recovered exactly (build_adjacency keeps each
// edge's (u, v) orientation only up to min/max, which tv_bridges never
// reads).  Eight lanes per vertex stride over its slots (degree ~16 on the
// road-like configs).  edges[] must be preset to 0xFF: an id no slot writes
// stays out of range and fails the endpoint check downstream; decreasing
// offsets raise flags[0].
__global__ void k_csr_coo(const u32* __restrict__ off, const u32* __restrict__ nbr,
                          const u32* __restrict__ eid, u32 n, uint2* __restrict__ edges,
                          u32* flags) {
  const u32 sub = threadIdx.x & 7;
  u32 bad = 0;
  for (u64 v = (u64(blockIdx.x) * blockDim.x + threadIdx.x) >> 3; v < n;
       v += (u64(gridDim.x) * blockDim.x) >> 3) {
    const u32 a = off[v], b = off[v + 1];
    bad |= a > b;
    for (u32 s = a + sub; s < b; s += 8) {
      const u32 w = nbr[s];
      if (static_cast<u32>(v) <= w) edges[eid[s]] = make_uint2(static_cast<u32>(v), w);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
}

// 0/1 mask bytes -> bits (LSB first), one 32-edge word per thread from two
// 16-B loads; the host-mask D2H then moves m/8 bytes.
__global__ void k_pack_bits(const uint8_t* __restrict__ mask, u32 m, u32* __restrict__ bits) {
  const u32 words = (m + 31) / 32;
  for (u32 w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x) {
    const u64 base = u64(w) * 32;
    u32 x = 0;
    if (base + 32 <= m) {
      const uint4 a = reinterpret_cast<const uint4*>(mask + base)[0];
      const uint4 b = reinterpret_cast<const uint4*>(mask + base)[1];
      const u32 v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const u32 t = v[i] & 0x01010101u;  // one bit per byte -> 4 bits
        x |= ((t * 0x10204080u) >> 28) << (4 * i);
      }
    } else {
      for (u64 i = base; i < m; ++i) x |= static_cast<u32>(mask[i] != 0) << (i - base);
    }
    bits[w] = x;
  }
}

// A caller's spanning-tree mask (char per edge, any non-zero = tree edge) as
// the tree bits the compaction counts: one 32-edge word per thread.
__global__ void k_mask_bits(const uint8_t* __restrict__ in, u32 m, u32* __restrict__ bits) {
  const u32 words = (m + 31) / 32;
  for (u32 w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x) {
    const u64 base = u64(w) * 32;
    u32 x = 0;
    for (u32 i = 0; i < 32 && base + i < m; ++i) x |= static_cast<u32>(in[base + i] != 0) << i;
    bits[w] = x;
  }
}

// Second-pass linking by priority: k_cc_hook_rest hooks a root under the
// root of lower uf_prio (a bijective hash of the id), so the forest stays
// shallow whatever the edge order.  Hooking the larger id under the smaller
// everywhere built a chain through every sampled group's root on an
// id-sorted path (10M-node path, sorted edge list: 5.43 -> 1.91 ms per
// call); the sampled pass keeps the id rule (config D: priority linking in
// both passes cost 3%, in the second only ~1%).  The streamed chunks of a
// host edge list (k_cc_hook<.., kPrio = true>) link by priority too.
// Invariant: every hooking kernel in flight uses ONE strict total order --
// two concurrent kernels with different orders could CAS two roots under
// each other and make uf_find loop -- and uf_prio must stay a bijection
// (mix32 is), so distinct roots never tie.  Kernels on one stream never
// overlap, so consecutive passes may use different orders.
__device__ __forceinline__ u32 uf_prio(u32 x) { return mix32(x); }

// Representative of x, starting from an already loaded cur = par[x].  The
// walk is read-only; only a start vertex that needed >= kShortcutHops hops is
// pointed straight at the root found (a benign race: the old root stays an
// ancestor).  Path halving -- a store at every hop -- made random graphs 10x
// slower (config C hooking 1.96 ms vs 0.21 ms): every find in a giant
// component wrote the same few upper-level entries from all SMs.  A pure
// read-only walk was fastest on C (0.18 ms) but let lattice chains grow on
// road graphs (config D 3.80 vs 2.31 ms); profiles/r1_bridges_tuning.md.
constexpr int kShortcutHops = 8;
__device__ __forceinline__ u32 uf_find_from(u32* par, u32 x, u32 cur) {
  if (cur == x) return x;
  u32 next;
  int hops = 1;
  while ((next = par[cur]) != cur) {
    cur = next;
    ++hops;
  }
  if (hops >= kShortcutHops) par[x] = cur;
  return cur;
}
__device__ __forceinline__ u32 uf_find(u32* par, u32 x) { return uf_find_from(par, x, par[x]); }

// One pass over the edges, kHookE edges per thread: their parent loads and
// first CAS attempts are issued together (the kernel is bound by dependent
// L2 latency, profiles/r1_ncu_bridges.md).  Each edge hooks the root a of one
// endpoint under the root b of the other with CAS, a being the later of the
// two in the kernel's strict total order (ids, or uf_prio with kPrio); on
// failure it retries from the value found.  A CAS only succeeds on a root
// (par[a] == a), so each success unions two distinct trees and exactly
// n - #components edges are marked.  Endpoints are range-checked here (the
// reference's build_adjacency check, core/src/graph.cpp:141-143) so the edge
// list is read once.

// Edge subset of a hooking pass: sample = 1 -> all edges; otherwise phase 0
// takes one group of kGroup consecutive edges out of every `sample` groups and
// phase 1 the others (Afforest-style: hook a sparse sample, compress, then
// most remaining edges find equal roots).  Groups are whole 32-B sectors of
// the 8-B edge array, so phase 0 reads 1/sample of the edge bytes; sampling
// every sample-th single edge touched every sector twice (ncu, config D:
// 2.6 GB DRAM read in each phase).
constexpr u32 kGroup = 4;
// goff: the group of each span phase 0 takes; lead: the leading groups of
// each span that earlier phase-0 rounds took, so phase 1 takes the others
// (ETTG_CC_ROUNDS: one sampled group per round, a compress after each).
struct EdgeSubset {
  u32 m, sample, phase, goff = 0, lead = 1;
  u32 total = 0;  // count(), filled in by launch_hook so the kernels do not loop
  u32 ebase = 0;  // index of edges[0] in the tree bit array (streamed chunks)
  // edges of group g summed over all spans
  __host__ __device__ __forceinline__ u64 group_count(u32 g) const {
    const u64 span = u64(kGroup) * sample;
    const u64 full = m / span, rest = m % span;
    const u64 lo = u64(g) * kGroup;
    const u64 part = rest > lo ? (rest - lo < kGroup ? rest - lo : kGroup) : 0;
    return full * kGroup + part;
  }
  __host__ __device__ __forceinline__ u64 count() const {
    if (sample <= 1) return m;
    if (phase == 0) return group_count(goff);
    u64 c = m;
    for (u32 g = 0; g < lead; ++g) c -= group_count(g);
    return c;
  }
  // phase 1 as (i * magic) >> shift == i / per, exact for i < 2^31
  // (Granlund-Montgomery; m < 2^31); host side: rest_divider()
  __device__ __forceinline__ u64 edge_rest(u64 i, u32 magic, u32 shift) const {
    const u32 span = kGroup * sample, skip = kGroup * lead, per = span - skip,
              j = static_cast<u32>(i);
    const u32 q = static_cast<u32>((static_cast<u64>(j) * magic) >> shift);
    return u64(q) * span + skip + (j - q * per);
  }
  void rest_divider(u32& magic, u32& shift) const {
    const u64 per = u64(kGroup) * (sample - lead);
    u32 l = 0;
    while ((u64(1) << l) < per) ++l;
    shift = 31 + l;
    magic = static_cast<u32>((u64(1) << shift) / per + 1);
  }
  __device__ __forceinline__ u64 edge(u64 i) const {
    if (sample <= 1) return i;
    const u64 span = u64(kGroup) * sample;
    if (phase == 0) return (i / kGroup) * span + u64(goff) * kGroup + (i % kGroup);
    const u64 skip = u64(kGroup) * lead, per = span - skip;  // edges of one span left for phase 1
    return (i / per) * span + skip + (i % per);
  }
};

__global__ void k_cc_compress(u32* par, u32 n) {
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    u32 r = par[v];
    while (par[r] != r) r = par[r];
    par[v] = r;
  }
}

// kCs: the edge stream is loaded with the evict-first (.cs) policy so that it
// does not push the union-find parents out of L2 (ETTG_BR_CS bit 0).
template <class T>
__device__ __forceinline__ T ld_edge(const T* p, bool cs) {
  return cs ? __ldcs(p) : *p;
}

template <int kHookE, int kMinB, bool kPrio = false, bool kCs = false>
__global__ void __launch_bounds__(256, kMinB)
    k_cc_hook(const uint2* __restrict__ edges, EdgeSubset sub, u32 n, u32* par,
              u32* __restrict__ tbits, u32* flags) {
  // 32-bit indices as in k_cc_hook_rest (m < 2^31)
  u32 bad = 0;
  const u32 stride = gridDim.x * blockDim.x;
  const u32 cnt = sub.total;
  const u32 span = kGroup * sub.sample, goff = kGroup * sub.goff;
  const bool sampled0 = sub.sample > 1 && sub.phase == 0;
  u32 eidx[kHookE];
  for (u32 base = blockIdx.x * blockDim.x + threadIdx.x; base < cnt; base += stride * kHookE) {
    uint2 uv[kHookE];
    bool ok[kHookE];
#pragma unroll
    for (int j = 0; j < kHookE; ++j) {
      const u32 i = base + j * stride;
      ok[j] = i < cnt;
      u32 e = 0;
      if (ok[j])
        e = sub.sample <= 1 ? i
            : sampled0      ? (i / kGroup) * span + goff + (i % kGroup)
                            : static_cast<u32>(sub.edge(i));  // phase 1 (ETTG_HOOK_REST=0 only)
      eidx[j] = e;
      uv[j] = ok[j] ? ld_edge(edges + e, kCs) : make_uint2(0, 0);
      if (ok[j] && (uv[j].x >= n || uv[j].y >= n)) {
        bad = 1;
        ok[j] = false;
      }
      if (!ok[j]) uv[j] = make_uint2(0, 0);
    }
    u32 a[kHookE], b[kHookE];
#pragma unroll
    for (int j = 0; j < kHookE; ++j) {
      a[j] = par[uv[j].x];
      b[j] = par[uv[j].y];
    }
#pragma unroll
    for (int j = 0; j < kHookE; ++j) {
      // equal parents => same tree: no find needed (after the compress pass
      // between the phases this settles most phase-1 edges with two loads)
      if (a[j] != b[j]) {
        a[j] = uf_find_from(par, uv[j].x, a[j]);
        b[j] = uf_find_from(par, uv[j].y, b[j]);
        if (kPrio ? uf_prio(a[j]) < uf_prio(b[j]) : a[j] < b[j]) {
          const u32 tmp = a[j];
          a[j] = b[j];
          b[j] = tmp;
        }
      }
    }
    u32 old[kHookE];
#pragma unroll
    for (int j = 0; j < kHookE; ++j)
      old[j] = (ok[j] && a[j] != b[j]) ? atomicCAS(&par[a[j]], a[j], b[j]) : a[j];
#pragma unroll
    for (int j = 0; j < kHookE; ++j) {
      bool t = false;
      if (ok[j] && a[j] != b[j]) {
        if (old[j] == a[j]) {
          t = true;
        } else {  // another thread re-rooted a: retry from what the CAS found
          u32 x = uf_find(par, old[j]), y = uf_find(par, b[j]);
          while (x != y) {
            if (kPrio ? uf_prio(x) < uf_prio(y) : x < y) {
              const u32 tmp = x;
              x = y;
              y = tmp;
            }
            const u32 o = atomicCAS(&par[x], x, y);
            if (o == x) {
              t = true;
              break;
            }
            x = uf_find(par, o);
            y = uf_find(par, y);
          }
        }
      }
      if (t) set_bit(tbits, sub.ebase + eidx[j]);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
}

// Second pass of the sampled hooking (the edges outside the sampled groups):
// the same body as k_cc_hook with i / per as a multiply-shift instead of an
// emulated u64 division per edge.  A separate kernel on purpose: changing
// the shared kernel's index code slowed the sampled pass 2x (see
// profiles/r1_bridges_tuning.md).
template <int kHookE, int kMinB, bool kCs = false>
__global__ void __launch_bounds__(256, kMinB)
    k_cc_hook_rest(const uint2* __restrict__ edges, EdgeSubset sub, u32 n, u32* par,
                   u32* __restrict__ tbits, u32* flags, u32 magic, u32 shift) {
  // 32-bit indices (m < 2^31; the grid is a few waves of resident CTAs): the
  // 64-bit index arithmetic was a large share of this pass's instructions
  u32 bad = 0;
  const u32 stride = gridDim.x * blockDim.x;
  const u32 cnt = sub.total;
  const u32 span = kGroup * sub.sample, skip = kGroup * sub.lead, per = span - skip;
  u32 eidx[kHookE];
  for (u32 base = blockIdx.x * blockDim.x + threadIdx.x; base < cnt; base += stride * kHookE) {
    uint2 uv[kHookE];
    bool ok[kHookE];
#pragma unroll
    for (int j = 0; j < kHookE; ++j) {
      const u32 i = base + j * stride;
      ok[j] = i < cnt;
      const u32 q = static_cast<u32>((static_cast<u64>(i) * magic) >> shift);  // i / per
      const u32 e = ok[j] ? q * span + skip + (i - q * per) : 0u;
      eidx[j] = e;
      uv[j] = ok[j] ? ld_edge(edges + e, kCs) : make_uint2(0, 0);
      if (ok[j] && (uv[j].x >= n || uv[j].y >= n)) {
        bad = 1;
        ok[j] = false;
      }
      if (!ok[j]) uv[j] = make_uint2(0, 0);
    }
    u32 a[kHookE], b[kHookE];
#pragma unroll
    for (int j = 0; j < kHookE; ++j) {
      a[j] = par[uv[j].x];
      b[j] = par[uv[j].y];
    }
#pragma unroll
    for (int j = 0; j < kHookE; ++j) {
      // equal parents => same tree: no find needed (after the compress pass
      // between the phases this settles most phase-1 edges with two loads)
      if (a[j] != b[j]) {
        a[j] = uf_find_from(par, uv[j].x, a[j]);
        b[j] = uf_find_from(par, uv[j].y, b[j]);
        // hook the higher priority value under the lower (the hash only when
        // the parents differ: most second-pass edges stop at equal parents)
        if (uf_prio(a[j]) < uf_prio(b[j])) {
          const u32 tmp = a[j];
          a[j] = b[j];
          b[j] = tmp;
        }
      }
    }
    u32 old[kHookE];
#pragma unroll
    for (int j = 0; j < kHookE; ++j)
      old[j] = (ok[j] && a[j] != b[j]) ? atomicCAS(&par[a[j]], a[j], b[j]) : a[j];
#pragma unroll
    for (int j = 0; j < kHookE; ++j) {
      bool t = false;
      if (ok[j] && a[j] != b[j]) {
        if (old[j] == a[j]) {
          t = true;
        } else {  // another thread re-rooted a: retry from what the CAS found
          u32 x = uf_find(par, old[j]), y = uf_find(par, b[j]);
          while (x != y) {
            if (uf_prio(x) < uf_prio(y)) {
              const u32 tmp = x;
              x = y;
              y = tmp;
            }
            const u32 o = atomicCAS(&par[x], x, y);
            if (o == x) {
              t = true;
              break;
            }
            x = uf_find(par, o);
            y = uf_find(par, y);
          }
        }
      }
      if (t) set_bit(tbits, sub.ebase + eidx[j]);
    }
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
}

__global__ void k_cc_range(const uint2* __restrict__ edges, u32 m, u32 n, u32* flags) {
  u32 bad = 0;
  for (u32 e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const uint2 uv = edges[e];
    bad |= (uv.x >= n) | (uv.y >= n);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flags, 1u);
}

// TV runs from the forest to the mask without a host round trip: the
// endpoint-range flag (words[0]) and the tree-edge count (words[1], which
// must be n - 1) stay on the device.  On a bad input the kernels that index
// by tree edge or key do nothing, and the host raises after its one final
// synchronisation.  Other engines pass abort = nullptr and check on the host.
__device__ __forceinline__ bool tv_abort(const u32* w, u32 n) {
  return w && (w[0] != 0u || w[1] != n - 1);
}

// Tree-edge compaction: tedge[t] = e for the t-th tree edge.
struct TreeOut {
  u32* tedge;
  u32 cap;
  __device__ __forceinline__ void operator()(u64 i, u32 rank) const {
    if (rank < cap) tedge[rank] = static_cast<u32>(i);
  }
};

// Rotation system of the spanning tree without sorting.  Half-edges of tree
// edge t = {u, v}: 2t = (u -> v), 2t+1 = (v -> u).  Each half-edge pushes
// itself onto its source's list with one atomicExch; the list order is the
// (arbitrary, race-dependent) cyclic rotation at that vertex.  Any rotation
// gives a valid Euler tour, and bridges do not depend on it, so this replaces
// the reference's two counting-sort passes (core/src/euler.cpp:58-69) by one
// scattered atomic per half-edge.  The half-edge that found an empty list at
// the root is the last of the root's rotation: the tour is cut before its twin.
// Push half-edge h onto vertex x's rotation list.  When every active lane of
// the warp pushes onto the same vertex (a hub whose edges are contiguous in
// the input, e.g. a source-sorted edge list), the lanes are chained among
// themselves and the warp does one atomicExch instead of 32 serialised ones
// on the hub's head (10M-leaf star: 8.8 -> 2.3 ms).  The check is two warp
// reductions, so bounded-degree graphs keep the plain per-lane atomic (a
// general match_any grouping cost 0.28 ms on config D).  The lane linking to
// an empty list is the list's tail; at the root it is remembered as the last
// half-edge of the root's rotation.
__device__ __forceinline__ void rot_push(u32 active, u32 x, u32 h, u32 root,
                                         u32* __restrict__ head, u32* __restrict__ nxt,
                                         u32* __restrict__ tails, u32* last_root) {
  const int lane = threadIdx.x & 31;
  u32 p;
  bool tail = true;
  if (__reduce_min_sync(active, x) == __reduce_max_sync(active, x)) {
    const int leader = __ffs(active) - 1;
    const u32 above = active & ~((2u << lane) - 1u);  // lanes after mine
    p = 0;
    if (lane == leader) p = atomicExch(&head[x], h);  // the leader's h becomes the head
    p = __shfl_sync(active, p, leader);
    const u32 nh = __shfl_sync(active, h, above ? __ffs(above) - 1 : lane);
    if (above) {
      p = nh;
      tail = false;
    }
  } else {
    p = atomicExch(&head[x], h);
  }
  nxt[h] = p;
  if (tail && p == kNone) {
    tails[x] = h;  // the list's last element: k_tree_close links it to head[x]
    if (x == root) *last_root = h;
  }
}

// (Fetching the next trip's endpoints before this trip's atomics made the
// rotation slower on config D: 0.76-0.77 vs 0.74 ms, gpurun_out/r2aa.)
__global__ void k_tree_rot(const uint2* __restrict__ edges, const u32* __restrict__ tedge, u32 T,
                           u32 root, u32* __restrict__ head, u32* __restrict__ nxt,
                           uint2* __restrict__ tend, u32* __restrict__ tails, u32* last_root,
                           const u32* abort, u32 n) {
  if (tv_abort(abort, n)) return;
  const u32 stride = gridDim.x * blockDim.x;
  for (u32 base = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); base < T; base += stride) {
    const u32 t = base + (threadIdx.x & 31);
    const u32 active = __ballot_sync(0xffffffffu, t < T);
    if (t >= T) continue;
    const uint2 uv = edges[tedge[t]];
    tend[t] = uv;
    rot_push(active, uv.x, 2 * t, root, head, nxt, tails, last_root);
    rot_push(active, uv.y, 2 * t + 1, root, head, nxt, tails, last_root);
  }
}

// Closes every rotation list into a cycle (nxt[tail(x)] = head(x)) except
// the root's, whose open end is the tour's cut.  Then for every half-edge
// succ(e) = nxt[e ^ 1] = next(twin(e)) in the cyclic rotation of e's
// destination (core/src/euler.cpp:85-88, :105), cut before head[root], and
// the list ranking reads the successor straight from nxt[e ^ 1] -- the same
// one dependent load per step, with no successor array to build (round 1
// built it in a separate pass: 0.30 ms and 512 MB of traffic on config D).
// A bad input (abort) leaves nxt unwritten: every link becomes a tail.
__global__ void k_tree_close(const u32* __restrict__ head, const u32* __restrict__ tails, u32 root,
                             u32* __restrict__ nxt, u32 k, const u32* abort, u32 n) {
  const bool off = tv_abort(abort, n);
  const u32 lim = off ? k : n;
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < lim; i += gridDim.x * blockDim.x) {
    if (off) {
      nxt[i] = kNone;
    } else if (i != root) {
      const u32 h = head[i];
      if (h != kNone) nxt[tails[i]] = h;
    }
  }
}

__global__ void k_tree_head(const u32* __restrict__ head, u32 root, const u32* last_root,
                            u32* words, const u32* abort, u32 n) {
  if (tv_abort(abort, n)) {
    words[2] = 0;
    words[3] = kNone;
    return;
  }
  words[2] = head[root];        // tour head: first half-edge of root's rotation
  words[3] = *last_root ^ 1u;   // its tour predecessor: twin of the last one
}

// flags[pos] = (t << 1) | is_down for the half-edge at tour position pos.
// A half-edge is down iff it precedes its twin (core/src/euler.cpp:134-139).
// (Round-1 A/B: also storing the twin position here -- as a second array or
// packed into 8 B -- made this phase slower, 1.5-2.0 vs 1.2 ms on config D,
// than re-gathering the two ranks in the scan epilogue.)
__global__ void k_tour_flags(Lr0View lr, u32 T, u32* __restrict__ flags) {
  const u32 S1 = *lr.d_S1;
  for (u32 t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    u32 r0, r1, d;
    lr.get(2 * t, S1, r0, d);
    lr.get(2 * t + 1, S1, r1, d);
    const u32 k = 2 * T;
    if (r0 < k) flags[r0] = (t << 1) | (r0 < r1 ? 1u : 0u);
    if (r1 < k) flags[r1] = (t << 1) | (r1 < r0 ? 1u : 0u);
  }
}

struct DownIn {
  const u32* flags;
  __device__ __forceinline__ u32 operator()(u64 i) const { return flags[i] & 1u; }
};

// Epilogue of the #downs scan: at a down half-edge (p -> c) at position pos
// with D downs before it, preorder(c) = D + 2, size(c) = (pos(twin) - pos + 1)/2
// (node_stats, core/src/euler.cpp:144-153).  Outputs are preorder-indexed
// (index = preorder - 1) so low/high and classification stream over them.
struct StatsOut {
  const u32* flags;
  const u32* tedge;
  const uint2* tend;
  Lr0View lr;
  u32 n;
  u32* pre_of;         // [n]   node -> preorder
  u32* size_by_pre;    // [n]
  u32* pedge_by_pre;   // [n]   input edge id to the parent
  uint2* rec_of;       // [n]   node -> {parent, level} (hybrid engine), or null
  u32* pedge_of;       // [n]   node -> parent edge (hybrid engine), or null
  __device__ __forceinline__ void operator()(u64 pos, u32 dbefore) const {
    const u32 f = flags[pos];
    if (!(f & 1u)) return;
    const u32 t = f >> 1;
    const u32 S1 = *lr.d_S1;
    u32 r0, r1, d;
    lr.get(2 * t, S1, r0, d);
    lr.get(2 * t + 1, S1, r1, d);
    const u32 e = tedge[t];
    const uint2 uv = tend[t];
    const bool first_is_down = r0 < r1;  // half-edge 2t = (u -> v)
    const u32 child = first_is_down ? uv.y : uv.x;
    const u32 pos_up = first_is_down ? r1 : r0;
    const u32 pre = dbefore + 2;
    if (child < n && pre <= n) {
      pre_of[child] = pre;
      size_by_pre[pre - 1] = (pos_up - static_cast<u32>(pos) + 1) >> 1;
      pedge_by_pre[pre - 1] = e;
      if (rec_of) {  // euler_root_tree's parent / level (core/src/bridges.cpp:184-193)
        rec_of[child] = make_uint2(first_is_down ? uv.x : uv.y,
                                   2 * dbefore - static_cast<u32>(pos) + 1);
        pedge_of[child] = e;
      }
    }
  }
};

__global__ void k_root_stats(u32 root, u32 n, u32* pre_of, u32* size_by_pre, u32* pedge_by_pre,
                             uint2* rec_of, u32* pedge_of) {
  pre_of[root] = 1;
  size_by_pre[0] = n;
  pedge_by_pre[0] = kNone;
  if (rec_of) {
    rec_of[root] = make_uint2(kNone, 0u);
    pedge_of[root] = kNone;
  }
}

// Non-tree edge {u, v} with pre(u) < pre(v): low(v) <- min(., pre(u)) and
// high(u) <- max(., pre(v))  (core/src/bridges.cpp:256-273).  kHookE edges per
// thread so their preorder gathers and extreme reads are in flight together;
// an atomic is issued only when it can change the slot.
template <int kHookE, int kMinB, bool kCheck = true>
__global__ void __launch_bounds__(256, kMinB)
    k_lowhigh_edges(const uint2* __restrict__ edges, const u32* __restrict__ tbits, u32 m,
                    const u32* __restrict__ pre_of, uint2* lh, const u32* abort, u32 n) {
  if (tv_abort(abort, n)) return;
  u32* w = reinterpret_cast<u32*>(lh);  // slot = preorder - 1; .x = low, .y = high
  const u64 stride = static_cast<u64>(gridDim.x) * blockDim.x;
  for (u64 base = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; base < m;
       base += stride * kHookE) {
    uint2 uv[kHookE];
    bool nt[kHookE];
#pragma unroll
    for (int j = 0; j < kHookE; ++j) {
      const u64 e = base + j * stride;
      nt[j] = e < m && !test_bit(tbits, e);
      uv[j] = nt[j] ? edges[e] : make_uint2(0, 0);
    }
    u32 pa[kHookE], pb[kHookE];
#pragma unroll
    for (int j = 0; j < kHookE; ++j) {
      pa[j] = nt[j] ? __ldg(pre_of + uv[j].x) : 0u;
      pb[j] = nt[j] ? __ldg(pre_of + uv[j].y) : 0u;
    }
    u32 cl[kHookE], ch[kHookE];
#pragma unroll
    for (int j = 0; j < kHookE; ++j) {
      if (pa[j] > pb[j]) {
        const u32 t = pa[j];
        pa[j] = pb[j];
        pb[j] = t;
      }
      nt[j] = nt[j] && pa[j] != pb[j];  // a self-loop changes nothing
      if (kCheck) {
        cl[j] = nt[j] ? w[2 * (pb[j] - 1)] : 0u;
        ch[j] = nt[j] ? w[2 * (pa[j] - 1) + 1] : 0xFFFFFFFFu;
      } else {
        cl[j] = nt[j] ? 0xFFFFFFFFu : 0u;
        ch[j] = nt[j] ? 0u : 0xFFFFFFFFu;
      }
    }
#pragma unroll
    for (int j = 0; j < kHookE; ++j) {
      if (cl[j] > pa[j]) atomicMin(&w[2 * (pb[j] - 1)], pa[j]);
      if (ch[j] < pb[j]) atomicMax(&w[2 * (pa[j] - 1) + 1], pb[j]);
    }
  }
}

// The same updates with runs of equal first endpoint combined.  Each thread
// takes kE consecutive edges; edges that share their first endpoint u (a
// source-grouped list: CSR-derived inputs, road-graph files, config D's
// generator) fold their u-side updates -- low(u) from neighbours with smaller
// keys, high(u) from larger ones -- into one filtered read and at most one
// atomic per run, while the v-side update stays per edge.  On inputs without
// runs every edge is its own run (the same work as k_lowhigh_edges).
// (Folding a run that continues into the next lane's chunk into this lane's
// u-side update -- two shuffles per chunk, one atomic pair instead of two --
// spilled at 48 registers and was no faster: 1.68 vs 1.66 ms on config D.)
template <int kE, bool kCs = false, int kMinB = 5>
__global__ void __launch_bounds__(256, kMinB)
    k_lowhigh_runs(const uint2* __restrict__ edges, const u32* __restrict__ tbits, u32 m,
                   const u32* __restrict__ key_of, uint2* lh, const u32* abort, u32 n) {
  static_assert(kE == 8, "vector loads are written for 8 edges per thread");
  if (tv_abort(abort, n)) return;
  u32* w = reinterpret_cast<u32*>(lh);  // slot = key - 1; [2s] = low, [2s + 1] = high
  const u64 nchunk = (static_cast<u64>(m) + kE - 1) / kE;
  const u64 gstride = static_cast<u64>(gridDim.x) * blockDim.x;
  auto load_chunk = [&](u64 cc, uint4* dst) {
    if ((cc + 1) * kE <= m) {
      const uint4* e4 = reinterpret_cast<const uint4*>(edges + cc * kE);
#pragma unroll
      for (int j = 0; j < kE / 2; ++j) dst[j] = kCs ? __ldcs(e4 + j) : __ldg(e4 + j);
    }
  };
  for (u64 c = static_cast<u64>(blockIdx.x) * blockDim.x + threadIdx.x; c < nchunk;
       c += gstride) {
    const u64 e0 = c * kE;
    uint2 uv[kE];
    bool nt[kE];
    if (e0 + kE <= m) {
      uint4 cv[kE / 2];
      load_chunk(c, cv);
#pragma unroll
      for (int j = 0; j < kE / 2; ++j) {
        const uint4 v = cv[j];
        uv[2 * j] = make_uint2(v.x, v.y);
        uv[2 * j + 1] = make_uint2(v.z, v.w);
      }
      // the 8 tree bits of this chunk: byte (e0 & 31) / 8 of its word
      const u32 f = __ldg(tbits + (e0 >> 5)) >> (e0 & 31);
#pragma unroll
      for (int j = 0; j < kE; ++j) nt[j] = ((f >> j) & 1u) == 0;
    } else {
#pragma unroll
      for (int j = 0; j < kE; ++j) {
        const bool in = e0 + j < m;
        uv[j] = in ? edges[e0 + j] : make_uint2(0, 0);
        nt[j] = in && !test_bit(tbits, e0 + j);
      }
    }
    u32 ku[kE], kv[kE];
#pragma unroll
    for (int j = 0; j < kE; ++j) {
      ku[j] = __ldg(key_of + uv[j].x);
      kv[j] = nt[j] ? __ldg(key_of + uv[j].y) : 0u;
    }
    // per edge the v-side update (slot word va, value = the key of u); after
    // the last edge of a run, the run's low and high for u (unfiltered:
    // a run's aggregate usually improves its slot)
    u32 va[kE], lv[kE], hv[kE];
    u32 accL = 0xFFFFFFFFu, accH = 0u;
#pragma unroll
    for (int j = 0; j < kE; ++j) {
      va[j] = 0xFFFFFFFFu;
      if (nt[j] && ku[j] != kv[j]) {
        if (kv[j] < ku[j]) {  // low(u) <- kv, high(v) <- ku
          accL = min(accL, kv[j]);
          va[j] = 2 * (kv[j] - 1) + 1;
        } else {              // high(u) <- kv, low(v) <- ku
          accH = max(accH, kv[j]);
          va[j] = 2 * (kv[j] - 1);
        }
      }
      const bool last = j == kE - 1 || uv[j + 1 < kE ? j + 1 : j].x != uv[j].x;
      lv[j] = last ? accL : 0xFFFFFFFFu;
      hv[j] = last ? accH : 0u;
      if (last) {
        accL = 0xFFFFFFFFu;
        accH = 0u;
      }
    }
    // v-side filter reads (low only falls, high only rises: a stale value
    // only lets an unneeded atomic through), then the atomics
    u32 cv[kE];
#pragma unroll
    for (int j = 0; j < kE; ++j) cv[j] = va[j] != 0xFFFFFFFFu ? w[va[j]] : 0u;
#pragma unroll
    for (int j = 0; j < kE; ++j) {
      if (va[j] != 0xFFFFFFFFu) {
        if (va[j] & 1u) {
          if (cv[j] < ku[j]) atomicMax(&w[va[j]], ku[j]);
        } else {
          if (cv[j] > ku[j]) atomicMin(&w[va[j]], ku[j]);
        }
      }
      if (lv[j] != 0xFFFFFFFFu) atomicMin(&w[2 * (ku[j] - 1)], lv[j]);
      if (hv[j] != 0u) atomicMax(&w[2 * (ku[j] - 1) + 1], hv[j]);
    }
  }
}

__device__ __forceinline__ uint2 lh_merge(uint2 a, uint2 b) {
  return make_uint2(min(a.x, b.x), max(a.y, b.y));
}

// Level 0 plus in-block prefix and suffix extrema (32-entry blocks), so a
// range that crosses a block boundary costs two gathers plus the sparse
// table instead of a scan of its partial blocks.  One array holds both: a
// key range [a, b] starts at a vertex's own slot a and ends at the slot b
// of its up half-edge, which never receives an update (neutral), so ps[i]
// is the suffix from i where lh[i] is set and the prefix up to i where it
// is neutral; nmask[block] has a bit per neutral slot.  A range starting at
// a neutral vertex slot takes the suffix from the next set slot of its
// block (k_classify_tour).  Half the stores of separate prefix and suffix
// arrays.
// Four slots per lane (one 32-B load / store), eight lanes per 32-slot
// block: in-lane prefix / suffix, then 3-step segmented shuffles across the
// block's lanes (12 shuffles per lane for 4 slots; one slot per lane needed
// 20 per slot and made the kernel L1/MIO-bound, 0.28 ms on config D).
__global__ void k_lh_block_ps(const uint2* __restrict__ lh, u32 n, u32 nb,
                              uint2* __restrict__ sp0, uint2* __restrict__ ps,
                              u32* __restrict__ nmask) {
  const u32 lane = threadIdx.x & 31, sub = lane & 7;  // lane within its block
  const u32 warps = (gridDim.x * blockDim.x) >> 5;
  const uint2 kNeutral = make_uint2(0xFFFFFFFFu, 0u);
  // a warp covers 4 blocks (128 slots)
  for (u32 w4 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; w4 * 4 < nb; w4 += warps) {
    const u32 i0 = w4 * 128 + lane * 4;  // first of this lane's 4 slots
    uint2 v[4];
    if (i0 + 4 <= n) {
      const uint4 p = reinterpret_cast<const uint4*>(lh + i0)[0];
      const uint4 q = reinterpret_cast<const uint4*>(lh + i0)[1];
      v[0] = make_uint2(p.x, p.y);
      v[1] = make_uint2(p.z, p.w);
      v[2] = make_uint2(q.x, q.y);
      v[3] = make_uint2(q.z, q.w);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) v[j] = i0 + j < n ? lh[i0 + j] : kNeutral;
    }
    // in-lane inclusive prefix / suffix
    uint2 pf[4], sf[4];
    pf[0] = v[0];
#pragma unroll
    for (int j = 1; j < 4; ++j) pf[j] = lh_merge(pf[j - 1], v[j]);
    sf[3] = v[3];
#pragma unroll
    for (int j = 2; j >= 0; --j) sf[j] = lh_merge(sf[j + 1], v[j]);
    // exclusive prefix / suffix of the lane aggregates within the block's 8 lanes
    uint2 ip = pf[3], is = sf[0];  // inclusive over lanes, built by shuffles
#pragma unroll
    for (int d = 1; d < 8; d <<= 1) {
      uint2 o;
      o.x = __shfl_up_sync(0xffffffffu, ip.x, d);
      o.y = __shfl_up_sync(0xffffffffu, ip.y, d);
      if (sub >= static_cast<u32>(d)) ip = lh_merge(ip, o);
      o.x = __shfl_down_sync(0xffffffffu, is.x, d);
      o.y = __shfl_down_sync(0xffffffffu, is.y, d);
      if (sub + d < 8) is = lh_merge(is, o);
    }
    uint2 ep, es;  // exclusive: lanes before / after this one in the block
    ep.x = __shfl_up_sync(0xffffffffu, ip.x, 1);
    ep.y = __shfl_up_sync(0xffffffffu, ip.y, 1);
    es.x = __shfl_down_sync(0xffffffffu, is.x, 1);
    es.y = __shfl_down_sync(0xffffffffu, is.y, 1);
    if (sub == 0) ep = kNeutral;
    if (sub == 7) es = kNeutral;
    u32 nib = 0;
    uint2 o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const bool neutral = v[j].x == 0xFFFFFFFFu && v[j].y == 0u;
      nib |= static_cast<u32>(neutral) << j;
      o[j] = neutral ? lh_merge(ep, pf[j]) : lh_merge(es, sf[j]);
    }
    if (i0 + 4 <= n) {
      reinterpret_cast<uint4*>(ps + i0)[0] = make_uint4(o[0].x, o[0].y, o[1].x, o[1].y);
      reinterpret_cast<uint4*>(ps + i0)[1] = make_uint4(o[2].x, o[2].y, o[3].x, o[3].y);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (i0 + j < n) ps[i0 + j] = o[j];
    }
    // block word: nibble of lane sub at bits 4 * sub (OR over the 8 lanes)
    u32 word = nib << (4 * sub);
#pragma unroll
    for (int d = 1; d < 8; d <<= 1) word |= __shfl_xor_sync(0xffffffffu, word, d);
    const u32 b = w4 * 4 + (lane >> 3);
    if (sub == 7 && b < nb) {
      sp0[b] = ip;  // block aggregate
      nmask[b] = word;
    }
  }
}

struct LhMerge {
  __device__ __forceinline__ uint2 operator()(uint2 a, uint2 b) const { return lh_merge(a, b); }
};

// ---- TV on Euler-tour positions (no preorder scan) -------------------------
// Any DFS numbering in which every subtree is contiguous serves the TV test
// (core/src/bridges.cpp:280-306); the tour itself is one.  Node key K(c) =
// rank(down(c)) + 2 (K(root) = 1) is order-isomorphic to the preorder, and
// c's subtree is exactly the nodes with keys in [K(c), U(c)), U(c) =
// rank(up(c)) + 2.  Low/high slots are indexed by key - 1 over 2n entries
// (up positions stay neutral), so the per-position "#downs before" scan of
// node_stats is not needed: bridge(c) iff low >= K(c) and high < U(c).
__global__ void k_tv_keys(Lr0View lr, u32 T, const uint2* __restrict__ tend, u32 root,
                          u32* __restrict__ key_of, uint2* __restrict__ kt, const u32* abort,
                          u32 n) {
  if (tv_abort(abort, n)) return;
  const u32 S1 = *lr.d_S1;
  for (u32 t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
    u32 r0, r1, d;
    lr.get(2 * t, S1, r0, d);
    lr.get(2 * t + 1, S1, r1, d);
    const uint2 uv = tend[t];
    const bool first_is_down = r0 < r1;  // half-edge 2t = (u -> v)
    const u32 child = first_is_down ? uv.y : uv.x;
    const u32 kd = min(r0, r1) + 2, ku = max(r0, r1) + 2;
    key_of[child] = kd;
    kt[t] = make_uint2(kd, ku);
    if (t == 0) key_of[root] = 1;
  }
}

// tv_bridges_on_tree only: a caller mask of n - 1 edges that is not a
// spanning tree (a cycle plus an unreached vertex, or a self-loop) can still
// yield a closed tour the list ranking accepts, when the cyclic part's
// rotation has a single face.  Then some non-root vertex is the child of no
// tree edge.  So: every non-root vertex must have a key (key_of preset to
// kNone) and the ranking must have succeeded; otherwise words[0] |= 4, which
// stops the later TV kernels (tv_abort) before they index by a bad key.
__global__ void k_tree_check(const u32* __restrict__ key_of, u32 n, u32 root, const u32* lr_err,
                             u32* words) {
  if (tv_abort(words, n)) return;
  bool bad = blockIdx.x == 0 && threadIdx.x == 0 && *lr_err != 0u;
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    bad |= v != root && key_of[v] == kNone;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&words[0], 4u);
}

__global__ void k_lh_neutral(uint2* __restrict__ lh, u32 len) {
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x)
    lh[i] = make_uint2(0xFFFFFFFFu, 0u);
}

// Extrema of the low/high slots [a, b] (b an up slot, so neutral), from the
// per-slot values, the in-block prefix / suffix array, the block sparse table
// and, for the widest rows, the superblock table.
__device__ __forceinline__ uint2 lh_range(const uint2* __restrict__ lh,
                                          const uint2* __restrict__ ps,
                                          const u32* __restrict__ nmask,
                                          const uint2* __restrict__ sp, u32 nb,
                                          const uint2* __restrict__ sps, u32 nsb, u32 a, u32 b) {
  const u32 la = a >> 5, lb = b >> 5;
  uint2 acc;
  if (la == lb) {
    acc = lh[a];
    for (u32 j = a + 1; j <= b; ++j) acc = lh_merge(acc, __ldg(lh + j));
  } else {
    // suffix of block la from a: ps[a], or from the next slot when a's
    // own slot is neutral (then ps[a] is a prefix); prefix of block lb
    // up to b: ps[b] (b is an up slot, always neutral)
    const u32 set = ~__ldg(nmask + la) & (0xFFFFFFFFu << (a & 31u));
    const uint2 sa = set ? __ldg(ps + (la << 5) + (__ffs(set) - 1)) : make_uint2(0xFFFFFFFFu, 0u);
    acc = lh_merge(sa, __ldg(ps + b));
    if (lb > la + 1) {
      constexpr int kTop = st_tile_log<uint2>();  // widest row kept with a superblock table
      const u32 cnt = lb - la - 1;
      const int kk = hb32(cnt);
      if (kk <= kTop || !sps) {
        const uint2* row = sp + static_cast<u64>(kk) * nb;
        acc = lh_merge(acc, lh_merge(row[la + 1], row[lb - (1u << kk)]));
      } else {
        // first and last 2^kTop blocks from the top row, whole superblocks
        // strictly between theirs from the superblock table
        const uint2* row = sp + static_cast<u64>(kTop) * nb;
        acc = lh_merge(acc, lh_merge(row[la + 1], row[lb - (1u << kTop)]));
        const u32 s1 = ((la + 1) >> kTop) + 1, s2e = (lb - 1) >> kTop;  // [s1, s2e)
        if (s1 < s2e) {
          const int k2 = hb32(s2e - s1);
          const uint2* srow = sps + static_cast<u64>(k2) * nsb;
          acc = lh_merge(acc, lh_merge(srow[s1], srow[s2e - (1u << k2)]));
        }
      }
    }
  }
  return acc;
}

__global__ void __launch_bounds__(256)
    k_classify_tour(const uint2* __restrict__ lh, const uint2* __restrict__ ps,
                    const u32* __restrict__ nmask, const uint2* __restrict__ sp, u32 nb,
                    const uint2* __restrict__ sps, u32 nsb, u32 len,
                    const uint2* __restrict__ kt, const u32* __restrict__ tedge, u32 T,
                    uint8_t* __restrict__ mask, u32 m, const u32* abort, u32 n) {
  if (tv_abort(abort, n)) return;
  const u32 stride = gridDim.x * blockDim.x;
  u32 t = blockIdx.x * blockDim.x + threadIdx.x;
  uint2 knext = t < T ? kt[t] : make_uint2(1, 1);
  for (; t < T; t += stride) {
    const uint2 k = knext;  // this trip's key range, loaded one trip ahead
    if (static_cast<u64>(t) + stride < T) knext = kt[t + stride];
    const uint2 acc = lh_range(lh, ps, nmask, sp, nb, sps, nsb, k.x - 1, min(k.y - 1, len - 1));
    // the mask was zeroed before the call: only bridges are stored (a
    // random byte store per tree edge would read-modify-write 32M sectors),
    // and only a bridge reads its input edge id
    if (acc.x >= k.x && acc.y < k.y) {
      const u32 e = tedge[t];
      if (e < m) mask[e] = 1;
    }
  }
}

// ettg_bridges_low_high (diagnostic, not on the timed path): the reference's
// low_high values (core/src/bridges.cpp:251-287) in preorder numbers.  cnt is
// the exclusive count of used key slots (cnt[K - 1] + 1 = preorder of the
// node with key K); a node's subtree holds the keys [K, U), so
// size = cnt[U - 1] - cnt[K - 1].  The slots hold only the updates that can
// move the TV test (k_lowhigh_runs); the reference's remaining ones are the
// node's own preorder, min'd / max'd in here: low = min(pre, slots),
// high = max(pre + size - 1, slots).  Thread T handles the root.
__global__ void k_lh_export(const uint2* __restrict__ lh, const uint2* __restrict__ ps,
                            const u32* __restrict__ nmask, const uint2* __restrict__ sp, u32 nb,
                            const uint2* __restrict__ sps, u32 nsb, u32 len,
                            const uint2* __restrict__ kt, const uint2* __restrict__ tend,
                            const u32* __restrict__ key_of, const u32* __restrict__ cnt, u32 T,
                            u32 root, int64_t* __restrict__ pre_out,
                            int64_t* __restrict__ low_out, int64_t* __restrict__ high_out,
                            const u32* abort, u32 n) {
  if (tv_abort(abort, n)) return;
  for (u32 t = blockIdx.x * blockDim.x + threadIdx.x; t <= T; t += gridDim.x * blockDim.x) {
    uint2 k;
    u32 node, pre, size;
    if (t < T) {
      k = kt[t];
      const uint2 uv = tend[t];
      node = key_of[uv.y] == k.x ? uv.y : uv.x;
      pre = cnt[k.x - 1] + 1;
      size = cnt[k.y - 1] - cnt[k.x - 1];
    } else {
      k = make_uint2(1u, len);
      node = root;
      pre = 1;
      size = n;
    }
    const uint2 acc = lh_range(lh, ps, nmask, sp, nb, sps, nsb, k.x - 1, min(k.y - 1, len - 1));
    const u32 lo = acc.x == 0xFFFFFFFFu ? pre : min(pre, cnt[acc.x - 1] + 1);
    const u32 hi = acc.y == 0u ? pre + size - 1 : max(pre + size - 1, cnt[acc.y - 1] + 1);
    pre_out[node] = pre;
    low_out[node] = lo;
    high_out[node] = hi;
  }
}

__global__ void k_key_used(const u32* __restrict__ key_of, u32 n, u32* __restrict__ used,
                           const u32* abort) {
  if (tv_abort(abort, n)) return;
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (key_of[v] - 1 < 2 * n - 1) used[key_of[v] - 1] = 1u;
}

__global__ void k_bits_to_bytes(const u32* __restrict__ bits, u32 m, uint8_t* __restrict__ out) {
  for (u32 e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x)
    out[e] = (bits[e >> 5] >> (e & 31)) & 1u;
}

// Edge-kernel launch shape: 2 edges per thread at 8 CTAs/SM (<= 32 regs),
// grid = whole waves of resident CTAs from the occupancy API.  A/B on config
// D (tools/trace_bridges.py, profiles/r1_bridges_tuning.md): hooking 2.88 ->
// 2.60 ms, low/high 2.12 -> 1.73 ms vs 4 edges/thread at 48-69 regs on a
// fixed 8-CTA/SM grid (6 resident: a one-third-full second wave).
constexpr int kEdgesPerThread = 2;

template <class K>
unsigned occ_grid(K kern, u64 work, int sms) {
  int per = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 256, 0));
  return static_cast<unsigned>(
      std::min<u64>(blocks_for(work, 256, ~0u), u64(sms) * std::max(per, 1)));
}

// Streamed-edge cache policy: bit 0 hooking, bit 1 low/high.  A/B on config
// D (profiles/r2_cache_hints.md): hooking 2.06 -> 2.00-2.02 ms with bit 0;
// bit 1 changes nothing, so the default is 1.
int br_cs() {
  static const int v = [] {
    const char* e = std::getenv("ETTG_BR_CS");
    return e ? std::atoi(e) : 1;
  }();
  return v;
}

void launch_hook(const uint2* edges, EdgeSubset sub, u32 n, u32* par, u32* tbits, u32* flags,
                 int sms, cudaStream_t st, bool prio = false) {
  sub.total = static_cast<u32>(sub.count());
  const u64 cnt = sub.total;
  bool rest_kernel = sub.sample > 1 && sub.phase == 1;
  if (const char* e = std::getenv("ETTG_HOOK_REST")) rest_kernel &= std::atoi(e) != 0;
  if (rest_kernel) {
    u32 magic = 0, shift = 0;
    sub.rest_divider(magic, shift);
    // (Loading the next trip's edges before this trip's finds -- 1 or 2
    // edges per thread, 6 or 8 CTAs/SM -- did not help: 1.88-2.09 vs 1.89 ms.)
    auto kern = br_cs() & 1 ? k_cc_hook_rest<kEdgesPerThread, 8, true>
                            : k_cc_hook_rest<kEdgesPerThread, 8, false>;
    kern<<<occ_grid(kern, (cnt + kEdgesPerThread - 1) / kEdgesPerThread, sms), 256, 0, st>>>(
        edges, sub, n, par, tbits, flags, magic, shift);
  } else {
    // (Sampled-pass shortcut after 2 / 4 / 16 / no hops instead of 8: config D
    // hooking 1.90 / 1.88 / 2.03 / 2.09 vs 1.91 ms, config C 0.20 / 0.18 /
    // 0.17 / 0.17 vs 0.17 ms; 8 kept, gpurun_out/r2bb.)
    auto kern = br_cs() & 1
                    ? (prio ? k_cc_hook<kEdgesPerThread, 8, true, true>
                            : k_cc_hook<kEdgesPerThread, 8, false, true>)
                    : (prio ? k_cc_hook<kEdgesPerThread, 8, true> : k_cc_hook<kEdgesPerThread, 8, false>);
    kern<<<occ_grid(kern, (cnt + kEdgesPerThread - 1) / kEdgesPerThread, sms), 256, 0, st>>>(
        edges, sub, n, par, tbits, flags);
  }
  CK_LAUNCH();
}

void launch_lowhigh(const uint2* edges, const u32* tbits, u32 m, const u32* pre_of, uint2* lh,
                    const u32* abort, u32 n, int sms, cudaStream_t st) {
  // Read-before-atomic filter: on config D (512 MB of key slots) it skips most
  // atomics (low/high 2.72 -> 1.96 ms); when the slots sit in L2 (config C,
  // 16 MB) the extra loads cost more L2 requests than they save (0.135 vs
  // 0.150 ms), so small slot arrays issue the atomics directly.
  bool check = static_cast<u64>(n) * 16 > (u64(64) << 20);
  if (const char* e = std::getenv("ETTG_LH_CHECK")) check = std::atoi(e) != 0;
  // (A warp-segmented min/max over runs of equal u, one u-side atomic pair
  // per run, cut the L2 reductions 254M -> 148M sectors on config D but
  // doubled the instructions and added reads: 2.37 vs 1.88 ms; round 2.)
  static const bool runs = [] {
    const char* e = std::getenv("ETTG_LH_RUNS");
    return !e || std::atoi(e) != 0;
  }();
  if (runs && check && reinterpret_cast<uintptr_t>(edges) % 16 == 0) {
    // 5 CTAs/SM (48 registers): 1.76 -> 1.67 ms on config D vs 4 at 64
    // registers; 6 spills (profiles/r2_bridges_notes.md)
    auto kr = br_cs() & 2 ? k_lowhigh_runs<8, true> : k_lowhigh_runs<8, false>;
    kr<<<occ_grid(kr, (u64(m) + 7) / 8, sms), 256, 0, st>>>(edges, tbits, m, pre_of, lh, abort, n);
    CK_LAUNCH();
    return;
  }
  auto kern = check ? k_lowhigh_edges<kEdgesPerThread, 8, true>
                    : k_lowhigh_edges<kEdgesPerThread, 8, false>;
  kern<<<occ_grid(kern, (u64(m) + kEdgesPerThread - 1) / kEdgesPerThread, sms), 256, 0, st>>>(
      edges, tbits, m, pre_of, lh, abort, n);
  CK_LAUNCH();
}

// Input of one bridges call: where the graph lives and in which form.
struct BridgeIn {
  enum Kind { kDevU32, kHostI64, kHostCsr } kind = kDevU32;
  const void* edges = nullptr;  // uint2[m] on the device, or int64[2m] on the host
  const int64_t *off = nullptr, *nbr = nullptr, *eid = nullptr;  // kHostCsr
  const uint8_t* tree = nullptr;  // caller spanning tree (tv_bridges_on_tree), or null
  bool tree_on_host = false;
  // kHostI64 from pageable memory: narrowed to u32 by host threads while
  // staging (8 B per edge over the link instead of 16)
  bool narrow = false;
  // ettg_bridges_low_high: host outputs (TV engine; tree_out may be null)
  int64_t *x_pre = nullptr, *x_low = nullptr, *x_high = nullptr;
  uint8_t* x_tree = nullptr;
};

// Host int64 (u, v) pairs -> device u32 pairs with the reference's endpoint
// range check (core/src/graph.cpp:141-143); returns true if one is out of
// range.  Pinned input: one DMA of the int64 pairs and a device narrowing
// pass (e64 is the landing buffer).  Pageable input: narrowed by the host
// threads into the pinned stage, so the link carries 8 B per edge.
bool upload_edges(const int64_t* h, u32 m, u32 n, longlong2* e64, uint2* e, u32* flags,
                  int device, cudaStream_t st) {
  if (!m) return false;
  if (!is_pinned(h) || narrow_enabled()) {
    return staged_h2d_narrow_u32(reinterpret_cast<u32*>(e), h, 2ull * m, n, false, device, st) !=
           0;
  }
  copy_h2d(e64, h, static_cast<u64>(m) * 16, device, st);
  k_edges_from_i64<<<std::min<unsigned>(sm_count(device) * 8, blocks_for(m, 256)), 256, 0, st>>>(
      e64, m, n, e, flags);
  CK_LAUNCH();
  u32 bad = 0;
  read_back(&bad, flags, 4, st);
  return bad != 0;
}

// AdjacencyIndex on the host -> device COO edge list (k_csr_coo); the three
// arrays are narrowed to u32 by the host threads while staging.  Errors are
// the reference's (bad shape, endpoint range) plus "malformed adjacency
// index" for ids the slots do not cover consistently.
struct CsrScratch {
  u32 *off = nullptr, *nbr = nullptr, *eid = nullptr;
  void carve(Carver& c, u32 n, u32 m) {
    off = c.take<u32>(static_cast<u64>(n) + 1);
    nbr = c.take<u32>(2ull * m + 1);
    eid = c.take<u32>(2ull * m + 1);
  }
};
void check_csr_shape(const int64_t* off, i64 n, i64 m) {
  if (!off) einval("null argument");
  if (off[0] != 0 || off[n] != 2 * m) einval("malformed adjacency index: offsets");
}
void upload_csr(const BridgeIn& in, u32 n, u32 m, const CsrScratch& cs, uint2* e, u32* flags,
                int device, cudaStream_t st) {
  if (staged_h2d_narrow_u32(cs.off, in.off, static_cast<u64>(n) + 1, 2ull * m + 1, false, device,
                            st))
    einval("malformed adjacency index: offsets");
  if (m) {
    if (staged_h2d_narrow_u32(cs.nbr, in.nbr, 2ull * m, n, false, device, st))
      einval("edge endpoint out of range");
    if (staged_h2d_narrow_u32(cs.eid, in.eid, 2ull * m, m, false, device, st))
      einval("malformed adjacency index: edge id out of range");
    CK(cudaMemsetAsync(e, 0xFF, static_cast<u64>(m) * 8, st));
  }
  k_csr_coo<<<blocks_for(static_cast<u64>(n) * 8, 256, sm_count(device) * 16), 256, 0, st>>>(
      cs.off, cs.nbr, cs.eid, n, e, flags);
  CK_LAUNCH();
  if (m) {
    k_cc_range<<<std::min<unsigned>(sm_count(device) * 8, blocks_for(m, 256)), 256, 0, st>>>(
        e, m, n, flags);
    CK_LAUNCH();
  }
  u32 bad = 0;
  read_back(&bad, flags, 4, st);
  if (bad) einval("malformed adjacency index");
}

struct BridgeWs {
  longlong2* e64 = nullptr;
  uint2* edges = nullptr;
  CsrScratch csr;
  u32* par = nullptr;
  u32* tbits = nullptr;  // spanning-forest flag per input edge, one bit each
  u64 tbits_bytes = 0;
  u64* scan_m = nullptr;
  u32* tedge = nullptr;
  u32* head = nullptr;
  u32* nxt = nullptr;
  uint2* tend = nullptr;
  u32* tails = nullptr;  // last element of each rotation list
  ListRankWs lr;
  u32* flags = nullptr;
  u64* scan_k = nullptr;
  u32* pre_of = nullptr;
  u32* size_by_pre = nullptr;
  u32* pedge_by_pre = nullptr;
  uint2* lh = nullptr;
  uint2* kt = nullptr;  // TV: (key, up key) per tree edge
  uint2* lh_ps = nullptr;  // TV: in-block suffix (set slots) / prefix (neutral slots) extrema
  u32* lh_nmask = nullptr;  // TV: neutral-slot bits per 32-slot block
  uint2* sp = nullptr;
  u32 nb = 0, levels = 0;
  uint2* sps = nullptr;  // TV: superblock table (build_sparse_rows_super), or null
  u32 nsb = 0, slev = 0;
  u32* words = nullptr;  // [0] edge-range flag, [1] tree-edge count, [2] head
  u32* bits = nullptr;   // the mask packed to bits for a host-mask D2H
  // CK / hybrid
  uint2* rec = nullptr;     // {parent, level} per node
  u32* pedge_of = nullptr;  // parent edge per node
  uint8_t* marked = nullptr;
  u32 *blevel = nullptr, *bparent = nullptr;
  BfsWs bfs;
  int64_t* x3 = nullptr;      // ettg_bridges_low_high: preorder, low, high
  uint8_t* xtree = nullptr;   // ettg_bridges_low_high: tree mask bytes
  void carve(Carver& c, u32 n, u32 m, const BridgeIn& in, int engine) {
    const u32 k = 2 * (n - 1);
    if (engine != ETTG_BRIDGES_TV) {
      rec = c.take<uint2>(n);
      pedge_of = c.take<u32>(n);
      marked = c.take<uint8_t>(n + 16);
    }
    if (engine == ETTG_BRIDGES_CK) {
      blevel = c.take<u32>(n);
      bparent = c.take<u32>(n);
      bfs.carve(c, n, m);
    }
    if (in.kind == BridgeIn::kHostI64 && !in.narrow) e64 = c.take<longlong2>(m);
    if (in.kind != BridgeIn::kDevU32) edges = c.take<uint2>(m);
    if (in.kind == BridgeIn::kHostCsr) csr.carve(c, n, m);
    par = c.take<u32>(n);
    // bits (32 MB on config D, L2-resident) instead of one byte per edge:
    // written by hooking, read by the compaction and low/high
    tbits_bytes = ((static_cast<u64>(m) + 31) / 32 + 4) * 4;
    tbits = c.take<u32>(tbits_bytes / 4);
    scan_m = c.take<u64>(scan_ws_words(m));
    tedge = c.take<u32>(n);
    head = c.take<u32>(n);
    nxt = c.take<u32>(k + 1);
    tend = c.take<uint2>(n);
    tails = c.take<u32>(n);
    // Tour ranks only (no down weights).  Level means 8 / 4 instead of 16 / 16:
    // the level-0 walk of a lattice spanning tree's tour is bound by its
    // tail (the longest sublist, ~L0 ln(k / L0) dependent steps) -- config D
    // walk0 1.19 -> 0.70 ms, list ranking 1.67 -> 1.46 ms
    // (profiles/r2_bridges_notes.md); random trees (the LCA build) keep 16 / 16.
    lr.carve(c, k > 0 ? k : 1, true, 8, 4);
    flags = c.take<u32>(k + 1);
    scan_k = c.take<u64>(scan_ws_words(k + 1));
    pre_of = c.take<u32>(n);
    size_by_pre = c.take<u32>(n);
    pedge_by_pre = c.take<u32>(n);
    const u32 lh_len = engine == ETTG_BRIDGES_TV ? 2 * n : n;
    lh = c.take<uint2>(lh_len);
    if (engine == ETTG_BRIDGES_TV) {
      kt = c.take<uint2>(n);
      lh_ps = c.take<uint2>(lh_len);
      lh_nmask = c.take<u32>((lh_len + 31) / 32);
    }
    nb = (lh_len + 31) / 32;
    levels = 32 - __builtin_clz(nb);
    u32 rows = levels;
    nsb = slev = 0;
    if (engine == ETTG_BRIDGES_TV) {
      st_super_shape<uint2>(nb, nsb, slev);
      if (nsb <= kStSuperMax) {
        rows = std::min<u32>(levels, st_tile_log<uint2>() + 1);
        if (nsb) sps = c.take<uint2>(static_cast<u64>(slev) * nsb);
      } else {
        nsb = slev = 0;
      }
    }
    sp = c.take<uint2>(static_cast<u64>(rows) * nb);
    words = c.take<u32>(16);
    bits = c.take<u32>((static_cast<u64>(m) + 31) / 32 + 1);
    if (in.x_pre) {
      x3 = c.take<int64_t>(3 * static_cast<u64>(n));
      xtree = c.take<uint8_t>(m + 16);
    }
  }
};

void run_bridges(const BridgeIn& in, i64 n64, i64 m64, int device, uint8_t* d_mask_user,
                 uint8_t* h_mask, cudaStream_t st_in, ettg_phase_times* times, int engine) {
  if (n64 <= 0) einval("empty graph");
  if (n64 >= (i64(1) << 31) || m64 >= (i64(1) << 31) || m64 < 0)
    einval("graph too large for packed hooking keys");
  if (engine != ETTG_BRIDGES_TV && engine != ETTG_BRIDGES_CK && engine != ETTG_BRIDGES_HYBRID)
    einval("unknown bridges engine");
  if (in.tree && engine != ETTG_BRIDGES_TV) einval("a caller spanning tree needs the TV engine");
  const bool on_tree = in.tree != nullptr;
  const u32 n = static_cast<u32>(n64), m = static_cast<u32>(m64);
  const int sms = sm_count(device);
  const unsigned g = sms * 8;
  cudaStream_t own = nullptr;
  if (!st_in) CK(cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking));
  cudaStream_t st = st_in ? st_in : own;
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      if (s) cudaStreamDestroy(s);
    }
  } sg{own};

  BridgeWs ws;
  Carver c;
  ws.carve(c, n, m, in, engine);
  uint8_t* d_mask = d_mask_user;
  if (!d_mask) d_mask = c.take<uint8_t>(m + 16);
  Lease lease(device, st, c.off);
  c = Carver{lease.base()};
  ws.carve(c, n, m, in, engine);
  if (!d_mask_user) d_mask = c.take<uint8_t>(m + 16);

  cudaEvent_t ev[4];
  for (auto& e : ev) CK(cudaEventCreate(&e));
  struct EvGuard {
    cudaEvent_t* e;
    ~EvGuard() {
      for (int i = 0; i < 4; ++i) cudaEventDestroy(e[i]);
    }
  } eg{ev};

  CK(cudaEventRecord(ev[0], st));
  Trace tr("bridges", st);
  CK(cudaMemsetAsync(ws.words, 0, 16 * sizeof(u32), st));
  CK(cudaMemsetAsync(ws.tbits, 0, ws.tbits_bytes, st));
  // Copies land in the leased arena: the copy stream is drained before the
  // lease is released (it is declared after the lease, so destroyed first).
  struct CopyGuard {
    cudaStream_t s = nullptr;
    cudaEvent_t e = nullptr;
    ~CopyGuard() {
      if (s) {
        cudaStreamSynchronize(s);
        cudaStreamDestroy(s);
      }
      if (e) cudaEventDestroy(e);
    }
  } copy_guard;
  const uint2* edges;
  bool hooked = false;  // spanning forest hooked while the edge list streamed in
  u32 kChunk = 16u << 20;
  if (const char* e = std::getenv("ETTG_BR_CHUNK")) kChunk = std::max(1, std::atoi(e));
  bool stream_hook = !on_tree && engine != ETTG_BRIDGES_CK && m > 2 * static_cast<u64>(kChunk);
  if (const char* e = std::getenv("ETTG_BR_STREAM")) stream_hook &= std::atoi(e) != 0;
  if (in.kind == BridgeIn::kHostI64 && in.narrow) {
    // Pageable host edge list: the host threads narrow each chunk to u32
    // pairs while filling the pinned stage (8 B per edge over the link); the
    // hooking of a chunk is enqueued behind its copy on the same stream.
    // The copies run on their own stream so that the hooking of chunk c
    // overlaps the copy of chunk c + 1.
    std::function<void(size_t, size_t)> hook_chunk;
    cudaStream_t cs = st;
    if (stream_hook) {
      CK(cudaStreamCreateWithFlags(&copy_guard.s, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&copy_guard.e, cudaEventDisableTiming));
      cs = copy_guard.s;
      CK(cudaEventRecord(ev[1], st));  // the arena lease and words clear come first
      CK(cudaStreamWaitEvent(cs, ev[1], 0));
      k_iota<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(ws.par, n);
      CK_LAUNCH();
      hook_chunk = [&](size_t lo, size_t cnt) {  // lo, cnt in u32 words (pairs: even)
        CK(cudaEventRecord(copy_guard.e, cs));
        CK(cudaStreamWaitEvent(st, copy_guard.e, 0));
        launch_hook(ws.edges + lo / 2,
                    EdgeSubset{static_cast<u32>(cnt / 2), 1, 0, 0, 1, 0, static_cast<u32>(lo / 2)},
                    n, ws.par, ws.tbits, ws.words, sms, st, true);
      };
    }
    // pinned: a chunk goes as int64 (narrowed on the device) whenever the
    // link has caught up with the host narrowing (kRawAdaptive)
    if (m && staged_h2d_narrow_u32(reinterpret_cast<u32*>(ws.edges),
                                   static_cast<const int64_t*>(in.edges), 2ull * m, n, false,
                                   device, cs, hook_chunk, raw_fraction(kRawAdaptive)))
      einval("edge endpoint out of range");
    if (cs != st) {  // everything after the input reads all of it
      CK(cudaEventRecord(copy_guard.e, cs));
      CK(cudaStreamWaitEvent(st, copy_guard.e, 0));
    }
    hooked = stream_hook;
    edges = ws.edges;
  } else if (in.kind == BridgeIn::kHostI64) {
    // Pinned host edge list: the H2D copy dominates an end-to-end call (16 B
    // per edge over PCIe vs ~35 ps of device work), and union-find hooking is
    // incremental, so large inputs arrive in 16M-edge chunks on a copy stream
    // while the previous chunk is converted and hooked (all its edges, no
    // sampling: the sampled two-pass order only matters when hooking is on
    // the critical path).  Any spanning forest gives the same bridge mask.
    const void* edges_in = in.edges;
    if (stream_hook) {
      CK(cudaStreamCreateWithFlags(&copy_guard.s, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&copy_guard.e, cudaEventDisableTiming));
      cudaStream_t cs = copy_guard.s;
      cudaEvent_t arrived = copy_guard.e;
      CK(cudaEventRecord(ev[1], st));  // words cleared before the first chunk lands
      CK(cudaStreamWaitEvent(cs, ev[1], 0));
      k_iota<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(ws.par, n);
      CK_LAUNCH();
      const auto* src = static_cast<const longlong2*>(edges_in);
      for (u32 lo = 0; lo < m; lo += kChunk) {
        const u32 cnt = std::min(kChunk, m - lo);
        copy_h2d(ws.e64 + lo, src + lo, static_cast<u64>(cnt) * 16, device, cs);
        CK(cudaEventRecord(arrived, cs));
        CK(cudaStreamWaitEvent(st, arrived, 0));
        k_edges_from_i64<<<std::min(g, blocks_for(cnt, 256)), 256, 0, st>>>(
            ws.e64 + lo, cnt, n, ws.edges + lo, ws.words);
        CK_LAUNCH();
        launch_hook(ws.edges + lo, EdgeSubset{cnt, 1, 0, 0, 1, 0, lo}, n, ws.par, ws.tbits,
                    ws.words, sms, st, true);
      }
      hooked = true;
    } else if (m) {
      copy_h2d(ws.e64, edges_in, static_cast<u64>(m) * 16, device, st);
      k_edges_from_i64<<<std::min(g, blocks_for(m, 256)), 256, 0, st>>>(ws.e64, m, n, ws.edges,
                                                                        ws.words);
      CK_LAUNCH();
    }
    edges = ws.edges;
  } else if (in.kind == BridgeIn::kHostCsr) {
    upload_csr(in, n, m, ws.csr, ws.edges, ws.words, device, st);
    edges = ws.edges;
  } else {
    edges = static_cast<const uint2*>(in.edges);  // range-checked inside k_cc_hook / below
  }
  if (on_tree) {
    // tv_bridges_on_tree (core/src/bridges.cpp:289-309): the caller's tree
    // replaces hooking.  Its edge count and acyclicity are checked by the
    // tour (count = words[1], cover = the list ranking's error flag).
    if (m) {
      const uint8_t* src = in.tree;
      if (in.tree_on_host) {  // d_mask is cleared below, after the conversion
        copy_h2d(d_mask, in.tree, m, device, st);
        src = d_mask;
      }
      k_mask_bits<<<std::min(g, blocks_for((m + 31) / 32, 256)), 256, 0, st>>>(src, m, ws.tbits);
      CK_LAUNCH();
      if (in.kind == BridgeIn::kDevU32) {
        k_cc_range<<<std::min(g, blocks_for(m, 256)), 256, 0, st>>>(edges, m, n, ws.words);
        CK_LAUNCH();
      }
    }
    hooked = true;
  }
  if (m) CK(cudaMemsetAsync(d_mask, 0, m, st));
  tr.mark("input");
  u32 lerr = 0;
  const u32* abort = nullptr;  // TV: device-side input checks (tv_abort)

  if (engine == ETTG_BRIDGES_CK) {
    // ---- ck_bridges (core/src/bridges.cpp:477-485): BFS tree + marking ----
    // BFS indexes vertices straight from the edge list: check the range first
    if (in.kind == BridgeIn::kDevU32 && m) {
      k_cc_range<<<std::min(g, blocks_for(m, 256)), 256, 0, st>>>(edges, m, n, ws.words);
      CK_LAUNCH();
    }
    u32 bad = 0;
    read_back(&bad, ws.words, 4, st);
    if (bad) einval("edge endpoint out of range");
    const u32 reached = run_bfs(edges, n, m, 0, ws.blevel, ws.bparent, ws.pedge_of, ws.tbits,
                                ws.bfs, st, sms);
    if (reached != n) einval("disconnected graph; extract the largest component first");
    tr.mark("bfs");
    CK(cudaEventRecord(ev[1], st));
    CK(cudaEventRecord(ev[2], st));
    k_pack_rec<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(ws.bparent, ws.blevel, n, ws.rec);
    CK_LAUNCH();
  } else {
    // ---- spanning forest --------------------------------------------------
    if (!hooked) {
      k_iota<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(ws.par, n);
      CK_LAUNCH();
    }
    // CK validates endpoints itself; device input to TV / hybrid is checked by k_cc_hook
    if (m && !hooked) {
      // Hook every 4th edge first, compress, then the rest (round-1 A/B on
      // config D: 3.28 vs 4.02 ms for one pass; ETTG_CC_SAMPLE overrides).
      u32 sample = 4, rounds = 1;
      if (const char* ev = std::getenv("ETTG_CC_SAMPLE")) sample = std::max(1, std::atoi(ev));
      if (const char* ev = std::getenv("ETTG_CC_ROUNDS")) rounds = std::max(1, std::atoi(ev));
      if (sample <= 1) {
        launch_hook(edges, EdgeSubset{m, 1, 0}, n, ws.par, ws.tbits, ws.words, sms, st);
      } else {
        rounds = std::min(rounds, sample - 1);
        for (u32 r = 0; r < rounds; ++r) {
          launch_hook(edges, EdgeSubset{m, sample, 0, r, 1}, n, ws.par, ws.tbits, ws.words, sms,
                      st);
          k_cc_compress<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(ws.par, n);
          CK_LAUNCH();
        }
        launch_hook(edges, EdgeSubset{m, sample, 1, 0, rounds}, n, ws.par, ws.tbits, ws.words, sms,
                    st);
      }
      tr.mark("cc_hook");
    }
    CK(cudaEventRecord(ev[1], st));

    // ---- Euler tour of the forest, rooted at 0 ---------------------------
    compact_bits(ws.tbits, m, TreeOut{ws.tedge, n}, ws.scan_m, ws.words + 1, st);
    const bool tv = engine == ETTG_BRIDGES_TV;
    if (!tv) {
      u32 w[2];
      CK(cudaMemcpyAsync(w, ws.words, sizeof w, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      if (w[0]) einval("edge endpoint out of range");
      if (w[1] != n - 1) einval("disconnected graph; extract the largest component first");
    }
    abort = tv ? ws.words : nullptr;  // TV: checked once at the end
    const u32 T = n - 1;

    if (n > 1) {
      const u32 k = 2 * T;
      CK(cudaMemsetAsync(ws.head, 0xFF, static_cast<u64>(n) * 4, st));
      tr.mark("compact");
      k_tree_rot<<<std::min(g, blocks_for(T, 256)), 256, 0, st>>>(
          edges, ws.tedge, T, 0, ws.head, ws.nxt, ws.tend, ws.tails, ws.words + 4, abort, n);
      CK_LAUNCH();
      k_tree_head<<<1, 1, 0, st>>>(ws.head, 0, ws.words + 4, ws.words, abort, n);
      CK_LAUNCH();
      // head and cut stay on the device (words[2], words[3])
      k_tree_close<<<std::min(g, blocks_for(std::max(n, k), 256)), 256, 0, st>>>(
          ws.head, ws.tails, 0, ws.nxt, k, abort, n);
      CK_LAUNCH();
      tr.mark("rotation");
      list_rank_core_h(k, DevHead{ws.words + 2}, NoDown{}, ws.lr, st, sms, nullptr, ws.nxt);
      tr.mark("list_rank");
      const Lr0View lv = lr0_view(ws.lr);
      if (engine == ETTG_BRIDGES_TV) {
        if (on_tree) CK(cudaMemsetAsync(ws.pre_of, 0xFF, static_cast<u64>(n) * 4, st));
        k_tv_keys<<<std::min(g, blocks_for(T, 256)), 256, 0, st>>>(lv, T, ws.tend, 0,
                                                                   ws.pre_of, ws.kt, abort, n);
        CK_LAUNCH();
        if (on_tree) {
          k_tree_check<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(
              ws.pre_of, n, 0, ws.lr.counters + LrCounters::kErr, ws.words);
          CK_LAUNCH();
        }
        tr.mark("keys");
      } else {
        k_tour_flags<<<std::min(g, blocks_for(T, 256)), 256, 0, st>>>(lv, T, ws.flags);
        CK_LAUNCH();
        scan_exclusive(DownIn{ws.flags},
                       StatsOut{ws.flags, ws.tedge, ws.tend, lv, n, ws.pre_of,
                                ws.size_by_pre, ws.pedge_by_pre, ws.rec, ws.pedge_of},
                       k, ws.scan_k, nullptr, st);
        tr.mark("preorder");
      }
    }
    if (engine != ETTG_BRIDGES_TV || n == 1) {
      k_root_stats<<<1, 1, 0, st>>>(0, n, ws.pre_of, ws.size_by_pre, ws.pedge_by_pre, ws.rec,
                                    ws.pedge_of);
      CK_LAUNCH();
    }
    CK(cudaEventRecord(ev[2], st));
  }

  if (engine == ETTG_BRIDGES_TV) {
    // ---- low / high over tour keys + classification ------------------------
    const u32 len = 2 * n;  // slots key - 1, keys in [1, 2n - 1]
    k_lh_neutral<<<std::min(g, blocks_for(len, 256)), 256, 0, st>>>(ws.lh, len);
    CK_LAUNCH();
    if (m && n > 1) launch_lowhigh(edges, ws.tbits, m, ws.pre_of, ws.lh, abort, n, sms, st);
    tr.mark("lowhigh_edges");
    k_lh_block_ps<<<blocks_for(static_cast<u64>(ws.nb) * 8, 256), 256, 0, st>>>(
        ws.lh, len, ws.nb, ws.sp, ws.lh_ps, ws.lh_nmask);
    CK_LAUNCH();
    if (!build_sparse_rows_super(ws.sp, ws.nb, ws.levels, ws.sps, LhMerge{}, st))
      build_sparse_rows(ws.sp, ws.nb, ws.levels, LhMerge{}, g, st);
    if (n > 1) {
      k_classify_tour<<<std::min(g, blocks_for(n - 1, 256)), 256, 0, st>>>(
          ws.lh, ws.lh_ps, ws.lh_nmask, ws.sp, ws.nb, ws.sps, ws.nsb, len, ws.kt, ws.tedge, n - 1,
          d_mask, m,
          abort, n);
      CK_LAUNCH();
    }
    tr.mark("rmq_classify");
    if (in.x_pre) {  // ettg_bridges_low_high (untimed diagnostic)
      CK(cudaMemsetAsync(ws.flags, 0, (2 * static_cast<u64>(n) - 1) * 4, st));
      k_key_used<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(ws.pre_of, n, ws.flags, abort);
      CK_LAUNCH();
      scan_exclusive(ArrayIn{ws.flags}, ArrayOut{ws.flags}, 2 * static_cast<u64>(n) - 1,
                     ws.scan_k, nullptr, st);
      int64_t* xp = ws.x3;
      k_lh_export<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(
          ws.lh, ws.lh_ps, ws.lh_nmask, ws.sp, ws.nb, ws.sps, ws.nsb, len, ws.kt, ws.tend,
          ws.pre_of, ws.flags, n - 1, 0, xp, xp + n, xp + 2 * static_cast<u64>(n), abort, n);
      CK_LAUNCH();
      if (m) {
        k_bits_to_bytes<<<std::min(g, blocks_for(m, 256)), 256, 0, st>>>(ws.tbits, m, ws.xtree);
        CK_LAUNCH();
      }
    }
  } else {
    // ---- CK marking (core/src/bridges.cpp:40-76) -------------------------
    CK(cudaMemsetAsync(ws.marked, 0, n, st));
    if (m) {
      k_ck_mark<<<std::min(g, blocks_for(m, 256)), 256, 0, st>>>(edges, ws.tbits, m, ws.rec,
                                                                 ws.marked);
      CK_LAUNCH();
    }
    k_ck_classify<<<std::min(g, blocks_for(n, 256)), 256, 0, st>>>(ws.pedge_of, ws.marked, n,
                                                                   d_mask, m);
    CK_LAUNCH();
    tr.mark("marking");
  }
  CK(cudaEventRecord(ev[3], st));
  bool mask_bits = true;
  if (const char* e = std::getenv("ETTG_MASK_BITS")) mask_bits = std::atoi(e) != 0;
  if (h_mask && m && !mask_bits) copy_d2h(h_mask, d_mask, m, device, st);
  if (h_mask && m && mask_bits) {
    // the mask as bits: m/8 bytes over the link, expanded by host threads
    k_pack_bits<<<std::min(g, blocks_for((m + 31) / 32, 256)), 256, 0, st>>>(d_mask, m, ws.bits);
    CK_LAUNCH();
    staged_d2h_expand_bits(h_mask, ws.bits, m, device, st);
  }
  if (n > 1 && engine != ETTG_BRIDGES_CK)
    CK(cudaMemcpyAsync(&lerr, ws.lr.counters + LrCounters::kErr, 4, cudaMemcpyDeviceToHost, st));
  if (in.x_pre) {
    const u64 nb8 = static_cast<u64>(n) * 8;
    CK(cudaMemcpyAsync(in.x_pre, ws.x3, nb8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(in.x_low, ws.x3 + n, nb8, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(in.x_high, ws.x3 + 2 * static_cast<u64>(n), nb8, cudaMemcpyDeviceToHost,
                       st));
    if (in.x_tree && m) CK(cudaMemcpyAsync(in.x_tree, ws.xtree, m, cudaMemcpyDeviceToHost, st));
  }
  u32 w[2] = {0, n - 1};
  if (abort) CK(cudaMemcpyAsync(w, abort, sizeof w, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (w[0] & 1u) einval("edge endpoint out of range");
  if (on_tree) {  // the reference's check_is_tree messages (core/src/euler.cpp:13-33)
    if (w[1] != n - 1) einval("not a tree: m != n - 1");
    if (lerr || (w[0] & 4u)) einval("not a tree: disconnected");
  }
  if (w[1] != n - 1) einval("disconnected graph; extract the largest component first");
  if (lerr) throw Error(ETTG_EINTERNAL, "bridges: spanning-tree tour ranking failed");
  if (times) {
    float a = 0, b = 0, d = 0, tot = 0;
    CK(cudaEventElapsedTime(&a, ev[0], ev[1]));
    CK(cudaEventElapsedTime(&b, ev[1], ev[2]));
    CK(cudaEventElapsedTime(&d, ev[2], ev[3]));
    CK(cudaEventElapsedTime(&tot, ev[0], ev[3]));
    times->spanning_ms = a;
    times->euler_ms = b;
    times->lowhigh_ms = engine == ETTG_BRIDGES_TV ? d : 0.0;
    times->marking_ms = engine == ETTG_BRIDGES_TV ? 0.0 : d;
    times->total_ms = tot;
  }
}

}  // namespace ettg

using namespace ettg;

extern "C" {

int ettg_bridges(const int64_t* edges, int64_t n, int64_t m, int device, uint8_t* is_bridge,
                 ettg_phase_times* times) {
  return ettg_bridges_engine(edges, n, m, device, ETTG_BRIDGES_TV, is_bridge, times);
}

int ettg_bridges_engine(const int64_t* edges, int64_t n, int64_t m, int device, int engine,
                        uint8_t* is_bridge, ettg_phase_times* times) {
  return guard([&] {
    if ((!edges || !is_bridge) && m > 0) einval("null argument");
    DeviceScope ds(device);
    check_host_ptr(is_bridge);
    BridgeIn in;
    in.kind = BridgeIn::kHostI64;
    in.edges = edges;
    in.narrow = m > 0 && (!is_pinned(edges) || narrow_enabled());
    run_bridges(in, n, m, device, nullptr, is_bridge, nullptr, times, engine);
  });
}

int ettg_bridges_dev(const uint32_t* d_edges, int64_t n, int64_t m, int device,
                     uint8_t* d_is_bridge, void* stream, ettg_phase_times* times) {
  return ettg_bridges_dev_engine(d_edges, n, m, device, ETTG_BRIDGES_TV, d_is_bridge, stream,
                                 times);
}

int ettg_bridges_dev_engine(const uint32_t* d_edges, int64_t n, int64_t m, int device,
                            int engine, uint8_t* d_is_bridge, void* stream,
                            ettg_phase_times* times) {
  return guard([&] {
    if ((!d_edges || !d_is_bridge) && m > 0) einval("null argument");
    DeviceScope ds(device);
    BridgeIn in;
    in.edges = d_edges;
    run_bridges(in, n, m, device, d_is_bridge, nullptr, static_cast<cudaStream_t>(stream), times,
                engine);
  });
}

int ettg_bridges_on_tree(const int64_t* edges, int64_t n, int64_t m, int device,
                         const uint8_t* tree_mask, uint8_t* is_bridge, ettg_phase_times* times) {
  return guard([&] {
    if ((!edges || !is_bridge || !tree_mask) && m > 0) einval("null argument");
    DeviceScope ds(device);
    check_host_ptr(is_bridge);
    check_host_ptr(tree_mask);
    BridgeIn in;
    in.kind = BridgeIn::kHostI64;
    in.edges = edges;
    in.narrow = m > 0 && (!is_pinned(edges) || narrow_enabled());
    static const uint8_t kEmpty = 0;
    in.tree = m ? tree_mask : &kEmpty;
    in.tree_on_host = true;
    run_bridges(in, n, m, device, nullptr, is_bridge, nullptr, times, ETTG_BRIDGES_TV);
  });
}

int ettg_bridges_low_high(const int64_t* edges, int64_t n, int64_t m, int device,
                          const uint8_t* tree_mask, uint8_t* tree_out, int64_t* preorder,
                          int64_t* low, int64_t* high) {
  return guard([&] {
    if ((!edges && m > 0) || !preorder || !low || !high) einval("null argument");
    DeviceScope ds(device);
    BridgeIn in;
    in.kind = BridgeIn::kHostI64;
    in.edges = edges;
    in.narrow = m > 0 && (!is_pinned(edges) || narrow_enabled());
    static const uint8_t kEmpty = 0;
    if (tree_mask) {
      check_host_ptr(tree_mask);
      in.tree = m ? tree_mask : &kEmpty;
      in.tree_on_host = true;
    }
    in.x_pre = preorder;
    in.x_low = low;
    in.x_high = high;
    in.x_tree = tree_out;
    run_bridges(in, n, m, device, nullptr, nullptr, nullptr, nullptr, ETTG_BRIDGES_TV);
  });
}

int ettg_bridges_dev_on_tree(const uint32_t* d_edges, int64_t n, int64_t m, int device,
                             const uint8_t* d_tree_mask, uint8_t* d_is_bridge, void* stream,
                             ettg_phase_times* times) {
  return guard([&] {
    if ((!d_edges || !d_is_bridge || !d_tree_mask) && m > 0) einval("null argument");
    DeviceScope ds(device);
    BridgeIn in;
    in.edges = d_edges;
    static const uint8_t kEmpty = 0;
    in.tree = m ? d_tree_mask : &kEmpty;
    run_bridges(in, n, m, device, d_is_bridge, nullptr, static_cast<cudaStream_t>(stream), times,
                ETTG_BRIDGES_TV);
  });
}

int ettg_bridges_csr(const int64_t* offsets, const int64_t* neighbors, const int64_t* edge_ids,
                     int64_t n, int64_t m, int device, int engine, const uint8_t* tree_mask,
                     uint8_t* is_bridge, ettg_phase_times* times) {
  return guard([&] {
    if (n <= 0) einval("empty graph");
    if ((!neighbors || !edge_ids || !is_bridge) && m > 0) einval("null argument");
    if (n >= (int64_t(1) << 31) || m >= (int64_t(1) << 31) || m < 0)
      einval("graph too large for packed hooking keys");
    check_csr_shape(offsets, n, m);
    DeviceScope ds(device);
    check_host_ptr(is_bridge);
    check_host_ptr(tree_mask);
    BridgeIn in;
    in.kind = BridgeIn::kHostCsr;
    in.off = offsets;
    in.nbr = neighbors;
    in.eid = edge_ids;
    static const uint8_t kEmpty = 0;
    if (tree_mask) {  // tv_bridges_on_tree
      in.tree = m ? tree_mask : &kEmpty;
      in.tree_on_host = true;
    }
    run_bridges(in, n, m, device, nullptr, is_bridge, nullptr, times, engine);
  });
}

namespace {
// Host edges -> device u32 pairs with the reference's range check.
struct HostGraph {
  uint2* d = nullptr;
  u32 n = 0, m = 0;
};
}  // namespace

int ettg_build_adjacency(const int64_t* edges, int64_t n, int64_t m, int device,
                         int64_t* offsets, int64_t* neighbors, int64_t* edge_ids) {
  return guard([&] {
    if (n <= 0 || n >= (int64_t(1) << 31) || m < 0 || m >= (int64_t(1) << 31))
      einval("bad graph size");
    if ((!edges && m) || !offsets || (m && (!neighbors || !edge_ids))) einval("null argument");
    DeviceScope ds(device);
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct SG {
      cudaStream_t s;
      ~SG() { cudaStreamDestroy(s); }
    } sg{st};
    const u32 nn = static_cast<u32>(n), mm = static_cast<u32>(m);
    struct Ws {
      longlong2* e64;
      uint2* e;
      u32 *offs, *nbr, *eid, *flags;
      CsrWs csr;
      void carve(Carver& c, u32 n, u32 m) {
        e64 = c.take<longlong2>(m + 1);
        e = c.take<uint2>(m + 1);
        offs = c.take<u32>(static_cast<u64>(n) + 1);
        nbr = c.take<u32>(2ull * m + 1);
        eid = c.take<u32>(2ull * m + 1);
        flags = c.take<u32>(8);
        csr.carve(c, n, m);
      }
    } ws;
    Carver c;
    ws.carve(c, nn, mm);
    Lease lease(device, st, c.off);
    c = Carver{lease.base()};
    ws.carve(c, nn, mm);
    const int sms = sm_count(device);
    CK(cudaMemsetAsync(ws.flags, 0, 32, st));
    if (upload_edges(edges, mm, nn, ws.e64, ws.e, ws.flags, device, st))
      einval("edge endpoint out of range");
    build_csr(ws.e, nn, mm, ws.offs, ws.nbr, ws.eid, ws.csr, st, sms);
    // values < 2^31: the kNone mapping of the widening never applies
    staged_d2h_widen_u32(offsets, ws.offs, static_cast<u64>(nn) + 1, device, st);
    if (mm) {
      staged_d2h_widen_u32(neighbors, ws.nbr, 2ull * mm, device, st);
      staged_d2h_widen_u32(edge_ids, ws.eid, 2ull * mm, device, st);
    }
  });
}

int ettg_largest_component(const int64_t* edges, int64_t n, int64_t m, int device,
                           int64_t* old_to_new, int64_t* n_out, int64_t* m_out,
                           int64_t* edges_out) {
  return guard([&] {
    if (n < 0 || n >= (int64_t(1) << 31) || m < 0 || m >= (int64_t(1) << 31))
      einval("bad graph size");
    if (!n_out || !m_out || (n && !old_to_new) || (m && (!edges || !edges_out)))
      einval("null argument");
    *n_out = 0;
    *m_out = 0;
    if (n == 0) return;
    DeviceScope ds(device);
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    struct SG {
      cudaStream_t s;
      ~SG() { cudaStreamDestroy(s); }
    } sg{st};
    const u32 nn = static_cast<u32>(n), mm = static_cast<u32>(m);
    struct Ws {
      longlong2* e64;
      uint2 *e, *eo;
      u32 *par, *size, *o2n, *flags, *counts;
      unsigned long long* best;
      u64 *sn, *se;
      void carve(Carver& c, u32 n, u32 m) {
        e64 = c.take<longlong2>(m + 1);
        e = c.take<uint2>(m + 1);
        eo = c.take<uint2>(m + 1);
        par = c.take<u32>(n);
        size = c.take<u32>(n);
        o2n = c.take<u32>(n);
        flags = c.take<u32>(8);
        counts = c.take<u32>(8);
        best = c.take<unsigned long long>(1);
        sn = c.take<u64>(scan_ws_words(n));
        se = c.take<u64>(scan_ws_words(m + 1));
      }
    } ws;
    Carver c;
    ws.carve(c, nn, mm);
    Lease lease(device, st, c.off);
    c = Carver{lease.base()};
    ws.carve(c, nn, mm);
    const int sms = sm_count(device);
    const unsigned g = sms * 8;
    CK(cudaMemsetAsync(ws.flags, 0, 32, st));
    CK(cudaMemsetAsync(ws.counts, 0, 32, st));
    CK(cudaMemsetAsync(ws.size, 0, nn * 4ull, st));
    CK(cudaMemsetAsync(ws.best, 0, 8, st));
    if (upload_edges(edges, mm, nn, ws.e64, ws.e, ws.flags, device, st))
      einval("edge endpoint out of range");
    k_iota<<<std::min(g, blocks_for(nn, 256)), 256, 0, st>>>(ws.par, nn);
    CK_LAUNCH();
    if (mm) {
      k_lcc_union<<<std::min(g, blocks_for(mm, 256)), 256, 0, st>>>(ws.e, mm, ws.par);
      CK_LAUNCH();
    }
    k_lcc_sizes<<<std::min(g, blocks_for(nn, 256)), 256, 0, st>>>(ws.par, nn, ws.size);
    CK_LAUNCH();
    k_lcc_best<<<std::min(g, blocks_for(nn, 256)), 256, 0, st>>>(ws.par, ws.size, nn, ws.best);
    CK_LAUNCH();
    scan_exclusive(LccNodeIn{ws.par, ws.best}, LccNodeOut{ws.par, ws.best, ws.o2n}, nn, ws.sn,
                   ws.counts, st);
    scan_exclusive(LccEdgeIn{ws.e, ws.o2n}, LccEdgeOut{ws.e, ws.o2n, ws.eo}, mm, ws.se,
                   ws.counts + 1, st);
    u32 cnt[2];
    CK(cudaMemcpyAsync(cnt, ws.counts, sizeof cnt, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    staged_d2h_widen_u32(old_to_new, ws.o2n, nn, device, st);
    if (cnt[1]) staged_d2h_widen_pairs(edges_out, ws.eo, cnt[1], device, st);
    *n_out = cnt[0];
    *m_out = cnt[1];
  });
}

namespace {
// bfs_tree (core/src/bridges.cpp:198-249) from an EdgeList or an AdjacencyIndex.
void bfs_tree_impl(const BridgeIn& in, int64_t n, int64_t m, int64_t root, int device,
                   uint8_t* tree_mask, int64_t* level, int64_t* parent, int64_t* parent_edge) {
  if (n <= 0 || n >= (int64_t(1) << 31) || m < 0 || m >= (int64_t(1) << 31))
    einval("graph too large for packed hooking keys");
  if (root < 0 || root >= n) einval("root out of range");
  if ((m && !tree_mask) || !level || !parent || !parent_edge) einval("null argument");
  if (in.kind == BridgeIn::kHostCsr) check_csr_shape(in.off, n, m);
  DeviceScope ds(device);
  for (const void* p : {static_cast<const void*>(tree_mask), static_cast<const void*>(level),
                        static_cast<const void*>(parent), static_cast<const void*>(parent_edge)})
    check_host_ptr(p);
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct SG {
    cudaStream_t s;
    ~SG() { cudaStreamDestroy(s); }
  } sg{st};
  const u32 nn = static_cast<u32>(n), mm = static_cast<u32>(m);
  const bool csr = in.kind == BridgeIn::kHostCsr;
  struct Ws {
    longlong2* e64;
    uint2* e;
    u32 *lev, *par, *pe, *flags;
    u32* tbits;
    CsrScratch cs;
    BfsWs bfs;
    void carve(Carver& c, u32 n, u32 m, bool csr) {
      e64 = c.take<longlong2>(m + 1);
      e = c.take<uint2>(m + 1);
      lev = c.take<u32>(n);
      par = c.take<u32>(n);
      pe = c.take<u32>(n);
      flags = c.take<u32>(8);
      tbits = c.take<u32>((static_cast<u64>(m) + 31) / 32 + 4);
      if (csr) cs.carve(c, n, m);
      bfs.carve(c, n, m);
    }
  } ws;
  Carver c;
  ws.carve(c, nn, mm, csr);
  Lease lease(device, st, c.off);
  c = Carver{lease.base()};
  ws.carve(c, nn, mm, csr);
  const int sms = sm_count(device);
  CK(cudaMemsetAsync(ws.flags, 0, 32, st));
  CK(cudaMemsetAsync(ws.tbits, 0, ((static_cast<u64>(mm) + 31) / 32 + 4) * 4, st));
  if (csr) {
    upload_csr(in, nn, mm, ws.cs, ws.e, ws.flags, device, st);
  } else if (upload_edges(static_cast<const int64_t*>(in.edges), mm, nn, ws.e64, ws.e, ws.flags,
                          device, st)) {
    einval("edge endpoint out of range");
  }
  const u32 reached = run_bfs(ws.e, nn, mm, static_cast<u32>(root), ws.lev, ws.par, ws.pe,
                              ws.tbits, ws.bfs, st, sms);
  if (reached != nn) einval("disconnected graph; extract the largest component first");
  staged_d2h_widen_u32(level, ws.lev, nn, device, st);
  staged_d2h_widen_u32(parent, ws.par, nn, device, st);
  staged_d2h_widen_u32(parent_edge, ws.pe, nn, device, st);
  if (mm) staged_d2h_expand_bits(tree_mask, ws.tbits, mm, device, st);
  CK(cudaStreamSynchronize(st));
}
}  // namespace

int ettg_bfs_tree(const int64_t* edges, int64_t n, int64_t m, int64_t root, int device,
                  uint8_t* tree_mask, int64_t* level, int64_t* parent, int64_t* parent_edge) {
  return guard([&] {
    if (!edges && m) einval("null argument");
    BridgeIn in;
    in.kind = BridgeIn::kHostI64;
    in.edges = edges;
    bfs_tree_impl(in, n, m, root, device, tree_mask, level, parent, parent_edge);
  });
}

int ettg_bfs_tree_csr(const int64_t* offsets, const int64_t* neighbors, const int64_t* edge_ids,
                      int64_t n, int64_t m, int64_t root, int device, uint8_t* tree_mask,
                      int64_t* level, int64_t* parent, int64_t* parent_edge) {
  return guard([&] {
    if ((!neighbors || !edge_ids) && m) einval("null argument");
    if (n <= 0) einval("graph too large for packed hooking keys");
    BridgeIn in;
    in.kind = BridgeIn::kHostCsr;
    in.off = offsets;
    in.nbr = neighbors;
    in.eid = edge_ids;
    bfs_tree_impl(in, n, m, root, device, tree_mask, level, parent, parent_edge);
  });
}

}  // extern "C"
