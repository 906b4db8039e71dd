// Graph ingestion and the BFS / Chaitanya-Kothapalli side of the bridges
// comparison, header-only so the bridges TU can
// carve everything from one scratch lease.
//
//   build_csr    build_adjacency (core/src/graph.cpp:135-173): CSR whose
//                slices are sorted by (neighbour, edge id) -- two stable
//                radix sorts of the 2m half-edges (by destination, then by
//                source), so the result is bit-identical to the reference's
//                per-slice std::sort of (neighbour, edge id) pairs.
//   run_bfs      bfs_tree (core/src/bridges.cpp:198-249): level-synchronous
//                BFS; every unvisited neighbour keeps the minimum
//                (parent << 32 | edge id) proposal, exactly the reference's
//                atomic_min_u64 rule, so levels, parents and the tree mask
//                match bit for bit.  Levels run in CUDA-graph chunks (the
//                road-like config has thousands of levels; launch latency,
//                not work, dominates) with one host check per chunk.
//   k_ck_mark    ck_marking (core/src/bridges.cpp:40-64): each non-tree edge
//                walks both endpoints up to their meeting point marking
//                tree edges; unmarked tree edges are bridges (:66-76).
#pragma once

#include "common.cuh"
#include "scan.cuh"
#include "sort.cuh"
#include "trace.cuh"

namespace ettg {
namespace {  // header-defined kernels: internal linkage per TU

// ---- CSR --------------------------------------------------------------------
__global__ void k_he_dst(const uint2* __restrict__ edges, u32 m, u32* __restrict__ keys,
                         u32* __restrict__ vals) {
  for (u32 e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const uint2 uv = edges[e];
    keys[2 * e] = uv.y;  // half-edge 2e = (u -> v), 2e+1 = (v -> u)
    vals[2 * e] = 2 * e;
    keys[2 * e + 1] = uv.x;
    vals[2 * e + 1] = 2 * e + 1;
  }
}

__global__ void k_he_src(const uint2* __restrict__ edges, const u32* __restrict__ vals, u64 k,
                         u32* __restrict__ keys) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < k;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 h = vals[i];
    const uint2 uv = edges[h >> 1];
    keys[i] = (h & 1u) ? uv.y : uv.x;
  }
}

__global__ void k_csr_fill(const uint2* __restrict__ edges, const u32* __restrict__ sval, u64 k,
                           u32* __restrict__ nbr, u32* __restrict__ eid, u32* __restrict__ deg) {
  for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < k;
       i += static_cast<u64>(gridDim.x) * blockDim.x) {
    const u32 h = sval[i];
    const uint2 uv = edges[h >> 1];
    nbr[i] = (h & 1u) ? uv.x : uv.y;
    eid[i] = h >> 1;
    atomicAdd(&deg[(h & 1u) ? uv.y : uv.x], 1u);
  }
}

struct CsrWs {
  u32 *keys = nullptr, *vals = nullptr, *k2 = nullptr, *v2 = nullptr, *deg = nullptr;
  SortWs sort;
  u64* scan = nullptr;
  void carve(Carver& c, u32 n, u32 m) {
    const u64 k = 2ull * m;
    keys = c.take<u32>(k + 1);
    vals = c.take<u32>(k + 1);
    k2 = c.take<u32>(k + 1);
    v2 = c.take<u32>(k + 1);
    sort.carve(c, k + 1);
    deg = c.take<u32>(static_cast<u64>(n) + 1);
    scan = c.take<u64>(scan_ws_words(static_cast<u64>(n) + 1));
  }
};

// offs[n+1], nbr[2m], eid[2m] (u32).  2m must fit in u32.
inline void build_csr(const uint2* edges, u32 n, u32 m, u32* offs, u32* nbr, u32* eid,
                      const CsrWs& ws, cudaStream_t st, int sms) {
  const u32 k = 2 * m;
  const unsigned g = sms * 8;
  CK(cudaMemsetAsync(ws.deg, 0, (static_cast<u64>(n) + 1) * 4, st));
  if (k) {
    k_he_dst<<<std::min(g, blocks_for(m, 256)), 256, 0, st>>>(edges, m, ws.keys, ws.vals);
    CK_LAUNCH();
    const int bits = bits_for(n - 1);
    sort_pairs(ws.keys, ws.vals, ws.k2, ws.v2, k, bits, ws.sort, st);  // by destination
    k_he_src<<<std::min(g, blocks_for(k, 256)), 256, 0, st>>>(edges, ws.v2, k, ws.keys);
    CK_LAUNCH();
    sort_pairs(ws.keys, ws.v2, ws.k2, ws.vals, k, bits, ws.sort, st);  // then by source
    k_csr_fill<<<std::min(g, blocks_for(k, 256)), 256, 0, st>>>(edges, ws.vals, k, nbr, eid,
                                                                ws.deg);
    CK_LAUNCH();
  }
  scan_exclusive(ArrayIn{ws.deg}, ArrayOut{offs}, static_cast<u64>(n) + 1, ws.scan, nullptr, st);
}

// ---- BFS --------------------------------------------------------------------
struct BfsState {
  u32* front[2];
  u32* size;     // [2] frontier sizes (parity), [2] visited count
  u64* cand;
  u32* level;
  u32* parent;
  u32* pedge;
  u32* tbits;  // tree-edge bit per input edge
};

// expand: every unvisited neighbour w of a frontier vertex u keeps the
// minimum (u << 32 | edge id)  (core/src/bridges.cpp:226-233)
__global__ void k_bfs_expand(BfsState s, int p, const u32* __restrict__ offs,
                             const u32* __restrict__ nbr, const u32* __restrict__ eid) {
  const u32 fsize = s.size[p];
  if (blockIdx.x == 0 && threadIdx.x == 0) s.size[1 - p] = 0;  // next frontier starts empty
  const u32* front = s.front[p];
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < fsize; i += gridDim.x * blockDim.x) {
    const u32 u = front[i];
    for (u32 j = offs[u]; j < offs[u + 1]; ++j) {
      const u32 w = nbr[j];
      if (s.level[w] == kNone) atomicMin(reinterpret_cast<unsigned long long*>(&s.cand[w]),
                                         (static_cast<unsigned long long>(u) << 32) | eid[j]);
    }
  }
}

// commit: the winning parent claims w (core/src/bridges.cpp:235-246)
__global__ void k_bfs_commit(BfsState s, int p, const u32* __restrict__ offs,
                             const u32* __restrict__ nbr) {
  const u32 fsize = s.size[p];
  const u32* front = s.front[p];
  u32 added = 0;
  for (u32 i = blockIdx.x * blockDim.x + threadIdx.x; i < fsize; i += gridDim.x * blockDim.x) {
    const u32 u = front[i];
    const u32 lu = s.level[u];
    for (u32 j = offs[u]; j < offs[u + 1]; ++j) {
      const u32 w = nbr[j];
      if (s.level[w] != kNone) continue;
      const u64 c = s.cand[w];
      if (static_cast<u32>(c >> 32) != u) continue;
      if (atomicCAS(&s.level[w], kNone, lu + 1) != kNone) continue;
      s.parent[w] = u;
      s.pedge[w] = static_cast<u32>(c);
      atomicOr(&s.tbits[static_cast<u32>(c) >> 5], 1u << (static_cast<u32>(c) & 31));
      s.front[1 - p][atomicAdd(&s.size[1 - p], 1u)] = w;
      ++added;
    }
  }
  if (added) atomicAdd(&s.size[2], added);
}

// ---- CK marking ---------------------------------------------------------------
// rec[v] = {parent, level}.  Racy duplicate stores of 1 are idempotent
// (core/src/bridges.cpp:40-41).
__global__ void k_ck_mark(const uint2* __restrict__ edges, const u32* __restrict__ tbits,
                          u32 m, const uint2* __restrict__ rec, uint8_t* marked) {
  for (u32 e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    if (test_bit(tbits, e)) continue;
    const uint2 uv = edges[e];
    u32 a = uv.x, b = uv.y;
    if (a == b) continue;
    uint2 ra = rec[a], rb = rec[b];
    while (a != b) {
      if (ra.y > rb.y) {
        marked[a] = 1;
        a = ra.x;
        ra = rec[a];
      } else if (rb.y > ra.y) {
        marked[b] = 1;
        b = rb.x;
        rb = rec[b];
      } else {
        marked[a] = 1;
        marked[b] = 1;
        a = ra.x;
        b = rb.x;
        ra = rec[a];
        rb = rec[b];
      }
    }
  }
}

// unmarked_tree_edges (core/src/bridges.cpp:66-76)
__global__ void k_ck_classify(const u32* __restrict__ pedge, const uint8_t* __restrict__ marked,
                              u32 n, uint8_t* __restrict__ mask, u32 m) {
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    const u32 e = pedge[v];
    if (e < m && !marked[v]) mask[e] = 1;  // zeroed before the call: bridges only
  }
}

__global__ void k_pack_rec(const u32* __restrict__ parent, const u32* __restrict__ level, u32 n,
                           uint2* __restrict__ rec) {
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    rec[v] = make_uint2(parent[v], level[v]);
}

struct BfsWs {
  u32* offs = nullptr;
  u32* nbr = nullptr;
  u32* eid = nullptr;
  CsrWs csr;
  u32* front0 = nullptr;
  u32* front1 = nullptr;
  u32* size = nullptr;
  u64* cand = nullptr;
  void carve(Carver& c, u32 n, u32 m) {
    offs = c.take<u32>(static_cast<u64>(n) + 1);
    nbr = c.take<u32>(2ull * m + 1);
    eid = c.take<u32>(2ull * m + 1);
    csr.carve(c, n, m);
    front0 = c.take<u32>(n);
    front1 = c.take<u32>(n);
    size = c.take<u32>(8);
    cand = c.take<u64>(n);
  }
};

__global__ void k_bfs_init(BfsState s, u32 n, u32 root) {
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    s.level[v] = v == root ? 0u : kNone;
    s.parent[v] = kNone;
    s.pedge[v] = kNone;
    s.cand[v] = ~0ull;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s.front[0][0] = root;
    s.size[0] = 1;
    s.size[1] = 0;
    s.size[2] = 1;  // visited
  }
}

constexpr int kBfsChunk = 16;  // levels per CUDA-graph replay

// Returns the number of vertices reached.  tbits[(m + 31) / 32] must be zeroed by the caller.
inline u32 run_bfs(const uint2* edges, u32 n, u32 m, u32 root, u32* level, u32* parent,
                   u32* pedge, u32* tbits, const BfsWs& ws, cudaStream_t st, int sms) {
  Trace tr("bfs", st);
  build_csr(edges, n, m, ws.offs, ws.nbr, ws.eid, ws.csr, st, sms);
  tr.mark("csr");
  BfsState s{{ws.front0, ws.front1}, ws.size, ws.cand, level, parent, pedge, tbits};
  const unsigned g = std::min<unsigned>(sms * 8, blocks_for(n, 256));
  k_bfs_init<<<g, 256, 0, st>>>(s, n, root);
  CK_LAUNCH();
  // Capture kBfsChunk levels (even/odd parity alternating) once, replay.
  cudaStream_t cap;
  CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  cudaGraph_t graph;
  CK(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
  for (int l = 0; l < kBfsChunk; ++l) {
    k_bfs_expand<<<g, 256, 0, cap>>>(s, l & 1, ws.offs, ws.nbr, ws.eid);
    k_bfs_commit<<<g, 256, 0, cap>>>(s, l & 1, ws.offs, ws.nbr);
  }
  CK(cudaStreamEndCapture(cap, &graph));
  cudaGraphExec_t exec;
  CK(cudaGraphInstantiate(&exec, graph, 0));
  tr.mark("capture");
  u32 sizes[3] = {1, 0, 1};
  u32 chunks = 0;
  for (u32 levels = 0; levels <= n; levels += kBfsChunk) {
    CK(cudaGraphLaunch(exec, st));
    CK(cudaMemcpyAsync(sizes, ws.size, sizeof sizes, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ++chunks;
    if (sizes[0] == 0 && sizes[1] == 0) break;
  }
  tr.mark(chunks > 4 ? "levels(>64)" : "levels");
  cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
  cudaStreamDestroy(cap);
  return sizes[2];
}

// ---- largest_component (core/src/graph.cpp:219-259) ----------------------------
// Union-find with min-id roots (so the reference's tie rule -- smallest
// minimum original id -- is the smaller root), sizes by warp-aggregated
// atomics, argmax by one packed atomicMax, then order-preserving relabel and
// edge compaction with the look-back scan.
__global__ void k_lcc_union(const uint2* __restrict__ edges, u32 m, u32* par) {
  for (u32 e = blockIdx.x * blockDim.x + threadIdx.x; e < m; e += gridDim.x * blockDim.x) {
    const uint2 uv = edges[e];
    u32 a = par[uv.x], b = par[uv.y];
    // find with path halving (par[x] <= x always)
    {
      u32 x = uv.x;
      while (a != x) {
        const u32 g2 = par[a];
        par[x] = g2;
        x = a;
        a = g2;
      }
      a = x;
    }
    {
      u32 x = uv.y;
      while (b != x) {
        const u32 g2 = par[b];
        par[x] = g2;
        x = b;
        b = g2;
      }
      b = x;
    }
    while (a != b) {
      if (a < b) {
        const u32 t = a;
        a = b;
        b = t;
      }
      const u32 old = atomicCAS(&par[a], a, b);
      if (old == a) break;
      a = old;
      while (par[a] != a) a = par[a];
      while (par[b] != b) b = par[b];
    }
  }
}

__global__ void k_lcc_sizes(u32* par, u32 n, u32* size) {
  const u32 lt = lanemask_lt();
  for (u32 base = blockIdx.x * blockDim.x; base < n; base += gridDim.x * blockDim.x) {
    const u32 v = base + threadIdx.x;
    u32 r = kNone;
    if (v < n) {
      r = par[v];
      while (par[r] != r) r = par[r];
      par[v] = r;  // full compression
    }
    const u32 peers = __match_any_sync(0xffffffffu, r);
    if (r != kNone && (peers & lt) == 0) atomicAdd(&size[r], __popc(peers));
  }
}

// best = max over roots of (size << 32 | ~root): larger size, then smaller root.
__global__ void k_lcc_best(const u32* __restrict__ par, const u32* __restrict__ size, u32 n,
                           unsigned long long* best) {
  unsigned long long b = 0;
  for (u32 v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    if (par[v] == v) b = max(b, (static_cast<unsigned long long>(size[v]) << 32) | (~v));
  for (int d = 16; d > 0; d >>= 1) b = max(b, __shfl_xor_sync(0xffffffffu, b, d));
  if ((threadIdx.x & 31) == 0 && b) atomicMax(best, b);
}

struct LccNodeIn {
  const u32* par;
  const unsigned long long* best;
  __device__ __forceinline__ u32 operator()(u64 v) const {
    return par[v] == ~static_cast<u32>(*best) ? 1u : 0u;
  }
};
struct LccNodeOut {
  const u32* par;
  const unsigned long long* best;
  u32* old_to_new;
  __device__ __forceinline__ void operator()(u64 v, u32 rank) const {
    old_to_new[v] = par[v] == ~static_cast<u32>(*best) ? rank : kNone;
  }
};
struct LccEdgeIn {
  const uint2* edges;
  const u32* old_to_new;
  __device__ __forceinline__ u32 operator()(u64 e) const {
    return old_to_new[edges[e].x] != kNone ? 1u : 0u;
  }
};
struct LccEdgeOut {
  const uint2* edges;
  const u32* old_to_new;
  uint2* out;
  __device__ __forceinline__ void operator()(u64 e, u32 rank) const {
    const uint2 uv = edges[e];
    const u32 a = old_to_new[uv.x];
    if (a != kNone) out[rank] = make_uint2(a, old_to_new[uv.y]);
  }
};

}  // namespace
}  // namespace ettg
