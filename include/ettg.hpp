// ettg.hpp -- header-only C++ shim over the C-ABI (ettg.h) with the
// reference's signatures and exceptions, so reference-style callers
// (tools/ett_bench.cpp:93-167, :303-339; tests/acceptance.cpp) can switch by
// changing the namespace:
//
//   ett::inlabel_build(const RootedTree&)        -> ettg::inlabel_build(...)
//   ett::answer_batch(lambda, queries, batch)    -> ettg::answer_batch(idx, queries, batch)
//   ett::rmq_lca_build / rmq_lca                 -> ettg::rmq_lca_build / answer_batch
//   ett::node_stats(linearize(...))              -> ettg::node_stats(tree)
//   ett::tv_bridges(const AdjacencyIndex&, PhaseTimes*) -> ettg::tv_bridges (same signature;
//     also an EdgeList overload), tv_bridges_on_tree, ck_bridges, hybrid_bridges,
//     dfs_bridges (answered by the device CK engine), PhaseTimes{nanos, add()}
//   ett::naive_build / naive_lca                 -> ettg::naive_build / answer_batch
//   ett::ancestor_doubling_levels                -> ettg::ancestor_doubling_levels
//   ett::build_adjacency / bfs_tree / largest_component -> same names
//   ett::parse_edge_list / parse_dimacs_gr (std::istream&) -> same names
//   ett::list_scan / segmented_reduce / RangeIndex, rmq_build/min/max -> same names
//     (segmented_reduce takes ettg::Min / Max / Plus instead of an arbitrary
//     lambda: the combiner runs on the device)
//
// Errors: std::invalid_argument / std::out_of_range exactly where the
// reference throws them (ETTG_EINVAL / ETTG_ERANGE); std::runtime_error for
// parse errors (ETTG_EPARSE, the reference's messages) and CUDA failures.  Link: -I<repo>/include -L<repo>/paper_2103_15217_b200/_lib -lettg
#ifndef ETTG_HPP_
#define ETTG_HPP_

#include <cstdint>
#include <istream>
#include <iterator>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ettg.h"

namespace ettg {

using i64 = std::int64_t;
using u64 = std::uint64_t;
inline constexpr i64 kNone = -1;

inline void check(int rc) {
  if (rc == ETTG_OK) return;
  std::string msg = ettg_last_error();
  if (rc == ETTG_EINVAL) throw std::invalid_argument(msg);
  if (rc == ETTG_ERANGE) throw std::out_of_range(msg);
  throw std::runtime_error(msg);
}

// Same field layout as ett::RootedTree / ett::EdgeList (graph.hpp:18-23, :66-70).
struct RootedTree {
  i64 n = 0;
  i64 root = 0;
  std::vector<i64> parent;
};

struct EdgeList {
  i64 n = 0;
  std::vector<std::pair<i64, i64>> edges;
  i64 m() const { return static_cast<i64>(edges.size()); }
};

struct NodeStats {
  std::vector<i64> preorder, size, level, parent;
};

struct BridgeMask {
  std::vector<char> is_bridge;
  i64 count() const {
    i64 c = 0;
    for (char b : is_bridge) c += b ? 1 : 0;
    return c;
  }
};

// PhaseTimes (core/include/ett/bridges.hpp:34-38): wall nanoseconds of an
// engine's phases under the reference's names; here the device time of each
// phase, measured with CUDA events.
struct PhaseTimes {
  std::vector<std::pair<std::string, i64>> nanos;

  void add(std::string name, i64 ns) { nanos.emplace_back(std::move(name), ns); }
};

// Owns the device index; movable, not copyable.
class LcaIndex {
 public:
  LcaIndex() = default;
  LcaIndex(ettg_lca* h, unsigned engine) : h_(h, &ettg_lca_free), engine_(engine) {}
  ettg_lca* get() const { return h_.get(); }
  unsigned engine() const { return engine_; }
  i64 n() const {
    i64 v = 0;
    check(ettg_lca_size(h_.get(), &v));
    return v;
  }

 private:
  std::unique_ptr<ettg_lca, void (*)(ettg_lca*)> h_{nullptr, &ettg_lca_free};
  unsigned engine_ = ETTG_ENGINE_INLABEL;
};

using InlabelIndex = LcaIndex;
using RmqLcaIndex = LcaIndex;

inline LcaIndex inlabel_build(const RootedTree& t, int device = 0) {
  if (static_cast<i64>(t.parent.size()) != t.n)
    throw std::invalid_argument("parent array size mismatch");
  ettg_lca* h = nullptr;
  check(ettg_lca_build(t.parent.data(), t.n, t.root, device, ETTG_ENGINE_INLABEL, &h));
  return LcaIndex(h, ETTG_ENGINE_INLABEL);
}

inline LcaIndex naive_build(const RootedTree& t, int device = 0) {
  if (static_cast<i64>(t.parent.size()) != t.n)
    throw std::invalid_argument("parent array size mismatch");
  ettg_lca* h = nullptr;
  check(ettg_lca_build(t.parent.data(), t.n, t.root, device, ETTG_ENGINE_NAIVE, &h));
  return LcaIndex(h, ETTG_ENGINE_NAIVE);
}

inline std::vector<i64> ancestor_doubling_levels(const RootedTree& t, int device = 0) {
  std::vector<i64> level(t.n);
  check(ettg_ancestor_levels(t.parent.data(), t.n, t.root, device, level.data()));
  return level;
}

inline LcaIndex rmq_lca_build(const RootedTree& t, int device = 0) {
  if (static_cast<i64>(t.parent.size()) != t.n)
    throw std::invalid_argument("parent array size mismatch");
  ettg_lca* h = nullptr;
  check(ettg_lca_build(t.parent.data(), t.n, t.root, device, ETTG_ENGINE_RMQ, &h));
  return LcaIndex(h, ETTG_ENGINE_RMQ);
}

// answer_batch (lca.hpp:50-65): answers in query order; batch < 1 throws.
inline std::vector<i64> answer_batch(const LcaIndex& idx,
                                     const std::vector<std::pair<i64, i64>>& queries,
                                     i64 batch_size) {
  std::vector<i64> out(queries.size());
  static_assert(sizeof(std::pair<i64, i64>) == 2 * sizeof(i64), "pair layout");
  check(ettg_lca_query_engine(idx.get(), idx.engine(),
                              reinterpret_cast<const int64_t*>(queries.data()),
                              static_cast<i64>(queries.size()), batch_size, out.data()));
  return out;
}

// Multi-GPU: query replicas of an inlabel index on
// `devices`, one grouped ncclBroadcast of the packed index; and a batch
// sharded across replicas, answers in query order.
inline std::vector<LcaIndex> replicate(const LcaIndex& idx, const std::vector<int>& devices) {
  std::vector<ettg_lca*> out(devices.size(), nullptr);
  check(ettg_lca_replicate(idx.get(), static_cast<int>(devices.size()), devices.data(),
                           out.data()));
  std::vector<LcaIndex> reps;
  for (ettg_lca* h : out) reps.emplace_back(h, ETTG_ENGINE_INLABEL);
  return reps;
}

inline std::vector<i64> answer_batch(const std::vector<LcaIndex>& replicas,
                                     const std::vector<std::pair<i64, i64>>& queries,
                                     i64 batch_size) {
  std::vector<ettg_lca*> hs;
  for (const auto& r : replicas) hs.push_back(r.get());
  std::vector<i64> out(queries.size());
  check(ettg_lca_query_multi(hs.data(), static_cast<int>(hs.size()), ETTG_ENGINE_INLABEL,
                             reinterpret_cast<const int64_t*>(queries.data()),
                             static_cast<i64>(queries.size()), batch_size, out.data()));
  return out;
}

inline i64 inlabel_lca(const LcaIndex& idx, i64 x, i64 y) {
  return answer_batch(idx, {{x, y}}, 1)[0];
}

inline NodeStats node_stats(const RootedTree& t, int device = 0) {
  LcaIndex idx = inlabel_build(t, device);
  NodeStats s;
  s.preorder.resize(t.n);
  s.size.resize(t.n);
  s.level.resize(t.n);
  s.parent.resize(t.n);
  check(ettg_lca_stats(idx.get(), s.preorder.data(), s.size.data(), s.level.data(),
                       s.parent.data()));
  return s;
}

// AdjacencyIndex (graph.hpp:44-61), the reference engines' input type.
struct AdjacencyIndex {
  i64 n = 0;
  i64 m = 0;
  std::vector<i64> offsets;    // n + 1
  std::vector<i64> neighbors;  // 2m
  std::vector<i64> edge_ids;   // 2m

  i64 degree(i64 v) const { return offsets[v + 1] - offsets[v]; }
};

// build_adjacency (graph.hpp:63) on the device; bit-identical CSR.
inline AdjacencyIndex build_adjacency(const EdgeList& g, int device = 0) {
  AdjacencyIndex a;
  a.n = g.n;
  a.m = g.m();
  a.offsets.resize(g.n + 1);
  a.neighbors.resize(2 * a.m);
  a.edge_ids.resize(2 * a.m);
  check(ettg_build_adjacency(reinterpret_cast<const int64_t*>(g.edges.data()), g.n, a.m, device,
                             a.offsets.data(), a.neighbors.data(), a.edge_ids.data()));
  return a;
}

namespace detail {
// Phase names as the reference records them (bridges.cpp:292-337).
inline void phases(PhaseTimes* times, int engine, bool on_tree, const ettg_phase_times& pt) {
  if (!times) return;
  auto ns = [](double ms) { return static_cast<i64>(ms * 1e6 + 0.5); };
  if (!on_tree) times->add("spanning", ns(pt.spanning_ms));
  if (engine != ETTG_BRIDGES_CK) times->add("euler", ns(pt.euler_ms));
  if (engine == ETTG_BRIDGES_TV)
    times->add("lowhigh", ns(pt.lowhigh_ms));
  else
    times->add("marking", ns(pt.marking_ms));
}
inline BridgeMask mask_of(const std::vector<uint8_t>& m) {
  BridgeMask out;
  out.is_bridge.assign(m.begin(), m.end());
  return out;
}
inline BridgeMask bridges_adj(const AdjacencyIndex& g, int engine, const std::vector<char>* tree,
                              PhaseTimes* times, int device) {
  std::vector<uint8_t> mask(static_cast<size_t>(g.m));
  ettg_phase_times pt{};
  if (tree && static_cast<i64>(tree->size()) != g.m)
    throw std::invalid_argument("tree mask size mismatch");
  check(ettg_bridges_csr(g.offsets.data(), g.neighbors.data(), g.edge_ids.data(), g.n, g.m,
                         device, engine,
                         tree ? reinterpret_cast<const uint8_t*>(tree->data()) : nullptr,
                         mask.data(), &pt));
  phases(times, engine, tree != nullptr, pt);
  return mask_of(mask);
}
inline BridgeMask bridges_edges(const EdgeList& g, int engine, PhaseTimes* times, int device) {
  std::vector<uint8_t> mask(g.edges.size());
  ettg_phase_times pt{};
  check(ettg_bridges_engine(reinterpret_cast<const int64_t*>(g.edges.data()), g.n, g.m(), device,
                            engine, mask.data(), &pt));
  phases(times, engine, false, pt);
  return mask_of(mask);
}
}  // namespace detail

// The engines with the reference's exact signatures (bridges.hpp:55-61), so
// `using BridgeFn = BridgeMask (*)(const AdjacencyIndex&, PhaseTimes*)`
// (tools/ett_bench.cpp:111) binds to them; the three-argument overloads pick
// the device.
inline BridgeMask tv_bridges(const AdjacencyIndex& g, PhaseTimes* times = nullptr) {
  return detail::bridges_adj(g, ETTG_BRIDGES_TV, nullptr, times, 0);
}
inline BridgeMask ck_bridges(const AdjacencyIndex& g, PhaseTimes* times = nullptr) {
  return detail::bridges_adj(g, ETTG_BRIDGES_CK, nullptr, times, 0);
}
inline BridgeMask hybrid_bridges(const AdjacencyIndex& g, PhaseTimes* times = nullptr) {
  return detail::bridges_adj(g, ETTG_BRIDGES_HYBRID, nullptr, times, 0);
}
// dfs_bridges (bridges.hpp:61) is the reference's sequential verification
// engine; a depth-first search has no parallel form, so the drop-in answers
// with the independent device algorithm -- BFS tree + Chaitanya-Kothapalli
// marking -- which shares no phase with TV.  Same contract: the bridge mask.
inline BridgeMask dfs_bridges(const AdjacencyIndex& g, PhaseTimes* times = nullptr) {
  return detail::bridges_adj(g, ETTG_BRIDGES_CK, nullptr, times, 0);
}
inline BridgeMask tv_bridges(const AdjacencyIndex& g, PhaseTimes* times, int device) {
  return detail::bridges_adj(g, ETTG_BRIDGES_TV, nullptr, times, device);
}
inline BridgeMask ck_bridges(const AdjacencyIndex& g, PhaseTimes* times, int device) {
  return detail::bridges_adj(g, ETTG_BRIDGES_CK, nullptr, times, device);
}
inline BridgeMask hybrid_bridges(const AdjacencyIndex& g, PhaseTimes* times, int device) {
  return detail::bridges_adj(g, ETTG_BRIDGES_HYBRID, nullptr, times, device);
}
// tv_bridges_on_tree (bridges.hpp:58-60): the caller's spanning tree
// replaces hooking; a mask that is not a spanning tree throws
// std::invalid_argument("not a tree: ...") like check_is_tree.
inline BridgeMask tv_bridges_on_tree(const AdjacencyIndex& g, const std::vector<char>& tree_mask,
                                     PhaseTimes* times = nullptr, int device = 0) {
  return detail::bridges_adj(g, ETTG_BRIDGES_TV, &tree_mask, times, device);
}

// Also straight from the EdgeList the AdjacencyIndex is built from (no CSR
// needed on the device: 8 B per edge over the link instead of 32).
inline BridgeMask tv_bridges(const EdgeList& g, PhaseTimes* times = nullptr, int device = 0) {
  return detail::bridges_edges(g, ETTG_BRIDGES_TV, times, device);
}
inline BridgeMask ck_bridges(const EdgeList& g, PhaseTimes* times = nullptr, int device = 0) {
  return detail::bridges_edges(g, ETTG_BRIDGES_CK, times, device);
}
inline BridgeMask hybrid_bridges(const EdgeList& g, PhaseTimes* times = nullptr, int device = 0) {
  return detail::bridges_edges(g, ETTG_BRIDGES_HYBRID, times, device);
}

// LowHigh (bridges.hpp) as the TV engine computes it, with the preorder it is
// numbered in (root 0) and the spanning tree used: tree_mask, or the engine's
// own hooking tree when null.  A diagnostic for checking the intermediate
// against the reference's low_high (core/src/bridges.cpp:251-287).
struct LowHigh {
  std::vector<i64> low, high, preorder;
  std::vector<char> tree_mask;
};
inline LowHigh low_high(const EdgeList& g, const std::vector<char>* tree_mask = nullptr,
                        int device = 0) {
  if (tree_mask && static_cast<i64>(tree_mask->size()) != g.m())
    throw std::invalid_argument("tree mask size mismatch");
  LowHigh out;
  out.low.resize(static_cast<size_t>(g.n));
  out.high.resize(static_cast<size_t>(g.n));
  out.preorder.resize(static_cast<size_t>(g.n));
  std::vector<uint8_t> tree(g.edges.size());
  check(ettg_bridges_low_high(reinterpret_cast<const int64_t*>(g.edges.data()), g.n, g.m(),
                              device,
                              tree_mask ? reinterpret_cast<const uint8_t*>(tree_mask->data())
                                        : nullptr,
                              tree.data(), out.preorder.data(), out.low.data(),
                              out.high.data()));
  if (tree_mask)
    out.tree_mask = *tree_mask;
  else
    out.tree_mask.assign(tree.begin(), tree.end());
  return out;
}

// SpanningTree fields of bfs_tree (bridges.hpp:12-18, :50).
struct SpanningTree {
  std::vector<char> is_tree_edge;
  std::vector<i64> level, parent, parent_edge;
};

inline SpanningTree bfs_tree(const EdgeList& g, i64 root, int device = 0) {
  SpanningTree st;
  std::vector<uint8_t> mask(g.edges.size());
  st.level.resize(g.n);
  st.parent.resize(g.n);
  st.parent_edge.resize(g.n);
  check(ettg_bfs_tree(reinterpret_cast<const int64_t*>(g.edges.data()), g.n, g.m(), root, device,
                      mask.data(), st.level.data(), st.parent.data(), st.parent_edge.data()));
  st.is_tree_edge.assign(mask.begin(), mask.end());
  return st;
}

inline SpanningTree bfs_tree(const AdjacencyIndex& g, i64 root, int device = 0) {
  SpanningTree st;
  std::vector<uint8_t> mask(static_cast<size_t>(g.m));
  st.level.resize(g.n);
  st.parent.resize(g.n);
  st.parent_edge.resize(g.n);
  check(ettg_bfs_tree_csr(g.offsets.data(), g.neighbors.data(), g.edge_ids.data(), g.n, g.m, root,
                          device, mask.data(), st.level.data(), st.parent.data(),
                          st.parent_edge.data()));
  st.is_tree_edge.assign(mask.begin(), mask.end());
  return st;
}

struct ComponentResult {  // graph.hpp:76-79
  EdgeList graph;
  std::vector<i64> old_to_new;
};

inline ComponentResult largest_component(const EdgeList& g, int device = 0) {
  ComponentResult r;
  r.old_to_new.resize(g.n);
  std::vector<int64_t> out(2 * g.edges.size() + 2);
  int64_t nn = 0, mm = 0;
  check(ettg_largest_component(reinterpret_cast<const int64_t*>(g.edges.data()), g.n, g.m(),
                               device, r.old_to_new.data(), &nn, &mm, out.data()));
  r.graph.n = nn;
  r.graph.edges.resize(mm);
  for (int64_t i = 0; i < mm; ++i) r.graph.edges[i] = {out[2 * i], out[2 * i + 1]};
  return r;
}

// ParseStats (graph.hpp:27-32) and the text parsers (graph.cpp:57-133).
struct ParseStats {
  i64 self_loops_removed = 0;
  i64 duplicates_removed = 0;
  i64 removed() const { return self_loops_removed + duplicates_removed; }
};

namespace detail {
template <class Fn>
EdgeList parse_stream(Fn fn, std::istream& in, ParseStats* stats, int device) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  const i64 cap = static_cast<i64>(text.size()) / 4 + 2;  // an edge line takes >= 4 bytes
  std::vector<i64> buf(2 * static_cast<size_t>(cap));
  i64 n = 0, m = 0;
  ettg_parse_stats st{0, 0};
  check(fn(text.data(), static_cast<i64>(text.size()), device, buf.data(), cap, &n, &m, &st));
  EdgeList g;
  g.n = n;
  g.edges.resize(static_cast<size_t>(m));
  for (i64 i = 0; i < m; ++i) g.edges[i] = {buf[2 * i], buf[2 * i + 1]};
  if (stats) *stats = ParseStats{st.self_loops_removed, st.duplicates_removed};
  return g;
}
}  // namespace detail

inline EdgeList parse_edge_list(std::istream& in, ParseStats* stats = nullptr, int device = 0) {
  return detail::parse_stream(ettg_parse_edge_list, in, stats, device);
}
inline EdgeList parse_dimacs_gr(std::istream& in, ParseStats* stats = nullptr, int device = 0) {
  return detail::parse_stream(ettg_parse_dimacs_gr, in, stats, device);
}

// ---- primitives (core/include/ett/primitives.hpp) ----------------------
inline constexpr i64 kPlusInf = INT64_MAX;
inline constexpr i64 kMinusInf = INT64_MIN;

struct LinkedListArray {  // primitives.hpp:17-24
  std::vector<i64> succ;
  i64 head = 0;
  i64 size() const { return static_cast<i64>(succ.size()); }
};

inline std::vector<i64> list_scan(const LinkedListArray& list, const std::vector<i64>& values,
                                  int device = 0) {
  if (static_cast<i64>(values.size()) != list.size())
    throw std::invalid_argument("list_scan: values size mismatch");
  std::vector<i64> out(values.size());
  if (!out.empty())
    check(ettg_list_scan(list.succ.data(), values.data(), list.size(), list.head, device,
                         out.data()));
  return out;
}

struct Min { static constexpr int op = ETTG_REDUCE_MIN; };
struct Max { static constexpr int op = ETTG_REDUCE_MAX; };
struct Plus { static constexpr int op = ETTG_REDUCE_SUM; };

template <class Combine>
std::vector<i64> segmented_reduce(const std::vector<i64>& values, const std::vector<i64>& offsets,
                                  Combine, i64 identity, int device = 0) {
  std::vector<i64> out(offsets.empty() ? 0 : offsets.size() - 1);
  check(ettg_segmented_reduce(values.data(), static_cast<i64>(values.size()), offsets.data(),
                              static_cast<i64>(offsets.size()), Combine::op, identity, device,
                              out.data()));
  return out;
}

// primitives.hpp:100-121.  min/max answer one inclusive range like the
// reference; mins/maxs answer a batch of (l, r) pairs in one launch.
class RangeIndex {
 public:
  explicit RangeIndex(const std::vector<i64>& keys, int device = 0) {
    ettg_range_index* h = nullptr;
    check(ettg_range_index_build(keys.data(), static_cast<i64>(keys.size()), device, &h));
    h_.reset(h);
  }
  i64 size() const { return ettg_range_index_size(h_.get()); }
  i64 min(i64 l, i64 r) const { return one(l, r, true); }
  i64 max(i64 l, i64 r) const { return one(l, r, false); }
  std::vector<i64> mins(const std::vector<std::pair<i64, i64>>& ranges) const {
    return batch(ranges, true);
  }
  std::vector<i64> maxs(const std::vector<std::pair<i64, i64>>& ranges) const {
    return batch(ranges, false);
  }
  const ettg_range_index* handle() const { return h_.get(); }

 private:
  struct Free {
    void operator()(ettg_range_index* h) const { ettg_range_index_free(h); }
  };
  std::unique_ptr<ettg_range_index, Free> h_;
  i64 one(i64 l, i64 r, bool want_min) const {
    const i64 q[2] = {l, r};
    i64 v = 0;
    check(ettg_range_index_query(h_.get(), q, 1, want_min ? &v : nullptr,
                                 want_min ? nullptr : &v));
    return v;
  }
  std::vector<i64> batch(const std::vector<std::pair<i64, i64>>& ranges, bool want_min) const {
    std::vector<i64> flat(2 * ranges.size()), out(ranges.size());
    for (size_t i = 0; i < ranges.size(); ++i) {
      flat[2 * i] = ranges[i].first;
      flat[2 * i + 1] = ranges[i].second;
    }
    if (!ranges.empty())
      check(ettg_range_index_query(h_.get(), flat.data(), static_cast<i64>(ranges.size()),
                                   want_min ? out.data() : nullptr,
                                   want_min ? nullptr : out.data()));
    return out;
  }
};

inline RangeIndex rmq_build(const std::vector<i64>& keys, int device = 0) {
  return RangeIndex(keys, device);
}
inline i64 rmq_min(const RangeIndex& idx, i64 l, i64 r) { return idx.min(l, r); }
inline i64 rmq_max(const RangeIndex& idx, i64 l, i64 r) { return idx.max(l, r); }

}  // namespace ettg

#endif  // ETTG_HPP_
