// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" face of the *unmodified* reference library (eulertools core/),
// compiled straight from /root/reference/proj/core/src/*.cpp by
// oracle/Makefile into oracle/_ref/libett_ref.so.  Tests use it to pin the
// C restatement (oracle/ettg_oracle.c) and the CUDA path; bench.py uses it as
// the "reference" CPU arm (cpu_baseline.kind = "reference").
//
// Every function returns 0 on success, 1 for std::invalid_argument,
// 2 for std::out_of_range, 3 for anything else; ref_last_error() holds the
// exception text.  Ids cross the boundary as int64 (the reference's i64).
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ett/bridges.hpp"
#include "ett/euler.hpp"
#include "ett/generators.hpp"
#include "ett/graph.hpp"
#include "ett/lca.hpp"
#include "ett/primitives.hpp"
#include "oracles.hpp"  // tests/oracles.hpp (recursive_low_high)
#include <pthread.h>

using namespace ett;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

RootedTree make_tree(int64_t n, const int64_t* parent, int64_t root) {
  RootedTree t;
  t.n = n;
  t.root = root;
  t.parent.assign(parent, parent + n);
  return t;
}

EdgeList make_edges(int64_t n, int64_t m, const int64_t* edges) {
  EdgeList g;
  g.n = n;
  g.edges.resize(m);
  for (int64_t i = 0; i < m; ++i) g.edges[i] = {edges[2 * i], edges[2 * i + 1]};
  return g;
}

std::vector<std::pair<i64, i64>> make_pairs(const int64_t* pairs, int64_t q) {
  std::vector<std::pair<i64, i64>> out(q);
  for (int64_t i = 0; i < q; ++i) out[i] = {pairs[2 * i], pairs[2 * i + 1]};
  return out;
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_workers(int w) { set_worker_count(w); }
int ref_workers() { return worker_count(); }

// ---- generators (core/src/generators.cpp) ---------------------------------
int ref_grasp_tree(int64_t n, uint64_t gamma, uint64_t seed, int64_t* parent) {
  return guard([&] {
    RootedTree t = grasp_tree({n, gamma, seed});
    std::memcpy(parent, t.parent.data(), n * sizeof(int64_t));
  });
}

int ref_barabasi_tree(int64_t n, uint64_t seed, int64_t* parent) {
  return guard([&] {
    RootedTree t = barabasi_tree(n, seed);
    std::memcpy(parent, t.parent.data(), n * sizeof(int64_t));
  });
}

int ref_permute_labels(int64_t n, const int64_t* parent, int64_t root,
                       uint64_t seed, int64_t* parent_out, int64_t* root_out) {
  return guard([&] {
    RootedTree t = permute_labels(make_tree(n, parent, root), seed);
    std::memcpy(parent_out, t.parent.data(), n * sizeof(int64_t));
    *root_out = t.root;
  });
}

int ref_sample_queries(int64_t n, int64_t q, uint64_t seed, int64_t* pairs) {
  return guard([&] {
    auto qs = sample_queries(n, q, seed);
    for (int64_t i = 0; i < q; ++i) {
      pairs[2 * i] = qs[i].first;
      pairs[2 * i + 1] = qs[i].second;
    }
  });
}

int ref_random_connected_graph(int64_t n, int64_t m, uint64_t seed,
                               int64_t* edges) {
  return guard([&] {
    EdgeList g = random_connected_graph(n, m, seed);
    for (int64_t i = 0; i < m; ++i) {
      edges[2 * i] = g.edges[i].first;
      edges[2 * i + 1] = g.edges[i].second;
    }
  });
}

// ---- primitives (core/src/primitives.cpp) ---------------------------------
int ref_list_rank(int64_t k, const int64_t* succ, int64_t head, int64_t* out) {
  return guard([&] {
    LinkedListArray l;
    l.succ.assign(succ, succ + k);
    l.head = head;
    auto r = list_rank(l);
    std::memcpy(out, r.data(), k * sizeof(int64_t));
  });
}

int ref_exclusive_scan_sum(int64_t n, const int64_t* in, int64_t* out) {
  return guard([&] {
    auto r = exclusive_scan(std::span<const i64>(in, n),
                            [](i64 a, i64 b) { return a + b; }, 0);
    std::memcpy(out, r.data(), n * sizeof(int64_t));
  });
}

int ref_list_scan(int64_t k, const int64_t* succ, int64_t head, const int64_t* values,
                  int64_t* out) {
  return guard([&] {
    LinkedListArray l;
    l.succ.assign(succ, succ + k);
    l.head = head;
    auto r = list_scan(l, std::span<const i64>(values, k));
    std::memcpy(out, r.data(), k * sizeof(int64_t));
  });
}

// op: 0 min, 1 max, 2 sum (the combiners the reference's callers pass).
int ref_segmented_reduce(int64_t nv, const int64_t* values, int64_t no, const int64_t* offsets,
                         int op, int64_t identity, int64_t* out) {
  return guard([&] {
    std::span<const i64> v(values, nv), o(offsets, no);
    std::vector<i64> r;
    if (op == 0)
      r = segmented_reduce(v, o, [](i64 a, i64 b) { return std::min(a, b); }, identity);
    else if (op == 1)
      r = segmented_reduce(v, o, [](i64 a, i64 b) { return std::max(a, b); }, identity);
    else
      r = segmented_reduce(v, o, [](i64 a, i64 b) { return a + b; }, identity);
    std::memcpy(out, r.data(), r.size() * sizeof(int64_t));
  });
}

// ranges[2q] = (l, r); mins/maxs may be null.  Throws on the first bad range.
int ref_range_index(int64_t n, const int64_t* keys, int64_t q, const int64_t* ranges,
                    int64_t* mins, int64_t* maxs) {
  return guard([&] {
    RangeIndex idx(std::span<const i64>(keys, n));
    for (int64_t i = 0; i < q; ++i) {
      if (mins) mins[i] = idx.min(ranges[2 * i], ranges[2 * i + 1]);
      if (maxs) maxs[i] = idx.max(ranges[2 * i], ranges[2 * i + 1]);
    }
  });
}

// ---- Euler tour (core/src/euler.cpp) --------------------------------------
// Tour of the tree given by `parent`, as (src,dst) pairs in tour order,
// 2(n-1) of them; plus node_stats.
int ref_euler_tour(int64_t n, const int64_t* parent, int64_t root,
                   int64_t* tour_src, int64_t* tour_dst) {
  return guard([&] {
    RootedTree t = make_tree(n, parent, root);
    validate_tree(t);
    EulerTour tour = linearize(build_half_edges(tree_edges(t), true), root);
    const auto& h = tour.structure;
    for (size_t i = 0; i < tour.order.size(); ++i) {
      tour_src[i] = h.src[tour.order[i]];
      tour_dst[i] = h.dst[tour.order[i]];
    }
  });
}

int ref_node_stats(int64_t n, const int64_t* parent, int64_t root,
                   int64_t* preorder, int64_t* size, int64_t* level,
                   int64_t* par) {
  return guard([&] {
    RootedTree t = make_tree(n, parent, root);
    validate_tree(t);
    NodeStats s =
        node_stats(linearize(build_half_edges(tree_edges(t), true), root));
    std::memcpy(preorder, s.preorder.data(), n * sizeof(int64_t));
    std::memcpy(size, s.size.data(), n * sizeof(int64_t));
    std::memcpy(level, s.level.data(), n * sizeof(int64_t));
    std::memcpy(par, s.parent.data(), n * sizeof(int64_t));
  });
}

// ---- LCA (core/src/lca.cpp) -----------------------------------------------
int ref_inlabel_index(int64_t n, const int64_t* parent, int64_t root,
                      int64_t* inlabel, uint64_t* ascendant, int64_t* head,
                      int64_t* level, int64_t* par) {
  return guard([&] {
    InlabelIndex idx = inlabel_build(make_tree(n, parent, root));
    std::memcpy(inlabel, idx.inlabel.data(), n * sizeof(int64_t));
    std::memcpy(ascendant, idx.ascendant.data(), n * sizeof(uint64_t));
    std::memcpy(head, idx.head.data(), (n + 1) * sizeof(int64_t));
    std::memcpy(level, idx.level.data(), n * sizeof(int64_t));
    std::memcpy(par, idx.parent.data(), n * sizeof(int64_t));
  });
}

// Opaque index handles so the bench can time build and query separately,
// exactly as tools/ett_bench.cpp:136-150 does.
void* ref_inlabel_new(int64_t n, const int64_t* parent, int64_t root,
                      int64_t* build_ns) {
  InlabelIndex* out = nullptr;
  int rc = guard([&] {
    RootedTree t = make_tree(n, parent, root);
    int64_t t0 = now_ns();
    out = new InlabelIndex(inlabel_build(t));
    if (build_ns) *build_ns = now_ns() - t0;
  });
  return rc == 0 ? out : nullptr;
}

void ref_inlabel_free(void* h) { delete static_cast<InlabelIndex*>(h); }

// answer_batch(inlabel_lca) over caller pairs; query_ns excludes the
// int64 pair marshalling.
int ref_inlabel_answer(void* h, const int64_t* pairs, int64_t q, int64_t batch,
                       int64_t* answers, int64_t* query_ns) {
  return guard([&] {
    const InlabelIndex& idx = *static_cast<InlabelIndex*>(h);
    auto qs = make_pairs(pairs, q);
    int64_t t0 = now_ns();
    auto a = answer_batch([&](i64 x, i64 y) { return inlabel_lca(idx, x, y); },
                          qs, batch);
    if (query_ns) *query_ns = now_ns() - t0;
    std::memcpy(answers, a.data(), q * sizeof(int64_t));
  });
}

int ref_lca(const char* engine, int64_t n, const int64_t* parent, int64_t root,
            const int64_t* pairs, int64_t q, int64_t batch, int64_t* answers) {
  return guard([&] {
    RootedTree t = make_tree(n, parent, root);
    auto qs = make_pairs(pairs, q);
    std::vector<i64> a;
    std::string e(engine);
    if (e == "inlabel") {
      InlabelIndex idx = inlabel_build(t);
      a = answer_batch([&](i64 x, i64 y) { return inlabel_lca(idx, x, y); },
                       qs, batch);
    } else if (e == "rmq") {
      RmqLcaIndex idx = rmq_lca_build(t);
      a = answer_batch([&](i64 x, i64 y) { return rmq_lca(idx, x, y); }, qs,
                       batch);
    } else if (e == "naive") {
      NaiveIndex idx = naive_build(t);
      a = answer_batch([&](i64 x, i64 y) { return naive_lca(idx, x, y); }, qs,
                       batch);
    } else {
      throw std::runtime_error("unknown engine " + e);
    }
    std::memcpy(answers, a.data(), q * sizeof(int64_t));
  });
}

// ---- bridges (core/src/bridges.cpp) ----------------------------------------
// engine: "tv" | "dfs" | "ck" | "hybrid" | "brute".  build_adjacency is
// excluded from phase_ns exactly as tools/ett_bench.cpp:310-317 excludes it.
// phase_ns receives up to 4 entries (tv: spanning, euler, lowhigh; total last).
int ref_bridges(const char* engine, int64_t n, int64_t m, const int64_t* edges,
                uint8_t* is_bridge, int64_t* phase_ns) {
  return guard([&] {
    AdjacencyIndex adj = build_adjacency(make_edges(n, m, edges));
    std::string e(engine);
    PhaseTimes pt;
    BridgeMask mask;
    int64_t t0 = now_ns();
    if (e == "tv") mask = tv_bridges(adj, &pt);
    else if (e == "dfs") mask = dfs_bridges(adj, &pt);
    else if (e == "ck") mask = ck_bridges(adj, &pt);
    else if (e == "hybrid") mask = hybrid_bridges(adj, &pt);
    else if (e == "brute") mask = brute_force_bridges(adj);
    else throw std::runtime_error("unknown engine " + e);
    int64_t total = now_ns() - t0;
    for (int64_t i = 0; i < m; ++i) is_bridge[i] = mask.is_bridge[i] ? 1 : 0;
    if (phase_ns) {
      for (int i = 0; i < 4; ++i) phase_ns[i] = 0;
      for (size_t i = 0; i < pt.nanos.size() && i < 3; ++i)
        phase_ns[i] = pt.nanos[i].second;
      phase_ns[3] = total;
    }
  });
}

// Spanning tree of the reference's deterministic hooking + its rooting,
// so low/high can be compared on an identical tree.
int ref_spanning_tree_hooking(int64_t n, int64_t m, const int64_t* edges,
                              uint8_t* tree_mask) {
  return guard([&] {
    AdjacencyIndex adj = build_adjacency(make_edges(n, m, edges));
    auto mask = spanning_tree_hooking(adj);
    for (int64_t i = 0; i < m; ++i) tree_mask[i] = mask[i] ? 1 : 0;
  });
}

// low_high (core/src/bridges.cpp:251-287) on the reference's own rooting of
// `tree_mask` (euler_root_tree, root 0): preorder, parent, low, high per node.
int ref_low_high(int64_t n, int64_t m, const int64_t* edges, const uint8_t* tree_mask,
                 int64_t* preorder, int64_t* parent, int64_t* low, int64_t* high) {
  return guard([&] {
    AdjacencyIndex adj = build_adjacency(make_edges(n, m, edges));
    std::vector<char> mask(tree_mask, tree_mask + m);
    SpanningTree st = euler_root_tree(adj, mask, 0);
    LowHigh lh = low_high(adj, st, *st.stats);
    for (int64_t v = 0; v < n; ++v) {
      preorder[v] = st.stats->preorder[v];
      parent[v] = st.rooted.parent[v];
      low[v] = lh.low[v];
      high[v] = lh.high[v];
    }
  });
}

// recursive_low_high (tests/oracles.hpp:166-201) over a caller rooted tree and
// preorder.  Its recursion is as deep as the tree, so it runs on a thread
// with a 1 GB stack.
int ref_recursive_low_high(int64_t n, int64_t m, const int64_t* edges,
                           const uint8_t* tree_mask, const int64_t* parent, int64_t root,
                           const int64_t* preorder, int64_t* low, int64_t* high) {
  return guard([&] {
    struct Job {
      EdgeList g;
      std::vector<char> mask;
      std::vector<i64> parent, pre;
      i64 root;
      oracle::LowHighOracle out;
    } job{make_edges(n, m, edges), std::vector<char>(tree_mask, tree_mask + m),
          std::vector<i64>(parent, parent + n), std::vector<i64>(preorder, preorder + n), root,
          {}};
    auto body = [](void* p) -> void* {
      auto* j = static_cast<Job*>(p);
      j->out = oracle::recursive_low_high(j->g, j->mask, j->parent, j->root, j->pre);
      return nullptr;
    };
    pthread_attr_t attr;
    pthread_attr_init(&attr);
    pthread_attr_setstacksize(&attr, size_t(1) << 30);
    pthread_t th;
    if (pthread_create(&th, &attr, body, &job) != 0) throw std::runtime_error("pthread_create");
    pthread_join(th, nullptr);
    pthread_attr_destroy(&attr);
    for (int64_t v = 0; v < n; ++v) {
      low[v] = job.out.low[v];
      high[v] = job.out.high[v];
    }
  });
}

// build_adjacency (core/src/graph.cpp:135-173): offsets[n+1], nbr[2m], eid[2m].
int ref_build_adjacency(int64_t n, int64_t m, const int64_t* edges, int64_t* offsets,
                        int64_t* neighbors, int64_t* edge_ids) {
  return guard([&] {
    AdjacencyIndex a = build_adjacency(make_edges(n, m, edges));
    std::memcpy(offsets, a.offsets.data(), (n + 1) * sizeof(int64_t));
    std::memcpy(neighbors, a.neighbors.data(), 2 * m * sizeof(int64_t));
    std::memcpy(edge_ids, a.edge_ids.data(), 2 * m * sizeof(int64_t));
  });
}

// largest_component (core/src/graph.cpp:219-259).
int ref_largest_component(int64_t n, int64_t m, const int64_t* edges, int64_t* old_to_new,
                          int64_t* n_out, int64_t* m_out, int64_t* edges_out) {
  return guard([&] {
    ComponentResult r = largest_component(make_edges(n, m, edges));
    std::memcpy(old_to_new, r.old_to_new.data(), n * sizeof(int64_t));
    *n_out = r.graph.n;
    *m_out = r.graph.m();
    for (int64_t i = 0; i < r.graph.m(); ++i) {
      edges_out[2 * i] = r.graph.edges[i].first;
      edges_out[2 * i + 1] = r.graph.edges[i].second;
    }
  });
}

// bfs_tree (core/src/bridges.cpp:198-249) from `root`.
int ref_bfs_tree(int64_t n, int64_t m, const int64_t* edges, int64_t root, uint8_t* tree_mask,
                 int64_t* level, int64_t* parent, int64_t* parent_edge) {
  return guard([&] {
    AdjacencyIndex a = build_adjacency(make_edges(n, m, edges));
    SpanningTree st = bfs_tree(a, root);
    for (int64_t e = 0; e < m; ++e) tree_mask[e] = st.is_tree_edge[e] ? 1 : 0;
    std::memcpy(level, st.level.data(), n * sizeof(int64_t));
    std::memcpy(parent, st.rooted.parent.data(), n * sizeof(int64_t));
    std::memcpy(parent_edge, st.parent_edge.data(), n * sizeof(int64_t));
  });
}

// parse_edge_list / parse_dimacs_gr (core/src/graph.cpp:57-133) over an
// in-memory text; parse errors (std::runtime_error) return 3 with the message.
int ref_parse(const char* kind, const char* text, int64_t len, int64_t* n, int64_t* m,
              int64_t* self_loops, int64_t* duplicates, int64_t* edges, int64_t cap) {
  return guard([&] {
    std::istringstream in(std::string(text, static_cast<size_t>(len)));
    ParseStats st;
    EdgeList g = std::strcmp(kind, "dimacs") == 0 ? parse_dimacs_gr(in, &st)
                                                   : parse_edge_list(in, &st);
    *n = g.n;
    *m = g.m();
    *self_loops = st.self_loops_removed;
    *duplicates = st.duplicates_removed;
    if (g.m() > cap) throw std::out_of_range("edge buffer too small");
    for (int64_t i = 0; i < g.m(); ++i) {
      edges[2 * i] = g.edges[i].first;
      edges[2 * i + 1] = g.edges[i].second;
    }
  });
}

}  // extern "C"
