// C++ caller through include/ettg.hpp, written like the reference's own tests
// (tests/lca_test.cpp:47-74, tests/bridges_test.cpp): exits non-zero on failure.
#include <algorithm>
#include <cstdio>
#include <sstream>
#include <stdexcept>

#include "ettg.hpp"

#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::fprintf(stderr, "CHECK failed: %s (line %d)\n", #c, __LINE__); \
      return 1;                                                    \
    }                                                              \
  } while (0)

int main() {
  ettg::RootedTree t{6, 0, {-1, 2, 0, 0, 0, 2}};
  auto idx = ettg::inlabel_build(t);
  CHECK(ettg::inlabel_lca(idx, 1, 5) == 2);
  CHECK(ettg::inlabel_lca(idx, 3, 4) == 0);
  auto ans = ettg::answer_batch(idx, {{1, 5}, {3, 4}, {5, 5}}, 2);
  CHECK(ans.size() == 3 && ans[0] == 2 && ans[1] == 0 && ans[2] == 5);
  {  // multi-GPU: replicas (NCCL broadcast) + a sharded batch, same answers
    auto reps = ettg::replicate(idx, {0, 0});
    auto multi = ettg::answer_batch(reps, {{1, 5}, {3, 4}, {5, 5}}, 2);
    CHECK(multi == ans);
  }
  auto r = ettg::rmq_lca_build(t);
  CHECK(ettg::answer_batch(r, {{1, 5}}, 1)[0] == 2);
  auto st = ettg::node_stats(t);
  CHECK(st.preorder == std::vector<ettg::i64>({1, 3, 2, 5, 6, 4}));
  bool threw = false;
  try {
    ettg::answer_batch(idx, {{0, 1}}, 0);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    ettg::inlabel_build(ettg::RootedTree{3, 0, {-1, 2, 1}});
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  ettg::EdgeList g{4, {{0, 1}, {1, 2}, {0, 2}, {2, 3}}};
  ettg::PhaseTimes pt;
  auto mask = ettg::tv_bridges(g, &pt);
  CHECK(mask.is_bridge == std::vector<char>({0, 0, 0, 1}));
  CHECK(mask.count() == 1 && pt.nanos.size() == 3 && pt.nanos[0].first == "spanning");
  auto nv = ettg::naive_build(t);
  CHECK(ettg::answer_batch(nv, {{1, 5}, {3, 4}}, 2) == std::vector<ettg::i64>({2, 0}));
  CHECK(ettg::ancestor_doubling_levels(t) == std::vector<ettg::i64>({0, 2, 1, 1, 1, 2}));
  CHECK(ettg::ck_bridges(g).is_bridge == std::vector<char>({0, 0, 0, 1}));
  ettg::PhaseTimes ph;
  CHECK(ettg::hybrid_bridges(g, &ph).is_bridge == std::vector<char>({0, 0, 0, 1}));
  CHECK(ph.nanos.size() == 3 && ph.nanos[2].first == "marking");
  auto adj = ettg::build_adjacency(g);
  CHECK(adj.offsets == std::vector<ettg::i64>({0, 2, 4, 7, 8}));
  CHECK(adj.neighbors == std::vector<ettg::i64>({1, 2, 0, 2, 0, 1, 3, 2}));
  {  // the reference engines' own input type and signature (bridges.hpp:55-61)
    using BridgeFn = ettg::BridgeMask (*)(const ettg::AdjacencyIndex&, ettg::PhaseTimes*);
    const BridgeFn fns[] = {ettg::tv_bridges, ettg::ck_bridges, ettg::hybrid_bridges,
                            ettg::dfs_bridges};
    for (BridgeFn f : fns) {
      ettg::PhaseTimes p;
      CHECK(f(adj, &p).is_bridge == std::vector<char>({0, 0, 0, 1}));
      CHECK(!p.nanos.empty() && p.nanos[0].first == "spanning");
    }
    // tests/bridges_test.cpp:163-169: the TV criterion does not depend on the tree
    ettg::PhaseTimes p;
    auto via_bfs = ettg::tv_bridges_on_tree(adj, ettg::bfs_tree(adj, 0).is_tree_edge, &p);
    CHECK(via_bfs.is_bridge == ettg::tv_bridges(adj).is_bridge);
    CHECK(p.nanos.size() == 2 && p.nanos[0].first == "euler" && p.nanos[1].first == "lowhigh");
    // check_is_tree messages (core/src/euler.cpp:13-33)
    std::string what;
    try {
      ettg::tv_bridges_on_tree(adj, {1, 1, 0, 0});
    } catch (const std::invalid_argument& e) {
      what = e.what();
    }
    CHECK(what == "not a tree: m != n - 1");
    what.clear();
    try {
      ettg::tv_bridges_on_tree(adj, {1, 1, 1, 0});  // the triangle: a cycle
    } catch (const std::invalid_argument& e) {
      what = e.what();
    }
    CHECK(what == "not a tree: disconnected");
  }
  {  // low/high intermediate (bridges.cpp:251-287) on the BFS tree {01, 02, 23}:
     // 3 is a leaf without non-tree edges; 1 and 2 see each other's preorder
    auto bfs = ettg::bfs_tree(g, 0).is_tree_edge;
    auto lh = ettg::low_high(g, &bfs);
    const auto& pre = lh.preorder;
    CHECK(pre[0] == 1 && lh.low[0] == 1 && lh.high[0] == 4);
    CHECK(lh.low[3] == pre[3] && lh.high[3] == pre[3]);
    CHECK(lh.low[1] == std::min(pre[1], pre[2]) && lh.low[2] == std::min(pre[1], pre[2]));
    CHECK(lh.high[1] == std::max(pre[1], pre[2]));
    CHECK(ettg::low_high(g).tree_mask.size() == g.edges.size());
  }
  auto bt = ettg::bfs_tree(g, 0);
  CHECK(bt.parent == std::vector<ettg::i64>({-1, 0, 0, 2}));
  auto lc = ettg::largest_component(ettg::EdgeList{6, {{0, 1}, {2, 3}, {3, 4}}});
  CHECK(lc.graph.n == 3 && lc.old_to_new == std::vector<ettg::i64>({-1, -1, 0, 1, 2, -1}));
  {  // tests/graph_test.cpp:21-31, :41-45
    std::istringstream in("0 1\n1 0\n0 0\n");
    ettg::ParseStats ps;
    auto g = ettg::parse_edge_list(in, &ps);
    CHECK((g.n == 2 && g.m() == 1 && g.edges[0].first == 0 && g.edges[0].second == 1));
    CHECK(ps.self_loops_removed == 1 && ps.duplicates_removed == 1);
    std::istringstream bad("0 1\nfoo 2\n");
    bool threw = false;
    try {
      ettg::parse_edge_list(bad);
    } catch (const std::runtime_error& e) {
      threw = std::string(e.what()).find("line 2") != std::string::npos;
    }
    CHECK(threw);
    std::istringstream gr("p sp 2 2\na 1 2 1\na 2 1 1\n");
    auto d = ettg::parse_dimacs_gr(gr);
    CHECK(d.n == 2 && d.m() == 1);
  }
  {  // tests/primitives_test.cpp:88-170
    CHECK(ettg::list_scan({{1, 2, -1}, 0}, {5, 7, 9}) == std::vector<ettg::i64>({0, 5, 12}));
    CHECK(ettg::segmented_reduce({3, 1, 2}, {0, 2, 3}, ettg::Min{}, ettg::kPlusInf) ==
          std::vector<ettg::i64>({1, 2}));
    CHECK(ettg::segmented_reduce({3, 1, 2}, {0, 0, 3}, ettg::Min{}, ettg::kPlusInf) ==
          std::vector<ettg::i64>({ettg::kPlusInf, 1}));
    bool threw = false;
    try {
      ettg::segmented_reduce({3, 1, 2}, {0, 2}, ettg::Max{}, ettg::kMinusInf);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
    auto idx = ettg::rmq_build({2, 9, 4, 1});
    CHECK(idx.size() == 4 && ettg::rmq_min(idx, 0, 3) == 1 && ettg::rmq_max(idx, 0, 3) == 9);
    CHECK(idx.min(1, 1) == 9);
    CHECK(idx.maxs({{0, 1}, {2, 3}}) == std::vector<ettg::i64>({9, 4}));
    threw = false;
    try {
      idx.min(0, 4);
    } catch (const std::out_of_range&) {
      threw = true;
    }
    CHECK(threw);
  }
  std::printf("shim ok\n");
  return 0;
}
