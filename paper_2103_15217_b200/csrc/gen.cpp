// Input generators (host C++).  Not on the hot path: they produce the
// synthetic inputs of BASELINE.json's configs.
//
// grasp_tree / barabasi_tree / permute_labels / sample_queries /
// random_connected_graph replay the reference's SplitMix64 streams
// (core/include/ett/rng.hpp:9-44, core/src/generators.cpp:21-111) so both
// sides see identical inputs.  planted_bridge_graph and road_like_graph are
// new: the reference's random generator plants no bridges,
// so these build graphs whose bridge set is known by construction.
#include <omp.h>

#include <algorithm>
#include <charconv>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <string>
#include <unordered_set>
#include <vector>

#include "../../include/ettg.h"

namespace {

thread_local std::string g_gen_err;

struct SplitMix64 {
  uint64_t s;
  explicit SplitMix64(uint64_t seed) : s(seed) {}
  uint64_t next() {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  uint64_t next_below(uint64_t bound) {  // Lemire with rejection
    uint64_t x = next();
    __uint128_t m = static_cast<__uint128_t>(x) * bound;
    uint64_t lo = static_cast<uint64_t>(m);
    if (lo < bound) {
      uint64_t threshold = (0 - bound) % bound;
      while (lo < threshold) {
        x = next();
        m = static_cast<__uint128_t>(x) * bound;
        lo = static_cast<uint64_t>(m);
      }
    }
    return static_cast<uint64_t>(m >> 64);
  }
  int64_t next_in(int64_t lo, int64_t hi) {
    return lo + static_cast<int64_t>(next_below(static_cast<uint64_t>(hi - lo + 1)));
  }
};

struct GenError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class F>
int gen_guard(F&& f) {
  try {
    f();
    return ETTG_OK;
  } catch (const GenError& e) {
    g_gen_err = e.what();
    return ETTG_EINVAL;
  } catch (const std::invalid_argument& e) {
    g_gen_err = e.what();
    return ETTG_EINVAL;
  } catch (const std::out_of_range& e) {
    g_gen_err = e.what();
    return ETTG_ERANGE;
  } catch (const std::exception& e) {
    g_gen_err = e.what();
    return ETTG_EINTERNAL;
  }
}

// Open-addressing set of packed (u,v) pairs.
struct PairSet {
  std::vector<uint64_t> slots;
  uint64_t mask;
  explicit PairSet(uint64_t expect) {
    uint64_t cap = 16;
    while (cap < expect * 2) cap <<= 1;
    slots.assign(cap, ~0ull);
    mask = cap - 1;
  }
  static uint64_t h(uint64_t k) {
    k ^= k >> 33;
    k *= 0xff51afd7ed558ccdULL;
    k ^= k >> 33;
    return k;
  }
  bool insert(uint64_t k) {  // true if new
    uint64_t i = h(k) & mask;
    while (true) {
      if (slots[i] == k) return false;
      if (slots[i] == ~0ull) {
        slots[i] = k;
        return true;
      }
      i = (i + 1) & mask;
    }
  }
};

inline uint64_t pack(int64_t u, int64_t v) {
  return (static_cast<uint64_t>(u) << 32) | static_cast<uint64_t>(v);
}

}  // namespace

extern "C" {

const char* ettg_gen_last_error(void) { return g_gen_err.c_str(); }

// grasp_tree (core/src/generators.cpp:21-37)
int ettg_gen_grasp_tree(int64_t n, uint64_t gamma, uint64_t seed, int64_t* parent) {
  return gen_guard([&] {
    if (n < 1 || gamma < 1) throw GenError("grasp_tree: n and gamma must be >= 1");
    SplitMix64 rng(seed);
    parent[0] = -1;
    for (int64_t i = 1; i < n; ++i) {
      int64_t lo = gamma >= static_cast<uint64_t>(i) ? 0 : i - static_cast<int64_t>(gamma);
      parent[i] = rng.next_in(lo, i - 1);
    }
  });
}

// barabasi_tree (core/src/generators.cpp:39-60)
int ettg_gen_barabasi_tree(int64_t n, uint64_t seed, int64_t* parent) {
  return gen_guard([&] {
    if (n < 1) throw GenError("barabasi_tree: n must be >= 1");
    parent[0] = -1;
    if (n == 1) return;
    SplitMix64 rng(seed);
    std::vector<int64_t> ends;
    ends.reserve(2 * (n - 1));
    parent[1] = 0;
    ends.push_back(0);
    ends.push_back(1);
    for (int64_t i = 2; i < n; ++i) {
      parent[i] = ends[rng.next_below(ends.size())];
      ends.push_back(parent[i]);
      ends.push_back(i);
    }
  });
}

// permute_labels (core/src/generators.cpp:62-78); the input is assumed valid.
int ettg_gen_permute_labels(int64_t n, const int64_t* parent, int64_t root, uint64_t seed,
                            int64_t* parent_out, int64_t* root_out) {
  return gen_guard([&] {
    if (n < 1) throw GenError("permute_labels: empty tree");
    std::vector<int64_t> perm(n);
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    SplitMix64 rng(seed);
    for (int64_t i = n - 1; i > 0; --i)
      std::swap(perm[i], perm[rng.next_below(static_cast<uint64_t>(i + 1))]);
    std::vector<int64_t> out(n, -1);
    for (int64_t v = 0; v < n; ++v)
      if (parent[v] != -1) out[perm[v]] = perm[parent[v]];
    std::memcpy(parent_out, out.data(), n * sizeof(int64_t));
    *root_out = perm[root];
  });
}

// sample_queries (core/src/generators.cpp:80-91)
int ettg_gen_sample_queries(int64_t n, int64_t q, uint64_t seed, int64_t* pairs) {
  return gen_guard([&] {
    if (n < 1 || q < 0) throw GenError("sample_queries: bad params");
    SplitMix64 rng(seed);
    for (int64_t i = 0; i < q; ++i) {
      pairs[2 * i] = static_cast<int64_t>(rng.next_below(static_cast<uint64_t>(n)));
      pairs[2 * i + 1] = static_cast<int64_t>(rng.next_below(static_cast<uint64_t>(n)));
    }
  });
}

// random_connected_graph (core/src/generators.cpp:93-111)
int ettg_gen_random_connected_graph(int64_t n, int64_t m, uint64_t seed, int64_t* edges) {
  return gen_guard([&] {
    if (n < 1 || m < n - 1 || m > n * (n - 1) / 2)
      throw GenError("random_connected_graph: infeasible edge count");
    std::vector<int64_t> parent(n);
    ettg_gen_grasp_tree(n, ~0ull, seed, parent.data());
    PairSet used(static_cast<uint64_t>(m));
    int64_t k = 0;
    for (int64_t v = 0; v < n; ++v) {
      if (parent[v] == -1) continue;
      int64_t a = std::min(v, parent[v]), b = std::max(v, parent[v]);
      used.insert(pack(a, b));
      edges[2 * k] = a;
      edges[2 * k + 1] = b;
      ++k;
    }
    SplitMix64 rng(seed ^ 0x6e6f6e2d74726565ULL);
    while (k < m) {
      int64_t u = static_cast<int64_t>(rng.next_below(static_cast<uint64_t>(n)));
      int64_t v = static_cast<int64_t>(rng.next_below(static_cast<uint64_t>(n)));
      if (u == v) continue;
      int64_t a = std::min(u, v), b = std::max(u, v);
      if (!used.insert(pack(a, b))) continue;
      edges[2 * k] = a;
      edges[2 * k + 1] = b;
      ++k;
    }
  });
}

// planted_bridge_graph: b+1 groups (>= 3 nodes each) of a seeded
// permutation; each group = Hamiltonian cycle + distinct random chords
// (2-edge-connected); group i >= 1 hangs off a uniform earlier group by one
// edge.  Exactly those b edges are bridges.  Edge order is shuffled.
int ettg_gen_planted_bridge_graph(int64_t n, int64_t m, int64_t b, uint64_t seed, int64_t* edges,
                                  uint8_t* truth) {
  return gen_guard([&] {
    if (b < 0 || n < 3 * (b + 1)) throw GenError("planted_bridge_graph: need n >= 3(b+1)");
    if (m < n + b) throw GenError("planted_bridge_graph: need m >= n + b");
    SplitMix64 rng(seed);
    std::vector<int64_t> perm(n);
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    for (int64_t i = n - 1; i > 0; --i)
      std::swap(perm[i], perm[rng.next_below(static_cast<uint64_t>(i + 1))]);
    const int64_t groups = b + 1;
    const int64_t base = n / groups, rem = n % groups;
    std::vector<int64_t> goff(groups + 1);
    for (int64_t g = 0; g < groups; ++g) goff[g + 1] = goff[g] + base + (g < rem ? 1 : 0);
    const int64_t extra_total = m - n - b;
    int64_t k = 0;
    auto emit = [&](int64_t u, int64_t v, uint8_t t) {
      edges[2 * k] = std::min(u, v);
      edges[2 * k + 1] = std::max(u, v);
      truth[k] = t;
      ++k;
    };
    // cycles
    for (int64_t g = 0; g < groups; ++g) {
      const int64_t s = goff[g], sz = goff[g + 1] - goff[g];
      for (int64_t j = 0; j < sz; ++j) emit(perm[s + j], perm[s + (j + 1) % sz], 0);
    }
    // bridges
    for (int64_t g = 1; g < groups; ++g) {
      const int64_t h = static_cast<int64_t>(rng.next_below(static_cast<uint64_t>(g)));
      const int64_t a = perm[goff[g] + rng.next_below(goff[g + 1] - goff[g])];
      const int64_t c = perm[goff[h] + rng.next_below(goff[h + 1] - goff[h])];
      emit(a, c, 1);
    }
    // chords, split proportionally to group size; the remainder goes one
    // each to the first groups
    int64_t assigned = 0;
    for (int64_t g = 0; g < groups; ++g) assigned += extra_total * (goff[g + 1] - goff[g]) / n;
    int64_t leftover = extra_total - assigned;
    for (int64_t g = 0; g < groups; ++g) {
      const int64_t s = goff[g], sz = goff[g + 1] - goff[g];
      int64_t want = extra_total * sz / n;
      if (leftover > 0) {
        ++want;
        --leftover;
      }
      const int64_t room = sz * (sz - 1) / 2 - sz;
      if (want > room) throw GenError("planted_bridge_graph: groups too small for m");
      std::vector<uint8_t> used(static_cast<size_t>(sz * sz), 0);
      for (int64_t j = 0; j < sz; ++j) {
        const int64_t j2 = (j + 1) % sz;
        used[j * sz + j2] = used[j2 * sz + j] = 1;
      }
      int64_t got = 0;
      while (got < want) {
        const int64_t x = static_cast<int64_t>(rng.next_below(sz));
        const int64_t y = static_cast<int64_t>(rng.next_below(sz));
        if (x == y || used[x * sz + y]) continue;
        used[x * sz + y] = used[y * sz + x] = 1;
        emit(perm[s + x], perm[s + y], 0);
        ++got;
      }
    }
    if (k != m) throw GenError("planted_bridge_graph: internal edge count mismatch");
    for (int64_t i = m - 1; i > 0; --i) {
      const int64_t j = static_cast<int64_t>(rng.next_below(static_cast<uint64_t>(i + 1)));
      std::swap(edges[2 * i], edges[2 * j]);
      std::swap(edges[2 * i + 1], edges[2 * j + 1]);
      std::swap(truth[i], truth[j]);
    }
  });
}

}  // extern "C"

namespace {

struct RoadShape {
  int64_t W, H, extra, r, pendant;
  std::vector<std::pair<int, int>> offs;  // forward half-window minus grid steps
  RoadShape(int64_t W_, int64_t H_, int64_t e, int64_t r_, int64_t p)
      : W(W_), H(H_), extra(e), r(r_), pendant(p) {
    for (int dy = 0; dy <= r; ++dy)
      for (int dx = -static_cast<int>(r); dx <= r; ++dx) {
        if (dy == 0 && dx <= 0) continue;
        if ((dx == 1 && dy == 0) || (dx == 0 && dy == 1)) continue;
        offs.push_back({dx, dy});
      }
  }
  // in-bounds extra candidates of node (x, y)
  int avail(int64_t x, int64_t y) const {
    int c = 0;
    for (auto [dx, dy] : offs)
      if (x + dx >= 0 && x + dx < W && y + dy < H) ++c;
    return c;
  }
  int64_t node_edges(int64_t x, int64_t y) const {
    int64_t e = (x + 1 < W ? 1 : 0) + (y + 1 < H ? 1 : 0);
    return e + std::min<int64_t>(extra, avail(x, y));
  }
};

}  // namespace

extern "C" {

int64_t ettg_road_like_edge_count(int64_t W, int64_t H, int64_t extra, int64_t r,
                                  int64_t pendant) {
  if (W < 2 || H < 2 || r < 1 || extra < 0 || pendant < 0) return -1;
  RoadShape sh(W, H, extra, r, pendant);
  int64_t total = 0;
#pragma omp parallel for reduction(+ : total) schedule(static)
  for (int64_t y = 0; y < H; ++y)
    for (int64_t x = 0; x < W; ++x) total += sh.node_edges(x, y);
  return total + pendant;
}

// road_like_graph: lattice ids y*W+x; grid edges right/down (a grid is
// 2-edge-connected, so no lattice edge is a bridge); `extra` distinct random
// edges from each node to forward neighbours within Chebyshev radius r
// (per-node SplitMix64 stream, so generation is parallel and deterministic);
// then `pendant` nodes W*H+i each attached to a uniform earlier node -- the
// pendant forest hangs off the lattice and every attaching edge is a bridge.
int ettg_gen_road_like_graph(int64_t W, int64_t H, int64_t extra, int64_t r, int64_t pendant,
                             uint64_t seed, int64_t* edges, uint8_t* truth) {
  return gen_guard([&] {
    if (W < 2 || H < 2 || r < 1 || extra < 0 || pendant < 0)
      throw GenError("road_like_graph: bad shape");
    RoadShape sh(W, H, extra, r, pendant);
    std::vector<int64_t> row_off(H + 1, 0);
#pragma omp parallel for schedule(static)
    for (int64_t y = 0; y < H; ++y) {
      int64_t c = 0;
      for (int64_t x = 0; x < W; ++x) c += sh.node_edges(x, y);
      row_off[y + 1] = c;
    }
    for (int64_t y = 0; y < H; ++y) row_off[y + 1] += row_off[y];
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t y = 0; y < H; ++y) {
      int64_t k = row_off[y];
      std::vector<int> cand;
      cand.reserve(sh.offs.size());
      for (int64_t x = 0; x < W; ++x) {
        const int64_t u = y * W + x;
        if (x + 1 < W) {
          edges[2 * k] = u;
          edges[2 * k + 1] = u + 1;
          truth[k++] = 0;
        }
        if (y + 1 < H) {
          edges[2 * k] = u;
          edges[2 * k + 1] = u + W;
          truth[k++] = 0;
        }
        cand.clear();
        for (int i = 0; i < static_cast<int>(sh.offs.size()); ++i) {
          auto [dx, dy] = sh.offs[i];
          if (x + dx >= 0 && x + dx < W && y + dy < H) cand.push_back(i);
        }
        const int take = static_cast<int>(std::min<int64_t>(extra, cand.size()));
        SplitMix64 rng(seed ^ (static_cast<uint64_t>(u) * 0xd1342543de82ef95ULL));
        for (int i = 0; i < take; ++i) {  // partial Fisher-Yates
          const int j = i + static_cast<int>(rng.next_below(cand.size() - i));
          std::swap(cand[i], cand[j]);
          auto [dx, dy] = sh.offs[cand[i]];
          edges[2 * k] = u;
          edges[2 * k + 1] = (y + dy) * W + (x + dx);
          truth[k++] = 0;
        }
      }
    }
    const int64_t nl = W * H;
    int64_t k = row_off[H];
    SplitMix64 rng(seed ^ 0x70656e64616e74ULL);
    for (int64_t i = 0; i < pendant; ++i) {
      const int64_t v = nl + i;
      const int64_t a = static_cast<int64_t>(rng.next_below(static_cast<uint64_t>(v)));
      edges[2 * k] = a;
      edges[2 * k + 1] = v;
      truth[k++] = 1;
    }
  });
}

// write_edge_list (core/src/graph.cpp:131-133): "u v\n" per edge into a
// caller buffer (host text formatting; the parsers' inverse).  *len receives
// the bytes needed; returns ETTG_ERANGE without writing past cap if short.
int ettg_write_edge_list(const int64_t* edges, int64_t m, char* out, int64_t cap, int64_t* len) {
  return gen_guard([&] {
    if (m < 0 || (m > 0 && !edges) || !len || cap < 0 || (cap > 0 && !out))
      throw std::invalid_argument("null or negative argument");
    int64_t pos = 0;
    char tmp[48];
    for (int64_t i = 0; i < m; ++i) {
      char* p = std::to_chars(tmp, tmp + 24, edges[2 * i]).ptr;
      *p++ = ' ';
      p = std::to_chars(p, tmp + 48, edges[2 * i + 1]).ptr;
      *p++ = '\n';
      const int64_t k = p - tmp;
      if (pos + k <= cap) std::memcpy(out + pos, tmp, static_cast<size_t>(k));
      pos += k;
    }
    *len = pos;
    if (pos > cap) throw std::out_of_range("text buffer too small (len returned)");
  });
}

}  // extern "C"
