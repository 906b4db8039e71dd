/* TEST INFRASTRUCTURE ONLY -- plain-C restatement of the reference hot path.
 * See ettg_oracle.h.  Every function cites the reference lines it restates
 * (paths relative to /root/reference/proj/).  Sequential by design: this is
 * the checker, never the thing measured as "ours".
 */
#include "ettg_oracle.h"

#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define NONE (-1)
#define PLUS_INF INT64_MAX
#define MINUS_INF INT64_MIN

static __thread char g_err[256];

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

const char* orc_last_error(void) { return g_err; }

static int hb64(uint64_t x) { return 63 - __builtin_clzll(x); }
static int tz64(uint64_t x) { return __builtin_ctzll(x); }

#define ALLOC(T, cnt) ((T*)calloc((size_t)((cnt) > 0 ? (cnt) : 1), sizeof(T)))

/* ---- validate_tree: core/src/graph.cpp:175-206 ---------------------------- */
int orc_validate_tree(int64_t n, const int64_t* parent, int64_t root) {
  if (n <= 0) return fail(1, "parent array size mismatch");
  if (root < 0 || root >= n || parent[root] != NONE) return fail(1, "root has no kNone parent entry");
  int64_t roots = 0;
  for (int64_t v = 0; v < n; ++v) {
    if (parent[v] == NONE) ++roots;
    else if (parent[v] < 0 || parent[v] >= n) return fail(1, "parent id out of range");
  }
  if (roots != 1) return fail(1, "tree must have exactly one root");
  char* ok = ALLOC(char, n);
  ok[root] = 1;
  for (int64_t v = 0; v < n; ++v) {
    int64_t u = v, steps = 0;
    while (!ok[u]) {
      u = parent[u];
      if (++steps > n) {
        free(ok);
        return fail(1, "cycle in parent array");
      }
    }
    u = v;
    while (!ok[u]) {
      ok[u] = 1;
      u = parent[u];
    }
  }
  free(ok);
  return 0;
}

/* ---- list_rank_sequential / list_scan_sequential:
 *      core/src/primitives.cpp:117-141, :164-167 (values == NULL: ranks) ---- */
static int list_prefix_seq(int64_t k, const int64_t* succ, int64_t head, const int64_t* values,
                           int64_t* out) {
  if (k == 0) return 0;
  if (head < 0 || head >= k) return fail(1, "list head out of range");
  char* visited = ALLOC(char, k);
  int64_t cur = head, acc = 0, count = 0;
  while (cur != NONE) {
    if (cur < 0 || cur >= k || visited[cur]) {
      free(visited);
      return fail(1, "linked list contains a cycle");
    }
    visited[cur] = 1;
    out[cur] = acc;
    acc = (int64_t)((uint64_t)acc + (values ? (uint64_t)values[cur] : 1u));
    ++count;
    cur = succ[cur];
  }
  free(visited);
  if (count != k) return fail(1, "linked list does not cover all elements");
  return 0;
}

int orc_list_rank(int64_t k, const int64_t* succ, int64_t head, int64_t* out) {
  return list_prefix_seq(k, succ, head, NULL, out);
}

int orc_list_scan(int64_t k, const int64_t* succ, int64_t head, const int64_t* values,
                  int64_t* out) {
  return list_prefix_seq(k, succ, head, values, out);
}

/* ---- segmented_reduce: core/include/ett/primitives.hpp:81-98 ---------------
 * op 0 min, 1 max, 2 sum (wrapping). */
int orc_segmented_reduce(int64_t nv, const int64_t* values, int64_t no, const int64_t* offsets,
                         int op, int64_t identity, int64_t* out) {
  if (no <= 0 || offsets[no - 1] != nv) return fail(1, "segmented_reduce: bad offsets");
  for (int64_t s = 0; s + 1 < no; ++s) {
    int64_t acc = identity;
    for (int64_t i = offsets[s]; i < offsets[s + 1]; ++i) {
      const int64_t v = values[i];
      if (op == 0) acc = v < acc ? v : acc;
      else if (op == 1) acc = v > acc ? v : acc;
      else acc = (int64_t)((uint64_t)acc + (uint64_t)v);
    }
    out[s] = acc;
  }
  return 0;
}

/* ---- exclusive_scan(+): core/include/ett/primitives.hpp:29-66 -------------- */
int orc_exclusive_scan(int64_t n, const int64_t* in, int64_t* out) {
  int64_t acc = 0;
  for (int64_t i = 0; i < n; ++i) {
    out[i] = acc;
    acc += in[i];
  }
  return 0;
}

/* ---- HalfEdgeStructure: core/src/euler.cpp:38-90 --------------------------- */
typedef struct {
  int64_t n, k;
  int64_t *src, *dst, *twin, *next, *first;
} HE;

static void he_free(HE* h) {
  free(h->src);
  free(h->dst);
  free(h->twin);
  free(h->next);
  free(h->first);
}

/* check_is_tree: core/src/euler.cpp:13-34 */
static int64_t uf_find(int64_t* uf, int64_t v) {
  while (uf[v] != v) v = uf[v] = uf[uf[v]];
  return v;
}

static int check_is_tree(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev) {
  if (m != n - 1) return fail(1, "not a tree: m != n - 1");
  int64_t* uf = ALLOC(int64_t, n);
  for (int64_t i = 0; i < n; ++i) uf[i] = i;
  int64_t merges = 0;
  for (int64_t i = 0; i < m; ++i) {
    int64_t a = uf_find(uf, eu[i]), b = uf_find(uf, ev[i]);
    if (a != b) {
      uf[a] = b;
      ++merges;
    }
  }
  free(uf);
  if (merges != n - 1) return fail(1, "not a tree: disconnected");
  return 0;
}

static void counting_pass(int64_t n, int64_t k, const int64_t* in, int64_t* out,
                          const int64_t* key) {
  int64_t* count = ALLOC(int64_t, n + 1);
  for (int64_t i = 0; i < k; ++i) ++count[key[in[i]] + 1];
  for (int64_t i = 0; i < n; ++i) count[i + 1] += count[i];
  for (int64_t i = 0; i < k; ++i) out[count[key[in[i]]]++] = in[i];
  free(count);
}

static int he_build(int64_t n, int64_t m, const int64_t* eu, const int64_t* ev, int validate,
                    HE* h) {
  memset(h, 0, sizeof *h);
  if (n <= 0) return fail(1, "empty node set");
  if (validate) {
    int rc = check_is_tree(n, m, eu, ev);
    if (rc) return rc;
  }
  const int64_t k = 2 * m;
  h->n = n;
  h->k = k;
  h->first = ALLOC(int64_t, n);
  for (int64_t i = 0; i < n; ++i) h->first[i] = NONE;
  h->src = ALLOC(int64_t, k);
  h->dst = ALLOC(int64_t, k);
  h->twin = ALLOC(int64_t, k);
  h->next = ALLOC(int64_t, k);
  if (k == 0) return 0;
  int64_t* as = ALLOC(int64_t, k);
  int64_t* ad = ALLOC(int64_t, k);
  for (int64_t i = 0; i < m; ++i) {
    as[2 * i] = eu[i];
    ad[2 * i] = ev[i];
    as[2 * i + 1] = ev[i];
    ad[2 * i + 1] = eu[i];
  }
  int64_t* perm = ALLOC(int64_t, k);
  int64_t* tmp = ALLOC(int64_t, k);
  for (int64_t i = 0; i < k; ++i) tmp[i] = i;
  counting_pass(n, k, tmp, perm, ad); /* by dst */
  memcpy(tmp, perm, k * sizeof(int64_t));
  counting_pass(n, k, tmp, perm, as); /* then by src: lexicographic (src, dst) */
  int64_t* inv = ALLOC(int64_t, k);
  for (int64_t b = 0; b < k; ++b) inv[perm[b]] = b;
  for (int64_t b = 0; b < k; ++b) {
    h->src[b] = as[perm[b]];
    h->dst[b] = ad[perm[b]];
    h->twin[b] = inv[perm[b] ^ 1];
  }
  for (int64_t b = 0; b < k; ++b)
    if (b == 0 || h->src[b - 1] != h->src[b]) h->first[h->src[b]] = b;
  for (int64_t b = 0; b < k; ++b)
    h->next[b] = (b + 1 < k && h->src[b + 1] == h->src[b]) ? b + 1 : h->first[h->src[b]];
  free(as);
  free(ad);
  free(perm);
  free(tmp);
  free(inv);
  return 0;
}

/* ---- linearize: core/src/euler.cpp:92-117 ----------------------------------- */
static int linearize(const HE* h, int64_t root, int64_t* order, int64_t* pos) {
  if (root < 0 || root >= h->n) return fail(1, "root out of range");
  const int64_t k = h->k;
  if (k == 0) return 0;
  int64_t* succ = ALLOC(int64_t, k);
  for (int64_t e = 0; e < k; ++e) succ[e] = h->next[h->twin[e]];
  int64_t last = h->first[root];
  while (h->next[last] != h->first[root]) last = h->next[last];
  succ[h->twin[last]] = NONE;
  int rc = list_prefix_seq(k, succ, h->first[root], NULL, pos);
  free(succ);
  if (rc) return rc;
  for (int64_t e = 0; e < k; ++e) order[pos[e]] = e;
  return 0;
}

/* ---- node_stats: core/src/euler.cpp:119-155 --------------------------------- */
static void node_stats(const HE* h, int64_t root, const int64_t* order, const int64_t* pos,
                       int64_t* pre, int64_t* size, int64_t* level, int64_t* par) {
  const int64_t n = h->n, k = h->k;
  for (int64_t v = 0; v < n; ++v) {
    pre[v] = size[v] = level[v] = 0;
    par[v] = NONE;
  }
  pre[root] = 1;
  size[root] = n;
  if (k == 0) return;
  int64_t d = 0, l = 0; /* running exclusive scans of down / level weights */
  for (int64_t t = 0; t < k; ++t) {
    const int64_t e = order[t];
    const int down = pos[e] < pos[h->twin[e]];
    if (down) {
      const int64_t v = h->dst[e];
      pre[v] = d + 2;
      level[v] = l + 1;
      par[v] = h->src[e];
      size[v] = (pos[h->twin[e]] - t + 1) / 2;
    }
    d += down ? 1 : 0;
    l += down ? 1 : -1;
  }
}

/* stats_for_tree: core/src/lca.cpp:12-16 (tree_edges graph.cpp:208-217) */
static int tree_stats(int64_t n, const int64_t* parent, int64_t root, int64_t* pre,
                      int64_t* size, int64_t* level, int64_t* par, HE* h_out, int64_t** order_out) {
  int rc = orc_validate_tree(n, parent, root);
  if (rc) return rc;
  int64_t* eu = ALLOC(int64_t, n);
  int64_t* ev = ALLOC(int64_t, n);
  int64_t m = 0;
  for (int64_t v = 0; v < n; ++v) {
    if (parent[v] == NONE) continue;
    eu[m] = v < parent[v] ? v : parent[v];
    ev[m] = v < parent[v] ? parent[v] : v;
    ++m;
  }
  HE h;
  rc = he_build(n, m, eu, ev, 0, &h);
  free(eu);
  free(ev);
  if (rc) return rc;
  int64_t* order = ALLOC(int64_t, h.k);
  int64_t* pos = ALLOC(int64_t, h.k);
  rc = linearize(&h, root, order, pos);
  if (!rc) node_stats(&h, root, order, pos, pre, size, level, par);
  free(pos);
  if (h_out && !rc) {
    *h_out = h;
    *order_out = order;
  } else {
    free(order);
    he_free(&h);
  }
  return rc;
}

int orc_node_stats(int64_t n, const int64_t* parent, int64_t root, int64_t* pre, int64_t* size,
                   int64_t* level, int64_t* par) {
  return tree_stats(n, parent, root, pre, size, level, par, NULL, NULL);
}

int orc_euler_tour(int64_t n, const int64_t* parent, int64_t root, int64_t* tour_src,
                   int64_t* tour_dst) {
  int64_t* a = ALLOC(int64_t, 4 * n);
  HE h;
  int64_t* order = NULL;
  int rc = tree_stats(n, parent, root, a, a + n, a + 2 * n, a + 3 * n, &h, &order);
  free(a);
  if (rc) return rc;
  for (int64_t t = 0; t < h.k; ++t) {
    tour_src[t] = h.src[order[t]];
    tour_dst[t] = h.dst[order[t]];
  }
  free(order);
  he_free(&h);
  return 0;
}

/* ---- inlabel_build: core/src/lca.cpp:20-82 ---------------------------------- */
int orc_inlabel_index(int64_t n, const int64_t* parent, int64_t root, int64_t* inlabel,
                      uint64_t* asc, int64_t* head, int64_t* level, int64_t* par) {
  if (n >= ((int64_t)1 << 62)) return fail(1, "tree too large for 64-bit inlabel masks");
  int64_t* pre = ALLOC(int64_t, n);
  int64_t* size = ALLOC(int64_t, n);
  int rc = tree_stats(n, parent, root, pre, size, level, par, NULL, NULL);
  if (rc) {
    free(pre);
    free(size);
    return rc;
  }
  for (int64_t v = 0; v < n; ++v) {
    const int64_t l = pre[v], r = pre[v] + size[v] - 1;
    if (l == r) inlabel[v] = l;
    else inlabel[v] = r & ~(((int64_t)1 << hb64((uint64_t)((l - 1) ^ r))) - 1);
  }
  for (int64_t i = 0; i <= n; ++i) head[i] = NONE;
  for (int64_t v = 0; v < n; ++v)
    if (par[v] == NONE || inlabel[par[v]] != inlabel[v]) head[inlabel[v]] = v;
  uint64_t* path_asc = ALLOC(uint64_t, n + 1);
  char* resolved = ALLOC(char, n + 1);
  const int max_rounds = hb64((uint64_t)n) + 2;
  for (int round = 0; round < max_rounds; ++round) {
    for (int64_t label = 0; label <= n; ++label) {
      const int64_t hd = head[label];
      if (hd == NONE || resolved[label]) continue;
      const uint64_t bit = (uint64_t)1 << tz64((uint64_t)label);
      if (par[hd] == NONE) {
        path_asc[label] = bit;
        resolved[label] = 1;
      } else {
        const int64_t up = inlabel[par[hd]];
        if (resolved[up]) {
          path_asc[label] = path_asc[up] | bit;
          resolved[label] = 1;
        }
      }
    }
  }
  for (int64_t v = 0; v < n; ++v) asc[v] = path_asc[inlabel[v]];
  free(path_asc);
  free(resolved);
  free(pre);
  free(size);
  return 0;
}

/* ---- inlabel_lca: core/src/lca.cpp:84-109 ----------------------------------- */
static int64_t inlabel_lca(const int64_t* inl, const uint64_t* asc, const int64_t* head,
                           const int64_t* level, const int64_t* par, int64_t x, int64_t y,
                           int64_t* lifts) {
  const int64_t ix = inl[x], iy = inl[y];
  if (ix == iy) return level[x] <= level[y] ? x : y;
  const int i = hb64((uint64_t)(ix ^ iy));
  uint64_t common = asc[x] & asc[y];
  common &= ~(((uint64_t)1 << i) - 1);
  const int j = tz64(common);
  const int64_t target = (int64_t)(((uint64_t)ix & ~(((uint64_t)2 << j) - 1)) | ((uint64_t)1 << j));
  int64_t hv[2];
  const int64_t vs[2] = {x, y};
  for (int s = 0; s < 2; ++s) {
    const int64_t v = vs[s];
    if (inl[v] == target) {
      hv[s] = v;
      continue;
    }
    const uint64_t below = asc[v] & (((uint64_t)1 << j) - 1);
    const int k = hb64(below);
    const int64_t w = (int64_t)(((uint64_t)inl[v] & ~(((uint64_t)2 << k) - 1)) | ((uint64_t)1 << k));
    hv[s] = par[head[w]];
    if (lifts) ++*lifts;
  }
  return level[hv[0]] <= level[hv[1]] ? hv[0] : hv[1];
}

int orc_inlabel_query(int64_t n, const int64_t* inl, const uint64_t* asc, const int64_t* head,
                      const int64_t* level, const int64_t* par, const int64_t* pairs, int64_t q,
                      int64_t* answers, int64_t* lifts) {
  if (lifts) *lifts = 0;
  for (int64_t i = 0; i < q; ++i) {
    const int64_t x = pairs[2 * i], y = pairs[2 * i + 1];
    if (x < 0 || x >= n || y < 0 || y >= n) return fail(2, "query node id out of range");
    answers[i] = inlabel_lca(inl, asc, head, level, par, x, y, lifts);
  }
  return 0;
}

int orc_lca_inlabel(int64_t n, const int64_t* parent, int64_t root, const int64_t* pairs,
                    int64_t q, int64_t* answers) {
  int64_t* inl = ALLOC(int64_t, n);
  uint64_t* asc = ALLOC(uint64_t, n);
  int64_t* head = ALLOC(int64_t, n + 1);
  int64_t* level = ALLOC(int64_t, n);
  int64_t* par = ALLOC(int64_t, n);
  int rc = orc_inlabel_index(n, parent, root, inl, asc, head, level, par);
  if (!rc) rc = orc_inlabel_query(n, inl, asc, head, level, par, pairs, q, answers, NULL);
  free(inl);
  free(asc);
  free(head);
  free(level);
  free(par);
  return rc;
}

/* ---- RangeIndex: core/src/primitives.cpp:169-206 ---------------------------- */
typedef struct {
  int64_t size, leaves;
  int64_t *mn, *mx;
} RI;

static void ri_build(RI* r, const int64_t* keys, int64_t size) {
  r->size = size;
  r->leaves = 1;
  while (r->leaves < (size > 1 ? size : 1)) r->leaves <<= 1;
  r->mn = ALLOC(int64_t, 2 * r->leaves);
  r->mx = ALLOC(int64_t, 2 * r->leaves);
  for (int64_t i = 0; i < 2 * r->leaves; ++i) {
    r->mn[i] = PLUS_INF;
    r->mx[i] = MINUS_INF;
  }
  for (int64_t i = 0; i < size; ++i) r->mn[r->leaves + i] = r->mx[r->leaves + i] = keys[i];
  for (int64_t i = r->leaves - 1; i >= 1; --i) {
    r->mn[i] = r->mn[2 * i] < r->mn[2 * i + 1] ? r->mn[2 * i] : r->mn[2 * i + 1];
    r->mx[i] = r->mx[2 * i] > r->mx[2 * i + 1] ? r->mx[2 * i] : r->mx[2 * i + 1];
  }
}

static int64_t ri_min(const RI* r, int64_t l, int64_t h) {
  int64_t res = PLUS_INF;
  for (l += r->leaves, h += r->leaves + 1; l < h; l >>= 1, h >>= 1) {
    if (l & 1) { int64_t v = r->mn[l++]; if (v < res) res = v; }
    if (h & 1) { int64_t v = r->mn[--h]; if (v < res) res = v; }
  }
  return res;
}

static int64_t ri_max(const RI* r, int64_t l, int64_t h) {
  int64_t res = MINUS_INF;
  for (l += r->leaves, h += r->leaves + 1; l < h; l >>= 1, h >>= 1) {
    if (l & 1) { int64_t v = r->mx[l++]; if (v > res) res = v; }
    if (h & 1) { int64_t v = r->mx[--h]; if (v > res) res = v; }
  }
  return res;
}

static void ri_free(RI* r) {
  free(r->mn);
  free(r->mx);
}

/* RangeIndex::min / ::max (core/src/primitives.cpp:184-206): the first bad
 * range fails the batch with out_of_range. */
int orc_range_index(int64_t n, const int64_t* keys, int64_t q, const int64_t* ranges,
                    int64_t* mins, int64_t* maxs) {
  RI r;
  ri_build(&r, keys, n);
  for (int64_t i = 0; i < q; ++i) {
    const int64_t l = ranges[2 * i], h = ranges[2 * i + 1];
    if (l < 0 || h >= n || l > h) {
      ri_free(&r);
      return fail(2, mins ? "RangeIndex::min: bad range" : "RangeIndex::max: bad range");
    }
    if (mins) mins[i] = ri_min(&r, l, h);
    if (maxs) maxs[i] = ri_max(&r, l, h);
  }
  ri_free(&r);
  return 0;
}

/* ---- rmq_lca_build / rmq_lca: core/src/lca.cpp:128-157 ---------------------- */
int orc_lca_rmq(int64_t n, const int64_t* parent, int64_t root, const int64_t* pairs, int64_t q,
                int64_t* answers) {
  int64_t* a = ALLOC(int64_t, 4 * n);
  HE h;
  int64_t* order = NULL;
  int rc = tree_stats(n, parent, root, a, a + n, a + 2 * n, a + 3 * n, &h, &order);
  if (rc) {
    free(a);
    return rc;
  }
  const int64_t* level = a + 2 * n;
  const int64_t steps = h.k + 1;
  int64_t* tour = ALLOC(int64_t, steps);
  int64_t* keys = ALLOC(int64_t, steps);
  tour[0] = root;
  keys[0] = 0;
  for (int64_t t = 0; t < steps - 1; ++t) {
    const int64_t v = h.dst[order[t]];
    tour[t + 1] = v;
    keys[t + 1] = (level[v] << 32) | (t + 1);
  }
  int64_t* first = ALLOC(int64_t, n);
  for (int64_t v = 0; v < n; ++v) first[v] = PLUS_INF;
  for (int64_t t = 0; t < steps; ++t)
    if (first[tour[t]] == PLUS_INF) first[tour[t]] = t;
  RI ri;
  ri_build(&ri, keys, steps);
  for (int64_t i = 0; i < q; ++i) {
    const int64_t x = pairs[2 * i], y = pairs[2 * i + 1];
    if (x < 0 || x >= n || y < 0 || y >= n) {
      rc = fail(2, "query node id out of range");
      break;
    }
    int64_t l = first[x], r = first[y];
    if (l > r) {
      int64_t t = l;
      l = r;
      r = t;
    }
    answers[i] = tour[ri_min(&ri, l, r) & 0xffffffff];
  }
  ri_free(&ri);
  free(first);
  free(keys);
  free(tour);
  free(order);
  he_free(&h);
  free(a);
  return rc;
}

/* ---- walk_up_lca: tests/oracles.hpp:30-53 ------------------------------------ */
int orc_lca_walk_up(int64_t n, const int64_t* parent, const int64_t* pairs, int64_t q,
                    int64_t* answers) {
  int64_t* depth = ALLOC(int64_t, n);
  for (int64_t v = 0; v < n; ++v) {
    int64_t u = v, d = 0;
    while (parent[u] != NONE) {
      u = parent[u];
      ++d;
    }
    depth[v] = d;
  }
  for (int64_t i = 0; i < q; ++i) {
    int64_t x = pairs[2 * i], y = pairs[2 * i + 1];
    int64_t dx = depth[x], dy = depth[y];
    while (dx > dy) { x = parent[x]; --dx; }
    while (dy > dx) { y = parent[y]; --dy; }
    while (x != y) { x = parent[x]; y = parent[y]; }
    answers[i] = x;
  }
  free(depth);
  return 0;
}

/* ---- build_adjacency: core/src/graph.cpp:135-173 ---------------------------- */
typedef struct {
  int64_t n, m;
  int64_t *off, *nbr, *eid;
} Adj;

static int cmp_pair(const void* a, const void* b) {
  const int64_t* x = (const int64_t*)a;
  const int64_t* y = (const int64_t*)b;
  if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
  if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
  return 0;
}

static int adj_build(int64_t n, int64_t m, const int64_t* e, Adj* g) {
  memset(g, 0, sizeof *g);
  g->n = n;
  g->m = m;
  int64_t* deg = ALLOC(int64_t, n);
  for (int64_t i = 0; i < m; ++i) {
    const int64_t u = e[2 * i], v = e[2 * i + 1];
    if (u < 0 || u >= n || v < 0 || v >= n) {
      free(deg);
      return fail(1, "edge endpoint out of range");
    }
    ++deg[u];
    ++deg[v];
  }
  g->off = ALLOC(int64_t, n + 1);
  for (int64_t v = 0; v < n; ++v) g->off[v + 1] = g->off[v] + deg[v];
  g->nbr = ALLOC(int64_t, 2 * m);
  g->eid = ALLOC(int64_t, 2 * m);
  int64_t* cur = deg;
  for (int64_t v = 0; v < n; ++v) cur[v] = g->off[v];
  for (int64_t i = 0; i < m; ++i) {
    const int64_t u = e[2 * i], v = e[2 * i + 1];
    g->nbr[cur[u]] = v;
    g->eid[cur[u]++] = i;
    g->nbr[cur[v]] = u;
    g->eid[cur[v]++] = i;
  }
  free(deg);
  int64_t* tmp = ALLOC(int64_t, 2 * (2 * m));
  for (int64_t v = 0; v < n; ++v) {
    const int64_t lo = g->off[v], hi = g->off[v + 1];
    for (int64_t i = lo; i < hi; ++i) {
      tmp[2 * (i - lo)] = g->nbr[i];
      tmp[2 * (i - lo) + 1] = g->eid[i];
    }
    qsort(tmp, (size_t)(hi - lo), 2 * sizeof(int64_t), cmp_pair);
    for (int64_t i = lo; i < hi; ++i) {
      g->nbr[i] = tmp[2 * (i - lo)];
      g->eid[i] = tmp[2 * (i - lo) + 1];
    }
  }
  free(tmp);
  return 0;
}

static void adj_free(Adj* g) {
  free(g->off);
  free(g->nbr);
  free(g->eid);
}

/* ---- spanning_tree_hooking: core/src/bridges.cpp:105-158 -------------------- */
static int hooking(const Adj* g, char* mask) {
  if (g->n >= ((int64_t)1 << 31) || g->m >= ((int64_t)1 << 31))
    return fail(1, "graph too large for packed hooking keys");
  if (g->n == 0) return fail(1, "empty graph");
  memset(mask, 0, (size_t)g->m);
  if (g->n == 1) return 0;
  const int64_t n = g->n;
  int64_t* comp = ALLOC(int64_t, n);
  int64_t* hook = ALLOC(int64_t, n);
  uint64_t* best = ALLOC(uint64_t, n);
  for (int64_t v = 0; v < n; ++v) comp[v] = v;
  int rc = 0;
  for (;;) {
    for (int64_t c = 0; c < n; ++c) {
      best[c] = UINT64_MAX;
      hook[c] = c;
    }
    for (int64_t u = 0; u < n; ++u)
      for (int64_t i = g->off[u]; i < g->off[u + 1]; ++i) {
        const int64_t cu = comp[u], cv = comp[g->nbr[i]];
        if (cu == cv) continue;
        const uint64_t key = ((uint64_t)cv << 32) | (uint64_t)g->eid[i];
        if (key < best[cu]) best[cu] = key;
      }
    int64_t hooks = 0;
    for (int64_t c = 0; c < n; ++c) {
      if (best[c] == UINT64_MAX) continue;
      const int64_t target = (int64_t)(best[c] >> 32);
      if (target >= c) continue;
      hook[c] = target;
      mask[best[c] & 0xffffffff] = 1;
      ++hooks;
    }
    if (hooks == 0) {
      for (int64_t v = 0; v < n; ++v)
        if (comp[v] != comp[0]) {
          rc = fail(1, "disconnected graph; extract the largest component first");
          break;
        }
      break;
    }
    for (int64_t v = 0; v < n; ++v) {
      int64_t r = comp[v];
      while (hook[r] != r) r = hook[r];
      comp[v] = r;
    }
  }
  free(comp);
  free(hook);
  free(best);
  return rc;
}

/* ---- tv_bridges: core/src/bridges.cpp:160-196, :251-316 --------------------- */
int orc_tv_bridges(int64_t n, int64_t m, const int64_t* edges, uint8_t* is_bridge) {
  Adj g;
  int rc = adj_build(n, m, edges, &g);
  if (rc) return rc;
  char* mask = ALLOC(char, m);
  rc = hooking(&g, mask);
  if (rc || n == 1) {
    if (!rc) memset(is_bridge, 0, (size_t)m);
    free(mask);
    adj_free(&g);
    return rc;
  }
  /* euler_root_tree (:160-196): tree edges in id order, endpoints from adj */
  int64_t* tid = ALLOC(int64_t, n);
  int64_t t = 0;
  for (int64_t e = 0; e < m; ++e)
    if (mask[e]) tid[t++] = e;
  int64_t* epu = ALLOC(int64_t, m);
  int64_t* epv = ALLOC(int64_t, m);
  for (int64_t e = 0; e < m; ++e) epu[e] = epv[e] = NONE;
  for (int64_t v = 0; v < n; ++v)
    for (int64_t i = g.off[v]; i < g.off[v + 1]; ++i)
      if (mask[g.eid[i]] && v < g.nbr[i]) {
        epu[g.eid[i]] = v;
        epv[g.eid[i]] = g.nbr[i];
      }
  int64_t* tu = ALLOC(int64_t, t);
  int64_t* tv = ALLOC(int64_t, t);
  for (int64_t i = 0; i < t; ++i) {
    tu[i] = epu[tid[i]];
    tv[i] = epv[tid[i]];
  }
  free(epu);
  free(epv);
  HE h;
  rc = he_build(n, t, tu, tv, 1, &h);
  int64_t *order = NULL, *pos = NULL, *pre = NULL, *size = NULL, *level = NULL, *par = NULL,
          *pedge = NULL;
  if (!rc) {
    order = ALLOC(int64_t, h.k);
    pos = ALLOC(int64_t, h.k);
    rc = linearize(&h, 0, order, pos);
  }
  if (!rc) {
    pre = ALLOC(int64_t, n);
    size = ALLOC(int64_t, n);
    level = ALLOC(int64_t, n);
    par = ALLOC(int64_t, n);
    node_stats(&h, 0, order, pos, pre, size, level, par);
    pedge = ALLOC(int64_t, n);
    for (int64_t v = 0; v < n; ++v) pedge[v] = NONE;
    for (int64_t i = 0; i < t; ++i) {
      const int64_t child = par[tu[i]] == tv[i] ? tu[i] : tv[i];
      pedge[child] = tid[i];
    }
    /* low_high (:251-287) */
    int64_t* nmin = ALLOC(int64_t, n);
    int64_t* nmax = ALLOC(int64_t, n);
    for (int64_t v = 0; v < n; ++v) {
      int64_t lo = PLUS_INF, hi = MINUS_INF;
      for (int64_t i = g.off[v]; i < g.off[v + 1]; ++i) {
        if (mask[g.eid[i]]) continue;
        const int64_t p = pre[g.nbr[i]];
        if (p < lo) lo = p;
        if (p > hi) hi = p;
      }
      nmin[v] = lo;
      nmax[v] = hi;
    }
    int64_t* bmin = ALLOC(int64_t, n);
    int64_t* bmax = ALLOC(int64_t, n);
    for (int64_t v = 0; v < n; ++v) {
      bmin[pre[v] - 1] = nmin[v] < pre[v] ? nmin[v] : pre[v];
      bmax[pre[v] - 1] = nmax[v] > pre[v] ? nmax[v] : pre[v];
    }
    RI rmin, rmax;
    ri_build(&rmin, bmin, n);
    ri_build(&rmax, bmax, n);
    /* classify (:301-306) */
    memset(is_bridge, 0, (size_t)m);
    for (int64_t v = 0; v < n; ++v) {
      if (pedge[v] == NONE) continue;
      const int64_t lo = pre[v] - 1, hi = lo + size[v] - 1;
      const int64_t low = ri_min(&rmin, lo, hi), high = ri_max(&rmax, lo, hi);
      is_bridge[pedge[v]] = (low >= pre[v] && high < pre[v] + size[v]) ? 1 : 0;
    }
    ri_free(&rmin);
    ri_free(&rmax);
    free(nmin);
    free(nmax);
    free(bmin);
    free(bmax);
  }
  free(order);
  free(pos);
  free(pre);
  free(size);
  free(level);
  free(par);
  free(pedge);
  free(tu);
  free(tv);
  free(tid);
  he_free(&h);
  free(mask);
  adj_free(&g);
  return rc;
}

/* ---- dfs_bridges: core/src/bridges.cpp:341-381 ------------------------------- */
int orc_dfs_bridges(int64_t n, int64_t m, const int64_t* edges, uint8_t* is_bridge) {
  Adj g;
  int rc = adj_build(n, m, edges, &g);
  if (rc) return rc;
  memset(is_bridge, 0, (size_t)m);
  if (n == 0) {
    adj_free(&g);
    return fail(1, "empty graph");
  }
  int64_t* pre = ALLOC(int64_t, n);
  int64_t* low = ALLOC(int64_t, n);
  int64_t* cursor = ALLOC(int64_t, n);
  int64_t* entry = ALLOC(int64_t, n);
  int64_t* stack = ALLOC(int64_t, n);
  for (int64_t v = 0; v < n; ++v) entry[v] = NONE;
  int64_t sp = 0, counter = 0;
  stack[sp++] = 0;
  pre[0] = low[0] = ++counter;
  while (sp > 0) {
    const int64_t v = stack[sp - 1];
    if (cursor[v] < g.off[v + 1] - g.off[v]) {
      const int64_t i = g.off[v] + cursor[v]++;
      const int64_t w = g.nbr[i], e = g.eid[i];
      if (e == entry[v]) continue;
      if (pre[w] == 0) {
        pre[w] = low[w] = ++counter;
        entry[w] = e;
        stack[sp++] = w;
      } else if (pre[w] < low[v]) {
        low[v] = pre[w];
      }
    } else {
      --sp;
      if (sp > 0) {
        const int64_t p = stack[sp - 1];
        if (low[v] < low[p]) low[p] = low[v];
        if (low[v] >= pre[v]) is_bridge[entry[v]] = 1;
      }
    }
  }
  if (counter != n) rc = fail(1, "disconnected graph; extract the largest component first");
  free(pre);
  free(low);
  free(cursor);
  free(entry);
  free(stack);
  adj_free(&g);
  return rc;
}
