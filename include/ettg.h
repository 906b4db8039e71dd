/*
 * ettg.h — C-ABI of the B200-native Euler-tour pipeline (arXiv 2103.15217).
 *
 * Drop-in boundary for the reference library's hot-path entry points
 * (namespace ett, /root/reference/proj/core/include/ett/):
 *
 *   ett::inlabel_build(const RootedTree&)            lca.hpp:26      -> ettg_lca_build
 *   ett::answer_batch(inlabel_lca, queries, batch)   lca.hpp:50-65   -> ettg_lca_query
 *   ett::rmq_lca_build / rmq_lca                     lca.hpp:46-47   -> ettg_lca_build(.., ETTG_ENGINE_RMQ)
 *                                                                       + ettg_lca_query_engine
 *   ett::node_stats(linearize(...))                  euler.hpp:55    -> ettg_lca_stats
 *   InlabelIndex fields                              lca.hpp:17-24   -> ettg_lca_inlabel_index
 *   ett::tv_bridges(const AdjacencyIndex&, PhaseTimes*) bridges.hpp:55 -> ettg_bridges
 *   ett::list_rank(const LinkedListArray&)           primitives.hpp:68 -> ettg_list_rank_dev
 *   ett::exclusive_scan(values, +, 0)                primitives.hpp:29 -> ettg_exclusive_scan_dev
 *                                                                       / ettg_exclusive_scan_i64_dev
 *   ett::list_scan(list, values)                     primitives.hpp:73 -> ettg_list_scan
 *   ett::segmented_reduce(values, offsets, f, id)    primitives.hpp:81 -> ettg_segmented_reduce
 *   ett::RangeIndex / rmq_build / rmq_min / rmq_max  primitives.hpp:100 -> ettg_range_index_*
 *   generators.hpp (grasp_tree, permute_labels, sample_queries, ...) -> ettg_gen_*
 *
 * Conventions
 *  - Ids are int64 at the host boundary (the reference's i64); kNone = -1.
 *    Device-resident variants (*_dev) take uint32 ids; 0xFFFFFFFF = none.
 *  - Host buffers are caller-owned.  A handle owns its device memory.
 *  - Host-buffer calls are synchronous.  *_dev calls enqueue on `stream`
 *    (a cudaStream_t, NULL = legacy default stream) and return immediately
 *    unless documented otherwise.
 *  - Host-buffer queries on one LCA handle from several host threads are
 *    serialised by the handle; device-resident (_dev) queries on a shared
 *    handle need no lock.  Building, exporting or freeing a handle while
 *    another thread uses it is not allowed.  Distinct handles are
 *    independent; the scratch arena and pinned staging buffers are shared
 *    per device and serialised internally.
 *  - Every function returns ETTG_OK or an error code; ettg_last_error()
 *    returns the message of the last failure on the calling thread.
 *    Error codes mirror the reference's exceptions:
 *      ETTG_EINVAL  <- std::invalid_argument (bad tree, disconnected graph,
 *                      batch < 1, n or m too large, not a list)
 *      ETTG_ERANGE  <- std::out_of_range / out-of-range query ids
 *  - There is no CPU fallback: without a usable CUDA device every compute
 *    entry point fails with ETTG_ECUDA.
 */
#ifndef ETTG_H_
#define ETTG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ETTG_OK 0
#define ETTG_EINVAL 1
#define ETTG_ERANGE 2
#define ETTG_ECUDA 3
#define ETTG_ENOMEM 4
#define ETTG_EINTERNAL 5
#define ETTG_EPARSE 6 /* malformed text input: the reference's std::runtime_error */
#define ETTG_ENCCL 7  /* NCCL failure while replicating an index across GPUs */

#define ETTG_ENGINE_INLABEL 1u /* Schieber-Vishkin inlabel (core/src/lca.cpp:20-109) */
#define ETTG_ENGINE_RMQ 2u     /* RMQ over the Euler tour (core/src/lca.cpp:128-157) */
#define ETTG_ENGINE_NAIVE 4u   /* walk-up over pointer-jumping levels (core/src/lca.cpp:111-126,
                                  core/src/primitives.cpp:208-241) */

/* Inlabel index layout (build flags, OR-ed into `engines`).  All layouts
 * give identical answers; by default the build picks one from the tree:
 *   WIDE    16-B node record {inlabel, ascendant, level}: one gather per
 *           endpoint; for trees between the two cases below.
 *   NARROW  8-B node record {inlabel, level} + ascendant per label: half the
 *           random-gather footprint, for few labels when COMPACT does not fit.
 *   COMPACT 4-B node word {label index, level - level(head)} + a dense
 *           per-label table: a quarter of the footprint, for deep trees with
 *           few inlabel paths (label-index bits + offset bits <= 32).
 *   SPLIT   8-B node record {inlabel, ascendant} + level in its own array,
 *           read only for endpoints that are not lifted (shallow trees).
 *   SPLIT_OWN 16-B {inlabel, ascendant, own-label lift record} + level:
 *           shallow-wide trees whose lifts go to the endpoint's own label
 *           (stars, caterpillars; chosen by a build-time query sample).
 *   SPLIT6  the split record packed into 6 B (n < 2^24): a 16M-node table of
 *           96 MB instead of 128 MB, which B200 gathers from ~1.3x faster.
 *   WIDE9   the wide record packed into 9 B, three per 32-B sector (n < 2^24):
 *           171 MB instead of 256 MB at 16M nodes (middle-depth trees).
 * ettg_lca_layout() reports the choice (0 wide, 1 narrow, 2 compact, 3 split,
 * 4 split_own, 5 split6, 6 wide9). */
#define ETTG_LAYOUT_WIDE 0x100u
#define ETTG_LAYOUT_NARROW 0x200u
#define ETTG_LAYOUT_COMPACT 0x400u
#define ETTG_LAYOUT_SPLIT 0x800u
#define ETTG_LAYOUT_SPLIT_OWN 0x1000u
#define ETTG_LAYOUT_SPLIT6 0x2000u
#define ETTG_LAYOUT_WIDE9 0x4000u

typedef struct ettg_lca ettg_lca;

/* Per-phase device times of one bridges call, named as the reference's
 * PhaseTimes (core/src/bridges.cpp:292-314). */
typedef struct ettg_phase_times {
  double spanning_ms; /* spanning tree: CC hooking (tv, hybrid) or BFS (ck) */
  double euler_ms;    /* Euler tour, list rank, preorder (tv, hybrid)       */
  double lowhigh_ms;  /* low/high, subtree RMQ, classification (tv)         */
  double total_ms;    /* device time of the whole call                     */
  double marking_ms;  /* CK marking + classification (ck, hybrid)          */
} ettg_phase_times;

/* Bridge engines (core/include/ett/bridges.hpp:55-62). */
#define ETTG_BRIDGES_TV 0     /* Tarjan-Vishkin (tv_bridges)                  */
#define ETTG_BRIDGES_CK 1     /* BFS tree + Chaitanya-Kothapalli marking     */
#define ETTG_BRIDGES_HYBRID 2 /* CC spanning tree + Euler rooting + marking  */

const char* ettg_last_error(void);
int ettg_version(void);
/* Number of CUDA devices visible (0 on a machine without a GPU). */
int ettg_device_count(int* count);

/* ---------------------------------------------------------------- LCA -- */

/* inlabel_build (core/src/lca.cpp:20): parent[root] == -1, every other
 * parent in [0,n).  `engines` is a bit set of ETTG_ENGINE_*; 0 means
 * ETTG_ENGINE_INLABEL.  Rejects non-trees with ETTG_EINVAL exactly where
 * validate_tree (core/src/graph.cpp:175-206) throws. */
int ettg_lca_build(const int64_t* parent, int64_t n, int64_t root, int device,
                   unsigned engines, ettg_lca** out);
/* Same, from a device-resident uint32 parent array (0xFFFFFFFF = root).
 * Synchronises `stream` before returning (the index is complete). */
int ettg_lca_build_dev(const uint32_t* d_parent, int64_t n, int64_t root,
                       int device, unsigned engines, void* stream,
                       ettg_lca** out);
void ettg_lca_free(ettg_lca* h);

int ettg_lca_size(const ettg_lca* h, int64_t* n);
/* Layout the inlabel engine queries with (0 wide, 1 narrow, 2 compact,
 * 3 split, 4 split_own, 5 split6, 6 wide9 -- also the layout code in the
 * blob header written by ettg_lca_index_export_dev) and the number of
 * inlabel paths (distinct labels) in the tree (0 for attached replicas). */
int ettg_lca_layout(const ettg_lca* h, int* layout, int64_t* labels);
/* Device time of the last build (ms), measured with CUDA events. */
int ettg_lca_build_ms(const ettg_lca* h, double* ms);

/* answer_batch(inlabel_lca, pairs, batch) (core/include/ett/lca.hpp:50-65):
 * pairs = x0,y0,x1,y1,... (2q int64), answers = q int64.  batch < 1 ->
 * ETTG_EINVAL; answers do not depend on batch.  Ids outside [0,n) give
 * ETTG_ERANGE (the reference leaves them undefined).  Host copies are
 * pipelined with the query kernel on two streams; ids and answers cross
 * the link as u32 (12 B per query), narrowed and widened by host threads. */
int ettg_lca_query(const ettg_lca* h, const int64_t* pairs, int64_t q,
                   int64_t batch, int64_t* answers);
int ettg_lca_query_engine(const ettg_lca* h, unsigned engine,
                          const int64_t* pairs, int64_t q, int64_t batch,
                          int64_t* answers);
/* Device-resident batch: d_pairs = 2q uint32, d_answers = q uint32.
 * Out-of-range ids answer 0xFFFFFFFF and raise the handle's sticky error
 * flag, which ettg_lca_query_dev_error reads (after the work on `stream`)
 * and clears: *bad = 1 if any _dev query since the last check had an id
 * outside [0, n). */
int ettg_lca_query_dev(const ettg_lca* h, unsigned engine,
                       const uint32_t* d_pairs, int64_t q, uint32_t* d_answers,
                       void* stream);
int ettg_lca_query_dev_error(const ettg_lca* h, void* stream, int* bad);

/* ancestor_doubling_levels (core/src/primitives.cpp:208-241): level[n] by
 * pointer jumping on the device (validates like validate_tree). */
int ettg_ancestor_levels(const int64_t* parent, int64_t n, int64_t root, int device,
                         int64_t* level);

/* NodeStats of the Euler tour (core/src/euler.cpp:119-155): 1-based
 * preorder, subtree size, level, parent (-1 at the root).  Any pointer may
 * be NULL.  Bit-identical to the reference (same DCEL child order). */
int ettg_lca_stats(const ettg_lca* h, int64_t* preorder, int64_t* size,
                   int64_t* level, int64_t* parent);
/* InlabelIndex fields (core/include/ett/lca.hpp:17-24): inlabel[n],
 * ascendant[n], head[n+1] (-1 where unused), level[n], parent[n]. */
int ettg_lca_inlabel_index(const ettg_lca* h, int64_t* inlabel,
                           uint64_t* ascendant, int64_t* head, int64_t* level,
                           int64_t* parent);

/* Multi-GPU replication of the inlabel index (query batches shard; the
 * index is broadcast once, e.g. with ncclBroadcast over NVLink).
 * index_bytes: size of the packed index; export copies it into a device
 * buffer of that size on the handle's device; attach builds a query-only
 * handle on `device` from such a buffer (copied). */
int ettg_lca_index_bytes(const ettg_lca* h, int64_t* bytes);
int ettg_lca_index_export_dev(const ettg_lca* h, void* d_dst, void* stream);
int ettg_lca_index_attach_dev(const void* d_src, int64_t n, int device,
                              void* stream, ettg_lca** out);
/* The CUDA device a handle's memory lives on. */
int ettg_lca_device(const ettg_lca* h, int* device);

/* ------------------------------------------------------------ multi-GPU -- */
/* the index is built once, broadcast with ncclBroadcast
 * (NVLink 5 / NVSwitch between B200s) and every GPU answers a contiguous
 * slice of the batch -- answer_batch semantics (core/include/ett/lca.hpp:
 * 50-65) over several devices, no per-query collective.  NCCL failures give
 * ETTG_ENCCL. */
#define ETTG_NCCL_ID_BYTES 128
/* Contiguous shard [*lo, *hi) of `total` units for rank `rank` of `world`
 * (sizes differ by at most one, larger first); needs no GPU. */
int ettg_shard_range(int64_t total, int rank, int world, int64_t* lo, int64_t* hi);
/* One process, many GPUs: out[i] is a query replica of `src` on devices[i]
 * (ncclCommInitAll over src's device + the distinct devices; one grouped
 * ncclBroadcast of the packed index).  Free each with ettg_lca_free. */
int ettg_lca_replicate(const ettg_lca* src, int ndev, const int* devices, ettg_lca** out);
/* One process per GPU (torchrun): every rank calls with the same
 * ETTG_NCCL_ID_BYTES id (made by ettg_nccl_unique_id on one rank and shared
 * by the caller); rank `root` passes its built index in *h, the others
 * *h == NULL (or an old replica, which is freed).  On return every rank's *h
 * answers for the root's tree on `device`. */
int ettg_nccl_unique_id(void* id);
int ettg_lca_replicate_rank(ettg_lca** h, int root, const void* id, int rank, int nranks,
                            int device);
/* A host batch sharded contiguously across `nrep` replicas (one host thread
 * each; pairs and answers as in ettg_lca_query_engine); answers in query
 * order and identical to one replica's. */
int ettg_lca_query_multi(ettg_lca* const* replicas, int nrep, unsigned engine,
                         const int64_t* pairs, int64_t q, int64_t batch,
                         int64_t* answers);

/* ------------------------------------------------------------ bridges -- */

/* tv_bridges (core/src/bridges.cpp:311-316) on the undirected simple graph
 * edges = u0,v0,u1,v1,... (2m int64, ids in [0,n)).  is_bridge[m] gets 1
 * for bridges, 0 otherwise, indexed by input edge id.  Disconnected input
 * -> ETTG_EINVAL.  times may be NULL.  The ids cross the link narrowed to
 * u32 by host threads (8 B per edge; ETTG_NARROW=0 ships pinned int64 as is). */
int ettg_bridges(const int64_t* edges, int64_t n, int64_t m, int device,
                 uint8_t* is_bridge, ettg_phase_times* times);
/* Device-resident: d_edges = 2m uint32, d_is_bridge = m bytes.  Returns
 * after the stream has completed (connectivity is checked on the host). */
int ettg_bridges_dev(const uint32_t* d_edges, int64_t n, int64_t m, int device,
                     uint8_t* d_is_bridge, void* stream,
                     ettg_phase_times* times);

/* ck_bridges / hybrid_bridges / tv_bridges by engine id. */
int ettg_bridges_engine(const int64_t* edges, int64_t n, int64_t m, int device,
                        int engine, uint8_t* is_bridge, ettg_phase_times* times);
int ettg_bridges_dev_engine(const uint32_t* d_edges, int64_t n, int64_t m,
                            int device, int engine, uint8_t* d_is_bridge,
                            void* stream, ettg_phase_times* times);

/* tv_bridges_on_tree (core/src/bridges.cpp:289-309): the TV criterion on a
 * caller-supplied spanning tree (tree_mask[m], non-zero = tree edge), which
 * replaces the hooking phase.  A mask that is not a spanning tree fails with
 * the reference's check_is_tree messages (core/src/euler.cpp:13-33):
 * ETTG_EINVAL "not a tree: m != n - 1" / "not a tree: disconnected".
 * The mask cannot change the answer (bridges are a graph property). */
int ettg_bridges_on_tree(const int64_t* edges, int64_t n, int64_t m, int device,
                         const uint8_t* tree_mask, uint8_t* is_bridge,
                         ettg_phase_times* times);
int ettg_bridges_dev_on_tree(const uint32_t* d_edges, int64_t n, int64_t m,
                             int device, const uint8_t* d_tree_mask,
                             uint8_t* d_is_bridge, void* stream,
                             ettg_phase_times* times);

/* low_high (core/src/bridges.cpp:251-287) as the TV engine computes it, for
 * checking the intermediate (diagnostic; not a timed path).  The spanning
 * tree is tree_mask (as ettg_bridges_on_tree) or, when tree_mask is NULL,
 * the engine's own hooking tree, returned in tree_out[m] (0/1) if non-NULL.
 * Per node, rooted at 0: preorder[v] (1-based, the Euler-tour order the
 * engine walks), low[v] / high[v] = the minimum / maximum preorder over v's
 * subtree and the non-tree neighbours of its subtree -- the reference's
 * LowHigh over that preorder (its test oracle recursive_low_high,
 * tests/oracles.hpp:166-201).  Errors as ettg_bridges / ettg_bridges_on_tree. */
int ettg_bridges_low_high(const int64_t* edges, int64_t n, int64_t m, int device,
                          const uint8_t* tree_mask, uint8_t* tree_out,
                          int64_t* preorder, int64_t* low, int64_t* high);

/* The engines over the reference's own input type, AdjacencyIndex
 * (core/include/ett/graph.hpp:44-61): offsets[n+1], neighbors[2m],
 * edge_ids[2m] -- what tv_bridges / ck_bridges / hybrid_bridges(const
 * AdjacencyIndex&, PhaseTimes*) (core/include/ett/bridges.hpp:55-61) take.
 * The edge list is recovered on the device by edge id (the slot of the
 * lower endpoint); the three arrays cross the link narrowed to 4 B.
 * tree_mask != NULL selects tv_bridges_on_tree (engine must be TV).
 * A CSR whose slots do not cover every edge id consistently fails with
 * ETTG_EINVAL "malformed adjacency index". */
int ettg_bridges_csr(const int64_t* offsets, const int64_t* neighbors,
                     const int64_t* edge_ids, int64_t n, int64_t m, int device,
                     int engine, const uint8_t* tree_mask, uint8_t* is_bridge,
                     ettg_phase_times* times);

/* ---------------------------------------------------------- ingestion -- */
/* build_adjacency (core/src/graph.cpp:135-173) on the device: offsets[n+1],
 * neighbors[2m], edge_ids[2m], slices sorted by (neighbor, edge id);
 * bit-identical to the reference. */
int ettg_build_adjacency(const int64_t* edges, int64_t n, int64_t m, int device,
                         int64_t* offsets, int64_t* neighbors,
                         int64_t* edge_ids);
/* bfs_tree (core/src/bridges.cpp:198-249): tree_mask[m], level[n],
 * parent[n], parent_edge[n] (-1 at the root); minimum (parent, edge id)
 * proposals, bit-identical to the reference. */
int ettg_bfs_tree(const int64_t* edges, int64_t n, int64_t m, int64_t root,
                  int device, uint8_t* tree_mask, int64_t* level,
                  int64_t* parent, int64_t* parent_edge);
/* bfs_tree(const AdjacencyIndex&, root) (core/include/ett/bridges.hpp:50). */
int ettg_bfs_tree_csr(const int64_t* offsets, const int64_t* neighbors,
                      const int64_t* edge_ids, int64_t n, int64_t m, int64_t root,
                      int device, uint8_t* tree_mask, int64_t* level,
                      int64_t* parent, int64_t* parent_edge);

/* largest_component (core/src/graph.cpp:219-259): old_to_new[n] (-1 outside),
 * the component's node count in *n_out, and its edges (renumbered, input
 * order kept) in edges_out (capacity 2m) with the count in *m_out.  Ties go to
 * the component with the smallest minimum original id, as in the reference. */
int ettg_largest_component(const int64_t* edges, int64_t n, int64_t m, int device,
                           int64_t* old_to_new, int64_t* n_out, int64_t* m_out,
                           int64_t* edges_out);

/* ------------------------------------------------------------ tuning -- */
/* cudaLimitMaxL2FetchGranularity for the device's context (bytes: 0..128).
 * Random 16-B record gathers over-fetch at the default; see DESIGN.md. */
int ettg_set_l2_fetch_granularity(int device, int bytes);
int ettg_get_l2_fetch_granularity(int device, int* bytes);

/* --------------------------------------------------------- primitives -- */

/* list_rank (core/src/primitives.cpp:145): rank[i] = links from head to i.
 * d_succ[k] uint32 with 0xFFFFFFFF as the tail.  Cycles / uncovered
 * elements -> ETTG_EINVAL.  Synchronous. */
int ettg_list_rank_dev(const uint32_t* d_succ, int64_t k, int64_t head,
                       uint32_t* d_rank, int device, void* stream);
/* exclusive_scan(values, +, 0) (core/include/ett/primitives.hpp:29-66)
 * over uint32 (sums modulo 2^32). */
int ettg_exclusive_scan_dev(const uint32_t* d_in, int64_t n, uint32_t* d_out,
                            int device, void* stream);
/* Stable sort of (key, value) uint32 pairs by key (LSD radix). */
int ettg_sort_pairs_dev(const uint32_t* d_keys, const uint32_t* d_vals,
                        int64_t n, uint32_t* d_keys_out, uint32_t* d_vals_out,
                        int device, void* stream);

/* exclusive_scan(values, +, 0) over int64 (sums wrap modulo 2^64).  d_out
 * may equal d_in. */
int ettg_exclusive_scan_i64_dev(const int64_t* d_in, int64_t n, int64_t* d_out,
                                int device, void* stream);

/* list_scan (core/src/primitives.cpp:156-162): out[i] = sum of values over
 * the elements strictly before i in list order.  succ[k] int64, -1 = tail.
 * Successors outside [-1, k), cycles and uncovered elements -> ETTG_EINVAL.
 * Synchronous. */
int ettg_list_scan(const int64_t* succ, const int64_t* values, int64_t k,
                   int64_t head, int device, int64_t* out);

/* segmented_reduce (core/include/ett/primitives.hpp:81-98):
 * out[s] = identity (op) values[offsets[s]] (op) ... (op) values[offsets[s+1]-1]
 * for s < n_offsets-1; an empty (or decreasing) segment yields identity.
 * n_offsets == 0 or offsets[n_offsets-1] != n_values -> ETTG_EINVAL
 * "segmented_reduce: bad offsets" (also for a non-empty segment reaching
 * outside [0, n_values), which the reference does not check).  The reference
 * takes any combiner; the device supports the three it uses. */
#define ETTG_REDUCE_MIN 0
#define ETTG_REDUCE_MAX 1
#define ETTG_REDUCE_SUM 2 /* wraps modulo 2^64 */
int ettg_segmented_reduce(const int64_t* values, int64_t n_values,
                          const int64_t* offsets, int64_t n_offsets, int op,
                          int64_t identity, int device, int64_t* out);
int ettg_segmented_reduce_dev(const int64_t* d_values, int64_t n_values,
                              const int64_t* d_offsets, int64_t n_offsets,
                              int op, int64_t identity, int64_t* d_out,
                              int device, void* stream); /* synchronous */

/* RangeIndex (core/include/ett/primitives.hpp:100-121,
 * core/src/primitives.cpp:169-206): inclusive range min/max over int64 keys.
 * ranges[2q] holds (l, r) pairs; mins or maxs may be NULL (not both).  Any
 * pair with l < 0, r >= n or l > r fails the whole batch with ETTG_ERANGE
 * "RangeIndex::min: bad range" ("::max" when mins is NULL).  Device layout:
 * 32-key blocks with in-block prefix/suffix {min,max} and a sparse table
 * over block extrema, so a query is at most four 16-B loads. */
typedef struct ettg_range_index ettg_range_index;
int ettg_range_index_build(const int64_t* keys, int64_t n, int device,
                           ettg_range_index** out);
int ettg_range_index_build_dev(const int64_t* d_keys, int64_t n, int device,
                               void* stream, ettg_range_index** out); /* synchronous */
int64_t ettg_range_index_size(const ettg_range_index* idx);
int ettg_range_index_query(const ettg_range_index* idx, const int64_t* ranges,
                           int64_t q, int64_t* mins, int64_t* maxs);
int ettg_range_index_query_dev(const ettg_range_index* idx,
                               const int64_t* d_ranges, int64_t q,
                               int64_t* d_mins, int64_t* d_maxs,
                               void* stream); /* synchronous (reads the error flag) */
void ettg_range_index_free(ettg_range_index* idx);

/* --------------------------------------------------------- generators -- */
/* Bit-identical to core/src/generators.cpp (SplitMix64, core/include/ett/rng.hpp). */
int ettg_gen_grasp_tree(int64_t n, uint64_t gamma, uint64_t seed,
                        int64_t* parent);
int ettg_gen_barabasi_tree(int64_t n, uint64_t seed, int64_t* parent);
int ettg_gen_permute_labels(int64_t n, const int64_t* parent, int64_t root,
                            uint64_t seed, int64_t* parent_out,
                            int64_t* root_out);
int ettg_gen_sample_queries(int64_t n, int64_t q, uint64_t seed,
                            int64_t* pairs);
int ettg_gen_random_connected_graph(int64_t n, int64_t m, uint64_t seed,
                                    int64_t* edges);
/* grasp_tree on the device in counter mode (parent[i] = draw i); u32 parent
 * array, 0xFFFFFFFF at the root 0.  *rejected as for ettg_gen_queries_dev. */
int ettg_gen_grasp_tree_dev(int64_t n, uint64_t gamma, uint64_t seed, uint32_t* d_parent,
                            int* rejected, int device, void* stream);
/* permute_labels on the device: the reference's Fisher-Yates swap sequence
 * executed as parallel rounds of deterministic reservations (bit-identical
 * to the sequential loop).  d_parent_out must not alias d_parent. */
int ettg_gen_permute_labels_dev(const uint32_t* d_parent, int64_t n, int64_t root,
                                uint64_t seed, uint32_t* d_parent_out, int64_t* root_out,
                                int* rejected, int device, void* stream);
/* sample_queries on the device in counter mode: query i of the stream
 * (offset + i) is SplitMix64 draws 2(offset+i)+1 and 2(offset+i)+2.
 * *rejected is set non-zero if any Lemire rejection occurred (the counter
 * replay is then invalid and the host generator must be used).
 * Synchronous. */
int ettg_gen_queries_dev(int64_t n, int64_t q, uint64_t seed, int64_t offset,
                         uint32_t* d_pairs, int* rejected, int device,
                         void* stream);
/* New generators for the bridge configs; truth[m] gets
 * the planted bridge mask, which is the exact answer by construction. */
int ettg_gen_planted_bridge_graph(int64_t n, int64_t m, int64_t b,
                                  uint64_t seed, int64_t* edges,
                                  uint8_t* truth);
/* Road-like: W x H lattice (row-major ids), grid edges + `extra` random
 * edges per node inside Chebyshev radius r, plus `pendant` pendant nodes
 * whose attaching edges are the planted bridges.  n = W*H + pendant,
 * m = ettg_road_like_edge_count(...). */
int64_t ettg_road_like_edge_count(int64_t W, int64_t H, int64_t extra,
                                  int64_t r, int64_t pendant);
int ettg_gen_road_like_graph(int64_t W, int64_t H, int64_t extra, int64_t r,
                             int64_t pendant, uint64_t seed, int64_t* edges,
                             uint8_t* truth);

/* ------------------------------------------------------------ ingestion -- */

/* ParseStats (core/include/ett/graph.hpp:27-32). */
typedef struct ettg_parse_stats {
  int64_t self_loops_removed;
  int64_t duplicates_removed;
} ettg_parse_stats;

/* parse_edge_list / parse_dimacs_gr (core/src/graph.cpp:57-133) on the
 * device.  `text` is the whole file (host memory, `len` bytes).  Output: n,
 * m and the normalised simple edge list (min, max) in first-occurrence
 * order into `edges` (2*cap int64).  If cap < m the call fails with
 * ETTG_ERANGE and *m holds the size needed (len/4 + 2 always suffices:
 * an edge line takes at least 4 bytes).  Malformed input gives ETTG_EPARSE with the reference's message
 * ("line N: ...").  Node ids must be < 2^32 (ETTG_ERANGE otherwise). */
int ettg_parse_edge_list(const char* text, int64_t len, int device, int64_t* edges,
                         int64_t cap, int64_t* n, int64_t* m, ettg_parse_stats* stats);
int ettg_parse_dimacs_gr(const char* text, int64_t len, int device, int64_t* edges,
                         int64_t cap, int64_t* n, int64_t* m, ettg_parse_stats* stats);
/* write_edge_list (core/src/graph.cpp:131-133): "u v\n" per edge into `out`
 * (host formatting).  *len = bytes needed; ETTG_ERANGE if cap < *len.
 * Errors are reported by ettg_gen_last_error(). */
int ettg_write_edge_list(const int64_t* edges, int64_t m, char* out, int64_t cap,
                         int64_t* len);

#ifdef __cplusplus
}
#endif
#endif /* ETTG_H_ */
