/* TEST INFRASTRUCTURE ONLY -- never linked into the product (libettg.so).
 *
 * Plain-C restatement of the reference's hot path (eulertools core/, see
 * /root/reference/proj/core/src/{graph,euler,primitives,lca,bridges}.cpp),
 * used by tests/, __graft_entry__.smoke() and bench.py's CPU baseline as the
 * checker.  Pinned in tests/test_oracle.py against the reference's golden
 * vectors (tests/{euler,lca,primitives,bridges}_test.cpp) and against the
 * compiled reference itself (oracle/_ref).
 *
 * Return codes: 0 ok, 1 invalid_argument, 2 out_of_range; orc_last_error().
 * Ids are int64 with -1 as kNone / kTail.
 */
#ifndef ETTG_ORACLE_H_
#define ETTG_ORACLE_H_
#include <stdint.h>

const char* orc_last_error(void);

int orc_validate_tree(int64_t n, const int64_t* parent, int64_t root);
int orc_list_rank(int64_t k, const int64_t* succ, int64_t head, int64_t* out);
int orc_exclusive_scan(int64_t n, const int64_t* in, int64_t* out);
int orc_list_scan(int64_t k, const int64_t* succ, int64_t head, const int64_t* values,
                  int64_t* out);
int orc_segmented_reduce(int64_t nv, const int64_t* values, int64_t no, const int64_t* offsets,
                         int op, int64_t identity, int64_t* out);
int orc_range_index(int64_t n, const int64_t* keys, int64_t q, const int64_t* ranges,
                    int64_t* mins, int64_t* maxs);
int orc_euler_tour(int64_t n, const int64_t* parent, int64_t root, int64_t* tour_src,
                   int64_t* tour_dst);
int orc_node_stats(int64_t n, const int64_t* parent, int64_t root, int64_t* preorder,
                   int64_t* size, int64_t* level, int64_t* par);
int orc_inlabel_index(int64_t n, const int64_t* parent, int64_t root, int64_t* inlabel,
                      uint64_t* ascendant, int64_t* head, int64_t* level, int64_t* par);
/* queries on an exported index; lifts (may be NULL) receives the total
 * number of label lifts (for the roofline byte model). */
int orc_inlabel_query(int64_t n, const int64_t* inlabel, const uint64_t* ascendant,
                      const int64_t* head, const int64_t* level, const int64_t* par,
                      const int64_t* pairs, int64_t q, int64_t* answers, int64_t* lifts);
int orc_lca_inlabel(int64_t n, const int64_t* parent, int64_t root, const int64_t* pairs,
                    int64_t q, int64_t* answers);
int orc_lca_rmq(int64_t n, const int64_t* parent, int64_t root, const int64_t* pairs, int64_t q,
                int64_t* answers);
int orc_lca_walk_up(int64_t n, const int64_t* parent, const int64_t* pairs, int64_t q,
                    int64_t* answers);
int orc_tv_bridges(int64_t n, int64_t m, const int64_t* edges, uint8_t* is_bridge);
int orc_dfs_bridges(int64_t n, int64_t m, const int64_t* edges, uint8_t* is_bridge);

#endif
