/*
 * mce_oracle.h -- TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C restatement of the reference `mce` package's CPU algorithm for the
 * maximal-clique-enumeration hot path.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 *
 * Pinned against the reference itself: the JSON vectors in tests/golden were produced by
 * importing /root/reference/pkg/src/mce (tests/golden/make_golden.py) and
 * tests/test_oracle.py checks this library against every vector.
 */
#ifndef MCE_ORACLE_H
#define MCE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCE_ORACLE_HIST_MAX 4096

typedef struct {
    int64_t cliques;                       /* number of maximal cliques */
    int64_t nodes;                         /* search-tree nodes visited (reference node accounting) */
    uint64_t hash;                         /* order-independent clique-set hash (sum of per-clique hashes) */
    int64_t max_size;                      /* largest clique size seen */
    int64_t hist[MCE_ORACLE_HIST_MAX];     /* hist[s] = number of maximal cliques of size s */
} mce_oracle_result;

/* Minimum-degree peeling with a lazy binary heap keyed (current degree, id):
 * restates mce/graph.py:degeneracy_order (graph.py:183-210).  Writes the
 * rank of every vertex into position[] and returns the degeneracy. */
int64_t mce_oracle_degeneracy_order(int64_t n, const int64_t* row_offsets,
                                    const int64_t* col_indices, int64_t* position);

/* Serial/OpenMP restatement of mce/scheduler.py:_Worker._execute
 * (scheduler.py:297-381) over first-level (roots_mode=1, bk.py:186-190) or
 * second-level (roots_mode=2, bk.py:198-204) subtree roots, with full
 * (induced_full=1, induced.py:95-103) or partial (induced_full=0,
 * induced.py:61-92) induced subgraphs and the split X_P / X_X state of
 * mce/xsets.py.  The graph must be canonical and degeneracy-reordered.
 *
 *  capacity_bits : bitset capacity (reference: round_up_capacity(max(d,1)))
 *  labels        : optional map vertex -> label used by the clique hash (NULL = identity)
 *  root_begin/end/stride : the roots processed (a bounded sample for timing)
 *  include_isolated : for roots_mode=2, report isolated vertices (scheduler.py:476-480)
 *  threads       : OpenMP threads (<=0: all)
 *  collect/collect_cap : optional flat output of cliques, each written as
 *                  [size, v0, v1, ...]; *collect_len receives the words used
 * Returns 0 on success, negative on error (capacity exceeded, bad mode). */
int mce_oracle_enumerate(int64_t n, const int64_t* row_offsets, const int64_t* col_indices,
                         int roots_mode, int induced_full, int64_t capacity_bits,
                         const int64_t* labels, int64_t root_begin, int64_t root_end,
                         int64_t root_stride, int include_isolated, int threads,
                         mce_oracle_result* out, int64_t* collect, int64_t collect_cap,
                         int64_t* collect_len);

/* Per-clique hash used by every component (shared definition). */
uint64_t mce_oracle_clique_hash(const int64_t* labels_of_members, int64_t size);

#ifdef __cplusplus
}
#endif
#endif
