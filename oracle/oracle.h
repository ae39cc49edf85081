/* oracle/oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's sequential branch-and-reduce algorithm
 * (/root/reference/proj/src/{graph,search_node,reductions,bounds,solver_seq}.cpp). It is the
 * CHECKER for the CUDA engine: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it. Parity of this restatement with the reference is pinned by
 * tests/test_oracle.py against oracle/_ref (the reference itself, compiled from its sources)
 * and against the committed fixtures in tests/golden/.
 */
#ifndef VC_ORACLE_H
#define VC_ORACLE_H
#include <stdint.h>

#define ORC_REMOVED 0xFFFFFFFFu /* search_node.hpp:14 kRemoved */

typedef struct {
    uint32_t n;
    uint64_t m;
    uint64_t* off; /* n+1 */
    uint32_t* nbr; /* 2m, every slice sorted ascending */
} orc_graph;

typedef struct {
    uint32_t size;
    int32_t feasible;
    int32_t status; /* 0 complete, 2 budget */
    uint32_t greedy_size;
    uint64_t nodes;
    uint64_t stack_high_water;
} orc_result;

/* graph.cpp:22-54 make_graph. pairs = 2*num_pairs ids. Returns 0 on success. */
int orc_make_graph(uint32_t n, uint64_t num_pairs, const uint32_t* pairs, orc_graph* out);
/* graph.cpp:161-185 complement */
int orc_complement(const orc_graph* g, orc_graph* out);
void orc_graph_free(orc_graph* g);
/* graph.cpp:14-20 has_edge */
int orc_has_edge(const orc_graph* g, uint32_t u, uint32_t v);

/* reductions.cpp:7-114. which: 0 reduce_to_fixpoint(best_or_k), 1 degree rules only,
 * 2 degree-one pass, 3 degree-two-triangle pass, 4 high-degree pass. Returns changed. */
int orc_reduce(const orc_graph* g, uint32_t* deg, uint32_t* cc, uint64_t* edges, int pvc,
               uint32_t k, uint32_t best_or_k, int which);
/* bounds.cpp:21-30 */
int orc_should_prune(uint32_t cc, uint64_t edges, int pvc, uint32_t k, uint32_t best);
/* bounds.cpp:7-19; cover receives internal ids ascending; returns size */
uint32_t orc_greedy(const orc_graph* g, uint32_t* cover);
/* bounds.cpp:32-45 */
int orc_verify_cover(const orc_graph* g, const uint32_t* cover, uint32_t len);
/* solver_seq.cpp:173-211; returns size or UINT32_MAX when n > 20 */
uint32_t orc_brute_force(const orc_graph* g, uint32_t* cover);
/* search_node.cpp:85-97 */
uint64_t orc_fingerprint(const uint32_t* deg, uint32_t n, uint32_t cc, uint64_t edges);
/* solver_seq.cpp:56-159 solve_seq. node_budget 0 = none. cover (internal ids) needs n slots.
 * Returns 0, -1 for pvc with k < 1. */
int orc_solve_seq(const orc_graph* g, int pvc, uint32_t k, uint64_t node_budget,
                  orc_result* out, uint32_t* cover);

#endif
