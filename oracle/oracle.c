/* oracle/oracle.c — TEST INFRASTRUCTURE ONLY (the checker; never linked into the product).
 *
 * Plain-C restatement of the reference's sequential algorithm. Each function cites the
 * reference file:line (paths relative to /root/reference/proj) it restates. Pinned against the
 * reference itself (oracle/_ref/libvcref.so) and tests/golden/ by tests/test_oracle.py.
 */
#include "oracle.h"

#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- graph (graph.cpp) */

static int cmp_pair(const void* a, const void* b) {
    const uint32_t* x = (const uint32_t*)a;
    const uint32_t* y = (const uint32_t*)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
    return 0;
}

/* graph.cpp:22-54: drop self-loops, orient u<v, sort, dedupe, count, prefix-sum, fill. */
int orc_make_graph(uint32_t n, uint64_t num_pairs, const uint32_t* pairs, orc_graph* out) {
    uint32_t* c = (uint32_t*)malloc((num_pairs ? num_pairs : 1) * 2 * sizeof(uint32_t));
    uint64_t k = 0;
    for (uint64_t i = 0; i < num_pairs; ++i) {
        uint32_t u = pairs[2 * i], v = pairs[2 * i + 1];
        if (u == v) continue;
        if (u > v) { uint32_t t = u; u = v; v = t; }
        if (v >= n) { free(c); return -1; }
        c[2 * k] = u; c[2 * k + 1] = v; ++k;
    }
    qsort(c, k, 2 * sizeof(uint32_t), cmp_pair);
    uint64_t m = 0;
    for (uint64_t i = 0; i < k; ++i) {
        if (m && c[2 * (m - 1)] == c[2 * i] && c[2 * (m - 1) + 1] == c[2 * i + 1]) continue;
        c[2 * m] = c[2 * i]; c[2 * m + 1] = c[2 * i + 1]; ++m;
    }
    out->n = n;
    out->m = m;
    out->off = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
    out->nbr = (uint32_t*)malloc((m ? 2 * m : 1) * sizeof(uint32_t));
    for (uint64_t i = 0; i < m; ++i) { out->off[c[2 * i] + 1]++; out->off[c[2 * i + 1] + 1]++; }
    for (uint32_t v = 0; v < n; ++v) out->off[v + 1] += out->off[v];
    uint64_t* cur = (uint64_t*)malloc(((size_t)n + 1) * sizeof(uint64_t));
    memcpy(cur, out->off, ((size_t)n + 1) * sizeof(uint64_t));
    /* (u,v) sorted lexicographically, so every slice is filled in ascending order. */
    for (uint64_t i = 0; i < m; ++i) {
        uint32_t u = c[2 * i], v = c[2 * i + 1];
        out->nbr[cur[u]++] = v;
        out->nbr[cur[v]++] = u;
    }
    free(cur);
    free(c);
    return 0;
}

/* graph.cpp:161-185 */
int orc_complement(const orc_graph* g, orc_graph* out) {
    uint64_t n = g->n;
    uint64_t total = n * (n - (n > 0 ? 1 : 0)) / 2;
    out->n = g->n;
    out->m = total - g->m;
    out->off = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
    out->nbr = (uint32_t*)malloc((out->m ? 2 * out->m : 1) * sizeof(uint32_t));
    uint64_t pos = 0;
    for (uint32_t v = 0; v < g->n; ++v) {
        out->off[v] = pos;
        uint64_t i = g->off[v], e = g->off[v + 1];
        for (uint32_t u = 0; u < g->n; ++u) {
            if (u == v) continue;
            while (i < e && g->nbr[i] < u) ++i;
            if (i < e && g->nbr[i] == u) continue;
            out->nbr[pos++] = u;
        }
    }
    out->off[g->n] = pos;
    return 0;
}

void orc_graph_free(orc_graph* g) {
    free(g->off);
    free(g->nbr);
    g->off = NULL;
    g->nbr = NULL;
}

/* graph.cpp:14-20: binary search in the shorter slice */
int orc_has_edge(const orc_graph* g, uint32_t u, uint32_t v) {
    if (u == v) return 0;
    if (g->off[u + 1] - g->off[u] > g->off[v + 1] - g->off[v]) { uint32_t t = u; u = v; v = t; }
    uint64_t lo = g->off[u], hi = g->off[u + 1];
    while (lo < hi) {
        uint64_t mid = lo + (hi - lo) / 2;
        if (g->nbr[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo < g->off[u + 1] && g->nbr[lo] == v;
}

/* ------------------------------------------------------ search node (search_node.cpp) */

typedef struct {
    uint32_t* deg;
    uint32_t cc;
    uint64_t edges;
} node_t;

/* search_node.cpp:16-25 */
static void remove_vertex(node_t* x, const orc_graph* g, uint32_t v) {
    uint32_t former = x->deg[v];
    x->deg[v] = ORC_REMOVED;
    x->cc++;
    for (uint64_t i = g->off[v]; i < g->off[v + 1]; ++i) {
        uint32_t u = g->nbr[i];
        if (x->deg[u] != ORC_REMOVED) x->deg[u]--;
    }
    x->edges -= former;
}

/* search_node.cpp:27-32 */
static void remove_neighbors(node_t* x, const orc_graph* g, uint32_t v) {
    for (uint64_t i = g->off[v]; i < g->off[v + 1]; ++i) {
        uint32_t u = g->nbr[i];
        if (x->deg[u] != ORC_REMOVED) remove_vertex(x, g, u);
    }
}

/* search_node.cpp:34-46: smallest-id alive vertex of maximum degree; n if none alive */
static uint32_t max_degree_vertex(const node_t* x, uint32_t n) {
    uint32_t best = n, bd = 0;
    for (uint32_t v = 0; v < n; ++v) {
        uint32_t d = x->deg[v];
        if (d == ORC_REMOVED) continue;
        if (best == n || d > bd) { best = v; bd = d; }
    }
    return best;
}

/* search_node.cpp:85-97 FNV-1a over degrees (as u64), cover_count, edge count */
uint64_t orc_fingerprint(const uint32_t* deg, uint32_t n, uint32_t cc, uint64_t edges) {
    uint64_t h = 1469598103934665603ull;
#define MIX(X) do { uint64_t x_ = (X); for (int i_ = 0; i_ < 8; ++i_) { \
        h ^= (x_ >> (8 * i_)) & 0xff; h *= 1099511628211ull; } } while (0)
    for (uint32_t v = 0; v < n; ++v) MIX(deg[v]);
    MIX(cc);
    MIX(edges);
#undef MIX
    return h;
}

/* ------------------------------------------------------------ rules (reductions.cpp) */

/* reductions.hpp:19-27 ReductionBound::current */
static uint32_t limit_for(int pvc, uint32_t k, uint32_t best_or_k, uint32_t cc) {
    if (pvc) return cc >= k ? 0 : k - cc;
    uint32_t spend = cc + 1;
    return best_or_k <= spend ? 0 : best_or_k - spend;
}

/* reductions.cpp:7-19: ascending pass, degree measured at visit time */
static int degree_one(node_t* x, const orc_graph* g) {
    int changed = 0;
    for (uint32_t v = 0; v < g->n; ++v) {
        if (x->deg[v] != 1) continue;
        for (uint64_t i = g->off[v]; i < g->off[v + 1]; ++i) {
            uint32_t u = g->nbr[i];
            if (x->deg[u] != ORC_REMOVED) { remove_vertex(x, g, u); changed = 1; break; }
        }
    }
    return changed;
}

/* reductions.cpp:22-40: first two alive base neighbours; both removed if adjacent */
static int degree_two_triangle(node_t* x, const orc_graph* g) {
    int changed = 0;
    for (uint32_t v = 0; v < g->n; ++v) {
        if (x->deg[v] != 2) continue;
        uint32_t p[2];
        int found = 0;
        for (uint64_t i = g->off[v]; i < g->off[v + 1] && found < 2; ++i) {
            uint32_t u = g->nbr[i];
            if (x->deg[u] != ORC_REMOVED) p[found++] = u;
        }
        if (found != 2) continue;
        if (!orc_has_edge(g, p[0], p[1])) continue;
        remove_vertex(x, g, p[0]);
        remove_vertex(x, g, p[1]);
        changed = 1;
    }
    return changed;
}

/* reductions.cpp:43-58: the limit is recomputed after every removal */
static int high_degree(node_t* x, const orc_graph* g, int pvc, uint32_t k, uint32_t best_or_k) {
    int changed = 0;
    uint32_t limit = limit_for(pvc, k, best_or_k, x->cc);
    for (uint32_t v = 0; v < g->n; ++v) {
        uint32_t d = x->deg[v];
        if (d == ORC_REMOVED || d == 0) continue;
        if (d > limit) {
            remove_vertex(x, g, v);
            changed = 1;
            limit = limit_for(pvc, k, best_or_k, x->cc);
        }
    }
    return changed;
}

/* reductions.cpp:63-90 reduce_loop with a constant bound (the plain overload :94-97) */
static void reduce_fixpoint(node_t* x, const orc_graph* g, int pvc, uint32_t k,
                            uint32_t best_or_k) {
    int changed = 1;
    while (changed) {
        if (x->edges == 0) break;
        changed = 0;
        changed |= degree_one(x, g);
        changed |= degree_two_triangle(x, g);
        changed |= high_degree(x, g, pvc, k, best_or_k);
    }
}

/* reductions.cpp:106-114 */
static void reduce_degree_rules(node_t* x, const orc_graph* g) {
    int changed = 1;
    while (changed) {
        if (x->edges == 0) break;
        changed = 0;
        changed |= degree_one(x, g);
        changed |= degree_two_triangle(x, g);
    }
}

int orc_reduce(const orc_graph* g, uint32_t* deg, uint32_t* cc, uint64_t* edges, int pvc,
               uint32_t k, uint32_t best_or_k, int which) {
    node_t x = {deg, *cc, *edges};
    int changed = 0;
    switch (which) {
        case 0: reduce_fixpoint(&x, g, pvc, k, best_or_k); break;
        case 1: reduce_degree_rules(&x, g); break;
        case 2: changed = degree_one(&x, g); break;
        case 3: changed = degree_two_triangle(&x, g); break;
        case 4: changed = high_degree(&x, g, pvc, k, best_or_k); break;
        default: return -1;
    }
    *cc = x.cc;
    *edges = x.edges;
    return changed;
}

/* ----------------------------------------------------------------- bounds (bounds.cpp) */

/* bounds.cpp:21-30 */
int orc_should_prune(uint32_t cc, uint64_t edges, int pvc, uint32_t k, uint32_t best) {
    if (pvc) {
        if (cc > k) return 1;
        uint64_t slack = k - cc;
        return edges > slack * slack;
    }
    if (cc >= best) return 1;
    uint64_t slack = best - cc - 1;
    return edges > slack * slack;
}

static void init_root(node_t* x, const orc_graph* g) {
    for (uint32_t v = 0; v < g->n; ++v) x->deg[v] = (uint32_t)(g->off[v + 1] - g->off[v]);
    x->cc = 0;
    x->edges = g->m;
}

static uint32_t cover_of(const node_t* x, uint32_t n, uint32_t* cover) {
    uint32_t c = 0;
    for (uint32_t v = 0; v < n; ++v)
        if (x->deg[v] == ORC_REMOVED) cover[c++] = v;
    return c;
}

/* bounds.cpp:7-19 */
uint32_t orc_greedy(const orc_graph* g, uint32_t* cover) {
    node_t x;
    x.deg = (uint32_t*)malloc(((size_t)g->n + 1) * sizeof(uint32_t));
    init_root(&x, g);
    for (;;) {
        reduce_degree_rules(&x, g);
        if (x.edges == 0) break;
        remove_vertex(&x, g, max_degree_vertex(&x, g->n));
    }
    cover_of(&x, g->n, cover);
    uint32_t size = x.cc;
    free(x.deg);
    return size;
}

/* bounds.cpp:32-45 */
int orc_verify_cover(const orc_graph* g, const uint32_t* cover, uint32_t len) {
    char* in = (char*)calloc((size_t)g->n + 1, 1);
    for (uint32_t i = 0; i < len; ++i) {
        if (cover[i] >= g->n) { free(in); return 0; }
        in[cover[i]] = 1;
    }
    int ok = 1;
    for (uint32_t v = 0; v < g->n && ok; ++v) {
        if (in[v]) continue;
        for (uint64_t i = g->off[v]; i < g->off[v + 1]; ++i) {
            uint32_t u = g->nbr[i];
            if (u > v && !in[u]) { ok = 0; break; }
        }
    }
    free(in);
    return ok;
}

/* solver_seq.cpp:173-211: the first minimum mask in increasing mask order wins */
uint32_t orc_brute_force(const orc_graph* g, uint32_t* cover) {
    uint32_t n = g->n;
    if (n > 20) return UINT32_MAX;
    if (n == 0) return 0;
    uint32_t best = n, best_mask = (1u << n) - 1u;
    for (uint32_t mask = 0; mask < (1u << n); ++mask) {
        uint32_t size = (uint32_t)__builtin_popcount(mask);
        if (size >= best) continue;
        int covers = 1;
        for (uint32_t v = 0; v < n && covers; ++v)
            for (uint64_t i = g->off[v]; i < g->off[v + 1]; ++i) {
                uint32_t u = g->nbr[i];
                if (v < u && !((mask >> u) & 1u) && !((mask >> v) & 1u)) { covers = 0; break; }
            }
        if (covers) { best = size; best_mask = mask; }
    }
    uint32_t c = 0;
    for (uint32_t v = 0; v < n; ++v)
        if ((best_mask >> v) & 1u) cover[c++] = v;
    return best;
}

/* ------------------------------------------------------ sequential solver (solver_seq.cpp) */

/* solver_seq.cpp:56-159: explicit-stack DFS; the remove-N(v) child is deferred, the
 * remove-v child is processed next. */
int orc_solve_seq(const orc_graph* g, int pvc, uint32_t k, uint64_t node_budget,
                  orc_result* out, uint32_t* cover) {
    if (pvc && k < 1) return -1;
    uint32_t n = g->n;
    memset(out, 0, sizeof(*out));
    uint32_t* best_cover = (uint32_t*)malloc(((size_t)n + 1) * sizeof(uint32_t));
    uint32_t best = orc_greedy(g, best_cover);
    out->greedy_size = best;
    uint32_t best_or_k = pvc ? k : best;
    int pvc_found = 0;
    uint64_t bound = pvc ? (k < n ? k : n) : best;
    size_t stride = (size_t)n + 1;
    uint32_t* stack = (uint32_t*)malloc((bound + 1) * stride * sizeof(uint32_t));
    uint32_t* stack_cc = (uint32_t*)malloc((bound + 1) * sizeof(uint32_t));
    uint64_t* stack_e = (uint64_t*)malloc((bound + 1) * sizeof(uint64_t));
    uint64_t top = 0;
    node_t x;
    x.deg = (uint32_t*)malloc(stride * sizeof(uint32_t));
    init_root(&x, g);
    int have = 1;
    for (;;) {
        if (!have) {
            if (top == 0) break;
            --top;
            memcpy(x.deg, stack + top * stride, n * sizeof(uint32_t));
            x.cc = stack_cc[top];
            x.edges = stack_e[top];
            have = 1;
        }
        out->nodes++;
        if (node_budget && out->nodes > node_budget) { out->status = 2; break; }
        reduce_fixpoint(&x, g, pvc, k, best_or_k);
        if (orc_should_prune(x.cc, x.edges, pvc, k, best)) { have = 0; continue; }
        if (x.edges == 0) {
            if (pvc) {
                best = x.cc;
                cover_of(&x, n, best_cover);
                pvc_found = 1;
                break;
            }
            if (x.cc < best) {
                best = x.cc;
                cover_of(&x, n, best_cover);
                best_or_k = best;
            }
            have = 0;
            continue;
        }
        uint32_t v = max_degree_vertex(&x, n);
        /* deferred = clone; remove N(v) in the clone; push */
        uint32_t* d = stack + top * stride;
        memcpy(d, x.deg, n * sizeof(uint32_t));
        node_t y = {d, x.cc, x.edges};
        remove_neighbors(&y, g, v);
        stack_cc[top] = y.cc;
        stack_e[top] = y.edges;
        ++top;
        if (top > out->stack_high_water) out->stack_high_water = top;
        remove_vertex(&x, g, v);
    }
    if (pvc) {
        out->feasible = pvc_found;
        out->size = pvc_found ? best : 0;
    } else {
        out->feasible = 1;
        out->size = best;
    }
    if (cover && out->feasible) memcpy(cover, best_cover, out->size * sizeof(uint32_t));
    free(x.deg);
    free(stack);
    free(stack_cc);
    free(stack_e);
    free(best_cover);
    return 0;
}
