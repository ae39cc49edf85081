// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never on the product path).
//
// A thin extern "C" surface over the UNMODIFIED reference solver, compiled together with the
// reference's own sources where they lie under /root/reference/proj/src (see oracle/Makefile,
// output oracle/_ref/libvcref.so, git-ignored). It lets the parity tests, the golden-fixture
// generator and bench.py's CPU arm call the reference exactly as its pybind11 module does
// (proj/python/bindings.cpp:60-99) without pybind11 or nlohmann/json.
//
// Every entry point forwards to the reference symbol named in its comment.
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "vcsolve/bounds.hpp"
#include "vcsolve/graph.hpp"
#include "vcsolve/metrics.hpp"
#include "vcsolve/reductions.hpp"
#include "vcsolve/scheduler.hpp"
#include "vcsolve/search_node.hpp"
#include "vcsolve/solver_seq.hpp"
#include "testutil.hpp"  // proj/tests/testutil.hpp: random_gnp, random_tree, ...

using namespace vcsolve;

namespace {
thread_local std::string g_err;
BaseGraph* as_graph(void* p) { return static_cast<BaseGraph*>(p); }
}  // namespace

extern "C" {

const char* vcref_last_error() { return g_err.c_str(); }

// BaseGraph from a caller CSR (bindings.cpp has no such entry; used to hand the reference the
// exact bytes our own loader produced).
void* vcref_graph_from_csr(uint32_t n, uint64_t m, const uint64_t* off, const uint32_t* nbr,
                           uint32_t id_base) {
    auto* g = new BaseGraph;
    g->num_vertices = n;
    g->num_edges = m;
    g->id_base = id_base;
    g->offsets.assign(off, off + n + 1);
    g->neighbors.assign(nbr, nbr + 2 * m);
    return g;
}

// make_graph (graph.cpp:22-54)
void* vcref_make_graph(uint32_t n, uint64_t num_pairs, const uint32_t* uv) {
    std::vector<std::pair<Vertex, Vertex>> e(num_pairs);
    for (uint64_t i = 0; i < num_pairs; ++i) e[i] = {uv[2 * i], uv[2 * i + 1]};
    return new BaseGraph(make_graph(n, e, 0));
}

// parse_edge_list / parse_dimacs (graph.cpp:81-159). Returns null and sets the error text
// (including the reference's "line N: ..." prefix) on ParseError.
void* vcref_parse(const char* text, int dimacs) {
    try {
        std::istringstream in(text);
        return new BaseGraph(dimacs ? parse_dimacs(in) : parse_edge_list(in));
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return nullptr;
    }
}

// testutil.hpp:62-70 random_gnp / :73-81 random_tree
void* vcref_gen_gnp(uint32_t n, double p, uint64_t seed) {
    return new BaseGraph(testutil::random_gnp(n, p, seed));
}
void* vcref_gen_tree(uint32_t n, uint64_t seed) {
    return new BaseGraph(testutil::random_tree(n, seed));
}

// complement (graph.cpp:161-185)
void* vcref_complement(void* g) { return new BaseGraph(complement(*as_graph(g))); }

void vcref_graph_free(void* g) { delete as_graph(g); }
uint32_t vcref_n(void* g) { return as_graph(g)->num_vertices; }
uint64_t vcref_m(void* g) { return as_graph(g)->num_edges; }
uint32_t vcref_id_base(void* g) { return as_graph(g)->id_base; }
void vcref_csr(void* g, uint64_t* off, uint32_t* nbr) {
    const BaseGraph& G = *as_graph(g);
    std::memcpy(off, G.offsets.data(), (G.num_vertices + 1) * sizeof(uint64_t));
    std::memcpy(nbr, G.neighbors.data(), G.neighbors.size() * sizeof(uint32_t));
}

// greedy_approx (bounds.cpp:7-19). Returns the size; cover in internal ids.
uint32_t vcref_greedy(void* g, uint32_t* cover) {
    GreedyResult r = greedy_approx(*as_graph(g));
    std::memcpy(cover, r.cover.data(), r.cover.size() * sizeof(uint32_t));
    return r.size;
}

// brute_force_mvc (solver_seq.cpp:173-211). Returns size, or UINT32_MAX when n > 20.
uint32_t vcref_brute_force(void* g, uint32_t* cover) {
    try {
        Solution s = brute_force_mvc(*as_graph(g));
        std::memcpy(cover, s.cover.data(), s.cover.size() * sizeof(uint32_t));
        return s.size;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return UINT32_MAX;
    }
}

// One reduce call on an explicit node (reductions.cpp:94-114). which: 0 = reduce_to_fixpoint
// (plain overload, constant best_or_k), 1 = reduce_degree_rules_to_fixpoint,
// 2 = apply_degree_one, 3 = apply_degree_two_triangle, 4 = apply_high_degree.
// Returns the rule's "changed" flag for the single-pass variants.
int vcref_reduce(void* g, uint32_t* degrees, uint32_t* cover_count, uint64_t* edges, int pvc,
                 uint32_t k, uint32_t best_or_k, int which) {
    const BaseGraph& G = *as_graph(g);
    SearchNode node;
    node.degrees.assign(degrees, degrees + G.num_vertices);
    node.cover_count = *cover_count;
    node.alive_edge_count = *edges;
    SolveMode mode = pvc ? SolveMode::pvc(k) : SolveMode::mvc();
    int changed = 0;
    switch (which) {
        case 0: reduce_to_fixpoint(node, G, mode, best_or_k); break;
        case 1: reduce_degree_rules_to_fixpoint(node, G); break;
        case 2: changed = apply_degree_one(node, G); break;
        case 3: changed = apply_degree_two_triangle(node, G); break;
        case 4: changed = apply_high_degree(node, G, mode, best_or_k); break;
        default: return -1;
    }
    std::memcpy(degrees, node.degrees.data(), G.num_vertices * sizeof(uint32_t));
    *cover_count = node.cover_count;
    *edges = node.alive_edge_count;
    return changed;
}

// should_prune (bounds.cpp:21-30)
int vcref_should_prune(uint32_t cover_count, uint64_t edges, int pvc, uint32_t k, uint32_t best) {
    SearchNode node;
    node.cover_count = cover_count;
    node.alive_edge_count = edges;
    return should_prune(node, pvc ? SolveMode::pvc(k) : SolveMode::mvc(), best) ? 1 : 0;
}

// node_fingerprint (search_node.cpp:85-97)
uint64_t vcref_fingerprint(const uint32_t* degrees, uint32_t n, uint32_t cover_count,
                           uint64_t edges) {
    SearchNode node;
    node.degrees.assign(degrees, degrees + n);
    node.cover_count = cover_count;
    node.alive_edge_count = edges;
    return node_fingerprint(node);
}

struct vcref_result {
    uint32_t size;
    int32_t feasible;
    int32_t status;  // 0 complete, 1 timeout, 2 budget (RunStatus order)
    uint32_t greedy_size;
    uint32_t cover_len;
    uint32_t num_workers;
    double wall_ms;
    uint64_t nodes_total;
    uint64_t wl_added, wl_removed, wl_max_size, wl_current_size;
    uint64_t stack_high_water;  // max over workers
};

// The solve dispatch of bindings.cpp:60-99: strategy 0 = "seq" (solve_mvc_seq/solve_pvc_seq),
// 1 = "hybrid" (run_hybrid), 2 = "stackonly" (run_stackonly). timeout_s < 0 and
// node_budget == 0 mean "none". cover (original ids) needs n entries; worker_nodes needs
// `workers` entries (1 for seq). Returns 0, or -1 with vcref_last_error() on
// std::invalid_argument.
int vcref_solve(void* g, int pvc, uint32_t k, int strategy, unsigned workers, uint64_t capacity,
                double threshold_fraction, unsigned depth, uint64_t backoff_us, double timeout_s,
                uint64_t node_budget, vcref_result* out, uint32_t* cover,
                uint64_t* worker_nodes) {
    try {
        const BaseGraph& G = *as_graph(g);
        SolveMode mode = pvc ? SolveMode::pvc(k) : SolveMode::mvc();
        SchedulerConfig config;
        config.num_workers = workers;
        config.worklist_capacity = capacity;
        config.threshold_fraction = threshold_fraction;
        config.stackonly_depth = depth;
        config.backoff = std::chrono::microseconds(backoff_us);
        if (timeout_s >= 0) config.limits.timeout_s = timeout_s;
        if (node_budget) config.limits.node_budget = node_budget;
        std::memset(out, 0, sizeof(*out));
        Solution sol;
        std::vector<WorkerMetrics> metrics;
        if (strategy == 0) {
            if (pvc && k < 1) throw std::invalid_argument("pvc requires k >= 1");
            SeqRun run = pvc ? solve_pvc_seq(G, k, config.limits) : solve_mvc_seq(G, config.limits);
            sol = run.solution;
            out->status = static_cast<int>(run.status);
            out->wall_ms = run.wall_ms;
            metrics.push_back(run.metrics);
            out->greedy_size = greedy_approx(G).size;
        } else {
            ParallelRun run = strategy == 1 ? run_hybrid(G, mode, config)
                                            : run_stackonly(G, mode, config);
            sol = run.solution;
            out->status = static_cast<int>(run.status);
            out->wall_ms = run.wall_ms;
            out->greedy_size = run.greedy_size;
            out->wl_added = run.worklist.added;
            out->wl_removed = run.worklist.removed;
            out->wl_max_size = run.worklist.max_size;
            out->wl_current_size = run.worklist.current_size;
            metrics = std::move(run.workers);
        }
        out->size = sol.size;
        out->feasible = sol.feasible ? 1 : 0;
        out->cover_len = static_cast<uint32_t>(sol.cover.size());
        std::memcpy(cover, sol.cover.data(), sol.cover.size() * sizeof(uint32_t));
        out->num_workers = static_cast<uint32_t>(metrics.size());
        for (std::size_t w = 0; w < metrics.size(); ++w) {
            worker_nodes[w] = metrics[w].nodes_visited;
            out->nodes_total += metrics[w].nodes_visited;
            if (metrics[w].stack_high_water > out->stack_high_water)
                out->stack_high_water = metrics[w].stack_high_water;
        }
        return 0;
    } catch (const std::exception& ex) {
        g_err = ex.what();
        return -1;
    }
}

}  // extern "C"
