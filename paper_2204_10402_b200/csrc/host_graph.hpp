// Host-side graph: the immutable CSR every solve starts from, its loaders and the host seed
// (greedy upper bound). Semantics follow the reference's graph-core module
// (proj/include/vcsolve/graph.hpp, proj/src/graph.cpp) and greedy_approx (proj/src/bounds.cpp).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace vcg {

constexpr uint32_t kRemoved = 0xFFFFFFFFu;  // search_node.hpp:14

// ParseError (graph.hpp:17-26): message prefixed with "line N: ".
struct ParseError : std::runtime_error {
    ParseError(const std::string& msg, size_t line)
        : std::runtime_error("line " + std::to_string(line) + ": " + msg) {}
};

struct DeviceGraph;  // engine.cu: per-device resident copies (CSR, adjacency bitmap)

struct Graph {
    uint32_t n = 0;
    uint64_t m = 0;
    uint32_t id_base = 0;
    std::vector<uint64_t> off;  // n+1
    std::vector<uint32_t> nbr;  // 2m, slices sorted ascending
    // device copies, one per device ordinal (lazily built by the engine)
    mutable std::vector<std::shared_ptr<DeviceGraph>> dev;

    uint32_t degree(uint32_t v) const { return static_cast<uint32_t>(off[v + 1] - off[v]); }
    bool has_edge(uint32_t u, uint32_t v) const;
};

// Builders / loaders (graph.cpp:22-193 semantics).
Graph make_graph(uint32_t n, const std::vector<std::pair<uint32_t, uint32_t>>& edges,
                 uint32_t id_base);
Graph parse_edge_list(const char* text, size_t len);
Graph parse_dimacs(const char* text, size_t len);
Graph complement(const Graph& g);
std::string write_edge_list(const Graph& g);
bool check_invariants(const Graph& g);

// greedy_approx (bounds.cpp:7-19), reproducing the reference cover exactly with
// bitset-indexed rule passes and a degree-bucket max-degree query.
struct Greedy {
    uint32_t size = 0;
    std::vector<uint32_t> cover;  // internal ids ascending
};
Greedy greedy_approx(const Graph& g);

// brute_force_mvc (solver_seq.cpp:173-211): n <= 20, first minimum mask in mask order.
uint32_t brute_force(const Graph& g, std::vector<uint32_t>& cover_internal);

// verify_cover (bounds.cpp:32-45) over internal ids.
bool verify_cover(const Graph& g, const uint32_t* cover, size_t len);

}  // namespace vcg
