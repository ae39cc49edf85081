// Host graph: CSR construction, loaders, complement, greedy seed, brute force, verification.
// Behaviour (results, error texts) follows proj/src/graph.cpp and proj/src/bounds.cpp; the
// implementation is our own (bitset candidate sets + lazy max-heap for the greedy seed).
#include "host_graph.hpp"

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cstdlib>
#include <limits>
#include <queue>
#include <string_view>

namespace vcg {

bool Graph::has_edge(uint32_t u, uint32_t v) const {
    // graph.cpp:14-20: binary search within the shorter of the two slices.
    if (u == v) return false;
    if (degree(u) > degree(v)) std::swap(u, v);
    const uint32_t* b = nbr.data() + off[u];
    const uint32_t* e = nbr.data() + off[u + 1];
    return std::binary_search(b, e, v);
}

Graph make_graph(uint32_t n, const std::vector<std::pair<uint32_t, uint32_t>>& edges,
                 uint32_t id_base) {
    // graph.cpp:22-54: self-loops dropped, (u,v) oriented u<v, sorted, duplicates dropped.
    std::vector<uint64_t> keys;
    keys.reserve(edges.size());
    for (auto [u, v] : edges) {
        if (u == v) continue;
        if (u >= n || v >= n) throw std::invalid_argument("vertex id out of range");
        uint32_t a = std::min(u, v), b = std::max(u, v);
        keys.push_back((uint64_t(a) << 32) | b);
    }
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    Graph g;
    g.n = n;
    g.m = keys.size();
    g.id_base = id_base;
    g.off.assign(size_t(n) + 1, 0);
    for (uint64_t k : keys) {
        ++g.off[(k >> 32) + 1];
        ++g.off[uint32_t(k) + 1];
    }
    for (uint32_t v = 0; v < n; ++v) g.off[v + 1] += g.off[v];
    g.nbr.resize(2 * g.m);
    std::vector<uint64_t> fill(g.off.begin(), g.off.end() - 1);
    // Keys ascend by (a, b): each a receives its larger neighbours b in ascending order, and
    // each b receives its smaller neighbours a in ascending order, before any larger ones
    // (those arrive later as (b, c) keys) — so every slice comes out sorted.
    for (uint64_t k : keys) {
        uint32_t a = uint32_t(k >> 32), b = uint32_t(k);
        g.nbr[fill[a]++] = b;
        g.nbr[fill[b]++] = a;
    }
    return g;
}

namespace {

// Line splitter with std::getline semantics: a trailing newline does not start a new line.
struct Lines {
    std::string_view text;
    size_t pos = 0;
    size_t line_no = 0;
    bool next(std::string_view& line) {
        if (pos >= text.size()) return false;
        size_t e = text.find('\n', pos);
        if (e == std::string_view::npos) e = text.size();
        line = text.substr(pos, e - pos);
        pos = e + 1;
        ++line_no;
        return true;
    }
};

// Whitespace tokenizer with istringstream >> std::string semantics.
struct Tokens {
    std::string_view s;
    size_t p = 0;
    bool next(std::string_view& tok) {
        while (p < s.size() && std::isspace(static_cast<unsigned char>(s[p]))) ++p;
        if (p >= s.size()) return false;
        size_t b = p;
        while (p < s.size() && !std::isspace(static_cast<unsigned char>(s[p]))) ++p;
        tok = s.substr(b, p - b);
        return true;
    }
};

// graph.cpp:66-78 parse_id: digits only, value <= UINT32_MAX - 1.
uint64_t parse_id(std::string_view tok, size_t line) {
    std::string t(tok);
    if (t.empty()) throw ParseError("empty vertex id", line);
    for (char c : t)
        if (!std::isdigit(static_cast<unsigned char>(c)))
            throw ParseError("malformed vertex id '" + t + "'", line);
    errno = 0;
    unsigned long long v = std::strtoull(t.c_str(), nullptr, 10);
    if (errno != 0 || v > std::numeric_limits<uint32_t>::max() - 1ull)
        throw ParseError("vertex id out of range '" + t + "'", line);
    return v;
}

// istream >> uint64_t on one whitespace token: an optional sign then a maximal digit prefix.
// Returns false on no digits / overflow; `rest` receives unconsumed characters.
bool stream_u64(std::string_view tok, uint64_t& out, std::string_view& rest) {
    size_t p = 0;
    bool neg = false;
    if (p < tok.size() && (tok[p] == '+' || tok[p] == '-')) neg = tok[p++] == '-';
    size_t b = p;
    unsigned long long v = 0;
    while (p < tok.size() && std::isdigit(static_cast<unsigned char>(tok[p]))) {
        unsigned d = unsigned(tok[p] - '0');
        if (v > (std::numeric_limits<unsigned long long>::max() - d) / 10) return false;
        v = v * 10 + d;
        ++p;
    }
    if (p == b) return false;
    out = neg ? uint64_t(0) - v : v;
    rest = tok.substr(p);
    return true;
}

bool comment_or_blank(std::string_view line) {
    for (char c : line) {
        if (std::isspace(static_cast<unsigned char>(c))) continue;
        return c == '#' || c == '%';
    }
    return true;
}

}  // namespace

Graph parse_edge_list(const char* text, size_t len) {
    // graph.cpp:81-114
    Lines lines{std::string_view(text, len)};
    std::string_view line;
    std::vector<std::pair<uint32_t, uint32_t>> edges;
    uint64_t lo = std::numeric_limits<uint64_t>::max(), hi = 0;
    bool any = false;
    while (lines.next(line)) {
        if (comment_or_blank(line)) continue;
        Tokens t{line};
        std::string_view a, b, extra;
        if (!t.next(a) || !t.next(b)) throw ParseError("expected 'u v' pair", lines.line_no);
        if (t.next(extra))
            throw ParseError("trailing token '" + std::string(extra) + "'", lines.line_no);
        uint64_t u = parse_id(a, lines.line_no);
        uint64_t v = parse_id(b, lines.line_no);
        any = true;
        lo = std::min(lo, std::min(u, v));
        hi = std::max(hi, std::max(u, v));
        edges.emplace_back(uint32_t(u), uint32_t(v));
    }
    if (!any) return make_graph(0, {}, 0);
    uint32_t base = lo >= 1 ? 1 : 0;  // 1-based iff no id 0 appears
    for (auto& [u, v] : edges) {
        u -= base;
        v -= base;
    }
    return make_graph(uint32_t(hi - base + 1), edges, base);
}

Graph parse_dimacs(const char* text, size_t len) {
    // graph.cpp:116-159
    Lines lines{std::string_view(text, len)};
    std::string_view line;
    std::vector<std::pair<uint32_t, uint32_t>> edges;
    bool have_problem = false;
    uint64_t n = 0;
    while (lines.next(line)) {
        Tokens t{line};
        std::string_view tag;
        if (!t.next(tag)) continue;
        if (tag == "c") continue;
        if (tag == "p") {
            if (have_problem) throw ParseError("duplicate 'p' line", lines.line_no);
            std::string_view fmt, tn, tm, rest;
            uint64_t m = 0;
            bool ok = t.next(fmt) && t.next(tn) && stream_u64(tn, n, rest) && rest.empty();
            // ">> n >> m": junk glued to n makes the m extraction fail; junk after m is left.
            ok = ok && t.next(tm) && stream_u64(tm, m, rest);
            if (!ok) throw ParseError("malformed 'p' line", lines.line_no);
            if (fmt != "edge" && fmt != "edges" && fmt != "col")
                throw ParseError("unsupported format '" + std::string(fmt) + "'", lines.line_no);
            if (n > std::numeric_limits<uint32_t>::max() - 1ull)
                throw ParseError("vertex count out of range", lines.line_no);
            have_problem = true;
            edges.reserve(std::min<uint64_t>(m, uint64_t(1) << 28));
            continue;
        }
        if (tag == "e") {
            if (!have_problem) throw ParseError("'e' line before 'p' line", lines.line_no);
            std::string_view a, b;
            if (!t.next(a) || !t.next(b)) throw ParseError("malformed 'e' line", lines.line_no);
            uint64_t u = parse_id(a, lines.line_no);
            uint64_t v = parse_id(b, lines.line_no);
            if (u < 1 || u > n || v < 1 || v > n)
                throw ParseError("edge endpoint outside 1.." + std::to_string(n), lines.line_no);
            edges.emplace_back(uint32_t(u - 1), uint32_t(v - 1));
            continue;
        }
        throw ParseError("unrecognized line type '" + std::string(tag) + "'", lines.line_no);
    }
    if (!have_problem)
        throw ParseError("missing 'p edge N M' line", lines.line_no == 0 ? 1 : lines.line_no);
    return make_graph(uint32_t(n), edges, 1);
}

Graph complement(const Graph& g) {
    // graph.cpp:161-185: u joins v's slice iff u != v and u is absent from g's slice.
    Graph out;
    out.n = g.n;
    out.id_base = g.id_base;
    uint64_t n = g.n;
    out.m = n * (n - (n > 0 ? 1 : 0)) / 2 - g.m;
    out.off.assign(size_t(n) + 1, 0);
    out.nbr.resize(2 * out.m);
    uint64_t pos = 0;
    for (uint32_t v = 0; v < g.n; ++v) {
        out.off[v] = pos;
        const uint32_t* s = g.nbr.data() + g.off[v];
        const uint32_t* e = g.nbr.data() + g.off[v + 1];
        for (uint32_t u = 0; u < g.n; ++u) {
            while (s < e && *s < u) ++s;
            if (u == v || (s < e && *s == u)) continue;
            out.nbr[pos++] = u;
        }
    }
    out.off[g.n] = pos;
    return out;
}

std::string write_edge_list(const Graph& g) {
    // graph.cpp:187-193: one "u v" line per edge with u < v, in original ids.
    std::string out;
    out.reserve(g.m * 12);
    char buf[32];
    for (uint32_t v = 0; v < g.n; ++v)
        for (uint64_t i = g.off[v]; i < g.off[v + 1]; ++i) {
            uint32_t u = g.nbr[i];
            if (v < u) {
                int k = std::snprintf(buf, sizeof buf, "%u %u\n", v + g.id_base, u + g.id_base);
                out.append(buf, size_t(k));
            }
        }
    return out;
}

bool check_invariants(const Graph& g) {
    // graph.cpp:195-211
    if (g.off.size() != size_t(g.n) + 1) return false;
    if (g.off.front() != 0 || g.off.back() != 2 * g.m) return false;
    if (g.nbr.size() != 2 * g.m) return false;
    for (uint32_t v = 0; v < g.n; ++v) {
        if (g.off[v] > g.off[v + 1]) return false;
        for (uint64_t i = g.off[v]; i < g.off[v + 1]; ++i) {
            uint32_t u = g.nbr[i];
            if (u >= g.n || u == v) return false;
            if (i > g.off[v] && g.nbr[i - 1] >= u) return false;
        }
    }
    // Symmetry (the reference's has_edge(u, v) for every slot) in one O(m) sweep: with sorted
    // duplicate-free slices, visiting v in ascending order must meet each u's slice entries in
    // order, so slot (v, u) matches the next unmatched entry of u's slice and every slice is
    // consumed exactly.
    std::vector<uint64_t> cur(g.off.begin(), g.off.end() - 1);
    for (uint32_t v = 0; v < g.n; ++v)
        for (uint64_t i = g.off[v]; i < g.off[v + 1]; ++i) {
            const uint32_t u = g.nbr[i];
            if (cur[u] >= g.off[u + 1] || g.nbr[cur[u]] != v) return false;
            ++cur[u];
        }
    for (uint32_t u = 0; u < g.n; ++u)
        if (cur[u] != g.off[u + 1]) return false;
    return true;
}

// ------------------------------------------------------------------------ greedy seed

namespace {

struct Bits {
    std::vector<uint64_t> w;
    explicit Bits(uint32_t n) : w((size_t(n) + 63) / 64, 0) {}
    void set(uint32_t i) { w[i >> 6] |= uint64_t(1) << (i & 63); }
    void clear(uint32_t i) { w[i >> 6] &= ~(uint64_t(1) << (i & 63)); }
    // first set index >= from, or UINT32_MAX
    uint32_t next(uint32_t from) const {
        size_t k = from >> 6;
        if (k >= w.size()) return UINT32_MAX;
        uint64_t x = w[k] & (~uint64_t(0) << (from & 63));
        while (true) {
            if (x) return uint32_t(k * 64 + __builtin_ctzll(x));
            if (++k >= w.size()) return UINT32_MAX;
            x = w[k];
        }
    }
};

// A search node (degree array + counters) with the candidate sets the reference's ascending
// rule passes and max_degree_vertex query. Degree buckets (one bitset per degree, O(1) moves)
// give deg==1 / deg==2 find-next and the smallest-id max-degree vertex; when
// (max degree + 1) x n/64 words would be too large, a lazy max-heap over (degree, -id) serves
// the max-degree query instead.
struct GreedyNode {
    const Graph& g;
    std::vector<uint32_t> deg;
    uint32_t cc = 0;
    uint64_t edges = 0;
    size_t words;
    bool bucketed;
    std::vector<uint64_t> bw;      // bucketed: (maxdeg + 1) x words
    std::vector<uint32_t> bcount;  // alive vertices per degree
    std::vector<size_t> bfirst;    // lowest possibly non-zero word per bucket
    uint32_t maxd = 0;
    Bits one, two;                 // heap mode only
    Bits nt;                       // degree-two vertices already found not to be in a triangle
    std::priority_queue<uint64_t> heap;  // heap mode: (deg << 32) | ~id

    explicit GreedyNode(const Graph& G)
        : g(G), deg(G.n), words((size_t(G.n) + 63) / 64), one(0), two(0), nt(G.n) {
        uint32_t md = 0;
        for (uint32_t v = 0; v < g.n; ++v) md = std::max(md, g.degree(v));
        bucketed = (size_t(md) + 1) * words <= (size_t(1) << 22);
        if (bucketed) {
            bw.assign((size_t(md) + 1) * words, 0);
            bcount.assign(size_t(md) + 1, 0);
            bfirst.assign(size_t(md) + 1, words);
            maxd = md;
        } else {
            one = Bits(g.n);
            two = Bits(g.n);
        }
        for (uint32_t v = 0; v < g.n; ++v) {
            deg[v] = g.degree(v);
            track(v, kRemoved, deg[v]);
        }
        edges = g.m;
    }
    void track(uint32_t v, uint32_t from, uint32_t to) {
        if (to == 2) nt.clear(v);  // a new degree-two vertex has new partners: check it again
        if (bucketed) {
            const uint64_t bit = uint64_t(1) << (v & 63);
            if (from != kRemoved) {
                bw[size_t(from) * words + (v >> 6)] &= ~bit;
                --bcount[from];
            }
            if (to != kRemoved) {
                bw[size_t(to) * words + (v >> 6)] |= bit;
                ++bcount[to];
                bfirst[to] = std::min(bfirst[to], size_t(v >> 6));
            }
            return;
        }
        if (from == 1) one.clear(v);
        if (from == 2) two.clear(v);
        if (to == 1) one.set(v);
        if (to == 2) two.set(v);
        if (to != kRemoved && to > 0) heap.push((uint64_t(to) << 32) | uint32_t(~v));
    }
    // first vertex >= from with degree d (d = 1 or 2), or UINT32_MAX
    uint32_t next_with(uint32_t d, uint32_t from) {
        if (!bucketed) return d == 1 ? one.next(from) : two.next(from);
        if (d >= bcount.size() || from >= g.n) return UINT32_MAX;
        const uint64_t* b = bw.data() + size_t(d) * words;
        size_t k = from >> 6;
        uint64_t x = b[k] & (~uint64_t(0) << (from & 63));
        while (true) {
            if (x) return uint32_t(k * 64 + __builtin_ctzll(x));
            if (++k >= words) return UINT32_MAX;
            x = b[k];
        }
    }
    // search_node.cpp:16-25
    void remove(uint32_t v) {
        uint32_t former = deg[v];
        deg[v] = kRemoved;
        track(v, former, kRemoved);
        ++cc;
        for (uint64_t i = g.off[v]; i < g.off[v + 1]; ++i) {
            uint32_t u = g.nbr[i];
            if (deg[u] != kRemoved) {
                --deg[u];
                track(u, deg[u] + 1, deg[u]);
            }
        }
        edges -= former;
    }
    uint32_t first_alive_neighbor(uint32_t v, uint64_t& i) const {
        for (; i < g.off[v + 1]; ++i)
            if (deg[g.nbr[i]] != kRemoved) return g.nbr[i];
        return UINT32_MAX;
    }
    // reductions.cpp:7-19 (find-next on the live set == the ascending visit-time scan)
    bool degree_one() {
        bool changed = false;
        for (uint32_t v = next_with(1, 0); v != UINT32_MAX; v = next_with(1, v + 1)) {
            uint64_t i = g.off[v];
            remove(first_alive_neighbor(v, i));
            changed = true;
        }
        return changed;
    }
    // reductions.cpp:22-40. A degree-two vertex keeps its partners (and so its non-triangle
    // verdict) until its degree changes, so verdicts are cached; the acting order is unchanged.
    bool degree_two_triangle() {
        bool changed = false;
        for (uint32_t v = next_with(2, 0); v != UINT32_MAX; v = next_with(2, v + 1)) {
            if ((nt.w[v >> 6] >> (v & 63)) & 1u) continue;
            uint64_t i = g.off[v];
            uint32_t a = first_alive_neighbor(v, i);
            ++i;
            uint32_t b = first_alive_neighbor(v, i);
            if (!g.has_edge(a, b)) {
                nt.set(v);
                continue;
            }
            remove(a);
            remove(b);
            changed = true;
        }
        return changed;
    }
    // search_node.cpp:34-46 (only queried while edges remain, so the max degree is >= 1)
    uint32_t max_degree_vertex() {
        if (bucketed) {
            while (bcount[maxd] == 0) --maxd;
            const uint64_t* b = bw.data() + size_t(maxd) * words;
            size_t k = bfirst[maxd];
            while (!b[k]) ++k;
            bfirst[maxd] = k;
            return uint32_t(k * 64 + __builtin_ctzll(b[k]));
        }
        while (true) {
            uint64_t top = heap.top();
            uint32_t v = ~uint32_t(top), d = uint32_t(top >> 32);
            if (deg[v] == d) return v;
            heap.pop();  // stale: degree changed or vertex removed since the push
        }
    }
};

}  // namespace

Greedy greedy_approx(const Graph& g) {
    // bounds.cpp:7-19 with reduce_degree_rules_to_fixpoint (reductions.cpp:106-114)
    GreedyNode x(g);
    while (true) {
        bool changed = true;
        while (changed) {
            if (x.edges == 0) break;
            changed = false;
            changed |= x.degree_one();
            changed |= x.degree_two_triangle();
        }
        if (x.edges == 0) break;
        x.remove(x.max_degree_vertex());
    }
    Greedy r;
    r.size = x.cc;
    r.cover.reserve(x.cc);
    for (uint32_t v = 0; v < g.n; ++v)
        if (x.deg[v] == kRemoved) r.cover.push_back(v);
    return r;
}

uint32_t brute_force(const Graph& g, std::vector<uint32_t>& cover) {
    // solver_seq.cpp:173-211: masks in increasing order; the first mask of minimum popcount
    // that covers every edge wins.
    uint32_t n = g.n;
    cover.clear();
    if (n == 0) return 0;
    std::vector<std::pair<uint32_t, uint32_t>> e;
    for (uint32_t v = 0; v < n; ++v)
        for (uint64_t i = g.off[v]; i < g.off[v + 1]; ++i)
            if (v < g.nbr[i]) e.emplace_back(v, g.nbr[i]);
    uint32_t best = n, best_mask = (1u << n) - 1u;
    for (uint32_t mask = 0; mask < (1u << n); ++mask) {
        uint32_t s = uint32_t(__builtin_popcount(mask));
        if (s >= best) continue;
        bool ok = true;
        for (auto [a, b] : e)
            if (!((mask >> a) & 1u) && !((mask >> b) & 1u)) {
                ok = false;
                break;
            }
        if (ok) {
            best = s;
            best_mask = mask;
        }
    }
    for (uint32_t v = 0; v < n; ++v)
        if ((best_mask >> v) & 1u) cover.push_back(v);
    return best;
}

bool verify_cover(const Graph& g, const uint32_t* cover, size_t len) {
    // bounds.cpp:32-45
    std::vector<char> in(g.n, 0);
    for (size_t i = 0; i < len; ++i) {
        if (cover[i] >= g.n) return false;
        in[cover[i]] = 1;
    }
    for (uint32_t v = 0; v < g.n; ++v) {
        if (in[v]) continue;
        for (uint64_t i = g.off[v]; i < g.off[v + 1]; ++i)
            if (g.nbr[i] > v && !in[g.nbr[i]]) return false;
    }
    return true;
}

}  // namespace vcg
