// vcsolve — the command-line front end of the B200 engine, a drop-in for the reference CLI
// (proj/tools/main.cpp) with `--strategy gpu` added to its strategy switch.
//
// Same options, subcommand, report formats and exit codes as the reference:
//   vcsolve --input FILE [--format dimacs|edgelist] [--complement] [--mode mvc|pvc] [--k K]
//           [--strategy seq|stackonly|hybrid|gpu|oracle] [--workers N] [--worklist-capacity C]
//           [--threshold-fraction F] [--depth D] [--backoff-us B] [--timeout-s T]
//           [--node-budget N] [--output json|csv|text] [--report PATH] [--device I]
//   vcsolve sweep --input FILE [--strategies a,b] [--workers 1,2] [--capacities ...]
//           [--fractions ...] [--depths ...] [--instances mvc,pvc-1,pvc,pvc+1]
//           [--timeout-s T] [--out PATH]
// Exit codes (main.cpp:26-28): 0 complete, 1 usage / error, 2 timeout or budget.
//
// Host side only, above the C-ABI (include/vcgpu.h): parsing and complement (graph.cpp), the
// search on the GPU (vcg_solve), brute force for "oracle" (vcg_brute_force). The report writers
// restate RunReport::to_json / to_csv_row / write_text (report.cpp:41-159) and collect_metrics
// (metrics.cpp:23-67); JSON keys come out sorted, as nlohmann::json's std::map objects do.
#include <algorithm>
#include <charconv>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <memory>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <variant>
#include <vector>

#include "vcgpu.h"

namespace {

constexpr int kExitOk = 0;
constexpr int kExitUsage = 1;
constexpr int kExitIncomplete = 2;

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------------------------ tiny JSON

struct Json {
    using Arr = std::vector<Json>;
    using Obj = std::map<std::string, Json>;
    std::variant<std::nullptr_t, bool, uint64_t, double, std::string, Arr, Obj> v;
    Json() : v(nullptr) {}
    Json(std::nullptr_t) : v(nullptr) {}
    Json(bool b) : v(b) {}
    Json(uint64_t x) : v(x) {}
    Json(uint32_t x) : v(uint64_t(x)) {}
    Json(unsigned long long x) : v(uint64_t(x)) {}
    Json(double x) : v(x) {}
    Json(const char* s) : v(std::string(s)) {}
    Json(std::string s) : v(std::move(s)) {}
    Json(Arr a) : v(std::move(a)) {}
    Json(Obj o) : v(std::move(o)) {}

    static void esc(std::ostream& o, const std::string& s) {
        o << '"';
        for (unsigned char c : s) {
            if (c == '"') o << "\\\"";
            else if (c == '\\') o << "\\\\";
            else if (c == '\n') o << "\\n";
            else if (c == '\t') o << "\\t";
            else if (c == '\r') o << "\\r";
            else if (c < 0x20) {
                char buf[8];
                std::snprintf(buf, sizeof buf, "\\u%04x", c);
                o << buf;
            } else o << c;
        }
        o << '"';
    }
    static void num(std::ostream& o, double x) {
        if (!std::isfinite(x)) {
            o << "null";
            return;
        }
        char buf[64];
        auto r = std::to_chars(buf, buf + sizeof buf, x);
        std::string s(buf, r.ptr);
        if (s.find_first_of(".e") == std::string::npos) s += ".0";
        o << s;
    }
    void dump(std::ostream& o, int indent, int level) const {
        std::string pad((level + 1) * indent, ' '), end(level * indent, ' ');
        if (std::holds_alternative<std::nullptr_t>(v)) o << "null";
        else if (auto b = std::get_if<bool>(&v)) o << (*b ? "true" : "false");
        else if (auto u = std::get_if<uint64_t>(&v)) o << *u;
        else if (auto d = std::get_if<double>(&v)) num(o, *d);
        else if (auto s = std::get_if<std::string>(&v)) esc(o, *s);
        else if (auto a = std::get_if<Arr>(&v)) {
            if (a->empty()) {
                o << "[]";
                return;
            }
            o << "[\n";
            for (size_t i = 0; i < a->size(); ++i) {
                o << pad;
                (*a)[i].dump(o, indent, level + 1);
                o << (i + 1 < a->size() ? ",\n" : "\n");
            }
            o << end << ']';
        } else {
            const Obj& m = std::get<Obj>(v);
            if (m.empty()) {
                o << "{}";
                return;
            }
            o << "{\n";
            size_t i = 0;
            for (const auto& [k, x] : m) {
                o << pad;
                esc(o, k);
                o << ": ";
                x.dump(o, indent, level + 1);
                o << (++i < m.size() ? ",\n" : "\n");
            }
            o << end << '}';
        }
    }
    std::string str(int indent = 2) const {
        std::ostringstream o;
        dump(o, indent, 0);
        return o.str();
    }
};

// ------------------------------------------------------------------------------ report

const char* kPhaseKeys[10] = {  // phase_key (metrics.cpp:7-21), Phase order (metrics.hpp:15-26)
    "worklist_remove", "worklist_add", "stack_ops", "reduce_degree_one",
    "reduce_degree_two_triangle", "reduce_high_degree", "max_degree_scan",
    "branch_remove_neighbors", "branch_remove_vertex", "prune_check"};

// RunReport (report.hpp:19-54) plus the engine's extras (reported under "engine").
struct RunReport {
    std::string file;
    bool complemented = false;
    uint32_t n = 0;
    uint64_t m = 0;
    std::string mode;
    std::optional<uint32_t> k;
    std::string strategy;
    unsigned workers = 1;
    uint64_t capacity = 0;
    double threshold_fraction = 0.0;
    unsigned depth = 0;
    std::optional<uint32_t> size;
    bool feasible = true;
    std::vector<uint32_t> cover;
    double wall_ms = 0.0;
    std::string status;
    std::vector<uint64_t> worker_nodes;
    std::vector<double> load_ratios;
    std::map<std::string, double> phase_shares;
    uint64_t wl_added = 0, wl_removed = 0, wl_max_size = 0;
    Json::Obj engine;  // device-side extras; empty for "oracle"

    Json to_json() const {  // report.cpp:41-70
        Json::Obj j;
        j["file"] = file;
        j["complemented"] = complemented;
        j["n"] = n;
        j["m"] = m;
        j["mode"] = mode;
        j["k"] = k ? Json(*k) : Json();
        j["strategy"] = strategy;
        j["workers"] = uint64_t(workers);
        j["capacity"] = capacity;
        j["threshold_fraction"] = threshold_fraction;
        j["depth"] = uint64_t(depth);
        j["size"] = size ? Json(*size) : Json();
        j["feasible"] = feasible;
        Json::Arr c;
        for (uint32_t v : cover) c.emplace_back(v);
        j["cover"] = std::move(c);
        j["wall_ms"] = wall_ms;
        j["status"] = status;
        Json::Arr wn, lr;
        for (uint64_t x : worker_nodes) wn.emplace_back(x);
        for (double x : load_ratios) lr.emplace_back(x);
        j["worker_nodes"] = std::move(wn);
        j["load_ratios"] = std::move(lr);
        Json::Obj ps;
        for (const auto& [key, x] : phase_shares) ps[key] = x;
        j["phase_shares"] = std::move(ps);
        j["worklist"] = Json::Obj{{"added", wl_added}, {"removed", wl_removed},
                                  {"max_size", wl_max_size}};
        if (!engine.empty()) j["engine"] = engine;
        return Json(std::move(j));
    }

    static std::string fmt(double x) {  // fmt_double (report.cpp:26-30)
        std::ostringstream o;
        o << std::setprecision(12) << x;
        return o.str();
    }
    static std::string csv_header() {  // report.cpp:101-104
        return "file,complemented,n,m,mode,k,strategy,workers,capacity,threshold_fraction,depth,"
               "size,feasible,wall_ms,status,worker_nodes,load_ratios,phase_shares";
    }
    std::string to_csv_row() const {  // report.cpp:106-125
        std::ostringstream o;
        o << file << ',' << (complemented ? 1 : 0) << ',' << n << ',' << m << ',' << mode << ',';
        if (k) o << *k;
        o << ',' << strategy << ',' << workers << ',' << capacity << ',' << fmt(threshold_fraction)
          << ',' << depth << ',';
        if (size) o << *size;
        o << ',' << (feasible ? 1 : 0) << ',' << fmt(wall_ms) << ',' << status << ',';
        for (size_t i = 0; i < worker_nodes.size(); ++i) o << (i ? ";" : "") << worker_nodes[i];
        o << ',';
        for (size_t i = 0; i < load_ratios.size(); ++i) o << (i ? ";" : "") << fmt(load_ratios[i]);
        o << ',';
        bool first = true;
        for (const auto& [key, x] : phase_shares) {
            o << (first ? "" : ";") << key << ':' << fmt(x);
            first = false;
        }
        return o.str();
    }
    void write_text(std::ostream& out) const {  // report.cpp:127-159
        out << "input:     " << (file.empty() ? "<none>" : file)
            << (complemented ? " (complemented)" : "") << "  n=" << n << " m=" << m << "\n";
        out << "problem:   " << mode;
        if (k) out << " k=" << *k;
        out << "\n";
        out << "strategy:  " << strategy << "  workers=" << workers;
        if (strategy == "hybrid" || strategy == "gpu")
            out << " capacity=" << capacity << " threshold_fraction=" << threshold_fraction;
        if (strategy == "stackonly") out << " depth=" << depth;
        out << "\n";
        out << "status:    " << status << "  wall_ms=" << fmt(wall_ms) << "\n";
        if (size)
            out << "result:    size=" << *size << (feasible ? "" : " (infeasible)") << "\n";
        else
            out << "result:    infeasible\n";
        if (!cover.empty()) {
            out << "cover:    ";
            for (uint32_t v : cover) out << ' ' << v;
            out << "\n";
        }
        if (!worker_nodes.empty()) {
            out << "nodes:    ";
            for (auto c : worker_nodes) out << ' ' << c;
            out << "\n";
            out << "load:     ";
            for (auto r : load_ratios) out << ' ' << fmt(r);
            out << "\n";
        }
        if (!phase_shares.empty()) {
            out << "phases:\n";
            for (const auto& [key, x] : phase_shares)
                out << "  " << std::left << std::setw(28) << key << fmt(x) << "\n";
        }
    }
};

// collect_metrics (metrics.cpp:23-67): the device sums phase cycles over workers, so a share is
// the cycle-weighted mean of per-worker shares; with no instrumentation every phase is 0 and
// "other" is 1 (the reference's uninstrumented case).
void collect_metrics(RunReport& r, const uint64_t* phase, uint64_t active) {
    uint64_t total = 0;
    for (uint64_t x : r.worker_nodes) total += x;
    double mean = r.worker_nodes.empty() ? 0.0 : double(total) / r.worker_nodes.size();
    r.load_ratios.clear();
    for (uint64_t x : r.worker_nodes) r.load_ratios.push_back(mean > 0.0 ? double(x) / mean : 1.0);
    double tracked = 0.0;
    for (int p = 0; p < 10; ++p) {
        double s = active ? double(phase ? phase[p] : 0) / double(active) : 0.0;
        r.phase_shares[kPhaseKeys[p]] = s;
        tracked += s;
    }
    r.phase_shares["other"] = active ? (tracked >= 1.0 ? 0.0 : 1.0 - tracked) : 1.0;
}

// ------------------------------------------------------------------------------ options

struct CommonOptions {
    std::string input, format, output = "json", report_path;
    bool complement_input = false;
};

struct SolveOptions {
    std::string mode = "mvc";
    std::optional<uint32_t> k;
    std::string strategy = "hybrid";
    std::optional<unsigned> workers;  // default: hardware threads (main.cpp:43); gpu: fill device
    uint64_t capacity = 4096;
    double threshold_fraction = 0.5;
    unsigned depth = 8;
    uint64_t backoff_us = 50;
    std::optional<double> timeout_s;
    std::optional<uint64_t> node_budget;
    int device = 0;
};

struct SweepOptions {
    std::vector<std::string> strategies = {"seq", "stackonly", "hybrid"};
    std::vector<unsigned> workers = {8};
    std::vector<uint64_t> capacities = {4096};
    std::vector<double> fractions = {0.5};
    std::vector<unsigned> depths = {8};
    std::vector<std::string> instances = {"mvc", "pvc-1", "pvc", "pvc+1"};
    std::optional<double> timeout_s;
    std::string out_path;
};

struct GraphDeleter {
    void operator()(vcg_graph* g) const { vcg_graph_destroy(g); }
};
using GraphPtr = std::unique_ptr<vcg_graph, GraphDeleter>;

void check(int rc) {
    if (rc == VCG_OK) return;
    std::string msg = vcg_last_error();
    if (rc == VCG_EPARSE) throw UsageError("parse error: " + msg);
    throw std::runtime_error(msg);
}

// load_graph (main.cpp:61-74): format from the flag, else from the extension.
GraphPtr load_graph(const CommonOptions& o) {
    std::ifstream in(o.input, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open input file: " + o.input);
    std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    std::string format = o.format;
    if (format.empty()) {
        auto dot = o.input.find_last_of('.');
        auto slash = o.input.find_last_of('/');
        std::string ext = (dot == std::string::npos || (slash != std::string::npos && dot < slash))
                              ? "" : o.input.substr(dot);
        format = (ext == ".clq" || ext == ".col" || ext == ".dimacs") ? "dimacs" : "edgelist";
    }
    vcg_graph* g = nullptr;
    check(format == "dimacs" ? vcg_parse_dimacs(text.data(), text.size(), &g)
                             : vcg_parse_edge_list(text.data(), text.size(), &g));
    GraphPtr gp(g);
    if (o.complement_input) {
        vcg_graph* c = nullptr;
        check(vcg_complement(gp.get(), &c));
        gp.reset(c);
    }
    return gp;
}

unsigned default_workers(const std::string& strategy) {
    if (strategy == "gpu") return 0;  // one worker per resident warp slot of the device
    return std::max(1u, std::thread::hardware_concurrency());
}

// run_one (main.cpp:88-125) with "gpu" added.
RunReport run_one(const vcg_graph* g, const SolveOptions& o) {
    RunReport r;
    r.n = vcg_graph_num_vertices(g);
    r.m = vcg_graph_num_edges(g);
    r.mode = o.mode;
    if (o.mode == "pvc") r.k = *o.k;
    r.strategy = o.strategy;
    r.capacity = o.capacity;
    r.threshold_fraction = o.threshold_fraction;
    r.depth = o.depth;
    unsigned workers = o.workers ? *o.workers : default_workers(o.strategy);

    if (o.strategy == "oracle") {  // main.cpp:99-116
        if (r.n > 20) throw std::runtime_error("oracle strategy is limited to 20 vertices");
        auto t0 = std::chrono::steady_clock::now();
        uint32_t size = 0;
        std::vector<uint32_t> cover(r.n + 1);
        check(vcg_brute_force(g, &size, cover.data()));
        cover.resize(size);
        bool feasible = true;
        if (o.mode == "pvc") {
            feasible = size <= *o.k;
            if (!feasible) cover.clear();
        }
        r.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0)
                        .count();
        r.workers = 1;
        r.feasible = feasible;
        if (feasible) r.size = size;
        r.cover = std::move(cover);
        r.status = "complete";
        r.worker_nodes = {r.n == 0 ? 1ull : (1ull << r.n)};
        collect_metrics(r, nullptr, 0);
        return r;
    }

    vcg_params p;
    vcg_params_init(&p);
    p.mode = o.mode == "pvc" ? VCG_PVC : VCG_MVC;
    p.k = o.mode == "pvc" ? *o.k : 0;
    p.strategy = o.strategy == "seq" ? VCG_SEQ : o.strategy == "stackonly" ? VCG_STACKONLY
                                                                           : VCG_HYBRID;
    // hybrid: the reference's worker count shapes the report, the device is filled; gpu: the
    // count is device workers (0 = fill the device); stackonly: device workers
    p.workers = o.strategy == "seq" ? 1 : o.strategy == "gpu" ? 0 : workers;
    if (o.strategy == "gpu") p.device_workers = workers;
    p.capacity = o.capacity;
    p.threshold_fraction = o.threshold_fraction;
    p.depth = o.depth;
    p.backoff_us = o.backoff_us;
    p.timeout_s = o.timeout_s ? *o.timeout_s : -1.0;
    p.node_budget = o.node_budget ? *o.node_budget : 0;
    p.device = o.device;
    // (donate_oldest: vcg_params_init's default, the tuned policy of a filled device)
    vcg_result res;
    std::memset(&res, 0, sizeof res);
    check(vcg_solve(g, &p, &res));
    struct Free {
        vcg_result* r;
        ~Free() { vcg_result_free(r); }
    } guard{&res};

    static const char* kStatus[] = {"complete", "timeout", "budget"};
    r.status = kStatus[std::clamp(res.status, 0, 2)];
    r.feasible = res.feasible != 0;
    if (r.feasible) r.size = res.size;
    r.cover.assign(res.cover, res.cover + res.cover_len);
    r.wall_ms = res.wall_ms;
    // the reference echoes the configured count (seq: 1); gpu reports the workers it ran
    r.workers = o.strategy == "seq" ? 1 : (workers ? workers : res.num_workers);
    r.worker_nodes.assign(res.worker_nodes, res.worker_nodes + res.num_workers);
    r.wl_added = res.wl_added;
    r.wl_removed = res.wl_removed;
    r.wl_max_size = res.wl_max_size;
    collect_metrics(r, res.phase_cycles, res.active_cycles);
    r.engine = Json::Obj{
        {"nodes_total", res.nodes_total},     {"greedy_size", res.greedy_size},
        {"device_ms", res.device_ms},         {"greedy_ms", res.greedy_ms},
        {"h2d_ms", res.h2d_ms},               {"cover_from_search", bool(res.cover_from_search)},
        {"engine", res.engine == 2 ? "sparse" : "dense"},
        {"grid_blocks", res.grid_blocks},     {"block_threads", res.block_threads},
        {"kernel_launches", res.kernel_launches}, {"device", uint64_t(o.device)},
        {"version", vcg_version()}};
    return r;
}

void emit_text(const std::string& body, const std::string& path) {
    if (path.empty()) {
        std::cout << body;
        return;
    }
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot write report file: " + path);
    out << body;
}

void emit(const RunReport& r, const std::string& output, const std::string& path) {  // :127-145
    std::ostringstream body;
    if (output == "json") body << r.to_json().str() << "\n";
    else if (output == "csv") body << RunReport::csv_header() << "\n" << r.to_csv_row() << "\n";
    else r.write_text(body);
    emit_text(body.str(), path);
}

int do_solve(const CommonOptions& c, const SolveOptions& o) {  // main.cpp:147-164
    if (o.mode == "pvc" && !o.k) {
        std::cerr << "error: --mode pvc requires --k\n";
        return kExitUsage;
    }
    if (o.mode == "pvc" && *o.k < 1) {
        std::cerr << "error: --k must be >= 1\n";
        return kExitUsage;
    }
    GraphPtr g = load_graph(c);
    RunReport r = run_one(g.get(), o);
    r.file = c.input;
    r.complemented = c.complement_input;
    emit(r, c.output, c.report_path);
    return r.status == "complete" ? kExitOk : kExitIncomplete;
}

struct SweepRow {
    std::string instance;
    RunReport report;
    bool best = false;
};

// do_sweep (main.cpp:173-299): PVC instances take k from a completed MVC solve (chained first
// when no "mvc" instance is requested); the fastest complete run per (instance, strategy) is
// flagged best.
int do_sweep(const CommonOptions& c, const SweepOptions& s) {
    GraphPtr g = load_graph(c);
    std::optional<uint32_t> min_size;
    bool wants_pvc = false, has_mvc = false;
    for (const auto& inst : s.instances) (inst == "mvc" ? has_mvc : wants_pvc) = true;
    if (wants_pvc && !has_mvc) {
        SolveOptions pre;
        pre.strategy = "hybrid";
        pre.workers = s.workers.empty() ? 1u : s.workers.front();
        pre.timeout_s = s.timeout_s;
        RunReport r = run_one(g.get(), pre);
        if (r.status == "complete" && r.size) min_size = *r.size;
    }

    std::vector<SweepRow> rows;
    auto run_configs = [&](const std::string& instance, const std::string& strategy,
                           const std::string& mode, std::optional<uint32_t> k) {
        size_t start = rows.size();
        SolveOptions o;
        o.mode = mode;
        o.k = k;
        o.strategy = strategy;
        o.timeout_s = s.timeout_s;
        auto push = [&](const SolveOptions& cfg) {
            RunReport r = run_one(g.get(), cfg);
            r.file = c.input;
            r.complemented = c.complement_input;
            rows.push_back({instance, std::move(r), false});
        };
        if (strategy == "seq" || strategy == "oracle") {
            o.workers = 1;
            push(o);
        } else if (strategy == "stackonly") {
            for (unsigned w : s.workers)
                for (unsigned d : s.depths) {
                    o.workers = w;
                    o.depth = d;
                    push(o);
                }
        } else {
            for (unsigned w : s.workers)
                for (uint64_t cap : s.capacities)
                    for (double f : s.fractions) {
                        o.workers = w;
                        o.capacity = cap;
                        o.threshold_fraction = f;
                        push(o);
                    }
        }
        size_t best = rows.size();
        for (size_t i = start; i < rows.size(); ++i) {
            if (rows[i].report.status != "complete") continue;
            if (best == rows.size() || rows[i].report.wall_ms < rows[best].report.wall_ms) best = i;
        }
        if (best < rows.size()) rows[best].best = true;
    };

    std::vector<std::string> ordered = s.instances;
    std::stable_partition(ordered.begin(), ordered.end(),
                          [](const std::string& x) { return x == "mvc"; });
    for (const auto& instance : ordered) {
        std::string mode = instance == "mvc" ? "mvc" : "pvc";
        std::optional<uint32_t> k;
        if (mode == "pvc") {
            if (!min_size) {
                std::cerr << "note: skipping " << instance << " (no completed MVC solve for min)\n";
                continue;
            }
            int64_t base = *min_size;
            int64_t kk = instance == "pvc-1" ? base - 1 : instance == "pvc+1" ? base + 1 : base;
            if (kk < 1) {
                std::cerr << "note: skipping " << instance << " (k would be " << kk << ")\n";
                continue;
            }
            k = uint32_t(kk);
        }
        for (const auto& strategy : s.strategies) run_configs(instance, strategy, mode, k);
        if (instance == "mvc" && !min_size) {
            for (const auto& row : rows)
                if (row.instance == "mvc" && row.report.status == "complete" && row.report.size) {
                    min_size = *row.report.size;
                    break;
                }
            if (!min_size && wants_pvc)
                std::cerr << "note: MVC did not complete; PVC instances will be skipped\n";
        }
    }

    std::ostringstream body;
    if (c.output == "csv" || c.output == "text") {
        body << "instance,best," << RunReport::csv_header() << "\n";
        for (const auto& row : rows)
            body << row.instance << ',' << (row.best ? 1 : 0) << ',' << row.report.to_csv_row()
                 << "\n";
    } else {
        Json::Arr arr;
        for (const auto& row : rows) {
            Json item = row.report.to_json();
            auto& obj = std::get<Json::Obj>(item.v);
            obj["instance"] = row.instance;
            obj["best"] = row.best;
            arr.push_back(std::move(item));
        }
        body << Json(std::move(arr)).str() << "\n";
    }
    emit_text(body.str(), s.out_path);
    return kExitOk;
}

// ------------------------------------------------------------------------------ parsing

template <class T>
T parse_num(const std::string& opt, const std::string& s) {
    T x{};
    const char* b = s.data();
    const char* e = b + s.size();
    std::from_chars_result r;
    if constexpr (std::is_floating_point_v<T>) {
        char* end = nullptr;
        x = std::strtod(s.c_str(), &end);
        r.ptr = end;
        r.ec = s.empty() ? std::errc::invalid_argument : std::errc();
    } else {
        r = std::from_chars(b, e, x);
    }
    if (r.ec != std::errc() || r.ptr != e)
        throw UsageError(opt + ": Value " + s + " could not be converted");
    return x;
}

std::vector<std::string> split(const std::string& s) {
    std::vector<std::string> out;
    std::string cur;
    std::istringstream in(s);
    while (std::getline(in, cur, ',')) out.push_back(cur);
    return out;
}

void member(const std::string& opt, const std::string& v, std::initializer_list<const char*> ok) {
    for (const char* x : ok)
        if (v == x) return;
    throw UsageError(opt + ": " + v + " not in {" + [&] {
        std::string s;
        for (const char* x : ok) s += (s.empty() ? "" : ",") + std::string(x);
        return s;
    }() + "}");
}

const char* kUsage =
    "Exact MVC/PVC solver with hybrid worklist load balancing (B200 engine)\n"
    "Usage: vcsolve [OPTIONS] [SUBCOMMAND]\n"
    "  --input FILE                Graph file (required)\n"
    "  --format dimacs|edgelist    Input format (default: from the extension)\n"
    "  --complement                Solve on the edge complement\n"
    "  --mode mvc|pvc              Problem variant\n"
    "  --k K                       Cover size bound for pvc\n"
    "  --strategy seq|stackonly|hybrid|gpu|oracle\n"
    "  --workers N                 Worker count (hybrid: report entries, the device is always\n"
    "                              filled; gpu/stackonly: warps on the device, gpu 0 = fill)\n"
    "  --worklist-capacity C       Hybrid worklist capacity\n"
    "  --threshold-fraction F      Hybrid donation threshold as a fraction of capacity\n"
    "  --depth D                   StackOnly sub-tree starting depth (1..30)\n"
    "  --backoff-us B              Idle back-off between worklist retries\n"
    "  --timeout-s T               Wall-clock limit per solve\n"
    "  --node-budget N             Visited-node limit per solve\n"
    "  --output json|csv|text      Report format\n"
    "  --report PATH               Write the report to this path\n"
    "  --device I                  CUDA device ordinal\n"
    "Subcommands:\n"
    "  sweep  --strategies --workers --capacities --fractions --depths --instances\n"
    "         --timeout-s --out   (comma-separated lists)\n";

}  // namespace

int main(int argc, char** argv) {
    CommonOptions common;
    SolveOptions solve;
    SweepOptions sweep;
    bool in_sweep = false, depth_given = false, have_input = false;
    try {
        std::vector<std::string> args(argv + 1, argv + argc);
        for (size_t i = 0; i < args.size(); ++i) {
            std::string a = args[i];
            if (a == "-h" || a == "--help") {
                std::cout << kUsage;
                return kExitOk;
            }
            if (a == "sweep" && !in_sweep) {
                in_sweep = true;
                continue;
            }
            std::string val;
            bool inline_val = false;
            if (auto eq = a.find('='); a.rfind("--", 0) == 0 && eq != std::string::npos) {
                val = a.substr(eq + 1);
                a = a.substr(0, eq);
                inline_val = true;
            }
            auto next = [&]() -> std::string {
                if (inline_val) return val;
                if (i + 1 >= args.size()) throw UsageError(a + ": 1 required argument missing");
                return args[++i];
            };
            if (a == "--complement") {
                common.complement_input = true;
                continue;
            }
            if (in_sweep) {  // sweep options shadow the parent's; the rest fall through
                if (a == "--strategies") {
                    sweep.strategies = split(next());
                    for (const auto& s : sweep.strategies)
                        member(a, s, {"seq", "stackonly", "hybrid", "gpu", "oracle"});
                    continue;
                }
                if (a == "--workers") {
                    sweep.workers.clear();
                    for (const auto& s : split(next())) sweep.workers.push_back(parse_num<unsigned>(a, s));
                    continue;
                }
                if (a == "--capacities") {
                    sweep.capacities.clear();
                    for (const auto& s : split(next())) sweep.capacities.push_back(parse_num<uint64_t>(a, s));
                    continue;
                }
                if (a == "--fractions") {
                    sweep.fractions.clear();
                    for (const auto& s : split(next())) sweep.fractions.push_back(parse_num<double>(a, s));
                    continue;
                }
                if (a == "--depths") {
                    sweep.depths.clear();
                    for (const auto& s : split(next())) sweep.depths.push_back(parse_num<unsigned>(a, s));
                    continue;
                }
                if (a == "--instances") {
                    sweep.instances = split(next());
                    for (const auto& s : sweep.instances) member(a, s, {"mvc", "pvc-1", "pvc", "pvc+1"});
                    continue;
                }
                if (a == "--timeout-s") {
                    sweep.timeout_s = parse_num<double>(a, next());
                    continue;
                }
                if (a == "--out") {
                    sweep.out_path = next();
                    continue;
                }
            }
            if (a == "--input") {
                common.input = next();
                have_input = true;
            } else if (a == "--format") {
                common.format = next();
                member(a, common.format, {"dimacs", "edgelist"});
            } else if (a == "--mode") {
                solve.mode = next();
                member(a, solve.mode, {"mvc", "pvc"});
            } else if (a == "--k") {
                solve.k = parse_num<uint32_t>(a, next());
            } else if (a == "--strategy") {
                solve.strategy = next();
                member(a, solve.strategy, {"seq", "stackonly", "hybrid", "gpu", "oracle"});
            } else if (a == "--workers") {
                solve.workers = parse_num<unsigned>(a, next());
            } else if (a == "--worklist-capacity") {
                solve.capacity = parse_num<uint64_t>(a, next());
            } else if (a == "--threshold-fraction") {
                solve.threshold_fraction = parse_num<double>(a, next());
            } else if (a == "--depth") {
                solve.depth = parse_num<unsigned>(a, next());
                if (solve.depth < 1 || solve.depth > 30)
                    throw UsageError("--depth: Value " + std::to_string(solve.depth) +
                                     " not in range [1 - 30]");
                depth_given = true;
            } else if (a == "--backoff-us") {
                solve.backoff_us = parse_num<uint64_t>(a, next());
            } else if (a == "--timeout-s") {
                solve.timeout_s = parse_num<double>(a, next());
            } else if (a == "--node-budget") {
                solve.node_budget = parse_num<uint64_t>(a, next());
            } else if (a == "--output") {
                common.output = next();
                member(a, common.output, {"json", "csv", "text"});
            } else if (a == "--report") {
                common.report_path = next();
            } else if (a == "--device") {
                solve.device = parse_num<int>(a, next());
            } else {
                throw UsageError("The following argument was not expected: " + a);
            }
        }
        if (!have_input) throw UsageError("--input is required");
    } catch (const std::exception& e) {
        std::cerr << e.what() << "\nRun with --help for more information.\n";
        return kExitUsage;
    }

    try {
        if (in_sweep) return do_sweep(common, sweep);
        if (depth_given && (solve.strategy == "hybrid" || solve.strategy == "gpu"))
            std::cerr << "warning: --depth has no effect with --strategy " << solve.strategy
                      << "; ignored\n";
        return do_solve(common, solve);
    } catch (const UsageError& e) {
        std::cerr << e.what() << "\n";
        return kExitUsage;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return kExitUsage;
    }
}
