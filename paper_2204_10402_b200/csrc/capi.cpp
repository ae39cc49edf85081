// capi.cpp — the extern "C" boundary (include/vcgpu.h). Maps C++ exceptions to status codes
// the way the reference's pybind11 layer maps them to Python (bindings.cpp:106 ParseError ->
// ValueError, std::invalid_argument -> ValueError) and runs the host part of run_hybrid
// (scheduler.cpp:328-359): validate, greedy seed, device search, certificate assembly.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <future>
#include <new>
#include <stdexcept>
#include <string>

#include "../../include/vcgpu.h"
#include "engine.hpp"
#include "host_graph.hpp"

struct vcg_graph {
    vcg::Graph g;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const vcg::ParseError& e) {
        return fail(VCG_EPARSE, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(VCG_EINVAL, e.what());
    } catch (const std::bad_alloc&) {
        return fail(VCG_ENOMEM, "out of memory");
    } catch (const std::runtime_error& e) {
        const std::string w = e.what();
        return fail(w.rfind("CUDA", 0) == 0 ? VCG_ECUDA : VCG_EINVAL, w);
    } catch (...) {
        return fail(VCG_EINVAL, "unknown error");
    }
}

int emit(vcg::Graph&& g, vcg_graph** out) {
    if (!out) return fail(VCG_EINVAL, "null output handle");
    *out = new vcg_graph{std::move(g)};
    return VCG_OK;
}

}  // namespace

extern "C" {

const char* vcg_last_error(void) { return g_err.c_str(); }
const char* vcg_version(void) { return "vcgpu 0.1.0 (sm_100a)"; }
int vcg_device_count(void) { return vcg::device_count(); }

int vcg_graph_from_csr(uint32_t n, uint64_t m, const uint64_t* offsets,
                       const uint32_t* neighbors, uint32_t id_base, vcg_graph** out) {
    return guarded([&]() -> int {
        if (!offsets || (m && !neighbors)) return fail(VCG_EINVAL, "null CSR array");
        vcg::Graph g;
        g.n = n;
        g.m = m;
        g.id_base = id_base;
        g.off.assign(offsets, offsets + size_t(n) + 1);
        g.nbr.assign(neighbors, neighbors + 2 * m);
        if (!vcg::check_invariants(g)) return fail(VCG_EINVAL, "CSR violates graph invariants");
        return emit(std::move(g), out);
    });
}

int vcg_make_graph(uint32_t n, uint64_t num_pairs, const uint32_t* pairs, uint32_t id_base,
                   vcg_graph** out) {
    return guarded([&]() -> int {
        if (num_pairs && !pairs) return fail(VCG_EINVAL, "null pairs");
        std::vector<std::pair<uint32_t, uint32_t>> e(num_pairs);
        for (uint64_t i = 0; i < num_pairs; ++i) e[i] = {pairs[2 * i], pairs[2 * i + 1]};
        return emit(vcg::make_graph(n, e, id_base), out);
    });
}

int vcg_parse_edge_list(const char* text, size_t len, vcg_graph** out) {
    return guarded([&]() -> int { return emit(vcg::parse_edge_list(text ? text : "", text ? len : 0), out); });
}

int vcg_parse_dimacs(const char* text, size_t len, vcg_graph** out) {
    return guarded([&]() -> int { return emit(vcg::parse_dimacs(text ? text : "", text ? len : 0), out); });
}

int vcg_complement(const vcg_graph* g, vcg_graph** out) {
    return guarded([&]() -> int {
        if (!g) return fail(VCG_EINVAL, "null graph");
        return emit(vcg::complement(g->g), out);
    });
}

int vcg_write_edge_list(const vcg_graph* g, char** text, size_t* len) {
    return guarded([&]() -> int {
        if (!g || !text || !len) return fail(VCG_EINVAL, "null argument");
        std::string s = vcg::write_edge_list(g->g);
        char* p = static_cast<char*>(std::malloc(s.size() + 1));
        if (!p) return fail(VCG_ENOMEM, "out of memory");
        std::memcpy(p, s.data(), s.size());
        p[s.size()] = 0;
        *text = p;
        *len = s.size();
        return VCG_OK;
    });
}

void vcg_free_buffer(void* p) { std::free(p); }
void vcg_graph_destroy(vcg_graph* g) { delete g; }
uint32_t vcg_graph_num_vertices(const vcg_graph* g) { return g ? g->g.n : 0; }
uint64_t vcg_graph_num_edges(const vcg_graph* g) { return g ? g->g.m : 0; }
uint32_t vcg_graph_id_base(const vcg_graph* g) { return g ? g->g.id_base : 0; }
const uint64_t* vcg_graph_offsets(const vcg_graph* g) { return g ? g->g.off.data() : nullptr; }
const uint32_t* vcg_graph_neighbors(const vcg_graph* g) { return g ? g->g.nbr.data() : nullptr; }

int vcg_has_edge(const vcg_graph* g, uint32_t u, uint32_t v) {
    if (!g || u >= g->g.n || v >= g->g.n) return 0;
    return g->g.has_edge(u, v) ? 1 : 0;
}

int vcg_graph_equal(const vcg_graph* a, const vcg_graph* b) {
    if (!a || !b) return 0;
    const vcg::Graph &x = a->g, &y = b->g;
    return x.n == y.n && x.m == y.m && x.id_base == y.id_base && x.off == y.off && x.nbr == y.nbr;
}

int vcg_check_invariants(const vcg_graph* g) { return g && vcg::check_invariants(g->g) ? 1 : 0; }

int vcg_greedy(const vcg_graph* g, uint32_t* size, uint32_t* cover) {
    return guarded([&]() -> int {
        if (!g || !size) return fail(VCG_EINVAL, "null argument");
        vcg::Greedy r = vcg::greedy_approx(g->g);
        *size = r.size;
        if (cover) std::memcpy(cover, r.cover.data(), r.cover.size() * 4);
        return VCG_OK;
    });
}

int vcg_brute_force(const vcg_graph* g, uint32_t* size, uint32_t* cover) {
    return guarded([&]() -> int {
        if (!g || !size) return fail(VCG_EINVAL, "null argument");
        if (g->g.n > 20) return fail(VCG_ERANGE, "brute force oracle is limited to 20 vertices");
        std::vector<uint32_t> c;
        *size = vcg::brute_force(g->g, c);
        if (cover)
            for (size_t i = 0; i < c.size(); ++i) cover[i] = c[i] + g->g.id_base;
        return VCG_OK;
    });
}

int vcg_verify_cover(const vcg_graph* g, const uint32_t* cover, uint32_t len, int* ok) {
    return guarded([&]() -> int {
        if (!g || !ok || (len && !cover)) return fail(VCG_EINVAL, "null argument");
        *ok = vcg::verify_cover(g->g, cover, len) ? 1 : 0;
        return VCG_OK;
    });
}

void vcg_params_init(vcg_params* p) {
    if (!p) return;
    std::memset(p, 0, sizeof(*p));
    p->mode = VCG_MVC;
    p->strategy = VCG_HYBRID;
    p->capacity = 4096;             // bindings.cpp:177
    p->threshold_fraction = 0.5;    // bindings.cpp:177
    p->depth = 8;                   // bindings.cpp:177
    p->backoff_us = 50;             // bindings.cpp:178
    p->timeout_s = -1.0;
    p->rules = VCG_RULES_REFERENCE;
    p->donate_oldest = 1;
}

namespace {

// validate_config (scheduler.cpp:20-29) + the k >= 1 check (:330); 0 when valid
int validate(const vcg_params* p) {
    if (p->capacity < 1) return fail(VCG_EINVAL, "worklist_capacity must be >= 1");
    if (!(p->threshold_fraction > 0.0) || p->threshold_fraction > 1.0)
        return fail(VCG_EINVAL, "threshold_fraction must be in (0, 1]");
    if (p->depth < 1 || p->depth > 30) return fail(VCG_EINVAL, "stackonly_depth must be in [1, 30]");
    if (p->mode == VCG_PVC && p->k < 1) return fail(VCG_EINVAL, "pvc requires k >= 1");
    if (p->strategy < VCG_HYBRID || p->strategy > VCG_STACKONLY)
        return fail(VCG_EINVAL, "unknown strategy");
    if (p->num_seeds && !p->seeds) return fail(VCG_EINVAL, "null seeds");
    return VCG_OK;
}

// The host half of run_hybrid (scheduler.cpp:328-359) around one device search: the greedy
// seed (scheduler.cpp:333-340, counted in wall_ms like the reference; MVC needs it as the initial
// bound, PVC only reports its size, so there it runs on a host thread while the device
// searches), the engine spec, and finish_run's result (scheduler.cpp:299-324).
struct HostRun {
    const vcg::Graph& g;
    const vcg_params* p;
    vcg_result* out;
    bool pvc;
    std::chrono::steady_clock::time_point t0;
    vcg::Greedy greedy;
    std::future<vcg::Greedy> greedy_async;
    vcg::SolveSpec s;

    bool greedy_deferred = false;  // PVC: computed by the caller while the search runs
    vcg::Greedy run_greedy() {
        const auto a = std::chrono::steady_clock::now();
        vcg::Greedy gr = vcg::greedy_approx(g);
        out->greedy_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
        return gr;
    }
    // defer_pvc_greedy: the caller runs the PVC greedy itself while the kernel searches
    // (vcg_solve: solve_on_device's while_running hook) instead of on a new host thread
    HostRun(const vcg::Graph& g_, const vcg_params* p_, vcg_result* out_, bool defer_pvc_greedy = false)
        : g(g_), p(p_), out(out_), pvc(p_->mode == VCG_PVC), t0(std::chrono::steady_clock::now()) {
        std::memset(out, 0, sizeof(*out));
        if (pvc && g.n > 0 && defer_pvc_greedy)
            greedy_deferred = true;
        else if (pvc && g.n > 0)
            greedy_async = std::async(std::launch::async, [this]() { return run_greedy(); });
        else
            greedy = run_greedy();
        s.pvc = pvc;
        s.k = p->k;
        s.strategy = p->strategy;
        // hybrid fills the device unless device_workers says otherwise; the reference's
        // num_workers only shapes the report (finish folds the device workers into it)
        s.workers = p->device_workers ? p->device_workers
                                      : (p->strategy == VCG_HYBRID ? 0u : p->workers);
        s.capacity = p->capacity;
        // worklist_threshold (scheduler.cpp:14-18)
        long long t = std::llround(p->threshold_fraction * double(p->capacity));
        s.threshold = (uint64_t)std::max<long long>(1, std::min<long long>(t, (long long)p->capacity));
        s.depth = p->depth;
        s.backoff_us = p->backoff_us;
        s.timeout_s = p->timeout_s;
        s.node_budget = p->node_budget;
        s.device = p->device;
        s.rules = p->rules;
        s.block_warps = p->block_warps;
        s.engine = p->engine;
        s.instrument = p->instrument != 0;
        s.donate_oldest = p->donate_oldest != 0;
        s.best = pvc ? p->k : greedy.size;
        if (!pvc && p->initial_best && p->initial_best < s.best) s.best = p->initial_best;
        // stack_bound_for (scheduler.cpp:118-121)
        s.stack_bound = pvc ? std::min<uint32_t>(p->k, g.n) : greedy.size;
        s.seeds = p->seeds;
        s.num_seeds = p->num_seeds;
        if (p->debug_flags & VCG_DEBUG_SMALL_STACK) s.stack_cap = 3;
        s.mailbox = p->mailbox;
        s.stream = p->stream;
    }
    ~HostRun() {  // the greedy thread never outlives the call, even on a device error
        if (greedy_async.valid()) greedy_async.wait();
    }

    void finish(vcg::SolveOut& r) {
        if (greedy_async.valid()) greedy = greedy_async.get();
        out->greedy_size = greedy.size;
        // finish_run (scheduler.cpp:299-324): certificate in original ids
        const std::vector<uint32_t>* cov = nullptr;
        if (pvc) {
            out->feasible = r.found ? 1 : 0;
            if (r.found) {
                cov = &r.cover;
                out->size = (uint32_t)r.cover.size();
                out->cover_from_search = 1;
            }
        } else {
            out->feasible = 1;
            if (r.found && r.cover.size() < greedy.size) {
                cov = &r.cover;
                out->cover_from_search = 1;
            } else {
                cov = &greedy.cover;
            }
            out->size = (uint32_t)cov->size();
        }
        if (cov && !cov->empty()) {
            out->cover = static_cast<uint32_t*>(std::malloc(cov->size() * 4));
            for (size_t i = 0; i < cov->size(); ++i) out->cover[i] = (*cov)[i] + g.id_base;
        }
        out->cover_len = cov ? (uint32_t)cov->size() : 0;
        out->status = r.status;
        // WorkerMetrics per reference worker: a hybrid solve that filled the device reports its
        // device workers folded into the configured num_workers (device worker i counts for
        // worker i % num_workers; stack high water = the maximum)
        const size_t dw = r.worker_nodes.size();
        const bool fold = p->strategy == VCG_HYBRID && !p->device_workers && p->workers && dw;
        const size_t nw = fold ? p->workers : dw;
        out->num_workers = (uint32_t)nw;
        out->worker_nodes = static_cast<uint64_t*>(std::calloc(std::max<size_t>(1, nw), 8));
        out->worker_stack_high_water = static_cast<uint64_t*>(std::calloc(std::max<size_t>(1, nw), 8));
        for (size_t i = 0; i < dw; ++i) {
            const size_t j = fold ? i % nw : i;
            out->worker_nodes[j] += r.worker_nodes[i];
            out->worker_stack_high_water[j] =
                std::max<uint64_t>(out->worker_stack_high_water[j], r.worker_high_water[i]);
            out->nodes_total += r.worker_nodes[i];
        }
        out->wl_added = r.wl_added;
        out->wl_removed = r.wl_removed;
        out->wl_max_size = r.wl_max_size;
        out->wl_current_size = r.wl_current;
        out->device_ms = r.device_ms;
        out->h2d_ms = r.h2d_ms;
        out->h2d_bytes = r.h2d_bytes;
        out->d2h_bytes = r.d2h_bytes;
        out->rounds = r.rounds;
        out->maxdeg_passes = r.maxdeg;
        out->children = r.children;
        out->removals = r.removals;
        out->donated = r.donated;
        out->removals_deg1 = r.rm1;
        out->removals_deg2 = r.rm2;
        out->removals_high = r.rmh;
        out->doomed = r.dooms;
        out->degree_bytes = r.degree_bytes;
        out->n_padded = r.n_padded;
        out->engine = r.engine;
        out->grid_blocks = r.grid;
        out->block_threads = r.block;
        out->kernel_launches = r.launches;
        for (int i = 0; i < 10; ++i) out->phase_cycles[i] = r.phase[i];
        out->active_cycles = r.active_cycles;
        for (int i = 0; i < 4; ++i) {
            out->t_first_ms[i] = r.t_first_ms[i];
            out->t_end_ms[i] = r.t_end_ms[i];
            out->t_lastwait_ms[i] = r.t_lastwait_ms[i];
        }
        out->idle_share = r.idle_share;
        out->donated_peer = r.donated_peer;
        out->wall_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }

    // verify_cover (bounds.cpp:32-45) on every cover the engine returns (O(n + m) on the host):
    // a cover that fails is an engine fault, reported as VCG_EVERIFY with the result freed.
    // (VCG_DEBUG_CORRUPT_COVER drops the first cover vertex first: the test of this check.)
    int verified() {
        if (!out->cover_len) return VCG_OK;
        if ((p->debug_flags & VCG_DEBUG_CORRUPT_COVER) && out->cover_len) {
            std::memmove(out->cover, out->cover + 1, (out->cover_len - 1) * 4);
            --out->cover_len;
        }
        std::vector<uint32_t> ids(out->cover, out->cover + out->cover_len);
        for (uint32_t& v : ids) v -= g.id_base;
        bool ok = vcg::verify_cover(g, ids.data(), ids.size());
        if (ok && pvc && out->cover_len > p->k) ok = false;
        if (ok) return VCG_OK;
        const std::string msg = "engine returned an invalid cover (size " +
                                std::to_string(out->cover_len) +
                                (pvc ? ", k " + std::to_string(p->k) : std::string()) +
                                "): verify_cover failed";
        vcg_result_free(out);
        return fail(VCG_EVERIFY, msg);
    }
};

}  // namespace

namespace {
// Debug option (VCG_DEBUG_CERTIFY): re-prove a parallel MVC optimum by PVC(s - 1). The PVC search
// has no bound dynamics (its tree and node count are the reference's exactly), so a "no" proves
// the size s found optimal and a "yes" improves the certificate and repeats. The parallel MVC
// search is exact on its own (the dense engine's edge-count prune uses the bound its reduction
// reached fixpoint under, even when a poll lowered the bound since; see settle() in
// dense_kernels.cuh), so this is off by default;
// it exists to cross-check that claim. Its nodes and device time are reported separately
// (certify_nodes / certify_ms), and it only spends what is left of the caller's time and node
// limits.
void certify_mvc(const vcg::Graph& g, HostRun& h, vcg::SolveOut& r, vcg_result* out) {
    if (r.status != 0) return;
    if (h.greedy_async.valid()) h.greedy = h.greedy_async.get();
    uint32_t best = h.greedy.size;
    if (h.s.best < best) best = h.s.best;  // an external bound (initial_best)
    if (r.found && r.cover.size() < best) best = (uint32_t)r.cover.size();
    uint64_t nodes_used = 0;
    for (uint64_t x : r.worker_nodes) nodes_used += x;
    while (best >= 2) {  // (a cover of size 0 exists only without edges: then best is 0)
        vcg::SolveSpec s2 = h.s;
        s2.pvc = true;
        s2.k = best - 1;
        s2.best = s2.k;
        s2.stack_bound = std::min<uint32_t>(s2.k, g.n);
        s2.mailbox = nullptr;
        if (h.s.timeout_s >= 0) {
            const double spent = std::chrono::duration<double>(std::chrono::steady_clock::now() - h.t0).count();
            s2.timeout_s = std::max(0.0, h.s.timeout_s - spent);
        }
        if (h.s.node_budget) {
            if (nodes_used >= h.s.node_budget) {
                r.status = 2;
                return;
            }
            s2.node_budget = h.s.node_budget - nodes_used;
        }
        vcg::SolveOut r2;
        vcg::solve_on_device(g, s2, r2);
        out->certify_ms += r2.device_ms;
        out->certify_launches += r2.launches;
        for (uint64_t x : r2.worker_nodes) {
            out->certify_nodes += x;
            nodes_used += x;
        }
        if (r2.status != 0) {
            r.status = r2.status;
            return;
        }
        if (!r2.found) return;  // PVC(best - 1) is a no-instance: best is the optimum
        if (r2.cover.size() >= best)
            throw std::runtime_error("certify: PVC(" + std::to_string(best - 1) +
                                     ") returned a cover of size " + std::to_string(r2.cover.size()));
        r.found = true;
        r.cover = r2.cover;
        best = (uint32_t)r2.cover.size();
    }
}
}  // namespace

int vcg_solve(const vcg_graph* gh, const vcg_params* p, vcg_result* out) {
    return guarded([&]() -> int {
        if (!gh || !p || !out) return fail(VCG_EINVAL, "null argument");
        std::memset(out, 0, sizeof(*out));
        if (const int e = validate(p)) return e;
        HostRun h(gh->g, p, out, true);
        vcg::SolveOut r;
        if (gh->g.n == 0) {
            // no vertex: one root visit, nothing to branch on (MVC 0; PVC feasible, empty)
            r.worker_nodes.assign(1, 1);
            r.worker_high_water.assign(1, 0);
            r.found = h.pvc;
            r.wl_added = r.wl_removed = 1;
        } else {
            vcg::solve_on_device(gh->g, h.s, r, [&h]() {
                if (h.greedy_deferred) {
                    h.greedy = h.run_greedy();
                    h.greedy_deferred = false;
                }
            });
            if (h.greedy_deferred) h.greedy = h.run_greedy();  // (not reached: the hook ran)
            if (!h.pvc && (p->debug_flags & VCG_DEBUG_CERTIFY) && h.s.strategy != VCG_SEQ)
                certify_mvc(gh->g, h, r, out);
        }
        h.finish(r);
        return h.verified();
    });
}

// ------------------------------------------------------------------ multi-shard sessions

struct vcg_session {
    const vcg_graph* g;
    vcg_params p;
    vcg_result* out = nullptr;   // filled by wait
    std::unique_ptr<HostRun> host;
    vcg::Session* ses = nullptr;
    vcg_result scratch;
    ~vcg_session() {
        if (ses) vcg::session_close(ses);
    }
};

int vcg_session_open(const vcg_graph* gh, const vcg_params* p, int with_root, vcg_session** out) {
    return guarded([&]() -> int {
        if (!gh || !p || !out) return fail(VCG_EINVAL, "null argument");
        *out = nullptr;
        if (const int e = validate(p)) return e;
        if (gh->g.n == 0) return fail(VCG_EINVAL, "multi-shard sessions need a non-empty graph");
        if (p->strategy != VCG_HYBRID) return fail(VCG_EINVAL, "multi-shard sessions run strategy hybrid/gpu");
        auto s = std::make_unique<vcg_session>();
        s->g = gh;
        s->p = *p;
        s->host = std::make_unique<HostRun>(gh->g, &s->p, &s->scratch);
        s->host->s.no_root = p->num_seeds == 0 && !with_root;
        s->ses = vcg::session_open(gh->g, s->host->s);
        *out = s.release();
        return VCG_OK;
    });
}

size_t vcg_session_handle_bytes(void) { return vcg::session_handle_bytes(); }

int vcg_session_export(const vcg_session* s, void* handle) {
    return guarded([&]() -> int {
        if (!s || !handle) return fail(VCG_EINVAL, "null argument");
        vcg::session_export(s->ses, handle);
        return VCG_OK;
    });
}

int vcg_session_link_ipc(vcg_session* s, uint32_t world, uint32_t rank, const void* handles,
                         const uint64_t* seeds_per_shard) {
    return guarded([&]() -> int {
        if (!s || !handles || !seeds_per_shard) return fail(VCG_EINVAL, "null argument");
        if (world < 1 || world > VCG_MAX_SHARDS || rank >= world)
            return fail(VCG_EINVAL, "bad shard rank / world");
        vcg::session_link_ipc(s->ses, world, rank, handles, seeds_per_shard);
        return VCG_OK;
    });
}

int vcg_session_link_local(vcg_session* const* shards, uint32_t world) {
    return guarded([&]() -> int {
        if (!shards) return fail(VCG_EINVAL, "null argument");
        if (world < 1 || world > VCG_MAX_SHARDS) return fail(VCG_EINVAL, "bad shard world");
        std::vector<vcg::Session*> v(world);
        for (uint32_t i = 0; i < world; ++i) {
            if (!shards[i]) return fail(VCG_EINVAL, "null shard");
            v[i] = shards[i]->ses;
        }
        vcg::session_link_local(v.data(), world);
        return VCG_OK;
    });
}

int vcg_session_reset(vcg_session* s) {
    return guarded([&]() -> int {
        if (!s) return fail(VCG_EINVAL, "null argument");
        s->host->t0 = std::chrono::steady_clock::now();
        vcg::session_reset(s->ses);
        return VCG_OK;
    });
}

int vcg_session_launch(vcg_session* s) {
    return guarded([&]() -> int {
        if (!s) return fail(VCG_EINVAL, "null argument");
        vcg::session_launch(s->ses);
        return VCG_OK;
    });
}

int vcg_session_wait(vcg_session* s, vcg_result* out) {
    return guarded([&]() -> int {
        if (!s || !out) return fail(VCG_EINVAL, "null argument");
        vcg::SolveOut r;
        vcg::session_wait(s->ses, r);
        HostRun& h = *s->host;
        if (h.greedy_async.valid()) h.greedy = h.greedy_async.get();  // (it writes scratch)
        std::memset(out, 0, sizeof(*out));
        out->greedy_ms = s->scratch.greedy_ms;
        h.out = out;
        h.finish(r);
        return h.verified();
    });
}

void vcg_session_close(vcg_session* s) { delete s; }

int vcg_device_workers(const vcg_graph* g, int32_t device, uint32_t* workers) {
    return guarded([&]() -> int {
        if (!g || !workers) return fail(VCG_EINVAL, "null argument");
        *workers = vcg::full_device_workers(g->g, device);
        return VCG_OK;
    });
}

int vcg_expand_frontier(const vcg_graph* gh, const vcg_params* p, uint64_t target,
                        vcg_frontier* out) {
    return guarded([&]() -> int {
        if (!gh || !p || !out) return fail(VCG_EINVAL, "null argument");
        std::memset(out, 0, sizeof(*out));
        if (p->mode == VCG_PVC && p->k < 1) return fail(VCG_EINVAL, "pvc requires k >= 1");
        const vcg::Graph& g = gh->g;
        const bool pvc = p->mode == VCG_PVC;
        vcg::Greedy greedy = vcg::greedy_approx(g);
        out->greedy_size = greedy.size;
        vcg::SolveSpec s;
        s.pvc = pvc;
        s.k = p->k;
        s.device = p->device;
        s.stream = p->stream;
        s.engine = p->engine;
        s.best = pvc ? p->k : greedy.size;
        if (!pvc && p->initial_best && p->initial_best < s.best) s.best = p->initial_best;
        vcg::Frontier f;
        if (g.n == 0) {
            f.nodes = 1;
            f.found = pvc;
            f.best = s.best;
        } else {
            vcg::expand_frontier(g, s, std::max<uint64_t>(target, 1), f);
        }
        out->num_seeds = f.count;
        if (f.count) {
            out->seeds = static_cast<uint32_t*>(std::malloc(f.records.size() * 4));
            std::memcpy(out->seeds, f.records.data(), f.records.size() * 4);
        }
        out->nodes_visited = f.nodes;
        out->levels = f.levels;
        out->best = f.best;
        out->found = f.found ? 1 : 0;
        out->kernel_launches = f.launches;
        const std::vector<uint32_t>& cov = f.found ? f.cover : greedy.cover;
        if (!(pvc && !f.found)) {
            // verify_cover (bounds.cpp:32-45) on the certificate handed back
            if (!vcg::verify_cover(g, cov.data(), cov.size()) || (pvc && cov.size() > p->k))
                return fail(VCG_EVERIFY, "frontier expansion returned an invalid cover");
            out->cover_len = (uint32_t)cov.size();
            out->cover = static_cast<uint32_t*>(std::malloc(std::max<size_t>(1, cov.size()) * 4));
            for (size_t i = 0; i < cov.size(); ++i) out->cover[i] = cov[i] + g.id_base;
        }
        return VCG_OK;
    });
}

void vcg_frontier_free(vcg_frontier* f) {
    if (!f) return;
    std::free(f->seeds);
    std::free(f->cover);
    f->seeds = nullptr;
    f->cover = nullptr;
}

int vcg_mailbox_alloc(uint32_t n_words, uint32_t** out) {
    return guarded([&]() -> int {
        if (!out || n_words < 4) return fail(VCG_EINVAL, "mailbox needs >= 4 words");
        *out = vcg::mailbox_alloc(n_words);
        return VCG_OK;
    });
}

void vcg_mailbox_free(uint32_t* p) { vcg::mailbox_free(p); }

void vcg_result_free(vcg_result* r) {
    if (!r) return;
    std::free(r->cover);
    std::free(r->worker_nodes);
    std::free(r->worker_stack_high_water);
    r->cover = nullptr;
    r->worker_nodes = nullptr;
    r->worker_stack_high_water = nullptr;
}

}  // extern "C"
