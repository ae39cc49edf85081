// Engine interface between the C-ABI (capi.cpp) and the CUDA side (dense_engine.cu).
#pragma once

#include <cstdint>
#include <functional>
#include <string>
#include <vector>

#include "host_graph.hpp"

namespace vcg {

struct SolveSpec {
    bool pvc = false;
    uint32_t k = 0;
    int strategy = 0;           // 0 hybrid, 1 seq, 2 stackonly
    uint32_t workers = 0;       // 0 = fill the device
    uint64_t capacity = 4096;
    uint64_t threshold = 2048;  // worklist_threshold (scheduler.cpp:14-18), computed on host
    uint32_t depth = 8;
    uint64_t backoff_us = 50;
    double timeout_s = -1.0;
    uint64_t node_budget = 0;
    int device = 0;
    int rules = 0;              // 0 reference order, 1 parallel
    uint32_t block_warps = 0;
    int engine = 0;
    bool instrument = false;
    bool donate_oldest = false;
    uint32_t best = 0;          // initial bound: greedy size (MVC, or tighter external) / k (PVC)
    uint32_t stack_bound = 0;   // stack_bound_for (scheduler.cpp:118-121)
    const uint32_t* seeds = nullptr;  // [cc, edges, deg[n]] records
    uint64_t num_seeds = 0;
    volatile uint32_t* mailbox = nullptr;
    void* stream = nullptr;     // caller's cudaStream_t (null: the library's stream)
    bool no_root = false;       // multi-shard: no seeds means an empty worklist, not the root
    uint32_t stack_cap = 0;     // debug (VCG_DEBUG_SMALL_STACK): cap the sparse local stack
};

struct SolveOut {
    int status = 0;             // 0 complete, 1 timeout, 2 budget
    bool found = false;         // a search cover was recorded (MVC: improved; PVC: yes)
    uint32_t found_size = 0;
    std::vector<uint32_t> cover;  // internal ids of the recorded cover
    std::vector<uint64_t> worker_nodes, worker_high_water;
    uint64_t wl_added = 0, wl_removed = 0, wl_max_size = 0, wl_current = 0;
    uint64_t rounds = 0, maxdeg = 0, children = 0, removals = 0, donated = 0;
    uint64_t rm1 = 0, rm2 = 0, rmh = 0, dooms = 0;
    uint64_t phase[10] = {0};
    uint64_t active_cycles = 0;
    // search timeline (dense engine): ms after the first warp started by which 10 / 50 / 90 /
    // 100% of the workers had taken their first node, and had exited
    double t_first_ms[4] = {0, 0, 0, 0}, t_end_ms[4] = {0, 0, 0, 0};
    double t_lastwait_ms[4] = {0, 0, 0, 0};  // ... and had entered their final wait (the tail)
    double idle_share = 0;  // share of the workers' time spent waiting for worklist nodes
    uint64_t donated_peer = 0;
    double device_ms = 0, h2d_ms = 0;
    uint64_t h2d_bytes = 0, d2h_bytes = 0;
    uint32_t degree_bytes = 2, n_padded = 0;
    int engine = 1;
    uint32_t grid = 0, block = 0;
    uint32_t launches = 0;
};

struct Frontier {
    uint64_t count = 0;              // frontier nodes
    std::vector<uint32_t> records;   // count x [cc, edges, deg[n]]
    uint64_t nodes = 0;              // nodes visited (processed) by the expansion
    uint32_t levels = 0, launches = 0;
    uint32_t best = 0;               // MVC bound after the expansion (k for PVC)
    bool found = false;              // a cover was found (PVC: yes-instance decided)
    std::vector<uint32_t> cover;     // internal ids
};

// Deterministic level-synchronous expansion of the search tree until >= target open nodes.
void expand_frontier(const Graph& g, const SolveSpec& s, uint64_t target, Frontier& f);

// Throws std::runtime_error (CUDA failures) / std::invalid_argument (bad configuration).
// while_running: host work to do while the search kernel runs (called after the launch).
void solve_on_device(const Graph& g, const SolveSpec& s, SolveOut& out,
                     const std::function<void()>& while_running = {});

// Multi-shard solves (one shard per GPU, or several on one device): each shard is a dense-engine
// run with its own worklist; linked shards donate work into each other's rings and share the
// MVC bound, the PVC found flag and termination through peer memory (NVLink P2P / CUDA IPC).
struct Session;
Session* session_open(const Graph& g, const SolveSpec& s);  // prepare: buffers + seeds
size_t session_handle_bytes();
void session_export(const Session* ses, void* handle);     // CUDA IPC handles of its exchange memory
// link to every shard's exported handles (this process owns shard `rank`)
void session_link_ipc(Session* ses, uint32_t world, uint32_t rank, const void* handles,
                      const uint64_t* seeds_per_shard);
// link shards living in this process (same or peer-accessible devices)
void session_link_local(Session* const* shards, uint32_t world);
void session_launch(Session* ses);                 // asynchronous
void session_reset(Session* ses);                  // fresh state for the next solve (kept links)
void session_wait(Session* ses, SolveOut& out);    // blocks, assembles the result
void session_close(Session* ses);
// Workers (warps) of a full-device dense solve of g: shards sharing a device split these.
uint32_t full_device_workers(const Graph& g, int dev);
int device_count();
uint32_t* mailbox_alloc(uint32_t n_words);
void mailbox_free(uint32_t* p);

}  // namespace vcg
