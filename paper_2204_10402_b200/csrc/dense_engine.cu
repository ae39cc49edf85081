// dense_engine.cu — the B200 hybrid search-tree traversal for graphs of n <= 1024 vertices.
//
// Reference path replaced: run_hybrid (proj/src/scheduler.cpp:328-359) with its worker loop
// hybrid_worker (:146-212), process_node (:125-144), reduce_to_fixpoint (reductions.cpp:63-104),
// the three rule passes (reductions.cpp:7-58), should_prune (bounds.cpp:21-30),
// max_degree_vertex / remove_*_into_cover (search_node.cpp:16-46) and GlobalWorklist
// (worklist.cpp:11-48). solve_mvc_seq/solve_pvc_seq (solver_seq.cpp:56-159) are the 1-worker,
// no-donation special case.
//
// Design:
//  * one WARP = one worker. The current search node lives in REGISTERS: lane l holds the
//    degrees of vertices 32*i + l, i < W (W = ceil(n/32) rounded up to 4/8/16/32), as u32
//    with kRemoved = 0xFFFFFFFF. Warp-wide ballots scan 32 vertices per instruction;
//    __reduce_max_sync gives the smallest-id max-degree vertex in one REDUX.
//  * the read-only graph is a W x n adjacency bitmap staged ONCE per CTA in shared memory
//    (uint4 groups of 4 row-words per vertex, column-coalesced). It replaces the CSR walks:
//    removing v decrements the degree of every alive neighbour from one broadcast row load;
//    removing N(v) (the deferred child) recomputes the surviving degrees as
//    d'(w) = d(w) - popc(A[w] & N_alive(v)) — W^2/4 conflict-free LDS.128 instead of
//    sum_{u in N(v)} deg(u) scattered decrements.
//  * rules run in the reference's sequential ascending order with "find next candidate at or
//    after pos" ballots, which reproduces the reference reduced node bit for bit (so PVC
//    no-instance node counts equal the reference's, and 1-worker MVC visits the same nodes).
//  * deferred children go to a per-warp stack in HBM (lane-major u16 records, L2-resident top)
//    or, while the global worklist is below its threshold, to a lock-free device ring queue
//    (ticket counters + per-slot sequence numbers, no mutex). Termination: a single `pending`
//    counter of queued items + active workers; done when it reaches zero.
//  * MVC bound: atomicMin on a device word, re-read once per node; certificate = per-worker
//    cover bitmap + a packed (size, worker) atomicMin. PVC: first finder raises `found`/`cancel`.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <tuple>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "dense_kernels.cuh"
#include "sparse_kernels.cuh"
#include "engine.hpp"

namespace vcg {

#define CUDA_CHECK(x)                                                                       \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess)                                                              \
            throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                     " at " #x);                                            \
    } while (0)

// ------------------------------------------------------------------ host side

struct DeviceGraph {
    int device = -1;
    uint32_t W = 0, npad = 0;
    uint4* at4 = nullptr;       // dense engine: adjacency bitmap
    size_t at4_bytes = 0;
    uint32_t* off = nullptr;    // sparse engine: CSR with u32 offsets
    uint32_t* nbr = nullptr;
    size_t csr_bytes = 0;
    ~DeviceGraph() {
        if (at4) cudaFree(at4);
        if (off) cudaFree(off);
        if (nbr) cudaFree(nbr);
    }
};

namespace {

// A grow-only per-device arena so repeated solves do not pay cudaMalloc each time.
struct Arena {
    void* p = nullptr;
    size_t bytes = 0;
    void* get(size_t need) {
        if (need > bytes) {
            if (p) CUDA_CHECK(cudaFree(p));
            p = nullptr;
            CUDA_CHECK(cudaMalloc(&p, need));
            bytes = need;
        }
        return p;
    }
};
// Grow-only pinned host staging for the end-of-solve readback (one async copy, no pageable
// bounce through the driver).
struct PinnedArena {
    void* p = nullptr;
    size_t bytes = 0;
    void* get(size_t need) {
        if (need > bytes) {
            if (p) CUDA_CHECK(cudaFreeHost(p));
            p = nullptr;
            CUDA_CHECK(cudaHostAlloc(&p, need, cudaHostAllocDefault));
            bytes = need;
        }
        return p;
    }
};
struct DeviceCtx {
    Arena stacks, wl, seq, misc, scratch, gdeg;
    PinnedArena host, seedbuf;
    cudaStream_t stream = nullptr;
    cudaEvent_t evh = nullptr, ev0 = nullptr, ev1 = nullptr;
    int sms = 0;
    // One solve at a time per device: the arenas, events and the graph's lazily built device
    // copy are shared state (the reference harness is synchronous too).
    std::mutex solve_mu;
};
std::mutex g_ctx_mu;
std::vector<std::unique_ptr<DeviceCtx>> g_ctx;

DeviceCtx& ctx_for(int dev) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    if ((int)g_ctx.size() <= dev) g_ctx.resize(dev + 1);
    if (!g_ctx[dev]) {
        auto c = std::make_unique<DeviceCtx>();
        CUDA_CHECK(cudaSetDevice(dev));
        CUDA_CHECK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
        CUDA_CHECK(cudaEventCreate(&c->evh));
        CUDA_CHECK(cudaEventCreate(&c->ev0));
        CUDA_CHECK(cudaEventCreate(&c->ev1));
        CUDA_CHECK(cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, dev));
        g_ctx[dev] = std::move(c);
    }
    return *g_ctx[dev];
}

__global__ void init_seq_kernel(unsigned long long* seq, uint32_t ring, uint32_t filled) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ring; i += gridDim.x * blockDim.x)
        seq[i] = i < filled ? i + 1ull : (unsigned long long)i;
}

// dst[j] = src[idx[j]] for node records of `vec16` 16-byte vectors (frontier compaction)
__global__ void gather_records_kernel(const unsigned char* src, const uint32_t* idx,
                                      unsigned char* dst, uint32_t count, uint32_t vec16) {
    for (uint32_t j = blockIdx.x; j < count; j += gridDim.x) {
        const uint4* s4 = reinterpret_cast<const uint4*>(src) + (size_t)idx[j] * vec16;
        uint4* d4 = reinterpret_cast<uint4*>(dst) + (size_t)j * vec16;
        for (uint32_t t = threadIdx.x; t < vec16; t += blockDim.x) d4[t] = s4[t];
    }
}

// Dynamic shared memory of the dense kernels (dense_scratch_base / dense_degree_base): the
// adjacency bitmap, a W-word slot per warp, W x 32 scratch words per warp, and with
// VCG_WIDE_SMEM the wide degrees (W x 32 words per warp, laid out after 8 warps of scratch).
size_t dense_smem_bytes(uint32_t W, uint32_t warps, int MW = -1, uint32_t BW = 8) {
    if (MW < 0) MW = default_mid((int)W);
    const size_t npad = 32 * (size_t)W;
    const size_t base = W * npad * 4 + BW * (size_t)W * 4;
    return VCG_WIDE_SMEM ? base + BW * (size_t)W * 32 * 4 + warps * (size_t)dense_degree_words(W, MW) * 4
                         : base + warps * (size_t)W * 32 * 4;
}

// One large CTA per SM for the W = 16 search kernels (the graph bitmap stored once per SM frees
// shared memory and the register file for more warps): warps per CTA for the dense-graph
// kernel (no mid layout), the 256-slot and the 128-slot mid kernels (8 = the 8-warp CTAs,
// several per SM; 0 = the same for the first two).
#ifndef VCG_BIG_CTA_DENSE
#define VCG_BIG_CTA_DENSE 28
#endif
#ifndef VCG_BIG_CTA_MID8
#define VCG_BIG_CTA_MID8 19
#endif
#ifndef VCG_BIG_CTA_MID4
#define VCG_BIG_CTA_MID4 28
#endif
#ifndef VCG_BIG_CTA_MULTI
#define VCG_BIG_CTA_MULTI 28  // the linked-shard kernel (sessions); 8 = 8-warp CTAs
#endif

#ifndef VCG_BACKOFF_CAP_NS
#define VCG_BACKOFF_CAP_NS 2000  // idle workers' exponential back-off cap
#endif
#ifndef VCG_FLUSH_EVERY
#define VCG_FLUSH_EVERY 64  // visits between a worker's node-counter flushes / limit checks
#endif

// sparse engine CTA shape: threads per CTA (one search node each), CTAs per SM at most, and
// the fewest shared-memory-node CTAs per SM worth keeping the node in shared memory (C4,
// budget 100k: 1024 x 1 3.6 M rule rounds/s, 256 x 4 3.9 M, 128 x 8 9.1 M)
#ifndef VCG_SPARSE_THREADS
#define VCG_SPARSE_THREADS 128
#endif
constexpr uint32_t kSparseThreads = VCG_SPARSE_THREADS;
#ifndef VCG_SPARSE_MAX_CTAS
#define VCG_SPARSE_MAX_CTAS 8
#endif
constexpr uint32_t kSparseMaxCtas = VCG_SPARSE_MAX_CTAS, kSparseMinCtas = VCG_SPARSE_MAX_CTAS < 4 ? VCG_SPARSE_MAX_CTAS : 4;

// average degree below which a W = 16 graph runs the <= 256-alive mid layout
constexpr double kMid8MaxAvgDegree = 24.0;
// edge density above which a W = 16 graph runs without the mid layout
constexpr double kMidOutOfLineDensity = 0.4;

uint32_t pick_w(uint32_t n) {
    if (n <= 128) return 4;
    if (n <= 256) return 8;
    if (n <= 512) return 16;
    return 32;
}

// Host image of the adjacency bitmap in the engine's layout: group q (words 4q..4q+3) of
// vertex w at uint4 index q*npad + w.
std::vector<uint32_t> build_bitmap(const Graph& g, uint32_t W, uint32_t npad) {
    std::vector<uint32_t> at((size_t)W * npad, 0);
    for (uint32_t w = 0; w < g.n; ++w)
        for (uint64_t e = g.off[w]; e < g.off[w + 1]; ++e) {
            uint32_t u = g.nbr[e];
            uint32_t j = u >> 5;
            at[((size_t)(j >> 2) * npad + w) * 4 + (j & 3)] |= 1u << (u & 31);
        }
    return at;
}

// Node record: the larger of the wide layout ([cc, edges, kind, 0] + lane-major u16 degrees
// (2W bytes per lane) + one word per lane of cached degree-two non-triangle verdicts) and the
// compact layout (CompactNode).
size_t dense_record_bytes(uint32_t W) {
    return std::max<size_t>(16 + 64 * (size_t)W + 128, kCompactRecordBytes);
}

// Pack one node record.
void pack_record(uint32_t W, uint32_t n, uint32_t cc, uint32_t edges, const uint32_t* deg,
                 unsigned char* rec) {
    std::memset(rec, 0, dense_record_bytes(W));  // no cached verdicts (nt = 0)
    uint32_t* h = reinterpret_cast<uint32_t*>(rec);
    h[0] = cc;
    h[1] = edges;
    uint16_t* dd = reinterpret_cast<uint16_t*>(rec + 16);
    for (uint32_t lane = 0; lane < 32; ++lane)
        for (uint32_t i = 0; i < W; ++i) {
            uint32_t v = 32 * i + lane;
            uint32_t x = v < n ? deg[v] : REM;
            dd[lane * W + i] = x == REM ? 0xFFFF : uint16_t(x);
        }
}

// Per-process caches of the kernels' shared-memory attribute and occupancy (the CUDA calls cost
// tens of microseconds on the host path of every solve otherwise).
std::mutex g_launch_mu;
std::map<std::tuple<int, const void*, size_t>, bool> g_smem_set;
std::map<std::tuple<int, const void*, uint32_t, size_t>, int> g_occupancy;
int current_device() {
    int d = 0;
    CUDA_CHECK(cudaGetDevice(&d));
    return d;
}
void set_smem_once(const void* k, size_t smem) {
    const auto key = std::make_tuple(current_device(), k, smem);
    std::lock_guard<std::mutex> lk(g_launch_mu);
    if (g_smem_set.count(key)) return;
    CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    g_smem_set[key] = true;
}

#ifndef VCG_MULTI_MOOL
#define VCG_MULTI_MOOL false  // the linked-shard kernel with the mid reduction out of line
#endif
// Instantiations: (instrumented | plain) single-shard kernels, plus the plain multi-shard one;
// W = 16 also with the wider mid layout (MW = 8, single-shard).
template <int W, bool INSTR, int MW = default_mid(W), bool MOOL = false, int BW = 8>
void launch_dense(const DenseArgs& a, uint32_t grid, uint32_t block, size_t smem, cudaStream_t s) {
    if (INSTR && a.world > 1)
        throw std::invalid_argument("instrumented runs are single-shard");
    void (*k)(DenseArgs);
    if constexpr (BW != 8) {
        k = a.world > 1 ? dense_kernel<W, false, true, false, default_mid(W), VCG_MULTI_MOOL, BW>
                        : dense_kernel<W, INSTR, false, false, MW, MOOL, BW>;  // (hybrid only)
    } else {
        k = a.world > 1 ? dense_kernel<W, false, true, false, default_mid(W), VCG_MULTI_MOOL>
            : (a.seq_mode || a.stackonly) ? dense_kernel<W, INSTR, false, true, MW, MOOL>
                                           : dense_kernel<W, INSTR, false, false, MW, MOOL>;
    }
    set_smem_once(reinterpret_cast<const void*>(k), smem);
    k<<<grid, block, smem, s>>>(a);
    CUDA_CHECK(cudaGetLastError());
}

template <int W, int MW = default_mid(W), bool MOOL = false, int BW = 8>
int occupancy(uint32_t block, size_t smem, bool instr, bool multi = false) {
    int nb = 0;
    auto k = multi ? dense_kernel<W, false, true, false, default_mid(W), VCG_MULTI_MOOL, BW>
                   : (instr ? dense_kernel<W, true, false, false, MW, MOOL, BW>
                            : dense_kernel<W, false, false, false, MW, MOOL, BW>);
    const auto key = std::make_tuple(current_device(), reinterpret_cast<const void*>(k), block, smem);
    {
        std::lock_guard<std::mutex> lk(g_launch_mu);
        auto it = g_occupancy.find(key);
        if (it != g_occupancy.end()) return it->second;
    }
    set_smem_once(reinterpret_cast<const void*>(k), smem);
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, (int)block, smem));
    std::lock_guard<std::mutex> lk(g_launch_mu);
    g_occupancy[key] = nb;
    return nb;
}

// Kernel done → control block + per-worker stats into pinned memory with one stream sync;
// device_ms from the kernel's events, h2d_ms from the upload's.
const WStats* finish_and_read(DeviceCtx& C, cudaStream_t st, const Ctl* ctl, const WStats* stats,
                              uint32_t workers, Ctl& hc, SolveOut& out) {
    CUDA_CHECK(cudaEventRecord(C.ev1, st));
    const size_t sb = (size_t)workers * sizeof(WStats);
    constexpr size_t kStatsAt = (sizeof(Ctl) + 255) / 256 * 256;
    unsigned char* h = static_cast<unsigned char*>(C.host.get(kStatsAt + sb));
    CUDA_CHECK(cudaMemcpyAsync(h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaMemcpyAsync(h + kStatsAt, stats, sb, cudaMemcpyDeviceToHost, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    float ms = 0;
    CUDA_CHECK(cudaEventElapsedTime(&ms, C.ev0, C.ev1));
    out.device_ms = ms;
    CUDA_CHECK(cudaEventElapsedTime(&ms, C.evh, C.ev0));
    out.h2d_ms = ms;
    std::memcpy(&hc, h, sizeof(Ctl));
    out.d2h_bytes += sizeof(Ctl) + sb;
    return reinterpret_cast<const WStats*>(h + kStatsAt);
}

// Per-worker counters → the run totals (WorkerMetrics, metrics.hpp:28-41).
void aggregate(const WStats* hs, uint32_t workers, SolveOut& out) {
    out.worker_nodes.resize(workers);
    out.worker_high_water.resize(workers);
    for (uint32_t w = 0; w < workers; ++w) {
        out.worker_nodes[w] = hs[w].nodes;
        out.worker_high_water[w] = hs[w].high_water;
        out.rounds += hs[w].rounds;
        out.maxdeg += hs[w].maxdeg;
        out.children += hs[w].children;
        out.removals += hs[w].rm1 + hs[w].rm2 + hs[w].rmh;
        out.rm1 += hs[w].rm1;
        out.rm2 += hs[w].rm2;
        out.rmh += hs[w].rmh;
        out.dooms += hs[w].dooms;
        out.donated += hs[w].donated;
        out.active_cycles += hs[w].active;
        out.donated_peer += hs[w].peer;
        out.wl_max_size = std::max<uint64_t>(out.wl_max_size, hs[w].max_queue);
        for (int p = 0; p < 10; ++p) out.phase[p] += hs[w].phase[p];
    }
    // timeline percentiles (workers that never took a node count as never starting)
    unsigned long long t0 = ~0ull;
    for (uint32_t w = 0; w < workers; ++w)
        if (hs[w].t_begin) t0 = std::min(t0, hs[w].t_begin);
    if (t0 == ~0ull) return;
    // (on the host's critical path between solves: reused buffers and O(n) selections)
    thread_local std::vector<double> tf, te, tw;
    tf.clear();
    te.clear();
    tw.clear();
    double idle = 0, span = 0;
    for (uint32_t w = 0; w < workers; ++w) {
        if (hs[w].t_end > hs[w].t_begin) {
            span += (double)(hs[w].t_end - hs[w].t_begin);
            idle += (double)hs[w].t_idle;
        }
        if (hs[w].t_first) tf.push_back((hs[w].t_first - t0) * 1e-6);
        if (hs[w].t_end) te.push_back((hs[w].t_end - t0) * 1e-6);
        if (hs[w].t_lastwait) tw.push_back((hs[w].t_lastwait - t0) * 1e-6);
    }
    auto pct = [](std::vector<double>& v, double* o, size_t total) {
        const double q[4] = {0.1, 0.5, 0.9, 1.0};
        size_t lo = 0;  // quantiles ascending: each selection works on the part above the last
        for (int i = 0; i < 4; ++i) {
            const size_t k = (size_t)std::ceil(q[i] * total);
            if (k == 0) {
                o[i] = 0.0;
            } else if (k > v.size()) {
                o[i] = -1.0;  // never reached
            } else {
                std::nth_element(v.begin() + lo, v.begin() + (k - 1), v.end());
                o[i] = v[k - 1];
                lo = k - 1;
            }
        }
    };
    pct(tf, out.t_first_ms, workers);
    pct(te, out.t_end_ms, workers);
    pct(tw, out.t_lastwait_ms, workers);
    out.idle_share = span > 0 ? idle / span : 0.0;
}

}  // namespace

uint32_t* mailbox_alloc(uint32_t n_words) {
    void* p = nullptr;
    CUDA_CHECK(cudaHostAlloc(&p, n_words * sizeof(uint32_t), cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(p, 0, n_words * sizeof(uint32_t));
    return static_cast<uint32_t*>(p);
}

void mailbox_free(uint32_t* p) {
    if (p) cudaFreeHost(p);
}

int device_count() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

static void solve_sparse(const Graph& g, const SolveSpec& s, SolveOut& out);

namespace {
// The adjacency bitmap of `g` on `dev`, uploaded once per device (the caller holds the device's
// solve lock).
const DeviceGraph& device_graph(const Graph& g, int dev, cudaStream_t st, SolveOut* out) {
    if ((int)g.dev.size() <= dev) g.dev.resize(dev + 1);
    if (!g.dev[dev]) {
        const uint32_t W = pick_w(g.n);
        auto dg = std::make_shared<DeviceGraph>();
        dg->device = dev;
        dg->W = W;
        dg->npad = 32 * W;
        std::vector<uint32_t> at = build_bitmap(g, W, dg->npad);
        dg->at4_bytes = at.size() * 4;
        CUDA_CHECK(cudaMalloc(&dg->at4, dg->at4_bytes));
        CUDA_CHECK(cudaMemcpyAsync(dg->at4, at.data(), dg->at4_bytes, cudaMemcpyHostToDevice, st));
        // (a pageable source is staged before cudaMemcpyAsync returns: `at` may go)
        if (out) out->h2d_bytes += dg->at4_bytes;
        g.dev[dev] = dg;
    }
    return *g.dev[dev];
}

}  // namespace

// One dense-engine solve on one device: prepare (buffers, seeds, kernel arguments), launch, and
// finish (result assembly). vcg_solve runs the three back to back on the device's reusable
// arenas under its solve lock; a multi-shard session owns its buffers, links its kernel to the
// peers' exchange memory between prepare and launch, and launches every shard before any waits.
struct DenseRun {
    const Graph& g;
    SolveSpec s;
    int dev;
    DeviceCtx& C;
    cudaStream_t st = nullptr;
    bool owned;  // own buffers and events (session) instead of the device arenas
    bool mid8 = false;  // W = 16 kernel with the <= 256-alive mid layout
    bool mool = false;  // W = 16 kernel without the mid layout (dense graphs)
    bool big = false;   // one large CTA per SM (VCG_BIG_CTA_*)
    std::vector<void*> allocs;
    void* host = nullptr;
    size_t host_bytes = 0;
    void* hseed_p = nullptr;
    size_t hseed_bytes = 0;
    cudaEvent_t evh = nullptr, ev0 = nullptr, ev1 = nullptr;
    std::vector<void*> ipc_opened;
    PeerRef* peers_dev = nullptr;
    uint32_t W = 0, npad = 0, block_warps = 0, block = 0, grid = 0, workers = 0, bound = 0;
    size_t entry = 0, smem = 0, wl_bytes = 0, seq_bytes = 0, misc_bytes = 0;
    uint64_t ring = 0, cap = 0, nseeds = 0;
    unsigned char *stacks = nullptr, *wl = nullptr, *misc = nullptr;
    unsigned long long* seq = nullptr;
    Ctl* ctl = nullptr;
    uint32_t* cover_slots = nullptr;
    WStats* stats = nullptr;
    DenseArgs a{};
    Ctl hc{};
    SolveOut out;

    DenseRun(const Graph& g_, const SolveSpec& s_, bool owned_)
        : g(g_), s(s_), dev(s_.device), C(ctx_for(s_.device)), owned(owned_) {}
    ~DenseRun() {
        cudaSetDevice(dev);
        for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
        if (peers_dev) cudaFree(peers_dev);
        for (void* p : allocs) cudaFree(p);
        if (host) cudaFreeHost(host);
        if (hseed_p) cudaFreeHost(hseed_p);
        if (owned) {
            if (evh) cudaEventDestroy(evh);
            if (ev0) cudaEventDestroy(ev0);
            if (ev1) cudaEventDestroy(ev1);
            if (st) cudaStreamDestroy(st);
        }
    }
    void* dalloc(Arena& arena, size_t bytes) {
        if (!owned) return arena.get(bytes);
        void* p = nullptr;
        CUDA_CHECK(cudaMalloc(&p, std::max<size_t>(bytes, 256)));
        allocs.push_back(p);
        return p;
    }
    // pinned staging of the initial control block and records (pageable copies would block)
    void* hseed(size_t bytes) {
        if (!owned) return C.seedbuf.get(bytes);
        if (bytes > hseed_bytes) {
            if (hseed_p) CUDA_CHECK(cudaFreeHost(hseed_p));
            hseed_p = nullptr;
            CUDA_CHECK(cudaHostAlloc(&hseed_p, bytes, cudaHostAllocDefault));
            hseed_bytes = bytes;
        }
        return hseed_p;
    }
    void* halloc(size_t bytes) {
        if (!owned) return C.host.get(bytes);
        if (bytes > host_bytes) {
            if (host) CUDA_CHECK(cudaFreeHost(host));
            host = nullptr;
            CUDA_CHECK(cudaHostAlloc(&host, bytes, cudaHostAllocDefault));
            host_bytes = bytes;
        }
        return host;
    }

    void prepare() {
        CUDA_CHECK(cudaSetDevice(dev));
        if (owned) {
            CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            CUDA_CHECK(cudaEventCreate(&evh));
            CUDA_CHECK(cudaEventCreate(&ev0));
            CUDA_CHECK(cudaEventCreate(&ev1));
        } else {
            st = s.stream ? static_cast<cudaStream_t>(s.stream) : C.stream;
            evh = C.evh;
            ev0 = C.ev0;
            ev1 = C.ev1;
        }
        W = pick_w(g.n);
        npad = 32 * W;
        entry = dense_record_bytes(W);
        out.engine = 1;
        out.degree_bytes = 2;
        out.n_padded = npad;

        CUDA_CHECK(cudaEventRecord(evh, st));
        const DeviceGraph* dgp;
        if (owned) {
            std::lock_guard<std::mutex> lk(C.solve_mu);  // (the lazily built device graph)
            dgp = &device_graph(g, dev, st, &out);
        } else {
            dgp = &device_graph(g, dev, st, &out);
        }
        const DeviceGraph& dg = *dgp;

        // worker grid: one warp per worker
        // The wider mid layout (<= 256 alive, 8 KB frames) for sparse graphs, whose nodes keep a
        // few hundred vertices alive (C2: 160-255); engine 5 forces it.
        mid8 = W == 16 && !owned && s.engine != 3 && s.engine != 4 && s.engine != 6 &&
               (s.engine == 5 || 2.0 * (double)g.m < kMid8MaxAvgDegree * (double)g.n);
        // dense graphs (C5, C3: nearly every visit compact) run without the mid layout: its code
        // only costs them instruction cache (C5: 1.3% of visits would be mid)
        mool = W == 16 && !owned && !mid8 && s.engine != 6 &&
               (s.engine == 4 || 2.0 * (double)g.m > kMidOutOfLineDensity * (double)g.n * (double)(g.n - 1));
        // one large CTA per SM for the hybrid single-shard kernels of those two classes
        const uint32_t big_warps = W != 16 ? 0u : owned ? VCG_BIG_CTA_MULTI
                                   : mid8 ? VCG_BIG_CTA_MID8 : mool ? VCG_BIG_CTA_DENSE : VCG_BIG_CTA_MID4;
        big = big_warps > 0 && !s.block_warps && s.strategy == 0;
        const uint32_t cta_warps = big ? big_warps : 8;
        block_warps = s.block_warps ? std::min<uint32_t>(s.block_warps, 8) : cta_warps;
        block = 32 * block_warps;
        // bitmap + per-warp slot (W words) + per-warp scratch and degree / frame words
        smem = dense_smem_bytes(W, block_warps, mid8 ? 8 : (mool ? 0 : -1), big ? block_warps : 8);
        int per_sm = 1;
        switch (W) {
            case 4: per_sm = occupancy<4>(block, smem, s.instrument, owned); break;
            case 8: per_sm = occupancy<8>(block, smem, s.instrument, owned); break;
            case 16:
                per_sm = big ? (owned ? occupancy<16, 4, false, VCG_BIG_CTA_MULTI>(block, smem, false, true)
                                : mid8 ? occupancy<16, 8, false, VCG_BIG_CTA_MID8>(block, smem, s.instrument, owned)
                                : mool ? occupancy<16, 0, false, VCG_BIG_CTA_DENSE>(block, smem, s.instrument, owned)
                                       : occupancy<16, 4, false, VCG_BIG_CTA_MID4>(block, smem, s.instrument, owned))
                             : mid8 ? occupancy<16, 8>(block, smem, s.instrument, owned)
                             : mool ? occupancy<16, 0>(block, smem, s.instrument, owned)
                                    : occupancy<16>(block, smem, s.instrument, owned);
                break;
            default: per_sm = occupancy<32>(block, smem, s.instrument, owned); break;
        }
        if (per_sm < 1) throw std::runtime_error("CUDA error: dense kernel cannot be resident");
        workers = s.workers;
        if (s.strategy == 1) workers = 1;
        if (workers == 0) workers = (uint32_t)C.sms * per_sm * block_warps;
        grid = (workers + block_warps - 1) / block_warps;
        out.grid = grid;
        out.block = block;

        // memory: stacks, worklist ring, control, cover slots, stats
        bound = std::max<uint32_t>(s.stack_bound, 1) + 1;
        cap = std::max<uint64_t>(std::max<uint64_t>(s.capacity, s.num_seeds), 1);
        if (cap > (1ull << 30)) throw std::invalid_argument("worklist capacity too large");
        ring = 2;
        while (ring < cap) ring <<= 1;
        const size_t stack_bytes = (size_t)workers * bound * entry;
        wl_bytes = (size_t)ring * entry;
        seq_bytes = ring * 8;
        stacks = (unsigned char*)dalloc(C.stacks, stack_bytes);
        wl = (unsigned char*)dalloc(C.wl, wl_bytes);
        seq = (unsigned long long*)dalloc(C.seq, seq_bytes);
        const size_t slots_bytes = (((size_t)workers * W * 4) + 255) / 256 * 256;
        misc_bytes = sizeof(Ctl) + slots_bytes + (size_t)workers * sizeof(WStats);
        misc = (unsigned char*)dalloc(C.misc, misc_bytes);
        ctl = reinterpret_cast<Ctl*>(misc);
        cover_slots = reinterpret_cast<uint32_t*>(misc + sizeof(Ctl));
        stats = reinterpret_cast<WStats*>(misc + sizeof(Ctl) + slots_bytes);

        seed();
        a = DenseArgs{};
        a.at4 = dg.at4;
        a.n = g.n;
        a.npad = npad;
        a.m = (uint32_t)g.m;
        a.pvc = s.pvc ? 1 : 0;
        a.k = s.k;
        a.capacity = (uint32_t)cap;
        a.ring_mask = (uint32_t)(ring - 1);
        a.threshold = (uint32_t)std::min<uint64_t>(s.threshold, cap);
        a.workers = workers;
        a.stack_bound = bound;
        a.entry_bytes = entry;
        a.stacks = stacks;
        a.wl = wl;
        a.seq = seq;
        a.ctl = ctl;
        a.cover_slots = cover_slots;
        a.stats = stats;
        a.node_budget = s.node_budget;
        a.timeout_ns = s.timeout_s >= 0 ? (unsigned long long)(s.timeout_s * 1e9) : 0ull;
        if (s.timeout_s >= 0 && a.timeout_ns == 0) a.timeout_ns = 1;
        a.flush_every = VCG_FLUSH_EVERY;
        if (s.node_budget)
            a.flush_every = std::max<uint64_t>(1, std::min<uint64_t>(64, s.node_budget / (4ull * workers)));
        // idle back-off: exponential from 32 ns, capped at backoff_us (at most 2 us on the device —
        // a polling warp costs one L2 read, an over-sleeping one leaves queued work unclaimed)
        a.backoff_ns = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(s.backoff_us * 1000, 64), VCG_BACKOFF_CAP_NS);
        a.seq_mode = s.strategy != 0 ? 1 : 0;  // seq and stackonly never donate
        a.donate_oldest = s.donate_oldest ? 1 : 0;
        a.compact = s.engine == 3 ? 0 : 1;
        a.mid = (s.engine == 3 || s.engine == 4) ? 0 : 1;
        a.stackonly = s.strategy == 2 ? 1 : 0;
        a.depth = s.depth;
        a.mailbox = s.mailbox;
        a.peers = nullptr;
        a.world = 1;
        a.rank = 0;
    }

    // The initial worklist and control state: the root (init_root, search_node.cpp:7-14), the
    // seeds, or nothing (a shard with an empty share). Run again by reset() for the next solve
    // of a persistent multi-shard session (buffers and peer mappings kept).
    void seed() {
        nseeds = s.num_seeds ? s.num_seeds : (s.no_root ? 0 : 1);
        // staging: [control block | records], pinned (the stream is idle until the copies land)
        constexpr size_t kRecsAt = (sizeof(Ctl) + 255) / 256 * 256;
        unsigned char* stage = static_cast<unsigned char*>(hseed(kRecsAt + nseeds * entry));
        unsigned char* recs = stage + kRecsAt;
        const size_t recs_bytes = nseeds * entry;
        if (s.num_seeds) {
            for (uint64_t i = 0; i < nseeds; ++i) {
                const uint32_t* r = s.seeds + i * (2 + (size_t)g.n);
                pack_record(W, g.n, r[0], r[1], r + 2, recs + i * entry);
            }
        } else if (nseeds) {
            std::vector<uint32_t> deg(g.n);
            for (uint32_t v = 0; v < g.n; ++v) deg[v] = g.degree(v);
            pack_record(W, g.n, 0, (uint32_t)g.m, deg.data(), recs);
        }
        std::memset(&hc, 0, sizeof(hc));
        hc.best = s.best;
        hc.head = 0;
        hc.tail = nseeds;
        hc.work = (nseeds << 32) | nseeds;
        hc.best_owner = ~0ull;
        hc.gactive = active_;  // (read from shard 0's copy only)
        std::memcpy(stage, &hc, sizeof(hc));
        CUDA_CHECK(cudaMemcpyAsync(ctl, stage, sizeof(hc), cudaMemcpyHostToDevice, st));
        if (nseeds)
            CUDA_CHECK(cudaMemcpyAsync(wl, recs, recs_bytes, cudaMemcpyHostToDevice, st));
        init_seq_kernel<<<64, 256, 0, st>>>(seq, (uint32_t)ring, (uint32_t)nseeds);
        CUDA_CHECK(cudaGetLastError());
        out.launches += 2;  // init_seq_kernel + dense_kernel
        CUDA_CHECK(cudaMemsetAsync(stats, 0, (size_t)workers * sizeof(WStats), st));
        out.h2d_bytes += sizeof(hc) + recs_bytes;
        if (owned) CUDA_CHECK(cudaStreamSynchronize(st));  // (peers may map it before launch)
    }
    uint32_t active_ = 0;  // multi-shard: shards with initial work (shard 0's gactive)

    // Next solve of a persistent session: the same graph and parameters, fresh state.
    void reset() {
        CUDA_CHECK(cudaSetDevice(dev));
        out = SolveOut();
        out.engine = 1;
        out.degree_bytes = 2;
        out.n_padded = npad;
        out.grid = grid;
        out.block = block;
        CUDA_CHECK(cudaEventRecord(evh, st));
        seed();
    }

    // Multi-shard: every shard's exchange memory (this one's included, at `rank`).
    void link(uint32_t world, uint32_t rank, const std::vector<PeerRef>& refs, uint32_t active) {
        CUDA_CHECK(cudaSetDevice(dev));
        CUDA_CHECK(cudaMalloc(&peers_dev, world * sizeof(PeerRef)));
        CUDA_CHECK(cudaMemcpy(peers_dev, refs.data(), world * sizeof(PeerRef), cudaMemcpyHostToDevice));
        a.peers = peers_dev;
        a.world = world;
        a.rank = rank;
        active_ = active;
        if (rank == 0)  // shard 0 holds the shard-activity count
            CUDA_CHECK(cudaMemcpy(&ctl->gactive, &active, 4, cudaMemcpyHostToDevice));
    }

    void launch() {
        CUDA_CHECK(cudaSetDevice(dev));
        CUDA_CHECK(cudaEventRecord(ev0, st));
        const bool I = s.instrument;
        switch (W) {
            case 4: I ? launch_dense<4, true>(a, grid, block, smem, st) : launch_dense<4, false>(a, grid, block, smem, st); break;
            case 8: I ? launch_dense<8, true>(a, grid, block, smem, st) : launch_dense<8, false>(a, grid, block, smem, st); break;
            case 16:
                if (big && mid8) I ? launch_dense<16, true, 8, false, VCG_BIG_CTA_MID8>(a, grid, block, smem, st) : launch_dense<16, false, 8, false, VCG_BIG_CTA_MID8>(a, grid, block, smem, st);
                else if (big && mool) I ? launch_dense<16, true, 0, false, VCG_BIG_CTA_DENSE>(a, grid, block, smem, st) : launch_dense<16, false, 0, false, VCG_BIG_CTA_DENSE>(a, grid, block, smem, st);
                else if (big && owned) launch_dense<16, false, 4, false, VCG_BIG_CTA_MULTI>(a, grid, block, smem, st);
                else if (big) I ? launch_dense<16, true, 4, false, VCG_BIG_CTA_MID4>(a, grid, block, smem, st) : launch_dense<16, false, 4, false, VCG_BIG_CTA_MID4>(a, grid, block, smem, st);
                else if (mid8) I ? launch_dense<16, true, 8>(a, grid, block, smem, st) : launch_dense<16, false, 8>(a, grid, block, smem, st);
                else if (mool) I ? launch_dense<16, true, 0>(a, grid, block, smem, st) : launch_dense<16, false, 0>(a, grid, block, smem, st);
                else I ? launch_dense<16, true>(a, grid, block, smem, st) : launch_dense<16, false>(a, grid, block, smem, st);
                break;
            default: I ? launch_dense<32, true>(a, grid, block, smem, st) : launch_dense<32, false>(a, grid, block, smem, st); break;
        }
        CUDA_CHECK(cudaEventRecord(ev1, st));
    }

    // Kernel done → control block + per-worker stats into pinned memory with one stream sync;
    // device_ms from the kernel's events, h2d_ms from the upload's.
    void finish() {
        CUDA_CHECK(cudaSetDevice(dev));
        const size_t sb = (size_t)workers * sizeof(WStats);
        constexpr size_t kStatsAt = (sizeof(Ctl) + 255) / 256 * 256;
        unsigned char* h = static_cast<unsigned char*>(halloc(kStatsAt + sb));
        CUDA_CHECK(cudaMemcpyAsync(h, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaMemcpyAsync(h + kStatsAt, stats, sb, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        float ms = 0;
        CUDA_CHECK(cudaEventElapsedTime(&ms, ev0, ev1));
        out.device_ms = ms;
        CUDA_CHECK(cudaEventElapsedTime(&ms, evh, ev0));
        out.h2d_ms = ms;
        std::memcpy(&hc, h, sizeof(Ctl));
        out.d2h_bytes += sizeof(Ctl) + sb;
        const WStats* hs = reinterpret_cast<const WStats*>(h + kStatsAt);
        out.status = hc.status;
        out.wl_added = hc.tail;  // every enqueue ticket is one added node (root/seeds included)
        out.wl_current = (uint32_t)hc.work;
        out.wl_removed = hc.tail - out.wl_current;
        out.wl_max_size = nseeds;
        aggregate(hs, workers, out);
        if (s.strategy == 2) out.wl_added = out.wl_removed = out.wl_current = out.wl_max_size = 0;
        if (hc.best_owner != ~0ull) {
            const uint32_t owner = (uint32_t)(hc.best_owner & 0xFFFFFFFFu);
            out.found = true;
            out.found_size = (uint32_t)(hc.best_owner >> 32);
            std::vector<uint32_t> bits(W);
            CUDA_CHECK(cudaMemcpy(bits.data(), cover_slots + (size_t)owner * W, W * 4, cudaMemcpyDeviceToHost));
            out.d2h_bytes += W * 4;
            out.cover.clear();
            for (uint32_t v = 0; v < g.n; ++v)
                if ((bits[v >> 5] >> (v & 31)) & 1u) out.cover.push_back(v);
        }
    }
};

namespace {
void check_dense_device(const Graph& g, const SolveSpec& s) {
    if (g.n > 1024)
        throw std::invalid_argument("graph has " + std::to_string(g.n) +
                                    " vertices; the dense engine handles n <= 1024");
    int ndev = device_count();
    if (ndev == 0) throw std::runtime_error("CUDA error: no CUDA device visible");
    if (s.device < 0 || s.device >= ndev) throw std::invalid_argument("device ordinal out of range");
}
}  // namespace

void solve_on_device(const Graph& g, const SolveSpec& s, SolveOut& out,
                     const std::function<void()>& while_running) {
    if (s.engine == 2 || s.engine == 7 || (s.engine == 0 && g.n > 1024)) {
        if (while_running) while_running();
        return solve_sparse(g, s, out);
    }
    check_dense_device(g, s);
    CUDA_CHECK(cudaSetDevice(s.device));
    DeviceCtx& C = ctx_for(s.device);
    std::lock_guard<std::mutex> solve_lock(C.solve_mu);
    DenseRun r(g, s, false);
    r.out = std::move(out);
    r.prepare();
    r.launch();
    if (while_running) while_running();  // host work overlapped with the search kernel
    r.finish();
    out = std::move(r.out);
}

// ------------------------------------------------------------------ multi-shard sessions

struct Session {
    std::unique_ptr<DenseRun> run;
};

Session* session_open(const Graph& g, const SolveSpec& s) {
    if (s.engine == 2 || s.engine == 7 || g.n > 1024)
        throw std::invalid_argument("multi-shard sessions need the dense engine (n <= 1024)");
    check_dense_device(g, s);
    if (s.strategy != 0) throw std::invalid_argument("multi-shard sessions run the hybrid strategies");
    auto ses = std::make_unique<Session>();
    ses->run = std::make_unique<DenseRun>(g, s, true);
    ses->run->prepare();
    return ses.release();
}

void session_close(Session* ses) { delete ses; }

size_t session_handle_bytes() { return 3 * sizeof(cudaIpcMemHandle_t); }

void session_export(const Session* ses, void* handle) {
    const DenseRun& r = *ses->run;
    CUDA_CHECK(cudaSetDevice(r.dev));
    cudaIpcMemHandle_t* h = static_cast<cudaIpcMemHandle_t*>(handle);
    CUDA_CHECK(cudaIpcGetMemHandle(&h[0], r.misc));
    CUDA_CHECK(cudaIpcGetMemHandle(&h[1], r.wl));
    CUDA_CHECK(cudaIpcGetMemHandle(&h[2], r.seq));
}

static uint32_t shard_active(const Session* ses) { return ses->run->nseeds ? 1u : 0u; }

void session_link_ipc(Session* ses, uint32_t world, uint32_t rank, const void* handles,
                      const uint64_t* seeds_per_shard) {
    DenseRun& r = *ses->run;
    if (world < 1 || rank >= world) throw std::invalid_argument("bad shard rank / world");
    CUDA_CHECK(cudaSetDevice(r.dev));
    const cudaIpcMemHandle_t* h = static_cast<const cudaIpcMemHandle_t*>(handles);
    std::vector<PeerRef> refs(world);
    uint32_t active = 0;
    for (uint32_t p = 0; p < world; ++p) {
        active += seeds_per_shard[p] ? 1u : 0u;
        if (p == rank) {
            refs[p] = PeerRef{r.ctl, r.wl, r.seq};
            continue;
        }
        void* ptr[3];
        for (int t = 0; t < 3; ++t) {
            CUDA_CHECK(cudaIpcOpenMemHandle(&ptr[t], h[3 * p + t], cudaIpcMemLazyEnablePeerAccess));
            r.ipc_opened.push_back(ptr[t]);
        }
        refs[p] = PeerRef{static_cast<Ctl*>(ptr[0]), static_cast<unsigned char*>(ptr[1]),
                          static_cast<unsigned long long*>(ptr[2])};
    }
    r.link(world, rank, refs, active);
}

void session_link_local(Session* const* shards, uint32_t world) {
    std::vector<PeerRef> refs(world);
    uint32_t active = 0;
    for (uint32_t p = 0; p < world; ++p) {
        const DenseRun& r = *shards[p]->run;
        refs[p] = PeerRef{r.ctl, r.wl, r.seq};
        active += shard_active(shards[p]);
    }
    for (uint32_t p = 0; p < world; ++p) {
        DenseRun& r = *shards[p]->run;
        for (uint32_t q = 0; q < world; ++q) {  // shards on different devices: peer access
            const int dq = shards[q]->run->dev;
            if (dq == r.dev) continue;
            CUDA_CHECK(cudaSetDevice(r.dev));
            const cudaError_t e = cudaDeviceEnablePeerAccess(dq, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CUDA_CHECK(e);
            cudaGetLastError();
        }
        r.link(world, p, refs, active);
    }
}

void session_launch(Session* ses) { ses->run->launch(); }

void session_reset(Session* ses) { ses->run->reset(); }

uint32_t full_device_workers(const Graph& g, int dev) {
    SolveSpec s;
    s.device = dev;
    check_dense_device(g, s);
    CUDA_CHECK(cudaSetDevice(dev));
    DeviceCtx& C = ctx_for(dev);
    const uint32_t W = pick_w(g.n);
    const uint32_t bw = W == 16 ? VCG_BIG_CTA_MULTI : 8;  // (as DenseRun sizes a session)
    const uint32_t block = 32 * bw;
    const size_t smem = dense_smem_bytes(W, bw, -1, bw);
    int per_sm = 1;
    switch (W) {
        case 4: per_sm = occupancy<4>(block, smem, false, true); break;
        case 8: per_sm = occupancy<8>(block, smem, false, true); break;
        case 16: per_sm = occupancy<16, 4, false, VCG_BIG_CTA_MULTI>(block, smem, false, true); break;
        default: per_sm = occupancy<32>(block, smem, false, true); break;
    }
    return (uint32_t)C.sms * per_sm * bw;
}

void session_wait(Session* ses, SolveOut& out) {
    ses->run->finish();
    out = std::move(ses->run->out);
}

// ------------------------------------------------------------------ sparse engine host side


static void solve_sparse(const Graph& g, const SolveSpec& s, SolveOut& out) {
    const int dev = s.device;
    const int ndev = device_count();
    if (ndev == 0) throw std::runtime_error("CUDA error: no CUDA device visible");
    if (dev < 0 || dev >= ndev) throw std::invalid_argument("device ordinal out of range");
    if (2 * g.m >= (1ull << 32)) throw std::invalid_argument("graph too large for u32 CSR offsets");
    CUDA_CHECK(cudaSetDevice(dev));
    DeviceCtx& C = ctx_for(dev);
    std::lock_guard<std::mutex> solve_lock(C.solve_mu);
    cudaStream_t st = s.stream ? static_cast<cudaStream_t>(s.stream) : C.stream;

    uint32_t maxdeg = 0;
    for (uint32_t v = 0; v < g.n; ++v) maxdeg = std::max(maxdeg, g.degree(v));
    if (maxdeg >= 0xFFFFu) throw std::invalid_argument("sparse engine: degree >= 65535");
    const uint32_t npad = (g.n + 7) / 8 * 8;
    const size_t entry = 16 + 2 * (size_t)npad;
    int max_smem = 0;
    CUDA_CHECK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    // CTA shape: small CTAs (kSparseThreads, block_warps overrides), as many per SM as fit, so
    // that one node's barrier waits overlap other nodes' work. The node's degree array sits in
    // shared memory when at least kSparseMinCtas such CTAs fit, else in global memory (GDEG
    // variant, kSparseMaxCtas per SM); engine 7 forces the global one.
    int sm_smem = 0;
    CUDA_CHECK(cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
    uint32_t threads = s.block_warps ? std::min<uint32_t>(s.block_warps, 32) * 32 : kSparseThreads;
    auto ctas_for = [&](uint32_t t, size_t& node_smem) {
        node_smem = 2 * (size_t)npad + (2 * (size_t)t + 1) * 4;
        const size_t cost = node_smem + sizeof(SpShared) + 1024;  // (+ the per-CTA reserve)
        return cost <= (size_t)max_smem ? (uint32_t)std::min<size_t>(kSparseMaxCtas, sm_smem / cost) : 0u;
    };
    size_t node_smem = 0;
    uint32_t smem_ctas = ctas_for(threads, node_smem);
    const bool fits_one = smem_ctas >= 1;
    const bool gdeg = s.engine == 7 || !fits_one || (smem_ctas < kSparseMinCtas && s.engine != 2);
    if (!gdeg && smem_ctas < kSparseMinCtas && !s.block_warps) {
        threads = SP_THREADS;  // (engine 2 forced on a big node: one 1024-thread CTA per SM)
        smem_ctas = ctas_for(threads, node_smem);
    }
    const size_t list_smem = (2 * (size_t)threads + 1) * 4;
    const size_t smem = gdeg ? list_smem : node_smem;
    const uint32_t thread_ctas = std::max<uint32_t>(1, 2048 / threads);
    const uint32_t per_sm = std::max<uint32_t>(
        1, std::min<uint32_t>(gdeg ? kSparseMaxCtas : smem_ctas, thread_ctas));
    out.engine = 2;
    out.degree_bytes = 2;
    out.n_padded = npad;

    CUDA_CHECK(cudaEventRecord(C.evh, st));
    if ((int)g.dev.size() <= dev) g.dev.resize(dev + 1);
    if (!g.dev[dev] || !g.dev[dev]->off) {
        auto dg = g.dev[dev] ? g.dev[dev] : std::make_shared<DeviceGraph>();
        dg->device = dev;
        std::vector<uint32_t> off32(g.n + 1);
        for (uint32_t v = 0; v <= g.n; ++v) off32[v] = (uint32_t)g.off[v];
        CUDA_CHECK(cudaMalloc(&dg->off, off32.size() * 4));
        CUDA_CHECK(cudaMalloc(&dg->nbr, std::max<size_t>(1, g.nbr.size()) * 4));
        CUDA_CHECK(cudaMemcpyAsync(dg->off, off32.data(), off32.size() * 4, cudaMemcpyHostToDevice, st));
        if (!g.nbr.empty())
            CUDA_CHECK(cudaMemcpyAsync(dg->nbr, g.nbr.data(), g.nbr.size() * 4, cudaMemcpyHostToDevice, st));
        dg->csr_bytes = off32.size() * 4 + g.nbr.size() * 4;
        out.h2d_bytes += dg->csr_bytes;
        g.dev[dev] = dg;
    }
    const DeviceGraph& dg = *g.dev[dev];

    uint32_t workers = s.workers;
    if (s.strategy == 1) workers = 1;
    if (workers == 0) workers = (uint32_t)C.sms * per_sm;
    out.grid = workers;
    out.block = threads;

    // stack depth: the reference bound (greedy / min(k, n)), capped by device memory
    size_t free_b = 0, total_b = 0;
    CUDA_CHECK(cudaMemGetInfo(&free_b, &total_b));
    const uint64_t cap = std::max<uint64_t>(std::max<uint64_t>(s.capacity, s.num_seeds), 1);
    uint64_t ring = 2;
    while (ring < cap) ring <<= 1;
    // per worker: 10n u32 lists, n u32 counters, n u64 claims, n u32 tags
    const size_t scratch_bytes = (size_t)workers * g.n * (12 * 4 + 4 + 8 + 4);
    const size_t gdeg_bytes = gdeg ? (size_t)workers * npad * 2 : 0;
    const size_t fixed = ring * entry + ring * 8 + scratch_bytes + gdeg_bytes + (64ull << 20);
    if (fixed >= free_b) throw std::runtime_error("CUDA error: out of device memory for the worklist");
    const uint64_t by_mem = (uint64_t)((free_b - fixed) * 0.6 / ((double)workers * entry));
    uint32_t bound = (uint32_t)std::min<uint64_t>((uint64_t)std::max<uint32_t>(s.stack_bound, 1) + 1,
                                                  std::max<uint64_t>(by_mem, 2));
    if (s.stack_cap) bound = std::min(bound, s.stack_cap);
    unsigned char* stacks = (unsigned char*)C.stacks.get((size_t)workers * bound * entry);
    unsigned char* wl = (unsigned char*)C.wl.get(ring * entry);
    unsigned long long* seq = (unsigned long long*)C.seq.get(ring * 8);
    const uint32_t cover_words = (g.n + 31) / 32;
    const size_t slots_bytes = ((size_t)workers * cover_words * 4 + 255) / 256 * 256;
    unsigned char* misc = (unsigned char*)C.misc.get(sizeof(Ctl) + slots_bytes + (size_t)workers * sizeof(WStats));
    Ctl* ctl = reinterpret_cast<Ctl*>(misc);
    uint32_t* cover_slots = reinterpret_cast<uint32_t*>(misc + sizeof(Ctl));
    WStats* stats = reinterpret_cast<WStats*>(misc + sizeof(Ctl) + slots_bytes);
    unsigned char* scr = (unsigned char*)C.scratch.get(scratch_bytes);
    const size_t wn = (size_t)workers * g.n;
    unsigned long long* owner = reinterpret_cast<unsigned long long*>(scr);  // 8-aligned first
    uint32_t* scratch = reinterpret_cast<uint32_t*>(scr + wn * 8);
    uint32_t* cnt = reinterpret_cast<uint32_t*>(scr + wn * 56);
    uint32_t* tag = reinterpret_cast<uint32_t*>(scr + wn * 60);
    CUDA_CHECK(cudaMemsetAsync(cnt, 0, wn * 4, st));        // counters start at zero
    CUDA_CHECK(cudaMemsetAsync(owner, 0xFF, wn * 8, st));   // no triangle claims
    CUDA_CHECK(cudaMemsetAsync(tag, 0, wn * 4, st));        // epochs start at 1
    uint16_t* gdeg_arr = gdeg ? (uint16_t*)C.gdeg.get(gdeg_bytes) : nullptr;

    // initial worklist: root (init_root) or the seeds, as u16 records
    const uint64_t nseeds = s.num_seeds ? s.num_seeds : 1;
    std::vector<unsigned char> recs(nseeds * entry, 0);
    for (uint64_t i = 0; i < nseeds; ++i) {
        unsigned char* rec = recs.data() + i * entry;
        uint32_t* h = reinterpret_cast<uint32_t*>(rec);
        uint16_t* dd = reinterpret_cast<uint16_t*>(rec + 16);
        if (s.num_seeds) {
            const uint32_t* r = s.seeds + i * (2 + (size_t)g.n);
            h[0] = r[0];
            h[1] = r[1];
            for (uint32_t v = 0; v < g.n; ++v) dd[v] = r[2 + v] == REM ? DREM : (uint16_t)r[2 + v];
        } else {
            h[0] = 0;
            h[1] = (uint32_t)g.m;
            for (uint32_t v = 0; v < g.n; ++v) dd[v] = (uint16_t)g.degree(v);
        }
        for (uint32_t v = g.n; v < npad; ++v) dd[v] = DREM;
    }
    Ctl hc;
    std::memset(&hc, 0, sizeof(hc));
    hc.best = s.best;
    hc.tail = nseeds;
    hc.work = (nseeds << 32) | nseeds;
    hc.best_owner = ~0ull;
    CUDA_CHECK(cudaMemcpyAsync(ctl, &hc, sizeof(hc), cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(wl, recs.data(), recs.size(), cudaMemcpyHostToDevice, st));
    init_seq_kernel<<<64, 256, 0, st>>>(seq, (uint32_t)ring, (uint32_t)nseeds);
    CUDA_CHECK(cudaGetLastError());
    CUDA_CHECK(cudaMemsetAsync(stats, 0, (size_t)workers * sizeof(WStats), st));
    out.h2d_bytes += sizeof(hc) + recs.size();
    out.launches += 2;

    SparseArgs a;
    a.off = dg.off;
    a.nbr = dg.nbr;
    a.n = g.n;
    a.npad = npad;
    a.pvc = s.pvc ? 1 : 0;
    a.k = s.k;
    a.capacity = (uint32_t)cap;
    a.ring_mask = (uint32_t)(ring - 1);
    a.threshold = (uint32_t)std::min<uint64_t>(s.threshold, cap);
    a.workers = workers;
    a.stack_bound = bound;
    a.entry_bytes = entry;
    a.stacks = stacks;
    a.wl = wl;
    a.seq = seq;
    a.ctl = ctl;
    a.cover_slots = cover_slots;
    a.cover_words = cover_words;
    a.stats = stats;
    a.scratch = scratch;
    a.cnt = cnt;
    a.owner = owner;
    a.tag = tag;
    a.node_budget = s.node_budget;
    a.timeout_ns = s.timeout_s >= 0 ? (unsigned long long)(s.timeout_s * 1e9) : 0ull;
    if (s.timeout_s >= 0 && a.timeout_ns == 0) a.timeout_ns = 1;
    a.flush_every = s.node_budget ? 1 : 16;
    a.backoff_ns = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(s.backoff_us * 1000, 64), 2000);
    a.seq_mode = s.strategy != 0 ? 1 : 0;  // seq and stackonly never donate
    a.donate_oldest = s.donate_oldest ? 1 : 0;
    a.stackonly = s.strategy == 2 ? 1 : 0;
    a.depth = s.depth;
    a.mailbox = s.mailbox;
    a.gdeg = gdeg_arr;

    auto kern = gdeg ? sparse_kernel<false, true> : sparse_kernel<false, false>;
    CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CUDA_CHECK(cudaEventRecord(C.ev0, st));
    kern<<<workers, threads, smem, st>>>(a);
    CUDA_CHECK(cudaGetLastError());
    const WStats* hs = finish_and_read(C, st, ctl, stats, workers, hc, out);
    if (hc.status >= 100) {
        uint32_t d[12] = {0};
        CUDA_CHECK(cudaMemcpy(d, cover_slots, sizeof d, cudaMemcpyDeviceToHost));
        std::string msg = "CUDA error: sparse engine invariant violated at check site " +
                          std::to_string(hc.status - 100) + " [";
        for (uint32_t x : d) msg += std::to_string(x) + " ";
        throw std::runtime_error(msg + "]");
    }
    if (hc.status == 4) {
        uint32_t d[3] = {0, 0, 0};
        CUDA_CHECK(cudaMemcpy(d, cover_slots, sizeof d, cudaMemcpyDeviceToHost));
        throw std::runtime_error("CUDA error: sparse engine invariant violated (edges " +
                                 std::to_string(d[0]) + " with no alive vertex; cc " +
                                 std::to_string(d[1]) + ", degree sum " + std::to_string(d[2]) + ")");
    }
    if (hc.status == 3)
        throw std::runtime_error("CUDA error: search stack depth exceeded the device-memory cap (" +
                                 std::to_string(bound) + " nodes per worker) with the worklist full");
    out.status = hc.status;
    out.wl_added = hc.tail;
    out.wl_current = (uint32_t)hc.work;
    out.wl_removed = hc.tail - out.wl_current;
    out.wl_max_size = nseeds;
    aggregate(hs, workers, out);
    if (s.strategy == 2) out.wl_added = out.wl_removed = out.wl_current = out.wl_max_size = 0;
    if (hc.best_owner != ~0ull) {
        const uint32_t ow = (uint32_t)(hc.best_owner & 0xFFFFFFFFu);
        out.found = true;
        out.found_size = (uint32_t)(hc.best_owner >> 32);
        std::vector<uint32_t> bits(cover_words);
        CUDA_CHECK(cudaMemcpy(bits.data(), cover_slots + (size_t)ow * cover_words, cover_words * 4,
                              cudaMemcpyDeviceToHost));
        out.d2h_bytes += cover_words * 4;
        out.cover.clear();
        for (uint32_t v = 0; v < g.n; ++v)
            if ((bits[v >> 5] >> (v & 31)) & 1u) out.cover.push_back(v);
    }
}


namespace {
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    void* get(size_t need) {
        if (need > bytes) {
            if (p) cudaFree(p);
            p = nullptr;
            CUDA_CHECK(cudaMalloc(&p, need));
            bytes = need;
        }
        return p;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};
}  // namespace

// The sparse engine's level-synchronous expansion (large n; sparse_expand_kernel): records are
// sparse records (16 + 2 npad bytes), one CTA per node of a level.
static void expand_frontier_sparse(const Graph& g, const SolveSpec& s, uint64_t target, Frontier& f) {
    const int dev = s.device;
    if (2 * g.m >= (1ull << 32)) throw std::invalid_argument("graph too large for u32 CSR offsets");
    uint32_t maxdeg = 0;
    for (uint32_t v = 0; v < g.n; ++v) maxdeg = std::max(maxdeg, g.degree(v));
    if (maxdeg >= 0xFFFFu) throw std::invalid_argument("sparse engine: degree >= 65535");
    CUDA_CHECK(cudaSetDevice(dev));
    DeviceCtx& C = ctx_for(dev);
    std::lock_guard<std::mutex> solve_lock(C.solve_mu);
    cudaStream_t st = s.stream ? static_cast<cudaStream_t>(s.stream) : C.stream;
    const uint32_t npad = (g.n + 7) / 8 * 8;
    const size_t entry = 16 + 2 * (size_t)npad;
    int max_smem = 0;
    CUDA_CHECK(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    const size_t list_smem = (2 * SP_THREADS + 1) * 4;
    const bool gdeg = s.engine == 7 || 2 * (size_t)npad + list_smem + sizeof(SpShared) + 1024 > (size_t)max_smem;
    const size_t smem = (gdeg ? 0 : 2 * (size_t)npad) + list_smem;
    if ((int)g.dev.size() <= dev) g.dev.resize(dev + 1);
    if (!g.dev[dev] || !g.dev[dev]->off) {
        auto dg = g.dev[dev] ? g.dev[dev] : std::make_shared<DeviceGraph>();
        dg->device = dev;
        std::vector<uint32_t> off32(g.n + 1);
        for (uint32_t v = 0; v <= g.n; ++v) off32[v] = (uint32_t)g.off[v];
        CUDA_CHECK(cudaMalloc(&dg->off, off32.size() * 4));
        CUDA_CHECK(cudaMalloc(&dg->nbr, std::max<size_t>(1, g.nbr.size()) * 4));
        CUDA_CHECK(cudaMemcpy(dg->off, off32.data(), off32.size() * 4, cudaMemcpyHostToDevice));
        if (!g.nbr.empty())
            CUDA_CHECK(cudaMemcpy(dg->nbr, g.nbr.data(), g.nbr.size() * 4, cudaMemcpyHostToDevice));
        dg->csr_bytes = off32.size() * 4 + g.nbr.size() * 4;
        g.dev[dev] = dg;
    }
    const DeviceGraph& dg = *g.dev[dev];
    const uint32_t ctas = (uint32_t)C.sms;
    const size_t wn = (size_t)ctas * g.n;
    const uint32_t cover_words = (g.n + 31) / 32;
    DevBuf bin, bout, bflags, bcov, bidx, bscr, bgdeg;
    unsigned char* scr = (unsigned char*)bscr.get(wn * (12 * 4 + 4 + 8 + 4));
    SparseExpandArgs e{};
    SparseArgs& a = e.s;
    a.off = dg.off;
    a.nbr = dg.nbr;
    a.n = g.n;
    a.npad = npad;
    a.pvc = s.pvc ? 1 : 0;
    a.k = s.k;
    a.entry_bytes = entry;
    a.cover_words = cover_words;
    a.owner = reinterpret_cast<unsigned long long*>(scr);
    a.scratch = reinterpret_cast<uint32_t*>(scr + wn * 8);
    a.cnt = reinterpret_cast<uint32_t*>(scr + wn * 56);
    a.tag = reinterpret_cast<uint32_t*>(scr + wn * 60);
    a.gdeg = gdeg ? (uint16_t*)bgdeg.get((size_t)ctas * npad * 2) : nullptr;
    {
        std::vector<unsigned char> root(entry, 0);
        uint32_t* h = reinterpret_cast<uint32_t*>(root.data());
        uint16_t* dd = reinterpret_cast<uint16_t*>(root.data() + 16);
        h[0] = 0;
        h[1] = (uint32_t)g.m;
        for (uint32_t v = 0; v < npad; ++v) dd[v] = v < g.n ? (uint16_t)g.degree(v) : DREM;
        CUDA_CHECK(cudaMemcpyAsync(bin.get(entry), root.data(), entry, cudaMemcpyHostToDevice, st));
    }
    auto kern = gdeg ? sparse_expand_kernel<true> : sparse_expand_kernel<false>;
    CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    uint64_t count = 1;
    f = Frontier();
    f.best = s.best;
    std::vector<uint32_t> flags, covers, idx;
    while (count > 0 && count < target) {
        // fresh claim / tag / counter state per level (epochs restart with every launch)
        CUDA_CHECK(cudaMemsetAsync(a.owner, 0xFF, wn * 8, st));
        CUDA_CHECK(cudaMemsetAsync(a.cnt, 0, wn * 4, st));
        CUDA_CHECK(cudaMemsetAsync(a.tag, 0, wn * 4, st));
        e.in = (unsigned char*)bin.p;
        e.out = (unsigned char*)bout.get(2 * count * entry);
        e.flags = (uint32_t*)bflags.get(count * 4);
        e.covers = (uint32_t*)bcov.get(count * (cover_words + 1) * 4);
        e.count = (uint32_t)count;
        e.best = f.best;
        const uint32_t grid = (uint32_t)std::min<uint64_t>(count, ctas);
        kern<<<grid, SP_THREADS, smem, st>>>(e);
        CUDA_CHECK(cudaGetLastError());
        ++f.launches;
        flags.resize(count);
        CUDA_CHECK(cudaMemcpyAsync(flags.data(), e.flags, count * 4, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        f.nodes += count;
        ++f.levels;
        bool any_cover = false;
        for (uint64_t i = 0; i < count; ++i) any_cover |= flags[i] == 1;
        if (any_cover) {
            covers.resize(count * (cover_words + 1));
            CUDA_CHECK(cudaMemcpy(covers.data(), e.covers, covers.size() * 4, cudaMemcpyDeviceToHost));
            for (uint64_t i = 0; i < count; ++i) {
                if (flags[i] != 1) continue;
                const uint32_t* c = &covers[i * (cover_words + 1)];
                if (s.pvc ? !f.found : c[0] < f.best) {
                    f.found = true;
                    if (!s.pvc) f.best = c[0];
                    f.cover.clear();
                    for (uint32_t v = 0; v < g.n; ++v)
                        if ((c[1 + (v >> 5)] >> (v & 31)) & 1u) f.cover.push_back(v);
                }
            }
        }
        if (s.pvc && f.found) {
            count = 0;
            break;
        }
        idx.clear();
        for (uint64_t i = 0; i < count; ++i)
            if (flags[i] == 2) {
                idx.push_back((uint32_t)(2 * i));
                idx.push_back((uint32_t)(2 * i + 1));
            }
        const uint64_t nc = idx.size();
        if (nc) {
            uint32_t* didx = (uint32_t*)bidx.get(nc * 4);
            CUDA_CHECK(cudaMemcpyAsync(didx, idx.data(), nc * 4, cudaMemcpyHostToDevice, st));
            unsigned char* dnext = (unsigned char*)bin.get(nc * entry);
            gather_records_kernel<<<(uint32_t)std::min<uint64_t>(nc, 65535), 256, 0, st>>>(
                e.out, didx, dnext, (uint32_t)nc, (uint32_t)(entry / 16));
            CUDA_CHECK(cudaGetLastError());
            ++f.launches;
        }
        count = nc;
    }
    std::vector<unsigned char> level(count * entry);
    if (count) {
        CUDA_CHECK(cudaMemcpyAsync(level.data(), bin.p, count * entry, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
    }
    f.records.assign(count * (2 + (size_t)g.n), 0);
    for (uint64_t i = 0; i < count; ++i) {
        const unsigned char* rec = level.data() + i * entry;
        uint32_t* r = f.records.data() + i * (2 + (size_t)g.n);
        r[0] = reinterpret_cast<const uint32_t*>(rec)[0];
        r[1] = reinterpret_cast<const uint32_t*>(rec)[1];
        const uint16_t* dd = reinterpret_cast<const uint16_t*>(rec + 16);
        for (uint32_t v = 0; v < g.n; ++v) r[2 + v] = dd[v] == DREM ? REM : dd[v];
    }
    f.count = count;
}

void expand_frontier(const Graph& g, const SolveSpec& s, uint64_t target, Frontier& f) {
    if (s.engine == 2 || s.engine == 7 || g.n > 1024) return expand_frontier_sparse(g, s, target, f);
    if (g.n > 1024)
        throw std::invalid_argument("frontier expansion needs the dense engine (n <= 1024)");
    const int dev = s.device;
    if (device_count() == 0) throw std::runtime_error("CUDA error: no CUDA device visible");
    CUDA_CHECK(cudaSetDevice(dev));
    DeviceCtx& C = ctx_for(dev);
    std::lock_guard<std::mutex> solve_lock(C.solve_mu);
    cudaStream_t st = s.stream ? static_cast<cudaStream_t>(s.stream) : C.stream;
    const uint32_t W = pick_w(g.n);
    const uint32_t npad = 32 * W;
    const size_t entry = dense_record_bytes(W);
    if ((int)g.dev.size() <= dev) g.dev.resize(dev + 1);
    if (!g.dev[dev]) {
        auto dg = std::make_shared<DeviceGraph>();
        dg->device = dev;
        dg->W = W;
        dg->npad = npad;
        std::vector<uint32_t> at = build_bitmap(g, W, npad);
        dg->at4_bytes = at.size() * 4;
        CUDA_CHECK(cudaMalloc(&dg->at4, dg->at4_bytes));
        CUDA_CHECK(cudaMemcpy(dg->at4, at.data(), dg->at4_bytes, cudaMemcpyHostToDevice));
        g.dev[dev] = dg;
    }
    const DeviceGraph& dg = *g.dev[dev];
    const size_t smem = dense_smem_bytes(W, 8);  // see dense_scratch_base

    // Levels stay on the device: per level only the flags come down and the gather list of
    // surviving children goes up; the final level is copied once.
    DevBuf bin, bout, bflags, bcov, bidx;
    {
        std::vector<unsigned char> root(entry);
        std::vector<uint32_t> deg(g.n);
        for (uint32_t v = 0; v < g.n; ++v) deg[v] = g.degree(v);
        pack_record(W, g.n, 0, (uint32_t)g.m, deg.data(), root.data());
        CUDA_CHECK(cudaMemcpyAsync(bin.get(entry), root.data(), entry, cudaMemcpyHostToDevice, st));
    }
    uint64_t count = 1;
    f = Frontier();
    f.best = s.best;
    std::vector<uint32_t> flags, covers, idx;
    while (count > 0 && count < target) {
        unsigned char* din = (unsigned char*)bin.p;
        unsigned char* dout = (unsigned char*)bout.get(2 * count * entry);
        uint32_t* dflags = (uint32_t*)bflags.get(count * 4);
        uint32_t* dcov = (uint32_t*)bcov.get(count * (W + 1) * 4);
        ExpandArgs a;
        a.at4 = dg.at4;
        a.n = g.n;
        a.npad = npad;
        a.pvc = s.pvc ? 1 : 0;
        a.k = s.k;
        a.best = f.best;
        a.count = (uint32_t)count;
        a.entry_bytes = entry;
        a.in = din;
        a.out = dout;
        a.flags = dflags;
        a.covers = dcov;
        const uint32_t grid = (uint32_t)std::min<uint64_t>((count + 7) / 8, 1184);
        switch (W) {
#define VCG_EXPAND(WW)                                                                        \
    case WW: {                                                                                \
        CUDA_CHECK(cudaFuncSetAttribute(expand_kernel<WW>,                                    \
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
        expand_kernel<WW><<<grid, 256, smem, st>>>(a);                                        \
        break;                                                                                \
    }
            VCG_EXPAND(4) VCG_EXPAND(8) VCG_EXPAND(16) VCG_EXPAND(32)
#undef VCG_EXPAND
        }
        CUDA_CHECK(cudaGetLastError());
        ++f.launches;
        flags.resize(count);
        CUDA_CHECK(cudaMemcpyAsync(flags.data(), dflags, count * 4, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        f.nodes += count;
        ++f.levels;
        // covers found on this level (fixed bound inside the level, improved between levels)
        bool any_cover = false;
        for (uint64_t i = 0; i < count; ++i) any_cover |= flags[i] == 1;
        if (any_cover) {
            covers.resize(count * (W + 1));
            CUDA_CHECK(cudaMemcpy(covers.data(), dcov, covers.size() * 4, cudaMemcpyDeviceToHost));
            for (uint64_t i = 0; i < count; ++i) {
                if (flags[i] != 1) continue;
                const uint32_t* c = &covers[i * (W + 1)];
                if (s.pvc ? !f.found : c[0] < f.best) {
                    f.found = true;
                    if (!s.pvc) f.best = c[0];
                    f.cover.clear();
                    for (uint32_t v = 0; v < g.n; ++v)
                        if ((c[1 + (v >> 5)] >> (v & 31)) & 1u) f.cover.push_back(v);
                }
            }
        }
        if (s.pvc && f.found) {
            count = 0;
            break;
        }
        idx.clear();
        for (uint64_t i = 0; i < count; ++i)
            if (flags[i] == 2) {
                idx.push_back((uint32_t)(2 * i));
                idx.push_back((uint32_t)(2 * i + 1));
            }
        const uint64_t nc = idx.size();
        if (nc) {
            uint32_t* didx = (uint32_t*)bidx.get(nc * 4);
            CUDA_CHECK(cudaMemcpyAsync(didx, idx.data(), nc * 4, cudaMemcpyHostToDevice, st));
            unsigned char* dnext = (unsigned char*)bin.get(nc * entry);
            gather_records_kernel<<<(uint32_t)std::min<uint64_t>(nc, 65535), 64, 0, st>>>(
                dout, didx, dnext, (uint32_t)nc, (uint32_t)(entry / 16));
            CUDA_CHECK(cudaGetLastError());
            ++f.launches;
        }
        count = nc;
    }
    std::vector<unsigned char> level(count * entry);
    if (count) {
        CUDA_CHECK(cudaMemcpyAsync(level.data(), bin.p, count * entry, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
    }
    // unpack the frontier into [cc, edges, deg[n]] records
    f.records.assign(count * (2 + (size_t)g.n), 0);
    for (uint64_t i = 0; i < count; ++i) {
        const unsigned char* rec = level.data() + i * entry;
        uint32_t* r = f.records.data() + i * (2 + (size_t)g.n);
        r[0] = reinterpret_cast<const uint32_t*>(rec)[0];
        r[1] = reinterpret_cast<const uint32_t*>(rec)[1];
        const uint16_t* dd = reinterpret_cast<const uint16_t*>(rec + 16);
        for (uint32_t v = 0; v < g.n; ++v) {
            const uint16_t x = dd[(v & 31) * W + (v >> 5)];
            r[2 + v] = x == 0xFFFF ? REM : x;
        }
    }
    f.count = count;
}

}  // namespace vcg
