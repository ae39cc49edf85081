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
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine.hpp"

namespace vcg {

#define CUDA_CHECK(x)                                                                       \
    do {                                                                                    \
        cudaError_t e_ = (x);                                                               \
        if (e_ != cudaSuccess)                                                              \
            throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + \
                                     " at " #x);                                            \
    } while (0)

constexpr uint32_t REM = 0xFFFFFFFFu;
constexpr unsigned FULL = 0xFFFFFFFFu;

// ------------------------------------------------------------------ device-global state

struct Ctl {
    // line 0: read by every worker once per node (two vector loads)
    uint32_t best;    // MVC bound (atomicMin); PVC: k
    uint32_t cancel;  // 1 = stop: PVC found, timeout, budget, host request
    uint32_t found;   // PVC: a cover of size <= k was recorded
    uint32_t pad0;
    // (pending << 32) | size: pending = queued items + active workers (termination when 0);
    // size = queued items + in-flight enqueue reservations (threshold gate, capacity)
    unsigned long long work;
    unsigned long long pad1;
    uint32_t pad2[24];
    // line 1: ring tickets (Vyukov-style slots with per-slot sequence numbers)
    unsigned long long head, tail;
    uint32_t pad3[28];
    // line 2: results
    unsigned long long nodes_total, best_owner;
    int32_t status;
    uint32_t pad4[27];
};
static_assert(sizeof(Ctl) == 384, "Ctl layout");

struct WStats {
    unsigned long long nodes, rounds, maxdeg, children, rm1, rm2, rmh, high_water, donated,
        active, max_queue, dooms;
    unsigned long long phase[10];
};

enum Phase { PH_WL_REMOVE, PH_WL_ADD, PH_STACK, PH_DEG1, PH_DEG2, PH_HIGH, PH_MAXDEG,
             PH_BRANCH_NBRS, PH_BRANCH_V, PH_PRUNE };  // metrics.hpp:15-26 order

struct DenseArgs {
    const uint4* at4;         // adjacency bitmap, [W/4][npad] uint4 groups
    uint32_t n, npad, m;
    int pvc;
    uint32_t k;
    uint32_t capacity;        // logical worklist capacity (try_add rejects at capacity)
    uint32_t ring_mask;       // physical ring slots - 1 (power of two >= max(capacity, 2))
    uint32_t threshold;
    uint32_t workers;
    uint32_t stack_bound;
    unsigned long long entry_bytes;
    unsigned char* stacks;    // workers * stack_bound * entry_bytes
    unsigned char* wl;        // ring slots * entry_bytes
    unsigned long long* seq;  // ring slots
    Ctl* ctl;
    uint32_t* cover_slots;    // workers * W words
    WStats* stats;
    unsigned long long node_budget;
    unsigned long long timeout_ns;
    unsigned long long flush_every;  // visits between node-counter flushes / limit checks
    uint32_t backoff_ns;
    int seq_mode;             // never donate (solve_*_seq semantics)
    int donate_oldest;        // donate the bottom (oldest) stack entry instead of the new child
    volatile uint32_t* mailbox;  // host-mapped: [0] ext best in, [1] cancel in, [2] best out, [3] found out
};

// ------------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint4 ld_volatile_v4(const void* p) {
    uint4 r;
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ int ld_relaxed_s32(const int* p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ ulonglong2 ld_volatile_v2u64(const void* p) {
    ulonglong2 r;
    asm volatile("ld.volatile.global.v2.u64 {%0,%1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ uint32_t comp(const uint4& r, int c) {
    return c == 0 ? r.x : c == 1 ? r.y : c == 2 ? r.z : r.w;
}

// ReductionBound::current (reductions.hpp:19-27)
__device__ __forceinline__ uint32_t limit_for(int pvc, uint32_t k, uint32_t best, uint32_t cc) {
    if (pvc) return cc >= k ? 0u : k - cc;
    uint32_t spend = cc + 1;
    return best <= spend ? 0u : best - spend;
}
// should_prune (bounds.cpp:21-30)
__device__ __forceinline__ bool should_prune(int pvc, uint32_t k, uint32_t best, uint32_t cc,
                                             uint32_t edges) {
    if (pvc) {
        if (cc > k) return true;
        unsigned long long s = k - cc;
        return (unsigned long long)edges > s * s;
    }
    if (cc >= best) return true;
    unsigned long long s = best - cc - 1;
    return (unsigned long long)edges > s * s;
}

// Host mailbox (pinned, mapped): one poller per device (worker 0) folds an external MVC bound
// into the device bound and turns a host cancel request into the device cancel flag.
__device__ __forceinline__ void poll_mailbox(const DenseArgs& a, Ctl* ctl) {
    const uint32_t eb = a.mailbox[0];
    if (!a.pvc && eb) atomicMin(&ctl->best, eb);
    if (a.mailbox[1]) atomicExch(&ctl->cancel, 1u);
}

// ------------------------------------------------------------------ the warp worker

template <int W, bool INSTR>
struct WarpNode {
    static constexpr int Q = W / 4;  // uint4 groups per bitmap row
    uint32_t d[W];                   // degree of vertex 32*i + lane
    uint32_t aw;                     // lane j < W: alive bitmap word j
    uint32_t cc, edges;              // uniform
    bool doom;                       // uniform: proven to be pruned (see pass_high)
    const uint4* sat;                // shared adjacency bitmap
    uint32_t npad;
    int lane;

    __device__ __forceinline__ uint32_t row_word(uint32_t u, uint32_t j) const {
        // word j of u's adjacency row
        return reinterpret_cast<const uint32_t*>(sat)[((j >> 2) * npad + u) * 4 + (j & 3)];
    }
    __device__ __forceinline__ void rebuild_alive() {
#pragma unroll
        for (int i = 0; i < W; ++i) {
            uint32_t b = __ballot_sync(FULL, d[i] != REM);
            if (lane == i) aw = b;
        }
    }
    __device__ __forceinline__ uint32_t deg_of(uint32_t u) const {
        uint32_t t = 0;
        const uint32_t ui = u >> 5;
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (i == ui) t = d[i];
        return __shfl_sync(FULL, t, u & 31);
    }
    // search_node.cpp:16-25 remove_vertex_into_cover(u), u alive
    __device__ __forceinline__ void remove_vertex(uint32_t u) {
        const uint32_t du = deg_of(u);
        const uint32_t ui = u >> 5, ul = u & 31;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint4 r = sat[q * npad + u];  // broadcast
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const int i = 4 * q + c;
                const uint32_t bit = (comp(r, c) >> lane) & 1u;
                uint32_t x = d[i];
                x = (x == REM) ? x : x - bit;
                if (i == ui && lane == ul) x = REM;
                d[i] = x;
            }
        }
        if (lane == ui) aw &= ~(1u << ul);
        cc += 1;
        edges -= du;
    }
    // first vertex >= pos satisfying pred at this moment (== the reference's ascending scan)
    template <class P>
    __device__ __forceinline__ int find_first(int pos, P pred) const {
        int v = -1;
        const int pi = pos >> 5;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            if (v < 0 && i >= pi) {
                uint32_t b = __ballot_sync(FULL, pred(d[i]));
                if (i == pi) b &= FULL << (pos & 31);
                if (b) v = 32 * i + __ffs(b) - 1;
            }
        }
        return v;
    }
    // lane j < W: word j of (row v AND alive)
    __device__ __forceinline__ uint32_t alive_row(uint32_t v) const {
        return lane < W ? (row_word(v, lane) & aw) : 0u;
    }
    __device__ __forceinline__ int first_bit(uint32_t xl, uint32_t skip_lanes = 0) const {
        uint32_t b = __ballot_sync(FULL, xl != 0) & ~skip_lanes;
        if (!b) return -1;
        int j = __ffs(b) - 1;
        uint32_t w = __shfl_sync(FULL, xl, j);
        return 32 * j + __ffs(w) - 1;
    }
    // reductions.cpp:7-19
    // A node whose cover already reaches the bound is pruned whatever the remaining rules do
    // (should_prune tests |S| first and rules only grow S), so the reduction may stop there.
    __device__ __forceinline__ bool doomed(int pvc, uint32_t k, uint32_t snap) const {
        return doom || (pvc ? cc > k : cc >= snap);
    }
    __device__ __forceinline__ bool pass_degree_one(unsigned long long& removals, int pvc,
                                                    uint32_t k, uint32_t snap) {
        bool changed = false;
        int pos = 0;
        while (!doomed(pvc, k, snap)) {
            int v = find_first(pos, [](uint32_t x) { return x == 1u; });
            if (v < 0) break;
            int u = first_bit(alive_row(v));
            remove_vertex(u);
            ++removals;
            changed = true;
            pos = v + 1;
        }
        return changed;
    }
    // reductions.cpp:22-40 (partners = the two alive neighbours, ascending)
    __device__ __forceinline__ bool pass_degree_two(unsigned long long& removals, int pvc,
                                                    uint32_t k, uint32_t snap) {
        bool changed = false;
        int pos = 0;
        while (!doomed(pvc, k, snap)) {
            int v = find_first(pos, [](uint32_t x) { return x == 2u; });
            if (v < 0) break;
            const uint32_t xl = alive_row(v);
            const uint32_t b = __ballot_sync(FULL, xl != 0);
            const int j0 = __ffs(b) - 1;
            const uint32_t w0 = __shfl_sync(FULL, xl, j0);
            const int p0 = 32 * j0 + __ffs(w0) - 1;
            const uint32_t w0b = w0 & (w0 - 1);
            int p1;
            if (w0b) {
                p1 = 32 * j0 + __ffs(w0b) - 1;
            } else {
                const uint32_t b2 = b & ~(1u << j0);
                const int j1 = __ffs(b2) - 1;
                p1 = 32 * j1 + __ffs(__shfl_sync(FULL, xl, j1)) - 1;
            }
            if ((row_word(p0, p1 >> 5) >> (p1 & 31)) & 1u) {
                remove_vertex(p0);
                remove_vertex(p1);
                removals += 2;
                changed = true;
            }
            pos = v + 1;
        }
        return changed;
    }
    // reductions.cpp:43-58 (limit recomputed after every removal)
    __device__ __forceinline__ bool pass_high(int pvc, uint32_t k, uint32_t snap,
                                              unsigned long long& removals) {
        bool changed = false;
        int pos = 0;
        uint32_t lim = limit_for(pvc, k, snap, cc);
        // Every alive vertex above the limit at pass start is removed by this pass (each
        // removal lowers the limit by one and a degree by at most one), so more than `lim` of
        // them take |S| past the bound: the node is pruned whatever else happens.
        uint32_t over = 0;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            const uint32_t x = d[i];
            over += __popc(__ballot_sync(FULL, x != REM && x > 0u && x > lim));
        }
        if (over > lim) {
            doom = true;
            return true;
        }
        while (!doomed(pvc, k, snap)) {
            int v = find_first(pos, [lim](uint32_t x) { return x != REM && x > 0u && x > lim; });
            if (v < 0) break;
            remove_vertex(v);
            ++removals;
            changed = true;
            lim = limit_for(pvc, k, snap, cc);
            pos = v + 1;
        }
        return changed;
    }
    // reduce_loop (reductions.cpp:63-90) with the bound snapshot taken per round
    template <class Cnt>
    __device__ __forceinline__ void reduce(int pvc, uint32_t k, uint32_t snap, Cnt& st) {
        while (true) {
            if (edges == 0) break;
            ++st.rounds;
            const uint32_t lim = limit_for(pvc, k, snap, cc);
            // fused quick test: if no vertex has degree 1 or 2 and none exceeds the limit, this
            // round cannot change anything (it is the final no-change round)
            uint32_t any = 0;
#pragma unroll
            for (int i = 0; i < W; ++i) {
                const uint32_t x = d[i];
                any |= __ballot_sync(FULL, x == 1u || x == 2u || (x != REM && x > lim && x > 0u));
            }
            if (!any) break;
            bool changed = false;
            long long t0 = INSTR ? clock64() : 0;
            changed |= pass_degree_one(st.rm1, pvc, k, snap);
            long long t1 = INSTR ? clock64() : 0;
            changed |= pass_degree_two(st.rm2, pvc, k, snap);
            long long t2 = INSTR ? clock64() : 0;
            changed |= pass_high(pvc, k, snap, st.rmh);
            if (INSTR) {
                long long t3 = clock64();
                st.phase[PH_DEG1] += t1 - t0;
                st.phase[PH_DEG2] += t2 - t1;
                st.phase[PH_HIGH] += t3 - t2;
            }
            if (!changed || doomed(pvc, k, snap)) break;
        }
    }
    // search_node.cpp:34-46: smallest id among alive vertices of maximum degree
    __device__ __forceinline__ uint32_t argmax() const {
        uint32_t mx = 0;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            const uint32_t x = d[i];
            const uint32_t key = x != REM ? ((x << 11) | (2047u - (32u * i + lane))) : 0u;
            mx = max(mx, key);
        }
        mx = __reduce_max_sync(FULL, mx);
        return 2047u - (mx & 2047u);
    }
    // Writes the remove-N(v) child (search_node.cpp:27-32 on a clone) as an entry record:
    // header {cc, edges} by lane 0, then lane-major u16 degrees.
    __device__ __forceinline__ void write_child_without_neighbors(uint32_t v,
                                                                  unsigned char* rec) const {
        const uint32_t xl = alive_row(v);
        uint32_t X[W];
#pragma unroll
        for (int j = 0; j < W; ++j) X[j] = __shfl_sync(FULL, xl, j);
        const uint32_t xcnt = __reduce_add_sync(FULL, __popc(xl));
        uint32_t packed[W / 2];
        uint32_t esum = 0;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            const uint32_t x = d[i];
            const bool alive_after = (x != REM) && !((X[i] >> lane) & 1u);
            uint32_t nd = REM;
            if (__any_sync(FULL, alive_after)) {
                uint32_t s = 0;
#pragma unroll
                for (int q = 0; q < Q; ++q) {
                    if ((X[4 * q] | X[4 * q + 1] | X[4 * q + 2] | X[4 * q + 3]) != 0u) {
                        const uint4 col = sat[q * npad + 32 * i + lane];
                        s += __popc(col.x & X[4 * q]) + __popc(col.y & X[4 * q + 1]) +
                             __popc(col.z & X[4 * q + 2]) + __popc(col.w & X[4 * q + 3]);
                    }
                }
                if (alive_after) nd = x - s;
            }
            esum += alive_after ? nd : 0u;
            const uint32_t h = alive_after ? nd : 0xFFFFu;
            if (i & 1) packed[i / 2] |= h << 16;
            else packed[i / 2] = h;
        }
        const uint32_t e2 = __reduce_add_sync(FULL, esum);
        if (lane == 0) {
            reinterpret_cast<uint32_t*>(rec)[0] = cc + xcnt;
            reinterpret_cast<uint32_t*>(rec)[1] = e2 / 2;
        }
        store_degrees(rec, packed);
    }
    __device__ __forceinline__ void store_degrees(unsigned char* rec, const uint32_t* packed) const {
        unsigned char* p = rec + 16 + lane * (2 * W);
        if constexpr (W == 4) {
            *reinterpret_cast<uint2*>(p) = make_uint2(packed[0], packed[1]);
        } else {
#pragma unroll
            for (int t = 0; t < W / 8; ++t)
                reinterpret_cast<uint4*>(p)[t] =
                    make_uint4(packed[4 * t], packed[4 * t + 1], packed[4 * t + 2], packed[4 * t + 3]);
        }
    }
    // Stores the current node as a record (header by lane 0, lane-major u16 degrees).
    __device__ __forceinline__ void store_current(unsigned char* rec) const {
        uint32_t packed[W / 2];
#pragma unroll
        for (int i = 0; i < W; ++i) {
            const uint32_t h = d[i] == REM ? 0xFFFFu : d[i];
            if (i & 1) packed[i / 2] |= h << 16;
            else packed[i / 2] = h;
        }
        if (lane == 0) {
            reinterpret_cast<uint32_t*>(rec)[0] = cc;
            reinterpret_cast<uint32_t*>(rec)[1] = edges;
        }
        store_degrees(rec, packed);
    }
    // Moves one record (header + lane-major degrees) between stack and worklist memory.
    __device__ __forceinline__ void copy_record(const unsigned char* src, unsigned char* dst) const {
        const unsigned char* p = src + 16 + lane * (2 * W);
        unsigned char* q = dst + 16 + lane * (2 * W);
        if constexpr (W == 4) {
            *reinterpret_cast<uint2*>(q) = *reinterpret_cast<const uint2*>(p);
        } else {
#pragma unroll
            for (int t = 0; t < W / 8; ++t)
                reinterpret_cast<uint4*>(q)[t] = reinterpret_cast<const uint4*>(p)[t];
        }
        if (lane == 0) *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
    }
    template <bool CG>
    __device__ __forceinline__ void load(const unsigned char* rec) {
        uint32_t packed[W / 2];
        const unsigned char* p = rec + 16 + lane * (2 * W);
        if constexpr (W == 4) {
            uint2 t = CG ? __ldcg(reinterpret_cast<const uint2*>(p)) : *reinterpret_cast<const uint2*>(p);
            packed[0] = t.x;
            packed[1] = t.y;
        } else {
#pragma unroll
            for (int t = 0; t < W / 8; ++t) {
                uint4 r = CG ? __ldcg(reinterpret_cast<const uint4*>(p) + t)
                             : reinterpret_cast<const uint4*>(p)[t];
                packed[4 * t] = r.x;
                packed[4 * t + 1] = r.y;
                packed[4 * t + 2] = r.z;
                packed[4 * t + 3] = r.w;
            }
        }
        uint32_t h0 = 0, h1 = 0;
        if (lane == 0) {
            const uint2 h = CG ? __ldcg(reinterpret_cast<const uint2*>(rec))
                               : *reinterpret_cast<const uint2*>(rec);
            h0 = h.x;
            h1 = h.y;
        }
        cc = __shfl_sync(FULL, h0, 0);
        edges = __shfl_sync(FULL, h1, 0);
        doom = false;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            const uint32_t h = (i & 1) ? (packed[i / 2] >> 16) : (packed[i / 2] & 0xFFFFu);
            d[i] = h == 0xFFFFu ? REM : h;
        }
        rebuild_alive();
    }
};

constexpr unsigned long long ONE_PENDING = 1ull << 32;

// GlobalWorklist::try_add (worklist.cpp:11-19): reserve capacity in the packed word (also
// counting the item in `pending` before it can be seen), then draw a ticket. Two always-
// succeeding atomics; no CAS loops (they collapse under thousands of contending warps).
__device__ __forceinline__ bool q_reserve(const DenseArgs& a, unsigned long long& pos_out,
                                          unsigned long long& size_seen) {
    Ctl* ctl = a.ctl;
    const unsigned long long old = atomicAdd(&ctl->work, ONE_PENDING | 1ull);
    const uint32_t size = (uint32_t)old;
    if (size >= a.capacity) {
        atomicAdd(&ctl->work, ~(ONE_PENDING | 1ull) + 1ull);  // undo (try_add rejects)
        return false;
    }
    size_seen = size + 1ull;
    pos_out = atomicAdd(&ctl->tail, 1ull);
    return true;
}

struct Counters {
    unsigned long long nodes = 0, rounds = 0, maxdeg = 0, children = 0, rm1 = 0, rm2 = 0,
                       rmh = 0, high_water = 0, donated = 0, max_queue = 0, dooms = 0;
    unsigned long long phase[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
};

template <int W, bool INSTR>
__global__ void __launch_bounds__(256, (W <= 8 ? 3 : (W == 16 ? 2 : 1))) dense_kernel(DenseArgs a) {
    extern __shared__ uint4 sat[];
    constexpr int Q = W / 4;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const uint32_t worker = blockIdx.x * (blockDim.x >> 5) + wib;

    // Stage the read-only adjacency bitmap once per CTA (coalesced 16-byte copies).
    for (uint32_t t = threadIdx.x; t < Q * a.npad; t += blockDim.x) sat[t] = a.at4[t];
    __syncthreads();
    if (worker >= a.workers) return;

    const unsigned long long t_start = globaltimer();
    const long long c_start = clock64();
    WarpNode<W, INSTR> x;
    x.sat = sat;
    x.npad = a.npad;
    x.lane = lane;
    Counters st;
    Ctl* ctl = a.ctl;
    unsigned char* const my_stack =
        a.stacks + (unsigned long long)worker * a.stack_bound * a.entry_bytes;
    // The local stack is a ring [base, base + sp) so the oldest entry can be donated.
    uint32_t base = 0, sp = 0;
    auto slot_at = [&](uint32_t i) {
        uint32_t j = base + i;
        if (j >= a.stack_bound) j -= a.stack_bound;
        return my_stack + (unsigned long long)j * a.entry_bytes;
    };
    bool have = false, idle = true;
    uint32_t best = a.pvc ? a.k : ctl->best;
    unsigned long long nodes_flushed = 0;
    const uint32_t last_word_mask = (a.n & 31) ? ((1u << (a.n & 31)) - 1u) : FULL;
    const int last_word = (int)((a.n + 31) / 32) - 1;

    while (true) {
        if (!have) {
            if (sp > 0) {
                long long t0 = INSTR ? clock64() : 0;
                --sp;
                x.template load<false>(slot_at(sp));
                have = true;
                if (INSTR) st.phase[PH_STACK] += clock64() - t0;
            } else {
                // GlobalWorklist::remove_or_done (worklist.cpp:21-48) on the device ring
                long long t0 = INSTR ? clock64() : 0;
                if (!idle) {
                    if (lane == 0) atomicAdd(&ctl->work, ~ONE_PENDING + 1ull);  // pending - 1
                    idle = true;
                }
                // take a ticket, then wait for that slot to be published, for termination
                // (pending == 0) or for a cancel
                unsigned long long pos = 0;
                if (lane == 0) pos = atomicAdd(&ctl->head, 1ull);
                pos = __shfl_sync(FULL, pos, 0);
                unsigned long long* sq = a.seq + (pos & a.ring_mask);
                uint32_t sleep = 32;
                int outcome = 0;  // 1 got, 2 done
                for (uint32_t spin = 0;; ++spin) {
                    int o = 0;
                    if (lane == 0) {
                        if (ld_acquire_u64(sq) == pos + 1) o = 1;
                        else if ((spin & 7) == 7) {
                            if (ld_volatile_v4(ctl).y) o = 2;
                            else if ((ld_relaxed_u64(&ctl->work) >> 32) == 0) o = 2;
                            else if (worker == 0 && a.mailbox) poll_mailbox(a, ctl);
                        }
                    }
                    outcome = __shfl_sync(FULL, o, 0);
                    if (outcome) break;
                    __nanosleep(sleep);
                    sleep = min(sleep * 2, a.backoff_ns);
                }
                if (outcome == 2) {
                    if (INSTR) st.phase[PH_WL_REMOVE] += clock64() - t0;
                    break;
                }
                (void)ld_acquire_u64(sq);  // every lane acquires the publication before reading
                x.template load<true>(a.wl + (pos & a.ring_mask) * a.entry_bytes);
                __threadfence();
                __syncwarp();
                if (lane == 0) {
                    st_release_u64(sq, pos + a.ring_mask + 1);  // free for the next lap
                    atomicAdd(&ctl->work, ~0ull);                // size - 1 (pending unchanged)
                }
                idle = false;
                have = true;
                if (INSTR) st.phase[PH_WL_REMOVE] += clock64() - t0;
            }
        }

        // Issue the read of the hot control line ({best, cancel} + queue size) now and consume
        // it after the reduction, so its L2 latency hides behind the rule passes. The rules use
        // the bound seen at the previous node (a stale, larger bound only prunes less).
        uint32_t h_best = 0, h_cancel = 0;
        unsigned long long h_size = 0;
        if (lane == 0) {
            const uint4 h = ld_volatile_v4(ctl);
            h_best = h.x;
            h_cancel = h.y;
            h_size = (uint32_t)ld_relaxed_u64(&ctl->work);
        }

        // visit_and_check_limits (scheduler.cpp:63-74), batched: one atomic per flush_every visits
        ++st.nodes;
        if (st.nodes - nodes_flushed >= a.flush_every) {
            int stop = 0;
            if (lane == 0) {
                unsigned long long tot = atomicAdd(&ctl->nodes_total, st.nodes - nodes_flushed) +
                                         (st.nodes - nodes_flushed);
                if (a.node_budget && tot > a.node_budget) stop = 2;
                else if (a.timeout_ns && globaltimer() - t_start >= a.timeout_ns) stop = 1;
                if (stop) {
                    atomicCAS(&ctl->status, 0, stop);
                    atomicExch(&ctl->cancel, 1u);
                }
                if (worker == 0 && a.mailbox) poll_mailbox(a, ctl);
            }
            nodes_flushed = st.nodes;
            if (__shfl_sync(FULL, stop, 0)) break;
        }

        // process_node (scheduler.cpp:125-144)
        x.reduce(a.pvc, a.k, best, st);
        if (__shfl_sync(FULL, h_cancel, 0)) break;
        if (!a.pvc) best = min(best, __shfl_sync(FULL, h_best, 0));
        const unsigned long long qsize = __shfl_sync(FULL, h_size, 0);
        long long tp = INSTR ? clock64() : 0;
        const bool prune = x.doom || should_prune(a.pvc, a.k, best, x.cc, x.edges);
        if (INSTR) st.phase[PH_PRUNE] += clock64() - tp;
        st.dooms += x.doom;
        if (prune) {
            have = false;
            continue;
        }
        if (x.edges == 0) {
            // record_cover (scheduler.cpp:84-108)
            uint32_t* slot = a.cover_slots + (unsigned long long)worker * W;
            uint32_t record = 0;
            if (lane == 0) {
                if (a.pvc) record = atomicCAS(&ctl->found, 0u, 1u) == 0u;
                else record = x.cc < atomicMin(&ctl->best, x.cc);
            }
            record = __shfl_sync(FULL, record, 0);
            if (record) {
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    uint32_t b = __ballot_sync(FULL, x.d[i] == REM);
                    b = i < last_word ? b : (i == last_word ? (b & last_word_mask) : 0u);
                    if (lane == i) slot[i] = b;
                }
                __threadfence();
                __syncwarp();
                if (lane == 0) {
                    atomicMin(&ctl->best_owner, ((unsigned long long)x.cc << 32) | worker);
                    if (a.pvc) atomicExch(&ctl->cancel, 1u);
                    if (a.mailbox) {
                        a.mailbox[2] = x.cc;
                        if (a.pvc) a.mailbox[3] = 1;
                    }
                }
            }
            if (a.pvc) break;  // the search is ended (solver_seq.cpp:108)
            best = min(best, x.cc);
            have = false;
            continue;
        }
        long long tm = INSTR ? clock64() : 0;
        const uint32_t v = x.argmax();
        ++st.maxdeg;
        if (INSTR) st.phase[PH_MAXDEG] += clock64() - tm;

        // Branch (scheduler.cpp:185-203): defer remove-N(v) — donated while the worklist is
        // below its threshold (optionally the oldest stacked node goes instead) — and continue
        // with remove-v.
        long long tb = INSTR ? clock64() : 0;
        bool child_placed = false;
        if (!a.seq_mode && qsize < a.threshold) {
            unsigned long long pos = 0, seen = 0;
            int ok = 0;
            if (lane == 0) ok = q_reserve(a, pos, seen);
            ok = __shfl_sync(FULL, ok, 0);
            if (ok) {
                pos = __shfl_sync(FULL, pos, 0);
                if (lane == 0) {
                    st.max_queue = max(st.max_queue, seen);
                    // the slot is free once the previous lap's reader released it
                    while (ld_acquire_u64(a.seq + (pos & a.ring_mask)) != pos) __nanosleep(32);
                }
                __syncwarp();
                unsigned char* dst = a.wl + (pos & a.ring_mask) * a.entry_bytes;
                if (a.donate_oldest && sp > 0) {
                    x.copy_record(slot_at(0), dst);
                    base = base + 1 == a.stack_bound ? 0 : base + 1;
                    --sp;
                } else {
                    x.write_child_without_neighbors(v, dst);
                    child_placed = true;
                }
                __threadfence();
                __syncwarp();
                if (lane == 0) st_release_u64(a.seq + (pos & a.ring_mask), pos + 1);
                ++st.donated;
                if (INSTR) st.phase[PH_WL_ADD] += clock64() - tb;
            }
        }
        if (!child_placed) {
            long long ts = INSTR ? clock64() : 0;
            x.write_child_without_neighbors(v, slot_at(sp));
            ++sp;
            if (sp > st.high_water) st.high_water = sp;
            if (INSTR) st.phase[PH_BRANCH_NBRS] += clock64() - ts;
        }
        ++st.children;
        long long tv = INSTR ? clock64() : 0;
        x.remove_vertex(v);
        if (INSTR) st.phase[PH_BRANCH_V] += clock64() - tv;
    }

    if (lane == 0) {
        if (st.nodes > nodes_flushed) atomicAdd(&ctl->nodes_total, st.nodes - nodes_flushed);
        WStats o;
        o.nodes = st.nodes;
        o.rounds = st.rounds;
        o.maxdeg = st.maxdeg;
        o.children = st.children;
        o.rm1 = st.rm1;
        o.rm2 = st.rm2;
        o.rmh = st.rmh;
        o.dooms = st.dooms;
        o.high_water = st.high_water;
        o.donated = st.donated;
        o.active = clock64() - c_start;
        o.max_queue = st.max_queue;
#pragma unroll
        for (int p = 0; p < 10; ++p) o.phase[p] = st.phase[p];
        a.stats[worker] = o;
        (void)t_start;
    }
}

// Level-synchronous frontier expansion (multi-GPU partitioning): warp i
// processes node i of a level exactly as process_node does (scheduler.cpp:125-144) with a
// FIXED bound, and writes its remove-N(v) child to out[2i] and its remove-v child to
// out[2i+1]. The result does not depend on scheduling, so every rank derives the same frontier.
struct ExpandArgs {
    const uint4* at4;
    uint32_t n, npad;
    int pvc;
    uint32_t k, best;
    uint32_t count;
    unsigned long long entry_bytes;
    const unsigned char* in;
    unsigned char* out;
    uint32_t* flags;   // per input: 0 pruned, 1 cover found (cc in covers[i*(W+1)]), 2 branched
    uint32_t* covers;  // per input: [cc, bitmap W words]
};

template <int W>
__global__ void __launch_bounds__(256) expand_kernel(ExpandArgs a) {
    extern __shared__ uint4 sat[];
    constexpr int Q = W / 4;
    const int lane = threadIdx.x & 31;
    for (uint32_t t = threadIdx.x; t < Q * a.npad; t += blockDim.x) sat[t] = a.at4[t];
    __syncthreads();
    const uint32_t warps = gridDim.x * (blockDim.x >> 5);
    const uint32_t last_word_mask = (a.n & 31) ? ((1u << (a.n & 31)) - 1u) : FULL;
    const int last_word = (int)((a.n + 31) / 32) - 1;
    WarpNode<W, false> x;
    x.sat = sat;
    x.npad = a.npad;
    x.lane = lane;
    Counters st;
    for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < a.count; i += warps) {
        x.template load<false>(a.in + (unsigned long long)i * a.entry_bytes);
        x.reduce(a.pvc, a.k, a.best, st);
        uint32_t flag;
        if (x.doom || should_prune(a.pvc, a.k, a.best, x.cc, x.edges)) {
            flag = 0;
        } else if (x.edges == 0) {
            flag = 1;
            uint32_t* c = a.covers + (unsigned long long)i * (W + 1);
#pragma unroll
            for (int j = 0; j < W; ++j) {
                uint32_t b = __ballot_sync(FULL, x.d[j] == REM);
                b = j < last_word ? b : (j == last_word ? (b & last_word_mask) : 0u);
                if (lane == j) c[1 + j] = b;
            }
            if (lane == 0) c[0] = x.cc;
        } else {
            flag = 2;
            const uint32_t v = x.argmax();
            x.write_child_without_neighbors(v, a.out + (2ull * i) * a.entry_bytes);
            x.remove_vertex(v);
            x.store_current(a.out + (2ull * i + 1) * a.entry_bytes);
        }
        if (lane == 0) a.flags[i] = flag;
    }
}

// ------------------------------------------------------------------ host side

struct DeviceGraph {
    int device = -1;
    uint32_t W = 0, npad = 0;
    uint4* at4 = nullptr;
    size_t at4_bytes = 0;
    ~DeviceGraph() {
        if (at4) cudaFree(at4);
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
struct DeviceCtx {
    Arena stacks, wl, seq, misc;
    cudaStream_t stream = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    int sms = 0;
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

// Pack one node record: [cc, edges, 0, 0] + lane-major u16 degrees.
void pack_record(uint32_t W, uint32_t n, uint32_t cc, uint32_t edges, const uint32_t* deg,
                 unsigned char* rec) {
    std::memset(rec, 0, 16 + 64 * (size_t)W);
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

template <int W, bool INSTR>
void launch_dense(const DenseArgs& a, uint32_t grid, uint32_t block, size_t smem, cudaStream_t s) {
    auto k = dense_kernel<W, INSTR>;
    CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<grid, block, smem, s>>>(a);
    CUDA_CHECK(cudaGetLastError());
}

template <int W>
int occupancy(uint32_t block, size_t smem, bool instr) {
    int nb = 0;
    auto k = instr ? dense_kernel<W, true> : dense_kernel<W, false>;
    CUDA_CHECK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, (int)block, smem));
    return nb;
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

void solve_on_device(const Graph& g, const SolveSpec& s, SolveOut& out) {
    if (g.n > 1024)
        throw std::invalid_argument("graph has " + std::to_string(g.n) +
                                    " vertices; the dense engine handles n <= 1024");
    const int dev = s.device;
    int ndev = device_count();
    if (ndev == 0) throw std::runtime_error("CUDA error: no CUDA device visible");
    if (dev < 0 || dev >= ndev) throw std::invalid_argument("device ordinal out of range");
    CUDA_CHECK(cudaSetDevice(dev));
    DeviceCtx& C = ctx_for(dev);
    cudaStream_t st = s.stream ? static_cast<cudaStream_t>(s.stream) : C.stream;

    const uint32_t W = pick_w(g.n);
    const uint32_t npad = 32 * W;
    const size_t entry = 16 + 64 * (size_t)W;
    out.engine = 1;
    out.degree_bytes = 2;
    out.n_padded = npad;

    auto th0 = std::chrono::steady_clock::now();
    // resident graph (adjacency bitmap), uploaded once per device
    if ((int)g.dev.size() <= dev) g.dev.resize(dev + 1);
    if (!g.dev[dev]) {
        auto dg = std::make_shared<DeviceGraph>();
        dg->device = dev;
        dg->W = W;
        dg->npad = npad;
        std::vector<uint32_t> at = build_bitmap(g, W, npad);
        dg->at4_bytes = at.size() * 4;
        CUDA_CHECK(cudaMalloc(&dg->at4, dg->at4_bytes));
        CUDA_CHECK(cudaMemcpyAsync(dg->at4, at.data(), dg->at4_bytes, cudaMemcpyHostToDevice, st));
        out.h2d_bytes += dg->at4_bytes;
        g.dev[dev] = dg;
    }
    const DeviceGraph& dg = *g.dev[dev];

    // worker grid: one warp per worker
    const uint32_t block_warps = s.block_warps ? std::min<uint32_t>(s.block_warps, 8) : 8;
    const uint32_t block = 32 * block_warps;
    const size_t smem = (size_t)W * npad * 4;
    int per_sm = 1;
    switch (W) {
        case 4: per_sm = occupancy<4>(block, smem, s.instrument); break;
        case 8: per_sm = occupancy<8>(block, smem, s.instrument); break;
        case 16: per_sm = occupancy<16>(block, smem, s.instrument); break;
        default: per_sm = occupancy<32>(block, smem, s.instrument); break;
    }
    if (per_sm < 1) throw std::runtime_error("CUDA error: dense kernel cannot be resident");
    uint32_t workers = s.workers;
    if (s.strategy == 1) workers = 1;
    if (workers == 0) workers = (uint32_t)C.sms * per_sm * block_warps;
    const uint32_t grid = (workers + block_warps - 1) / block_warps;
    out.grid = grid;
    out.block = block;

    // memory: stacks, worklist ring, control, cover slots, stats
    const uint32_t bound = std::max<uint32_t>(s.stack_bound, 1) + 1;
    const uint64_t cap = std::max<uint64_t>(std::max<uint64_t>(s.capacity, s.num_seeds), 1);
    if (cap > (1ull << 30)) throw std::invalid_argument("worklist capacity too large");
    uint64_t ring = 2;
    while (ring < cap) ring <<= 1;
    const size_t stack_bytes = (size_t)workers * bound * entry;
    const size_t wl_bytes = (size_t)ring * entry;
    unsigned char* stacks = (unsigned char*)C.stacks.get(stack_bytes);
    unsigned char* wl = (unsigned char*)C.wl.get(wl_bytes);
    unsigned long long* seq = (unsigned long long*)C.seq.get(ring * 8);
    const size_t slots_bytes = (((size_t)workers * W * 4) + 255) / 256 * 256;
    const size_t misc_bytes = sizeof(Ctl) + slots_bytes + (size_t)workers * sizeof(WStats);
    unsigned char* misc = (unsigned char*)C.misc.get(misc_bytes);
    Ctl* ctl = reinterpret_cast<Ctl*>(misc);
    uint32_t* cover_slots = reinterpret_cast<uint32_t*>(misc + sizeof(Ctl));
    WStats* stats = reinterpret_cast<WStats*>(misc + sizeof(Ctl) + slots_bytes);

    // initial worklist content: the root (init_root, search_node.cpp:7-14) or the seeds
    const uint64_t nseeds = s.num_seeds ? s.num_seeds : 1;
    std::vector<unsigned char> recs(nseeds * entry);
    if (s.num_seeds) {
        for (uint64_t i = 0; i < nseeds; ++i) {
            const uint32_t* r = s.seeds + i * (2 + (size_t)g.n);
            pack_record(W, g.n, r[0], r[1], r + 2, recs.data() + i * entry);
        }
    } else {
        std::vector<uint32_t> deg(g.n);
        for (uint32_t v = 0; v < g.n; ++v) deg[v] = g.degree(v);
        pack_record(W, g.n, 0, (uint32_t)g.m, deg.data(), recs.data());
    }
    Ctl hc;
    std::memset(&hc, 0, sizeof(hc));
    hc.best = s.best;
    hc.head = 0;
    hc.tail = nseeds;
    hc.work = (nseeds << 32) | nseeds;
    hc.best_owner = ~0ull;
    CUDA_CHECK(cudaMemcpyAsync(ctl, &hc, sizeof(hc), cudaMemcpyHostToDevice, st));
    CUDA_CHECK(cudaMemcpyAsync(wl, recs.data(), recs.size(), cudaMemcpyHostToDevice, st));
    init_seq_kernel<<<64, 256, 0, st>>>(seq, (uint32_t)ring, (uint32_t)nseeds);
    CUDA_CHECK(cudaGetLastError());
    out.launches += 2;  // init_seq_kernel + dense_kernel
    CUDA_CHECK(cudaMemsetAsync(stats, 0, (size_t)workers * sizeof(WStats), st));
    out.h2d_bytes += sizeof(hc) + recs.size();
    CUDA_CHECK(cudaStreamSynchronize(st));
    out.h2d_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - th0).count();

    DenseArgs a;
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
    a.flush_every = 64;
    if (s.node_budget) a.flush_every = std::max<uint64_t>(1, std::min<uint64_t>(64, s.node_budget / (4ull * workers)));
    // idle back-off: exponential from 32 ns, capped at backoff_us (at most 2 us on the device —
    // a polling warp costs one L2 read, an over-sleeping one leaves queued work unclaimed)
    a.backoff_ns = (uint32_t)std::min<uint64_t>(std::max<uint64_t>(s.backoff_us * 1000, 64), 2000);
    a.seq_mode = s.strategy == 1 ? 1 : 0;
    a.donate_oldest = s.donate_oldest ? 1 : 0;
    a.mailbox = s.mailbox;

    CUDA_CHECK(cudaEventRecord(C.ev0, st));
    const bool I = s.instrument;
    switch (W) {
        case 4: I ? launch_dense<4, true>(a, grid, block, smem, st) : launch_dense<4, false>(a, grid, block, smem, st); break;
        case 8: I ? launch_dense<8, true>(a, grid, block, smem, st) : launch_dense<8, false>(a, grid, block, smem, st); break;
        case 16: I ? launch_dense<16, true>(a, grid, block, smem, st) : launch_dense<16, false>(a, grid, block, smem, st); break;
        default: I ? launch_dense<32, true>(a, grid, block, smem, st) : launch_dense<32, false>(a, grid, block, smem, st); break;
    }
    CUDA_CHECK(cudaEventRecord(C.ev1, st));
    CUDA_CHECK(cudaStreamSynchronize(st));
    float ms = 0;
    CUDA_CHECK(cudaEventElapsedTime(&ms, C.ev0, C.ev1));
    out.device_ms = ms;

    // readback
    CUDA_CHECK(cudaMemcpy(&hc, ctl, sizeof(hc), cudaMemcpyDeviceToHost));
    std::vector<WStats> hs(workers);
    CUDA_CHECK(cudaMemcpy(hs.data(), stats, workers * sizeof(WStats), cudaMemcpyDeviceToHost));
    out.d2h_bytes += sizeof(hc) + workers * sizeof(WStats);
    out.status = hc.status;
    out.wl_added = hc.tail;  // every enqueue ticket is one added node (root/seeds included)
    out.wl_current = (uint32_t)hc.work;
    out.wl_removed = hc.tail - out.wl_current;
    out.wl_max_size = nseeds;
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
        out.wl_max_size = std::max<uint64_t>(out.wl_max_size, hs[w].max_queue);
        for (int p = 0; p < 10; ++p) out.phase[p] += hs[w].phase[p];
    }
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

void expand_frontier(const Graph& g, const SolveSpec& s, uint64_t target, Frontier& f) {
    if (g.n > 1024)
        throw std::invalid_argument("frontier expansion needs the dense engine (n <= 1024)");
    const int dev = s.device;
    if (device_count() == 0) throw std::runtime_error("CUDA error: no CUDA device visible");
    CUDA_CHECK(cudaSetDevice(dev));
    DeviceCtx& C = ctx_for(dev);
    cudaStream_t st = s.stream ? static_cast<cudaStream_t>(s.stream) : C.stream;
    const uint32_t W = pick_w(g.n);
    const uint32_t npad = 32 * W;
    const size_t entry = 16 + 64 * (size_t)W;
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
    const size_t smem = (size_t)W * npad * 4;

    // level 0: the root
    std::vector<unsigned char> level(entry);
    {
        std::vector<uint32_t> deg(g.n);
        for (uint32_t v = 0; v < g.n; ++v) deg[v] = g.degree(v);
        pack_record(W, g.n, 0, (uint32_t)g.m, deg.data(), level.data());
    }
    uint64_t count = 1;
    f = Frontier();
    f.best = s.best;
    while (count > 0 && count < target) {
        unsigned char *din = nullptr, *dout = nullptr;
        uint32_t *dflags = nullptr, *dcov = nullptr;
        CUDA_CHECK(cudaMalloc(&din, count * entry));
        CUDA_CHECK(cudaMalloc(&dout, 2 * count * entry));
        CUDA_CHECK(cudaMalloc(&dflags, count * 4));
        CUDA_CHECK(cudaMalloc(&dcov, count * (W + 1) * 4));
        CUDA_CHECK(cudaMemcpyAsync(din, level.data(), count * entry, cudaMemcpyHostToDevice, st));
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
        std::vector<uint32_t> flags(count), covers(count * (W + 1));
        std::vector<unsigned char> out(2 * count * entry);
        CUDA_CHECK(cudaMemcpyAsync(flags.data(), dflags, count * 4, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaMemcpyAsync(covers.data(), dcov, covers.size() * 4, cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaMemcpyAsync(out.data(), dout, out.size(), cudaMemcpyDeviceToHost, st));
        CUDA_CHECK(cudaStreamSynchronize(st));
        cudaFree(din);
        cudaFree(dout);
        cudaFree(dflags);
        cudaFree(dcov);
        f.nodes += count;
        ++f.levels;
        // covers found on this level (fixed bound inside the level, improved between levels)
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
        if (s.pvc && f.found) {
            count = 0;
            level.clear();
            break;
        }
        std::vector<unsigned char> next;
        next.reserve(2 * count * entry);
        uint64_t nc = 0;
        for (uint64_t i = 0; i < count; ++i) {
            if (flags[i] != 2) continue;
            next.insert(next.end(), out.begin() + (2 * i) * entry, out.begin() + (2 * i + 2) * entry);
            nc += 2;
        }
        level.swap(next);
        count = nc;
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
