// dense_kernels.cuh — device code of the dense engine (n <= 1024): the warp-per-node hybrid
// traversal kernel and the level-synchronous frontier expansion kernel.
//
// Reference path replaced: run_hybrid (proj/src/scheduler.cpp:328-359) — hybrid_worker
// (:146-212), process_node (:125-144) — reduce_to_fixpoint and the three rule passes
// (reductions.cpp:7-104), should_prune (bounds.cpp:21-30), max_degree_vertex and
// remove_*_into_cover (search_node.cpp:16-46), GlobalWorklist (worklist.cpp:11-48).
//
// Layout:
//  * one WARP = one worker. A node is WIDE (WarpNode: lane l owns vertices 32*i + l, i < W; the
//    u32 degrees in the warp's shared-memory slots, alive / verdict bits in registers) until at
//    most 64 vertices are alive, then COMPACT (CompactNode: the alive vertices renumbered in id
//    order, each lane holding the induced 64-bit adjacency rows and degrees of its two slots in
//    registers, warp-uniform 64-bit candidate masks). 97% of C5's visits are compact.
//  * the read-only graph is an adjacency bitmap staged once per CTA in shared memory, word j of
//    vertex w's row at uint4 group (j/4)*npad + w (column-coalesced, row-broadcast);
//  * deferred nodes are records {cover_count, edge_count, kind, 0} + a wide body (lane-major
//    u16 degrees and one word per lane of cached degree-two non-triangle verdicts) or a compact
//    body (alive / verdict masks, induced rows, slot ids); they live in a per-warp ring stack
//    in HBM (L2-resident top) or in the device worklist ring.
//  * both layouts run the same reduce_node: the reference's rule order, bit for bit.
//
// Instruction footprint matters here: with the rule code inlined at every call site the wide
// W=16 kernel was 128 KB of SASS and 64% of warp stalls were `no_instruction`. Every primitive
// therefore has one call site per layout, the three rule passes share one rolled loop, cold
// paths (cover recording, peer donation, cancel broadcast, slot waits) are out of line, and the
// multi-shard and one-worker (seq / StackOnly) variants are separate instantiations.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <type_traits>

namespace vcg {

constexpr uint32_t REM = 0xFFFFFFFFu;
constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr unsigned long long ONE_PENDING = 1ull << 32;

// ------------------------------------------------------------------ device-global state

#ifndef VCG_SPLIT_TICKETS
#define VCG_SPLIT_TICKETS 1
#endif
#ifndef VCG_SPLIT_WORK
#define VCG_SPLIT_WORK 0
#endif
struct Ctl {
    // line 0: read by every worker once per node (one vector load + one scalar load)
    uint32_t best;    // MVC bound (atomicMin); PVC: k
    uint32_t cancel;  // 1 = stop: PVC found, timeout, budget, host request
#if !VCG_SPLIT_WORK
    // (pending << 32) | size: pending = queued items + active workers (termination at 0);
    // size = queued items + in-flight enqueue reservations (threshold gate, capacity).
    // {best, cancel, work} are the first 16 bytes: the dense workers' poll copies them to
    // shared memory with one cp.async.
    unsigned long long work;
    uint32_t found;   // PVC: a cover of size <= k was recorded
    uint32_t pad0;
    unsigned long long pad1;
    uint32_t pad2[24];
#else
    uint32_t found;
    uint32_t pad0;
    uint32_t pad2[28];
    // line 0b: the packed worklist word on its own line (its atomics do not contend with the
    // reads of the bound / cancel words)
    unsigned long long work;
    uint32_t pad7[30];
#endif
    // line 1: the consumers' ring ticket (per-slot sequence numbers publish / free each slot)
    unsigned long long head;
    // shard 0 only (multi-shard solves): number of shards whose `pending` is non-zero; the
    // whole solve is done when it reaches zero
    uint32_t gactive;
    uint32_t pad3[29];
#if VCG_SPLIT_TICKETS
    // line 2: the producers' ticket, on its own line (producers and consumers do not contend
    // on one L2 line)
    unsigned long long tail;
    uint32_t pad5[30];
#endif
    // results
    unsigned long long nodes_total, best_owner;
    int32_t status;
    uint32_t pad4[27];
#if !VCG_SPLIT_TICKETS
    unsigned long long tail;
    uint32_t pad6[30];
#endif
};
static_assert(sizeof(Ctl) == (VCG_SPLIT_WORK ? 640 : 512), "Ctl layout");

// A peer shard's exchange memory (another GPU over NVLink P2P / CUDA IPC, or another shard on
// this device): its control block, ring slots and slot sequence numbers.
struct PeerRef {
    Ctl* ctl;
    unsigned char* wl;
    unsigned long long* seq;
};

struct WStats {
    unsigned long long nodes, rounds, maxdeg, children, rm1, rm2, rmh, high_water, donated,
        active, max_queue, dooms, peer;
    unsigned long long phase[10];
    // timeline (globaltimer ns): kernel start, first node taken, exit — the ramp-up and tail of
    // the search (dense engine)
    unsigned long long t_begin, t_first, t_end;
    unsigned long long t_idle;      // ns waiting for a worklist node
    unsigned long long t_lastwait;  // start of the last wait (from then on: the tail)
};

enum Phase { PH_WL_REMOVE, PH_WL_ADD, PH_STACK, PH_DEG1, PH_DEG2, PH_HIGH, PH_MAXDEG,
             PH_BRANCH_NBRS, PH_BRANCH_V, PH_PRUNE };  // metrics.hpp:15-26 order

struct DenseArgs {
    const uint4* at4;         // adjacency bitmap, [W/4][npad] uint4 groups
    uint32_t n, npad, m;
    int pvc;
    uint32_t k;
    uint32_t capacity;        // logical worklist capacity (try_add rejects at capacity)
    uint32_t ring_mask;       // ring slots - 1 (power of two >= max(capacity, 2))
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
    int donate_oldest;        // donate the bottom (oldest) stacked node instead of the new child
    int compact;              // renumber nodes with <= 64 alive vertices (CompactNode)
    int mid;                  // (W >= 16) renumber nodes with <= 128 alive vertices into a
                              // per-warp frame (the mid layout, WarpNode<4, ., W>)
    int stackonly;            // StackOnly strategy (scheduler.cpp:214-297): claim sub-tree ids
    uint32_t depth;           // StackOnly sub-tree depth (2^depth sub-trees)
    volatile uint32_t* mailbox;  // host-mapped: [0] ext best in, [1] cancel in, [2] best out,
                                 // [3] found out
    // multi-shard solves (world > 1): every shard's exchange memory, this shard's index
    const PeerRef* peers;
    uint32_t world, rank;
};

// ------------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint4 ld_volatile_v4(const void* p) {
    uint4 r;
    asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}
__device__ __forceinline__ uint2 ld_volatile_v2(const void* p) {
    uint2 r;
    asm volatile("ld.volatile.global.v2.u32 {%0,%1}, [%2];" : "=r"(r.x), "=r"(r.y) : "l"(p));
    return r;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const void* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// system scope: ring publications and control words shared with other GPUs
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
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
    const uint32_t spend = cc + 1;
    return best <= spend ? 0u : best - spend;
}
// should_prune (bounds.cpp:21-30)
__device__ __forceinline__ bool should_prune(int pvc, uint32_t k, uint32_t best, uint32_t cc,
                                             uint32_t edges) {
    if (pvc) {
        if (cc > k) return true;
        const unsigned long long s = k - cc;
        return (unsigned long long)edges > s * s;
    }
    if (cc >= best) return true;
    const unsigned long long s = best - cc - 1;
    return (unsigned long long)edges > s * s;
}

// The bound B of a search: a node is pruned once |S| > B (PVC: B = k; MVC: B = best - 1), and
// ReductionBound::current (reductions.hpp:19-27) and should_prune (bounds.cpp:21-30) are both
// functions of B - |S| alone — one code path for both modes, no per-node mode branches.
__device__ __forceinline__ int bound_of(int pvc, uint32_t k, uint32_t best) {
    return pvc ? (int)k : (int)best - 1;
}
__device__ __forceinline__ uint32_t limit_of(int B, uint32_t cc) {
    return B > (int)cc ? (uint32_t)(B - (int)cc) : 0u;
}
__device__ __forceinline__ bool prune_at(int B, uint32_t cc, uint32_t edges) {
    if ((int)cc > B) return true;
    const unsigned long long s = (uint32_t)(B - (int)cc);
    return (unsigned long long)edges > s * s;
}

// Host mailbox (pinned, mapped): one poller per device (worker 0) folds an external MVC bound
// into the device bound and turns a host cancel request into the device cancel flag.
__device__ __noinline__ void poll_mailbox(volatile uint32_t* mb, int pvc, Ctl* ctl) {
    const uint32_t eb = mb[0];
    if (!pvc && eb) atomicMin(&ctl->best, eb);
    if (mb[1]) atomicExch(&ctl->cancel, 1u);
}

template <class T>
struct CountersT {
    T nodes = 0, rounds = 0, maxdeg = 0, children = 0, rm1 = 0, rm2 = 0, rmh = 0, donated = 0,
      dooms = 0, peer = 0;
    T high_water = 0, max_queue = 0;  // maxima
    unsigned long long phase[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
};
using Counters = CountersT<unsigned long long>;
// The dense worker keeps 32-bit deltas (half the registers) and folds them into its WStats
// slot at every flush (at most every 64 nodes, so no delta can overflow).
using Counters32 = CountersT<uint32_t>;
__device__ __forceinline__ void fold_stats(WStats* o, Counters32& st) {
    o->nodes += st.nodes;
    o->rounds += st.rounds;
    o->maxdeg += st.maxdeg;
    o->children += st.children;
    o->rm1 += st.rm1;
    o->rm2 += st.rm2;
    o->rmh += st.rmh;
    o->donated += st.donated;
    o->dooms += st.dooms;
    o->peer += st.peer;
}
__device__ __forceinline__ void reset_deltas(Counters32& st) {
    st.nodes = st.rounds = st.maxdeg = st.children = st.rm1 = st.rm2 = st.rmh = st.donated =
        st.dooms = st.peer = 0;
}

// ------------------------------------------------------------------ one search node per warp

// Cover count of a stacked marker standing for a child proven pruned at birth.
constexpr uint32_t DEAD_NODE = 0xFFFFFFFFu;
// Record kinds (header word 2): wide (WarpNode layout) or compact (CompactNode layout).
constexpr uint32_t REC_WIDE = 0, REC_COMPACT = 1, REC_MID = 2;

#ifndef VCG_POLL_EVERY
#define VCG_POLL_EVERY 32  // nodes between reads of the control line (power of two; C5: 4 → 12.3 ms,
                           // 8 → 10.1, 16 → 9.4, 32 → 9.0, 64 → 9.4)
#endif
constexpr uint32_t kPoll = VCG_POLL_EVERY;
#ifndef VCG_CHILD_DMAX
#define VCG_CHILD_DMAX 0  // skip the child doom test's bookkeeping when max degree <= limit (C5: 10.3 -> 11.3 ms, C2 unchanged: off)
#endif
#ifndef VCG_TIMELINE
#define VCG_TIMELINE 1    // per-warp first-node time (the timeline's ramp-up)
#endif
#ifndef VCG_EXPECT
#define VCG_EXPECT 0  // branch-likelihood hints in the node loop (C5 neutral, mid-heavy graphs 6% slower: off)
#endif
#if VCG_EXPECT
#define VCG_LIKELY(x) __builtin_expect(!!(x), 1)
#define VCG_UNLIKELY(x) __builtin_expect(!!(x), 0)
#else
#define VCG_LIKELY(x) (x)
#define VCG_UNLIKELY(x) (x)
#endif
#ifndef VCG_TEST_GPU_ACQ
#define VCG_TEST_GPU_ACQ 0  // A/B only (unsound across GPUs): gpu-scope acquires in the shard kernel
#endif
#ifndef VCG_WIDE_SMEM
#define VCG_WIDE_SMEM 1   // wide degrees in shared memory (fewer registers) instead of registers
#endif
#ifndef VCG_FROM_WIDE_BALLOT
#define VCG_FROM_WIDE_BALLOT 1  // compact conversion: rows by ballots over slots (see from_wide)
#endif
#ifndef VCG_RELAXED_FREE
#define VCG_RELAXED_FREE 0  // A/B only: the slot-free signal as a relaxed store (the slot's values
                            // are consumed before it, but the PTX model does not order them)
#endif
#ifndef VCG_POLL_SMEM
#define VCG_POLL_SMEM 0  // (W >= 16) the control-line poll lands in shared memory by cp.async:
                         // no registers across the reduction (C5 kernel spills 36 -> 4 B) but
                         // measured C5 equal, C5-scale 2% slower than register polls: off
#endif
#ifndef VCG_CNT_SMEM
#define VCG_CNT_SMEM 1  // (W >= 16) per-branch counters in the warp's shared slot, not registers
#endif
#ifndef VCG_CHILD_UNROLL
#define VCG_CHILD_UNROLL 1  // vertex words per iteration of write_child's popcount loop
#endif
constexpr int kChildUnroll = VCG_CHILD_UNROLL;

// Dynamic shared memory of the dense kernels (BW warps per CTA): the adjacency bitmap
// ([W/4][32W] uint4 groups), then a W-word slot per warp, then per warp W x 32 scratch words,
// then per warp its degree / frame words.
extern __shared__ uint4 dense_smem[];
template <int W, int BW = 8>
__device__ __forceinline__ uint32_t dense_scratch_base(uint32_t wib) {
    return (W / 4) * (32 * W) * 4 + BW * W + wib * W * 32;
}
// (VCG_WIDE_SMEM) per-warp degree words after the scratch words of 8 warps; with a mid layout
// of width MW the region also holds the warp's frame bitmap ([MW/4][32 MW] uint4), which
// overlays the wide degrees (a warp holds one current node).
__host__ __device__ constexpr uint32_t dense_degree_words(int W, int MW) {
    return (uint32_t)W * 32 > (uint32_t)(MW / 4) * (32 * MW) * 4 ? (uint32_t)W * 32
                                                                  : (uint32_t)(MW / 4) * (32 * MW) * 4;
}
// the mid width of the default instantiation: 4 (<= 128 alive) where the graph is >= 16 words
__host__ __device__ constexpr int default_mid(int W) { return W >= 16 ? 4 : 0; }
template <int W, int MW = default_mid(W), int BW = 8>
__device__ __forceinline__ uint32_t dense_degree_base(uint32_t wib) {
    return dense_scratch_base<W, BW>(BW) + wib * dense_degree_words(W, MW);
}

// WG == 0: the WIDE layout over the whole graph (vertex v at lane v & 31, word v >> 5). WG != 0:
// the MID layout (induced, "frame" renumbering): at most 32*W alive vertices of a graph of width WG
// renumbered in id order into slots, their induced adjacency rows in a per-warp FRAME bitmap in
// shared memory, degrees in registers. Every primitive is the wide one on a W-word bitmap, so
// the same reduce_node runs on it and, slots keeping the id order, acts on the same vertices.
// (VCG_WIDE_COLD, A/B only) the wide layout's record load, child pass and child store out of
// line, to take their large bodies out of the compact hot loop's instruction footprint.
// Measured: C5 8.9 -> 10.0 ms, C5-scale -5% (the calls' register saves and restores add
// spills at the 72-register budget): off.
#ifndef VCG_WIDE_COLD
#define VCG_WIDE_COLD 0
#endif
template <class N>
__device__ __noinline__ void wide_load_cold(N& x, const unsigned char* rec) { x.load_body(rec); }
template <class N>
__device__ __noinline__ bool wide_child_pass_cold(const N& x, uint32_t xl, uint32_t xcnt, int B,
                                                  uint32_t& keep, uint32_t dmax) {
    return x.template child_pass<true>(xl, xcnt, B, keep, dmax);
}
template <class N>
__device__ __noinline__ void wide_store_child_cold(const N& x, uint32_t keepm, uint32_t xcnt,
                                                   unsigned char* rec) {
    x.store_child(keepm, xcnt, rec);
}

template <int W, bool INSTR, int WG = 0>
struct WarpNode {
    static constexpr bool kInstr = INSTR;
    static constexpr bool IND = WG != 0;
    static constexpr int kW = W;
    static constexpr int kPassUnroll = 1;  // (rolled: the wide pass body is large)
    static constexpr int Q = W / 4;  // uint4 groups per bitmap row
    // Wide degrees live in the warp's shared slots (VCG_WIDE_SMEM): the wide layout then holds
    // no degree registers, so the kernel's register budget (and with it the occupancy of the
    // compact hot path) is set by the compact layout. The mid layout keeps its W in registers.
#if VCG_WIDE_SMEM
    static constexpr bool kDegSmem = !IND;
#else
    static constexpr bool kDegSmem = false;
#endif
    uint32_t dsb;                    // u32 index of this warp's W x 32 degree words (kDegSmem)
    mutable uint32_t dr[kDegSmem ? 1 : W];  // degree of vertex 32*i + lane (!kDegSmem)
    __device__ __forceinline__ uint32_t& D(int i) const {
        if constexpr (kDegSmem) return reinterpret_cast<uint32_t*>(dense_smem)[dsb + i * 32 + lane];
        else return dr[i];
    }
    uint32_t alv;                    // bit i: vertex 32*i + lane is alive (not in the cover)
    uint32_t aw;                     // lane j < W: alive bitmap word j (vertices 32j..32j+31)
    uint32_t nt;                     // bit i: vertex 32*i + lane has degree two and was found
                                     // not to close a triangle; valid until its degree changes
    uint32_t cc, edges;              // uniform
    bool doom;                       // uniform: proven to be pruned (see reduce)
    // Shared memory is addressed through the dynamic-smem symbol with constant strides (a
    // pointer member costs a generic→shared conversion and an address rebuild per load).
    static constexpr uint32_t NPAD = 32 * W;  // bitmap columns (vertex slots)
    uint32_t ssb;                    // u32 index of this warp's W x 32 scratch words
    int lane;
    // mid layout only: the frame
    uint32_t rb;                     // uint4 index of the frame bitmap ([Q][NPAD] uint4 groups)
    uint32_t idb;                    // u16 index of the frame's slot -> vertex id table (32W)
    uint32_t tgi;                    // u64 index of this warp's current frame tag
    uint32_t ns;                     // uniform: slots of the frame

    __device__ __forceinline__ const uint4& grp(uint32_t q, uint32_t v) const {
        if constexpr (IND) return dense_smem[rb + q * NPAD + v];
        else return dense_smem[q * NPAD + v];  // row v, words 4q..4q+3
    }
    __device__ __forceinline__ uint32_t& scratch(int i) const {
        return reinterpret_cast<uint32_t*>(dense_smem)[ssb + i * 32 + lane];
    }
    __device__ __forceinline__ bool alive(int i) const { return (alv >> i) & 1u; }
    __device__ __forceinline__ uint32_t row_word(uint32_t u, uint32_t j) const {
        const uint32_t b = IND ? rb * 4 : 0u;
        return reinterpret_cast<const uint32_t*>(dense_smem)[b + ((j >> 2) * NPAD + u) * 4 + (j & 3)];
    }
    __device__ __forceinline__ void rebuild_aw() {
#pragma unroll
        for (int i = 0; i < W; ++i) {
            const uint32_t b = __ballot_sync(FULL, alive(i));
            if (lane == i) aw = b;
        }
    }
    // search_node.cpp:16-25 remove_vertex_into_cover(u), u alive: its degree is the popcount of
    // its alive row; one broadcast row load per 4 words decrements every neighbour.
    __device__ __forceinline__ void remove_vertex(uint32_t u) {
        uint32_t du = lane < W ? __popc(row_word(u, lane) & aw) : 0u;
        du = __reduce_add_sync(FULL, du);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const uint4 r = grp(q, u);
#pragma unroll
            for (int c = 0; c < 4; ++c) D(4 * q + c) -= (comp(r, c) >> lane) & 1u;
        }
        // (no verdict to invalidate: a cached non-triangle verdict is consulted only at degree
        // two, and a degree never rises, so once it leaves two the stale bit is never read)
        if (lane == (int)(u & 31)) alv &= ~(1u << (u >> 5));
        if (lane == (int)(u >> 5)) aw &= ~(1u << (u & 31));
        cc += 1;
        edges -= du;
    }
    // Candidate masks are bit-sliced: each lane builds the mask of its own candidates (bit i =
    // vertex 32*i + lane); first_in's one REDUX then picks the smallest id >= pos — exactly the
    // next vertex the reference's ascending pass would act on.
    __device__ __forceinline__ uint32_t eq_mask(uint32_t c) const {
        uint32_t m = 0;
#pragma unroll
        for (int i = 0; i < W; ++i) m |= (D(i) == c ? 1u : 0u) << i;
        return m & alv;
    }
    // Alive vertices of degree > lim: the sign of lim - d (both < 2^16) funnel-shifted into the
    // mask, two instructions per word.
    __device__ __forceinline__ uint32_t above_mask(uint32_t lim) const {
        uint32_t m = 0;
#pragma unroll
        for (int i = W - 1; i >= 0; --i) m = __funnelshift_l(lim - D(i), m, 1);
        return m & alv;
    }
    // smallest vertex id >= pos in the bit-sliced candidate mask m; -1 if none
    __device__ __forceinline__ int first_in(uint32_t m, int pos) const {
        const uint32_t pi = (uint32_t)pos >> 5;
        m &= lane >= (pos & 31) ? (FULL << pi) : (pi + 1 < 32 ? FULL << (pi + 1) : 0u);
        const uint32_t key = m ? (((uint32_t)__ffs(m) - 1u) << 5) | (uint32_t)lane : FULL;
        const uint32_t v = __reduce_min_sync(FULL, key);
        return v == FULL ? -1 : (int)v;
    }
    // The first two alive neighbours of v in id order (= CSR order; the second is -1 if absent).
    __device__ __forceinline__ void first_neighbors(uint32_t v, int& p0, int& p1) const {
        const uint32_t xl = lane < W ? (row_word(v, lane) & aw) : 0u;
        const uint32_t b = __ballot_sync(FULL, xl != 0);
        const int j0 = __ffs(b) - 1;
        const uint32_t w0 = __shfl_sync(FULL, xl, j0 & 31);
        p0 = 32 * j0 + __ffs(w0) - 1;
        const uint32_t w0b = w0 & (w0 - 1);
        const uint32_t b2 = b & ~(1u << j0);
        const int j1 = w0b ? j0 : __ffs(b2) - 1;
        const uint32_t w1 = w0b ? w0b : __shfl_sync(FULL, xl, j1 & 31);
        p1 = (w0b || b2) ? 32 * j1 + __ffs(w1) - 1 : -1;
    }
    // search_node.cpp:34-46: smallest id among alive vertices of maximum degree
    __device__ __forceinline__ uint32_t argmax() const {
        uint32_t dmax;
        return argmax(dmax);
    }
    // (and the maximum degree itself)
    __device__ __forceinline__ uint32_t argmax(uint32_t& dmax) const {
        uint32_t mx = 0;
#pragma unroll
        for (int i = 0; i < W; ++i)
            mx = max(mx, alive(i) ? ((D(i) << 11) | (2047u - (32u * i + lane))) : 0u);
        mx = __reduce_max_sync(FULL, mx);
        dmax = mx >> 11;
        return 2047u - (mx & 2047u);
    }
    // A node whose cover reaches the bound is pruned whatever the remaining rules do
    // (should_prune tests |S| first and rules only grow S), so the reduction may stop there.
    __device__ __forceinline__ bool doomed(int B) const { return doom || (int)cc > B; }

    // reduce_loop (reductions.cpp:63-90), shared with the compact node (reduce_node below).
    // Candidate masks are bit-sliced per lane (bit i = vertex 32*i + lane).
    using Mask = uint32_t;
    __device__ __forceinline__ static bool any(Mask m) { return __any_sync(FULL, m != 0); }
    __device__ __forceinline__ static uint32_t count(Mask m) {
        return __reduce_add_sync(FULL, __popc(m));
    }
    template <class Cnt>
    __device__ __forceinline__ void reduce(int B, Cnt& st);
    // candidate masks of passes 1 and 2 (alive, degree one / degree two without a cached
    // non-triangle verdict)
    __device__ __forceinline__ void deg_masks(uint32_t& m1, uint32_t& m2) const {
        m1 = m2 = 0;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            m1 |= (D(i) == 1u ? 1u : 0u) << i;
            m2 |= (D(i) == 2u ? 1u : 0u) << i;
        }
        m1 &= alv;
        m2 &= alv & ~nt;
    }
    __device__ __forceinline__ bool is_edge(uint32_t p, uint32_t q) const {
        return (row_word(p, q >> 5) >> (q & 31)) & 1u;
    }
    __device__ __forceinline__ void mark_nt(uint32_t v) {
        if (lane == (int)(v & 31)) nt |= 1u << (v >> 5);
    }
    // alive vertices (warp-uniform)
    __device__ __forceinline__ uint32_t alive_count() const {
        return __reduce_add_sync(FULL, __popc(alv));
    }

    // The remove-N(v) child (search_node.cpp:27-32 on a clone) written straight to a record:
    // d'(w) = d(w) - popc(A[w] & X) for the survivors w, X = N(v) ∩ alive, staged in shared
    // memory so the word loop stays rolled.
    // Lane j < W: word j of X = N(v) ∩ alive (the vertices the remove-N(v) child covers).
    __device__ __forceinline__ uint32_t branch_mask(uint32_t v) const {
        return lane < W ? (row_word(v, lane) & aw) : 0u;
    }
    // The child interface shared with CompactNode (see the kernel's branch step).
    struct Child {
        uint32_t xl, xcnt, keepm;
    };
    __device__ __forceinline__ void child_begin(uint32_t v, Child& c) const {
        c.xl = branch_mask(v);
        c.xcnt = __reduce_add_sync(FULL, __popc(c.xl));
    }
    template <bool TEST>
    __device__ __forceinline__ bool child_pass(Child& c, int B, uint32_t dmax) const {
        if constexpr (!IND && VCG_WIDE_COLD && TEST)
            return wide_child_pass_cold(*this, c.xl, c.xcnt, B, c.keepm, dmax);
        else
            return child_pass<TEST>(c.xl, c.xcnt, B, c.keepm, dmax);
    }
    __device__ __forceinline__ void child_store(const Child& c, unsigned char* rec) const {
        if constexpr (!IND && VCG_WIDE_COLD) wide_store_child_cold(*this, c.keepm, c.xcnt, rec);
        else store_child(c.keepm, c.xcnt, rec);
    }
    template <int WW>
    __device__ __forceinline__ uint32_t cover_word(uint32_t* sb) const {
        if constexpr (IND) return mid_cover_word(sb);
        else return cover_word();
    }
    __device__ __forceinline__ void write_child(uint32_t xl, uint32_t xcnt,
                                                unsigned char* rec) const {
        uint32_t keepm;
        (void)child_pass<false>(xl, xcnt, 0, keepm, 0u);
        store_child(keepm, xcnt, rec);
    }
    // The popcount pass of the remove-N(v) child: for every survivor w, the degree it loses,
    // |N(w) ∩ X|, parked in shared scratch; keepm = this lane's survivors.
    // With TEST, the pass also decides whether the child is pruned whatever happens when it is
    // visited — its cover already reaches the bound, or more survivors than its high-degree
    // limit stay above that limit (the doom test of reduce on the child's state; `snap` is the
    // bound it would see at best) — and stops as soon as the count passes the limit. Returns
    // true for such a dead child (scratch is then incomplete).
    template <bool TEST>
    // (dmax: the node's maximum degree — when even it is within the child's limit no survivor
    // can stay above it, and the pass skips the doom test's headroom bookkeeping)
    __device__ __forceinline__ bool child_pass(uint32_t xl, uint32_t xcnt, int B,
                                               uint32_t& keep_out, uint32_t dmax) const {
        // X in registers on every lane; xm = this lane's vertices that X removes
        uint32_t X[W];
        uint32_t xm = 0;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            X[j] = __shfl_sync(FULL, xl, j);
            xm |= ((X[j] >> lane) & 1u) << j;
        }
        const uint32_t keepm = alv & ~xm;  // survivors
        keep_out = keepm;
        uint32_t lim = 0;
        bool test = TEST;
        if (TEST) {
            const uint32_t c2 = cc + xcnt;
            if ((int)c2 > B) return true;
            lim = limit_of(B, c2);
            test = !VCG_CHILD_DMAX || dmax > lim;
            // headroom d - lim of the survivors above the child's limit (0: not a candidate);
            // such a survivor stays above iff it loses less than its headroom
            if (test)
#pragma unroll
                for (int i = 0; i < W; ++i)
                    scratch(i) = ((keepm >> i) & 1u) ? (uint32_t)max((int)(D(i) - lim), 0) : 0u;
        }
        uint32_t above = 0;
        // rolled pass over vertex words
#pragma unroll kChildUnroll
        for (int i = 0; i < W; ++i) {
            uint32_t s = 0;
            if (__any_sync(FULL, (keepm >> i) & 1u)) {
#pragma unroll
                for (int q = 0; q < Q; ++q) {  // straight-line: Q loads at constant strides
                    const uint4 c = grp(q, 32 * i + lane);
                    s += __popc(c.x & X[4 * q]) + __popc(c.y & X[4 * q + 1]) +
                         __popc(c.z & X[4 * q + 2]) + __popc(c.w & X[4 * q + 3]);
                }
            }
            if (TEST && test) {
                above += __reduce_add_sync(FULL, s < scratch(i) ? 1u : 0u);
                if (above > lim) return true;
            }
            scratch(i) = s;
        }
        return false;
    }
    __device__ __forceinline__ void store_child(uint32_t keepm, uint32_t xcnt,
                                                unsigned char* rec) const {
        if constexpr (IND) {
            uint32_t esum = 0;
#pragma unroll
            for (int i = 0; i < W; ++i) esum += ((keepm >> i) & 1u) ? D(i) - scratch(i) : 0u;
            store_mid(rec, cc + xcnt, __reduce_add_sync(FULL, esum) / 2, keepm, nt & keepm);
            return;
        }
        uint32_t packed[W / 2];
        uint32_t esum = 0;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            const bool keep = (keepm >> i) & 1u;
            const uint32_t lost = scratch(i);  // own writes: no sync needed
            const uint32_t nd = keep ? D(i) - lost : 0xFFFFu;
            esum += keep ? nd : 0u;
            if (i & 1) packed[i / 2] |= nd << 16;
            else packed[i / 2] = nd;
        }
        const uint32_t e2 = __reduce_add_sync(FULL, esum);
        if (lane == 0) *reinterpret_cast<uint4*>(rec) = make_uint4(cc + xcnt, e2 / 2, REC_WIDE, 0u);
        store_degrees(rec, packed);
        store_nt(rec, nt & keepm);  // stale bits of vertices below degree two are never read
    }
    // The cached non-triangle verdicts travel with the record (one word per lane).
    __device__ __forceinline__ void store_nt(unsigned char* rec, uint32_t m) const {
        reinterpret_cast<uint32_t*>(rec + 16 + 64 * W)[lane] = m;
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
    __device__ __forceinline__ void store_current(unsigned char* rec) const {
        if constexpr (IND) {
            store_mid(rec, cc, edges, alv, nt);
            return;
        }
        uint32_t packed[W / 2];
#pragma unroll
        for (int i = 0; i < W; ++i) {
            const uint32_t h = alive(i) ? D(i) : 0xFFFFu;
            if (i & 1) packed[i / 2] |= h << 16;
            else packed[i / 2] = h;
        }
        if (lane == 0) *reinterpret_cast<uint4*>(rec) = make_uint4(cc, edges, REC_WIDE, 0u);
        store_degrees(rec, packed);
        store_nt(rec, nt);
    }
    // Loads a record through L2 (it may come from another SM's worklist donation).
    __device__ __forceinline__ void load(const unsigned char* rec) {
        if constexpr (IND) load_mid(rec);
        else if constexpr (VCG_WIDE_COLD) wide_load_cold(*this, rec);
        else load_body(rec);
    }
    __device__ __forceinline__ void load_body(const unsigned char* rec) {
        uint32_t packed[W / 2];
        const unsigned char* p = rec + 16 + lane * (2 * W);
        if constexpr (W == 4) {
            const uint2 t = __ldcg(reinterpret_cast<const uint2*>(p));
            packed[0] = t.x;
            packed[1] = t.y;
        } else {
#pragma unroll
            for (int t = 0; t < W / 8; ++t) {
                const uint4 r = __ldcg(reinterpret_cast<const uint4*>(p) + t);
                packed[4 * t] = r.x;
                packed[4 * t + 1] = r.y;
                packed[4 * t + 2] = r.z;
                packed[4 * t + 3] = r.w;
            }
        }
        uint2 h = make_uint2(0, 0);
        if (lane == 0) h = __ldcg(reinterpret_cast<const uint2*>(rec));
        cc = __shfl_sync(FULL, h.x, 0);
        edges = __shfl_sync(FULL, h.y, 0);
        doom = false;
        nt = __ldcg(reinterpret_cast<const uint32_t*>(rec + 16 + 64 * W) + lane);
        alv = 0;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            const uint32_t x = (i & 1) ? (packed[i / 2] >> 16) : (packed[i / 2] & 0xFFFFu);
            D(i) = x;
            alv |= (x != 0xFFFFu ? 1u : 0u) << i;
        }
        rebuild_aw();
    }
    // Word `lane` (< W) of the cover bitmap; bits of padding vertices (id >= n) are set and
    // are masked by the host.
    __device__ __forceinline__ uint32_t cover_word() const {
        uint32_t mine = 0;
#pragma unroll
        for (int i = 0; i < W; ++i) {
            const uint32_t b = __ballot_sync(FULL, !alive(i));
            if (lane == i) mine = b;
        }
        return mine;
    }

    // ---- the mid layout's frame and records (IND)
    //
    // Record: {cc, edges, REC_MID, ns} {tag lo, tag hi, 0, 0} + alive words (W u32, word j =
    // slots 32j..32j+31) + per-lane cached verdicts (32 u32) + the frame's slot -> vertex ids
    // (32W u16). Degrees are not stored: they are the popcounts of the alive rows. A record is
    // reloaded on the frame it was made on when the warp still holds that frame (the tag
    // matches: its own depth-first subtree); otherwise (a donated record, or the warp has moved
    // on) its alive vertices are renumbered into a fresh frame (rebuild).
    static constexpr uint32_t kMidNt = 32 + 4 * W, kMidIds = 32 + 4 * W + 128;
    static constexpr uint32_t kMidBytes = kMidIds + 64 * W;
    __device__ __forceinline__ uint32_t graph_id(uint32_t slot) const {
        return reinterpret_cast<const uint16_t*>(dense_smem)[idb + slot];
    }
    __device__ __forceinline__ unsigned long long& frame_tag() const {
        return reinterpret_cast<unsigned long long*>(dense_smem)[tgi];
    }
    __device__ __forceinline__ void store_mid(unsigned char* rec, uint32_t rcc, uint32_t redges,
                                              uint32_t keep, uint32_t rnt) const {
        uint32_t word = 0;  // alive word `lane` (< W)
#pragma unroll
        for (int i = 0; i < W; ++i) {
            const uint32_t b = __ballot_sync(FULL, (keep >> i) & 1u);
            if (lane == i) word = b;
        }
        if (lane == 0) {
            const unsigned long long t = frame_tag();
            reinterpret_cast<uint4*>(rec)[0] = make_uint4(rcc, redges, REC_MID, ns);
            reinterpret_cast<uint4*>(rec)[1] = make_uint4((uint32_t)t, (uint32_t)(t >> 32), 0u, 0u);
        }
        if (lane < W) reinterpret_cast<uint32_t*>(rec + 32)[lane] = word;
        reinterpret_cast<uint32_t*>(rec + kMidNt)[lane] = rnt;
        // ids: 32W u16 = 2W bytes per lane
        const unsigned char* src = reinterpret_cast<const unsigned char*>(dense_smem) + 2 * idb;
        if constexpr (W == 4)
            reinterpret_cast<uint2*>(rec + kMidIds)[lane] = reinterpret_cast<const uint2*>(src)[lane];
        else
#pragma unroll
            for (int t = 0; t < W / 8; ++t)
                reinterpret_cast<uint4*>(rec + kMidIds)[lane + 32 * t] =
                    reinterpret_cast<const uint4*>(src)[lane + 32 * t];
    }
    // degrees = popcounts of the alive induced rows (aw words gathered on every lane)
    __device__ __forceinline__ void set_degrees() {
        uint32_t a[W];
#pragma unroll
        for (int j = 0; j < W; ++j) a[j] = __shfl_sync(FULL, aw, j);
#pragma unroll
        for (int i = 0; i < W; ++i) {
            uint32_t d = 0;
#pragma unroll
            for (int q = 0; q < Q; ++q) {
                const uint4 r = grp(q, 32 * i + lane);
                d += __popc(r.x & a[4 * q]) + __popc(r.y & a[4 * q + 1]) +
                     __popc(r.z & a[4 * q + 2]) + __popc(r.w & a[4 * q + 3]);
            }
            D(i) = alive(i) ? d : 0u;
        }
    }
    // A fresh frame over the nalive vertices whose ids are in the frame id table (ascending):
    // induced rows by ballots — lane l tests A[id(32i + l)][id(t)], so by symmetry the W
    // ballots for slot t are row t — then alive masks, degrees and a new tag.
    // (the warp's tag counter sits right after its current tag: tags are unique per shard, warp
    // and frame — (rank << 56) | ((worker + 1) << 36) | count, set up by the kernel)
    __device__ __forceinline__ unsigned long long next_tag() const {
        unsigned long long t = 0;
        if (lane == 0) t = ++reinterpret_cast<unsigned long long*>(dense_smem)[tgi + 1];
        return __shfl_sync(FULL, t, 0);
    }
    template <int GW>
    __device__ __noinline__ void build_frame(uint32_t nalive) {
        const unsigned long long tag = next_tag();
        constexpr uint32_t GNPAD = 32 * GW;
        const uint32_t* gw = reinterpret_cast<const uint32_t*>(dense_smem);
        if constexpr (W >= 8) {
            // Sparse graphs (the <= 256-slot frames run only there): each lane compresses the
            // graph rows of its own slots — for every frame neighbour (a set bit of row(id) ∩ F,
            // F = the frame's vertex set as a graph bitmap) its slot is the rank of its bit in F.
            // O(degree) per slot instead of the ballot build's O(frame slots).
            uint32_t* F = reinterpret_cast<uint32_t*>(dense_smem) + ssb;  // GW words
            uint32_t* P = F + GW;                                          // prefix ranks
            if (lane < GW) F[lane] = 0;
            __syncwarp();
#pragma unroll
            for (int i = 0; i < W; ++i)
                if (32u * i + lane < nalive) {
                    const uint32_t id = graph_id(32 * i + lane);
                    atomicOr(&F[id >> 5], 1u << (id & 31));
                }
            __syncwarp();
            const uint32_t pc = lane < GW ? __popc(F[lane]) : 0u;
            uint32_t incl = pc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(FULL, incl, o);
                if (lane >= o) incl += t;
            }
            if (lane < GW) P[lane] = incl - pc;
            __syncwarp();
#pragma unroll 1
            for (int i = 0; i < W; ++i) {
                const uint32_t s = 32u * i + lane;
                uint32_t row[W];
#pragma unroll
                for (int k = 0; k < W; ++k) row[k] = 0;
                if (s < nalive) {
                    const uint32_t id = graph_id(s);
#pragma unroll 1
                    for (uint32_t j = 0; j < GW; ++j) {
                        const uint32_t f = F[j];
                        uint32_t m = gw[((j >> 2) * GNPAD + id) * 4 + (j & 3)] & f;
                        while (m) {
                            const uint32_t b = __ffs(m) - 1;
                            m &= m - 1;
                            const uint32_t t = P[j] + __popc(f & ((1u << b) - 1u));
#pragma unroll
                            for (int k = 0; k < W; ++k) row[k] |= (t >> 5) == (uint32_t)k ? 1u << (t & 31) : 0u;
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < Q; ++q)
                    dense_smem[rb + q * NPAD + s] =
                        make_uint4(row[4 * q], row[4 * q + 1], row[4 * q + 2], row[4 * q + 3]);
            }
        } else {
            uint32_t myid[W];
#pragma unroll
            for (int i = 0; i < W; ++i) myid[i] = 32 * i + lane < nalive ? graph_id(32 * i + lane) : 0xFFFFu;
#pragma unroll 1
            for (uint32_t t = 0; t < nalive; ++t) {
                const uint32_t idt = graph_id(t);
                const uint32_t wj = idt >> 5, bit = idt & 31u;
                uint32_t row[W];
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    const bool b = myid[i] != 0xFFFFu &&
                                   ((gw[((wj >> 2) * GNPAD + myid[i]) * 4 + (wj & 3)] >> bit) & 1u);
                    row[i] = __ballot_sync(FULL, b);
                }
                if (lane < Q)
#pragma unroll
                    for (int q = 0; q < Q; ++q)
                        if (lane == q)
                            dense_smem[rb + q * NPAD + t] =
                                make_uint4(row[4 * q], row[4 * q + 1], row[4 * q + 2], row[4 * q + 3]);
            }
        }
        alv = 0;
#pragma unroll
        for (int i = 0; i < W; ++i) alv |= (32u * i + lane < nalive ? 1u : 0u) << i;
        ns = nalive;
        nt = 0;  // (verdicts are a cache: starting empty only re-runs tests)
        __syncwarp();
        rebuild_aw();
        set_degrees();
        if (lane == 0) frame_tag() = tag;
        __syncwarp();
    }
    // Renumbers a reduced wide node with at most 32W alive vertices into a fresh frame.
    template <bool I2>
    __device__ __forceinline__ void from_wide(const WarpNode<WG, I2>& w) {
        cc = w.cc;
        edges = w.edges;
        doom = false;
        const uint32_t pc = lane < WG ? __popc(w.aw) : 0u;
        uint32_t incl = pc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t base = incl - pc;  // lane j < WG: first slot of word j
        const uint32_t nalive = __shfl_sync(FULL, incl, 31);
        uint16_t* sid = reinterpret_cast<uint16_t*>(dense_smem) + idb;
#pragma unroll 1
        for (int i = 0; i < WG; ++i) {
            const uint32_t awi = __shfl_sync(FULL, w.aw, i);
            const uint32_t bi = __shfl_sync(FULL, base, i);
            if ((w.alv >> i) & 1u) sid[bi + __popc(awi & ((1u << lane) - 1u))] = (uint16_t)(32 * i + lane);
        }
        __syncwarp();
        build_frame<WG>(nalive);
    }
    // Loads a mid record: on the frame it was made on if the warp holds it, else renumbered
    // into a fresh frame.
    __device__ __forceinline__ void load_mid(const unsigned char* rec) {
        uint4 h0 = make_uint4(0, 0, 0, 0);
        uint2 h1 = make_uint2(0, 0);
        int same = 0;
        if (lane == 0) {
            h0 = __ldcg(reinterpret_cast<const uint4*>(rec));
            h1 = __ldcg(reinterpret_cast<const uint2*>(rec + 16));
            same = frame_tag() == (((unsigned long long)h1.y << 32) | h1.x);
        }
        cc = __shfl_sync(FULL, h0.x, 0);
        edges = __shfl_sync(FULL, h0.y, 0);
        doom = false;
        aw = lane < W ? __ldcg(reinterpret_cast<const uint32_t*>(rec + 32) + lane) : 0u;
        if (__shfl_sync(FULL, same, 0)) {
            ns = __shfl_sync(FULL, h0.w, 0);
            alv = 0;
#pragma unroll
            for (int i = 0; i < W; ++i) alv |= ((__shfl_sync(FULL, aw, i) >> lane) & 1u) << i;
            nt = __ldcg(reinterpret_cast<const uint32_t*>(rec + kMidNt) + lane);
            set_degrees();
            return;
        }
        rebuild_from(rec);
    }
    // The record's alive vertices (ids through its own id table) renumbered into a fresh frame.
    __device__ __noinline__ void rebuild_from(const unsigned char* rec) {
        uint32_t a[W], below[W];
        uint32_t run = 0;
#pragma unroll
        for (int j = 0; j < W; ++j) {
            a[j] = __shfl_sync(FULL, aw, j);
            below[j] = run;
            run += __popc(a[j]);
        }
        const uint16_t* rid = reinterpret_cast<const uint16_t*>(rec + kMidIds);
        uint16_t* sid = reinterpret_cast<uint16_t*>(dense_smem) + idb;
#pragma unroll
        for (int j = 0; j < W; ++j)
            if ((a[j] >> lane) & 1u)
                sid[below[j] + __popc(a[j] & ((1u << lane) - 1u))] = __ldcg(rid + 32 * j + lane);
        __syncwarp();
        build_frame<WG>(run);
    }
    // Word `lane` (< WG) of the cover bitmap (graph vertices not alive), in shared scratch.
    __device__ __forceinline__ uint32_t mid_cover_word(uint32_t* sb) const {
        if (lane < WG) sb[lane] = FULL;
        __syncwarp();
#pragma unroll
        for (int i = 0; i < W; ++i)
            if (alive(i)) {
                const uint32_t id = graph_id(32 * i + lane);
                atomicAnd(&sb[id >> 5], ~(1u << (id & 31)));
            }
        __syncwarp();
        const uint32_t w = lane < WG ? sb[lane] : 0u;
        __syncwarp();
        return w;
    }
};

// ------------------------------------------------------------------ compact search node

// Deep in the tree only a few dozen vertices are still alive (C5: 34 on average at a branch, of
// 500), yet the wide node scans all 32*W slots and reads the whole bitmap per child. Once at most
// 64 are alive, the node is renumbered: slot c (0..63) = the c-th alive vertex in id order, at
// lane c & 31, half c >> 5, and each lane keeps the INDUCED adjacency rows of its two slots as
// 64-bit masks in registers. Removing a slot, finding a partner, the triangle test, the whole
// remove-N(v) child and its doom test become a handful of shuffles and popcounts, with no shared
// memory traffic. Renumbering keeps the id order, so every rule acts on the same vertex as in
// the wide layout (and in the reference): node counts are unchanged. The alive set only shrinks,
// so every descendant of a compact node stays compact with the same slots.
constexpr uint32_t kCompactSlots = 64;
// Compact record: {cc, edges, kind, 0, alive lo, alive hi, verdicts lo, verdicts hi} + per lane
// {row of slot lane, row of slot lane+32} (16 B) + per lane packed ids (2 x u16).
constexpr uint32_t kCompactRecordBytes = 32 + 32 * 16 + 32 * 4;

template <bool INSTR>
struct CompactNode {
    static constexpr bool kInstr = INSTR;
#ifndef VCG_COMPACT_PASS_UNROLL
#define VCG_COMPACT_PASS_UNROLL 3
#endif
    // the three passes unrolled: candidate selection and pass tests become compile-time
    static constexpr int kPassUnroll = VCG_COMPACT_PASS_UNROLL;
    static constexpr int H = 2;          // slots per lane
    // Candidate masks are WARP-UNIFORM 64-bit slot masks built with two ballots: counting and
    // "first candidate >= pos" are then plain ALU work on every lane, with no reductions.
    using Mask = unsigned long long;
    unsigned long long r[H];             // induced row of slot 32*i + lane (bit c: slot c adjacent)
    uint32_t d[H];                       // degree of slot 32*i + lane (meaningless once removed)
    Mask am;                             // alive slots
    Mask nt;                             // cached degree-two non-triangle verdicts
    uint32_t ids;                        // vertex ids of slots lane (low 16) and lane + 32 (high)
    uint32_t cc, edges;                  // uniform
    bool doom;                           // uniform
    int lane;

    __device__ __forceinline__ static Mask ballot2(bool p0, bool p1) {
        return ((Mask)__ballot_sync(FULL, p1) << 32) | __ballot_sync(FULL, p0);
    }
    __device__ __forceinline__ static bool any(Mask m) { return m != 0; }
    __device__ __forceinline__ static uint32_t count(Mask m) { return __popcll(m); }
    __device__ __forceinline__ bool alive(int i) const { return (am >> (32 * i + lane)) & 1ull; }
    // the row of slot u on every lane
    __device__ __forceinline__ unsigned long long row(uint32_t u) const {
        return __shfl_sync(FULL, (u >> 5) ? r[1] : r[0], u & 31);
    }
    __device__ __forceinline__ void remove_vertex(uint32_t u) {  // search_node.cpp:16-25
        const unsigned long long ru = row(u);
        const uint32_t du = __popcll(ru & am);
#pragma unroll
        for (int i = 0; i < H; ++i) d[i] -= (uint32_t)(ru >> (32 * i + lane)) & 1u;
        am &= ~(1ull << u);
        cc += 1;
        edges -= du;
    }
    __device__ __forceinline__ Mask eq_mask(uint32_t c) const {
        return ballot2(d[0] == c, d[1] == c) & am;
    }
    __device__ __forceinline__ Mask above_mask(uint32_t lim) const {
        return ballot2(d[0] > lim, d[1] > lim) & am;
    }
    __device__ __forceinline__ void deg_masks(Mask& m1, Mask& m2) const {
        m1 = eq_mask(1u);
        m2 = eq_mask(2u) & ~nt;
    }
    __device__ __forceinline__ static int first_in(Mask m, int pos) {
        m = pos < 64 ? m & (~0ull << pos) : 0ull;
        return __ffsll((long long)m) - 1;
    }
    __device__ __forceinline__ void first_neighbors(uint32_t v, int& p0, int& p1) const {
        unsigned long long x = row(v) & am;
        p0 = __ffsll((long long)x) - 1;
        x &= x - 1;
        p1 = __ffsll((long long)x) - 1;
    }
    __device__ __forceinline__ bool is_edge(uint32_t p, uint32_t q) const {
        return (row(p) >> q) & 1ull;
    }
    __device__ __forceinline__ void mark_nt(uint32_t v) { nt |= 1ull << v; }
    __device__ __forceinline__ uint32_t argmax(uint32_t& dmax) const {  // search_node.cpp:34-46
        uint32_t mx = 0;
#pragma unroll
        for (int i = 0; i < H; ++i)
            mx = max(mx, alive(i) ? ((d[i] << 11) | (2047u - (32u * i + lane))) : 0u);
        mx = __reduce_max_sync(FULL, mx);
        dmax = mx >> 11;
        return 2047u - (mx & 2047u);
    }
    __device__ __forceinline__ bool doomed(int B) const { return doom || (int)cc > B; }
    template <class Cnt>
    __device__ __forceinline__ void reduce(int B, Cnt& st);

    // ---- the remove-N(v) child (search_node.cpp:27-32 on a clone)
    struct Child {
        Mask X;                // slots the child covers: N(v) ∩ alive
        uint32_t xcnt;         // |X|
        uint32_t nd[H];        // the survivors' degrees in the child
    };
    __device__ __forceinline__ void child_begin(uint32_t v, Child& c) const {
        c.X = row(v) & am;
        c.xcnt = __popcll(c.X);
    }
    // Degrees of the child; with TEST, true if it is pruned whatever happens when visited (its
    // cover exceeds the bound, or more survivors than its limit stay above it — the round-start
    // doom test of reduce_node on the child's state).
    template <bool TEST>
    __device__ __forceinline__ bool child_pass(Child& c, int B, uint32_t) const {
#pragma unroll
        for (int i = 0; i < H; ++i) c.nd[i] = d[i] - __popcll(r[i] & c.X);
        if (!TEST) return false;
        const uint32_t c2 = cc + c.xcnt;
        if ((int)c2 > B) return true;
        const uint32_t lim = limit_of(B, c2);
        return __popcll(ballot2(c.nd[0] > lim, c.nd[1] > lim) & am & ~c.X) > lim;
    }
    __device__ __forceinline__ void child_store(const Child& c, unsigned char* rec) const {
        const Mask keep = am & ~c.X;
        uint32_t esum = 0;
#pragma unroll
        for (int i = 0; i < H; ++i) esum += ((keep >> (32 * i + lane)) & 1ull) ? c.nd[i] : 0u;
        const uint32_t e2 = __reduce_add_sync(FULL, esum);
        store(rec, cc + c.xcnt, e2 / 2, keep, nt & keep);
    }
    __device__ __forceinline__ void store(unsigned char* rec, uint32_t rcc, uint32_t redges,
                                          Mask ram, Mask rnt) const {
        if (lane == 0) {
            reinterpret_cast<uint4*>(rec)[0] = make_uint4(rcc, redges, REC_COMPACT, 0u);
            reinterpret_cast<uint4*>(rec)[1] = make_uint4((uint32_t)ram, (uint32_t)(ram >> 32),
                                                          (uint32_t)rnt, (uint32_t)(rnt >> 32));
        }
        reinterpret_cast<uint4*>(rec + 32)[lane] =
            make_uint4((uint32_t)r[0], (uint32_t)(r[0] >> 32), (uint32_t)r[1], (uint32_t)(r[1] >> 32));
        reinterpret_cast<uint32_t*>(rec + 32 + 512)[lane] = ids;
    }
    __device__ __forceinline__ void store_current(unsigned char* rec) const {
        store(rec, cc, edges, am, nt);
    }
    // Loads a compact record through L2; degrees are recomputed from the rows.
    __device__ __forceinline__ void load(const unsigned char* rec) {
        uint4 h0 = make_uint4(0, 0, 0, 0), h1 = make_uint4(0, 0, 0, 0);
        if (lane == 0) {
            h0 = __ldcg(reinterpret_cast<const uint4*>(rec));
            h1 = __ldcg(reinterpret_cast<const uint4*>(rec) + 1);
        }
        const uint4 rr = __ldcg(reinterpret_cast<const uint4*>(rec + 32) + lane);
        ids = __ldcg(reinterpret_cast<const uint32_t*>(rec + 32 + 512) + lane);
        cc = __shfl_sync(FULL, h0.x, 0);
        edges = __shfl_sync(FULL, h0.y, 0);
        am = ((Mask)__shfl_sync(FULL, h1.y, 0) << 32) | __shfl_sync(FULL, h1.x, 0);
        nt = ((Mask)__shfl_sync(FULL, h1.w, 0) << 32) | __shfl_sync(FULL, h1.z, 0);
        r[0] = ((unsigned long long)rr.y << 32) | rr.x;
        r[1] = ((unsigned long long)rr.w << 32) | rr.z;
        set_degrees();
        doom = false;
    }
    __device__ __forceinline__ void set_degrees() {
#pragma unroll
        for (int i = 0; i < H; ++i) d[i] = __popcll(r[i] & am);
    }
    // Renumbers a reduced wide node with at most 64 alive vertices. `sb` is the warp's shared
    // scratch (at least 64 u16 + W words).
    template <int W, bool I2, int WG2>
    __device__ __forceinline__ void from_wide(const WarpNode<W, I2, WG2>& w, uint32_t* sb) {
        lane = w.lane;
        cc = w.cc;
        edges = w.edges;
        doom = false;
        // slot of an alive vertex 32j + b: (alive before word j) + (alive below b in word j)
        const uint32_t pc = lane < W ? __popc(w.aw) : 0u;
        uint32_t incl = pc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += t;
        }
        const uint32_t base = incl - pc;  // lane j < W: first slot of word j
        uint16_t* sid = reinterpret_cast<uint16_t*>(sb);
        const uint32_t nalive = __shfl_sync(FULL, incl, 31);
        sid[lane] = 0xFFFFu;
        sid[lane + 32] = 0xFFFFu;
        __syncwarp();
        // vertex 32 i + lane (alive bit i of this lane) → slot
#pragma unroll 1
        for (int i = 0; i < W; ++i) {
            const uint32_t awi = __shfl_sync(FULL, w.aw, i);
            const uint32_t bi = __shfl_sync(FULL, base, i);
            if ((w.alv >> i) & 1u) sid[bi + __popc(awi & ((1u << lane) - 1u))] = (uint16_t)(32 * i + lane);
        }
        __syncwarp();
        const uint32_t id0 = sid[lane], id1 = sid[lane + 32];
        __syncwarp();
        if constexpr (WG2 != 0)  // from a mid node: slots -> graph ids through its frame
            ids = (id0 != 0xFFFFu ? w.graph_id(id0) : 0xFFFFu) |
                  ((id1 != 0xFFFFu ? w.graph_id(id1) : 0xFFFFu) << 16);
        else
            ids = id0 | (id1 << 16);
        am = nalive >= 64 ? ~0ull : ((1ull << nalive) - 1ull);
        nt = 0;  // (verdicts are a cache: starting empty only re-runs tests)
#if VCG_FROM_WIDE_BALLOT
        // induced rows, one slot t at a time: lane l tests A[id_l][id_t] and A[id_{l+32}][id_t];
        // by symmetry the two ballots are row t itself (uniform work, no per-bit loops)
        // Slots are the alive vertices in id order, so walking the alive words and their set
        // bits in order visits slot t = 0, 1, ...: each lane loads its two rows' word j once
        // per word (not once per slot) and the slot's column is a register bit test.
        r[0] = r[1] = 0;
        uint32_t t = 0;
#pragma unroll 1
        for (int j = 0; j < W; ++j) {
            uint32_t awj = __shfl_sync(FULL, w.aw, j);  // (uniform)
            if (!awj) continue;
            const uint32_t w0 = id0 != 0xFFFFu ? w.row_word(id0, j) : 0u;
            const uint32_t w1 = id1 != 0xFFFFu ? w.row_word(id1, j) : 0u;
#pragma unroll 1
            while (awj) {
                const uint32_t bit = __ffs(awj) - 1;
                awj &= awj - 1;
                const unsigned long long row = ballot2((w0 >> bit) & 1u, (w1 >> bit) & 1u);
                if (lane == (int)(t & 31u)) {
                    if (t >> 5) r[1] = row;
                    else r[0] = row;
                }
                ++t;
            }
        }
#else
        // induced rows: compress row(id) over the alive set, word by word
        r[0] = r[1] = 0;
#pragma unroll 1
        for (int j = 0; j < W; ++j) {
            const uint32_t awj = __shfl_sync(FULL, w.aw, j);
            const uint32_t bj = __shfl_sync(FULL, base, j);
#pragma unroll
            for (int h = 0; h < H; ++h) {
                const uint32_t id = h ? id1 : id0;
                if (id == 0xFFFFu) continue;
                uint32_t m = w.row_word(id, j) & awj;
                while (m) {
                    const uint32_t b = __ffs(m) - 1;
                    m &= m - 1;
                    r[h] |= 1ull << (bj + __popc(awj & ((1u << b) - 1u)));
                }
            }
        }
#endif
        set_degrees();
    }
    // Word `lane` (< W) of the cover bitmap (vertices not alive), built in shared scratch.
    template <int W>
    __device__ __forceinline__ uint32_t cover_word(uint32_t* sb) const {
        if (lane < W) sb[lane] = FULL;
        __syncwarp();
#pragma unroll
        for (int i = 0; i < H; ++i) {
            const uint32_t id = (ids >> (16 * i)) & 0xFFFFu;
            if (alive(i)) atomicAnd(&sb[id >> 5], ~(1u << (id & 31)));
        }
        __syncwarp();
        const uint32_t w = lane < W ? sb[lane] : 0u;
        __syncwarp();
        return w;
    }
};

// reduce_loop (reductions.cpp:63-90) on either node layout: rounds of {degree-one,
// degree-two-triangle, high-degree} passes, each an ascending scan acting at visit time
// (first_in: the next candidate >= pos at this moment), until a round changes nothing.
template <class N, class Cnt>
__device__ __forceinline__ void reduce_node(N& x, int B, Cnt& st) {
    using Mask = typename N::Mask;
    while (x.edges != 0) {
        ++st.rounds;
        // Doom test at every round start (see pass 3): a node loaded from a record is usually
        // decided here, before any rule runs.
        const uint32_t lim0 = limit_of(B, x.cc);
        const Mask above = x.above_mask(lim0);
        if (N::count(above) > lim0) {
            x.doom = true;
            return;
        }
        // Candidate masks of the three passes at round start; they stay exact until the next
        // removal, so a pass without candidates is skipped and the first scan of a pass reuses
        // its mask.
        Mask m1, m2;
        x.deg_masks(m1, m2);
        if (!N::any(m1 | m2 | above)) break;  // the final no-change round
        bool removed = false;  // a removal happened since the round-start masks
        bool changed = false;
#pragma unroll (N::kPassUnroll)
        for (int pass = 1; pass <= 3; ++pass) {
            long long t0 = N::kInstr ? clock64() : 0;
            uint32_t c = pass;  // passes 1, 2: the degree; pass 3: the limit
            Mask cand = pass == 1 ? m1 : pass == 2 ? m2 : above;
            bool stale = removed;  // cand must be recomputed before use
            if (pass == 3) {
                const uint32_t lim = limit_of(B, x.cc);
                // Every alive vertex above the limit at pass start is removed by this pass (each
                // removal lowers the limit by one and any degree by at most one), so more than
                // `lim` of them take |S| past the bound: the node is pruned.
                if (removed) {  // (otherwise lim == lim0 and the round-start test holds)
                    cand = x.above_mask(lim);
                    if (N::count(cand) > lim) x.doom = true;
                    stale = false;
                }
                c = lim;
            }
            if (!stale && !N::any(cand)) continue;
            int pos = 0;
#pragma unroll 1
            while (!x.doomed(B)) {
                // (a degree-two vertex already known not to close a triangle is skipped: its
                // partners are unchanged while its degree is, so the test would fail)
                if (stale) {
                    cand = pass == 3 ? x.above_mask(c) : x.eq_mask(c);
                    if (pass == 2) cand &= ~x.nt;
                    stale = false;
                }
                const int v = x.first_in(cand, pos);
                if (v < 0) break;
                pos = v + 1;
                int u0 = v, u1 = -1;
                if (pass < 3) {
                    int p0, p1;
                    x.first_neighbors(v, p0, p1);
                    u0 = p0;  // degree one: its unique alive neighbour (reductions.cpp:7-19)
                    if (pass == 2) {  // degree two: both partners iff adjacent (:22-40)
                        const bool tri = x.is_edge(p0, p1);
                        u0 = tri ? p0 : -1;
                        u1 = tri ? p1 : -1;
                        if (!tri) x.mark_nt(v);
                    }
                }
#pragma unroll (N::kPassUnroll == 1 ? 1 : 2)
                for (int t = 0; t < 2; ++t) {
                    const int u = t ? u1 : u0;
                    if (u < 0) break;
                    x.remove_vertex((uint32_t)u);
                    changed = true;
                    removed = stale = true;
                    st.rm1 += pass == 1;
                    st.rm2 += pass == 2;
                    st.rmh += pass == 3;
                }
                if (pass == 3) c = limit_of(B, x.cc);  // :50-56
            }
            if (N::kInstr) st.phase[PH_DEG1 + pass - 1] += clock64() - t0;
            if (x.doomed(B)) return;
        }
        if (!changed) break;
    }
}

template <int W, bool INSTR, int WG>
template <class Cnt>
__device__ __forceinline__ void WarpNode<W, INSTR, WG>::reduce(int B, Cnt& st) {
    reduce_node(*this, B, st);
}
// The wide reduction out of line (VCG_WIDE_NOINLINE): the wide layout is the cold one, and its
// rule code inlined next to the compact hot loop costs instruction-cache misses. Counter deltas
// come back by value (a reference to the kernel's counters would move them to local memory).
struct RuleDeltas {
    uint32_t rounds, rm1, rm2, rmh;
};
template <class N>
__device__ __noinline__ RuleDeltas wide_reduce(N& x, int B) {
    CountersT<uint32_t> c;
    reduce_node(x, B, c);
    return RuleDeltas{c.rounds, c.rm1, c.rm2, c.rmh};
}
#ifndef VCG_WIDE_NOINLINE
#define VCG_WIDE_NOINLINE 1
#endif

template <bool INSTR>
template <class Cnt>
__device__ __forceinline__ void CompactNode<INSTR>::reduce(int B, Cnt& st) {
    reduce_node(*this, B, st);
}

// ------------------------------------------------------------------ device worklist

// GlobalWorklist::try_add (worklist.cpp:11-19): reserve capacity in the packed word (also
// counting the item in `pending` before anyone can see it), then draw a ticket. Two always-
// succeeding atomics; CAS loops collapse under thousands of contending warps.
__device__ __forceinline__ bool q_reserve(const DenseArgs& a, unsigned long long& pos_out,
                                          unsigned long long& size_seen) {
    Ctl* ctl = a.ctl;
    const unsigned long long old = atomicAdd(&ctl->work, ONE_PENDING | 1ull);
    const uint32_t size = (uint32_t)old;
    if (size >= a.capacity) {
        atomicAdd(&ctl->work, ~(ONE_PENDING | 1ull) + 1ull);  // undo: try_add rejects
        return false;
    }
    size_seen = size + 1ull;
    pos_out = atomicAdd(&ctl->tail, 1ull);
    return true;
}

// (By value: a reference to the kernel parameters would force them into local memory.)
__device__ __noinline__ void cancel_all_(Ctl* ctl, const PeerRef* peers, uint32_t world,
                                         uint32_t rank) {
    atomicExch(&ctl->cancel, 1u);
    for (uint32_t p = 0; p < world; ++p)
        if (p != rank) atomicExch_system(&peers[p].ctl->cancel, 1u);
}
#define cancel_all(a) cancel_all_((a).ctl, (a).peers, (a).world, (a).rank)

// Waits until ring slot `publish` is free for ticket `pos` (its previous lap's reader released
// it). After a cancel that reader may have left for good, so the wait gives up when `cancel`
// is raised (returns false: the caller keeps its record and leaves at its next poll).
__device__ __noinline__ bool wait_slot_free(const unsigned long long* publish,
                                            unsigned long long pos, const uint32_t* cancel,
                                            bool sys) {
#pragma unroll 1
    for (uint32_t spin = 0;; ++spin) {
        if ((sys ? ld_acquire_sys_u64(publish) : ld_acquire_u64(publish)) == pos) return true;
        if ((spin & 15) == 15 && *reinterpret_cast<const volatile uint32_t*>(cancel)) return false;
        __nanosleep(32);
    }
}

// Copies one node record (either layout) through L2: `vec16` 16-byte vectors spread over the
// warp's lanes.
__device__ __forceinline__ void copy_record_raw(const unsigned char* src, unsigned char* dst,
                                                uint32_t vec16, int lane) {
#pragma unroll 1
    for (uint32_t t = lane; t < vec16; t += 32)
        reinterpret_cast<uint4*>(dst)[t] = __ldcg(reinterpret_cast<const uint4*>(src) + t);
}

// Work donation between shards (cold): reserve a slot in peer `pr`'s ring, copy the record at
// `src` into it over NVLink / IPC, publish it with a system-scope release. Warp-collective.
__device__ __noinline__ bool donate_to_peer(const PeerRef* pr, Ctl* ctl0, Ctl* own,
                                            uint32_t capacity, uint32_t ring_mask,
                                            unsigned long long entry_bytes,
                                            const unsigned char* src, int lane) {
    uint32_t* const gactive = &ctl0->gactive;
    unsigned long long pos = 0;
    int ok = 0;
    if (lane == 0) {
        const unsigned long long old = atomicAdd_system(&pr->ctl->work, ONE_PENDING | 1ull);
        if ((old >> 32) == 0) atomicAdd_system(gactive, 1u);  // the peer's pending 0 -> 1
        if ((uint32_t)old >= capacity) {
            const unsigned long long o2 =
                atomicAdd_system(&pr->ctl->work, ~(ONE_PENDING | 1ull) + 1ull);
            if ((o2 >> 32) == 1) atomicSub_system(gactive, 1u);  // and back 1 -> 0
        } else {
            pos = atomicAdd_system(&pr->ctl->tail, 1ull);
            ok = 1;
        }
    }
    if (!__shfl_sync(FULL, ok, 0)) return false;
    pos = __shfl_sync(FULL, pos, 0);
    unsigned long long* publish = pr->seq + (pos & ring_mask);
    int freed = 1;
    if (lane == 0 && ld_acquire_sys_u64(publish) != pos)
        freed = wait_slot_free(publish, pos, &own->cancel, true);
    if (!__shfl_sync(FULL, freed, 0)) return false;
    copy_record_raw(src, pr->wl + (pos & ring_mask) * entry_bytes, (uint32_t)(entry_bytes / 16), lane);
    __syncwarp();
    if (lane == 0) st_release_sys_u64(publish, pos + 1);
    return true;
}

// The exchange helper of a linked shard (warp 0 of the shard kernel; it never searches). The
// search warps run the single-shard loop against their own device worklist; this warp moves
// queued nodes from it into the worklists of peer shards that run low — over NVLink P2P /
// CUDA IPC: reserve a slot in the peer's ring with system-scope atomics, copy the record,
// publish with a system-scope release (the peer's workers acquire at system scope) — and so
// keeps the peer-specific code and registers out of the search warps (which then hold the
// single-shard kernel's 24 warps per SM). A node moves only from a shard with more queued
// nodes than the peer; the peer's `pending` is raised before this shard's drops (termination:
// see donate_to_peer).
__device__ __noinline__ void exchange_helper(Ctl* ctl, const PeerRef* peers, uint32_t world,
                                             uint32_t rank, uint32_t capacity, uint32_t ring_mask,
                                             uint32_t threshold, unsigned long long entry_bytes,
                                             unsigned char* wl, unsigned long long* seq,
                                             WStats* stats, int lane) {
    uint32_t* const gactive = &peers[0].ctl->gactive;
    unsigned long long moved = 0;
    uint32_t rr = 0, sleep = 64;
#pragma unroll 1
    while (true) {
        // 1. stop: cancel, or every shard idle (no queued node, no active worker anywhere)
        int act = 0;  // 0 wait, 1 move to `target`, 2 stop
        uint32_t target = 0;
        if (lane == 0) {
            const unsigned long long w = ld_relaxed_sys_u64(&ctl->work);
            if (*reinterpret_cast<volatile uint32_t*>(&ctl->cancel)) {
                act = 2;
            } else if ((w >> 32) == 0 && ld_acquire_sys_u32(gactive) == 0) {
                act = 2;
            } else {
                // 2. the poorest peer below its donation threshold, if this shard is richer
                const uint32_t mine = (uint32_t)w;
                uint32_t best = ~0u;
                for (uint32_t i = 1; i < world; ++i) {
                    const uint32_t p = (rank + i + rr) % world;
                    const uint32_t q = (uint32_t)ld_relaxed_sys_u64(&peers[p].ctl->work);
                    if (q < threshold && q + 1 < mine && q < best) {
                        best = q;
                        target = p;
                    }
                }
                ++rr;
                act = best != ~0u ? 1 : 0;
            }
        }
        act = __shfl_sync(FULL, act, 0);
        if (act == 2) break;
        if (act == 0) {
            __nanosleep(sleep);
            sleep = min(sleep * 2, 2048u);
            continue;
        }
        sleep = 64;
        target = __shfl_sync(FULL, target, 0);
        // 3. take the next local node: a ticket, then its publication (it may be a peer's)
        unsigned long long pos = 0;
        int got = 0;
        if (lane == 0) {
            pos = atomicAdd(&ctl->head, 1ull);
#pragma unroll 1
            for (uint32_t spin = 0;; ++spin) {
                // (relaxed polls — an acquire invalidates the SM's L1, the search warps' spill
                // and local-memory lines included; every lane acquires once it has matched)
                if (ld_relaxed_sys_u64(seq + (pos & ring_mask)) == pos + 1) {
                    got = 1;
                    break;
                }
                if ((spin & 7) == 7) {
                    if (*reinterpret_cast<volatile uint32_t*>(&ctl->cancel)) break;
                    if ((ld_relaxed_sys_u64(&ctl->work) >> 32) == 0 && ld_acquire_sys_u32(gactive) == 0)
                        break;
                }
                __nanosleep(64);
            }
        }
        if (!__shfl_sync(FULL, got, 0)) break;
        pos = __shfl_sync(FULL, pos, 0);
        (void)ld_acquire_sys_u64(seq + (pos & ring_mask));  // (every lane acquires it)
        const unsigned char* src = wl + (pos & ring_mask) * entry_bytes;
        // 4. into the peer's ring (full — a race with other donors — means it has plenty: retry
        // until it drains; a cancel ends the search anyway)
        bool sent = false;
#pragma unroll 1
        for (uint32_t back = 64;; back = min(back * 2, 2048u)) {
            sent = donate_to_peer(peers + target, peers[0].ctl, ctl, capacity, ring_mask, entry_bytes,
                                  src, lane);
            if (sent) break;
            int c = 0;
            if (lane == 0) c = *reinterpret_cast<volatile uint32_t*>(&ctl->cancel);
            if (__shfl_sync(FULL, c, 0)) break;
            __nanosleep(back);
        }
        __syncwarp();
        // 5. release the local slot; this shard's queue and pending each drop by one (the peer's
        // pending was raised first, so the active-shard count never touches zero in between)
        if (lane == 0) {
            st_release_sys_u64(seq + (pos & ring_mask), pos + ring_mask + 1);
            __threadfence_system();
            const unsigned long long o = atomicAdd_system(&ctl->work, ~(ONE_PENDING | 1ull) + 1ull);
            if ((o >> 32) == 1) atomicSub_system(gactive, 1u);
        }
        moved += sent;
    }
    if (lane == 0) stats->peer = moved;
}

// record_cover (scheduler.cpp:84-108) once the warp holds a cover: MVC keeps it if it beats the
// bound (every shard's bound is lowered), PVC keeps the first and ends the search everywhere.
// Returns true when the search is over (PVC). Cold: out of the node loop's code.
__device__ __noinline__ bool record_cover_(Ctl* ctl, uint32_t* cover_slots, volatile uint32_t* mailbox,
                                           const PeerRef* peers, uint32_t world, uint32_t rank,
                                           int pvc, uint32_t W, uint32_t worker, uint32_t cc,
                                           uint32_t wbits, int lane) {
    uint32_t record = 0;
    if (lane == 0) {
        if (pvc) record = atomicCAS(&ctl->found, 0u, 1u) == 0u;
        else record = cc < atomicMin(&ctl->best, cc);
    }
    if (__shfl_sync(FULL, record, 0)) {
        if (lane < (int)W) cover_slots[(unsigned long long)worker * W + lane] = wbits;
        __threadfence();
        __syncwarp();
        if (lane == 0) {
            atomicMin(&ctl->best_owner, ((unsigned long long)cc << 32) | worker);
            if (pvc) {
                cancel_all_(ctl, peers, world, rank);
            } else {
                for (uint32_t p = 0; p < world; ++p)  // the bound reaches every shard
                    if (p != rank) atomicMin_system(&peers[p].ctl->best, cc);
            }
            if (mailbox) {
                mailbox[2] = cc;
                if (pvc) mailbox[3] = 1;
            }
        }
    }
    return pvc != 0;
}
#define record_cover(a, worker, cc, wbits, lane)                                                 \
    record_cover_((a).ctl, (a).cover_slots, (a).mailbox, (a).peers, (a).world, (a).rank, (a).pvc, \
                  W, worker, cc, wbits, lane)

// ------------------------------------------------------------------ the traversal kernel

enum { ACT_CONT = 0, ACT_POP = 1, ACT_BREAK = 2, ACT_BRANCH = 3 };

template <int W, bool INSTR, bool MULTI, bool ONEW = false, int MW = default_mid(W), bool MOOL = false,
          int BW = 8>
#ifndef VCG_MINB16
#define VCG_MINB16 3  // CTAs of 8 warps per SM targeted by the W=16 register allocation
#endif               // (wide degrees in smem: 3 → 80 regs, C5 10.2 ms; 2 → 127 regs, 10.8 ms; 4 → 64 + spills, 12.9)
#ifndef VCG_MINB8
#define VCG_MINB8 3   // the same for W <= 8 (C1: 3 → 0.98 ms, 4 → 1.08 ms)
#endif
#ifndef VCG_MINB_MULTI
#define VCG_MINB_MULTI 3  // the linked-shard instantiation: the single-shard kernel's 24 warps per
                          // SM (its peer code lives in the exchange helper warp)
#endif
// MW: the mid layout's width (0 none, 4: <= 128 alive, 8: <= 256 alive — its 8 KB frames leave
// room for 2 CTAs per SM; for sparse graphs whose nodes stay wide). MOOL: the mid reduction out
// of line (an A/B option: out of line, the mid node's register degrees go through local memory
// around the call; dense graphs, whose visits are nearly all compact, run MW = 0 instead — the
// mid code inlined costs their compact hot loop registers and instruction cache).
// BW: warps per CTA — 8 (several CTAs per SM, each with its own copy of the graph bitmap), or one
// large CTA per SM (the bitmap stored once leaves room for more warps' frames / registers).
__global__ void __launch_bounds__(32 * BW, (BW != 8 ? 1 : (W <= 8 ? VCG_MINB8 : (W == 16 ? (MULTI ? VCG_MINB_MULTI : (MW == 8 ? 2 : VCG_MINB16)) : 1)))) dense_kernel(DenseArgs a) {
    constexpr int Q = W / 4;
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    const uint32_t worker = blockIdx.x * (blockDim.x >> 5) + wib;

    // Stage the read-only adjacency bitmap once per CTA (coalesced 16-byte copies).
    for (uint32_t t = threadIdx.x; t < Q * a.npad; t += blockDim.x) dense_smem[t] = a.at4[t];
    __syncthreads();
    if (worker >= a.workers) return;

    // start times live in the warp's scratch words while the search runs (read only for
    // timeout checks and the final stats): two fewer 64-bit registers on the hot path
    // (the warp's W-word slot between the bitmap and the scratch words; W >= 4)
    unsigned long long* const t0s = reinterpret_cast<unsigned long long*>(
        reinterpret_cast<uint32_t*>(dense_smem) + (W / 4) * (32 * W) * 4 + wib * W);
    // (W >= 16: words 4..7 of the slot hold the mid layout's current frame tag and tag counter)
    static_assert(MW == 0 || (W >= 16 && (MW == 4 || MW == 8)), "mid layout width");
    // (W >= 16, VCG_CNT_SMEM: words 8..10 hold lane 0's per-branch counters — branches,
    // children stored and donations packed 10 bits each (deltas between flushes, at most
    // flush_every <= 64 each), stack high water, queue maximum — instead of five registers
    // live across the node loop: the hot loop's register budget sets the occupancy, and the
    // counters change at most once per branch. Words 12..15: the poll's copy of the control
    // line's first 16 bytes {best, cancel, work}, landed by cp.async — no registers held from
    // the poll's issue to its use after the reduction.)
    constexpr bool kCntSmem = VCG_CNT_SMEM && W >= 16;
    constexpr bool kPollSmem = VCG_POLL_SMEM && W >= 16 && !VCG_SPLIT_WORK;
    uint32_t* const cw = reinterpret_cast<uint32_t*>(t0s) + 8;
    enum { CW_PACKED = 0, CW_HIGH = 1, CW_MAXQ = 2 };
    constexpr uint32_t CWP_MAXDEG = 1u, CWP_CHILDREN = 1u << 10, CWP_DONATED = 1u << 20;
    uint32_t* const pw = reinterpret_cast<uint32_t*>(t0s) + 12;
    if (lane == 0) {
        t0s[0] = globaltimer();
        t0s[1] = (unsigned long long)clock64();
        if (kCntSmem)
#pragma unroll
            for (int i = 0; i < 3; ++i) cw[i] = 0;
        if (MW) {
            t0s[2] = 0;  // no frame
            t0s[3] = ((unsigned long long)a.rank << 56) | ((unsigned long long)(worker + 1) << 36);
        }
    }
    __syncwarp();
    if constexpr (MULTI) {
        if (worker == 0) {  // linked shards: warp 0 moves queued nodes to starving peers
            exchange_helper(a.ctl, a.peers, a.world, a.rank, a.capacity, a.ring_mask, a.threshold,
                            a.entry_bytes, a.wl, a.seq, a.stats, lane);
            return;
        }
    }
#define t_start (t0s[0])
#define c_start ((long long)t0s[1])
    // The current node is WIDE (x: all 32*W vertex slots) until at most 64 vertices are alive,
    // then COMPACT (y: renumbered induced subgraph, see CompactNode).
    WarpNode<W, INSTR> x;
    x.ssb = dense_scratch_base<W, BW>(wib);
#if VCG_WIDE_SMEM
    x.dsb = dense_degree_base<W, MW, BW>(wib);
#endif
    x.lane = lane;
    CompactNode<INSTR> y;
    y.lane = lane;
    // the mid layout (64 < alive <= 32 MW): its frame bitmap in the warp's wide degree words,
    // its scratch and frame id table in the warp's wide scratch words (unused while mid)
    WarpNode<MW ? MW : 4, INSTR, W> m;
    m.lane = lane;
    m.ssb = x.ssb;
    m.rb = dense_degree_base<W, MW, BW>(wib) / 4;
    m.idb = (x.ssb + (MW ? MW : 4) * 32) * 2;
    m.tgi = (uint32_t)(reinterpret_cast<uint32_t*>(t0s) - reinterpret_cast<uint32_t*>(dense_smem)) / 2 + 2;
    enum { M_WIDE = 0, M_COMPACT = 1, M_MID = 2 };
    uint32_t mode = M_WIDE;
    // (derived on use rather than held in registers: the hot path's register budget sets the
    // occupancy)
#define sb (reinterpret_cast<uint32_t*>(dense_smem) + x.ssb)  // warp scratch
#define vec16 ((uint32_t)(a.entry_bytes / 16))
    Counters32 st;
    Ctl* ctl = a.ctl;
#define my_stats (a.stats + worker)
    auto fold_cw = [&]() {  // (lane 0)
        const uint32_t pk = cw[CW_PACKED];
        my_stats->maxdeg += pk & 1023u;
        my_stats->children += (pk >> 10) & 1023u;
        my_stats->donated += pk >> 20;
        cw[CW_PACKED] = 0;
    };
#define my_stack (a.stacks + (unsigned long long)worker * a.stack_bound * a.entry_bytes)
    // The local stack is a ring [base, base + sp) so its oldest entry can be donated.
    uint32_t base = 0, sp = 0;
    auto slot_at = [&](uint32_t i) {
        uint32_t j = base + i;
        if (j >= a.stack_bound) j -= a.stack_bound;
        return my_stack + (unsigned long long)j * a.entry_bytes;
    };
    bool have = false, idle = true;
    unsigned long long subtree = 0;  // StackOnly: current sub-tree id
    uint32_t replay = 0xFFFFFFFFu;   // StackOnly: levels of the root path replayed so far
    uint32_t best = a.pvc ? a.k : ctl->best;
    int B = bound_of(a.pvc, a.k, best);  // prune once |S| > B
    // (small graphs, W <= 8: short trees whose time is latency — bound and cancel news must
    // travel fast, so they keep polling every 8 nodes)
    constexpr uint32_t kPollK = W <= 8 ? 8u : kPoll;
    uint32_t qsize = 0, polls = kPollK - 1;  // (the first node polls)
    bool poll = false;
    uint2 h = make_uint2(0, 0);  // control line: {best, cancel}
    uint32_t hw = 0;             // worklist size
    // (the one-worker strategies — seq, StackOnly — are a separate instantiation: the hybrid
    // kernel carries none of their marker / replay code)
    const bool seq_mode_ = ONEW && a.seq_mode;
    const bool stackonly_ = ONEW && a.stackonly;
    const bool multi = MULTI;  // linked shards (a separate instantiation: the single-shard
                               // kernel carries none of the peer code)

    // process_node (scheduler.cpp:125-144) up to the branch: reduce, prune, record a cover.
    auto reduce_under_B = [&](auto& n) {
        using NT = typename std::remove_reference<decltype(n)>::type;
        // (only the wide layout out of line: its degrees are in shared memory anyway, while a
        // call taking the mid node by reference would move its register degrees to local memory)
        if constexpr (VCG_WIDE_NOINLINE && !INSTR &&
                      (std::is_same<NT, WarpNode<W, INSTR>>::value ||
                       (MOOL && !std::is_same<NT, CompactNode<INSTR>>::value))) {
            const RuleDeltas dl = wide_reduce(n, B);
            st.rounds += dl.rounds;
            st.rm1 += dl.rm1;
            st.rm2 += dl.rm2;
            st.rmh += dl.rmh;
        } else {
            n.reduce(B, st);
        }
    };
    auto settle = [&](auto& n) -> int {
        // The edge-count prune (should_prune, bounds.cpp:27-29) is a proof only when every
        // alive degree is within the high-degree limit of the SAME bound (reductions.hpp:25-26):
        // a cover of L = B - |S| vertices of degree <= L covers at most L^2 edges. The reference
        // reads one `best` for both (scheduler.cpp:127-132, reductions.cpp:70-87); here the poll
        // below may lower B after the reduction ran, so the edge test uses Br, the bound the
        // reduction reached fixpoint under (no cover of size <= Br - |S| proves none <= B - |S|
        // either), while |S| > B and the doom test prune under the newest bound. (Round 2 first
        // re-ran the reduction under the lowered bound: a second inlined copy of the compact
        // reduction in the hot loop, 8% on C5 through instruction-cache misses.)
        const int Br = B;
        reduce_under_B(n);
        if (VCG_UNLIKELY(poll)) {
            uint32_t pb, pc, pq;  // the polled {best, cancel, size}
            if constexpr (kPollSmem) {
                if (lane == 0) asm volatile("cp.async.wait_all;" ::: "memory");
                __syncwarp();
                pb = pw[0];
                pc = pw[1];
                pq = pw[2];
            } else {
                pb = __shfl_sync(FULL, h.x, 0);
                pc = __shfl_sync(FULL, h.y, 0);
                pq = __shfl_sync(FULL, hw, 0);
            }
            if (pc) return ACT_BREAK;
            if (!a.pvc) {
                best = min(best, pb);
                B = bound_of(0, 0, best);
            }
            qsize = pq;
        }
        const bool prune = n.doom || prune_at(Br, n.cc, n.edges) || (int)n.cc > B;
        st.dooms += n.doom;
        if (prune) return ACT_POP;
        if (VCG_UNLIKELY(n.edges == 0)) {
            // record_cover (scheduler.cpp:84-108)
            const uint32_t wbits = n.template cover_word<W>(sb);
            if (record_cover(a, worker, n.cc, wbits, lane)) return ACT_BREAK;  // PVC: ended
            best = min(best, n.cc);
            B = bound_of(0, 0, best);
            return ACT_POP;
        }
        return ACT_BRANCH;
    };

    // Branch (scheduler.cpp:185-203) on the smallest-id max-degree vertex v: defer remove-N(v)
    // — donated while the worklist is below its threshold (with donate_oldest the oldest stacked
    // node goes instead and the child is stacked) — and continue with remove-v.
    auto branch = [&](auto& n) -> int {
        long long tm = INSTR ? clock64() : 0;
        uint32_t dmax;
        const uint32_t v = n.argmax(dmax);
        if (kCntSmem) { if (lane == 0) cw[CW_PACKED] += CWP_MAXDEG; } else ++st.maxdeg;
        if (INSTR) st.phase[PH_MAXDEG] += clock64() - tm;
        long long tb = INSTR ? clock64() : 0;
        // StackOnly replay of the root path: branch bit `replay` of the sub-tree id picks the
        // child (0 = remove v_max, 1 = remove N(v_max), scheduler.cpp:303-309), nothing deferred
        const bool replaying = stackonly_ && replay < a.depth;
        const bool right = replaying && ((subtree >> replay) & 1ull);
        replay += replaying;
        unsigned char* child = nullptr;
        unsigned long long* publish = nullptr;
        unsigned long long pos = 0;
        // (After a full reduction every alive degree is within the high-degree limit, so
        // |S| + |N(v)| stays below the bound: the deferred child is never dead on arrival.)
        typename std::remove_reference<decltype(n)>::type::Child c;
        n.child_begin(v, c);
        const bool build = !replaying || right;
        bool dead = false;
        if (build) {
            // A child pruned whatever happens is not stored, queued and reloaded: it is counted
            // as visited right here (the reference counts it when it pops it). The one-worker
            // strategies keep the reference's visit ORDER — a search that stops early (PVC yes,
            // budget) must not count it — so they stack a 16-byte marker in its place instead.
            dead = n.template child_pass<true>(c, B, dmax);
            if (!seq_mode_) {
                st.nodes += dead;
                st.dooms += dead;
            }
        }
        const bool oldest = a.donate_oldest && sp > 0;
        if (!seq_mode_ && qsize < a.threshold && (oldest || !dead)) {
            unsigned long long seen = 0;
            int ok = 0;
            if (lane == 0) ok = q_reserve(a, pos, seen);
            if (lane == 0 && ok) {
                if (kCntSmem) cw[CW_MAXQ] = max(cw[CW_MAXQ], (uint32_t)seen);
                else st.max_queue = max(st.max_queue, (uint32_t)seen);
                // the slot is free once the previous lap's reader released it
                if (ld_acquire_u64(a.seq + (pos & a.ring_mask)) != pos)  // (rarely not yet)
                    ok = wait_slot_free(a.seq + (pos & a.ring_mask), pos, &ctl->cancel, false);
            }
            if (__shfl_sync(FULL, ok, 0)) {
                pos = __shfl_sync(FULL, pos, 0);
                publish = a.seq + (pos & a.ring_mask);
                unsigned char* dst = a.wl + (pos & a.ring_mask) * a.entry_bytes;
                if (oldest) {
                    copy_record_raw(slot_at(0), dst, vec16, lane);
                    base = base + 1 == a.stack_bound ? 0 : base + 1;
                    --sp;
                } else {
                    child = dst;
                }
                if (kCntSmem) { if (lane == 0) cw[CW_PACKED] += CWP_DONATED; } else ++st.donated;
            }
        }
        if (build && (!dead || seq_mode_)) {
            if (!child) {
                child = slot_at(sp);
                ++sp;
                if (kCntSmem) { if (lane == 0 && sp > cw[CW_HIGH]) cw[CW_HIGH] = sp; }
                else if (sp > st.high_water) st.high_water = sp;
            }
            if (dead) {
                if (lane == 0) *reinterpret_cast<uint4*>(child) = make_uint4(DEAD_NODE, 0u, 0u, 0u);
            } else {
                n.child_store(c, child);
                if (kCntSmem) { if (lane == 0) cw[CW_PACKED] += CWP_CHILDREN; } else ++st.children;
            }
        }
        if (publish) {
            __syncwarp();  // (the release by lane 0 is cumulative over the warp's stores)
            if (lane == 0) st_release_u64(publish, pos + 1);
        }
        if (INSTR) st.phase[publish ? PH_WL_ADD : PH_BRANCH_NBRS] += clock64() - tb;
        if (right) return ACT_POP;  // replay continues with the remove-N(v) child just stacked
        long long tv = INSTR ? clock64() : 0;
        n.remove_vertex(v);
        if (INSTR) st.phase[PH_BRANCH_V] += clock64() - tv;
        return ACT_CONT;
    };

#pragma unroll 1
    while (true) {
        if (!have) {
            long long t0 = INSTR ? clock64() : 0;
            const unsigned char* src;
            unsigned long long* release = nullptr;
            unsigned long long pos = 0;
            if (sp > 0) {
                --sp;
                src = slot_at(sp);
            } else if (stackonly_) {
                // stackonly_worker (scheduler.cpp:279-281): claim the next sub-tree id and
                // replay its root path from the root record (ring slot 0, never consumed)
                unsigned long long t = 0;
                int o = 0;
                if (lane == 0) {
                    t = atomicAdd(&ctl->head, 1ull);
                    o = (t >> a.depth) == 0 && !ld_volatile_v4(ctl).y;
                }
                if (!__shfl_sync(FULL, o, 0)) break;
                if (VCG_TIMELINE && lane == 0 && !my_stats->t_first) my_stats->t_first = globaltimer();
                subtree = __shfl_sync(FULL, t, 0);
                replay = 0;
                src = a.wl;
            } else {
                // GlobalWorklist::remove_or_done (worklist.cpp:21-48): take a ticket, then wait
                // for that slot's publication, for termination (pending == 0) or a cancel.
                if (!idle) {
                    if (lane == 0) {
                        const unsigned long long o = atomicAdd(&ctl->work, ~ONE_PENDING + 1ull);
                        if (multi && (o >> 32) == 1) {  // this shard went idle
                            __threadfence_system();
                            atomicSub_system(&a.peers[0].ctl->gactive, 1u);
                        }
                    }
                    idle = true;
                }
                if (lane == 0) pos = atomicAdd(&ctl->head, 1ull);
                pos = __shfl_sync(FULL, pos, 0);
                release = a.seq + (pos & a.ring_mask);
                uint32_t sleep = 32;
                int outcome = 0;  // 1 got, 2 done
                const unsigned long long w0 = lane == 0 ? globaltimer() : 0ull;
#pragma unroll 1
                for (uint32_t spin = 0;; ++spin) {
                    int o = 0;
                    if (lane == 0) {
                        // relaxed polls: an acquire load invalidates the SM's whole L1 (CCTL.IVALL),
                        // the working warps' local-memory lines included, at every spin of every
                        // idle warp; the publication is acquired once, below, after the match
                        if ((multi && !VCG_TEST_GPU_ACQ ? ld_relaxed_sys_u64(release) : ld_relaxed_u64(release)) == pos + 1) o = 1;
                        else if ((spin & 7) == 7) {
                            if (ld_volatile_v4(ctl).y) o = 2;
                            else if ((ld_relaxed_u64(&ctl->work) >> 32) == 0 &&
                                     (!multi || ld_acquire_sys_u32(&a.peers[0].ctl->gactive) == 0))
                                o = 2;  // every shard idle: nothing can create work again
                            else if (worker == (MULTI ? 1u : 0u) && a.mailbox) poll_mailbox(a.mailbox, a.pvc, ctl);
                            else if (a.timeout_ns && globaltimer() - t_start >= a.timeout_ns) {
                                atomicCAS(&ctl->status, 0, 1);
                                cancel_all(a);
                                o = 2;
                            }
                        }
                    }
                    outcome = __shfl_sync(FULL, o, 0);
                    if (outcome) break;
                    __nanosleep(sleep);
                    sleep = min(sleep * 2, a.backoff_ns);
                }
                if (lane == 0) {  // (cold: the idle path)
                    const unsigned long long now = globaltimer();
                    my_stats->t_idle += now - w0;
                    my_stats->t_lastwait = w0;
                    // the first node of a worker always comes off the worklist: its time is
                    // kept here, off the hot loop (a first-pop flag held in a register across
                    // the loop cost C5 5% through spills)
                    if (VCG_TIMELINE && outcome == 1 && !my_stats->t_first) my_stats->t_first = now;
                }
                if (outcome == 2) {
                    if (INSTR) st.phase[PH_WL_REMOVE] += clock64() - t0;
                    break;
                }
                // every lane acquires the publication
                (void)(multi && !VCG_TEST_GPU_ACQ ? ld_acquire_sys_u64(release) : ld_acquire_u64(release));
                src = a.wl + (pos & a.ring_mask) * a.entry_bytes;
                idle = false;
            }
            uint2 kc = make_uint2(0, 0);  // {cover count, kind}
            if (lane == 0) {
                const uint4 hd = __ldcg(reinterpret_cast<const uint4*>(src));
                kc = make_uint2(hd.x, hd.z);
            }
            const uint32_t kind = __shfl_sync(FULL, kc.y, 0);
            if (kind == REC_COMPACT) {
                mode = M_COMPACT;
                y.load(src);
            } else if (MW && kind == REC_MID) {
                mode = M_MID;
                m.load(src);
            } else {
                mode = M_WIDE;
                if (seq_mode_ && __shfl_sync(FULL, kc.x, 0) == DEAD_NODE) {
                    x.cc = DEAD_NODE;  // a dead child's marker (see below): nothing to load
                } else {
                    x.load(src);
                    if (MW && lane == 0) t0s[2] = 0;  // the wide degrees overwrote the frame
                }
            }
            if (release) {
                // every lane's read of the slot is ordered before lane 0's release by the
                // warp barrier (cumulativity): no full fence needed
                __syncwarp();
                if (lane == 0) {
                    if (VCG_RELAXED_FREE && !multi)  // (A/B only, see VCG_RELAXED_FREE)
                        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(release), "l"(pos + a.ring_mask + 1) : "memory");
                    else
                        st_release_u64(release, pos + a.ring_mask + 1);  // free for the next lap
                    atomicAdd(&ctl->work, ~0ull);                     // size - 1
                }
            }
            have = true;
            if (INSTR) st.phase[release ? PH_WL_REMOVE : PH_STACK] += clock64() - t0;
        }

        // Every worker polling the one control line at every node queues thousands of reads on
        // one L2 slice (and the scoreboard wait lands inside the reduction), so it is polled
        // every kPoll nodes; in between the warp uses the last bound / queue size it saw (a
        // stale bound only prunes less; the queue size only steers donation). The read is
        // issued here and consumed after the reduction.
        poll = (++polls & (kPollK - 1)) == 0;
        if (poll && lane == 0) {
            if constexpr (kPollSmem) {
                // L2 -> shared memory (.cg: not through L1, so the line is as fresh as a relaxed
                // load's; a stale bound only prunes less, a stale size only steers donation)
                const uint32_t dst = (uint32_t)__cvta_generic_to_shared(pw);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n\tcp.async.commit_group;"
                             ::"r"(dst), "l"(ctl) : "memory");
            } else {
                h = ld_volatile_v2(ctl);
                hw = ld_relaxed_u32(&ctl->work);  // (low word: size)
            }
        }

        // visit_and_check_limits (scheduler.cpp:63-74), batched per flush_every visits
        ++st.nodes;
        if (VCG_UNLIKELY(st.nodes >= a.flush_every)) {
            int stop = 0;
            if (lane == 0) {
                // (without a node budget the total is never read back: a fire-and-forget
                // reduction, no round trip to the contended counter)
                if (a.node_budget) {
                    const unsigned long long tot =
                        atomicAdd(&ctl->nodes_total, (unsigned long long)st.nodes) + st.nodes;
                    if (tot > a.node_budget) stop = 2;
                } else {
                    atomicAdd(&ctl->nodes_total, (unsigned long long)st.nodes);
                }
                if (!stop && a.timeout_ns && globaltimer() - t_start >= a.timeout_ns) stop = 1;
                if (stop) {
                    atomicCAS(&ctl->status, 0, stop);
                    cancel_all(a);
                }
                if (worker == (MULTI ? 1u : 0u) && a.mailbox) poll_mailbox(a.mailbox, a.pvc, ctl);
                fold_stats(my_stats, st);
                if (kCntSmem) fold_cw();
            }
            reset_deltas(st);
            if (__shfl_sync(FULL, stop, 0)) break;
        }

        // a doomed child's marker: visited, pruned (markers exist only in the one-worker
        // strategies; the hybrid kernel never reads the wide node's local-memory copy here)
        if (seq_mode_ && mode == M_WIDE && x.cc == DEAD_NODE) {
            ++st.dooms;
            have = false;
            continue;
        }
        int act;
        if (VCG_LIKELY(mode == M_COMPACT)) {
            act = settle(y);
        } else if (MW && mode == M_MID) {
            act = settle(m);
            if (act == ACT_BRANCH && m.alive_count() <= kCompactSlots) {
                y.from_wide(m, sb);
                mode = M_COMPACT;
            }
        } else {
            act = settle(x);
            if (act == ACT_BRANCH && a.compact) {
                const uint32_t na = x.alive_count();
                if (na <= kCompactSlots) {
                    y.from_wide(x, sb);
                    mode = M_COMPACT;
                } else if (MW && a.mid && na <= 32u * MW) {
                    m.from_wide(x);
                    mode = M_MID;
                }
            }
        }
        if (act == ACT_BRANCH)
            act = VCG_LIKELY(mode == M_COMPACT) ? branch(y) : (MW && mode == M_MID) ? branch(m) : branch(x);
        if (act == ACT_BREAK) break;
        if (act == ACT_POP) have = false;
    }

    if (lane == 0) {
        if (kPollSmem) asm volatile("cp.async.wait_all;" ::: "memory");  // (a poll left in flight)
        if (st.nodes) atomicAdd(&ctl->nodes_total, (unsigned long long)st.nodes);
        fold_stats(my_stats, st);
        if (kCntSmem) fold_cw();
        my_stats->high_water = kCntSmem ? cw[CW_HIGH] : st.high_water;
        my_stats->active = clock64() - c_start;
        my_stats->t_begin = t0s[0];
        my_stats->t_end = globaltimer();
        my_stats->max_queue = kCntSmem ? cw[CW_MAXQ] : st.max_queue;
#pragma unroll
        for (int p = 0; p < 10; ++p) my_stats->phase[p] = INSTR ? st.phase[p] : 0ull;
    }
#undef t_start
#undef c_start
#undef sb
#undef vec16
#undef my_stats
#undef my_stack
}

// ------------------------------------------------------------------ frontier expansion

// Level-synchronous expansion (multi-GPU partitioning): warp i processes node i
// of a level exactly as process_node does (scheduler.cpp:125-144) with a FIXED bound, and writes
// its remove-N(v) child to out[2i] and its remove-v child to out[2i+1]. The result does not
// depend on scheduling, so every rank derives the same frontier.
struct ExpandArgs {
    const uint4* at4;
    uint32_t n, npad;
    int pvc;
    uint32_t k, best;
    uint32_t count;
    unsigned long long entry_bytes;
    const unsigned char* in;
    unsigned char* out;
    uint32_t* flags;   // per input: 0 pruned, 1 cover found, 2 branched
    uint32_t* covers;  // per input: [cc, bitmap W words]
};

template <int W>
__global__ void __launch_bounds__(256) expand_kernel(ExpandArgs a) {
    constexpr int Q = W / 4;
    const int lane = threadIdx.x & 31;
    for (uint32_t t = threadIdx.x; t < Q * a.npad; t += blockDim.x) dense_smem[t] = a.at4[t];
    __syncthreads();
    const uint32_t warps = gridDim.x * (blockDim.x >> 5);
    WarpNode<W, false> x;
    x.ssb = dense_scratch_base<W>(threadIdx.x >> 5);
#if VCG_WIDE_SMEM
    x.dsb = dense_degree_base<W>(threadIdx.x >> 5);
#endif
    x.lane = lane;
    Counters st;
#pragma unroll 1
    for (uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < a.count; i += warps) {
        x.load(a.in + (unsigned long long)i * a.entry_bytes);
        const int B = bound_of(a.pvc, a.k, a.best);
        x.reduce(B, st);
        uint32_t flag;
        if (x.doom || prune_at(B, x.cc, x.edges)) {
            flag = 0;
        } else if (x.edges == 0) {
            flag = 1;
            uint32_t* c = a.covers + (unsigned long long)i * (W + 1);
            const uint32_t wbits = x.cover_word();
            if (lane < W) c[1 + lane] = wbits;
            if (lane == 0) c[0] = x.cc;
        } else {
            flag = 2;
            const uint32_t v = x.argmax();
            const uint32_t xl = x.branch_mask(v);
            x.write_child(xl, __reduce_add_sync(FULL, __popc(xl)), a.out + (2ull * i) * a.entry_bytes);
            x.remove_vertex(v);
            x.store_current(a.out + (2ull * i + 1) * a.entry_bytes);
        }
        if (lane == 0) a.flags[i] = flag;
    }
}

}  // namespace vcg
