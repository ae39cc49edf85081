// sparse_kernels.cuh — device code of the sparse engine (large n, e.g. C4: BA n=100k): one
// CTA per worker, the current node's degree array resident in SHARED memory as u16.
//
// Reference path replaced: the same as the dense engine (run_hybrid, scheduler.cpp:146-212,
// process_node :125-144, reductions.cpp:7-104, search_node.cpp:16-46, worklist.cpp:11-48), with
// the reduction rules applied BLOCK-PARALLEL per round (SPEC.md §IV-D):
//   * degree one   — every leaf v takes its alive neighbour u; a leaf pair (isolated edge) lets
//                    the smaller id act; claims on a shared neighbour dedupe;
//   * degree two   — every degree-two vertex whose partners are adjacent proposes its
//                    triangle; of overlapping triangles the smallest proposer acts, so acting
//                    triangles are vertex-disjoint;
//   * high degree  — every alive vertex above the limit at the snapshot is forced into any
//                    improving cover containing S, so all are removed at once (and if more than
//                    the limit exist, the node is pruned — the dense engine's exact test).
// Each phase is sound applied to its snapshot; the fixpoint conditions are the
// reference's, so answers (MVC size, PVC yes/no) are exact, while the visited tree — and so
// node counts — may differ from the reference's sequential order.
//
// Work is incremental: a popped record gets one full scan; after that the candidate lists are
// fed by the decrement phase itself (a vertex whose degree drops to 1 or 2 is appended), |E|
// is maintained from the decrements, and the high-degree pass only scans when the max-degree
// bound exceeds the limit. One closing scan yields the smallest-id max-degree vertex.
//
// Layout: u16 degrees (0xFFFF = in the cover) in smem, decremented with 32-bit shared atomics
// on the containing word; CSR (u32 offsets / neighbours) read through L2; deferred nodes are
// 16 + 2*npad byte records {cover_count, edge_count, 0, 0, u16 degrees[npad]}.
#pragma once

#include "dense_kernels.cuh"

namespace vcg {

constexpr uint32_t SP_THREADS = 1024;  // the largest CTA (the host picks smaller ones, several
                                       // per SM; see kSparseThreads)
constexpr uint16_t DREM = 0xFFFFu;

struct SparseArgs {
    const uint32_t* off;      // CSR offsets, n+1
    const uint32_t* nbr;      // CSR neighbours, 2m
    uint32_t n, npad;         // npad: n rounded up to a multiple of 8
    int pvc;
    uint32_t k;
    uint32_t capacity, ring_mask, threshold, workers, stack_bound;
    unsigned long long entry_bytes;  // 16 + 2*npad
    unsigned char* stacks;    // workers * stack_bound * entry_bytes
    unsigned char* wl;        // ring slots * entry_bytes
    unsigned long long* seq;
    Ctl* ctl;
    uint32_t* cover_slots;    // workers * cover_words
    uint32_t cover_words;     // ceil(n / 32)
    WStats* stats;
    uint32_t* scratch;        // workers * 12n u32: A1, A2, N1, N2, L3, RL, T, P(2n), L, PP(2n)
    unsigned long long* owner;  // workers * n (triangle claims, epoch-tagged)
    uint32_t* tag;            // workers * n (phase / branch-set membership, epoch-tagged)
    uint32_t* cnt;            // workers * n (per-vertex counters, zero between uses)
    unsigned long long node_budget, timeout_ns, flush_every;
    uint32_t backoff_ns;
    int seq_mode, donate_oldest;
    int stackonly;            // StackOnly strategy (scheduler.cpp:214-297)
    uint32_t depth;
    volatile uint32_t* mailbox;
    uint16_t* gdeg;           // GDEG kernels: workers * npad u16 degree arrays in global memory
};

// CTA-wide shared control block (decisions are made here and read after a barrier)
struct SpShared {
    uint32_t a1, a2, n1, n2, cH, nrem, nT, nX, nA;  // list lengths
    uint32_t scan_total;
    uint32_t eX, ecut;                               // edge bookkeeping
    unsigned long long sumdeg, maxkey;               // scan results
    uint32_t cc, edges, doom, maxdeg;
    int outcome;
    unsigned long long pos;
    uint32_t red[32];
};

// Debug builds (VCG_SPARSE_CHECKS=1): vertex ids read from the candidate / removal lists are
// checked against n; a violation records its site in the status word (100 + site), cancels the
// search and clamps the id (the host then throws).
#ifndef VCG_SPARSE_CHECKS
#define VCG_SPARSE_CHECKS 0
#endif
#define SP_CHECK(a, id, site)                                                              \
    do {                                                                                   \
        if (VCG_SPARSE_CHECKS && (id) >= (a)->n) {                                         \
            atomicCAS(&(a)->ctl->status, 0, 100 + (site));                                 \
            atomicExch(&(a)->ctl->cancel, 1u);                                             \
            (id) = 0;                                                                      \
        }                                                                                  \
    } while (0)

// ---------------------------------------------------------------- block-level helpers

// atomically set deg[v] = 0xFFFF; returns the previous value
__device__ __forceinline__ uint32_t dclaim(uint16_t* deg, uint32_t v) {
    uint32_t* w = reinterpret_cast<uint32_t*>(deg) + (v >> 1);
    const uint32_t sh = (v & 1) * 16;
    const uint32_t old = atomicOr(w, 0xFFFFu << sh);
    return (old >> sh) & 0xFFFFu;
}
// deg[v] -= 1 for an alive v (never borrows: an alive neighbour has degree >= 1);
// returns the new degree
__device__ __forceinline__ uint32_t ddec(uint16_t* deg, uint32_t v) {
    uint32_t* w = reinterpret_cast<uint32_t*>(deg) + (v >> 1);
    const uint32_t sh = (v & 1) * 16;
    return ((atomicSub(w, 1u << sh) >> sh) & 0xFFFFu) - 1u;
}

// Warp-aggregated append of `item` (when `pred`) to list[*count++]. Warp-uniform call sites only.
__device__ __forceinline__ void append(bool pred, uint32_t item, uint32_t* list, uint32_t* count) {
    const unsigned b = __ballot_sync(FULL, pred);
    if (!b) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(b) - 1;
    uint32_t base = 0;
    if (lane == leader) base = atomicAdd(count, (uint32_t)__popc(b));
    base = __shfl_sync(FULL, base, leader);
    if (pred) list[base + __popc(b & ((1u << lane) - 1u))] = item;
}

__device__ __forceinline__ uint32_t block_sum(uint32_t x, SpShared& s) {
    x = __reduce_add_sync(FULL, x);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s.red[threadIdx.x >> 5] = x;
    __syncthreads();
    uint32_t t = (threadIdx.x < (blockDim.x >> 5)) ? s.red[threadIdx.x] : 0u;
    t = __reduce_add_sync(FULL, t);
    __syncthreads();
    if (threadIdx.x == 0) s.red[0] = t;
    __syncthreads();
    return s.red[0];
}

// Exclusive block scan of x over 1024 threads; `total` receives the sum.
__device__ __forceinline__ uint32_t block_exscan(uint32_t x, uint32_t& total, SpShared& s) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(FULL, inc, o);
        if (lane >= o) inc += y;
    }
    __syncthreads();
    if (lane == 31) s.red[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const uint32_t t = lane < (int)(blockDim.x >> 5) ? s.red[lane] : 0u;
        uint32_t ti = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, ti, o);
            if (lane >= o) ti += y;
        }
        s.red[lane] = ti - t;
        if (lane == 31) s.scan_total = ti;
    }
    __syncthreads();
    total = s.scan_total;
    const uint32_t r = s.red[wid] + inc - x;
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------- the node of one CTA

struct CtaNode {
    uint16_t* deg;        // smem, npad entries
    uint32_t* cbuf;       // smem, blockDim.x: chunk vertices
    uint32_t* cstart;     // smem, blockDim.x + 1: chunk prefix offsets
    SpShared* sh;
    const SparseArgs* a;
    uint32_t *A1, *A2, *N1, *N2;  // candidate lists: this round (A) and the next (N)
    uint32_t *L3, *RL, *T, *P;    // above-limit list, removal list, triangle proposers/partners
    uint32_t *L, *PP;             // candidates still at degree one / two; their alive partners
                                  // (PP[2v], PP[2v+1], indexed by vertex)
    uint32_t* cnt;
    unsigned long long* owner;
    uint32_t* tag;
    uint32_t epoch;
    bool fresh;           // the candidate lists describe the current degrees

    // Full scan. With `lists`, rebuilds A1 (degree one), A2 (degree two) and L3 (above lim);
    // always: alive degree sum (|E| = sum / 2) and the max-degree key (degree << 32 | ~id).
    __device__ void scan(uint32_t lim, bool lists) {
        SpShared& s = *sh;
        if (threadIdx.x == 0) {
            if (lists) s.a1 = s.a2 = s.cH = 0;
            s.sumdeg = 0;
            s.maxkey = 0;
        }
        __syncthreads();
        uint32_t sum = 0;
        unsigned long long mk = 0;
        const uint32_t n = a->n;
        const uint4* d4 = reinterpret_cast<const uint4*>(deg);
        for (uint32_t base = 0; base < a->npad; base += 8 * blockDim.x) {
            const uint32_t v0 = base + 8 * threadIdx.x;
            const uint4 q = v0 < a->npad ? d4[v0 >> 3] : make_uint4(FULL, FULL, FULL, FULL);
            bool any = false;
            uint32_t cand1 = 0, cand2 = 0, candH = 0;  // bit h: element h is a candidate
#pragma unroll
            for (int h = 0; h < 8; ++h) {
                const uint32_t d = (comp(q, h >> 1) >> (16 * (h & 1))) & 0xFFFFu;
                const uint32_t v = v0 + h;
                if (d != DREM && v < n) {
                    sum += d;
                    const unsigned long long key = ((unsigned long long)d << 32) | (0xFFFFFFFFu - v);
                    mk = key > mk ? key : mk;
                    cand1 |= (d == 1) << h;
                    cand2 |= (d == 2) << h;
                    candH |= (d > lim) << h;
                }
            }
            any = lists && (cand1 | cand2 | candH);
            if (__any_sync(FULL, any)) {
#pragma unroll
                for (int h = 0; h < 8; ++h) {
                    append((cand1 >> h) & 1u, v0 + h, A1, &s.a1);
                    append((cand2 >> h) & 1u, v0 + h, A2, &s.a2);
                    append((candH >> h) & 1u, v0 + h, L3, &s.cH);
                }
            }
        }
        sum = __reduce_add_sync(FULL, sum);
        mk = max(mk, __shfl_xor_sync(FULL, mk, 16));
        mk = max(mk, __shfl_xor_sync(FULL, mk, 8));
        mk = max(mk, __shfl_xor_sync(FULL, mk, 4));
        mk = max(mk, __shfl_xor_sync(FULL, mk, 2));
        mk = max(mk, __shfl_xor_sync(FULL, mk, 1));
        if ((threadIdx.x & 31) == 0) {
            atomicAdd(&s.sumdeg, (unsigned long long)sum);
            atomicMax(&s.maxkey, mk);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s.edges = (uint32_t)(s.sumdeg / 2);
            s.maxdeg = (uint32_t)(s.maxkey >> 32);
        }
        __syncthreads();
    }

    // f(valid, u, w) for every (u in list, w in N(u)), load-balanced over the neighbour slices
    // (block scan of the slice lengths, then a binary search per item). Every thread runs the
    // same number of iterations, so f may use warp collectives.
    template <class F>
    __device__ void for_each_neighbor(const uint32_t* list, uint32_t count, F f) {
        SpShared& s = *sh;
        for (uint32_t base = 0; base < count; base += blockDim.x) {
            const uint32_t t = base + threadIdx.x;
            uint32_t u = t < count ? list[t] : 0u;
            SP_CHECK(a, u, 1);
            const uint32_t dg = t < count ? a->off[u + 1] - a->off[u] : 0u;
            uint32_t total;
            const uint32_t st = block_exscan(dg, total, s);
            cbuf[threadIdx.x] = u;
            cstart[threadIdx.x] = st;
            __syncthreads();
            const uint32_t items = min(count - base, (uint32_t)blockDim.x);
            for (uint32_t ib = 0; ib < total; ib += blockDim.x) {
                const uint32_t idx = ib + threadIdx.x;
                const bool valid = idx < total;
                uint32_t uu = 0, w = 0;
                if (valid) {
                    uint32_t lo = 0, hi = items - 1;
                    while (lo < hi) {
                        const uint32_t mid = (lo + hi + 1) >> 1;
                        if (cstart[mid] <= idx) lo = mid;
                        else hi = mid - 1;
                    }
                    uu = cbuf[lo];
                    SP_CHECK(a, uu, 2);
                    if (VCG_SPARSE_CHECKS && a->off[uu] + (idx - cstart[lo]) >= a->off[uu + 1]) {
                        if (atomicCAS(&a->ctl->status, 0, 100 + 7) == 0) {
                            uint32_t* d = a->cover_slots;  // (diagnostics for the host)
                            d[0] = idx; d[1] = lo; d[2] = items; d[3] = total; d[4] = cstart[lo];
                            d[5] = a->off[uu + 1] - a->off[uu]; d[6] = count; d[7] = base;
                            d[8] = threadIdx.x; d[9] = lo + 1 < items ? cstart[lo + 1] : 0xFFFFFFFFu;
                            d[10] = uu; d[11] = blockDim.x;
                        }
                        atomicExch(&a->ctl->cancel, 1u);
                    }
                    w = a->nbr[a->off[uu] + (idx - cstart[lo])];
                }
                f(valid, uu, w);
            }
            __syncthreads();
        }
    }

    // Decrement the alive neighbours of the claimed RL[0..count) (all tagged with `ep`);
    // vertices whose degree drops to 1 / 2 join the candidate lists `to1` / `to2`; |E| and |S|
    // are updated (edges to alive neighbours + edges inside RL, counted once).
    __device__ void remove_claimed(uint32_t count, uint32_t ep, uint32_t* to1, uint32_t* c1,
                                   uint32_t* to2, uint32_t* c2) {
        SpShared& s = *sh;
        uint16_t* dg = deg;
        const uint32_t* tg = tag;
        uint32_t cut = 0;
        for_each_neighbor(RL, count, [&](bool valid, uint32_t u, uint32_t w) {
            uint32_t nd = 0xFFFFu;
            if (valid) {
                if (dg[w] != DREM) {
                    nd = ddec(dg, w);
                    ++cut;
                } else if (tg[w] == ep && w > u) {
                    ++cut;
                }
            }
            append(nd == 1, w, to1, c1);
            append(nd == 2, w, to2, c2);
        });
        cut = __reduce_add_sync(FULL, cut);
        if ((threadIdx.x & 31) == 0 && cut) atomicAdd(&s.ecut, cut);
        __syncthreads();
        if (threadIdx.x == 0) {
            s.cc += count;
            s.edges -= s.ecut;
            s.ecut = 0;
        }
        __syncthreads();
    }

    // graph.cpp:14-20: binary search in the shorter slice
    __device__ bool has_edge(uint32_t u, uint32_t v) const {
        const uint32_t a0 = a->off[u], a1 = a->off[u + 1], b0 = a->off[v], b1 = a->off[v + 1];
        uint32_t lo, hi, key;
        if (a1 - a0 <= b1 - b0) {
            lo = a0; hi = a1; key = v;
        } else {
            lo = b0; hi = b1; key = u;
        }
        const uint32_t end = hi;
        while (lo < hi) {
            const uint32_t mid = (lo + hi) >> 1;
            if (a->nbr[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        return lo < end && a->nbr[lo] == key;
    }

    // claim u (if still alive) into RL, tagged with the phase epoch
    __device__ __forceinline__ void claim_into_rl(bool want, uint32_t u, uint32_t ep) {
        if (want) SP_CHECK(a, u, 3);
        const bool got = want && dclaim(deg, u) != DREM;
        if (got) tag[u] = ep;
        append(got, u, RL, &sh->nrem);
    }

    // The alive partners of the candidates in `list` that still have degree `d` (1 or 2): the
    // candidates go to L (count in s.nA), their partners to PP[2v..]. The adjacency slices are
    // walked load-balanced over the whole block (for_each_neighbor): a per-thread walk of one
    // slice is a chain of dependent L2 loads as long as the vertex's ORIGINAL degree — a hub
    // that dropped to degree one kept every other thread waiting at the next barrier.
    __device__ void find_partners(const uint32_t* list, uint32_t count, uint32_t d) {
        SpShared& s = *sh;
        if (threadIdx.x == 0) s.nA = 0;
        __syncthreads();
        for (uint32_t base = 0; base < count; base += blockDim.x) {
            const uint32_t i = base + threadIdx.x;
            uint32_t v = i < count ? list[i] : 0u;
            SP_CHECK(a, v, 4);
            const bool c = i < count && deg[v] == d;
            if (c) PP[2 * v] = PP[2 * v + 1] = REM;  // (no partner found yet)
            append(c, v, L, &s.nA);
        }
        __syncthreads();
        const uint16_t* dg = deg;
        uint32_t* ct = cnt;
        uint32_t* pp = PP;
        for_each_neighbor(L, s.nA, [&](bool valid, uint32_t v, uint32_t w) {
            if (valid && dg[w] != DREM) {
                if (d == 1) {
                    pp[2 * v] = w;  // the unique alive neighbour
                } else {
                    // (bounded: a candidate listed twice walks its slice twice; the first two
                    // partners found are then not necessarily distinct, which only skips a
                    // reduction — never unsound)
                    const uint32_t slot = atomicAdd(ct + v, 1u);
                    if (slot < 2) pp[2 * v + slot] = w;
                }
            }
        });
    }

    // degree one over A1 (entries whose degree is still 1); new degree-1 vertices go to N1
    // (next round), new degree-2 ones to A2 (this round's degree-two phase)
    __device__ uint32_t phase_degree_one() {
        SpShared& s = *sh;
        const uint32_t ep = ++epoch;
        find_partners(A1, s.a1, 1);
        const uint32_t c = s.nA;
        if (threadIdx.x == 0) s.nrem = 0;
        __syncthreads();
        for (uint32_t base = 0; base < c; base += blockDim.x) {
            const uint32_t i = base + threadIdx.x;
            bool take = false;
            uint32_t u = 0;
            if (i < c) {
                const uint32_t v = L[i];
                u = PP[2 * v];
                // isolated edge: the smaller id acts (reductions.cpp:7-19 visits it first)
                take = u != REM && !(deg[u] == 1 && u < v);
            }
            claim_into_rl(take, u, ep);
        }
        __syncthreads();
        const uint32_t nrem = s.nrem;
        if (nrem) remove_claimed(nrem, ep, N1, &s.n1, A2, &s.a2);
        return nrem;
    }

    // degree two over A2 (entries whose degree is still 2); new candidates go to N1 / N2
    __device__ uint32_t phase_degree_two() {
        SpShared& s = *sh;
        const uint32_t ep = ++epoch;
        const unsigned long long key_hi = (unsigned long long)(~ep) << 32;
        find_partners(A2, s.a2, 2);
        const uint32_t c = s.nA;
        if (threadIdx.x == 0) {
            s.nT = 0;
            s.nrem = 0;
        }
        __syncthreads();
        for (uint32_t base = 0; base < c; base += blockDim.x) {
            const uint32_t i = base + threadIdx.x;
            bool tri = false;
            uint32_t v = 0, p0 = 0, p1 = 0;
            if (i < c) {
                v = L[i];
                {
                    p0 = PP[2 * v];
                    p1 = PP[2 * v + 1];
                    cnt[v] = 0;  // (counters are zero between uses)
                    tri = p0 != REM && p1 != REM && p0 != p1 && has_edge(p0, p1);
                    if (tri) {
                        const unsigned long long key = key_hi | v;
                        atomicMin(owner + v, key);
                        atomicMin(owner + p0, key);
                        atomicMin(owner + p1, key);
                    }
                }
            }
            const unsigned b = __ballot_sync(FULL, tri);
            if (b) {
                const int lane = threadIdx.x & 31, leader = __ffs(b) - 1;
                uint32_t slot = 0;
                if (lane == leader) slot = atomicAdd(&s.nT, (uint32_t)__popc(b));
                slot = __shfl_sync(FULL, slot, leader) + __popc(b & ((1u << lane) - 1u));
                if (tri) {
                    T[slot] = v;
                    P[2 * slot] = p0;
                    P[2 * slot + 1] = p1;
                }
            }
        }
        __syncthreads();
        const uint32_t nT = s.nT;
        // the smallest proposer of overlapping triangles acts: winners are vertex-disjoint
        for (uint32_t base = 0; base < nT; base += blockDim.x) {
            const uint32_t i = base + threadIdx.x;
            bool win = false;
            uint32_t v = 0, p0 = 0, p1 = 0;
            if (i < nT) {
                v = T[i];
                p0 = P[2 * i];
                p1 = P[2 * i + 1];
                const unsigned long long key = key_hi | v;
                win = owner[v] == key && owner[p0] == key && owner[p1] == key;
            }
            claim_into_rl(win, p0, ep);
            claim_into_rl(win, p1, ep);
            // a losing proposer whose triangle survives untouched must be tried again
            append(i < nT && !win, v, N2, &s.n2);
        }
        __syncthreads();
        const uint32_t nrem = s.nrem;
        if (nrem) remove_claimed(nrem, ep, N1, &s.n1, N2, &s.n2);
        return nrem;
    }

    // high degree over L3 (from a fresh scan)
    __device__ uint32_t phase_high(uint32_t lim) {
        SpShared& s = *sh;
        const uint32_t c = s.cH;
        if (c > lim) {  // every one of them would enter S: |S| passes the bound
            if (threadIdx.x == 0) s.doom = 1;
            __syncthreads();
            return 0;
        }
        const uint32_t ep = ++epoch;
        for (uint32_t i = threadIdx.x; i < c; i += blockDim.x) {
            uint32_t u = L3[i];
            SP_CHECK(a, u, 5);
            (void)dclaim(deg, u);
            tag[u] = ep;
            RL[i] = u;
        }
        __syncthreads();
        remove_claimed(c, ep, N1, &s.n1, N2, &s.n2);
        return c;
    }

    __device__ bool doomed(uint32_t snap) const {
        const SpShared& s = *sh;
        return s.doom || (a->pvc ? s.cc > a->k : s.cc >= snap);
    }

    // reduce_to_fixpoint with block-parallel rounds {degree one, degree two, high degree}
    template <class Cnt>
    __device__ void reduce(uint32_t snap, Cnt& st) {
        SpShared& s = *sh;
        if (!fresh) {
            const uint32_t lim0 = limit_for(a->pvc, a->k, snap, s.cc);
            scan(lim0, true);
            if (s.cH > lim0) {  // the doom test of phase_high, on the loaded node
                if (threadIdx.x == 0) s.doom = 1;
                __syncthreads();
                return;
            }
        }
        while (true) {
            if (s.edges == 0) break;
            const uint32_t lim = limit_for(a->pvc, a->k, snap, s.cc);
            const bool high = s.maxdeg > lim;  // an upper bound: degrees only decrease
            if (s.a1 == 0 && s.a2 == 0 && !high) break;  // no rule can fire
            ++st.rounds;
            if (threadIdx.x == 0) s.n1 = s.n2 = 0;
            __syncthreads();
            bool changed = false;
            if (s.a1) {
                const uint32_t r = phase_degree_one();
                st.rm1 += r;
                changed |= r != 0;
                if (doomed(snap)) return;
            }
            if (s.a2 && s.edges) {
                const uint32_t r = phase_degree_two();
                st.rm2 += r;
                changed |= r != 0;
                if (doomed(snap)) return;
            }
            bool rescan = false;
            const uint32_t lim2 = limit_for(a->pvc, a->k, snap, s.cc);
            if (s.maxdeg > lim2 && s.edges) {
                scan(lim2, true);  // the above-limit list needs the current degrees
                const uint32_t r = phase_high(lim2);
                st.rmh += r;
                changed |= r != 0;
                if (doomed(snap)) return;
                rescan = r != 0;  // the scan's A1/A2 predate these removals
            }
            if (rescan) {
                scan(limit_for(a->pvc, a->k, snap, s.cc), true);
            } else {
                // next round's candidates: what this round's decrements produced
                uint32_t* t;
                t = A1; A1 = N1; N1 = t;
                t = A2; A2 = N2; N2 = t;
                if (threadIdx.x == 0) {
                    s.a1 = s.n1;
                    s.a2 = s.n2;
                }
                __syncthreads();
            }
            if (!changed) break;
        }
    }

    __device__ void load_record(const unsigned char* rec) {
        const uint4* src = reinterpret_cast<const uint4*>(rec + 16);
        uint4* dst = reinterpret_cast<uint4*>(deg);
        const uint32_t nvec = a->npad / 8;
        for (uint32_t i = threadIdx.x; i < nvec; i += blockDim.x) dst[i] = __ldcg(src + i);
        if (threadIdx.x == 0) {
            const uint2 h = __ldcg(reinterpret_cast<const uint2*>(rec));
            sh->cc = h.x;
            sh->edges = h.y;
            sh->doom = 0;
        }
        fresh = false;
        __syncthreads();
    }
    // the current node as a record {cc, edges, 0, 0} + u16 degrees
    __device__ void store_current(unsigned char* rec) const {
        const uint4* s4 = reinterpret_cast<const uint4*>(deg);
        uint4* d4 = reinterpret_cast<uint4*>(rec + 16);
        for (uint32_t i = threadIdx.x; i < a->npad / 8; i += blockDim.x) d4[i] = s4[i];
        if (threadIdx.x == 0) *reinterpret_cast<uint4*>(rec) = make_uint4(sh->cc, sh->edges, 0u, 0u);
        __syncthreads();
    }
    __device__ void copy_record(const unsigned char* src, unsigned char* dst) const {
        const uint4* s4 = reinterpret_cast<const uint4*>(src);
        uint4* d4 = reinterpret_cast<uint4*>(dst);
        const uint32_t nvec = (uint32_t)(a->entry_bytes / 16);
        for (uint32_t i = threadIdx.x; i < nvec; i += blockDim.x) d4[i] = __ldcg(s4 + i);
        __syncthreads();
    }

    // The remove-N(v) child written straight to `rec`: copy the degrees, cover X = N(v) ∩
    // alive, and subtract from each affected survivor w its number of neighbours in X.
    __device__ void write_child(uint32_t v, unsigned char* rec) {
        SpShared& s = *sh;
        const uint32_t ep = ++epoch;
        if (threadIdx.x == 0) {
            s.nX = 0;
            s.nA = 0;
            s.eX = 0;
        }
        __syncthreads();
        // X (in RL), tagged with the epoch
        const uint32_t b0 = a->off[v], b1 = a->off[v + 1];
        for (uint32_t base = b0; base < b1; base += blockDim.x) {
            const uint32_t e = base + threadIdx.x;
            const uint32_t w = e < b1 ? a->nbr[e] : 0u;
            const bool al = e < b1 && deg[w] != DREM;
            if (al) tag[w] = ep;
            append(al, w, RL, &s.nX);
        }
        // bulk copy of the parent's degrees
        uint4* d4 = reinterpret_cast<uint4*>(rec + 16);
        const uint4* s4 = reinterpret_cast<const uint4*>(deg);
        for (uint32_t i = threadIdx.x; i < a->npad / 8; i += blockDim.x) d4[i] = s4[i];
        __syncthreads();
        const uint32_t nX = s.nX;
        uint16_t* rd = reinterpret_cast<uint16_t*>(rec + 16);
        uint32_t sx = 0;
        for (uint32_t i = threadIdx.x; i < nX; i += blockDim.x) {
            uint32_t u = RL[i];
            SP_CHECK(a, u, 6);
            sx += deg[u];
            rd[u] = DREM;
        }
        sx = block_sum(sx, s);
        // count each survivor's neighbours in X
        const uint16_t* dg = deg;
        uint32_t* tg = tag;
        uint32_t* ct = cnt;
        uint32_t* LA = A1;  // free after the reduction
        uint32_t ex = 0;
        for_each_neighbor(RL, nX, [&](bool valid, uint32_t u, uint32_t w) {
            bool first = false;
            if (valid && dg[w] != DREM) {
                if (tg[w] == ep) ex += w > u;
                else first = atomicAdd(ct + w, 1u) == 0u;
            }
            append(first, w, LA, &s.nA);
        });
        ex = __reduce_add_sync(FULL, ex);
        if ((threadIdx.x & 31) == 0 && ex) atomicAdd(&s.eX, ex);
        __syncthreads();
        const uint32_t na = s.nA;
        for (uint32_t i = threadIdx.x; i < na; i += blockDim.x) {
            const uint32_t w = LA[i];
            rd[w] = (uint16_t)(deg[w] - cnt[w]);
            cnt[w] = 0;
        }
        if (threadIdx.x == 0) {
            const uint32_t cc2 = s.cc + nX;
            const uint32_t e2 = s.edges - sx + s.eX;
            *reinterpret_cast<uint4*>(rec) = make_uint4(cc2, e2, 0, 0);
        }
        __syncthreads();
    }

    // search_node.cpp:16-25 for the branch vertex (the remove-v child); its decrements seed
    // the child's candidate lists, so its reduction needs no opening scan.
    __device__ void remove_branch_vertex(uint32_t v) {
        SpShared& s = *sh;
        const uint32_t ep = ++epoch;
        if (threadIdx.x == 0) {
            (void)dclaim(deg, v);
            tag[v] = ep;
            RL[0] = v;
            s.a1 = s.a2 = 0;
            s.doom = 0;
        }
        __syncthreads();
        remove_claimed(1, ep, A1, &s.a1, A2, &s.a2);
        fresh = true;  // maxdeg from the closing scan stays a valid upper bound
    }
};

// One CTA's node and its per-worker scratch (lists in global memory, claims, tags, counters).
template <bool GDEG>
__device__ __forceinline__ void init_cta_node(CtaNode& x, const SparseArgs& a, uint32_t worker,
                                              uint4* smem4, SpShared& sh) {
    if constexpr (GDEG) {
        x.deg = a.gdeg + (unsigned long long)worker * a.npad;
        x.cbuf = reinterpret_cast<uint32_t*>(smem4);
    } else {
        x.deg = reinterpret_cast<uint16_t*>(smem4);
        x.cbuf = reinterpret_cast<uint32_t*>(x.deg + a.npad);
    }
    x.cstart = x.cbuf + blockDim.x;
    x.sh = &sh;
    x.a = &a;
    uint32_t* scr = a.scratch + (unsigned long long)worker * 12ull * a.n;
    x.A1 = scr;
    x.A2 = scr + 1ull * a.n;
    x.N1 = scr + 2ull * a.n;
    x.N2 = scr + 3ull * a.n;
    x.L3 = scr + 4ull * a.n;
    x.RL = scr + 5ull * a.n;
    x.T = scr + 6ull * a.n;
    x.P = scr + 7ull * a.n;  // 2n
    x.L = scr + 9ull * a.n;
    x.PP = scr + 10ull * a.n;  // 2n
    x.cnt = a.cnt + (unsigned long long)worker * a.n;
    x.owner = a.owner + (unsigned long long)worker * a.n;
    x.tag = a.tag + (unsigned long long)worker * a.n;
    x.epoch = 0;
    x.fresh = false;
}

// GDEG: the global-memory node variant for graphs whose degree array does not
// fit in shared memory (n beyond ~110k): the current node's u16 degrees live in a per-worker
// array in global memory (L2-resident: 148 workers x 2n bytes), everything else is unchanged.
template <bool INSTR, bool GDEG = false>
__global__ void __launch_bounds__(SP_THREADS, 1) sparse_kernel(SparseArgs a) {
    extern __shared__ uint4 smem4[];
    __shared__ SpShared sh;
    const uint32_t worker = blockIdx.x;
    if (worker >= a.workers) return;
    const int tid = threadIdx.x;

    CtaNode x;
    init_cta_node<GDEG>(x, a, worker, smem4, sh);
    if (tid == 0) sh.ecut = 0;

    const unsigned long long t_start = globaltimer();
    const long long c_start = clock64();
    Counters st;
    Ctl* ctl = a.ctl;
    unsigned char* const my_stack =
        a.stacks + (unsigned long long)worker * a.stack_bound * a.entry_bytes;
    uint32_t base = 0, sp = 0;
    auto slot_at = [&](uint32_t i) {
        uint32_t j = base + i;
        if (j >= a.stack_bound) j -= a.stack_bound;
        return my_stack + (unsigned long long)j * a.entry_bytes;
    };
    bool have = false, idle = true;
    unsigned long long subtree = 0;  // StackOnly: current sub-tree id
    uint32_t replay = 0xFFFFFFFFu;   // StackOnly: root-path levels replayed so far
    uint32_t best = a.pvc ? a.k : ctl->best;
    unsigned long long nodes_flushed = 0;

    while (true) {
        if (!have) {
            if (sp > 0) {
                --sp;
                x.load_record(slot_at(sp));
            } else if (a.stackonly) {
                // stackonly_worker (scheduler.cpp:279-281): next sub-tree id, replay from the root
                if (tid == 0) {
                    const unsigned long long t = atomicAdd(&ctl->head, 1ull);
                    sh.outcome = (t >> a.depth) == 0 && !ld_volatile_v4(ctl).y;
                    sh.pos = t;
                }
                __syncthreads();
                if (!sh.outcome) break;
                subtree = sh.pos;
                replay = 0;
                x.load_record(a.wl);
            } else {
                // GlobalWorklist::remove_or_done: ticket, then publication / termination / cancel
                if (tid == 0) {
                    if (!idle) atomicAdd(&ctl->work, ~ONE_PENDING + 1ull);
                    const unsigned long long pos = atomicAdd(&ctl->head, 1ull);
                    unsigned long long* rel = a.seq + (pos & a.ring_mask);
                    uint32_t sleep = 32;
                    int o = 0;
                    for (uint32_t spin = 0;; ++spin) {
                        if (ld_acquire_u64(rel) == pos + 1) { o = 1; break; }
                        if ((spin & 7) == 7) {
                            if (ld_volatile_v4(ctl).y) { o = 2; break; }
                            if ((ld_relaxed_u64(&ctl->work) >> 32) == 0) { o = 2; break; }
                            if (worker == 0 && a.mailbox) poll_mailbox(a.mailbox, a.pvc, ctl);
                        }
                        __nanosleep(sleep);
                        sleep = min(sleep * 2, a.backoff_ns);
                    }
                    sh.outcome = o;
                    sh.pos = pos;
                }
                idle = true;
                __syncthreads();
                if (sh.outcome == 2) break;
                const unsigned long long pos = sh.pos;
                unsigned long long* rel = a.seq + (pos & a.ring_mask);
                (void)ld_acquire_u64(rel);
                x.load_record(a.wl + (pos & a.ring_mask) * a.entry_bytes);
                __threadfence();
                __syncthreads();
                if (tid == 0) {
                    st_release_u64(rel, pos + a.ring_mask + 1);
                    atomicAdd(&ctl->work, ~0ull);
                }
                idle = false;
            }
            have = true;
        }

        // control line, node counter, limits (thread 0), broadcast through shared memory
        ++st.nodes;
        if (tid == 0) {
            const uint4 h = ld_volatile_v4(ctl);
            sh.red[0] = h.y;
            sh.red[1] = h.x;
            sh.red[2] = (uint32_t)ld_relaxed_u64(&ctl->work);
            int stop = 0;
            if (st.nodes - nodes_flushed >= a.flush_every) {
                const unsigned long long tot =
                    atomicAdd(&ctl->nodes_total, st.nodes - nodes_flushed) + (st.nodes - nodes_flushed);
                nodes_flushed = st.nodes;
                if (a.node_budget && tot > a.node_budget) stop = 2;
                else if (a.timeout_ns && globaltimer() - t_start >= a.timeout_ns) stop = 1;
                if (stop) {
                    atomicCAS(&ctl->status, 0, stop);
                    atomicExch(&ctl->cancel, 1u);
                }
                if (worker == 0 && a.mailbox) poll_mailbox(a.mailbox, a.pvc, ctl);
            }
            sh.red[3] = stop;
        }
        __syncthreads();
        const uint32_t cancel = sh.red[0], hbest = sh.red[1], qsize = sh.red[2], stop = sh.red[3];
        __syncthreads();
        if (cancel || stop) break;
        if (!a.pvc) best = min(best, hbest);

        // process_node
        x.reduce(best, st);
        // The reduced node's state, read by every thread BEFORE anyone moves on: a thread that
        // prunes and pops the next record rewrites sh.cc / sh.edges / sh.doom (load_record)
        // while a slower warp may still be deciding on this node — with small CTAs that skew
        // split the CTA's control flow and desynchronised its barriers.
        const uint32_t ncc = sh.cc, nedges = sh.edges;
        const bool ndoom = sh.doom != 0;
        __syncthreads();
        const bool prune = ndoom || should_prune(a.pvc, a.k, best, ncc, nedges);
        st.dooms += ndoom;
        if (prune) {
            have = false;
            continue;
        }
        if (nedges == 0) {
            if (tid == 0) {
                uint32_t rec;
                if (a.pvc) rec = atomicCAS(&ctl->found, 0u, 1u) == 0u;
                else rec = ncc < atomicMin(&ctl->best, ncc);
                sh.red[4] = rec;
            }
            __syncthreads();
            if (sh.red[4]) {
                uint32_t* slot = a.cover_slots + (unsigned long long)worker * a.cover_words;
                for (uint32_t w = tid; w < a.cover_words; w += blockDim.x) {
                    uint32_t bits = 0;
                    for (int j = 0; j < 32; ++j) {
                        const uint32_t v = 32 * w + j;
                        if (v < a.n && x.deg[v] == DREM) bits |= 1u << j;
                    }
                    slot[w] = bits;
                }
                __threadfence();
                __syncthreads();
                if (tid == 0) {
                    atomicMin(&ctl->best_owner, ((unsigned long long)ncc << 32) | worker);
                    if (a.pvc) atomicExch(&ctl->cancel, 1u);
                    if (a.mailbox) {
                        a.mailbox[2] = ncc;
                        if (a.pvc) a.mailbox[3] = 1;
                    }
                }
            }
            __syncthreads();
            if (a.pvc) break;
            best = min(best, ncc);
            have = false;
            continue;
        }
        // the smallest id among max-degree alive vertices (search_node.cpp:34-46)
        x.scan(0xFFFFu, false);
        const uint32_t v = 0xFFFFFFFFu - (uint32_t)(sh.maxkey & 0xFFFFFFFFull);
        ++st.maxdeg;
        if (v >= a.n) {  // invariant: |E| > 0 implies an alive vertex (fail loudly, status 4)
            if (tid == 0) {
                atomicCAS(&ctl->status, 0, 4);
                atomicExch(&ctl->cancel, 1u);
                a.cover_slots[0] = sh.edges;
                a.cover_slots[1] = sh.cc;
                a.cover_slots[2] = (uint32_t)sh.sumdeg;
            }
            break;
        }

        // branch (scheduler.cpp:185-203)
        unsigned char* child = nullptr;
        unsigned long long* publish = nullptr;
        unsigned long long pos = 0;
        if (!a.seq_mode && qsize < a.threshold) {
            if (tid == 0) {
                const unsigned long long old = atomicAdd(&ctl->work, ONE_PENDING | 1ull);
                int ok = (uint32_t)old < a.capacity;
                if (!ok) {
                    atomicAdd(&ctl->work, ~(ONE_PENDING | 1ull) + 1ull);
                } else {
                    st.max_queue = max(st.max_queue, (unsigned long long)((uint32_t)old + 1));
                    sh.pos = atomicAdd(&ctl->tail, 1ull);
                    // (gives up after a cancel: the previous lap's reader may have left)
                    if (ld_acquire_u64(a.seq + (sh.pos & a.ring_mask)) != sh.pos)
                        ok = wait_slot_free(a.seq + (sh.pos & a.ring_mask), sh.pos, &ctl->cancel, false);
                }
                sh.outcome = ok;
            }
            __syncthreads();
            if (sh.outcome) {
                pos = sh.pos;
                publish = a.seq + (pos & a.ring_mask);
                unsigned char* dst = a.wl + (pos & a.ring_mask) * a.entry_bytes;
                if (a.donate_oldest && sp > 0) {
                    x.copy_record(slot_at(0), dst);
                    base = base + 1 == a.stack_bound ? 0 : base + 1;
                    --sp;
                } else {
                    child = dst;
                }
                ++st.donated;
            }
            __syncthreads();
        }
        // StackOnly replay: bit `replay` of the sub-tree id picks the child, nothing deferred
        const bool replaying = a.stackonly && replay < a.depth;
        const bool right = replaying && ((subtree >> replay) & 1ull);
        replay += replaying;
        if (!replaying || right) {
            if (!child && sp >= a.stack_bound && !a.seq_mode) {
                // The local stack reached its device-memory cap: its oldest node moves to the
                // device worklist (the shared HBM pool), whatever the donation threshold.
                if (tid == 0) {
                    int ok = 0;
                    const unsigned long long old = atomicAdd(&ctl->work, ONE_PENDING | 1ull);
                    if ((uint32_t)old >= a.capacity) {
                        atomicAdd(&ctl->work, ~(ONE_PENDING | 1ull) + 1ull);
                    } else {
                        sh.pos = atomicAdd(&ctl->tail, 1ull);
                        ok = 1;
                        if (ld_acquire_u64(a.seq + (sh.pos & a.ring_mask)) != sh.pos)
                            ok = wait_slot_free(a.seq + (sh.pos & a.ring_mask), sh.pos, &ctl->cancel, false) ? 1 : 2;
                    }
                    sh.outcome = ok;
                }
                __syncthreads();
                const int ok = sh.outcome;
                if (ok == 1) {
                    const unsigned long long p2 = sh.pos;
                    x.copy_record(slot_at(0), a.wl + (p2 & a.ring_mask) * a.entry_bytes);
                    base = base + 1 == a.stack_bound ? 0 : base + 1;
                    --sp;
                    ++st.donated;
                    __threadfence();
                    __syncthreads();
                    if (tid == 0) st_release_u64(a.seq + (p2 & a.ring_mask), p2 + 1);
                }
            }
            if (!child) {
                if (sp >= a.stack_bound) {  // the worklist is full too: fail loudly
                    if (tid == 0) {
                        atomicCAS(&ctl->status, 0, 3);
                        atomicExch(&ctl->cancel, 1u);
                    }
                    break;
                }
                child = slot_at(sp);
                ++sp;
                if (sp > st.high_water) st.high_water = sp;
            }
            x.write_child(v, child);
            ++st.children;
        }
        if (publish) {
            __threadfence();
            __syncthreads();
            if (tid == 0) st_release_u64(publish, pos + 1);
        }
        if (right) {  // continue with the remove-N(v) child just stacked
            have = false;
            continue;
        }
        x.remove_branch_vertex(v);
    }

    __syncthreads();
    if (tid == 0) {
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
        o.peer = 0;
        o.active = clock64() - c_start;
        o.max_queue = st.max_queue;
        o.t_begin = o.t_first = o.t_end = o.t_idle = o.t_lastwait = 0;  // (the timeline is the dense engine's)
#pragma unroll
        for (int p = 0; p < 10; ++p) o.phase[p] = 0;
        a.stats[worker] = o;
        (void)t_start;
    }
}

// Level-synchronous frontier expansion on the sparse engine (multi-GPU partitioning for large
// n): CTA i processes node i of a level exactly as process_node does
// (scheduler.cpp:125-144) with a FIXED bound, writes its remove-N(v) child to out[2i] and its
// remove-v child to out[2i+1]. The block-parallel rules reach the same fixpoint whatever the
// thread schedule, so every rank derives the same frontier.
struct SparseExpandArgs {
    SparseArgs s;             // graph, scratch (gridDim.x workers), gdeg
    const unsigned char* in;
    unsigned char* out;
    uint32_t* flags;          // per input: 0 pruned, 1 cover found, 2 branched
    uint32_t* covers;         // per input: [cc, bitmap cover_words]
    uint32_t count, best;
};

template <bool GDEG>
__global__ void __launch_bounds__(SP_THREADS, 1) sparse_expand_kernel(SparseExpandArgs e) {
    extern __shared__ uint4 smem4[];
    __shared__ SpShared sh;
    const SparseArgs& a = e.s;
    CtaNode x;
    init_cta_node<GDEG>(x, a, blockIdx.x, smem4, sh);
    if (threadIdx.x == 0) sh.ecut = 0;
    Counters st;
    for (uint32_t i = blockIdx.x; i < e.count; i += gridDim.x) {
        x.load_record(e.in + (unsigned long long)i * a.entry_bytes);
        x.reduce(e.best, st);
        uint32_t flag;
        if (sh.doom || should_prune(a.pvc, a.k, e.best, sh.cc, sh.edges)) {
            flag = 0;
        } else if (sh.edges == 0) {
            flag = 1;
            uint32_t* c = e.covers + (unsigned long long)i * (a.cover_words + 1);
            for (uint32_t w = threadIdx.x; w < a.cover_words; w += blockDim.x) {
                uint32_t bits = 0;
                for (int j = 0; j < 32; ++j) {
                    const uint32_t v = 32 * w + j;
                    if (v < a.n && x.deg[v] == DREM) bits |= 1u << j;
                }
                c[1 + w] = bits;
            }
            if (threadIdx.x == 0) c[0] = sh.cc;
        } else {
            flag = 2;
            x.scan(0xFFFFu, false);
            const uint32_t v = 0xFFFFFFFFu - (uint32_t)(sh.maxkey & 0xFFFFFFFFull);
            x.write_child(v, e.out + (2ull * i) * a.entry_bytes);
            x.remove_branch_vertex(v);
            x.store_current(e.out + (2ull * i + 1) * a.entry_bytes);
        }
        if (threadIdx.x == 0) e.flags[i] = flag;
        __syncthreads();
    }
}

}  // namespace vcg
