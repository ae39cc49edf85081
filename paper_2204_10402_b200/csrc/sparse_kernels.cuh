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
//                    the limit exist, the node is pruned — the same exact test as the dense
//                    engine's).
// Each phase is sound applied to the snapshot (DESIGN.md §4 has the arguments); the fixpoint
// conditions are the reference's, so answers (MVC size, PVC yes/no) are exact, while the
// visited tree — and so node counts — may differ from the reference's sequential order.
//
// Layout: u16 degrees (0xFFFF = in the cover) in smem, decremented with 32-bit shared atomics
// on the containing word; CSR (u32 offsets / neighbours) read through L2; deferred nodes are
// 16 + 2*npad byte records {cover_count, edge_count, 0, 0, u16 degrees[npad]}.
#pragma once

#include "dense_kernels.cuh"

namespace vcg {

constexpr uint32_t SP_THREADS = 1024;
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
    uint32_t* scratch;        // workers * 8n: L1, L2, L3, RL, T, cnt, P (2n)
    unsigned long long* owner;  // workers * n (triangle claims, epoch-tagged)
    uint32_t* tag;            // workers * n (branch-set membership, epoch-tagged)
    unsigned long long node_budget, timeout_ns, flush_every;
    uint32_t backoff_ns;
    int seq_mode, donate_oldest;
    volatile uint32_t* mailbox;
};

// CTA-wide shared control block (decisions are made here and read after a barrier)
struct SpShared {
    uint32_t c1, c2, cH, nrem, nT, nX, nA;   // list lengths
    uint32_t scan_total;
    uint32_t eX, sumX;                        // branch bookkeeping
    unsigned long long sumdeg, maxkey;        // scan results
    uint32_t cc, edges, doom;
    int outcome;
    unsigned long long pos;
    uint32_t red[32];                         // block reductions
    unsigned long long red64[32];
};

// ---------------------------------------------------------------- block-level helpers

__device__ __forceinline__ uint16_t dget(const uint16_t* deg, uint32_t v) { return deg[v]; }

// atomically set deg[v] = 0xFFFF; returns the previous value
__device__ __forceinline__ uint32_t dclaim(uint16_t* deg, uint32_t v) {
    uint32_t* w = reinterpret_cast<uint32_t*>(deg) + (v >> 1);
    const uint32_t sh = (v & 1) * 16;
    const uint32_t old = atomicOr(w, 0xFFFFu << sh);
    return (old >> sh) & 0xFFFFu;
}
// deg[v] -= 1 for an alive v (never borrows: an alive neighbour has degree >= 1)
__device__ __forceinline__ void ddec(uint16_t* deg, uint32_t v) {
    uint32_t* w = reinterpret_cast<uint32_t*>(deg) + (v >> 1);
    atomicSub(w, 1u << ((v & 1) * 16));
}

// Warp-aggregated append of `item` (when `pred`) to list[*count++].
__device__ __forceinline__ void append(bool pred, uint32_t item, uint32_t* list, uint32_t* count) {
    const unsigned b = __ballot_sync(FULL, pred);
    if (!b) return;
    const int lane = threadIdx.x & 31;
    uint32_t base = 0;
    if (lane == __ffs(b) - 1) base = atomicAdd(count, (uint32_t)__popc(b));
    base = __shfl_sync(FULL, base, __ffs(b) - 1);
    if (pred) list[base + __popc(b & ((1u << lane) - 1u))] = item;
}

__device__ __forceinline__ uint32_t block_sum(uint32_t x, SpShared& s) {
    x = __reduce_add_sync(FULL, x);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) s.red[threadIdx.x >> 5] = x;
    __syncthreads();
    uint32_t t = (threadIdx.x < 32) ? s.red[threadIdx.x] : 0u;
    t = __reduce_add_sync(FULL, t);
    __syncthreads();
    if (threadIdx.x == 0) s.red[0] = t;
    __syncthreads();
    return s.red[0];
}

// Exclusive block scan of x over 1024 threads; returns the exclusive prefix, total via ref.
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
        uint32_t t = s.red[lane], ti = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, ti, o);
            if (lane >= o) ti += y;
        }
        s.red[lane] = ti - t;  // exclusive warp offsets
        if (lane == 31) s.scan_total = ti;
    }
    __syncthreads();
    total = s.scan_total;
    const uint32_t r = s.red[wid] + inc - x;
    __syncthreads();
    return r;
}

// ---------------------------------------------------------------- the node of one CTA

template <bool INSTR>
struct CtaNode {
    uint16_t* deg;        // smem, npad entries
    uint32_t* cbuf;       // smem, SP_THREADS: chunk vertices
    uint32_t* cstart;     // smem, SP_THREADS + 1: chunk prefix offsets
    SpShared* sh;
    const SparseArgs* a;
    uint32_t* L1;         // global scratch lists (n each)
    uint32_t* L2;
    uint32_t* L3;
    uint32_t* RL;         // removal list (claimed vertices)
    uint32_t* T;          // triangle proposers
    uint32_t* P;          // their partners (2 per proposer)
    uint32_t* cnt;        // per-vertex counters, all zero between uses
    unsigned long long* owner;
    uint32_t* tag;
    uint32_t epoch;

    // Full scan: degree-one / degree-two / above-limit candidate lists, alive degree sum and
    // the max-degree key (degree << 32 | ~id: smallest id wins ties).
    __device__ void scan(uint32_t lim, bool lists) {
        SpShared& s = *sh;
        if (threadIdx.x == 0) {
            s.c1 = s.c2 = s.cH = 0;
            s.sumdeg = 0;
            s.maxkey = 0;
        }
        __syncthreads();
        uint32_t sum = 0;
        unsigned long long mk = 0;
        const uint32_t n = a->n;
        for (uint32_t base = 0; base < n; base += 2 * SP_THREADS) {
            const uint32_t v0 = base + 2 * threadIdx.x;
            uint32_t pair = v0 < n ? reinterpret_cast<const uint32_t*>(deg)[v0 >> 1] : 0xFFFFFFFFu;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t v = v0 + h;
                const uint32_t d = (pair >> (16 * h)) & 0xFFFFu;
                const bool al = v < n && d != DREM;
                if (al) {
                    sum += d;
                    const unsigned long long key = ((unsigned long long)d << 32) | (0xFFFFFFFFu - v);
                    mk = key > mk ? key : mk;
                }
                if (lists) {
                    append(al && d == 1, v, L1, &s.c1);
                    append(al && d == 2, v, L2, &s.c2);
                    append(al && d > lim, v, L3, &s.cH);
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
        if (threadIdx.x == 0) s.edges = (uint32_t)(s.sumdeg / 2);
        __syncthreads();
    }

    // Decrement the alive neighbours of every vertex of list[0..count) (already claimed),
    // load-balanced over the neighbour slices with a block scan (merge-path style).
    template <class F>
    __device__ void for_each_neighbor(const uint32_t* list, uint32_t count, F f) {
        SpShared& s = *sh;
        for (uint32_t base = 0; base < count; base += SP_THREADS) {
            const uint32_t t = base + threadIdx.x;
            const uint32_t u = t < count ? list[t] : 0u;
            const uint32_t dg = t < count ? a->off[u + 1] - a->off[u] : 0u;
            uint32_t total;
            const uint32_t st = block_exscan(dg, total, s);
            cbuf[threadIdx.x] = u;
            cstart[threadIdx.x] = st;
            if (threadIdx.x == 0) cstart[SP_THREADS] = total;
            __syncthreads();
            const uint32_t items = min(count - base, SP_THREADS);
            for (uint32_t idx = threadIdx.x; idx < total; idx += SP_THREADS) {
                // last j with cstart[j] <= idx
                uint32_t lo = 0, hi = items - 1;
                while (lo < hi) {
                    const uint32_t mid = (lo + hi + 1) >> 1;
                    if (cstart[mid] <= idx) lo = mid;
                    else hi = mid - 1;
                }
                const uint32_t uu = cbuf[lo];
                f(uu, a->nbr[a->off[uu] + (idx - cstart[lo])]);
            }
            __syncthreads();
        }
    }

    __device__ void remove_claimed(uint32_t count) {
        uint16_t* dg = deg;
        for_each_neighbor(RL, count, [dg](uint32_t, uint32_t w) {
            if (dg[w] != DREM) ddec(dg, w);
        });
        if (threadIdx.x == 0) sh->cc += count;
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

    // Returns the number of vertices this phase put into the cover.
    __device__ uint32_t phase_degree_one() {
        SpShared& s = *sh;
        const uint32_t c1 = s.c1;
        if (threadIdx.x == 0) s.nrem = 0;
        __syncthreads();
        for (uint32_t base = 0; base < c1; base += SP_THREADS) {
            const uint32_t i = base + threadIdx.x;
            bool take = false;
            uint32_t u = 0;
            if (i < c1) {
                const uint32_t v = L1[i];
                for (uint32_t e = a->off[v]; e < a->off[v + 1]; ++e) {
                    const uint32_t w = a->nbr[e];
                    if (deg[w] != DREM) {
                        u = w;
                        take = true;
                        break;
                    }
                }
                // isolated edge: the smaller id acts (reductions.cpp:7-19 visits it first)
                if (take && deg[u] == 1 && u < v) take = false;
                if (take) take = dclaim(deg, u) != DREM;
            }
            append(take, u, RL, &s.nrem);
        }
        __syncthreads();
        const uint32_t nrem = s.nrem;
        if (nrem) remove_claimed(nrem);
        return nrem;
    }

    __device__ uint32_t phase_degree_two() {
        SpShared& s = *sh;
        const uint32_t c2 = s.c2;
        ++epoch;
        const unsigned long long ep = (unsigned long long)(~epoch) << 32;
        if (threadIdx.x == 0) s.nT = 0;
        __syncthreads();
        // propose triangles (T: proposers, P: their partners)
        for (uint32_t base = 0; base < c2; base += SP_THREADS) {
            const uint32_t i = base + threadIdx.x;
            bool tri = false;
            uint32_t v = 0, p0 = 0, p1 = 0;
            if (i < c2) {
                v = L2[i];
                int f = 0;
                for (uint32_t e = a->off[v]; e < a->off[v + 1] && f < 2; ++e) {
                    const uint32_t w = a->nbr[e];
                    if (deg[w] != DREM) {
                        if (f == 0) p0 = w;
                        else p1 = w;
                        ++f;
                    }
                }
                tri = f == 2 && has_edge(p0, p1);
                if (tri) {
                    const unsigned long long key = ep | v;
                    atomicMin(owner + v, key);
                    atomicMin(owner + p0, key);
                    atomicMin(owner + p1, key);
                }
            }
            const unsigned b = __ballot_sync(FULL, tri);
            const int lane = threadIdx.x & 31;
            uint32_t slot = 0;
            if (b) {
                if (lane == __ffs(b) - 1) slot = atomicAdd(&s.nT, (uint32_t)__popc(b));
                slot = __shfl_sync(FULL, slot, __ffs(b) - 1) + __popc(b & ((1u << lane) - 1u));
                if (tri) {
                    T[slot] = v;
                    P[2 * slot] = p0;
                    P[2 * slot + 1] = p1;
                }
            }
        }
        __syncthreads();
        const uint32_t nT = s.nT;
        if (threadIdx.x == 0) s.nrem = 0;
        __syncthreads();
        // vertex-disjoint winners remove both partners
        for (uint32_t base = 0; base < nT; base += SP_THREADS) {
            const uint32_t i = base + threadIdx.x;
            bool win = false;
            uint32_t p0 = 0, p1 = 0;
            if (i < nT) {
                const uint32_t v = T[i];
                p0 = P[2 * i];
                p1 = P[2 * i + 1];
                const unsigned long long key = ep | v;
                win = owner[v] == key && owner[p0] == key && owner[p1] == key;
            }
            const bool c0 = win && dclaim(deg, p0) != DREM;
            const bool c1 = win && dclaim(deg, p1) != DREM;
            append(c0, p0, RL, &s.nrem);
            append(c1, p1, RL, &s.nrem);
        }
        __syncthreads();
        const uint32_t nrem = s.nrem;
        if (nrem) remove_claimed(nrem);
        return nrem;
    }

    __device__ uint32_t phase_high(uint32_t lim) {
        SpShared& s = *sh;
        const uint32_t cH = s.cH;
        if (cH > lim) {  // every one of them would enter S: |S| passes the bound
            if (threadIdx.x == 0) s.doom = 1;
            __syncthreads();
            return 0;
        }
        for (uint32_t i = threadIdx.x; i < cH; i += SP_THREADS) {
            const uint32_t u = L3[i];
            (void)dclaim(deg, u);
            RL[i] = u;
        }
        __syncthreads();
        remove_claimed(cH);
        return cH;
    }

    __device__ bool doomed(uint32_t snap) const {
        const SpShared& s = *sh;
        return s.doom || (a->pvc ? s.cc > a->k : s.cc >= snap);
    }

    // reduce_to_fixpoint with block-parallel rounds {degree one, degree two, high degree}
    template <class Cnt>
    __device__ void reduce(uint32_t snap, Cnt& st) {
        SpShared& s = *sh;
        while (true) {
            uint32_t lim = limit_for(a->pvc, a->k, snap, s.cc);
            scan(lim, true);
            if (s.edges == 0) break;
            ++st.rounds;
            if (s.c1 == 0 && s.c2 == 0 && s.cH == 0) break;  // no rule can fire
            bool changed = false;
            if (s.c1) {
                const uint32_t r = phase_degree_one();
                st.rm1 += r;
                changed |= r != 0;
                if (doomed(snap)) return;
                if (r) scan(limit_for(a->pvc, a->k, snap, s.cc), true);
            }
            if (s.c2 && s.edges) {
                const uint32_t r = phase_degree_two();
                st.rm2 += r;
                changed |= r != 0;
                if (doomed(snap)) return;
                if (r) scan(limit_for(a->pvc, a->k, snap, s.cc), true);
            }
            lim = limit_for(a->pvc, a->k, snap, s.cc);
            if (s.cH && s.edges) {
                const uint32_t r = phase_high(lim);
                st.rmh += r;
                changed |= r != 0;
                if (doomed(snap)) return;
            }
            if (!changed) break;  // the last scan saw no applicable rule
        }
    }

    __device__ void load_record(const unsigned char* rec) {
        const uint4* src = reinterpret_cast<const uint4*>(rec + 16);
        uint4* dst = reinterpret_cast<uint4*>(deg);
        const uint32_t nvec = a->npad / 8;
        for (uint32_t i = threadIdx.x; i < nvec; i += SP_THREADS) dst[i] = __ldcg(src + i);
        if (threadIdx.x == 0) {
            const uint2 h = __ldcg(reinterpret_cast<const uint2*>(rec));
            sh->cc = h.x;
            sh->edges = h.y;
            sh->doom = 0;
        }
        __syncthreads();
    }
    __device__ void copy_record(const unsigned char* src, unsigned char* dst) const {
        const uint4* s4 = reinterpret_cast<const uint4*>(src);
        uint4* d4 = reinterpret_cast<uint4*>(dst);
        const uint32_t nvec = (uint32_t)(a->entry_bytes / 16);
        for (uint32_t i = threadIdx.x; i < nvec; i += SP_THREADS) d4[i] = __ldcg(s4 + i);
        __syncthreads();
    }

    // The remove-N(v) child written straight to `rec`: copy the degrees, cover X = N(v) ∩
    // alive, and subtract from each affected survivor w its number of neighbours in X.
    __device__ void write_child(uint32_t v, unsigned char* rec) {
        SpShared& s = *sh;
        ++epoch;
        if (threadIdx.x == 0) {
            s.nX = 0;
            s.nA = 0;
            s.eX = 0;
            s.sumX = 0;
        }
        __syncthreads();
        // X (in L1), tagged with the epoch
        const uint32_t b0 = a->off[v], b1 = a->off[v + 1];
        for (uint32_t base = b0; base < b1; base += SP_THREADS) {
            const uint32_t e = base + threadIdx.x;
            const uint32_t w = e < b1 ? a->nbr[e] : 0u;
            const bool al = e < b1 && deg[w] != DREM;
            if (al) tag[w] = epoch;
            append(al, w, L1, &s.nX);
        }
        // bulk copy of the parent's degrees
        uint4* d4 = reinterpret_cast<uint4*>(rec + 16);
        const uint4* s4 = reinterpret_cast<const uint4*>(deg);
        for (uint32_t i = threadIdx.x; i < a->npad / 8; i += SP_THREADS) d4[i] = s4[i];
        __syncthreads();
        const uint32_t nX = s.nX;
        uint16_t* rd = reinterpret_cast<uint16_t*>(rec + 16);
        uint32_t sx = 0;
        for (uint32_t i = threadIdx.x; i < nX; i += SP_THREADS) {
            const uint32_t u = L1[i];
            sx += deg[u];
            rd[u] = DREM;
        }
        sx = block_sum(sx, s);
        // count each survivor's neighbours in X
        const uint16_t* dg = deg;
        uint32_t* tg = tag;
        uint32_t* ct = cnt;
        uint32_t* LA = L2;
        uint32_t* nA = &s.nA;
        uint32_t* eX = &s.eX;
        const uint32_t ep = epoch;
        for_each_neighbor(L1, nX, [dg, tg, ct, LA, nA, eX, ep](uint32_t u, uint32_t w) {
            if (dg[w] == DREM) return;
            if (tg[w] == ep) {
                if (w > u) atomicAdd(eX, 1u);
                return;
            }
            if (atomicAdd(ct + w, 1u) == 0u) LA[atomicAdd(nA, 1u)] = w;
        });
        const uint32_t na = s.nA;
        for (uint32_t i = threadIdx.x; i < na; i += SP_THREADS) {
            const uint32_t w = L2[i];
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

    // search_node.cpp:16-25 for one vertex (the remove-v branch)
    __device__ void remove_one(uint32_t v) {
        if (threadIdx.x == 0) {
            (void)dclaim(deg, v);
            RL[0] = v;
        }
        __syncthreads();
        remove_claimed(1);
        // edges: recomputed by the next scan
    }
};

template <bool INSTR>
__global__ void __launch_bounds__(SP_THREADS, 1) sparse_kernel(SparseArgs a) {
    extern __shared__ uint4 smem4[];
    __shared__ SpShared sh;
    const uint32_t worker = blockIdx.x;
    if (worker >= a.workers) return;
    const int tid = threadIdx.x;

    CtaNode<INSTR> x;
    x.deg = reinterpret_cast<uint16_t*>(smem4);
    x.cbuf = reinterpret_cast<uint32_t*>(x.deg + a.npad);
    x.cstart = x.cbuf + SP_THREADS;
    x.sh = &sh;
    x.a = &a;
    uint32_t* scr = a.scratch + (unsigned long long)worker * 8ull * a.n;
    x.L1 = scr;
    x.L2 = scr + a.n;
    x.L3 = scr + 2ull * a.n;
    x.RL = scr + 3ull * a.n;
    x.T = scr + 4ull * a.n;
    x.cnt = scr + 5ull * a.n;
    x.P = scr + 6ull * a.n;
    x.owner = a.owner + (unsigned long long)worker * a.n;
    x.tag = a.tag + (unsigned long long)worker * a.n;
    x.epoch = 0;

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
    uint32_t best = a.pvc ? a.k : ctl->best;
    unsigned long long nodes_flushed = 0;

    while (true) {
        if (!have) {
            if (sp > 0) {
                --sp;
                x.load_record(slot_at(sp));
            } else {
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

        // control line, node counter, limits
        if (tid == 0) {
            const uint4 h = ld_volatile_v4(ctl);
            sh.red[0] = h.y;
            sh.red[1] = h.x;
            sh.red[2] = (uint32_t)ld_relaxed_u64(&ctl->work);
            int stop = 0;
            ++st.nodes;
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
        } else {
            ++st.nodes;
        }
        __syncthreads();
        const uint32_t cancel = sh.red[0], hbest = sh.red[1], qsize = sh.red[2], stop = sh.red[3];
        __syncthreads();
        if (cancel || stop) break;
        if (!a.pvc) best = min(best, hbest);

        // process_node
        x.reduce(best, st);
        const bool prune = sh.doom || should_prune(a.pvc, a.k, best, sh.cc, sh.edges);
        st.dooms += sh.doom;
        if (prune) {
            have = false;
            continue;
        }
        if (sh.edges == 0) {
            if (tid == 0) {
                uint32_t rec;
                if (a.pvc) rec = atomicCAS(&ctl->found, 0u, 1u) == 0u;
                else rec = sh.cc < atomicMin(&ctl->best, sh.cc);
                sh.red[4] = rec;
            }
            __syncthreads();
            if (sh.red[4]) {
                uint32_t* slot = a.cover_slots + (unsigned long long)worker * a.cover_words;
                for (uint32_t w = tid; w < a.cover_words; w += SP_THREADS) {
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
                    atomicMin(&ctl->best_owner, ((unsigned long long)sh.cc << 32) | worker);
                    if (a.pvc) atomicExch(&ctl->cancel, 1u);
                    if (a.mailbox) {
                        a.mailbox[2] = sh.cc;
                        if (a.pvc) a.mailbox[3] = 1;
                    }
                }
            }
            __syncthreads();
            if (a.pvc) break;
            best = min(best, sh.cc);
            have = false;
            continue;
        }
        // argmax from the last scan (smallest id among max degree)
        const uint32_t v = 0xFFFFFFFFu - (uint32_t)(sh.maxkey & 0xFFFFFFFFull);
        ++st.maxdeg;

        // branch
        unsigned char* child = nullptr;
        unsigned long long* publish = nullptr;
        unsigned long long pos = 0;
        if (!a.seq_mode && qsize < a.threshold) {
            if (tid == 0) {
                const unsigned long long old = atomicAdd(&ctl->work, ONE_PENDING | 1ull);
                int ok = (uint32_t)old < a.capacity;
                if (!ok) atomicAdd(&ctl->work, ~(ONE_PENDING | 1ull) + 1ull);
                else {
                    st.max_queue = max(st.max_queue, (unsigned long long)((uint32_t)old + 1));
                    sh.pos = atomicAdd(&ctl->tail, 1ull);
                    unsigned long long* p = a.seq + (sh.pos & a.ring_mask);
                    while (ld_acquire_u64(p) != sh.pos) __nanosleep(32);
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
        if (!child) {
            if (sp >= a.stack_bound) {  // cannot happen within the provisioned depth
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
        if (publish) {
            __threadfence();
            __syncthreads();
            if (tid == 0) st_release_u64(publish, pos + 1);
        }
        ++st.children;
        x.remove_one(v);
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
        o.active = clock64() - c_start;
        o.max_queue = st.max_queue;
#pragma unroll
        for (int p = 0; p < 10; ++p) o.phase[p] = 0;
        a.stats[worker] = o;
        (void)t_start;
    }
}

}  // namespace vcg
