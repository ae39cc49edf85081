/* include/vcgpu.h — the C-ABI of the B200-native vertex-cover search engine (libvcgpu.so).
 *
 * Plain pointers and sizes only. Every entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj). All functions return an int status code
 * (VCG_OK = 0); on failure vcg_last_error() holds a thread-local message whose text follows the
 * reference's exception text where one exists (e.g. ParseError "line N: ...", graph.hpp:17-26).
 *
 * Limits (both fail loudly with VCG_EINVAL / VCG_ECUDA, never silently):
 *   - dense engine (n <= 1024): per-worker node stacks of stack_bound records (greedy size, or
 *     min(k, n)) of 16 + 64 W + 128 bytes, W = 4/8/16/32 words per row — C5 (n = 500, 3552
 *     warps): 3552 x 484 x 1168 B = 2.0 GB;
 *   - sparse engine (any n): u16 degrees, so every vertex degree must be < 65535; CSR offsets
 *     are u32 on the device, so 2m < 2^32; the node's degree array sits in shared memory up to
 *     about 110k vertices, in global memory beyond (the GDEG variant, engine 7); per-worker
 *     scratch of 64 n bytes and node records of 16 + 2n bytes; a local stack deeper than its
 *     device-memory cap hands its oldest node to the worklist, and only a full worklist then
 *     ends the solve with an error.
 *
 * Ownership: the caller owns every buffer it passes in (never retained beyond the call, except
 * that vcg_graph_* copy their inputs). The library owns vcg_graph objects (free with
 * vcg_graph_destroy) and the arrays inside a vcg_result (free with vcg_result_free). Device
 * copies of a graph are created lazily by the first solve on a device and live until
 * vcg_graph_destroy.
 */
#ifndef VCGPU_H
#define VCGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VCG_API __attribute__((visibility("default")))

/* status codes */
enum {
    VCG_OK = 0,
    VCG_EINVAL = 1,   /* std::invalid_argument in the reference (scheduler.cpp:20-29,330) */
    VCG_EPARSE = 2,   /* vcsolve::ParseError (graph.hpp:17-26) */
    VCG_ECUDA = 3,    /* CUDA/device error: no reference counterpart (CPU-only reference) */
    VCG_ENOMEM = 4,
    VCG_ERANGE = 5,   /* brute_force_mvc limit (solver_seq.cpp:174-175) */
    VCG_EVERIFY = 6   /* a cover the engine returned failed verify_cover (bounds.cpp:32-45):
                         an engine fault, never expected; the result is freed */
};

typedef struct vcg_graph vcg_graph; /* opaque: BaseGraph (graph.hpp:34-53) + device copies */

/* ------------------------------------------------------------------ graph (host side) */

/* BaseGraph from an already-built CSR (offsets u64[n+1], neighbors u32[2m], sorted,
 * duplicate-free, symmetric). Validated; replaces constructing BaseGraph directly. */
VCG_API int vcg_graph_from_csr(uint32_t n, uint64_t m, const uint64_t* offsets,
                               const uint32_t* neighbors, uint32_t id_base, vcg_graph** out);
/* make_graph (graph.hpp:57-59, graph.cpp:22-54): pairs = 2*num_pairs ids in [0, n). */
VCG_API int vcg_make_graph(uint32_t n, uint64_t num_pairs, const uint32_t* pairs,
                           uint32_t id_base, vcg_graph** out);
/* parse_edge_list (graph.hpp:64, graph.cpp:81-114) and parse_dimacs (graph.hpp:68,
 * graph.cpp:116-159) over an in-memory text of `len` bytes. VCG_EPARSE on malformed input. */
VCG_API int vcg_parse_edge_list(const char* text, size_t len, vcg_graph** out);
VCG_API int vcg_parse_dimacs(const char* text, size_t len, vcg_graph** out);
/* complement (graph.hpp:71, graph.cpp:161-185) */
VCG_API int vcg_complement(const vcg_graph* g, vcg_graph** out);
/* write_edge_list (graph.hpp:74, graph.cpp:187-193): *text is library-owned until
 * vcg_free_buffer. */
VCG_API int vcg_write_edge_list(const vcg_graph* g, char** text, size_t* len);
VCG_API void vcg_free_buffer(void* p);
VCG_API void vcg_graph_destroy(vcg_graph* g);

VCG_API uint32_t vcg_graph_num_vertices(const vcg_graph* g);
VCG_API uint64_t vcg_graph_num_edges(const vcg_graph* g);
VCG_API uint32_t vcg_graph_id_base(const vcg_graph* g);
/* Borrowed views of the CSR (valid until vcg_graph_destroy). */
VCG_API const uint64_t* vcg_graph_offsets(const vcg_graph* g);
VCG_API const uint32_t* vcg_graph_neighbors(const vcg_graph* g);
/* BaseGraph::has_edge (graph.cpp:14-20); BaseGraph::operator== (graph.hpp:52) */
VCG_API int vcg_has_edge(const vcg_graph* g, uint32_t u, uint32_t v);
VCG_API int vcg_graph_equal(const vcg_graph* a, const vcg_graph* b);
/* check_graph_invariants (graph.cpp:195-211) */
VCG_API int vcg_check_invariants(const vcg_graph* g);

/* greedy_approx (bounds.hpp:28-32, bounds.cpp:7-19): same cover as the reference.
 * cover needs n slots, receives internal ids ascending. */
VCG_API int vcg_greedy(const vcg_graph* g, uint32_t* size, uint32_t* cover);
/* brute_force_mvc (solver_seq.hpp:50-52, solver_seq.cpp:173-211): VCG_ERANGE when n > 20.
 * cover receives ORIGINAL ids (internal + id_base), like the reference. */
VCG_API int vcg_brute_force(const vcg_graph* g, uint32_t* size, uint32_t* cover);
/* verify_cover (bounds.hpp:44, bounds.cpp:32-45) over internal ids. */
VCG_API int vcg_verify_cover(const vcg_graph* g, const uint32_t* cover, uint32_t len, int* ok);

/* ------------------------------------------------------------------------------ solve */

enum { VCG_MVC = 0, VCG_PVC = 1 };                         /* SolveMode (bounds.hpp:13-22) */
enum { VCG_HYBRID = 0, VCG_SEQ = 1, VCG_STACKONLY = 2 };   /* bindings.cpp:75-93 strategies */
enum { VCG_COMPLETE = 0, VCG_TIMEOUT = 1, VCG_BUDGET = 2 }; /* RunStatus (solver_seq.hpp:22) */
enum { VCG_RULES_REFERENCE = 0, VCG_RULES_PARALLEL = 1 };

/* SchedulerConfig (scheduler.hpp:17-25) + SolveLimits (solver_seq.hpp:28-31) + GPU knobs.
 * Initialise with vcg_params_init (reference defaults: capacity 4096, fraction 0.5, depth 8,
 * backoff 50 us, bindings.cpp:174-202). */
typedef struct {
    int32_t mode;               /* VCG_MVC | VCG_PVC */
    uint32_t k;                 /* PVC parameter, >= 1 */
    int32_t strategy;           /* VCG_HYBRID | VCG_SEQ | VCG_STACKONLY */
    uint32_t workers;           /* the reference's num_workers. VCG_HYBRID: the device is
                                   always filled (see device_workers) and the per-worker report
                                   is folded into this many entries (device worker i counts for
                                   entry i % workers; 0 = one entry per device worker).
                                   VCG_STACKONLY: device workers (one warp or one block each). */
    uint64_t capacity;          /* worklist capacity (entries) */
    double threshold_fraction;  /* (0, 1] → threshold = clamp(llround(f*cap), 1, cap) */
    uint32_t depth;             /* StackOnly sub-tree depth in [1, 30] */
    uint64_t backoff_us;        /* idle back-off (maps to __nanosleep) */
    double timeout_s;           /* < 0: none */
    uint64_t node_budget;       /* 0: none */
    int32_t device;             /* CUDA device ordinal */
    int32_t rules;              /* VCG_RULES_REFERENCE (bit-exact reference node order) or
                                   VCG_RULES_PARALLEL (block-parallel rule rounds) */
    uint32_t block_warps;       /* warps per CTA, 0 = auto */
    int32_t engine;             /* 0 auto, 1 dense (n <= 1024, warp per node),
                                   2 sparse (any n, CTA per node),
                                   3 dense without renumbering (every node in the wide 32*W-slot
                                     layout; for A/B tests),
                                   4 dense without the mid (per-warp frame) layout (wide and
                                     compact only; for A/B tests),
                                   5 / 6 dense with the mid layout forced to <= 256 / <= 128
                                     alive vertices (n in 257..512; auto picks 256 for sparse
                                     graphs, average degree < 24),
                                   7 sparse with the node's degree array in global memory (the
                                     variant auto picks when n is beyond the shared-memory limit,
                                     about 110k vertices) */
    int32_t instrument;         /* 1: per-worker phase cycle counters */
    int32_t donate_oldest;      /* 1 (vcg_params_init's default): when donating, hand over the
                                   OLDEST stacked node (largest expected sub-tree) and stack the
                                   new child; 0: donate the new remove-N(v) child as the reference
                                   does (scheduler.cpp:191-199) */
    uint32_t initial_best;      /* MVC: external upper bound (e.g. from another rank),
                                   0 = none; never replaces the greedy certificate */
    /* Seeding (multi-GPU frontier shares): when num_seeds > 0, the worklist starts with these
       nodes instead of the root. seeds = num_seeds records of
       [cover_count u32, edge_count u32, degrees u32[n]] (kRemoved = 0xFFFFFFFF). */
    uint64_t num_seeds;
    const uint32_t* seeds;
    /* Mailbox (pinned host memory, written by the host, polled by the device ~every 50 us):
       mailbox[0] = external best bound (MVC, 0 = none), mailbox[1] = cancel request.
       Null = none. */
    volatile uint32_t* mailbox;
    /* CUDA stream (cudaStream_t) to launch on; null = the library's own stream. The call stays
       blocking: it synchronizes this stream before returning. */
    void* stream;
    /* Debug options (0 in production):
       VCG_DEBUG_CERTIFY — after a parallel MVC search of size s, prove PVC(s - 1) infeasible
         (repeating on "yes"); reported as certify_nodes / certify_ms, within the caller's
         remaining timeout / node budget. A cross-check: the search is exact without it.
       VCG_DEBUG_CORRUPT_COVER — drop one vertex from the returned cover before verification
         (tests the engine's own verify_cover check, which then fails with VCG_EVERIFY).
       VCG_DEBUG_SMALL_STACK — cap the sparse engine's local stacks at 3 nodes (tests the
         hand-over of the oldest node to the worklist when a stack is full). */
    uint32_t debug_flags;
    /* Device workers (warps of the dense engine, CTAs of the sparse engine) to run. 0 = every
       SM filled (VCG_HYBRID) / `workers` (VCG_STACKONLY). Set it to run a fixed number, e.g.
       to give several shards on one device their share. */
    uint32_t device_workers;
} vcg_params;
enum { VCG_DEBUG_CERTIFY = 1, VCG_DEBUG_CORRUPT_COVER = 2, VCG_DEBUG_SMALL_STACK = 4 };

typedef struct {
    int32_t status;             /* VCG_COMPLETE | VCG_TIMEOUT | VCG_BUDGET */
    uint32_t size;              /* Solution.size (0 for infeasible PVC) */
    int32_t feasible;
    uint32_t greedy_size;       /* ParallelRun.greedy_size */
    uint32_t cover_len;
    uint32_t* cover;            /* ORIGINAL ids (internal + id_base), ascending */
    int32_t cover_from_search;  /* 0: the greedy certificate was the answer */
    uint32_t num_workers;
    uint64_t* worker_nodes;     /* WorkerMetrics.nodes_visited, per worker */
    uint64_t* worker_stack_high_water;
    uint64_t nodes_total;
    uint64_t wl_added, wl_removed, wl_max_size, wl_current_size; /* GlobalWorklist::Stats */
    double wall_ms;             /* ParallelRun.wall_ms: greedy + setup + search + readback */
    double device_ms;           /* search kernel(s), CUDA events */
    double greedy_ms;
    double h2d_ms;
    uint64_t h2d_bytes, d2h_bytes;
    /* roofline counters: rule rounds, max-degree passes, children built */
    uint64_t rounds, maxdeg_passes, children, removals;
    uint64_t donated;           /* nodes handed to the worklist by workers */
    uint64_t removals_deg1, removals_deg2, removals_high; /* rule removals, per rule */
    uint64_t doomed;            /* nodes cut short by the exact high-degree doom test */
    uint32_t degree_bytes;      /* w: bytes per degree entry in the engine's node layout */
    uint32_t n_padded;          /* n rounded to the engine's lane layout */
    int32_t engine;             /* engine that ran: 1 dense, 2 sparse */
    uint32_t grid_blocks, block_threads;
    uint32_t kernel_launches;   /* device kernels this solve launched */
    uint64_t phase_cycles[10];  /* Phase order of metrics.hpp:15-26, summed over workers */
    uint64_t active_cycles;     /* summed over workers */
    uint64_t donated_peer;      /* of `donated`: nodes written into another shard's worklist */
    /* VCG_DEBUG_CERTIFY only: the certificate's PVC searches (not in nodes_total / device_ms) */
    uint64_t certify_nodes;
    double certify_ms;
    uint32_t certify_launches;
    /* search timeline (dense engine): ms after the first worker started by which 10 / 50 / 90 /
       100% of the workers had taken their first node (the ramp-up), and had exited (the tail);
       -1 = that share never got work */
    double t_first_ms[4];
    double t_end_ms[4];
    double idle_share;          /* share of the workers' time spent waiting for worklist nodes */
    double t_lastwait_ms[4];    /* ... by which 10/50/90/100% had entered their final wait: the
                                   search's tail runs from there to t_end_ms */
} vcg_result;

VCG_API void vcg_params_init(vcg_params* p);
/* run_hybrid / run_stackonly (scheduler.hpp:48,55) and solve_mvc_seq / solve_pvc_seq
 * (solver_seq.hpp:43-48) on the GPU: greedy seed (host), CSR upload, one persistent kernel,
 * result readback, verify_cover of the returned cover (VCG_EVERIFY if it fails). Blocking. */
VCG_API int vcg_solve(const vcg_graph* g, const vcg_params* p, vcg_result* out);
VCG_API void vcg_result_free(vcg_result* r);

/* Multi-GPU partitioning: expands the search tree level by level on the device
 * — every node processed exactly as the search would, with a fixed bound per level — until at
 * least `target` open nodes exist. Deterministic: every rank computes the same frontier and
 * takes its share (records i with i % world == rank) as vcg_params.seeds. The nodes the
 * expansion visits are counted in nodes_visited (count them once, on one rank). */
typedef struct {
    uint64_t num_seeds;
    uint32_t* seeds;            /* num_seeds x [cover_count, edge_count, degrees u32[n]] */
    uint64_t nodes_visited;
    uint32_t levels;
    uint32_t best;              /* MVC: greedy size or better after expansion; PVC: k */
    uint32_t greedy_size;
    int32_t found;              /* a cover was found during the expansion */
    uint32_t cover_len;
    uint32_t* cover;            /* best certificate so far, ORIGINAL ids (greedy if none) */
    uint32_t kernel_launches;
} vcg_frontier;
VCG_API int vcg_expand_frontier(const vcg_graph* g, const vcg_params* p, uint64_t target,
                                vcg_frontier* out);
VCG_API void vcg_frontier_free(vcg_frontier* f);

/* Multi-shard solves with device-to-device work donation (SURVEY.md §8e "exchange step").
 * A shard is one dense-engine search (n <= 1024, strategy hybrid) on one GPU with its own device
 * worklist. Linked shards (one per GPU, or several on one device):
 *   - hand queued nodes straight into the ring of a shard whose worklist is below its
 *     threshold (an exchange-helper warp per shard: remote stores + a system-scope release
 *     over NVLink P2P / CUDA IPC);
 *   - propagate an improved MVC bound with peer atomicMin and a PVC "found" / timeout / budget
 *     as a cancel store into every shard;
 *   - terminate together: shard 0 counts the shards whose `pending` (queued + active) is
 *     non-zero, maintained by whoever moves a shard's pending between 0 and 1.
 * Replaces the reference's single shared GlobalWorklist (worklist.cpp:11-48) across GPUs.
 *
 * open    : validate + greedy + buffers + seeds on p->device (p->seeds = this shard's share;
 *           with no seeds the shard starts with the root if with_root, else empty).
 * export  : CUDA IPC handles of the shard's exchange memory (vcg_session_handle_bytes()).
 * link_ipc: map every other shard's handles (handles = world x handle bytes, in rank order;
 *           seeds_per_shard = each shard's seed count, root counted as 1).
 * link_local: link shards opened in this process (same device or P2P-capable devices).
 * launch  : asynchronous; launch EVERY shard before waiting on any (they finish together).
 * wait    : blocks; fills the result like vcg_solve, for this shard's part of the search.
 * On one device, shards must leave room for each other (params.device_workers), or the later ones
 * cannot become resident. */
#define VCG_MAX_SHARDS 16
typedef struct vcg_session vcg_session;
VCG_API int vcg_session_open(const vcg_graph* g, const vcg_params* p, int with_root,
                             vcg_session** out);
VCG_API size_t vcg_session_handle_bytes(void);
VCG_API int vcg_session_export(const vcg_session* s, void* handle);
VCG_API int vcg_session_link_ipc(vcg_session* s, uint32_t world, uint32_t rank,
                                 const void* handles, const uint64_t* seeds_per_shard);
VCG_API int vcg_session_link_local(vcg_session* const* shards, uint32_t world);
VCG_API int vcg_session_launch(vcg_session* s);
/* Fresh search state for the next solve of the same session (same graph and parameters):
 * buffers, IPC mappings and links are kept. Every linked shard must reset (and the caller must
 * synchronise: all reset before any launches) between two solves. */
VCG_API int vcg_session_reset(vcg_session* s);
VCG_API int vcg_session_wait(vcg_session* s, vcg_result* out);
VCG_API void vcg_session_close(vcg_session* s);
/* Workers (warps) of a full-device dense-engine solve of g on `device` (shards sharing a device
   * split them through params.device_workers). Warp 0 of every linked shard is its exchange
 * helper (it moves queued nodes to starving peers; the other warps search). */
VCG_API int vcg_device_workers(const vcg_graph* g, int32_t device, uint32_t* workers);

/* Pinned, device-mapped host words for vcg_params.mailbox (zeroed); n_words >= 4. */
VCG_API int vcg_mailbox_alloc(uint32_t n_words, uint32_t** out);
VCG_API void vcg_mailbox_free(uint32_t* p);

/* Number of CUDA devices visible (0 when no driver / no GPU). */
VCG_API int vcg_device_count(void);
/* Thread-local text of the last error. */
VCG_API const char* vcg_last_error(void);
/* Library version string. */
VCG_API const char* vcg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* VCGPU_H */
