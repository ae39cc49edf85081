/* tools/tree_stats.c — offline analysis (not product, not test): walks the C5 PVC tree in the
 * dense engine's order on the CPU (bitmap node, reference rule order, doom tests, doomed
 * children counted at birth) and prints where the per-node work goes, to evaluate kernel ideas
 * without GPU time.  Usage: tree_stats graph.clq k [complement] [node cap]
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAXN 1024
#define MAXW (MAXN / 32)
static uint32_t n, W, A[MAXN][MAXW];

typedef struct {
    uint32_t d[MAXN];
    uint32_t alive[MAXW];
    uint32_t cc, edges;
} node_t;

static uint64_t st_nodes, st_rounds, st_branch, st_dead, st_stored, st_doom_start, st_pass_scans[4],
    st_pass_skipped[4], st_rm[4], st_words_dead, st_words_live, st_cand_words_dead, st_xsize,
    st_alive_at_branch, st_lim_child, st_dead_hist[17], st_first_round_doom, st_rounds_hist[8],
    st_nonempty_xwords, st_surv_words, st_alive_visit[17], st_alive_branch_h[17];
static uint32_t alive_count(const void* xv);

static int is_alive(const node_t* x, uint32_t v) { return (x->alive[v >> 5] >> (v & 31)) & 1; }
static void remove_v(node_t* x, uint32_t u) {
    uint32_t du = 0;
    for (uint32_t j = 0; j < W; ++j) du += __builtin_popcount(A[u][j] & x->alive[j]);
    for (uint32_t j = 0; j < W; ++j) {
        uint32_t m = A[u][j];
        while (m) {
            int b = __builtin_ctz(m);
            m &= m - 1;
            x->d[32 * j + b] -= 1;
        }
    }
    x->alive[u >> 5] &= ~(1u << (u & 31));
    x->cc++;
    x->edges -= du;
}
static uint32_t lim_of(uint32_t k, uint32_t cc) { return cc >= k ? 0 : k - cc; }
static int first_cand(const node_t* x, int pos, int pass, uint32_t c) {
    for (uint32_t v = pos; v < n; ++v) {
        if (!is_alive(x, v)) continue;
        if (pass == 3 ? x->d[v] > c : x->d[v] == c) return v;
    }
    return -1;
}
static void first2(const node_t* x, uint32_t v, int* p0, int* p1) {
    *p0 = *p1 = -1;
    for (uint32_t u = 0; u < n; ++u)
        if (((A[v][u >> 5] >> (u & 31)) & 1) && is_alive(x, u)) {
            if (*p0 < 0) *p0 = u;
            else { *p1 = u; return; }
        }
}
/* returns 1 if doomed/pruned */
static int reduce(node_t* x, uint32_t k) {
    int doom = 0;
    int rounds = 0;
    while (x->edges) {
        st_rounds++;
        rounds++;
        uint32_t lim0 = lim_of(k, x->cc), above = 0;
        int any = 0;
        for (uint32_t v = 0; v < n; ++v)
            if (is_alive(x, v)) {
                above += x->d[v] > lim0;
                any |= x->d[v] == 1 || x->d[v] == 2 || x->d[v] > lim0;
            }
        if (above > lim0) {
            st_doom_start++;
            if (rounds == 1) st_first_round_doom++;
            return 1;
        }
        if (!any) break;
        int changed = 0;
        for (int pass = 1; pass <= 3; ++pass) {
            uint32_t c = pass;
            if (pass == 3) {
                uint32_t lim = lim_of(k, x->cc), cnt = 0;
                for (uint32_t v = 0; v < n; ++v) cnt += is_alive(x, v) && x->d[v] > lim;
                if (cnt > lim) doom = 1;
                c = lim;
            }
            int pos = 0;
            while (!doom && x->cc <= k) {
                st_pass_scans[pass]++;
                int v = first_cand(x, pos, pass, c);
                if (v < 0) break;
                pos = v + 1;
                int u0 = v, u1 = -1;
                if (pass < 3) {
                    int p0, p1;
                    first2(x, v, &p0, &p1);
                    u0 = p0;
                    if (pass == 2) {
                        int tri = (A[p0][p1 >> 5] >> (p1 & 31)) & 1;
                        u0 = tri ? p0 : -1;
                        u1 = tri ? p1 : -1;
                    }
                }
                if (u0 >= 0) { remove_v(x, u0); st_rm[pass]++; changed = 1; }
                if (u1 >= 0) { remove_v(x, u1); st_rm[pass]++; }
                if (pass == 3) c = lim_of(k, x->cc);
            }
            if (doom || x->cc > k) return 1;
        }
        if (!changed) break;
    }
    st_rounds_hist[rounds < 7 ? rounds : 7]++;
    if (x->cc > k) return 1;
    uint64_t s = k - x->cc;
    return (uint64_t)x->edges > s * s;
}

static node_t stack_[4096];
static uint32_t depth_[4096];
static uint32_t pw_[4096], pc_[4096], pb_[4096][3];  /* wide / compact visits on the root path;
                                                      wide by alive band 65-128, 129-256, >256 */
static uint64_t best_w, best_c, best_cost, best_b[3];
static uint64_t wide_depth_h[1024];
static uint32_t alive_count(const void* xv) {
    const node_t* x = xv;
    uint32_t a = 0;
    for (uint32_t j = 0; j < W; ++j) a += __builtin_popcount(x->alive[j]);
    return a;
}

int main(int argc, char** argv) {
    FILE* f = fopen(argv[1], "r");
    uint32_t k = atoi(argv[2]);
    char line[256];
    uint64_t m = 0;
    while (fgets(line, sizeof line, f)) {
        if (line[0] == 'p') sscanf(line, "p %*s %u %lu", &n, &m);
        else if (line[0] == 'e') {
            uint32_t u, v;
            sscanf(line, "e %u %u", &u, &v);
            --u, --v;
            if (u == v) continue;
            A[u][v >> 5] |= 1u << (v & 31);
            A[v][u >> 5] |= 1u << (u & 31);
        }
    }
    if (argc > 3 && atoi(argv[3])) /* complement */
        for (uint32_t u = 0; u < n; ++u)
            for (uint32_t v = 0; v < n; ++v)
                if (u != v) A[u][v >> 5] ^= 1u << (v & 31);
    W = (n + 31) / 32;
    W = W <= 4 ? 4 : W <= 8 ? 8 : W <= 16 ? 16 : 32;
    node_t* root = &stack_[0];
    memset(root, 0, sizeof *root);
    uint64_t e2 = 0;
    for (uint32_t v = 0; v < n; ++v) {
        root->alive[v >> 5] |= 1u << (v & 31);
        for (uint32_t j = 0; j < W; ++j) root->d[v] += __builtin_popcount(A[v][j]);
        e2 += root->d[v];
    }
    root->edges = e2 / 2;
    int sp = 1;
    node_t x;
    depth_[0] = 0;
    while (sp > 0) {
        uint32_t dep = depth_[--sp];
        uint32_t pw = pw_[sp], pc = pc_[sp], pb[3] = {pb_[sp][0], pb_[sp][1], pb_[sp][2]};
        x = stack_[sp];
        for (;;) {
            st_nodes++;
            if (argc > 4 && st_nodes >= (uint64_t)atoll(argv[4])) goto done;
            {
                uint32_t a = alive_count(&x);
                st_alive_visit[a >= 512 ? 16 : a / 32]++;
                if (a > 64) wide_depth_h[dep < 1023 ? dep : 1023]++;
                if (a > 64) pw++; else pc++;
                if (a > 64) pb[a > 256 ? 2 : a > 128 ? 1 : 0]++;
                uint64_t cost = 8ull * pw + pc;
                if (cost > best_cost) { best_cost = cost; best_w = pw; best_c = pc; memcpy(best_b, (uint64_t[3]){pb[0], pb[1], pb[2]}, sizeof best_b); }
            }
            if (reduce(&x, k)) break;
            if (x.edges == 0) { printf("cover found (yes-instance)\n"); return 0; }
            /* argmax: smallest id of max degree */
            uint32_t v = 0, best = 0;
            int have = 0;
            for (uint32_t u = 0; u < n; ++u)
                if (is_alive(&x, u) && (!have || x.d[u] > best)) { best = x.d[u]; v = u; have = 1; }
            st_branch++;
            /* child: X = N(v) ∩ alive */
            uint32_t X[MAXW], xcnt = 0, nz = 0;
            for (uint32_t j = 0; j < W; ++j) {
                X[j] = A[v][j] & x.alive[j];
                xcnt += __builtin_popcount(X[j]);
                nz += X[j] != 0;
            }
            st_nonempty_xwords += nz;
            st_xsize += xcnt;
            uint32_t na = 0;
            for (uint32_t j = 0; j < W; ++j) na += __builtin_popcount(x.alive[j]);
            st_alive_at_branch += na;
            st_alive_branch_h[na >= 512 ? 16 : na / 32]++;
            uint32_t c2 = x.cc + xcnt;
            int dead = c2 > k;
            uint32_t words = 0, candw = 0;
            node_t ch;
            if (!dead) {
                uint32_t lim = lim_of(k, c2), above = 0;
                st_lim_child += lim;
                ch = x;
                for (uint32_t i = 0; i < W && !dead; ++i) {
                    int surv = 0, cand = 0;
                    for (uint32_t l = 0; l < 32; ++l) {
                        uint32_t w = 32 * i + l;
                        if (w >= n || !is_alive(&x, w) || ((X[i] >> l) & 1)) continue;
                        surv = 1;
                        uint32_t s = 0;
                        for (uint32_t j = 0; j < W; ++j) s += __builtin_popcount(A[w][j] & X[j]);
                        ch.d[w] = x.d[w] - s;
                        if (x.d[w] > lim) cand = 1;
                        above += ch.d[w] > lim;
                    }
                    st_surv_words += surv;
                    words++;
                    candw += cand;
                    if (above > lim) dead = 1;
                }
                if (dead) { st_words_dead += words; st_cand_words_dead += candw; st_dead_hist[words]++; }
                else st_words_live += words;
            }
            if (dead) {
                st_dead++;
                st_nodes++;
            } else {
                for (uint32_t j = 0; j < W; ++j) ch.alive[j] = x.alive[j] & ~X[j];
                ch.cc = c2;
                uint64_t e = 0;
                for (uint32_t w = 0; w < n; ++w) if (is_alive(&ch, w)) e += ch.d[w];
                ch.edges = e / 2;
                depth_[sp] = dep + 1;
                pw_[sp] = pw;
                pc_[sp] = pc;
                memcpy(pb_[sp], pb, sizeof pb);
                stack_[sp++] = ch;
                st_stored++;
            }
            remove_v(&x, v);
            dep++;
        }
    }
done:
    printf("nodes %lu rounds %lu branch %lu dead %lu stored %lu doom_at_round_start %lu (first round %lu)\n",
           st_nodes, st_rounds, st_branch, st_dead, st_stored, st_doom_start, st_first_round_doom);
    printf("scans p1 %lu p2 %lu p3 %lu; removals p1 %lu p2 %lu p3 %lu\n", st_pass_scans[1],
           st_pass_scans[2], st_pass_scans[3], st_rm[1], st_rm[2], st_rm[3]);
    printf("rounds hist (completed reductions):");
    for (int i = 0; i < 8; ++i) printf(" %d:%lu", i, st_rounds_hist[i]);
    printf("\navg |X| %.1f, alive at branch %.1f, child lim %.1f, nonempty X words %.2f\n",
           (double)st_xsize / st_branch, (double)st_alive_at_branch / st_branch,
           (double)st_lim_child / st_branch, (double)st_nonempty_xwords / st_branch);
    printf("words per dead child %.2f (cand words %.2f), per live child %.2f, surv words/child %.2f\n",
           (double)st_words_dead / st_dead, (double)st_cand_words_dead / st_dead,
           (double)st_words_live / (st_branch - st_dead), (double)st_surv_words / st_branch);
    printf("alive at visit (x32):");
    for (int i = 0; i <= 16; ++i) printf(" %d:%lu", i, st_alive_visit[i]);
    printf("\nalive at branch (x32):");
    for (int i = 0; i <= 16; ++i) printf(" %d:%lu", i, st_alive_branch_h[i]);
    printf("\ncritical path (8 x wide + compact): %lu wide + %lu compact visits (wide by alive: 65-128 %lu, 129-256 %lu, >256 %lu)", best_w, best_c, best_b[0], best_b[1], best_b[2]);
    printf("\nwide visits by depth:");
    for (int i = 0; i < 1024; ++i) if (wide_depth_h[i]) printf(" %d:%lu", i, wide_depth_h[i]);
    printf("\ndead words hist:");
    for (int i = 0; i <= 16; ++i) printf(" %d:%lu", i, st_dead_hist[i]);
    printf("\n");
    return 0;
}
