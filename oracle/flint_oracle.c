/*
 * flint_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker).
 *
 * A sequential, single-threaded CPU restatement of the reference's hot path,
 * used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs.  Nothing in paper_2604_17550_b200/ links or calls it.
 *
 * Parity pinning: checked against the reference Python implementation
 * (trainsim, imported read-only in the build container) on the golden corpus
 * under tests/golden/ (hand schedules, randomized world/rank graphs, the
 * cross-rank race witness, synthesized DP/FSDP/TP families, C3 points at
 * R=1024), see tests/test_oracle_golden.py.
 *
 * What it restates (reference file:line, relative to pkg/src/trainsim/):
 *   or_analytical_time      collectives.py:243-293 (+ round_half_up traceio.py:68-70)
 *   or_duration_from_flops  traceio.py:184
 *   or_simulate             simulator.py:203-367 (dispatch :247-268, loop :279-340,
 *                           stats :342-356, _merge/_total/_overlap :121-149,
 *                           _peak_mem :370-393, _coll_duration :109-114,
 *                           _pair_messages :177-200, transfer_ns/route
 *                           topology.py:68-102, collective_instances
 *                           collectives.py:419-453)
 *   or_critical_path        simulator.py:400-460
 *
 * One algorithmic liberty, result-preserving: the reference re-runs the
 * host/compute start phase for *every* rank after every pop
 * (simulator.py:282-297).  That phase is a no-op for a rank unless it has a
 * ready node and a free stream at `now`, and running it is idempotent, so we
 * only visit ranks whose earliest possible start ("wake" time) is <= now.
 * critical_path computes each collective's union-of-deps maximum once per
 * instance instead of materializing the union per member (simulator.py:419-428);
 * the longest-path value is identical.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

enum { K_HOST = 0, K_COMP = 1, K_COLL = 2, K_SEND = 3, K_RECV = 4 };
enum { C_AR = 0, C_AG = 1, C_RS = 2 };
enum { A_RING = 0, A_TREE = 1, A_MESH = 2 };
enum { OR_OK = 0, OR_INVALID = 1, OR_DEADLOCK = 3, OR_UNSUPPORTED = 4, OR_INCONSISTENT = 5 };

typedef struct {
    int64_t n_ranks;
    const int64_t *rank_value;   /* [n_ranks], graphs list order              */
    const int64_t *node_off;     /* [n_ranks+1] flat node index of each rank  */
    const int64_t *rank_base;    /* [n_ranks] first structure node of a rank  */
    /* Per-node arrays below are indexed by STRUCTURE node (SV(G, flat)): ranks
     * that share one node list (synth.py:331-335) share one copy, so a graph
     * set costs O(structures), not O(R x N) -- and a full-world group list is
     * stored once per structure node instead of R times (R x C x R at 8192). */
    const int64_t *node_id;
    const int32_t *node_kind;
    const int64_t *node_dur;     /* duration_ns, -1 for None                  */
    const int64_t *dep_off;      /* dep_ids() = data_deps + ctrl ids, raw     */
    const int64_t *dep_ids;
    const int64_t *in_off, *in_tid;
    const int64_t *out_off, *out_tid;
    const int32_t *coll_kind;    /* -1 when not a collective                  */
    const int64_t *coll_bytes;
    const int64_t *grp_off, *grp_rank;
    const int64_t *p2p_peer, *p2p_bytes, *p2p_tag;
    const int64_t *tens_lo, *tens_hi;  /* [n_ranks] per-rank tensor table range */
    const int64_t *tens_id, *tens_bytes;
    const int64_t *sv;           /* internal: flat node -> structure node (set by the entry points) */
} or_graphs;

#define SV(G, v) ((G)->sv[v])

/* flat -> structure node map; the entry points run on a copy of G carrying it */
static int64_t *build_sv(const or_graphs *G) {
    int64_t nr = G->n_ranks, total = G->node_off[nr];
    int64_t *sv = malloc((size_t)(total + 1) * sizeof(int64_t));
    for (int64_t r = 0; r < nr; r++)
        for (int64_t v = G->node_off[r]; v < G->node_off[r + 1]; v++) sv[v] = G->rank_base[r] + (v - G->node_off[r]);
    return sv;
}

typedef struct {
    int32_t topo_kind;           /* 0 switch, 1 mesh2d */
    int32_t algo;                /* 0 ring, 1 tree, 2 mesh-hier */
    int64_t world_size;
    double bw;
    int64_t latency;
    int64_t rows, cols;
    int32_t compute_streams, comm_streams;
} or_config;

typedef struct {
    int64_t makespan;
    int64_t *rank_stats;         /* [n_ranks*5]: finish, comp, comm, exposed, peak */
    int64_t *ev_start, *ev_end;  /* optional [total_nodes] */
    int64_t *link_busy;          /* optional [n_links]; -1 = link never used */
    int64_t n_links;
} or_sim_out;

static void set_err(char *err, int len, const char *msg) {
    if (err && len > 0) { strncpy(err, msg, (size_t)len - 1); err[len - 1] = 0; }
}

/* ---------------------------------------------------------------- costs */

static int64_t rhu(double x) { return (int64_t)floor(x + 0.5); }   /* traceio.py:68-70 */

static double ring_rs(int64_t n, double s, double a, double b) {   /* collectives.py:243-244 */
    double t1 = (double)(n - 1) * a;
    double t2 = (double)(n - 1) / (double)n;
    t2 = t2 * s;
    t2 = t2 * b;
    return t1 + t2;
}

static double ring_ar(int64_t n, double s, double a, double b) {   /* collectives.py:247-248 */
    double t1 = (double)(2 * (n - 1)) * a;
    double t2 = (double)(2 * (n - 1)) / (double)n;
    t2 = t2 * s;
    t2 = t2 * b;
    return t1 + t2;
}

static int64_t ceil_log2(int64_t n) {  /* math.ceil(math.log2(n)), exact for n < 2^48 */
    int64_t k = 0;
    while (((int64_t)1 << k) < n) k++;
    return k;
}

int64_t or_analytical_time(int kind, int64_t size_bytes, int64_t n, int algo, double alpha,
                           double beta, int64_t rows, int64_t cols, int *status) {
    *status = OR_OK;
    if (n <= 1) return 0;
    double a = alpha, b = beta, s = (double)size_bytes, t;
    if (algo == A_RING) {
        t = kind == C_AR ? ring_ar(n, s, a, b) : ring_rs(n, s, a, b);
    } else if (algo == A_TREE) {
        if (kind != C_AR) { *status = OR_UNSUPPORTED; return 0; }
        double t1 = (double)(2 * ceil_log2(n)) * a;
        double t2 = (2.0 * s) * b;
        t = t1 + t2;
    } else {
        if (rows <= 0 || cols <= 0 || rows * cols != n) { *status = OR_UNSUPPORTED; return 0; }
        double sc = s / (double)cols, sr = s / (double)rows;
        if (kind == C_AR) {
            t = ring_rs(cols, s, a, b) + ring_ar(rows, sc, a, b);
            t = t + ring_rs(cols, s, a, b);
        } else if (kind == C_AG) {
            t = ring_rs(cols, sr, a, b) + ring_rs(rows, s, a, b);
        } else {
            t = ring_rs(cols, s, a, b) + ring_rs(rows, sc, a, b);
        }
    }
    return rhu(t);
}

int64_t or_duration_from_flops(int64_t flops, double peak, double eff) {
    double d = peak * eff;
    double x = (double)flops / d;
    return rhu(x * 1e9);
}

/* simulator.py:109-114 */
static int64_t coll_duration(const or_graphs *G, int64_t v, const or_config *cfg, int *st) {
    int64_t n = G->grp_off[SV(G, v) + 1] - G->grp_off[SV(G, v)];
    int64_t size = G->coll_kind[SV(G, v)] == C_AG ? G->coll_bytes[SV(G, v)] * n : G->coll_bytes[SV(G, v)];
    int mesh = cfg->topo_kind == 1;
    double beta = 1e9 / cfg->bw;
    return or_analytical_time(G->coll_kind[SV(G, v)], size, n, cfg->algo, (double)cfg->latency, beta,
                              mesh ? cfg->rows : 0, mesh ? cfg->cols : 0, st);
}

/* ------------------------------------------------------------ utilities */

typedef struct { int64_t *a; int64_t n, cap; } vec;
static void vpush(vec *v, int64_t x) {
    if (v->n == v->cap) { v->cap = v->cap ? 2 * v->cap : 8; v->a = realloc(v->a, (size_t)v->cap * sizeof(int64_t)); }
    v->a[v->n++] = x;
}

static int cmp_i64(const void *x, const void *y) {
    int64_t a = *(const int64_t *)x, b = *(const int64_t *)y;
    return a < b ? -1 : a > b;
}

/* generic binary min-heap over fixed-size int64 tuples, lexicographic */
typedef struct { int64_t *a; int64_t n, cap; int w; } heap;
static int hless(const heap *h, int64_t i, int64_t j) {
    const int64_t *x = h->a + i * h->w, *y = h->a + j * h->w;
    for (int k = 0; k < h->w; k++) { if (x[k] != y[k]) return x[k] < y[k]; }
    return 0;
}
static void hswap(heap *h, int64_t i, int64_t j) {
    for (int k = 0; k < h->w; k++) { int64_t t = h->a[i * h->w + k]; h->a[i * h->w + k] = h->a[j * h->w + k]; h->a[j * h->w + k] = t; }
}
static void hpush(heap *h, const int64_t *x) {
    if (h->n == h->cap) { h->cap = h->cap ? 2 * h->cap : 8; h->a = realloc(h->a, (size_t)(h->cap * h->w) * sizeof(int64_t)); }
    memcpy(h->a + h->n * h->w, x, (size_t)h->w * sizeof(int64_t));
    int64_t i = h->n++;
    while (i > 0) { int64_t p = (i - 1) / 2; if (!hless(h, i, p)) break; hswap(h, i, p); i = p; }
}
static void hpop(heap *h, int64_t *out) {
    memcpy(out, h->a, (size_t)h->w * sizeof(int64_t));
    h->n--;
    if (h->n > 0) {
        memcpy(h->a, h->a + h->n * h->w, (size_t)h->w * sizeof(int64_t));
        int64_t i = 0;
        for (;;) {
            int64_t l = 2 * i + 1, r = l + 1, m = i;
            if (l < h->n && hless(h, l, m)) m = l;
            if (r < h->n && hless(h, r, m)) m = r;
            if (m == i) break;
            hswap(h, i, m); i = m;
        }
    }
}

/* rank value -> index, and (rank, node id) -> flat node index */
typedef struct {
    int64_t nr;
    int64_t *sorted_vals, *sorted_idx;      /* rank values sorted, with their index */
    int64_t **ids, **flat;                  /* per rank: sorted node ids + flat index */
    int64_t *cnt;
} lookup;

static int64_t find_sorted(const int64_t *keys, int64_t n, int64_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) { int64_t mid = (lo + hi) / 2; if (keys[mid] < key) lo = mid + 1; else hi = mid; }
    return (lo < n && keys[lo] == key) ? lo : -1;
}
static int64_t rank_index(const lookup *L, int64_t value) {
    int64_t p = find_sorted(L->sorted_vals, L->nr, value);
    return p < 0 ? -1 : L->sorted_idx[p];
}
static int64_t node_index(const lookup *L, int64_t r, int64_t id) {
    int64_t p = find_sorted(L->ids[r], L->cnt[r], id);
    return p < 0 ? -1 : L->flat[r][p];
}

static int build_lookup(const or_graphs *G, lookup *L) {
    int64_t nr = G->n_ranks;
    L->nr = nr;
    L->sorted_vals = malloc((size_t)(nr + 1) * sizeof(int64_t));
    L->sorted_idx = malloc((size_t)(nr + 1) * sizeof(int64_t));
    int64_t *pairs = malloc((size_t)(2 * nr + 2) * sizeof(int64_t));
    for (int64_t r = 0; r < nr; r++) { pairs[2 * r] = G->rank_value[r]; pairs[2 * r + 1] = r; }
    /* sort pairs by value (insertion into sorted arrays via qsort on packed struct) */
    typedef struct { int64_t v, i; } pr;
    qsort(pairs, (size_t)nr, sizeof(pr), cmp_i64);   /* first field is the key */
    int dup = 0;
    for (int64_t r = 0; r < nr; r++) {
        L->sorted_vals[r] = pairs[2 * r]; L->sorted_idx[r] = pairs[2 * r + 1];
        if (r > 0 && pairs[2 * r] == pairs[2 * r - 2]) dup = 1;
    }
    free(pairs);
    L->ids = calloc((size_t)nr + 1, sizeof(int64_t *));
    L->flat = calloc((size_t)nr + 1, sizeof(int64_t *));
    L->cnt = calloc((size_t)nr + 1, sizeof(int64_t));
    for (int64_t r = 0; r < nr; r++) {
        int64_t b = G->node_off[r], e = G->node_off[r + 1], c = e - b;
        int64_t *pp = malloc((size_t)(2 * c + 2) * sizeof(int64_t));
        for (int64_t k = 0; k < c; k++) { pp[2 * k] = G->node_id[SV(G, b + k)]; pp[2 * k + 1] = b + k; }
        qsort(pp, (size_t)c, 2 * sizeof(int64_t), cmp_i64);
        L->ids[r] = malloc((size_t)(c + 1) * sizeof(int64_t));
        L->flat[r] = malloc((size_t)(c + 1) * sizeof(int64_t));
        for (int64_t k = 0; k < c; k++) { L->ids[r][k] = pp[2 * k]; L->flat[r][k] = pp[2 * k + 1]; }
        L->cnt[r] = c;
        free(pp);
    }
    return dup;
}
static void free_lookup(lookup *L) {
    for (int64_t r = 0; r < L->nr; r++) { free(L->ids[r]); free(L->flat[r]); }
    free(L->ids); free(L->flat); free(L->cnt); free(L->sorted_vals); free(L->sorted_idx);
}

/* -------------------------------------------------- collective instances */

typedef struct {
    int64_t n_inst;
    int64_t *mem_off;    /* [n_inst+1] */
    int64_t *mem_rank;   /* rank index, group order */
    int64_t *mem_node;   /* flat node */
    int64_t *lead;       /* flat node of members[0] */
} instances;

static int cmp_pair(const void *a, const void *b) {
    const int64_t *x = a, *y = b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    return x[1] < y[1] ? -1 : x[1] > y[1];
}

/* (rank value, dependency id) pairs of the members' dependencies, ranks taken from `rk`
 * (member q's rank index) -- sorted, for the set comparison below. */
static int64_t dep_pairs(const or_graphs *G, const vec *members, const int64_t *rk, int64_t **out) {
    int64_t n = 0;
    for (int64_t q = 0; q < members->n; q++) {
        int64_t sv = SV(G, members->a[q]);
        n += G->dep_off[sv + 1] - G->dep_off[sv];
    }
    int64_t *p = malloc((size_t)(2 * n + 2) * sizeof(int64_t)), k = 0;
    for (int64_t q = 0; q < members->n; q++) {
        int64_t sv = SV(G, members->a[q]);
        for (int64_t d = G->dep_off[sv]; d < G->dep_off[sv + 1]; d++) {
            p[2 * k] = G->rank_value[rk[q]]; p[2 * k + 1] = G->dep_ids[d]; k++;
        }
    }
    qsort(p, (size_t)n, 2 * sizeof(int64_t), cmp_pair);
    int64_t u = 0;                                   /* set semantics */
    for (int64_t i = 0; i < n; i++)
        if (u == 0 || p[2 * i] != p[2 * u - 2] || p[2 * i + 1] != p[2 * u - 1]) { p[2 * u] = p[2 * i]; p[2 * u + 1] = p[2 * i + 1]; u++; }
    *out = p;
    return u;
}

/* zip(group, members) equals the natural pairing: members[q] carries the node_id of rank
 * group[q]'s own member, and the union of dependencies is the same under both pairings. */
static int zip_pairing_is_natural(const or_graphs *G, const lookup *L, int64_t g0, const vec *members,
                                  const vec *mrank) {
    int64_t n = members->n;
    int64_t *zr = malloc((size_t)(n + 1) * sizeof(int64_t));
    int ok = 1;
    for (int64_t q = 0; q < n && ok; q++) {
        int64_t r = rank_index(L, G->grp_rank[g0 + q]);
        zr[q] = r;
        int64_t own = -1;
        for (int64_t j = 0; j < n; j++) if (mrank->a[j] == r) { own = members->a[j]; break; }
        ok = own >= 0 && G->node_id[SV(G, own)] == G->node_id[SV(G, members->a[q])];
    }
    if (ok) {
        int64_t *a, *b;
        int64_t na = dep_pairs(G, members, mrank->a, &a), nb = dep_pairs(G, members, zr, &b);
        ok = na == nb && memcmp(a, b, (size_t)(2 * na) * sizeof(int64_t)) == 0;
        free(a); free(b);
    }
    free(zr);
    return ok;
}

/* collectives.py:419-453 (instance order = discovery order) */
static int match_instances(const or_graphs *G, const lookup *L, instances *I, int64_t *inst_of,
                           char *err, int errlen) {
    int64_t nr = G->n_ranks;
    vec *colls = calloc((size_t)nr + 1, sizeof(vec));
    for (int64_t r = 0; r < nr; r++)
        for (int64_t v = G->node_off[r]; v < G->node_off[r + 1]; v++)
            if (G->node_kind[SV(G, v)] == K_COLL) vpush(&colls[r], v);
    int64_t *idx = calloc((size_t)nr + 1, sizeof(int64_t));
    vec off = {0}, mr = {0}, mn = {0}, lead = {0};
    vpush(&off, 0);
    int rc = OR_OK;
    for (;;) {
        int64_t start = -1;
        for (int64_t p = 0; p < nr; p++) {           /* sorted(per_rank) */
            int64_t r = L->sorted_idx[p];
            if (idx[r] < colls[r].n) { start = r; break; }
        }
        if (start < 0) break;
        int64_t lv = colls[start].a[idx[start]];
        int64_t g0 = G->grp_off[SV(G, lv)], g1 = G->grp_off[SV(G, lv) + 1];
        /* members = [lead] + others in group order; pairs = zip(group, members) */
        vec members = {0}, mrank = {0};
        vpush(&members, lv);
        vpush(&mrank, start);
        for (int64_t k = g0; k < g1; k++) {
            int64_t rv = G->grp_rank[k];
            int64_t r = rank_index(L, rv);
            if (r == start) continue;
            if (r < 0 || idx[r] >= colls[r].n) {
                char m[256];
                snprintf(m, sizeof m, "rank %lld is missing a collective of the group", (long long)rv);
                set_err(err, errlen, m); rc = OR_INCONSISTENT; free(members.a); goto done;
            }
            int64_t ov = colls[r].a[idx[r]];
            int same = G->coll_kind[SV(G, ov)] == G->coll_kind[SV(G, lv)] && G->coll_bytes[SV(G, ov)] == G->coll_bytes[SV(G, lv)] &&
                       (G->grp_off[SV(G, ov) + 1] - G->grp_off[SV(G, ov)]) == (g1 - g0);
            if (same)
                for (int64_t q = 0; q < g1 - g0; q++)
                    if (G->grp_rank[G->grp_off[SV(G, ov)] + q] != G->grp_rank[g0 + q]) { same = 0; break; }
            if (!same) {
                set_err(err, errlen, "collective disagrees across ranks");
                rc = OR_INCONSISTENT; free(members.a); free(mrank.a); goto done;
            }
            vpush(&members, ov);
            vpush(&mrank, r);
        }
        /* The reference pairs zip(group, members) (simulator.py:222-223, :419-425): rank
         * group[q] with members[q], where members = [lead] + the others in group order.  With
         * the lead listed first (ascending groups, as every producer emits) that is each rank
         * with its own node.  Otherwise it is the same pairing exactly when members[q] has the
         * node_id of rank group[q]'s own collective and the zipped union of the members'
         * dependencies equals the natural one (critical_path, simulator.py:419-428); anything
         * else is rejected (the reference fails there with a KeyError or a spurious cycle). */
        if (members.n != g1 - g0) {
            set_err(err, errlen, "collective group lists a rank twice");
            rc = OR_INCONSISTENT; free(members.a); free(mrank.a); goto done;
        }
        if (rank_index(L, G->grp_rank[g0]) != start &&
            !zip_pairing_is_natural(G, L, g0, &members, &mrank)) {
            set_err(err, errlen, "collective group pairs ranks with other ranks' nodes (zip(group, members))");
            rc = OR_INCONSISTENT; free(members.a); free(mrank.a); goto done;
        }
        int64_t id = lead.n;
        for (int64_t q = 0; q < members.n; q++) {
            vpush(&mr, mrank.a[q]); vpush(&mn, members.a[q]);
            inst_of[members.a[q]] = id;
        }
        vpush(&lead, lv);
        vpush(&off, mr.n);
        for (int64_t k = g0; k < g1; k++) { int64_t r = rank_index(L, G->grp_rank[k]); idx[r]++; }
        free(members.a);
        free(mrank.a);
    }
done:
    for (int64_t r = 0; r < nr; r++) free(colls[r].a);
    free(colls); free(idx);
    I->n_inst = lead.n; I->mem_off = off.a; I->mem_rank = mr.a; I->mem_node = mn.a; I->lead = lead.a;
    return rc;
}

/* ----------------------------------------------------------- messages */

typedef struct { int64_t send, recv, nbytes, send_t, recv_t; } message;

/* simulator.py:177-200; msg_of[flat node] = message index or -1 */
static int pair_messages(const or_graphs *G, const lookup *L, message **out, int64_t *nmsg,
                         int64_t *msg_of, char *err, int errlen) {
    int64_t total = G->node_off[G->n_ranks];
    /* key rows: (src value, dst value, tag, is_recv, node_id, flat) */
    int64_t cnt = 0;
    for (int64_t v = 0; v < total; v++) if (G->node_kind[SV(G, v)] == K_SEND || G->node_kind[SV(G, v)] == K_RECV) cnt++;
    int64_t *rows = malloc((size_t)(cnt * 6 + 6) * sizeof(int64_t));
    int64_t k = 0;
    for (int64_t r = 0; r < G->n_ranks; r++)
        for (int64_t v = G->node_off[r]; v < G->node_off[r + 1]; v++) {
            int kd = G->node_kind[SV(G, v)];
            if (kd != K_SEND && kd != K_RECV) continue;
            int64_t *row = rows + 6 * k++;
            row[0] = kd == K_SEND ? G->rank_value[r] : G->p2p_peer[SV(G, v)];
            row[1] = kd == K_SEND ? G->p2p_peer[SV(G, v)] : G->rank_value[r];
            row[2] = G->p2p_tag[SV(G, v)];
            row[3] = kd == K_RECV;
            row[4] = G->node_id[SV(G, v)];
            row[5] = v;
        }
    /* lexicographic sort of 6-wide rows: simple insertion-free approach via qsort on index */
    int64_t *ord = malloc((size_t)(cnt + 1) * sizeof(int64_t));
    for (int64_t i = 0; i < cnt; i++) ord[i] = i;
    /* bubble-free: use a heap to sort */
    heap h = {0}; h.w = 6;
    for (int64_t i = 0; i < cnt; i++) hpush(&h, rows + 6 * i);
    for (int64_t i = 0; i < cnt; i++) hpop(&h, rows + 6 * i);   /* rows now sorted (in place reuse ok: heap owns copies) */
    free(h.a); free(ord);
    message *msgs = malloc((size_t)(cnt / 2 + 1) * sizeof(message));
    int64_t nm = 0;
    int rc = OR_OK;
    for (int64_t i = 0; i < cnt;) {
        int64_t j = i;
        while (j < cnt && rows[6 * j] == rows[6 * i] && rows[6 * j + 1] == rows[6 * i + 1] && rows[6 * j + 2] == rows[6 * i + 2]) j++;
        int64_t ns = 0, nrv = 0;
        for (int64_t q = i; q < j; q++) { if (rows[6 * q + 3]) nrv++; else ns++; }
        if (ns != nrv) {
            set_err(err, errlen, "channel has unequal sends and recvs");
            rc = OR_DEADLOCK; break;
        }
        /* sends come first (is_recv=0), each sorted by node id */
        for (int64_t q = 0; q < ns; q++) {
            int64_t sv = rows[6 * (i + q) + 5], rv = rows[6 * (i + ns + q) + 5];
            msgs[nm].send = sv; msgs[nm].recv = rv; msgs[nm].nbytes = G->p2p_bytes[SV(G, sv)];
            msgs[nm].send_t = -1; msgs[nm].recv_t = -1;
            msg_of[sv] = nm; msg_of[rv] = nm;
            nm++;
        }
        i = j;
    }
    (void)L;
    free(rows);
    *out = msgs; *nmsg = nm;
    return rc;
}

/* topology.py:68-102.  Link ids: switch eg(src)=2*idx, in(dst)=2*idx+1;
 * mesh "a->b" = 4*a + dir (0:+col 1:-col 2:+row 3:-row). */
static int route(const or_config *cfg, const lookup *L, int64_t src, int64_t dst, int64_t *links) {
    if (src == dst) return 0;
    if (cfg->topo_kind == 0) { links[0] = 2 * rank_index(L, src); links[1] = 2 * rank_index(L, dst) + 1; return 2; }
    int64_t cols = cfg->cols, r = src / cols, c = src % cols, r1 = dst / cols, c1 = dst % cols;
    int n = 0;
    while (c != c1) { int64_t a = r * cols + c; links[n++] = 4 * a + (c1 > c ? 0 : 1); c += c1 > c ? 1 : -1; }
    while (r != r1) { int64_t a = r * cols + c; links[n++] = 4 * a + (r1 > r ? 2 : 3); r += r1 > r ? 1 : -1; }
    return n;
}
static int64_t transfer_ns(const or_config *cfg, int64_t src, int64_t dst, int64_t nbytes) {
    if (src == dst) return 0;
    int64_t hops = 1;
    if (cfg->topo_kind == 1) {
        int64_t cols = cfg->cols;
        hops = llabs(src / cols - dst / cols) + llabs(src % cols - dst % cols);
    }
    double beta = 1e9 / cfg->bw;
    double x = (double)(hops * cfg->latency) + (double)nbytes * beta;
    return rhu(x);
}

/* --------------------------------------------------- interval statistics */

typedef struct { int64_t s, e; } iv;
static int cmp_iv(const void *x, const void *y) {
    const iv *a = x, *b = y;
    if (a->s != b->s) return a->s < b->s ? -1 : 1;
    return a->e < b->e ? -1 : a->e > b->e;
}
/* simulator.py:121-131; merges in place, returns count */
static int64_t merge_iv(iv *a, int64_t n) {
    qsort(a, (size_t)n, sizeof(iv), cmp_iv);
    int64_t m = 0;
    for (int64_t i = 0; i < n; i++) {
        if (a[i].e <= a[i].s) continue;
        if (m > 0 && a[i].s <= a[m - 1].e) { if (a[i].e > a[m - 1].e) a[m - 1].e = a[i].e; }
        else a[m++] = a[i];
    }
    return m;
}
static int64_t total_iv(const iv *a, int64_t n) { int64_t t = 0; for (int64_t i = 0; i < n; i++) t += a[i].e - a[i].s; return t; }
static int64_t overlap_iv(const iv *a, int64_t na, const iv *b, int64_t nb) {   /* :138-149 */
    int64_t i = 0, j = 0, tot = 0;
    while (i < na && j < nb) {
        int64_t s = a[i].s > b[j].s ? a[i].s : b[j].s, e = a[i].e < b[j].e ? a[i].e : b[j].e;
        if (e > s) tot += e - s;
        if (a[i].e < b[j].e) i++; else j++;
    }
    return tot;
}

typedef struct { int64_t t, kind, delta; } memev;
static int cmp_memev(const void *x, const void *y) {
    const memev *a = x, *b = y;
    if (a->t != b->t) return a->t < b->t ? -1 : 1;
    if (a->kind != b->kind) return a->kind < b->kind ? -1 : 1;
    return a->delta < b->delta ? -1 : a->delta > b->delta;
}

/* simulator.py:370-393 */
static int64_t peak_mem(const or_graphs *G, int64_t r, const int64_t *st, const int64_t *en, int64_t finish) {
    int64_t b = G->node_off[r], e = G->node_off[r + 1];
    int64_t t0 = G->tens_lo[r], t1 = G->tens_hi[r], nt = t1 - t0;
    if (nt <= 0) return 0;
    /* tensor ids of this rank's table, sorted for lookup */
    int64_t *tid = malloc((size_t)(2 * nt + 2) * sizeof(int64_t));
    for (int64_t k = 0; k < nt; k++) { tid[2 * k] = G->tens_id[t0 + k]; tid[2 * k + 1] = k; }
    qsort(tid, (size_t)nt, 2 * sizeof(int64_t), cmp_i64);
    int64_t *keys = malloc((size_t)(nt + 1) * sizeof(int64_t)), *pos = malloc((size_t)(nt + 1) * sizeof(int64_t));
    for (int64_t k = 0; k < nt; k++) { keys[k] = tid[2 * k]; pos[k] = tid[2 * k + 1]; }
    free(tid);
    int64_t *alloc = malloc((size_t)(nt + 1) * sizeof(int64_t)), *freet = malloc((size_t)(nt + 1) * sizeof(int64_t));
    char *hasp = calloc((size_t)nt + 1, 1), *hasc = calloc((size_t)nt + 1, 1);
    for (int64_t v = b; v < e; v++) {
        for (int64_t q = G->out_off[SV(G, v)]; q < G->out_off[SV(G, v) + 1]; q++) {   /* producer[t] = last */
            int64_t p = find_sorted(keys, nt, G->out_tid[q]);
            if (p >= 0) { alloc[pos[p]] = st[v]; hasp[pos[p]] = 1; }
        }
        for (int64_t q = G->in_off[SV(G, v)]; q < G->in_off[SV(G, v) + 1]; q++) {
            int64_t p = find_sorted(keys, nt, G->in_tid[q]);
            if (p >= 0) {
                int64_t k = pos[p];
                if (!hasc[k] || en[v] > freet[k]) freet[k] = en[v];
                hasc[k] = 1;
            }
        }
    }
    memev *ev = malloc((size_t)(2 * nt + 2) * sizeof(memev));
    for (int64_t k = 0; k < nt; k++) {
        int64_t by = G->tens_bytes[t0 + k];
        ev[2 * k].t = hasp[k] ? alloc[k] : 0; ev[2 * k].kind = 0; ev[2 * k].delta = by;
        ev[2 * k + 1].t = hasc[k] ? freet[k] : finish; ev[2 * k + 1].kind = 1; ev[2 * k + 1].delta = -by;
    }
    qsort(ev, (size_t)(2 * nt), sizeof(memev), cmp_memev);
    int64_t cur = 0, peak = 0;
    for (int64_t k = 0; k < 2 * nt; k++) { cur += ev[k].delta; if (cur > peak) peak = cur; }
    free(ev); free(keys); free(pos); free(alloc); free(freet); free(hasp); free(hasc);
    return peak;
}

/* ------------------------------------------------------------ simulate */

typedef struct {
    heap host_ready, comp_ready;   /* (node_id, flat) */
    int64_t host_slot;
    int64_t *comp_slots, *comm_slots;
    int64_t wake_version;
    vec comm_iv;                   /* flattened (s, e) pairs */
} rank_state;

/* earliest time at which this rank's start phase could start something */
static int64_t wake_time(const rank_state *R, int ncs) {
    int64_t w = INT64_MAX;
    if (R->host_ready.n && R->host_slot < w) w = R->host_slot;
    if (R->comp_ready.n) { for (int k = 0; k < ncs; k++) if (R->comp_slots[k] < w) w = R->comp_slots[k]; }
    return w;
}

static int simulate_impl(const or_graphs *G, const or_config *cfg, or_sim_out *out, char *err, int errlen);
int or_simulate(const or_graphs *G0, const or_config *cfg, or_sim_out *out, char *err, int errlen) {
    or_graphs g = *G0;
    int64_t *sv = build_sv(G0);
    g.sv = sv;
    int rc = simulate_impl(&g, cfg, out, err, errlen);
    free(sv);
    return rc;
}

static int simulate_impl(const or_graphs *G, const or_config *cfg, or_sim_out *out, char *err, int errlen) {
    int64_t nr = G->n_ranks, total = G->node_off[nr];
    int ncs = cfg->compute_streams, nms = cfg->comm_streams;
    if (ncs < 1 || nms < 1) { set_err(err, errlen, "stream counts must be >= 1"); return OR_INVALID; }
    lookup L;
    if (build_lookup(G, &L)) { free_lookup(&L); set_err(err, errlen, "duplicate rank in graphs"); return OR_INVALID; }
    int rc = OR_OK;
    int64_t *rank_of = malloc((size_t)(total + 1) * sizeof(int64_t));
    for (int64_t r = 0; r < nr; r++) for (int64_t v = G->node_off[r]; v < G->node_off[r + 1]; v++) rank_of[v] = r;

    /* remaining / dependents (simulator.py:212-218) */
    int64_t *remaining = calloc((size_t)total + 1, sizeof(int64_t));
    int64_t *dcount = calloc((size_t)total + 1, sizeof(int64_t));
    int64_t *tmp = NULL; int64_t tmpcap = 0;
    vec edges = {0};   /* (dep flat, node flat) in iteration order */
    for (int64_t v = 0; v < total; v++) {
        int64_t n = G->dep_off[SV(G, v) + 1] - G->dep_off[SV(G, v)];
        if (n > tmpcap) { tmpcap = n; tmp = realloc(tmp, (size_t)tmpcap * sizeof(int64_t)); }
        memcpy(tmp, G->dep_ids + G->dep_off[SV(G, v)], (size_t)n * sizeof(int64_t));
        qsort(tmp, (size_t)n, sizeof(int64_t), cmp_i64);
        int64_t u = 0;
        for (int64_t k = 0; k < n; k++) if (k == 0 || tmp[k] != tmp[k - 1]) tmp[u++] = tmp[k];
        remaining[v] = u;
        for (int64_t k = 0; k < u; k++) {
            int64_t d = node_index(&L, rank_of[v], tmp[k]);
            if (d >= 0) { vpush(&edges, d); vpush(&edges, v); dcount[d]++; }
        }
    }
    free(tmp);
    int64_t *doff = calloc((size_t)total + 2, sizeof(int64_t));
    for (int64_t v = 0; v < total; v++) doff[v + 1] = doff[v] + dcount[v];
    int64_t *dlist = malloc((size_t)(edges.n / 2 + 1) * sizeof(int64_t));
    int64_t *fillp = calloc((size_t)total + 1, sizeof(int64_t));
    for (int64_t k = 0; k < edges.n / 2; k++) { int64_t d = edges.a[2 * k], v = edges.a[2 * k + 1]; dlist[doff[d] + fillp[d]++] = v; }
    free(edges.a); free(fillp); free(dcount);

    /* collective instances (simulator.py:220-226) */
    int64_t *inst_of = malloc((size_t)(total + 1) * sizeof(int64_t));
    for (int64_t v = 0; v < total; v++) inst_of[v] = -1;
    instances I = {0};
    int64_t *inst_dur = NULL, *inst_wait = NULL, *inst_ready = NULL;
    message *msgs = NULL; int64_t nmsg = 0;
    int64_t *msg_of = NULL;
    rank_state *RS = NULL;
    int64_t *st = NULL, *en = NULL;
    rc = match_instances(G, &L, &I, inst_of, err, errlen);
    if (rc) goto cleanup;
    inst_dur = malloc((size_t)(I.n_inst + 1) * sizeof(int64_t));
    inst_wait = malloc((size_t)(I.n_inst + 1) * sizeof(int64_t));
    inst_ready = calloc((size_t)I.n_inst + 1, sizeof(int64_t));
    for (int64_t i = 0; i < I.n_inst; i++) {
        int s2;
        inst_dur[i] = coll_duration(G, I.lead[i], cfg, &s2);
        if (s2) { rc = s2; set_err(err, errlen, "collective algorithm not defined on this topology"); goto cleanup; }
        inst_wait[i] = I.mem_off[i + 1] - I.mem_off[i];
    }
    msg_of = malloc((size_t)(total + 1) * sizeof(int64_t));
    for (int64_t v = 0; v < total; v++) msg_of[v] = -1;
    rc = pair_messages(G, &L, &msgs, &nmsg, msg_of, err, errlen);
    if (rc) goto cleanup;

    RS = calloc((size_t)nr + 1, sizeof(rank_state));
    for (int64_t r = 0; r < nr; r++) {
        RS[r].host_ready.w = 2; RS[r].comp_ready.w = 2;
        RS[r].comp_slots = calloc((size_t)ncs, sizeof(int64_t));
        RS[r].comm_slots = calloc((size_t)nms, sizeof(int64_t));
    }
    st = malloc((size_t)(total + 1) * sizeof(int64_t));
    en = malloc((size_t)(total + 1) * sizeof(int64_t));
    for (int64_t v = 0; v < total; v++) { st[v] = -1; en[v] = -1; }
    int64_t n_links = cfg->topo_kind == 0 ? 2 * nr : 4 * cfg->rows * cfg->cols;
    int64_t *link_free = calloc((size_t)n_links + 1, sizeof(int64_t));
    int64_t *link_busy = malloc((size_t)(n_links + 1) * sizeof(int64_t));
    for (int64_t k = 0; k < n_links; k++) link_busy[k] = -1;

    heap ev = {0}; ev.w = 4;          /* (end, rank value, node id, flat) */
    heap wake = {0}; wake.w = 3;      /* (time, rank idx, version) */
    vec pend_c = {0}, pend_m = {0};
    int64_t done = 0;
    int64_t *links = malloc((size_t)(4 + 2 * (cfg->rows + cfg->cols) + 2) * sizeof(int64_t));

#define FINISH(v, s_, e_) do { st[v] = (s_); en[v] = (e_); int64_t k_[4] = {(e_), G->rank_value[rank_of[v]], G->node_id[SV(G, v)], (v)}; hpush(&ev, k_); } while (0)
#define REWAKE(r) do { int64_t w_ = wake_time(&RS[r], ncs); RS[r].wake_version++; if (w_ != INT64_MAX) { int64_t k_[3] = {w_, (r), RS[r].wake_version}; hpush(&wake, k_); } } while (0)

    /* dispatch (simulator.py:247-268) */
#define DISPATCH(v, now_) do { \
        int64_t r_ = rank_of[v]; int kd_ = G->node_kind[SV(G, v)]; \
        if (kd_ == K_HOST) { int64_t k_[2] = {G->node_id[SV(G, v)], (v)}; hpush(&RS[r_].host_ready, k_); REWAKE(r_); } \
        else if (kd_ == K_COMP) { int64_t k_[2] = {G->node_id[SV(G, v)], (v)}; hpush(&RS[r_].comp_ready, k_); REWAKE(r_); } \
        else if (kd_ == K_COLL) { int64_t i_ = inst_of[v]; inst_wait[i_]--; if ((now_) > inst_ready[i_]) inst_ready[i_] = (now_); \
            if (inst_wait[i_] == 0) vpush(&pend_c, i_); } \
        else { int64_t m_ = msg_of[v]; \
            if (m_ < 0) { set_err(err, errlen, "unmatched send/recv"); rc = OR_DEADLOCK; goto loop_end; } \
            if (msgs[m_].send == (v)) msgs[m_].send_t = (now_); else msgs[m_].recv_t = (now_); \
            if (msgs[m_].send_t >= 0 && msgs[m_].recv_t >= 0) vpush(&pend_m, m_); } \
    } while (0)

    for (int64_t v = 0; v < total; v++) if (remaining[v] == 0) DISPATCH(v, 0);

    int64_t now = 0;
    int64_t tmpk[4];
    for (;;) {
        /* host phase then comp phase, for every rank whose wake time <= now */
        while (wake.n && wake.a[0] <= now) {
            int64_t wk[3]; hpop(&wake, wk);
            int64_t r = wk[1];
            if (wk[2] != RS[r].wake_version) continue;
            rank_state *R = &RS[r];
            while (R->host_ready.n && R->host_slot <= now) {
                hpop(&R->host_ready, tmpk);
                int64_t v = tmpk[1], d = G->node_dur[SV(G, v)] < 0 ? 0 : G->node_dur[SV(G, v)];
                R->host_slot = now + d;
                FINISH(v, now, now + d);
            }
            while (R->comp_ready.n) {
                int k = 0;
                for (int q = 1; q < ncs; q++) if (R->comp_slots[q] < R->comp_slots[k]) k = q;
                if (R->comp_slots[k] > now) break;
                hpop(&R->comp_ready, tmpk);
                int64_t v = tmpk[1], d = G->node_dur[SV(G, v)] < 0 ? 0 : G->node_dur[SV(G, v)];
                R->comp_slots[k] = now + d;
                FINISH(v, now, now + d);
            }
            REWAKE(r);
        }
        if (pend_c.n) {   /* stable sort by (ready_ns, lead node_id) (:298-309) */
            for (int64_t a = 1; a < pend_c.n; a++) {
                int64_t x = pend_c.a[a], b = a - 1;
                while (b >= 0) {
                    int64_t y = pend_c.a[b];
                    int gt = inst_ready[y] > inst_ready[x] ||
                             (inst_ready[y] == inst_ready[x] && G->node_id[SV(G, I.lead[y])] > G->node_id[SV(G, I.lead[x])]);
                    if (!gt) break;
                    pend_c.a[b + 1] = y; b--;
                }
                pend_c.a[b + 1] = x;
            }
            for (int64_t q = 0; q < pend_c.n; q++) {
                int64_t i = pend_c.a[q], s = inst_ready[i];
                for (int64_t m = I.mem_off[i]; m < I.mem_off[i + 1]; m++) {
                    rank_state *R = &RS[I.mem_rank[m]];
                    for (int k = 0; k < nms; k++) if (R->comm_slots[k] > s) s = R->comm_slots[k];
                }
                int64_t e = s + inst_dur[i];
                for (int64_t m = I.mem_off[i]; m < I.mem_off[i + 1]; m++) {
                    rank_state *R = &RS[I.mem_rank[m]];
                    for (int k = 0; k < nms; k++) R->comm_slots[k] = e;
                    vpush(&R->comm_iv, s); vpush(&R->comm_iv, e);
                    FINISH(I.mem_node[m], s, e);
                }
            }
            pend_c.n = 0;
        }
        if (pend_m.n) {   /* stable sort by (max(send_t, recv_t), src rank, src node id) (:310-327) */
            for (int64_t a = 1; a < pend_m.n; a++) {
                int64_t x = pend_m.a[a], b = a - 1;
                message *mx = &msgs[x];
                int64_t kx0 = mx->send_t > mx->recv_t ? mx->send_t : mx->recv_t;
                int64_t kx1 = G->rank_value[rank_of[mx->send]], kx2 = G->node_id[SV(G, mx->send)];
                while (b >= 0) {
                    message *my = &msgs[pend_m.a[b]];
                    int64_t ky0 = my->send_t > my->recv_t ? my->send_t : my->recv_t;
                    int64_t ky1 = G->rank_value[rank_of[my->send]], ky2 = G->node_id[SV(G, my->send)];
                    int gt = ky0 > kx0 || (ky0 == kx0 && (ky1 > kx1 || (ky1 == kx1 && ky2 > kx2)));
                    if (!gt) break;
                    pend_m.a[b + 1] = pend_m.a[b]; b--;
                }
                pend_m.a[b + 1] = x;
            }
            for (int64_t q = 0; q < pend_m.n; q++) {
                message *M = &msgs[pend_m.a[q]];
                int64_t sr = rank_of[M->send], dr = rank_of[M->recv];
                int64_t sv = G->rank_value[sr], dv = G->rank_value[dr];
                int nl = route(cfg, &L, sv, dv, links);
                int64_t s = M->send_t > M->recv_t ? M->send_t : M->recv_t;
                for (int k = 0; k < nl; k++) if (link_free[links[k]] > s) s = link_free[links[k]];
                int64_t e = s + transfer_ns(cfg, sv, dv, M->nbytes);
                for (int k = 0; k < nl; k++) {
                    link_free[links[k]] = e;
                    link_busy[links[k]] = (link_busy[links[k]] < 0 ? 0 : link_busy[links[k]]) + (e - s);
                }
                vpush(&RS[sr].comm_iv, s); vpush(&RS[sr].comm_iv, e);
                if (dr != sr) { vpush(&RS[dr].comm_iv, s); vpush(&RS[dr].comm_iv, e); }
                FINISH(M->send, s, e);
                FINISH(M->recv, s, e);
            }
            pend_m.n = 0;
        }
        if (!ev.n) {
            if (done < total) { set_err(err, errlen, "nodes never became runnable"); rc = OR_DEADLOCK; }
            break;
        }
        int64_t top[4]; hpop(&ev, top);
        now = top[0];
        int64_t x = top[3];
        done++;
        for (int64_t q = doff[x]; q < doff[x + 1]; q++) {
            int64_t v = dlist[q];
            if (--remaining[v] == 0) DISPATCH(v, now);
        }
    }
loop_end:
    if (rc == OR_OK) {
        int64_t makespan = 0;
        for (int64_t v = 0; v < total; v++) if (en[v] > makespan) makespan = en[v];
        out->makespan = makespan;
        iv *cbuf = malloc((size_t)(total + 1) * sizeof(iv));
        for (int64_t r = 0; r < nr; r++) {
            int64_t nc = 0, fin = 0;
            for (int64_t v = G->node_off[r]; v < G->node_off[r + 1]; v++) {
                if (G->node_kind[SV(G, v)] == K_COMP) { cbuf[nc].s = st[v]; cbuf[nc].e = en[v]; nc++; }
                if (en[v] > fin) fin = en[v];
            }
            nc = merge_iv(cbuf, nc);
            int64_t nm = RS[r].comm_iv.n / 2;
            iv *mb = (iv *)RS[r].comm_iv.a;
            nm = nm ? merge_iv(mb, nm) : 0;
            int64_t comm = total_iv(mb, nm);
            int64_t *o = out->rank_stats + 5 * r;
            o[0] = fin;
            o[1] = total_iv(cbuf, nc);
            o[2] = comm;
            o[3] = comm - overlap_iv(mb, nm, cbuf, nc);
            o[4] = peak_mem(G, r, st, en, fin);
        }
        free(cbuf);
        if (out->ev_start) for (int64_t v = 0; v < total; v++) { out->ev_start[v] = st[v]; out->ev_end[v] = en[v]; }
        if (out->link_busy) for (int64_t k = 0; k < n_links && k < out->n_links; k++) out->link_busy[k] = link_busy[k];
        out->n_links = n_links;
    }
    free(ev.a); free(wake.a); free(pend_c.a); free(pend_m.a); free(link_free); free(link_busy); free(links);
cleanup:
    if (RS) for (int64_t r = 0; r < nr; r++) {
        free(RS[r].host_ready.a); free(RS[r].comp_ready.a); free(RS[r].comp_slots); free(RS[r].comm_slots); free(RS[r].comm_iv.a);
    }
    free(RS); free(st); free(en); free(msgs); free(msg_of);
    free(inst_dur); free(inst_wait); free(inst_ready);
    free(I.mem_off); free(I.mem_rank); free(I.mem_node); free(I.lead);
    free(inst_of); free(remaining); free(doff); free(dlist); free(rank_of);
    free_lookup(&L);
    return rc;
#undef FINISH
#undef REWAKE
#undef DISPATCH
}

/* ------------------------------------------------------- critical path */

/* critical_path, optionally with every node's finish and start, its collective
 * instance (-1: none) and, for a RECV, its SEND (-1: none) -- the inputs of the
 * node-trace rule in pyoracle.critical_path_trace.  Flat node order. */
static int critical_path_impl(const or_graphs *G, const or_config *cfg, int64_t *result, int64_t *node_fin,
                              int64_t *node_start, int64_t *node_inst, int64_t *node_send, char *err, int errlen);
int or_critical_path_ex(const or_graphs *G0, const or_config *cfg, int64_t *result, int64_t *node_fin,
                        int64_t *node_start, int64_t *node_inst, int64_t *node_send, char *err, int errlen) {
    or_graphs g = *G0;
    int64_t *sv = build_sv(G0);
    g.sv = sv;
    int rc = critical_path_impl(&g, cfg, result, node_fin, node_start, node_inst, node_send, err, errlen);
    free(sv);
    return rc;
}

static int critical_path_impl(const or_graphs *G, const or_config *cfg, int64_t *result, int64_t *node_fin,
                              int64_t *node_start, int64_t *node_inst, int64_t *node_send, char *err, int errlen) {
    int64_t nr = G->n_ranks, total = G->node_off[nr];
    lookup L;
    if (build_lookup(G, &L)) { free_lookup(&L); set_err(err, errlen, "duplicate rank in graphs"); return OR_INVALID; }
    int rc = OR_OK;
    int64_t *rank_of = malloc((size_t)(total + 1) * sizeof(int64_t));
    for (int64_t r = 0; r < nr; r++) for (int64_t v = G->node_off[r]; v < G->node_off[r + 1]; v++) rank_of[v] = r;
    int64_t *inst_of = malloc((size_t)(total + 1) * sizeof(int64_t));
    for (int64_t v = 0; v < total; v++) inst_of[v] = -1;
    instances I = {0};
    message *msgs = NULL; int64_t nmsg = 0;
    int64_t *msg_of = malloc((size_t)(total + 1) * sizeof(int64_t));
    for (int64_t v = 0; v < total; v++) msg_of[v] = -1;
    /* vertices: nodes 0..total-1 not in an instance, plus one vertex per instance */
    int64_t *vdur = NULL, *vfin = NULL, *indeg = NULL, *soff = NULL, *slist = NULL, *vert_of = NULL;
    vec pe = {0};
    rc = match_instances(G, &L, &I, inst_of, err, errlen);
    if (rc) goto cleanup;
    rc = pair_messages(G, &L, &msgs, &nmsg, msg_of, err, errlen);
    if (rc) goto cleanup;
    int64_t nv = total + I.n_inst;
    vert_of = malloc((size_t)(total + 1) * sizeof(int64_t));
    for (int64_t v = 0; v < total; v++) vert_of[v] = inst_of[v] >= 0 ? total + inst_of[v] : v;
    vdur = calloc((size_t)nv + 1, sizeof(int64_t));
    for (int64_t v = 0; v < total; v++) vdur[v] = G->node_dur[SV(G, v)] < 0 ? 0 : G->node_dur[SV(G, v)];
    for (int64_t i = 0; i < I.n_inst; i++) {
        int s2;
        vdur[total + i] = coll_duration(G, I.lead[i], cfg, &s2);
        if (s2) { rc = s2; set_err(err, errlen, "collective algorithm not defined on this topology"); goto cleanup; }
    }
    /* predecessor pairs (pred flat node or -1-dangling, vertex) -- deduplicated per vertex */
    char *live = calloc((size_t)nv + 1, 1);
    for (int64_t v = 0; v < total; v++) live[vert_of[v]] = 1;
    int64_t dangling_tag = 0;
    {
        /* per vertex, collect raw preds then dedup by sort */
        vec *pv = calloc((size_t)nv + 1, sizeof(vec));
        for (int64_t v = 0; v < total; v++) {
            int64_t w = vert_of[v];
            for (int64_t q = G->dep_off[SV(G, v)]; q < G->dep_off[SV(G, v) + 1]; q++) {
                int64_t d = node_index(&L, rank_of[v], G->dep_ids[q]);
                vpush(&pv[w], d >= 0 ? d : -(++dangling_tag));   /* dangling dep: never finishes */
            }
            if (G->node_kind[SV(G, v)] == K_RECV && msg_of[v] >= 0) vpush(&pv[w], msgs[msg_of[v]].send);
        }
        indeg = calloc((size_t)nv + 1, sizeof(int64_t));
        vec edges = {0};
        for (int64_t w = 0; w < nv; w++) {
            if (!live[w]) continue;
            qsort(pv[w].a, (size_t)pv[w].n, sizeof(int64_t), cmp_i64);
            for (int64_t k = 0; k < pv[w].n; k++) {
                if (k > 0 && pv[w].a[k] == pv[w].a[k - 1]) continue;
                indeg[w]++;
                if (pv[w].a[k] >= 0) { vpush(&edges, pv[w].a[k]); vpush(&edges, w); }
            }
            free(pv[w].a);
        }
        free(pv);
        int64_t *cnt = calloc((size_t)total + 1, sizeof(int64_t));
        for (int64_t k = 0; k < edges.n / 2; k++) cnt[edges.a[2 * k]]++;
        soff = calloc((size_t)total + 2, sizeof(int64_t));
        for (int64_t v = 0; v < total; v++) soff[v + 1] = soff[v] + cnt[v];
        slist = malloc((size_t)(edges.n / 2 + 1) * sizeof(int64_t));
        memset(cnt, 0, (size_t)(total + 1) * sizeof(int64_t));
        for (int64_t k = 0; k < edges.n / 2; k++) { int64_t d = edges.a[2 * k]; slist[soff[d] + cnt[d]++] = edges.a[2 * k + 1]; }
        free(cnt); free(edges.a);
    }
    vfin = calloc((size_t)nv + 1, sizeof(int64_t));
    int64_t *vstart = calloc((size_t)nv + 1, sizeof(int64_t));
    int64_t *queue = malloc((size_t)(nv + 1) * sizeof(int64_t));
    int64_t qh = 0, qt = 0, seen = 0;
    for (int64_t w = 0; w < nv; w++) if (live[w] && indeg[w] == 0) queue[qt++] = w;
    while (qh < qt) {
        int64_t w = queue[qh++];
        int64_t start = vstart[w];
        if (w < total && G->node_kind[SV(G, w)] == K_RECV && msg_of[w] >= 0) {   /* :450-452 */
            message *M = &msgs[msg_of[w]];
            int64_t sv = G->rank_value[rank_of[M->send]], dv = G->rank_value[rank_of[M->recv]];
            int64_t wire = vfin[vert_of[M->send]] + transfer_ns(cfg, sv, dv, M->nbytes);
            if (wire > start) start = wire;
        }
        vfin[w] = start + vdur[w];
        vstart[w] = start;
        seen += w < total ? 1 : (I.mem_off[w - total + 1] - I.mem_off[w - total]);
        /* successors of every node that maps to this vertex */
        if (w < total) {
            for (int64_t q = soff[w]; q < soff[w + 1]; q++) {
                int64_t s = slist[q];
                if (vfin[w] > vstart[s]) vstart[s] = vfin[w];
                if (--indeg[s] == 0) queue[qt++] = s;
            }
        } else {
            int64_t i = w - total;
            for (int64_t m = I.mem_off[i]; m < I.mem_off[i + 1]; m++) {
                int64_t v = I.mem_node[m];
                for (int64_t q = soff[v]; q < soff[v + 1]; q++) {
                    int64_t s = slist[q];
                    if (vfin[w] > vstart[s]) vstart[s] = vfin[w];
                    if (--indeg[s] == 0) queue[qt++] = s;
                }
            }
        }
    }
    if (seen != total) { set_err(err, errlen, "cyclic cross-rank wait in critical path"); rc = OR_DEADLOCK; }
    else {
        int64_t best = 0;
        for (int64_t w = 0; w < nv; w++) if (live[w] && vfin[w] > best) best = vfin[w];
        *result = best;
        if (node_fin)
            for (int64_t v = 0; v < total; v++) {
                node_fin[v] = vfin[vert_of[v]];
                node_start[v] = vstart[vert_of[v]];
                node_inst[v] = inst_of[v];
                node_send[v] = (G->node_kind[SV(G, v)] == K_RECV && msg_of[v] >= 0) ? msgs[msg_of[v]].send : -1;
            }
    }
    free(vstart); free(queue); free(live);
cleanup:
    (void)pe;
    free(vdur); free(vfin); free(indeg); free(soff); free(slist); free(vert_of);
    free(msgs); free(msg_of);
    free(I.mem_off); free(I.mem_rank); free(I.mem_node); free(I.lead);
    free(inst_of); free(rank_of);
    free_lookup(&L);
    return rc;
}

int or_critical_path(const or_graphs *G, const or_config *cfg, int64_t *result, char *err, int errlen) {
    return or_critical_path_ex(G, cfg, result, NULL, NULL, NULL, NULL, err, errlen);
}
