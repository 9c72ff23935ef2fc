// capi.cu -- the extern "C" boundary declared in include/flint_b200.h.
//
// Owns device memory for compiled graph sets (fl_graph) and their per-CTA
// scratch, validates descriptors, launches the engine kernels.  No torch
// types cross this boundary; the Python layer binds it with ctypes.

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <array>
#include <string>
#include <vector>

#include "flint_b200.h"
#include "engine_internal.h"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string &msg) {
    g_err = msg;
    return code;
}

#define CK(expr)                                                                      \
    do {                                                                              \
        cudaError_t e_ = (expr);                                                      \
        if (e_ != cudaSuccess)                                                        \
            return fail(FL_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
    } while (0)

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

struct fl_graph {
    int device;
    fl::DevGraph dg;
    std::vector<void *> allocs;
    // scratch, grown on demand
    unsigned char *scratch = nullptr;
    size_t scratch_bytes = 0;
    fl::DevScratch sc{};
    // staging for fl_sweep_run (host-buffer entry point), grown on demand: a device block and
    // its pinned host mirror, so inputs go up in one copy and rows come back in one
    unsigned char *stage = nullptr;
    size_t stage_bytes = 0;
    unsigned char *hstage = nullptr;
    size_t hstage_bytes = 0;
    unsigned char *hstage_dev = nullptr;   // its device alias (mapped pinned memory)
    cudaStream_t stream = nullptr;  // fl_sweep_run's own non-blocking stream (not the legacy one)
    int grid_cap = 0;
    int links_sm_cap = 0;           // link-table capacity reserved in shared memory
    int block = 32;
    int cluster = 1;
    size_t smem = 0;
};

namespace {

template <typename T>
int upload(fl_graph *g, const T *host, size_t n, const T **dev) {
    if (n == 0) n = 1;   // keep a valid pointer for empty tables
    void *p = nullptr;
    CK(cudaMalloc(&p, n * sizeof(T)));
    g->allocs.push_back(p);
    if (host) CK(cudaMemcpy(p, host, n * sizeof(T), cudaMemcpyHostToDevice));
    else CK(cudaMemset(p, 0, n * sizeof(T)));
    *dev = static_cast<const T *>(p);
    return FL_OK;
}

#define UP(field, n)                                                   \
    do {                                                               \
        int rc_ = upload(g, d->field, (size_t)(n), &g->dg.field);      \
        if (rc_) return rc_;                                           \
    } while (0)

int create(const fl_graph_desc *d, int32_t device, fl_graph *g) {
    if (!d || d->n_ranks < 1 || d->n_structs < 1) return fail(FL_ERR_INVALID, "empty graph set");
    if (d->n_ranks > FL_MAX_RANKS)
        return fail(FL_ERR_CAPACITY, "this build evaluates at most " + std::to_string(FL_MAX_RANKS) + " ranks per design point");
    const int R = d->n_ranks, S = d->n_structs;
    int max_nodes = 0;
    for (int s = 0; s < S; s++) {
        int n = d->s_node_off[s + 1] - d->s_node_off[s];
        if (n > FL_MAX_NODES_PER_RANK)
            return fail(FL_ERR_CAPACITY, "a rank graph has more than " + std::to_string(FL_MAX_NODES_PER_RANK) + " nodes");
        max_nodes = n > max_nodes ? n : max_nodes;
    }
    for (int r = 0; r < R; r++)
        if (d->rank_struct[r] < 0 || d->rank_struct[r] >= S) return fail(FL_ERR_INVALID, "rank_struct out of range");
    const int total = d->s_node_off[S], total_t = d->s_tens_off[S];
    for (int i = 0; i < total; i++) {
        int k = d->node_kind[i];
        if (k > FL_RECV) return fail(FL_ERR_INVALID, "bad node kind");
        if (d->succ_off[i + 1] - d->succ_off[i] >= 4096) return fail(FL_ERR_CAPACITY, "node fan-out >= 4096");
    }
    CK(cudaSetDevice(device));
    g->device = device;
    fl::DevGraph &dg = g->dg;
    dg.R = R;
    dg.S = S;
    dg.n_inst = d->n_inst;
    dg.coll_stride = d->coll_stride > 0 ? d->coll_stride : 1;
    dg.max_nodes = max_nodes > 0 ? max_nodes : 1;
    dg.max_words = (dg.max_nodes + 63) / 64;
    dg.total_nodes = total;
    dg.total_tens = total_t;
    dg.n_succ = d->succ_off[total];
    const int ne_pred = d->pred_off[total], ne_succ = d->succ_off[total], ne_free = d->free_off[total];
    const int ne_cons = d->tens_cons_off[total_t], ne_init = d->s_init_off[S];
    const int64_t ne_mem = d->inst_mem_off[d->n_inst];
    UP(rank_struct, R);
    UP(s_node_off, S + 1);
    UP(s_tens_off, S + 1);
    UP(s_init_off, S + 1);
    UP(s_ncoll, S);
    UP(s_init_alloc, S);
    UP(node_kind, total);
    UP(node_flags, total);
    UP(node_dur, total);
    UP(node_flops, total);
    UP(node_alloc, total);
    UP(node_coll_ord, total);
    UP(pred_off, total + 1);
    UP(pred_idx, ne_pred);
    UP(succ_off, total + 1);
    UP(succ_idx, ne_succ);
    UP(free_off, total + 1);
    UP(init_list, ne_init);
    UP(tens_bytes, total_t);
    UP(tens_cons_off, total_t + 1);
    UP(tens_cons, ne_cons);
    UP(inst_kind, d->n_inst);
    UP(inst_n, d->n_inst);
    UP(inst_bytes, d->n_inst);
    UP(inst_lead_id, d->n_inst);
    UP(inst_init_key, d->n_inst);
    UP(inst_mem_off, d->n_inst + 1);
    UP(inst_mem_rank, ne_mem);
    UP(inst_mem_node, ne_mem);
    if (d->n_msg < 0 || d->p2p_stride > FL_MAX_P2P_PER_RANK) return fail(FL_ERR_CAPACITY, "too many SEND/RECV nodes per rank");
    dg.n_msg = d->n_msg;
    dg.p2p_stride = d->p2p_stride > 0 ? d->p2p_stride : 1;
    UP(rank_value, R);
    UP(msg_send_rank, d->n_msg);
    UP(msg_send_node, d->n_msg);
    UP(msg_recv_rank, d->n_msg);
    UP(msg_recv_node, d->n_msg);
    UP(msg_bytes, d->n_msg);
    UP(msg_send_id, d->n_msg);
    if (d->n_msg > 0 || dg.p2p_stride > 1) {
        // every SEND/RECV must be paired (simulator.py:177-200); an unmatched channel would make the
        // kernel index message -1, so refuse it here (the Python layer raises DeadlockError first)
        std::vector<int> s_p2p(S, 0);
        for (int s = 0; s < S; s++)
            for (int i = d->s_node_off[s]; i < d->s_node_off[s + 1]; i++)
                s_p2p[s] += d->node_kind[i] == FL_SEND || d->node_kind[i] == FL_RECV;
        for (int r = 0; r < R; r++) {
            const int c = s_p2p[d->rank_struct[r]];
            if (c > dg.p2p_stride) return fail(FL_ERR_INVALID, "p2p_stride below a rank's SEND/RECV count");
            for (int q = 0; q < c; q++) {
                const int m = d->rank_p2p_msg[(size_t)r * dg.p2p_stride + q];
                if (m < 0 || m >= d->n_msg) return fail(FL_ERR_DEADLOCK, "a SEND/RECV has no matching peer (unmatched channel)");
            }
        }
    }
    {
        int rc = upload(g, d->rank_p2p_msg, (size_t)R * dg.p2p_stride, &dg.rank_p2p_msg);
        if (rc) return rc;
        // the message phase's static tie order (simulator.py:311: source rank, then SEND node_id)
        std::vector<int32_t> by((size_t)(d->n_msg > 0 ? d->n_msg : 1)), ord(by.size(), 0);
        for (int m = 0; m < d->n_msg; m++) by[m] = m;
        std::sort(by.begin(), by.begin() + d->n_msg, [&](int a, int b) {
            const int64_t ra = d->rank_value[d->msg_send_rank[a]], rb = d->rank_value[d->msg_send_rank[b]];
            if (ra != rb) return ra < rb;
            if (d->msg_send_id[a] != d->msg_send_id[b]) return d->msg_send_id[a] < d->msg_send_id[b];
            return a < b;
        });
        for (int k = 0; k < d->n_msg; k++) ord[by[k]] = k;
        rc = upload(g, ord.data(), ord.size(), &dg.msg_ord);
        if (rc) return rc;
        dg.msg_self = 0;
        dg.msg_min_bytes = INT64_MAX;
        for (int m = 0; m < d->n_msg; m++) {
            dg.msg_self |= d->msg_send_rank[m] == d->msg_recv_rank[m];
            dg.msg_min_bytes = std::min<int64_t>(dg.msg_min_bytes, d->msg_bytes[m]);
        }
    }
    {
        int rc = upload(g, d->rank_coll_inst, (size_t)R * dg.coll_stride, &dg.rank_coll_inst);
        if (rc) return rc;
        std::vector<int32_t> full((size_t)(d->n_inst > 0 ? d->n_inst : 1), -1);
        for (int i = 0; i < d->n_inst; i++) {
            const int64_t m0 = d->inst_mem_off[i], nm = d->inst_mem_off[i + 1] - m0;
            if (nm != R) continue;
            const int node = d->inst_mem_node[m0];
            bool ok = true;
            for (int64_t j = 0; j < nm && ok; j++) ok = d->inst_mem_rank[m0 + j] == j && d->inst_mem_node[m0 + j] == node;
            if (ok) full[i] = node;
        }
        rc = upload(g, full.data(), full.size(), &dg.inst_full_node);
        if (rc) return rc;
    }

    // packed node records and tensor consumer ranges (engine.cu node record layout)
    {
        std::vector<uint4> rec(2 * (size_t)(total > 0 ? total : 1));
        std::vector<int32_t> mfree_off((size_t)(total > 0 ? total : 1), 0);
        std::vector<int32_t> mfree;
        mfree.reserve((size_t)ne_free + 1);
        // static hosts: zero in-degree, zero duration, no tensors (all start and end at t=0)
        std::vector<char> is_static((size_t)total + 1, 0);
        std::vector<int32_t> s_nstatic(S, 0), s_fold(S, 1), trig_off(S + 1, 0), static_off(S + 1, 0), static_list;
        std::vector<int4> trig;
        for (int s = 0; s < S; s++) {
            for (int i = d->s_node_off[s]; i < d->s_node_off[s + 1]; i++) {
                const bool zero_in = d->pred_off[i + 1] == d->pred_off[i] && !(d->node_flags[i] & 1);
                if (d->node_kind[i] == FL_HOST && zero_in && d->node_dur[i] == 0) {
                    is_static[i] = 1;
                    s_nstatic[s]++;
                    static_list.push_back(i - d->s_node_off[s]);
                    if (d->free_off[i + 1] != d->free_off[i] || d->node_alloc[i] != 0) s_fold[s] = 0;
                }
            }
            static_off[s + 1] = (int32_t)static_list.size();
        }
        // A tensor is freed when its last consumer completes (simulator.py:384-388).
        // When one consumer depends (transitively) on all the others it is always the
        // last to finish, so the free can be attributed to it statically.
        std::vector<int32_t> last_cons((size_t)(total_t > 0 ? total_t : 1), -1);
        // Dependency-edge classes (engine.cu pop_event), with static hosts folded away:
        // when a node's remaining predecessors are totally ordered by ancestry, the order
        // in which they complete is the same in every schedule, so its readiness needs no
        // counting -- the first only writes the critical-path accumulator, the middle ones
        // max into it without reading it back, and the last reads it and dispatches.
        std::vector<int32_t> succ_ent((size_t)(ne_succ > 0 ? ne_succ : 1));
        int n_acc = 1;
        for (int q = 0; q < ne_succ; q++) succ_ent[q] = d->succ_idx[q];      // class 0: counted
        for (int s = 0; s < S; s++) {
            const int nb = d->s_node_off[s], n = d->s_node_off[s + 1] - nb;
            const int tb = d->s_tens_off[s], nt = d->s_tens_off[s + 1] - tb;
            const int W = (n + 63) / 64;
            std::vector<uint64_t> anc((size_t)n * (W > 0 ? W : 1), 0);
            std::vector<int> indeg(n), order;
            order.reserve(n);
            for (int v = 0; v < n; v++) {
                indeg[v] = d->pred_off[nb + v + 1] - d->pred_off[nb + v];
                if (!indeg[v]) order.push_back(v);
            }
            for (size_t k = 0; k < order.size(); k++) {
                const int v = order[k];
                for (int q = d->succ_off[nb + v]; q < d->succ_off[nb + v + 1]; q++) {
                    const int w = d->succ_idx[q];
                    uint64_t *aw = &anc[(size_t)w * W];
                    const uint64_t *av = &anc[(size_t)v * W];
                    for (int k2 = 0; k2 < W; k2++) aw[k2] |= av[k2];
                    aw[v >> 6] |= 1ull << (v & 63);
                    if (--indeg[w] == 0) order.push_back(w);
                }
            }
            if ((int)order.size() != n) continue;   // cyclic: leave every free to the run-time check
            {
                auto is_anc = [&](int a, int b) { return (anc[(size_t)b * W + (a >> 6)] >> (a & 63)) & 1ull; };
                std::vector<int> P;
                for (int x = 0; x < n; x++) {
                    if (is_static[nb + x]) continue;
                    for (int q = d->succ_off[nb + x]; q < d->succ_off[nb + x + 1]; q++) {
                        const int w = d->succ_idx[q];
                        P.clear();
                        for (int u = d->pred_off[nb + w]; u < d->pred_off[nb + w + 1]; u++)
                            if (!is_static[nb + d->pred_idx[u]]) P.push_back(d->pred_idx[u]);
                        int cls = 0;
                        if (P.size() == 1) {
                            cls = fl::FL_EDGE_SINGLE;
                        } else {
                            bool ordered = true, first = true, last = true;
                            for (size_t i = 0; i < P.size() && ordered; i++)
                                for (size_t j = i + 1; j < P.size() && ordered; j++)
                                    ordered = is_anc(P[i], P[j]) || is_anc(P[j], P[i]);
                            for (int p : P) {
                                if (p == x) continue;
                                first &= is_anc(x, p);
                                last &= is_anc(p, x);
                            }
                            if (ordered) cls = first ? fl::FL_EDGE_FIRST : last ? fl::FL_EDGE_LAST : fl::FL_EDGE_MID;
                        }
                        succ_ent[q] = w | (cls << 16);
                    }
                }
                // Accumulator slots.  A statically ordered node's accumulator is live from the
                // completion of its first dependency (the FIRST write) to that of its last (the
                // LAST read): [pop(first), pop(last)].  When last(a) is a proper ancestor of
                // first(b), pop(last(a)) precedes first(b)'s dispatch in every schedule, so a and
                // b can share one word.  Greedy colouring in order of the first dependency; nodes
                // that wait on a missing node get a slot of their own.  (C3: 319 nodes, 15 slots
                // -- 120 KB per 1024-rank point instead of the 6.8 MB [node][rank] table, which
                // keeps the accumulator traffic in L2.)
                std::vector<std::array<int, 3>> ord;     // {first, last, node}
                std::vector<int> slot_of(n, -1);
                for (int w = 0; w < n; w++) {
                    P.clear();
                    for (int u = d->pred_off[nb + w]; u < d->pred_off[nb + w + 1]; u++)
                        if (!is_static[nb + d->pred_idx[u]]) P.push_back(d->pred_idx[u]);
                    if (P.size() < 2) continue;
                    int f = -1, l = -1;
                    bool ordered = true;
                    for (size_t i = 0; i < P.size() && ordered; i++)
                        for (size_t j = i + 1; j < P.size() && ordered; j++)
                            ordered = is_anc(P[i], P[j]) || is_anc(P[j], P[i]);
                    if (!ordered) continue;
                    for (int p : P) {
                        bool isf = true, isl = true;
                        for (int o : P) if (o != p) { isf &= is_anc(p, o); isl &= is_anc(o, p); }
                        if (isf) f = p;
                        if (isl) l = p;
                    }
                    ord.push_back({f, l, w});
                }
                std::sort(ord.begin(), ord.end());
                std::vector<std::vector<std::array<int, 3>>> slots;
                for (const auto &e : ord) {
                    const bool never = d->node_flags[nb + e[2]] & 1;
                    size_t k = 0;
                    for (; !never && k < slots.size(); k++) {
                        bool ok = !slots[k].empty() && !(d->node_flags[nb + slots[k][0][2]] & 1);
                        for (size_t m = 0; m < slots[k].size() && ok; m++) {
                            const auto &o = slots[k][m];
                            ok = is_anc(o[1], e[0]) || is_anc(e[1], o[0]);
                        }
                        if (ok) break;
                    }
                    if (never || k == slots.size()) slots.emplace_back();
                    k = never ? slots.size() - 1 : k;
                    slots[k].push_back(e);
                    slot_of[e[2]] = (int)k;
                }
                if (slots.size() >= 8192) return fail(FL_ERR_CAPACITY, "more than 8191 accumulator slots");
                n_acc = std::max<int>(n_acc, (int)slots.size());
                for (int x = 0; x < n; x++)
                    for (int q = d->succ_off[nb + x]; q < d->succ_off[nb + x + 1]; q++) {
                        const int cls = (succ_ent[q] >> 16) & 7;
                        if (cls == fl::FL_EDGE_FIRST || cls == fl::FL_EDGE_MID || cls == fl::FL_EDGE_LAST) {
                            const int w = d->succ_idx[q];
                            if (slot_of[w] < 0) return fail(FL_ERR_INVALID, "ordered edge without an accumulator slot");
                            succ_ent[q] |= slot_of[w] << 19;
                        }
                    }
            }
            for (int t = 0; t < nt; t++) {
                const int c0 = d->tens_cons_off[tb + t], c1 = d->tens_cons_off[tb + t + 1];
                if (c1 - c0 < 2) continue;
                for (int a = c0; a < c1; a++) {
                    const int cand = d->tens_cons[a];
                    bool dom = true;
                    for (int b = c0; b < c1 && dom; b++) {
                        const int o = d->tens_cons[b];
                        if (o != cand) dom = (anc[(size_t)cand * W + (o >> 6)] >> (o & 63)) & 1ull;
                    }
                    if (dom) { last_cons[tb + t] = cand; break; }
                }
            }
        }
        // tracked consumers: the nodes whose completion the run-time free check of a shared
        // tensor reads (the `done` bitmap); a lean variant's other pops skip the bitmap write
        std::vector<uint8_t> tracked((size_t)(total > 0 ? total : 1), 0);
        for (int s = 0; s < S; s++) {
            const int nb = d->s_node_off[s], tb = d->s_tens_off[s], nt = d->s_tens_off[s + 1] - tb;
            for (int t = 0; t < nt; t++) {
                const int c0 = d->tens_cons_off[tb + t], c1 = d->tens_cons_off[tb + t + 1];
                if (c1 - c0 < 2 || last_cons[tb + t] >= 0) continue;
                for (int a = c0; a < c1; a++) tracked[nb + d->tens_cons[a]] = 1;
            }
        }
        if (ne_succ >= (1 << 30)) return fail(FL_ERR_CAPACITY, "too many dependency edges");
        int s_of = 0;
        for (int i = 0; i < total; i++) {
            while (s_of + 1 < S && i >= d->s_node_off[s_of + 1]) s_of++;
            const int nb = d->s_node_off[s_of], tb = d->s_tens_off[s_of];
            const int indeg = d->pred_off[i + 1] - d->pred_off[i];
            if (indeg > 1023) return fail(FL_ERR_CAPACITY, "node in-degree > 1023");
            int indeg_nh = 0;
            for (int q = d->pred_off[i]; q < d->pred_off[i + 1]; q++) indeg_nh += !is_static[nb + d->pred_idx[q]];
            uint64_t ufree = 0;
            const uint32_t m0 = (uint32_t)mfree.size();
            for (int q = d->free_off[i]; q < d->free_off[i + 1]; q++) {
                const int t = d->free_tens[q];
                const int nc = d->tens_cons_off[tb + t + 1] - d->tens_cons_off[tb + t];
                if (nc == 1 || last_cons[tb + t] == i - nb) ufree += (uint64_t)d->tens_bytes[tb + t];
                else if (last_cons[tb + t] < 0) mfree.push_back(t);     // decided at run time (done bitmap)
            }
            const uint64_t alloc = (uint64_t)d->node_alloc[i];
            const unsigned meta = (unsigned)d->node_kind[i] | ((unsigned)(d->node_flags[i] & 1) << 4) |
                                  ((unsigned)is_static[i] << 5) | ((unsigned)indeg_nh << 6) | ((unsigned)indeg << 16);
            const uint32_t nmf = (uint32_t)mfree.size() - m0;
            if (nmf > 0xfff) return fail(FL_ERR_CAPACITY, "a node frees more than 4095 shared tensors");
            // offset + 1 of the node's first "last" dependency edge (its accumulator read is
            // issued before the other edges are processed), 0 when none or beyond 255
            uint32_t lo = 0;
            for (int q = d->succ_off[i]; q < d->succ_off[i + 1] && q - d->succ_off[i] < 255; q++)
                if (((uint32_t)succ_ent[q] >> 16 & 7u) == (uint32_t)fl::FL_EDGE_LAST) { lo = q - d->succ_off[i] + 1; break; }
            mfree_off[i] = (int32_t)m0;
            rec[2 * i] = make_uint4((unsigned)d->succ_off[i] | ((unsigned)tracked[i] << 31),
                                    (unsigned)(d->succ_off[i + 1] - d->succ_off[i]) | (nmf << 12) | (lo << 24),
                                    (uint32_t)ufree, (uint32_t)(ufree >> 32));
            rec[2 * i + 1] = make_uint4(meta, (unsigned)(d->node_coll_ord[i] < 0 ? 0 : d->node_coll_ord[i]),
                                        (uint32_t)alloc, (uint32_t)(alloc >> 32));
        }
        // nodes whose every dependency is a static host become ready during the t=0 pops of
        // those hosts, right after the highest-id one (the trigger); listed by (trigger, position)
        for (int s = 0; s < S; s++) {
            const int nb = d->s_node_off[s];
            for (int h = nb; h < d->s_node_off[s + 1]; h++) {
                if (!is_static[h]) continue;
                int seq = 0;
                for (int q = d->succ_off[h]; q < d->succ_off[h + 1]; q++, seq++) {
                    const int v = nb + d->succ_idx[q];
                    if (d->node_flags[v] & 1) continue;
                    bool host_only = true;
                    int last = -1;
                    for (int u = d->pred_off[v]; u < d->pred_off[v + 1]; u++) {
                        host_only &= is_static[nb + d->pred_idx[u]] != 0;
                        last = d->pred_idx[u] > last ? d->pred_idx[u] : last;
                    }
                    if (host_only && last == h - nb) trig.push_back(make_int4(h - nb, v - nb, seq, 0));
                }
            }
            trig_off[s + 1] = (int32_t)trig.size();
        }
        // the initial dispatch list without static hosts (what the folded t = 0 visits)
        std::vector<int32_t> init_ns_off(S + 1, 0), init_ns;
        for (int s = 0; s < S; s++) {
            const int nb = d->s_node_off[s];
            for (int q = d->s_init_off[s]; q < d->s_init_off[s + 1]; q++) {
                const int v = d->init_list[q];
                if (!is_static[nb + v] && !(d->node_flags[nb + v] & 1)) init_ns.push_back(v);
            }
            init_ns_off[s + 1] = (int32_t)init_ns.size();
        }
        if (init_ns.empty()) init_ns.push_back(0);
        int fold_ok = 1;
        for (int s = 0; s < S; s++) fold_ok &= s_fold[s];
        dg.fold_ok = fold_ok;
        dg.dyn_host = 0;
        for (int i = 0; i < total; i++) dg.dyn_host |= d->node_kind[i] == FL_HOST && !is_static[i];
        std::vector<int2> tc((size_t)(total_t > 0 ? total_t : 1));
        for (int i = 0; i < total_t; i++) tc[i] = make_int2(d->tens_cons_off[i], d->tens_cons_off[i + 1]);
        dg.needs_done = !mfree.empty();
        if (mfree.empty()) mfree.push_back(0);
        if (trig.empty()) trig.push_back(make_int4(0, 0, 0, 0));
        if (static_list.empty()) static_list.push_back(0);
        int rc = upload(g, rec.data(), rec.size(), &dg.node_rec);
        if (!rc) rc = upload(g, tc.data(), tc.size(), &dg.tens_rng);
        if (!rc) rc = upload(g, mfree.data(), mfree.size(), &dg.free_tens);
        if (!rc) rc = upload(g, s_nstatic.data(), s_nstatic.size(), &dg.s_nstatic);
        // sinks: every node precedes one, so a rank whose sinks all popped popped everything, its
        // last pop is a sink and so is its largest critical-path finish (engine.cu pop_event, lean)
        std::vector<int32_t> s_nsink(S, 0);
        for (int s = 0; s < S; s++)
            for (int i = d->s_node_off[s]; i < d->s_node_off[s + 1]; i++)
                s_nsink[s] += d->succ_off[i + 1] == d->succ_off[i] && !is_static[i];
        if (!rc) rc = upload(g, s_nsink.data(), s_nsink.size(), &dg.s_nsink);
        if (!rc) rc = upload(g, succ_ent.data(), succ_ent.size(), &dg.succ_ent);
        dg.n_acc = n_acc;
        if (!rc) rc = upload(g, mfree_off.data(), mfree_off.size(), &dg.mfree_off);
        if (!rc) rc = upload(g, init_ns_off.data(), init_ns_off.size(), &dg.s_init_ns_off);
        if (!rc) rc = upload(g, init_ns.data(), init_ns.size(), &dg.init_ns);
        if (!rc) rc = upload(g, trig_off.data(), trig_off.size(), &dg.trig_off);
        if (!rc) rc = upload(g, trig.data(), trig.size(), &dg.trig);
        if (!rc) rc = upload(g, static_off.data(), static_off.size(), &dg.static_off);
        if (!rc) rc = upload(g, static_list.data(), static_list.size(), &dg.static_list);
        if (rc) return rc;
    }

    // launch geometry: one thread per rank; a design point runs on one CTA, or on a
    // cluster of CS CTAs of ceil(R / CS) ranks each when it has more ranks than a CTA has
    // threads.  The kernel is issue-bound with one CTA per SM, so a point's time scales with
    // the ranks per CTA, and clusters must fit inside a GPC: CS is the size that maximizes
    // (co-resident clusters) / (ranks per CTA) -- on B200 a 9-CTA cluster of 911 ranks
    // leaves fewer SMs idle than 8 CTAs of 1024 (FL_CLUSTER_CTAS forces a size, for A/B).
    int sms = 0, optin = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
    const int cs_min = (R + 1023) / 1024;
    int cs_lo = cs_min, cs_hi = cs_min > 1 ? 16 : 1;
    if (cs_min > 1) {
        if (const char *ev = getenv("FL_CLUSTER_CTAS")) {
            const int f = atoi(ev);
            if (f >= cs_min && f <= 16) cs_lo = cs_hi = f;
        }
    }
    int best_cs = -1;
    double best_score = -1.0;
    for (int pass = 0; pass < 2; pass++) {
    for (int CS = cs_lo; CS <= cs_hi; CS++) {
    if (pass == 1 && CS != best_cs) continue;
    const int per = (R + CS - 1) / CS;
    g->cluster = CS;
    g->block = (per + 31) / 32 * 32;
    if (CS > 1 && (CS - 1) * g->block >= R) continue;     // the last CTA would own no rank

    // per-CTA scratch (global) layout
    fl::DevScratch &sc = g->sc;
    const size_t inst_bytes = (size_t)(d->n_inst > 0 ? d->n_inst : 1) * (5 * 8 + 2 * 4);
    const size_t dur_bytes = (size_t)(total > 0 ? total : 1) * 8;
    const size_t done_bytes = (size_t)dg.max_words * R * 8;
    size_t off = 0;
    sc.off_bits = off; off = align_up(off + 5 * done_bytes, 256);
    sc.off_cp = off;   off = align_up(off + (size_t)dg.max_nodes * R * 8, 256);
    sc.off_acc = off;  off = align_up(off + (size_t)dg.n_acc * R * 8, 256);
    sc.off_ring = off; off = align_up(off + 2 * (size_t)dg.coll_stride * R * 4, 256);
    sc.off_dur = off;  off = align_up(off + dur_bytes * CS, 256);      // one copy per CTA of a cluster
    sc.off_inst = off; off = align_up(off + inst_bytes, 256);
    sc.off_inst_se = off; off = align_up(off + 16 * (size_t)(d->n_inst > 0 ? d->n_inst : 1) * CS, 256);
    // links: switch eg/in per rank; mesh 4 per position.  The table is the last piece of a
    // slot, sized at create from the largest rank id and grown per launch (fl_sweep_run knows
    // its points' mesh shapes) -- see grow_links.
    int64_t maxv = 0;
    for (int r = 0; r < R; r++) maxv = d->rank_value[r] > maxv ? d->rank_value[r] : maxv;
    bool neg = false;
    for (int r = 0; r < R; r++) neg |= d->rank_value[r] < 0;
    if (d->n_msg > 0 && (maxv >= ((int64_t)1 << 27) || neg))
        return fail(FL_ERR_CAPACITY, "rank ids of graphs with SEND/RECV must be in [0, 2^27) (link ids)");
    sc.link_cap = d->n_msg > 0 ? (int)std::max<int64_t>(2 * (int64_t)R, 8 * (maxv + 1)) : 0;
    sc.off_msg = off;                 // [n_msg] 64-byte message records | completion list | in-flight lists
    off = align_up(off + (size_t)d->n_msg * 64 + (size_t)d->n_msg * 4 + 2 * (size_t)dg.p2p_stride * R * 4 + 64, 256);
    sc.off_mlist_se = off;
    off = align_up(off + (d->n_msg > 0 ? 2 * (size_t)dg.p2p_stride * R * 8 : 0), 256);
    sc.off_ctr = off;  off = align_up(off + 64, 256);
    sc.off_links = off;
    sc.slot_bytes = align_up(off + (size_t)sc.link_cap * 24, 256);

    // shared memory: header | comm_end, stats, ring tails | [instances] | [durations] | [done bitmap]
    size_t sm = fl::sweep_shared_header_bytes();
    sc.sm_off_dyn = (unsigned)sm;
    const size_t B = (size_t)g->block;              // shared per-rank arrays have blockDim stride
    sm = align_up(sm + (size_t)fl::sweep_plane_lanes(g->block, CS) * fl::sweep_shared_bytes_per_rank(d->n_msg > 0),
                  16);   // per-rank fields (engine.cu F_*, Q_*, M_*)
    const size_t budget = (size_t)optin - 1024;   // the kernel's static shared memory (Ctx) comes off the top
    const size_t sbits = (size_t)dg.max_words * B * 8;   // a bitmap over this CTA's ranks
    sc.inst_in_smem = CS == 1 && sm + inst_bytes <= budget;   // clusters share instance state in HBM
    // (the durations, when they fit beside the instance table, come first: their offset is then the
    // end of the planes, a compile-time constant of each kernel variant -- engine.cu dur_off)
    sc.dur_in_smem = align_up(sm + (sc.inst_in_smem ? inst_bytes : 0), 16) + dur_bytes <= budget;
    if (sc.dur_in_smem) { sc.sm_off_dur = (unsigned)sm; sm = align_up(sm + dur_bytes, 16); }
    if (sc.inst_in_smem) { sc.sm_off_inst = (unsigned)sm; sm = align_up(sm + inst_bytes, 16); }
    dg.dur_sm_off = sc.dur_in_smem ? sc.sm_off_dur : 0;
    sc.done_in_smem = dg.needs_done && sm + sbits <= budget;
    if (sc.done_in_smem) { sc.sm_off_done = (unsigned)sm; sm = align_up(sm + sbits, 16); }
#ifdef FL_NO_TOUCH
    sc.touch_in_smem = false;       // first dependency recognised by its accumulator's epoch tag
#else
    sc.touch_in_smem = sm + sbits <= budget;
#endif
    if (sc.touch_in_smem) { sc.sm_off_touch = (unsigned)sm; sm = align_up(sm + sbits, 16); }
    // the accumulator slot table [n_acc][R] (single-CTA points: its words are per-rank columns
    // that only the rank's own thread touches, so plain shared-memory accesses replace the L2
    // reads on the critical chain of every "last" edge)
    const size_t acc_bytes = (size_t)dg.n_acc * R * 8;
#ifdef FL_NO_ACC_SMEM
    sc.acc_in_smem = false;
#else
    sc.acc_in_smem = CS == 1 && acc_bytes <= 64 * 1024 && sm + acc_bytes <= budget;   // (small tables only: occupancy)
#endif
    if (sc.acc_in_smem) { sc.sm_off_acc = (unsigned)sm; sm = align_up(sm + acc_bytes, 16); }
    // the link table [3][link_cap] of the message phase, which only the (lead) CTA runs; a
    // launch whose meshes need a larger table than reserved here uses the slot's copy in HBM
    g->links_sm_cap = 0;
    if (d->n_msg > 0 && sm + (size_t)sc.link_cap * 24 <= budget) {
        sc.sm_off_links = (unsigned)sm;
        sm = align_up(sm + (size_t)sc.link_cap * 24, 16);
        g->links_sm_cap = sc.link_cap;
    }
    if (sm > budget) {
        if (pass == 0 && CS < cs_hi) continue;
        if (pass == 0 && best_cs > 0) continue;
        return fail(FL_ERR_CAPACITY, "per-rank state exceeds shared memory");
    }
    g->smem = sm;
    {
        // the kernels' dynamic shared-memory limit is per function and device, shared by every
        // handle: only ever raise it (a handle created later with a smaller footprint must not
        // invalidate the launches of one created earlier)
        static std::mutex mu;
        static size_t smem_max[64] = {};
        std::lock_guard<std::mutex> lock(mu);
        if (device < 0 || device >= 64) return fail(FL_ERR_INVALID, "device ordinal out of range");
        if (sm > smem_max[device]) {
            CK(fl::sweep_set_smem(sm));
            smem_max[device] = sm;
        }
    }
    int occ = 0;
    if (fl::sweep_occupancy(g->block, g->smem, CS, &occ) != cudaSuccess) { cudaGetLastError(); occ = 0; }
    if (pass == 0) {
        const double score = (double)occ / g->block;
        if (occ >= 1 && score > best_score * 1.0001) { best_score = score; best_cs = CS; }
        continue;
    }
    if (occ < 1) return fail(FL_ERR_CAPACITY, "engine kernel cannot be resident with this shared-memory footprint");
    g->grid_cap = CS > 1 ? occ : sms * occ;           // concurrent design points (clusters or CTAs)
    return FL_OK;
    }   // CS
    if (best_cs < 0) return fail(FL_ERR_CAPACITY, "engine kernel cannot be resident with this shared-memory footprint");
    }   // pass
    return fail(FL_ERR_INVALID, "launch geometry");
}

// A launch whose mesh points need more links than the slot holds grows the table (the
// reference accepts any mesh at least as large as the ranks, topology.py:68-102).
void grow_links(fl_graph *g, int need) {
    if (g->dg.n_msg <= 0 || need <= g->sc.link_cap) return;
    g->sc.link_cap = need;
    g->sc.slot_bytes = align_up(g->sc.off_links + (size_t)need * 24, 256);
}

int ensure_scratch(fl_graph *g, int grid) {
    size_t need = g->sc.slot_bytes * (size_t)grid;
    if (need <= g->scratch_bytes) return FL_OK;
    if (g->scratch) cudaFree(g->scratch);
    g->scratch = nullptr;
    g->scratch_bytes = 0;
    CK(cudaMalloc(&g->scratch, need));
    g->scratch_bytes = need;
    g->sc.base = g->scratch;
    return FL_OK;
}

// defer / deferred: fl::launch_sweep's deferred second pass; retry_only: launch that pass
int launch(fl_graph *g, const fl_points *pts, fl_outputs *out, cudaStream_t stream, int *launches = nullptr,
           bool defer = false, bool *deferred = nullptr, bool retry_only = false) {
    if (launches) *launches = 0;
    if (pts->n_points <= 0) return FL_OK;
    int cs = pts->compute_streams;
    if (cs < 1 || cs > 8) return fail(FL_ERR_CAPACITY, "compute_streams must be 1..8 in this build");
    int grid = pts->n_points < g->grid_cap ? pts->n_points : g->grid_cap;   // design points in flight
    int rc = ensure_scratch(g, grid);
    if (rc) return rc;
    fl::DevPoints dp;
    dp.n = pts->n_points;
    dp.algo = pts->algo;
    dp.topo_kind = pts->topo_kind;
    dp.bw = pts->bw;
    dp.latency = pts->latency;
    dp.rows = pts->rows;
    dp.cols = pts->cols;
    dp.peak_flops = pts->peak_flops;
    dp.efficiency = pts->efficiency;
    dp.compute_streams = cs;
    dp.retry = retry_only ? 1 : 0;
    fl::DevScratch sc = g->sc;
    sc.links_in_smem = g->links_sm_cap > 0 && sc.link_cap <= g->links_sm_cap;
    fl::DevOut dout;
    dout.status = out->status;
    dout.rows = out->rows;
    dout.rank_stats = out->rank_stats;
    dout.ev_start = out->ev_start;
    dout.ev_end = out->ev_end;
    dout.link_busy = out->link_busy;
    dout.link_cap = out->link_cap;
    dout.trace = out->trace_len ? out->trace : nullptr;
    dout.trace_len = out->trace_len;
    dout.trace_cap = out->trace ? out->trace_cap : 0;
    int nl = 0;
    // kernel variants exist for 1, 2, 4 and 8 streams: a count in between runs on the next one
    // up with the extra slots never free (simulator.py:250-257 picks the lowest free stream)
    CK(fl::launch_sweep(cs <= 2 ? cs : cs <= 4 ? 4 : 512, grid * g->cluster, g->block, g->smem, stream, g->cluster, g->dg, dp, dout,
                        sc, &nl, defer, deferred));
    if (launches) *launches = nl;
    return FL_OK;
}

template <typename T>
int to_dev(const T *host, size_t n, T **dev, std::vector<void *> &tmp) {
    *dev = nullptr;
    if (!host) return FL_OK;
    void *p = nullptr;
    CK(cudaMalloc(&p, (n ? n : 1) * sizeof(T)));
    tmp.push_back(p);
    if (n) CK(cudaMemcpy(p, host, n * sizeof(T), cudaMemcpyHostToDevice));
    *dev = static_cast<T *>(p);
    return FL_OK;
}

void free_all(std::vector<void *> &v) {
    for (void *p : v) cudaFree(p);
    v.clear();
}

}  // namespace

extern "C" {

int fl_version(void) { return FL_ABI_VERSION; }

const char *fl_last_error(void) { return g_err.c_str(); }

int fl_device_count(int32_t *count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    *count = e == cudaSuccess ? n : 0;
    if (e != cudaSuccess) return fail(FL_ERR_CUDA, cudaGetErrorString(e));
    return FL_OK;
}

int fl_graph_create(const fl_graph_desc *desc, int32_t device, fl_graph **out) {
    *out = nullptr;
    fl_graph *g = new fl_graph();
    int rc = create(desc, device, g);
    if (rc) {
        fl_graph_destroy(g);
        return rc;
    }
    *out = g;
    return FL_OK;
}

int fl_graph_destroy(fl_graph *g) {
    if (!g) return FL_OK;
    cudaSetDevice(g->device);
    for (void *p : g->allocs) cudaFree(p);
    if (g->scratch) cudaFree(g->scratch);
    if (g->stage) cudaFree(g->stage);
    if (g->hstage) cudaFreeHost(g->hstage);
    if (g->stream) cudaStreamDestroy(g->stream);
    delete g;
    return FL_OK;
}

int32_t fl_graph_max_nodes(const fl_graph *g) { return g ? g->dg.max_nodes : 0; }

int fl_sweep_run_device(fl_graph *g, const fl_points *dev_points, fl_outputs *dev_out, void *stream,
                        int32_t *launches) {
    if (!g || !dev_points || !dev_out) return fail(FL_ERR_INVALID, "null argument");
    CK(cudaSetDevice(g->device));
    int nl = 0;
    int rc = launch(g, dev_points, dev_out, static_cast<cudaStream_t>(stream), &nl);
    if (launches) *launches = rc == FL_OK ? nl : 0;
    return rc;
}

int fl_sweep_run(fl_graph *g, const fl_points *hp, fl_outputs *ho) {
    if (!g || !hp || !ho) return fail(FL_ERR_INVALID, "null argument");
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != g->device) CK(cudaSetDevice(g->device));
    const size_t n = (size_t)hp->n_points;
    if (n == 0) return FL_OK;
    if (!g->stream) CK(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    if (g->dg.n_msg > 0 && hp->topo_kind && hp->rows && hp->cols) {
        int64_t need = 0;
        for (size_t i = 0; i < n; i++)
            if (hp->topo_kind[i] == FL_MESH2D && hp->rows[i] > 0 && hp->cols[i] > 0)
                need = std::max<int64_t>(need, 4 * (int64_t)hp->rows[i] * hp->cols[i]);
        if (need > (int64_t)1 << 28) return fail(FL_ERR_CAPACITY, "mesh too large for the link table");
        grow_links(g, (int)need);
    }
    cudaStream_t st = g->stream;
    const size_t R = (size_t)g->dg.R, MN = (size_t)g->dg.max_nodes;
    // One staging block, mirrored in pinned host memory: the packed inputs (one H2D copy),
    // then the per-point outputs (status, rows, trace lengths: one D2H copy), then the
    // optional bulk outputs, which are copied straight into the caller's buffers.
    struct Part { const void *src; size_t bytes; size_t off; };
    Part in[8] = {{hp->algo, n, 0}, {hp->topo_kind, n, 0}, {hp->bw, 8 * n, 0}, {hp->latency, 8 * n, 0},
                  {hp->rows, 4 * n, 0}, {hp->cols, 4 * n, 0},
                  {hp->peak_flops, hp->peak_flops ? 8 * n : 0, 0}, {hp->efficiency, hp->efficiency ? 8 * n : 0, 0}};
    size_t off = 0;
    for (auto &p : in) { p.off = off; off = align_up(off + p.bytes, 16); }
    const size_t in_bytes = off;
    off = align_up(off, 256);
    const size_t o_status = off; off = align_up(off + 4 * n, 16);
    const size_t o_tl = off; off = align_up(off + (ho->trace_len ? 4 * n : 0), 16);
    const size_t o_rows = off; off = align_up(off + 48 * n, 256);
    const size_t small_end = off;                  // [o_status, small_end): copied back in one piece
    const size_t o_rs = off; off = align_up(off + (ho->rank_stats ? 40 * n * R : 0), 256);
    const size_t o_es = off; off = align_up(off + (ho->ev_start ? 8 * n * R * MN : 0), 256);
    const size_t o_ee = off; off = align_up(off + (ho->ev_start ? 8 * n * R * MN : 0), 256);
    const size_t LC = ho->link_busy ? (size_t)(ho->link_cap > 0 ? ho->link_cap : 0) : 0;
    const size_t o_lb = off; off = align_up(off + 8 * n * LC, 256);
    const size_t TC = ho->trace_len ? (size_t)(ho->trace && ho->trace_cap > 0 ? ho->trace_cap : 0) : 0;
    const size_t o_tr = off; off = align_up(off + 8 * n * TC, 256);
    if (off > g->stage_bytes) {
        if (g->stage) cudaFree(g->stage);
        g->stage = nullptr;
        g->stage_bytes = 0;
        CK(cudaMalloc(&g->stage, off));
        g->stage_bytes = off;
    }
    if (small_end > g->hstage_bytes) {
        if (g->hstage) cudaFreeHost(g->hstage);
        g->hstage = nullptr;
        g->hstage_bytes = 0;
        CK(cudaHostAlloc(&g->hstage, small_end, cudaHostAllocMapped));
        g->hstage_bytes = small_end;
        void *dh = nullptr;
        CK(cudaHostGetDevicePointer(&dh, g->hstage, 0));
        g->hstage_dev = static_cast<unsigned char *>(dh);
    }
    unsigned char *S = g->stage, *H = g->hstage;
    for (auto &p : in)
        if (p.bytes) memcpy(H + p.off, p.src, p.bytes);
    // With at most one design point per CTA, the kernel reads each point's parameters once and
    // writes its row once, so it does so over the bus from the mapped staging block itself:
    // no copy engine round trips for a few KB (the bulk outputs below still use copies).
    const bool zc = n <= (size_t)g->grid_cap;
    unsigned char *small = S;                      // where the inputs and per-point outputs live
    if (zc) {
        small = g->hstage_dev;
    } else {
        CK(cudaMemcpyAsync(S, H, in_bytes, cudaMemcpyHostToDevice, st));
    }
    fl_points dp = *hp;
    dp.algo = small + in[0].off;
    dp.topo_kind = small + in[1].off;
    dp.bw = reinterpret_cast<const double *>(small + in[2].off);
    dp.latency = reinterpret_cast<const int64_t *>(small + in[3].off);
    dp.rows = reinterpret_cast<const int32_t *>(small + in[4].off);
    dp.cols = reinterpret_cast<const int32_t *>(small + in[5].off);
    dp.peak_flops = hp->peak_flops ? reinterpret_cast<const double *>(small + in[6].off) : nullptr;
    dp.efficiency = hp->efficiency ? reinterpret_cast<const double *>(small + in[7].off) : nullptr;
    fl_outputs dout{};
    dout.status = reinterpret_cast<int32_t *>(small + o_status);
    dout.rows = reinterpret_cast<int64_t *>(small + o_rows);
    dout.rank_stats = ho->rank_stats ? reinterpret_cast<int64_t *>(S + o_rs) : nullptr;
    dout.ev_start = ho->ev_start ? reinterpret_cast<int64_t *>(S + o_es) : nullptr;
    dout.ev_end = ho->ev_start ? reinterpret_cast<int64_t *>(S + o_ee) : nullptr;
    dout.link_busy = LC ? reinterpret_cast<int64_t *>(S + o_lb) : nullptr;
    dout.link_cap = (int32_t)LC;
    dout.trace = TC ? reinterpret_cast<int64_t *>(S + o_tr) : nullptr;
    dout.trace_len = ho->trace_len ? reinterpret_cast<int32_t *>(small + o_tl) : nullptr;
    dout.trace_cap = (int32_t)TC;
    // The statuses come back to the host anyway, so the lean variant's second pass (the points
    // it left as FL_RETRY: zero-length nodes, engine.cu "Lean variants") is launched only when
    // one of them says so -- for most sweeps never, saving a launch and a kernel on the call.
    bool deferred = false;
    int rc = launch(g, &dp, &dout, st, nullptr, true, &deferred);
    if (rc) return rc;
    auto copy_back = [&]() -> int {
        if (!zc) CK(cudaMemcpyAsync(H + o_status, S + o_status, small_end - o_status, cudaMemcpyDeviceToHost, st));
        if (ho->rank_stats) CK(cudaMemcpyAsync(ho->rank_stats, dout.rank_stats, 40 * n * R, cudaMemcpyDeviceToHost, st));
        if (LC) CK(cudaMemcpyAsync(ho->link_busy, dout.link_busy, 8 * n * LC, cudaMemcpyDeviceToHost, st));
        if (TC) CK(cudaMemcpyAsync(ho->trace, dout.trace, 8 * n * TC, cudaMemcpyDeviceToHost, st));
        if (ho->ev_start) {
            CK(cudaMemcpyAsync(ho->ev_start, dout.ev_start, 8 * n * R * MN, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(ho->ev_end, dout.ev_end, 8 * n * R * MN, cudaMemcpyDeviceToHost, st));
        }
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return fail(FL_ERR_CUDA, std::string("engine kernel: ") + cudaGetErrorString(e));
        return FL_OK;
    };
    if ((rc = copy_back())) return rc;
    if (deferred) {
        const int32_t *hs = reinterpret_cast<const int32_t *>(H + o_status);
        bool any = false;
        for (size_t i = 0; i < n && !any; i++) any = hs[i] == fl::FL_RETRY;
        if (any) {
            if ((rc = launch(g, &dp, &dout, st, nullptr, false, nullptr, true))) return rc;
            if ((rc = copy_back())) return rc;
        }
    }
    memcpy(ho->status, H + o_status, 4 * n);
    memcpy(ho->rows, H + o_rows, 48 * n);
    if (ho->trace_len) memcpy(ho->trace_len, H + o_tl, 4 * n);
    return FL_OK;
}

static int critical_path_impl(fl_graph *g, const fl_points *hp, int32_t nv, const int32_t *order,
                              const int32_t *vkind, const int32_t *va, const int32_t *vb, const int32_t *vsend,
                              const int32_t *vmsg, const int32_t *pred_off, const int32_t *pred_idx,
                              int64_t *out_cp, int32_t *out_status, int64_t *out_vals) {
    if (!g || !hp || nv < 0) return fail(FL_ERR_INVALID, "bad argument");
    CK(cudaSetDevice(g->device));
    const size_t n = (size_t)hp->n_points;
    if (n == 0) return FL_OK;
    std::vector<void *> tmp;
    uint8_t *algo, *topo;
    double *bw, *peak = nullptr, *eff = nullptr;
    int64_t *lat, *vals, *dout;
    int32_t *rows, *cols, *dst, *dorder, *dk, *da, *db, *ds, *dm, *dpo, *dpi;
    int rc;
    const size_t V = (size_t)(nv > 0 ? nv : 1), E = (size_t)(pred_off ? pred_off[nv] : 0);
    if ((rc = to_dev(hp->algo, n, &algo, tmp)) || (rc = to_dev(hp->topo_kind, n, &topo, tmp)) ||
        (rc = to_dev(hp->bw, n, &bw, tmp)) || (rc = to_dev(hp->latency, n, &lat, tmp)) ||
        (rc = to_dev(hp->rows, n, &rows, tmp)) || (rc = to_dev(hp->cols, n, &cols, tmp)) ||
        (rc = to_dev(hp->peak_flops, n, &peak, tmp)) || (rc = to_dev(hp->efficiency, n, &eff, tmp)) ||
        (rc = to_dev(order, V, &dorder, tmp)) || (rc = to_dev(vkind, V, &dk, tmp)) || (rc = to_dev(va, V, &da, tmp)) ||
        (rc = to_dev(vb, V, &db, tmp)) || (rc = to_dev(vsend, V, &ds, tmp)) || (rc = to_dev(vmsg, V, &dm, tmp)) ||
        (rc = to_dev(pred_off, V + 1, &dpo, tmp)) || (rc = to_dev(pred_idx, E ? E : 1, &dpi, tmp)) ||
        (rc = to_dev(out_cp, n, &dout, tmp)) || (rc = to_dev(out_status, n, &dst, tmp))) {
        free_all(tmp);
        return rc;
    }
    void *pv = nullptr;
    if (cudaMalloc(&pv, n * V * 8 * (out_vals ? 2 : 1)) != cudaSuccess) { free_all(tmp); return fail(FL_ERR_CUDA, "cp scratch"); }
    tmp.push_back(pv);
    vals = static_cast<int64_t *>(pv);
    int64_t *starts = out_vals ? vals + n * V : nullptr;
    fl::DevPoints dp;
    dp.n = (int)n; dp.algo = algo; dp.topo_kind = topo; dp.bw = bw; dp.latency = lat; dp.rows = rows;
    dp.cols = cols; dp.peak_flops = peak; dp.efficiency = eff; dp.compute_streams = 1;
    cudaError_t e = fl::launch_cp(g->dg, dp, nv, dorder, dk, da, db, ds, dm, dpo, dpi, vals, starts, dout, dst);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(out_cp, dout, n * 8, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(out_status, dst, n * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && out_vals) e = cudaMemcpy(out_vals, vals, 2 * n * V * 8, cudaMemcpyDeviceToHost);
    free_all(tmp);
    if (e != cudaSuccess) return fail(FL_ERR_CUDA, cudaGetErrorString(e));
    return FL_OK;
}

int fl_critical_path(fl_graph *g, const fl_points *hp, int32_t nv, const int32_t *order, const int32_t *vkind,
                     const int32_t *va, const int32_t *vb, const int32_t *vsend, const int32_t *vmsg,
                     const int32_t *pred_off, const int32_t *pred_idx, int64_t *out_cp, int32_t *out_status) {
    return critical_path_impl(g, hp, nv, order, vkind, va, vb, vsend, vmsg, pred_off, pred_idx, out_cp, out_status,
                              nullptr);
}

int fl_critical_path_values(fl_graph *g, const fl_points *hp, int32_t nv, const int32_t *order,
                            const int32_t *vkind, const int32_t *va, const int32_t *vb, const int32_t *vsend,
                            const int32_t *vmsg, const int32_t *pred_off, const int32_t *pred_idx,
                            int64_t *out_cp, int32_t *out_status, int64_t *out_vals) {
    if (!out_vals) return fail(FL_ERR_INVALID, "out_vals is required");
    return critical_path_impl(g, hp, nv, order, vkind, va, vb, vsend, vmsg, pred_off, pred_idx, out_cp, out_status,
                              out_vals);
}

int fl_cost_only(int32_t n, const uint8_t *kind, const int64_t *size_bytes, const int64_t *group_n,
                 const uint8_t *algo, const double *alpha, const double *beta, const int32_t *rows,
                 const int32_t *cols, int64_t *out_ns, int32_t *out_status, int32_t m,
                 const int64_t *flops, const double *peak, const double *eff, int64_t *out_comp_ns) {
    std::vector<void *> tmp;
    uint8_t *dk = nullptr, *da = nullptr;
    int64_t *ds = nullptr, *dn = nullptr, *dout = nullptr, *dfl = nullptr, *dcomp = nullptr;
    double *dal = nullptr, *dbe = nullptr, *dpk = nullptr, *def = nullptr;
    int32_t *dr = nullptr, *dc = nullptr, *dst = nullptr;
    int rc;
    const size_t N = n > 0 ? n : 0, M = m > 0 ? m : 0;
    if ((rc = to_dev(kind, N, &dk, tmp)) || (rc = to_dev(size_bytes, N, &ds, tmp)) ||
        (rc = to_dev(group_n, N, &dn, tmp)) || (rc = to_dev(algo, N, &da, tmp)) ||
        (rc = to_dev(alpha, N, &dal, tmp)) || (rc = to_dev(beta, N, &dbe, tmp)) ||
        (rc = to_dev(rows, N, &dr, tmp)) || (rc = to_dev(cols, N, &dc, tmp)) ||
        (rc = to_dev(flops, M, &dfl, tmp)) || (rc = to_dev(peak, M, &dpk, tmp)) ||
        (rc = to_dev(eff, M, &def, tmp)) || (rc = to_dev(out_ns, N, &dout, tmp)) ||
        (rc = to_dev(out_status, N, &dst, tmp)) || (rc = to_dev(out_comp_ns, M, &dcomp, tmp))) {
        free_all(tmp);
        return rc;
    }
    int total = (int)(N > M ? N : M);
    if (total > 0) {
        cudaError_t e = fl::launch_cost_only((int)N, dk, ds, dn, da, dal, dbe, dr, dc, dout, dst, (int)M, dfl,
                                             dpk, def, dcomp);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            free_all(tmp);
            return fail(FL_ERR_CUDA, cudaGetErrorString(e));
        }
        if (N && e == cudaSuccess) e = cudaMemcpy(out_ns, dout, N * 8, cudaMemcpyDeviceToHost);
        if (N && e == cudaSuccess) e = cudaMemcpy(out_status, dst, N * 4, cudaMemcpyDeviceToHost);
        if (M && e == cudaSuccess) e = cudaMemcpy(out_comp_ns, dcomp, M * 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) {
            free_all(tmp);
            return fail(FL_ERR_CUDA, cudaGetErrorString(e));
        }
    }
    free_all(tmp);
    return FL_OK;
}

int fl_topo_order(fl_graph *g, int32_t *out_order, int32_t *out_level) {
    if (!g || !out_order || !out_level) return fail(FL_ERR_INVALID, "null argument");
    CK(cudaSetDevice(g->device));
    const size_t n = (size_t)(g->dg.total_nodes > 0 ? g->dg.total_nodes : 1);
    int32_t *dw = nullptr;
    CK(cudaMalloc(&dw, 3 * n * sizeof(int32_t)));
    cudaError_t e = fl::launch_topo(g->dg, dw, dw + n, dw + 2 * n);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(out_order, dw + n, (size_t)g->dg.total_nodes * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(out_level, dw + 2 * n, (size_t)g->dg.total_nodes * 4, cudaMemcpyDeviceToHost);
    cudaFree(dw);
    if (e != cudaSuccess) return fail(FL_ERR_CUDA, cudaGetErrorString(e));
    return FL_OK;
}

}  // extern "C"
