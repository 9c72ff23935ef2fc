// engine.cu -- batched design-point evaluation of per-rank workload graphs on B200.
//
// One CTA evaluates one design point at a time (persistent grid-stride loop
// over points); thread r of the CTA owns rank r.  Inside a point the CTA
// replays the reference's discrete-event list scheduler exactly
// (pkg/src/trainsim/simulator.py:203-367) as a sequence of global time steps:
//
//   * every step, a block-wide min over the ranks' next event times gives the
//     step time t and the lowest rank r_min holding an event at t;
//   * each rank then pops its own events at t in node-id order, releasing
//     dependents and re-running its start phase after every pop -- the
//     reference's per-pop loop restricted to one rank, which is exact because
//     a rank's host/compute phases only read that rank's state;
//   * the reference additionally runs every rank's start phase after *other*
//     ranks' pops.  That phase is idempotent, and it can only change a rank's
//     schedule when the rank has an event of its own at t and a lower rank
//     popped first (the cross-rank tie race).  So
//     rank r runs one extra start phase before its pops iff r > r_min;
//   * collectives that complete during the step are reserved afterwards, in
//     the reference's order (completing pop, then lead node id,
//     simulator.py:298-309), by a block-wide max over member comm streams.
//     A reservation only pushes events at e > t unless its duration is 0;
//     design points with a zero-duration collective run the same machinery
//     one pop per block iteration instead ("serial mode"), which is the
//     reference loop verbatim.
//
// The same pass computes, per (rank, node), the contention-free longest-path
// finish time (critical_path, simulator.py:400-460): when a node becomes
// ready all its predecessors -- for a collective, all members' predecessors --
// have completed in the simulation, so its critical-path start is final.
// Per-rank statistics (compute/comm busy, exposed comm, peak memory,
// simulator.py:342-393) are accumulated on-line from the step timeline.
//
// Numerics: every fp64 operation of the cost model uses an explicit
// round-to-nearest intrinsic and the file is compiled with -fmad=false, so
// each expression is the reference's Python evaluation order with no FMA
// contraction.  Times are int64 ns.

#include <cuda_runtime.h>
#include <stdint.h>

#include "flint_b200.h"
#include "engine_internal.h"

namespace fl {

// ------------------------------------------------------------------ costs

__device__ __forceinline__ int64_t rhu(double x) {          // traceio.py:68-70
    return (int64_t)floor(__dadd_rn(x, 0.5));
}

__device__ __forceinline__ double ring_rs(int64_t n, double s, double a, double b) {  // collectives.py:243-244
    double t1 = __dmul_rn((double)(n - 1), a);
    double t2 = __ddiv_rn((double)(n - 1), (double)n);
    t2 = __dmul_rn(t2, s);
    t2 = __dmul_rn(t2, b);
    return __dadd_rn(t1, t2);
}

__device__ __forceinline__ double ring_ar(int64_t n, double s, double a, double b) {  // collectives.py:247-248
    double t1 = __dmul_rn((double)(2 * (n - 1)), a);
    double t2 = __ddiv_rn((double)(2 * (n - 1)), (double)n);
    t2 = __dmul_rn(t2, s);
    t2 = __dmul_rn(t2, b);
    return __dadd_rn(t1, t2);
}

// collectives.py:251-293.  Returns -1 for UnsupportedAlgoTopologyError.
__device__ int64_t analytical_time(int kind, int64_t size, int64_t n, int algo, double a,
                                   double b, int64_t rows, int64_t cols) {
    if (n <= 1) return 0;
    double s = (double)size, t;
    if (algo == FL_RING) {
        t = kind == FL_ALL_REDUCE ? ring_ar(n, s, a, b) : ring_rs(n, s, a, b);
    } else if (algo == FL_TREE) {
        if (kind != FL_ALL_REDUCE) return -1;
        int64_t lg = 64 - __clzll((unsigned long long)(n - 1));   // ceil(log2 n), n >= 2
        t = __dadd_rn(__dmul_rn((double)(2 * lg), a), __dmul_rn(__dmul_rn(2.0, s), b));
    } else {
        if (rows <= 0 || cols <= 0 || rows * cols != n) return -1;
        double sc = __ddiv_rn(s, (double)cols), sr = __ddiv_rn(s, (double)rows);
        if (kind == FL_ALL_REDUCE)
            t = __dadd_rn(__dadd_rn(ring_rs(cols, s, a, b), ring_ar(rows, sc, a, b)), ring_rs(cols, s, a, b));
        else if (kind == FL_ALL_GATHER)
            t = __dadd_rn(ring_rs(cols, sr, a, b), ring_rs(rows, s, a, b));
        else
            t = __dadd_rn(ring_rs(cols, s, a, b), ring_rs(rows, sc, a, b));
    }
    return rhu(t);
}

__device__ __forceinline__ int64_t flops_to_ns(int64_t flops, double peak, double eff) {  // traceio.py:184
    return rhu(__dmul_rn(__ddiv_rn((double)flops, __dmul_rn(peak, eff)), 1e9));
}

// simulator.py:109-114: ALL_GATHER is timed on the gathered size.
__device__ __forceinline__ int64_t coll_time(const DevGraph &g, int i, int algo, int topo, double bw,
                                             int64_t lat, int32_t rows, int32_t cols) {
    int64_t n = g.inst_n[i];
    int kind = g.inst_kind[i];
    int64_t size = kind == FL_ALL_GATHER ? g.inst_bytes[i] * n : g.inst_bytes[i];
    bool mesh = topo == FL_MESH2D;
    return analytical_time(kind, size, n, algo, (double)lat, __ddiv_rn(1e9, bw),
                           mesh ? rows : 0, mesh ? cols : 0);
}

__global__ void cost_only_kernel(int n, const uint8_t *kind, const int64_t *size, const int64_t *gn,
                                 const uint8_t *algo, const double *alpha, const double *beta,
                                 const int32_t *rows, const int32_t *cols, int64_t *out,
                                 int32_t *status, int m, const int64_t *flops, const double *peak,
                                 const double *eff, int64_t *out_comp) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        int64_t v = analytical_time(kind[i], size[i], gn[i], algo[i], alpha[i], beta[i], rows[i], cols[i]);
        out[i] = v < 0 ? 0 : v;
        status[i] = v < 0 ? FL_ERR_UNSUPPORTED_ALGO : FL_OK;
    }
    if (i < m) out_comp[i] = flops_to_ns(flops[i], peak[i], eff[i]);
}

// ------------------------------------------------------- block primitives

constexpr unsigned FULL = 0xffffffffu;
constexpr int64_t TINF = INT64_MAX;
constexpr uint64_t KINF = ~0ull;

struct Shared {
    uint64_t red[2][32];
    int64_t redi[2][32];
    int parity;
    int ncomp;
    int flag;
};

__device__ __forceinline__ uint64_t block_min_u64(uint64_t v, Shared &sh, int &par) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) { uint64_t w = __shfl_xor_sync(FULL, v, o); v = w < v ? w : v; }
    uint64_t *b = sh.red[par];
    par ^= 1;
    if (lane == 0) b[warp] = v;
    __syncthreads();
    v = lane < nw ? b[lane] : KINF;
#pragma unroll
    for (int o = 16; o; o >>= 1) { uint64_t w = __shfl_xor_sync(FULL, v, o); v = w < v ? w : v; }
    return v;
}

__device__ __forceinline__ int64_t block_max_i64(int64_t v, Shared &sh, int &par) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) { int64_t w = __shfl_xor_sync(FULL, v, o); v = w > v ? w : v; }
    int64_t *b = sh.redi[par];
    par ^= 1;
    if (lane == 0) b[warp] = v;
    __syncthreads();
    v = lane < nw ? b[lane] : INT64_MIN;
#pragma unroll
    for (int o = 16; o; o >>= 1) { int64_t w = __shfl_xor_sync(FULL, v, o); v = w > v ? w : v; }
    return v;
}

// ---------------------------------------------------------- rank state

// Bitmaps are stored word-major, rank-minor ([word][rank]) so the 32 ranks of
// a warp that step in lockstep touch one contiguous 256-byte segment.
struct Bits {
    uint64_t *p;
    int R;
    __device__ __forceinline__ uint64_t &w(int word, int r) const { return p[(size_t)word * R + r]; }
};

template <int K>
struct Rank {
    int r, nb, N, tb;            // rank, global node base, node count, global tensor base
    uint64_t due_s, rc_s, rh_s;  // non-empty-word summaries of the due / ready-comp / ready-host sets
    int64_t host_slot, host_e;
    int host_n;
    int64_t slot[K], occ_e[K];
    int occ_n[K];
    int ring_head, ring_acur;
    int64_t comp_busy, comm_busy, overlap, finish, cur, peak, alloc_t, free_t, cpmax;
    int done_cnt, pop_seq;
};

struct Cfg {                      // per design point, uniform over the CTA
    int64_t *dur;                 // per node duration for this point
    int serial;
    uint64_t step;
    int init;
};

__device__ __forceinline__ void bm_insert(const Bits &b, uint64_t &sum, int r, int idx) {
    int w = idx >> 6;
    b.w(w, r) |= 1ull << (idx & 63);
    sum |= 1ull << w;
}

__device__ __forceinline__ int bm_pop(const Bits &b, uint64_t &sum, int r) {
    int w = __ffsll((long long)sum) - 1;
    uint64_t word = b.w(w, r);
    int bit = __ffsll((long long)word) - 1;
    word &= word - 1;
    b.w(w, r) = word;
    if (!word) sum &= sum - 1;
    return (w << 6) | bit;
}

__device__ __forceinline__ int bm_peek(const Bits &b, uint64_t sum, int r) {
    int w = __ffsll((long long)sum) - 1;
    return (w << 6) | (__ffsll((long long)b.w(w, r)) - 1);
}

__device__ __forceinline__ bool bm_test(const Bits &b, int r, int idx) {
    return (b.w(idx >> 6, r) >> (idx & 63)) & 1ull;
}

struct Ctx {
    DevGraph g;
    DevPoints p;
    DevOut o;
    Bits done, rdyc, rdyh, due;
    int64_t *cp;                  // [max_nodes][R] critical-path finish per (node, rank)
    int32_t *ring_inst, *ring_node;  // [coll_stride][R] per-rank comm FIFO
    int64_t *dur;                 // [total_nodes]
    int64_t *inst_dur, *inst_s, *inst_e, *inst_cpmax;
    unsigned long long *inst_ckey;
    int32_t *inst_wait, *complist;
    int64_t *comm_end;            // shared: [R]
    int32_t *ring_tail;           // shared: [R]
    int *ncomp;                   // shared: instances completed in this step
};

template <int K>
__device__ __forceinline__ void record(const Ctx &c, int cfg, const Rank<K> &s, int x, int64_t st, int64_t en) {
    if (c.o.ev_start) {
        size_t at = ((size_t)cfg * c.g.R + s.r) * c.g.max_nodes + x;
        c.o.ev_start[at] = st;
        c.o.ev_end[at] = en;
    }
}

// One rank's start phase at time t (simulator.py:282-297 for this rank).
template <int K>
__device__ void start_phase(const Ctx &c, const Cfg &f, Rank<K> &s, int64_t t, int cfg) {
    const int r = s.r;
    while (s.rh_s && s.host_slot <= t) {
        int h = bm_pop(c.rdyh, s.rh_s, r);
        int64_t e = t + f.dur[s.nb + h];
        s.host_slot = e;
        s.alloc_t += c.g.node_alloc[s.nb + h];
        record(c, cfg, s, h, t, e);
        if (e == t) bm_insert(c.due, s.due_s, r, h);
        else { s.host_e = e; s.host_n = h; }
    }
    while (s.rc_s) {
        int k = 0;
#pragma unroll
        for (int q = 1; q < K; q++) if (s.slot[q] < s.slot[k]) k = q;
        if (s.slot[k] > t) break;
        int x = bm_pop(c.rdyc, s.rc_s, r);
        int64_t e = t + f.dur[s.nb + x];
        s.alloc_t += c.g.node_alloc[s.nb + x];
        record(c, cfg, s, x, t, e);
#pragma unroll
        for (int q = 0; q < K; q++) {
            if (q == k) {
                s.slot[q] = e;
                if (e == t) bm_insert(c.due, s.due_s, r, x);
                else { s.occ_e[q] = e; s.occ_n[q] = x; }
            }
        }
    }
}

// A node whose every dependency completed (simulator.py:247-268).
template <int K>
__device__ void dispatch(const Ctx &c, const Cfg &f, Rank<K> &s, int d, int seq) {
    const int r = s.r, R = c.g.R;
    const int gd = s.nb + d;
    int64_t cps = 0;
    for (int q = c.g.pred_off[gd]; q < c.g.pred_off[gd + 1]; q++) {
        int64_t v = c.cp[(size_t)c.g.pred_idx[q] * R + r];
        cps = v > cps ? v : cps;
    }
    int kind = c.g.node_kind[gd];
    if (kind == FL_COLL) {
        int i = c.g.rank_coll_inst[(size_t)r * c.g.coll_stride + c.g.node_coll_ord[gd]];
        atomicMax((unsigned long long *)&c.inst_cpmax[i], (unsigned long long)cps);
        if (!f.init) {
            unsigned long long key = (f.step << 39) | ((unsigned long long)r << 25) |
                                     ((unsigned long long)s.pop_seq << 12) | (unsigned long long)seq;
            atomicMax(&c.inst_ckey[i], key);
        }
        if (atomicSub(&c.inst_wait[i], 1) == 1) c.complist[atomicAdd(c.ncomp, 1)] = i;
        return;
    }
    int64_t fin = cps + f.dur[gd];
    c.cp[(size_t)d * R + r] = fin;
    s.cpmax = fin > s.cpmax ? fin : s.cpmax;
    if (kind == FL_COMP) bm_insert(c.rdyc, s.rc_s, r, d);
    else bm_insert(c.rdyh, s.rh_s, r, d);
}

// Pop one completion event (simulator.py:335-340) plus its tensor frees.
template <int K>
__device__ void pop_event(const Ctx &c, const Cfg &f, Rank<K> &s, int x, int64_t t) {
    const int r = s.r;
    const int gx = s.nb + x;
    c.done.w(x >> 6, r) |= 1ull << (x & 63);
    s.done_cnt++;
    s.pop_seq++;
    s.finish = t;
    // a tensor is freed when its last consumer completes (simulator.py:384-388)
    for (int q = c.g.free_off[gx]; q < c.g.free_off[gx + 1]; q++) {
        int tt = s.tb + c.g.free_tens[q];
        bool all = true;
        for (int u = c.g.tens_cons_off[tt]; u < c.g.tens_cons_off[tt + 1] && all; u++)
            all = bm_test(c.done, r, c.g.tens_cons[u]);
        if (all) s.free_t += c.g.tens_bytes[tt];
    }
    int seq = 0;
    for (int q = c.g.succ_off[gx]; q < c.g.succ_off[gx + 1]; q++, seq++) {
        int d = c.g.succ_idx[q];
        int gd = s.nb + d;
        if (c.g.node_flags[gd] & 1) continue;
        bool ready = true;
        for (int u = c.g.pred_off[gd]; u < c.g.pred_off[gd + 1] && ready; u++)
            ready = bm_test(c.done, r, c.g.pred_idx[u]);
        if (ready) dispatch(c, f, s, d, seq);
    }
}

template <int K>
__device__ __forceinline__ int64_t next_time(const Ctx &c, const Rank<K> &s, int64_t tcur) {
    if (s.due_s) return tcur;
    int64_t nt = TINF;
    if (s.host_n >= 0) nt = s.host_e;
#pragma unroll
    for (int q = 0; q < K; q++) if (s.occ_n[q] >= 0 && s.occ_e[q] < nt) nt = s.occ_e[q];
    if (s.ring_head < c.ring_tail[s.r]) {
        int64_t e = c.inst_e[c.ring_inst[(size_t)s.ring_head * c.g.R + s.r]];
        nt = e < nt ? e : nt;
    }
    return nt;
}

// Events already scheduled for exactly t join the due set.
template <int K>
__device__ __forceinline__ void gather_due(const Ctx &c, Rank<K> &s, int64_t t) {
    const int r = s.r;
    if (s.host_n >= 0 && s.host_e == t) { bm_insert(c.due, s.due_s, r, s.host_n); s.host_n = -1; }
#pragma unroll
    for (int q = 0; q < K; q++)
        if (s.occ_n[q] >= 0 && s.occ_e[q] == t) { bm_insert(c.due, s.due_s, r, s.occ_n[q]); s.occ_n[q] = -1; }
    const int tail = c.ring_tail[r];
    while (s.ring_head < tail) {
        size_t at = (size_t)s.ring_head * c.g.R + r;
        if (c.inst_e[c.ring_inst[at]] != t) break;
        bm_insert(c.due, s.due_s, r, c.ring_node[at]);
        s.ring_head++;
    }
}

// Close the interval [tcur, tnew): busy/overlap integration and the
// alloc-before-free memory high-water mark at tcur (simulator.py:381-393).
template <int K>
__device__ __forceinline__ void advance(const Ctx &c, Rank<K> &s, int64_t tcur, int64_t tnew) {
    const int r = s.r;
    const int tail = c.ring_tail[r];
    while (s.ring_acur < tail) {   // collectives that started by tcur allocate their outputs then
        size_t at = (size_t)s.ring_acur * c.g.R + r;
        if (c.inst_s[c.ring_inst[at]] > tcur) break;
        s.alloc_t += c.g.node_alloc[s.nb + c.ring_node[at]];
        s.ring_acur++;
    }
    s.cur += s.alloc_t;
    s.peak = s.cur > s.peak ? s.cur : s.peak;
    s.cur -= s.free_t;
    s.alloc_t = s.free_t = 0;
    if (tnew == TINF) return;
    int64_t dt = tnew - tcur;
    bool comp_on = false;
#pragma unroll
    for (int q = 0; q < K; q++) comp_on |= s.occ_n[q] >= 0;
    bool comm_on = false;
    if (s.ring_head < tail) comm_on = c.inst_s[c.ring_inst[(size_t)s.ring_head * c.g.R + r]] <= tcur;
    if (comp_on) s.comp_busy += dt;
    if (comm_on) s.comm_busy += dt;
    if (comp_on && comm_on) s.overlap += dt;
}

__device__ __forceinline__ bool comp_before(const Ctx &c, int a, int b, bool init) {
    // reservation order of instances that completed in the same step
    int64_t la = c.g.inst_lead_id[a], lb = c.g.inst_lead_id[b];
    if (init) {
        if (la != lb) return la < lb;
        return c.g.inst_init_key[a] < c.g.inst_init_key[b];
    }
    unsigned long long ka = c.inst_ckey[a] >> 12, kb = c.inst_ckey[b] >> 12;
    if (ka != kb) return ka < kb;
    if (la != lb) return la < lb;
    return (c.inst_ckey[a] & 0xfff) < (c.inst_ckey[b] & 0xfff);
}

// Reserve the comm streams for every instance completed in this step
// (simulator.py:298-309); block-wide.  Returns max critical-path value seen.
__device__ int64_t reserve(const Ctx &c, Shared &sh, int &par, int64_t t, bool init, int cfg) {
    __syncthreads();
    const int nc = sh.ncomp;
    int64_t cpm = 0;
    if (nc == 0) return 0;
    if (threadIdx.x == 0) {
        for (int a = 1; a < nc; a++) {
            int x = c.complist[a], b = a - 1;
            while (b >= 0 && comp_before(c, x, c.complist[b], init)) { c.complist[b + 1] = c.complist[b]; b--; }
            c.complist[b + 1] = x;
        }
    }
    __syncthreads();
    for (int q = 0; q < nc; q++) {
        const int i = c.complist[q];
        const int64_t m0 = c.g.inst_mem_off[i], nm = c.g.inst_mem_off[i + 1] - m0;
        int64_t local = t;
        for (int64_t j = threadIdx.x; j < nm; j += blockDim.x) {
            int64_t ce = c.comm_end[c.g.inst_mem_rank[m0 + j]];
            local = ce > local ? ce : local;
        }
        const int64_t s = block_max_i64(local, sh, par);
        const int64_t e = s + c.inst_dur[i];
        const int64_t cpv = c.inst_cpmax[i] + c.inst_dur[i];
        cpm = cpv > cpm ? cpv : cpm;
        for (int64_t j = threadIdx.x; j < nm; j += blockDim.x) {
            int m = c.g.inst_mem_rank[m0 + j], node = c.g.inst_mem_node[m0 + j];
            c.comm_end[m] = e;
            int slot = c.ring_tail[m]++;
            c.ring_inst[(size_t)slot * c.g.R + m] = i;
            c.ring_node[(size_t)slot * c.g.R + m] = node;
            c.cp[(size_t)node * c.g.R + m] = cpv;
            if (c.o.ev_start) {
                size_t at = ((size_t)cfg * c.g.R + m) * c.g.max_nodes + node;
                c.o.ev_start[at] = s;
                c.o.ev_end[at] = e;
            }
        }
        if (threadIdx.x == 0) { c.inst_s[i] = s; c.inst_e[i] = e; }
        __syncthreads();
    }
    if (threadIdx.x == 0) sh.ncomp = 0;
    __syncthreads();
    return cpm;
}

template <int K>
__global__ void __launch_bounds__(1024, 1) sweep_kernel(DevGraph g, DevPoints p, DevOut o, DevScratch sc) {
    extern __shared__ __align__(16) unsigned char smem[];
    Shared &sh = *reinterpret_cast<Shared *>(smem);
    int64_t *comm_end = reinterpret_cast<int64_t *>(smem + sizeof(Shared));
    int32_t *ring_tail = reinterpret_cast<int32_t *>(comm_end + g.R);

    // per-CTA scratch slot
    unsigned char *base = sc.base + (size_t)blockIdx.x * sc.slot_bytes;
    Ctx c;
    c.g = g; c.p = p; c.o = o;
    const size_t bw = (size_t)g.max_words * g.R;
    uint64_t *bits = reinterpret_cast<uint64_t *>(base + sc.off_bits);
    c.done = Bits{bits, g.R};
    c.rdyc = Bits{bits + bw, g.R};
    c.rdyh = Bits{bits + 2 * bw, g.R};
    c.due = Bits{bits + 3 * bw, g.R};
    c.cp = reinterpret_cast<int64_t *>(base + sc.off_cp);
    c.ring_inst = reinterpret_cast<int32_t *>(base + sc.off_ring);
    c.ring_node = c.ring_inst + (size_t)g.coll_stride * g.R;
    c.dur = reinterpret_cast<int64_t *>(base + sc.off_dur);
    c.inst_dur = reinterpret_cast<int64_t *>(base + sc.off_inst);
    c.inst_s = c.inst_dur + g.n_inst;
    c.inst_e = c.inst_s + g.n_inst;
    c.inst_cpmax = c.inst_e + g.n_inst;
    c.inst_ckey = reinterpret_cast<unsigned long long *>(c.inst_cpmax + g.n_inst);
    c.inst_wait = reinterpret_cast<int32_t *>(c.inst_ckey + g.n_inst);
    c.complist = c.inst_wait + g.n_inst;
    c.comm_end = comm_end;
    c.ring_tail = ring_tail;
    c.ncomp = &sh.ncomp;

    const int tid = threadIdx.x, bd = blockDim.x;
    int par = 0;
    if (tid == 0) { sh.parity = 0; sh.ncomp = 0; sh.flag = 0; }

    for (int cfg = blockIdx.x; cfg < p.n; cfg += gridDim.x) {
        // ---- cost stage (K1): this point's durations ----
        const int algo = p.algo[cfg], topo = p.topo_kind[cfg];
        const double bwv = p.bw[cfg];
        const int64_t lat = p.latency[cfg];
        int bad = 0, zero = 0;
        for (int i = tid; i < g.n_inst; i += bd) {
            int64_t d = coll_time(g, i, algo, topo, bwv, lat, p.rows[cfg], p.cols[cfg]);
            if (d < 0) { bad = 1; d = 0; }
            zero |= d == 0;
            c.inst_dur[i] = d;
            c.inst_cpmax[i] = 0;
            c.inst_ckey[i] = 0ull;
            c.inst_wait[i] = (int32_t)(g.inst_mem_off[i + 1] - g.inst_mem_off[i]);
            c.inst_s[i] = 0;
            c.inst_e[i] = 0;
        }
        const bool recost = p.peak_flops != nullptr;
        for (int n = tid; n < g.total_nodes; n += bd) {
            int64_t d = g.node_dur[n];
            if (recost && g.node_kind[n] == FL_COMP && g.node_flops[n] >= 0)
                d = flops_to_ns(g.node_flops[n], p.peak_flops[cfg], p.efficiency[cfg]);
            c.dur[n] = d;
        }
        for (size_t i = tid; i < 4 * bw; i += bd) bits[i] = 0;
        for (int r = tid; r < g.R; r += bd) { comm_end[r] = 0; ring_tail[r] = 0; }
        bad = __syncthreads_or(bad);
        zero = __syncthreads_or(zero);
        if (bad) {
            if (tid == 0) o.status[cfg] = FL_ERR_UNSUPPORTED_ALGO;
            continue;
        }
        Cfg f;
        f.dur = c.dur;
        f.serial = zero;
        f.step = 0;
        f.init = 1;

        // ---- per-rank state ----
        Rank<K> s;
        const bool active = tid < g.R;
        s.r = active ? tid : 0;
        const int st = g.rank_struct[s.r];
        s.nb = g.s_node_off[st];
        s.N = active ? g.s_node_off[st + 1] - s.nb : 0;
        s.tb = g.s_tens_off[st];
        s.due_s = s.rc_s = s.rh_s = 0;
        s.host_slot = 0; s.host_e = 0; s.host_n = -1;
        const int ncs = p.compute_streams;
#pragma unroll
        for (int q = 0; q < K; q++) { s.slot[q] = q < ncs ? 0 : TINF; s.occ_e[q] = 0; s.occ_n[q] = -1; }
        s.ring_head = s.ring_acur = 0;
        s.comp_busy = s.comm_busy = s.overlap = s.finish = s.cur = s.peak = s.free_t = s.cpmax = 0;
        s.alloc_t = active ? g.s_init_alloc[st] : 0;
        s.done_cnt = 0;
        s.pop_seq = 0;

        // ---- t = 0: initial dispatch + start phase (simulator.py:275-277) ----
        if (active) {
            for (int q = g.s_init_off[st]; q < g.s_init_off[st + 1]; q++) {
                int d = g.init_list[q];
                if (g.node_flags[s.nb + d] & 1) continue;
                dispatch(c, f, s, d, 0);
            }
            start_phase(c, f, s, 0, cfg);
        }
        int64_t cpm = reserve(c, sh, par, 0, true, cfg);
        f.init = 0;
        int64_t tcur = 0;
        bool overflow = false;

        // ---- event loop ----
        for (;;) {
            int64_t nt = active ? next_time(c, s, tcur) : TINF;
            const int64_t TCAP = (int64_t)1 << 49;   // keys pack (t, rank) into 64 bits
            uint64_t key = nt == TINF ? KINF : ((uint64_t)(nt < TCAP ? nt : TCAP) << 14) | (uint64_t)s.r;
            uint64_t kmin = block_min_u64(key, sh, par);
            if (kmin == KINF) break;
            const int64_t t = (int64_t)(kmin >> 14);
            const int rmin = (int)(kmin & 0x3fff);
            if (t >= TCAP || f.step >= (1ull << 25) - 2) { overflow = true; break; }
            if (t > tcur) {
                if (active) advance(c, s, tcur, t);
                tcur = t;
            }
            f.step++;
            if (!f.serial) {
                if (active) {
                    gather_due(c, s, t);
                    if (s.r > rmin) start_phase(c, f, s, t, cfg);
                    s.pop_seq = 0;
                    while (s.due_s) {
                        int x = bm_pop(c.due, s.due_s, s.r);
                        pop_event(c, f, s, x, t);
                        start_phase(c, f, s, t, cfg);
                    }
                }
                int64_t v = reserve(c, sh, par, t, false, cfg);
                cpm = v > cpm ? v : cpm;
            } else {
                // serial mode: the reference loop verbatim, one pop per iteration
                if (active) gather_due(c, s, t);
                for (;;) {
                    uint64_t k2 = (active && s.due_s) ? (((uint64_t)s.r << 13) | (uint64_t)bm_peek(c.due, s.due_s, s.r)) : KINF;
                    uint64_t m2 = block_min_u64(k2, sh, par);
                    if (m2 == KINF) break;
                    f.step++;
                    if (active && (int)(m2 >> 13) == s.r) {
                        s.pop_seq = 0;
                        int x = bm_pop(c.due, s.due_s, s.r);
                        pop_event(c, f, s, x, t);
                    }
                    if (active) start_phase(c, f, s, t, cfg);
                    int64_t v = reserve(c, sh, par, t, false, cfg);
                    cpm = v > cpm ? v : cpm;
                    if (active) gather_due(c, s, t);
                }
            }
        }
        if (active) advance(c, s, tcur, TINF);

        // ---- row: reductions over ranks (cli.py:336-341) ----
        int dead = active && s.done_cnt != s.N;
        dead = __syncthreads_or(dead);
        int64_t exposed = s.comm_busy - s.overlap;
        int64_t vals[6] = {s.finish, s.cpmax > cpm ? s.cpmax : cpm, s.comp_busy, s.comm_busy, exposed, s.peak};
        if (!active) for (int k = 0; k < 6; k++) vals[k] = 0;
        if (o.rank_stats && active) {
            int64_t *rs = o.rank_stats + ((size_t)cfg * g.R + s.r) * 5;
            rs[0] = s.finish; rs[1] = s.comp_busy; rs[2] = s.comm_busy; rs[3] = exposed; rs[4] = s.peak;
        }
        for (int k = 0; k < 6; k++) {
            int64_t v = block_max_i64(vals[k], sh, par);
            if (tid == 0) o.rows[(size_t)cfg * 6 + k] = v;
        }
        if (tid == 0) o.status[cfg] = overflow ? FL_ERR_CAPACITY : dead ? FL_ERR_DEADLOCK : FL_OK;
        __syncthreads();
    }
}

// ------------------------------------------------------------ host side

cudaError_t launch_sweep(int K, int grid, int block, size_t smem, cudaStream_t st, const DevGraph &g,
                         const DevPoints &p, const DevOut &o, const DevScratch &sc) {
    if (K == 1) sweep_kernel<1><<<grid, block, smem, st>>>(g, p, o, sc);
    else if (K == 2) sweep_kernel<2><<<grid, block, smem, st>>>(g, p, o, sc);
    else sweep_kernel<4><<<grid, block, smem, st>>>(g, p, o, sc);
    return cudaGetLastError();
}

cudaError_t sweep_occupancy(int block, size_t smem, int *occ) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, sweep_kernel<1>, block, smem);
}

cudaError_t launch_cost_only(int n, const uint8_t *kind, const int64_t *size, const int64_t *gn,
                             const uint8_t *algo, const double *alpha, const double *beta,
                             const int32_t *rows, const int32_t *cols, int64_t *out, int32_t *status,
                             int m, const int64_t *flops, const double *peak, const double *eff,
                             int64_t *out_comp) {
    int total = n > m ? n : m;
    if (total <= 0) return cudaSuccess;
    cost_only_kernel<<<(total + 255) / 256, 256>>>(n, kind, size, gn, algo, alpha, beta, rows, cols, out,
                                                   status, m, flops, peak, eff, out_comp);
    return cudaGetLastError();
}

}  // namespace fl
