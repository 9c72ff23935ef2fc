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
// What makes it fast (with the A/B measurements):
//   * dependency edges whose order is fixed by ancestry are classed on the host
//     (capi.cu): first / middle / last writes, maxes and reads of the accumulator
//     replace per-edge read-modify-writes (pop_event);
//   * per-rank state lives in registers (what every step reads) and in shared-
//     memory planes with a compile-time stride (everything else, F_* / Q_*);
//   * collective arrivals are aggregated per warp (dispatch);
//   * design points wider than 1024 ranks run on thread-block clusters whose
//     per-step reduction goes through st.async + mbarrier (cl_step_min).
//
// Numerics: every fp64 operation of the cost model uses an explicit
// round-to-nearest intrinsic and the file is compiled with -fmad=false, so
// each expression is the reference's Python evaluation order with no FMA
// contraction.  Times are int64 ns.

#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

#include "flint_b200.h"
#include "engine_internal.h"

namespace fl {

namespace cg = cooperative_groups;

extern __shared__ __align__(16) unsigned char fl_smem[];   // the sweep kernel's dynamic shared memory

#ifdef FL_PROFILE     // development only: per-segment cycle counts of warp 0 of CTA 0
static __device__ unsigned long long fl_prof[16];
static __shared__ long long fl_prof_t;
#define PROF_MARK(k)                                                                      \
    do {                                                                                  \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                        \
            const long long now_ = clock64();                                             \
            atomicAdd(&fl_prof[k], (unsigned long long)(now_ - fl_prof_t));               \
            fl_prof_t = now_;                                                             \
        }                                                                                 \
    } while (0)
#else
#define PROF_MARK(k) do {} while (0)
#endif

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
static __device__ int64_t analytical_time(int kind, int64_t size, int64_t n, int algo, double a,
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

#ifndef FL_BASE
#define FL_BASE 0       // 0: this translation unit instantiates every kernel variant
#endif
#define FL_COMMON (FL_BASE == 0 || FL_BASE == 1)   // non-template kernels and the dispatchers
#ifndef FL_LEAN
#define FL_LEAN 1               // 0: never launch the lean variant (A/B)
#endif
#ifndef FL_LEAN_STEP
#define FL_LEAN_STEP 1          // lean: no due-set test in next_time, no t > tcur test per step
#endif
#ifndef FL_LEAN_TRACK
#define FL_LEAN_TRACK 1         // lean variants set `done` bits for tracked consumers only
#endif
#ifndef FL_RS1
#define FL_RS1 1                // single-CTA points also skip the step reduction after a full-world reservation
#endif
#ifndef FL_LEAN_FULL
#define FL_LEAN_FULL 1          // lean single-CTA variants assume every lane is a rank (block == R)
#endif

#if FL_COMMON
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
#endif

// ------------------------------------------------------- block primitives

constexpr unsigned FULL = 0xffffffffu;
constexpr int64_t TINF = INT64_MAX;
constexpr uint64_t KINF = ~0ull;

struct Shared {
    alignas(16) uint64_t xbuf[2][16][2];   // cluster step exchange: {min key, completions} per CTA (st.async)
    int tr_r, tr_x;                 // critical-path trace walk: the current (rank, local node)
    int seq_ovf;                    // a rank popped more than 8191 events at one time (ordering key capacity)
    unsigned long long xmbar[2];    // their mbarriers
    int cflag;                      // a rank of this CTA completed a collective / message since the last exchange
    int ncons;                      // cluster without messages: completion-list entries reserved so far
    int fifo_empty;                 // rank 0's comm FIFO was empty before this step's reservations
    uint64_t red[2][32];
    int64_t redi[2][32];
    int64_t cend_all;               // every rank's comm stream ends here (valid iff cend_uniform)
    int cend_uniform;
    int ncomp;
    int nmcomp;
    int pcols;                      // this design point's mesh columns
    int have_dur, dev_zdur;         // the previous point's device: durations in place, a zero-length node
    double dev_pk, dev_ef;
    double mbeta;                   // this design point's 1e9 / bw and latency (message wire times)
    int64_t mlat;
    // cluster variant: per-CTA partial results, written by every CTA of the cluster (DSMEM)
    uint64_t xkmin[2][16];
    int64_t xvmax[2][16];
    int xvor[2][16];
};

// Warp-wide 64-bit min / max by two REDUX each: the extreme of the high words, then of the low
// words among the lanes that hold it.  (A lockstep shortcut -- one shuffle and a vote when every
// lane holds the same time -- with a five-level shuffle tree behind it measured 1.5-2.4% slower
// on every workload: REDUX has no data-dependent branch and half the latency of the tree.)
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
    const unsigned hi = (unsigned)(v >> 32), mh = __reduce_min_sync(FULL, hi);
    const unsigned ml = __reduce_min_sync(FULL, hi == mh ? (unsigned)v : 0xffffffffu);
    return ((uint64_t)mh << 32) | ml;
}

__device__ __forceinline__ int64_t warp_max_i64(int64_t v) {
    const uint64_t u = (uint64_t)v ^ (1ull << 63);      // order-preserving signed -> unsigned
    const unsigned hi = (unsigned)(u >> 32), mh = __reduce_max_sync(FULL, hi);
    const unsigned ml = __reduce_max_sync(FULL, hi == mh ? (unsigned)u : 0u);
    return (int64_t)((((uint64_t)mh << 32) | ml) ^ (1ull << 63));
}

// Block-wide min of step keys (time << 14 | rank) or any 64-bit keys.
__device__ __forceinline__ uint64_t block_min_u64(uint64_t v, Shared &sh, int &par) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_min_u64(v);
    uint64_t *b = sh.red[par];
    par ^= 1;
    if (lane == 0) b[warp] = v;
    __syncthreads();
    v = lane < nw ? b[lane] : KINF;
    return warp_min_u64(v);
}

__device__ __forceinline__ uint64_t block_min_any(uint64_t v, Shared &sh, int &par) { return block_min_u64(v, sh, par); }

__device__ __forceinline__ int64_t block_max_i64(int64_t v, Shared &sh, int &par) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_max_i64(v);
    int64_t *b = sh.redi[par];
    par ^= 1;
    if (lane == 0) b[warp] = v;
    __syncthreads();
    v = lane < nw ? b[lane] : INT64_MIN;
    return warp_max_i64(v);
}

// A design point with more ranks than one CTA holds runs on a thread-block
// cluster (one CTA per 1024 ranks); its reductions and barriers span the
// cluster through distributed shared memory.  CL selects that variant.  The
// per-CTA partials are double-buffered on the same parity as the block-level
// buffers, so each buffer is reused only after another cluster barrier.
template <bool CL>
__device__ __forceinline__ void gsync() {
    if (CL) cg::this_cluster().sync();
    else __syncthreads();
}

template <bool CL>
__device__ __forceinline__ uint64_t gmin_key(uint64_t v, Shared &sh, int &par) {
    v = block_min_u64(v, sh, par);
    if (!CL) return v;
    cg::cluster_group cl = cg::this_cluster();
    const int n = (int)cl.num_blocks(), me = (int)cl.block_rank(), q = par ^ 1;
    if ((int)threadIdx.x < n) *cl.map_shared_rank(&sh.xkmin[q][me], (int)threadIdx.x) = v;
    cl.sync();
    uint64_t m = KINF;
    for (int j = 0; j < n; j++) m = sh.xkmin[q][j] < m ? sh.xkmin[q][j] : m;
    return m;
}

template <bool CL>
__device__ __forceinline__ int64_t gmax_i64(int64_t v, Shared &sh, int &par) {
    v = block_max_i64(v, sh, par);
    if (!CL) return v;
    cg::cluster_group cl = cg::this_cluster();
    const int n = (int)cl.num_blocks(), me = (int)cl.block_rank(), q = par ^ 1;
    if ((int)threadIdx.x < n) *cl.map_shared_rank(&sh.xvmax[q][me], (int)threadIdx.x) = v;
    cl.sync();
    int64_t m = INT64_MIN;
    for (int j = 0; j < n; j++) m = sh.xvmax[q][j] > m ? sh.xvmax[q][j] : m;
    return m;
}

template <bool CL>
__device__ __forceinline__ int gor(int v, Shared &sh, int &par) {
    v = __syncthreads_or(v);
    if (!CL) return v;
    cg::cluster_group cl = cg::this_cluster();
    const int n = (int)cl.num_blocks(), me = (int)cl.block_rank(), q = par;
    par ^= 1;
    if ((int)threadIdx.x < n) *cl.map_shared_rank(&sh.xvor[q][me], (int)threadIdx.x) = v;
    cl.sync();
    int m = 0;
    for (int j = 0; j < n; j++) m |= sh.xvor[q][j];
    return m;
}

// The per-step reduction of a cluster without cluster.sync: cluster.sync is a
// MEMBAR.ALL.GPU + CCTL.IVALL (it invalidates L1, so every step would re-read the node
// records from L2).  Each CTA st.async's its {block min, completion flag} into every
// CTA's exchange slot, which completes a transaction count on that CTA's mbarrier;
// waiting on the local mbarrier (acquire, CTA scope) makes all slots visible.  Steps
// in which some rank completed a collective or message then take a full cluster
// barrier before the reservation reads the shared instance state in HBM.
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t cl_step_min(uint64_t v, int &any, Shared &sh, int &par, unsigned &xk) {
    PROF_MARK(12);                              // (profile builds: exchange entry)
    v = block_min_u64(v, sh, par);              // (its barrier also orders this CTA's pops before cflag)
    PROF_MARK(13);                              // block min
    const int p = xk & 1;
    const unsigned ph = (xk >> 1) & 1;
    xk++;
    cg::cluster_group cl = cg::this_cluster();
    const unsigned n = cl.num_blocks(), me = cl.block_rank();
    const unsigned mb = smem_u32(&sh.xmbar[p]);
    if (threadIdx.x < 32) {         // warp 0: lane j sends to CTA j
        unsigned long long f = 0;
        if (threadIdx.x == 0) {
            f = (unsigned long long)sh.cflag;
            sh.cflag = 0;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(16u * n) : "memory");
        }
        f = __shfl_sync(FULL, f, 0);
        if (threadIdx.x < n) {
            const unsigned slot = smem_u32(&sh.xbuf[p][me][0]);
            unsigned ra, rmb;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(slot), "r"(threadIdx.x));
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rmb) : "r"(mb), "r"(threadIdx.x));
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];"
                         ::"r"(ra), "l"(v), "l"(f), "r"(rmb) : "memory");
        }
    }
    PROF_MARK(14);                              // sends
    unsigned done;
    do {
        asm volatile("{ .reg .pred q; mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 q, [%1], %2; "
                     "selp.u32 %0, 1, 0, q; }" : "=r"(done) : "r"(mb), "r"(ph) : "memory");
    } while (!done);
    // lane j reads CTA j's slot; the warp reduces them (two REDUX for the 64-bit min)
    const unsigned lane = threadIdx.x & 31u;
    const uint64_t x = lane < n ? sh.xbuf[p][lane][0] : KINF;
    const unsigned f = lane < n ? (unsigned)sh.xbuf[p][lane][1] : 0u;
    const unsigned hi = (unsigned)(x >> 32), mh = __reduce_min_sync(FULL, hi);
    const unsigned ml = __reduce_min_sync(FULL, hi == mh ? (unsigned)x : 0xffffffffu);
    any = (int)__reduce_or_sync(FULL, f);
    return ((uint64_t)mh << 32) | ml;
}

// ---------------------------------------------------------- rank state


// Node record built by capi.cu, two 16-byte words per node so that one
// broadcast load per word serves the 32 ranks of a warp visiting the node (an L1
// hit: the records of a graph set are a few tens of KB):
//   a = {succ_off | tracked << 31, succ_cnt | mfree_cnt << 12 | (first "last" edge + 1) << 24, ufree_lo, ufree_hi}
//       dependents; tensors with more than one consumer it may free (from g.mfree_off);
//       bytes of tensors it is the only (or statically last) consumer of; tracked: a consumer of a
//       tensor whose last consumer is decided at run time
//   b = {meta, coll_ord, alloc_lo, alloc_hi}        bytes allocated when the node starts
//   meta bits: 0-3 kind, 4 never-ready (waits on a missing node), 5 static host,
//   6-15 in-degree from non-static nodes, 16-25 in-degree
__device__ __forceinline__ int rec_kind(const uint4 &b) { return (int)(b.x & 15u); }
__device__ __forceinline__ bool rec_never(const uint4 &b) { return (b.x >> 4) & 1u; }
__device__ __forceinline__ bool rec_static(const uint4 &b) { return (b.x >> 5) & 1u; }
__device__ __forceinline__ uint64_t rec_indeg(const uint4 &b, bool fold) { return (b.x >> (fold ? 6 : 16)) & 0x3ffu; }
__device__ __forceinline__ int64_t rec_u64(uint32_t lo, uint32_t hi) { return (int64_t)(((uint64_t)hi << 32) | lo); }
__device__ __forceinline__ uint4 rec_a(const DevGraph &g, int gn) { return g.node_rec[2 * gn]; }
__device__ __forceinline__ uint4 rec_b(const DevGraph &g, int gn) { return g.node_rec[2 * gn + 1]; }

// Per-(node, rank) accumulator word, one int64 in global memory ([node][rank]):
//   bits 58-63  epoch of the design point that wrote it (stale words read as empty)
//   bits 48-57  dependencies still outstanding (in-degree <= 1023)
//   bits  0-47  max critical-path finish over the completed dependencies; once the
//               node is dispatched, its own critical-path finish
// so a dependency's completion is one read-modify-write that both counts it
// down (simulator.py:337-340) and relaxes the contention-free longest path
// (simulator.py:449-453) -- no per-rank in-degree table to initialize.
constexpr uint64_t VAL48 = (1ull << 48) - 1;

// Per-rank state that is not needed on every step lives in shared memory, one
// [field][blockDim] plane per field (a warp touches 256 contiguous bytes), addressed
// from the kernel's own shared symbol so every access is an LDS/STS.  Registers
// hold only what each step reads (the set heads, stream occupancy, the comm-FIFO
// head): a CTA of 1024 ranks has 64 registers per rank, and what does not fit would
// spill to local memory, i.e. to L2.
//   *_CP: contention-free critical-path finish of the node at the head of a set /
//   on a stream, carried along with it so that popping a node needs no HBM read;
//   a node that overflows a set's head into its bitmap parks the value in the
//   node's accumulator word instead (simulator.py:449-453 values, see below).
// Shared-memory planes, one per field.  The plane stride is a compile-time constant,
// so a field access is one LDS/STS at an immediate offset from the lane's own address
// (A/B: keeping the colder fields in HBM instead cost 9%).
enum {
    F_DUE_CP = 0, F_RC_CP, F_OCC_CP,                // heads of the due / ready-compute sets, running compute node
    F_COMM_END,                                     // end of this rank's comm stream (FIFO tail)
    F_FIN, F_CPMAX,                                 // last pop time; max critical-path finish popped
    F_COMP, F_OVL, F_COMP_A,                        // compute busy, compute-under-comm, commcum at compute start
    F_ALLOC, F_FREE, F_CUR, F_PEAK,                 // bytes allocated / freed at this step; memory in use, peak
    F_RH_CP, F_HOST_E, F_HOST_CP,                   // host stream (its slot is free at t iff host_n < 0)
    F_N64
};
enum { F_DUE_SUM = -1, F_RC_SUM = -1, F_RH_SUM = -1 };   // (sets keep no summaries: see MinSet)
// Plane stride (lanes), a compile-time constant per kernel variant: bits 5-6 of the
// variant word K select 1024 (0), 256 (1) or 64 (2), the smallest that holds the block,
// so small design points keep many CTAs per SM.
template <int K> __host__ __device__ constexpr int plane_lanes() { return ((K >> 5) & 3) == 0 ? 1024 : ((K >> 5) & 3) == 1 ? 256 : 64; }
constexpr int FL_SR = 1024;                         // widest plane (HBM fallback fields, capacity)
enum { Q_RING_TAIL = 0, Q_RING_HEAD, Q_RING_SEEN, Q_HEAD_NODE, Q_HEAD_INST, Q_DONE,
       Q_N32,                       // (the planes above are cleared per design point)
       Q_NB = Q_N32, Q_TB, Q_MYN,   // per CTA: the rank's first node / tensor in the graph set, its node count
       Q_ALL };

constexpr unsigned SM_HDR = (sizeof(Shared) + 15) / 16 * 16;
template <int K>
__device__ __forceinline__ int64_t &F64(int k, int lr) {
    constexpr int SR = plane_lanes<K>();
    return reinterpret_cast<int64_t *>(fl_smem + SM_HDR)[k * SR + lr];
}
template <int K>
__device__ __forceinline__ int32_t &F32(int k, int lr) {
    constexpr int SR = plane_lanes<K>();
    return reinterpret_cast<int32_t *>(fl_smem + SM_HDR + (size_t)F_N64 * 8 * SR)[k * SR + lr];
}
// Variants with messages (K & 8) add per-rank summaries of the rank's in-flight messages,
// so that a step reads no message state from HBM unless one of them starts or ends:
// the earliest end, the earliest start, the earliest start of one whose outputs are not
// yet allocated (TINF when none), and the list length (the list itself is unordered, in HBM).
enum { MF_E = 0, MF_S, MF_NA, MF_N64 };
template <int K>
__device__ __forceinline__ int64_t &FM64(int k, int lr) {
    constexpr int SR = plane_lanes<K>();
    return reinterpret_cast<int64_t *>(fl_smem + SM_HDR + (size_t)(F_N64 * 8 + Q_ALL * 4) * SR)[k * SR + lr];
}
template <int K>
__device__ __forceinline__ int32_t &QMN(int lr) {
    constexpr int SR = plane_lanes<K>();
    return reinterpret_cast<int32_t *>(fl_smem + SM_HDR + (size_t)(F_N64 * 8 + Q_ALL * 4 + MF_N64 * 8) * SR)[lr];
}

// Dynamic state of one point-to-point message (expanded comm mode), one 64-byte record:
// both endpoints' dispatch times and critical-path starts (simulator.py:259-268), the wire
// reservation [s, e) (simulator.py:310-327), the completion key and the endpoints to come.
struct alignas(64) MsgState {
    int64_t sendt, recvt, cps_s, cps_r, s, e;
    unsigned long long ckey;
    int32_t wait, pad;              // (ckey and wait are reset together: one 16-byte store)
};

// Per-CTA (block-uniform) state pointers.  Bitmaps are word-major,
// rank-minor ([word][rank]) so a warp's 32 ranks touch one 256-byte segment;
// `done` lives in shared memory when it fits.
struct Ctx {
    int R;
    int RL;                         // ranks owned by this CTA
    int base;                       // first rank owned by this CTA (clusters of CTAs share a design point)
    int BR, DR;                     // strides of the touched / done bitmaps (RL in shared memory, else R)
    bool lead_cta;                  // the cluster's first CTA (its thread 0 does the serial work)
    // [w][R] arrays are addressed [w * R + L.lr]: a cluster CTA's pointers below are offset by
    // its first rank (c.base), so only the *_g views index another CTA's columns by global rank
    // (and the cluster variant keeps no base + tid register: the compiler re-derived it ~70 times)
    uint64_t *done, *rdyc, *rdyh, *due;
    uint64_t *touched;              // [word][rank]: accumulator written in this design point
    int64_t *cp;                    // [max_nodes][R]: counted accumulators, parked set members
    int64_t *cp_g;                  // the same, not offset (message grants, trace walk)
    int64_t *acc;                   // [n_acc][R]: accumulators of statically ordered nodes, by slot
    int32_t *ring_inst, *ring_node; // [coll_stride][R] per-rank comm FIFO
    int64_t *dur;                   // [total_nodes] this design point's durations
    int64_t *inst_dur, *inst_s, *inst_e, *inst_cpmax;
    unsigned long long *inst_ckey;
    int32_t *inst_wait, *complist;
    int *ncomp;                     // shared
    // point-to-point messages (expanded comm mode), simulator.py:177-200, :310-327
    MsgState *msg;                  // [n_msg]
    int32_t *mcomplist;
    int *nmcomp;                    // shared: messages completed in this step
    int64_t *link_free, *link_busy; // [link_cap]
    unsigned long long *link_owner; // [link_cap] message-phase claims (KINF when free)
    int link_cap;
    int32_t *mlist;                 // [p2p_stride][R] per-rank in-flight messages (id | MSG_ALLOC), unordered
    int32_t *mlist_node;            // [p2p_stride][R] this rank's endpoint node of that message
    int64_t *mlist_s, *mlist_e;     // [p2p_stride][R] its wire reservation (copies: the list is read per step,
                                    // the message records are scattered over HBM)
    int32_t *mlist_g, *mlist_node_g;   // the in-flight lists, not offset (message grants)
    int64_t *mlist_s_g, *mlist_e_g;
};

// This design point's duration of node n: an LDS when the durations are in shared memory
// (g.dur_sm_off), else through the CTA's HBM copy.
__device__ __forceinline__ int64_t dur_of(const DevGraph &g, const Ctx &c, int n) {
    return g.dur_sm_off ? reinterpret_cast<const int64_t *>(fl_smem + g.dur_sm_off)[n] : c.dur[n];
}
// Bit 7 of the variant word: the lean variant, launched when the run needs no event record, no
// trace, no shared-memory first-dependency bitmap or slot table, and has the durations in shared
// memory -- those branches compile away (fewer live values under the 64-register cap).
template <int K> __host__ __device__ constexpr bool lean() { return (K & 128) != 0; }
// Bits 0-2: compute streams (1, 2 or 4); bit 9 instead: 8 compute streams (5-8 requested, the
// slots above the count never free)
template <int K> __host__ __device__ constexpr int nstreams() { return (K & 512) ? 8 : (K & 7); }
// bit 8 (lean variants only): the first-dependency bitmap and the slot table are both in shared
// memory (small design points) -- else both are not
template <int K> __host__ __device__ constexpr bool lean_sm() { return (K & 256) != 0; }
// A lean variant also assumes static hosts are folded (launched only for graph sets without a
// non-static HOST, so the host stream is never used) -- a design point that cannot fold (a
// zero-length node, engine.cu "t = 0 host pops") is marked FL_RETRY and evaluated by the
// general variant in a second pass (launch_sweep).
template <int K> __host__ __device__ constexpr bool nohost() { return lean<K>(); }
// where capi.cu puts the durations when they are in shared memory: right after the per-rank
// planes (a lean launch checks g.dur_sm_off against it)
template <int K> __host__ __device__ constexpr unsigned dur_off() {
    return (SM_HDR + (unsigned)plane_lanes<K>() * (8u * F_N64 + 4u * Q_ALL + ((K & 8) ? 8u * MF_N64 + 4u : 0u)) + 15u) / 16u * 16u;
}
template <int K>
__device__ __forceinline__ int64_t dur_of(const DevGraph &g, const Ctx &c, int n) {
    if constexpr (lean<K>()) return reinterpret_cast<const int64_t *>(fl_smem + dur_off<K>())[n];
    else return dur_of(g, c, n);
}

constexpr int32_t MSG_ALLOC = 1 << 30;   // mlist entry flag: the endpoint's outputs are allocated

// Per-thread rank identity: element w of rank r in a [w][R] array is at w * R + r.
struct Lane {
    int r, nb, tb;
    int lr;                         // this thread's lane of the shared per-rank fields (threadIdx.x)
    int br, dr;                     // column of the touched / done bitmaps (lr: shared memory, or HBM
                                    // through the offset pointers)
};

// Per-rank indices and strides.  Bit 16 of K marks the cluster variant, whose
// shared-memory arrays and bitmaps cover only this CTA's ranks (index lr,
// stride blockDim); a single CTA indexes everything by rank (index r, stride R).
// R is the caller's register copy of c.R (Ctx lives in shared memory, and a
// re-read after every shared store would cost an LDS per access).
template <int K> __device__ __forceinline__ uint64_t &done_ref(const Ctx &c, const Lane &L, int R, int w) {
    if constexpr ((K & 16) != 0) return c.done[w * c.DR + L.dr];
    else return c.done[w * R + L.lr];
}
template <int K> __device__ __forceinline__ uint64_t &touch_ref(const Ctx &c, const Lane &L, int R, int w) {
    if constexpr ((K & 16) != 0) return c.touched[w * c.BR + L.br];
    else return c.touched[w * R + L.lr];
}

// A node set with its minimum cached in a register and the rest in a global
// bitmap ([word][rank]).  head < 0: empty; else bits 0-15 = the minimum, bits 17-30 =
// the number of bitmap members (saturating at MS_SAT: then "some, maybe none"), so
// the bitmap is scanned only when it holds a member (invariant: the minimum < every
// bitmap member).  The due / ready sets rarely hold more than one node, so most
// inserts and pops are register operations; a pop with bitmap members scans the words
// above the minimum.
struct MinSet {
    int head;
};
constexpr int MS_SAT = 0x3fff;
__device__ __forceinline__ int ms_min(const MinSet &m) { return m.head & 0xffff; }
__device__ __forceinline__ int ms_cnt(const MinSet &m) { return m.head >> 17; }     // (head >= 0)
__device__ __forceinline__ int ms_inc(int cnt) { return (cnt + (cnt < MS_SAT)) << 17; }

#ifndef FL_REGF
#define FL_REGF 1
#endif
// Narrow single-CTA variants (planes of 64 or 256 lanes: at most 256 threads, so no register
// cap below 255) keep the own-lane busy and memory fields F_COMP..F_PEAK, which advance and
// gather_due update every step, in registers instead of shared-memory planes (no other lane
// reads them).  A/B on C2: +4%; also moving F_OCC_CP, F_FIN and F_CPMAX was +2%, and every
// own-lane field (the set heads too) +0%: the longer live ranges cost what the loads saved.
template <int K> __host__ __device__ constexpr bool regf() { return FL_REGF && !(K & 16) && ((K >> 5) & 3) != 0; }
constexpr int F_REG0 = F_COMP, F_REGN = F_PEAK + 1 - F_COMP;

template <int K>
struct Rank {
    int64_t rf[regf<K>() ? F_REGN : 1];   // (regf variants) own-lane fields, see regf()
    MinSet due, rc, rh;             // due events at t / ready compute nodes / ready host nodes
    int64_t slot[nstreams<K>()];            // compute stream free-at times (K > 1 only: with one stream
                                    // the stream is busy at t iff it has an occupant)
    int64_t occ_e[nstreams<K>()];           // end of the node running on each compute stream
    int64_t head_s, head_e;         // comm-FIFO head: start (HS_ALLOC once its outputs are allocated),
                                    // end (TINF when the FIFO is empty); FIFO indices in Q_RING_*
    int64_t commcum;                // integral of "comm stream busy" up to the current step (= comm busy)
    int host_n;                     // node running on the host stream (end in F_HOST_E), or -1
    int occ_n[nstreams<K>()];
    int pop_seq;
};

// An own-lane field: a register in regf variants, else the lane's shared-memory plane word.
template <int K>
__device__ __forceinline__ int64_t &RF(Rank<K> &s, int k, int lr) {
    if constexpr (regf<K>()) return s.rf[k - F_REG0];
    else return F64<K>(k, lr);
}

struct Step {                       // block-uniform per-step context
    uint64_t step;
    uint64_t epoch;                 // design-point epoch << 58 (accumulator tag)
    int init;
    int fold;                       // static hosts folded (see "t = 0 host pops")
    int touch;                      // first-dependency bitmap in shared memory (else epoch tags)
    int trace;                      // record every node's critical-path finish for the trace walk
    int acc_sm;                     // the accumulator slot table is in shared memory
};

__device__ __forceinline__ void bm_set(uint64_t *b, int R, int r, int idx) {
    b[(idx >> 6) * R + r] |= 1ull << (idx & 63);
}

// pops the smallest member above `from`, or returns -1 when there is none
__device__ __forceinline__ int bm_pop(uint64_t *b, int R, int r, int from, int nwords) {
    for (int w = from >> 6; w < nwords; w++) {
        uint64_t *p = b + (w * R + r);
        const uint64_t word = *p;
        if (word) {
            *p = word & (word - 1);
            return (w << 6) | (__ffsll((long long)word) - 1);
        }
    }
    return -1;
}

// Sets carrying each member's critical-path finish: the minimum's in shared field F,
// bitmap members' in their accumulator word cp[node][rank].
template <int K, int F, int FS>
__device__ __forceinline__ void ms_insert_cp(MinSet &m, uint64_t *b, int64_t *cp, int R, const Lane &L, int idx,
                                             int64_t v) {
    if (m.head < 0) {
        m.head = idx;
        F64<K>(F, L.lr) = v;
    } else if (idx < ms_min(m)) {
        const int h = ms_min(m);
        cp[h * R + L.lr] = F64<K>(F, L.lr);
        bm_set(b, R, L.lr, h);
        m.head = idx | ms_inc(ms_cnt(m));
        F64<K>(F, L.lr) = v;
    } else {
        cp[idx * R + L.lr] = v;
        bm_set(b, R, L.lr, idx);
        m.head = ms_min(m) | ms_inc(ms_cnt(m));
    }
}

template <int K, int F, int FS>
__device__ __forceinline__ int ms_pop_cp(MinSet &m, uint64_t *b, const int64_t *cp, int R, const Lane &L,
                                         int64_t &v, int nwords) {
    const int x = ms_min(m);
    v = F64<K>(F, L.lr);
    const int n = ms_cnt(m);
    if (n) {
        const int h = bm_pop(b, R, L.lr, x, nwords);
        if (h >= 0) {
            m.head = h | ((n - (n < MS_SAT)) << 17);
            F64<K>(F, L.lr) = cp[h * R + L.lr] & (int64_t)VAL48;
        } else {
            m.head = -1;
        }
    } else {
        m.head = -1;
    }
    return x;
}

template <int K>
__device__ __forceinline__ void record(const DevGraph &g, const DevOut &o, int cfg, int r, int x, int64_t st,
                                       int64_t en) {
    if (!lean<K>() && o.ev_start) {
        size_t at = ((size_t)cfg * g.R + r) * g.max_nodes + x;
        o.ev_start[at] = st;
        o.ev_end[at] = en;
    }
}

// One rank's start phase at time t (simulator.py:282-297 restricted to this rank).
template <int K>
__device__ __forceinline__ void start_phase(const DevGraph &g, const DevOut &o, const Ctx &c, const Lane &L,
                                            Rank<K> &s, const Step &f, int64_t t, int cfg) {
    const int R = g.R;                      // (a kernel parameter: no shared-memory load)
    while (!nohost<K>() && s.rh.head >= 0 && s.host_n < 0) {      // the host stream is free at t (gather_due ran at t)
        int64_t v;
        const int h = ms_pop_cp<K, F_RH_CP, F_RH_SUM>(s.rh, c.rdyh, c.cp, R, L, v, g.max_words);
        const int64_t e = t + dur_of<K>(g, c, L.nb + h);
        { const uint4 hb = rec_b(g, L.nb + h); RF<K>(s, F_ALLOC, L.lr) += rec_u64(hb.z, hb.w); }
        record<K>(g, o, cfg, L.r, h, t, e);
        if (e == t) {
            ms_insert_cp<K, F_DUE_CP, F_DUE_SUM>(s.due, c.due, c.cp, R, L, h, v);
        } else {
            F64<K>(F_HOST_E, L.lr) = e;
            F64<K>(F_HOST_CP, L.lr) = v;
            s.host_n = h;
        }
    }
    while (s.rc.head >= 0) {
        int k = 0;
        if constexpr (nstreams<K>() == 1) {
            if (s.occ_n[0] >= 0) break;   // the occupant ends after t (gather_due ran at t)
        } else {
#pragma unroll
            for (int q = 1; q < nstreams<K>(); q++) if (s.slot[q] < s.slot[k]) k = q;
            int64_t sk = s.slot[0];
#pragma unroll
            for (int q = 1; q < nstreams<K>(); q++) if (q == k) sk = s.slot[q];
            if (sk > t) break;
        }
        int64_t v;
        // (the node's record and duration are read before the pop's own shared-memory traffic)
        const uint2 xal = *reinterpret_cast<const uint2 *>(&g.node_rec[2 * (L.nb + ms_min(s.rc)) + 1].z);
        const int64_t dx = dur_of<K>(g, c, L.nb + ms_min(s.rc));
        const int x = ms_pop_cp<K, F_RC_CP, F_RC_SUM>(s.rc, c.rdyc, c.cp, R, L, v, g.max_words);
        const int64_t e = t + dx;
        RF<K>(s, F_ALLOC, L.lr) += rec_u64(xal.x, xal.y);
        record<K>(g, o, cfg, L.r, x, t, e);
        if (nstreams<K>() == 1 && e > t) {      // one compute stream: its busy intervals are disjoint
            RF<K>(s, F_COMP, L.lr) += e - t;
            RF<K>(s, F_COMP_A, L.lr) = s.commcum;
        }

#pragma unroll
        for (int q = 0; q < nstreams<K>(); q++) {
            if (q == k) {
                if constexpr (nstreams<K>() > 1) s.slot[q] = e;
                if (e == t) {
                    ms_insert_cp<K, F_DUE_CP, F_DUE_SUM>(s.due, c.due, c.cp, R, L, x, v);
                } else {
                    s.occ_e[q] = e;
                    s.occ_n[q] = x;
                    if (q == 0) F64<K>(F_OCC_CP, L.lr) = v;
                    else c.cp[x * R + L.lr] = v;     // streams 1..3: the running node's own accumulator word
                }
            }
        }
    }
}

// max of a 64-bit value over the lanes of `grp` (all of which call this)
__device__ __forceinline__ unsigned long long group_max_u64(unsigned grp, unsigned long long v) {
    const unsigned hi = (unsigned)(v >> 32), lo = (unsigned)v;
    const unsigned mh = __reduce_max_sync(grp, hi);
    const unsigned ml = __reduce_max_sync(grp, hi == mh ? lo : 0u);
    return ((unsigned long long)mh << 32) | ml;
}

// A node whose every dependency has completed (simulator.py:247-268); `cps`
// is its contention-free critical-path start (simulator.py:449).
template <int K>
__device__ __forceinline__ void dispatch(const DevGraph &g, const Ctx &c, const Lane &L, Rank<K> &s,
                                         const Step &f, int d, const uint4 &rb, int64_t cps, int seq, int64_t t) {
    const int R = g.R;                      // (a kernel parameter: no shared-memory load)
    const int kind = rec_kind(rb);
    if ((K & 8) && kind >= FL_SEND) {   // simulator.py:259-268: the message is granted once both ends are ready
        const int m = g.rank_p2p_msg[L.r * g.p2p_stride + (int)rb.y];
        MsgState &ms = c.msg[m];
        if (kind == FL_SEND) { ms.sendt = t; ms.cps_s = cps; }
        else { ms.recvt = t; ms.cps_r = cps; }
        if (f.step) {
            const unsigned long long key = ((unsigned long long)f.step << 39) | ((unsigned long long)L.r << 25) |
                                           ((unsigned long long)s.pop_seq << 12) | (unsigned long long)seq;
            atomicMax(&ms.ckey, key);
        }
        if (atomicSub(&ms.wait, 1) == 1) {
            c.mcomplist[atomicAdd(c.nmcomp, 1)] = m;
            if (K & 16) reinterpret_cast<Shared *>(fl_smem)->cflag = 1;
        }
        return;
    }
    if (kind == FL_COLL) {
        const int i = g.rank_coll_inst[L.r * g.coll_stride + (int)rb.y];
        // warp-aggregated: the lanes arriving at the same instance together update it once
        const unsigned grp = __match_any_sync(__activemask(), i);
        const unsigned long long cm = group_max_u64(grp, (unsigned long long)cps);
        const unsigned long long key = (f.step << 39) | ((unsigned long long)L.r << 25) |
                                       ((unsigned long long)s.pop_seq << 12) | (unsigned long long)seq;
        const unsigned long long km = f.init ? 0ull : group_max_u64(grp, key);
        if ((int)(threadIdx.x & 31) == __ffs(grp) - 1) {
            atomicMax((unsigned long long *)&c.inst_cpmax[i], cm);
            if (!f.init) atomicMax(&c.inst_ckey[i], km);
            const int cnt = __popc(grp);
            if (atomicSub(&c.inst_wait[i], cnt) == cnt) {
                c.complist[atomicAdd(c.ncomp, 1)] = i;
                if (K & 16) reinterpret_cast<Shared *>(fl_smem)->cflag = 1;
            }
        }
        return;
    }
    const int64_t fin = cps + dur_of<K>(g, c, L.nb + d);
    if (kind == FL_COMP) ms_insert_cp<K, F_RC_CP, F_RC_SUM>(s.rc, c.rdyc, c.cp, R, L, d, fin);
    else if (!nohost<K>()) ms_insert_cp<K, F_RH_CP, F_RH_SUM>(s.rh, c.rdyh, c.cp, R, L, d, fin);
}

// A statically ordered node's accumulator word (capi.cu "Accumulator slots"): in shared
// memory when the slot table fits there, else an L2 read that bypasses L1 (the words are
// written with RED operations).
__device__ __forceinline__ uint64_t acc_read(const Ctx &c, const Step &f, int idx) {
    return f.acc_sm ? (uint64_t)c.acc[idx] : (uint64_t)__ldcg(c.acc + idx);
}

// Pop one completion event (simulator.py:335-340) and free tensors whose last
// consumer it was (simulator.py:384-388).
template <int K>
__device__ __forceinline__ void pop_event(const DevGraph &g, const Ctx &c, const Lane &L, Rank<K> &s,
                                          const Step &f, int x, int64_t fx64, int64_t t) {
    const int R = g.R;                      // (a kernel parameter: no shared-memory load)
    const uint4 xa = rec_a(g, L.nb + x);
    // the `done` bit of a consumer whose completion a run-time free check reads (lean: only those)
    if ((lean<K>() && FL_LEAN_TRACK) ? (xa.x >> 31) != 0 : g.needs_done) done_ref<K>(c, L, R, x >> 6) |= 1ull << (x & 63);
    // 13-bit field of the keys (a lean launch has at most 8191 nodes per rank graph: cannot overflow)
    if (++s.pop_seq > 8191 && !lean<K>()) reinterpret_cast<Shared *>(fl_smem)->seq_ovf = 1;
    // pops counted (deadlock check), the rank's finish and its largest critical-path finish: a
    // lean variant updates them at sinks only -- every node precedes a sink of its rank graph,
    // with a finish no later than the sink's (capi.cu s_nsink)
    if (!lean<K>() || (xa.y & 0xfffu) == 0) {
        F32<K>(Q_DONE, L.lr)++;
        F64<K>(F_FIN, L.lr) = t;
        const int64_t cm = F64<K>(F_CPMAX, L.lr);
        if (fx64 > cm) F64<K>(F_CPMAX, L.lr) = fx64;
    }
    int64_t freed = rec_u64(xa.z, xa.w);
    const uint32_t nmf = (xa.y >> 12) & 0xfffu;
    if (nmf) for (uint32_t q = (uint32_t)g.mfree_off[L.nb + x], qe = q + nmf; q < qe; q++) {
        const int tt = L.tb + g.free_tens[q];
        const int2 cr = g.tens_rng[tt];
        bool all = true;
        for (int u = cr.x; u < cr.y && all; u++) {
            const int q = g.tens_cons[u];
            all = (done_ref<K>(c, L, R, q >> 6) >> (q & 63)) & 1;
        }
        if (all) freed += g.tens_bytes[tt];
    }
    if (freed) RF<K>(s, F_FREE, L.lr) += freed;
    PROF_MARK(9);                           // pop: records, statistics
    const uint64_t fx = (uint64_t)fx64;     // this node's critical-path finish
    // trace: the node's own word is dead once it is popped (its accumulator and its parking
    // as a set member are behind it), so it keeps the finish for the walk-back
    if (f.trace) c.cp[x * R + L.lr] = (int64_t)(f.epoch | fx);
    int seq = 0;
    const int32_t *sl = g.succ_ent;
    // the first "last" edge's accumulator read goes out before the other edges are processed
    const uint32_t lo = xa.y >> 24;
    const uint32_t q0 = xa.x & 0x7fffffffu;  // first successor entry
    const uint32_t qlast = lo && f.fold ? q0 + lo - 1 : 0xffffffffu;
    uint64_t alast = 0;
    if (qlast != 0xffffffffu) alast = acc_read(c, f, (int)((uint32_t)sl[qlast] >> 19) * R + L.lr);
    for (uint32_t q = q0, qe = q0 + (xa.y & 0xfffu); q < qe; q++, seq++) {
        const uint32_t ent = (uint32_t)sl[q];
        const int d = (int)(ent & 0xffffu);
        const int cls = f.fold ? (int)((ent >> 16) & 7u) : FL_EDGE_COUNTED;
        // Statically ordered predecessors (capi.cu): no counting, and only the last one
        // reads the accumulator -- a word of the small slot table [n_acc][R] that nodes with
        // disjoint accumulator lifetimes share (capi.cu "Accumulator slots"), so it stays in
        // L2.  A node that waits on a missing one is never dispatched.
        if (cls == FL_EDGE_FIRST) {
            c.acc[(int)(ent >> 19) * R + L.lr] = (int64_t)(f.epoch | fx);
            continue;
        }
        if (cls == FL_EDGE_MID) {
            int64_t *const w = c.acc + ((int)(ent >> 19) * R + L.lr);
            if (f.acc_sm) { if ((int64_t)(f.epoch | fx) > *w) *w = (int64_t)(f.epoch | fx); }   // (own column)
            else atomicMax(reinterpret_cast<unsigned long long *>(w), (unsigned long long)(f.epoch | fx));
            continue;
        }
        int64_t *slot = c.cp + (d * R + L.lr);
        const uint4 db = rec_b(g, L.nb + d);
        if (rec_never(db)) continue;
        if (cls == FL_EDGE_SINGLE) {
            dispatch(g, c, L, s, f, d, db, (int64_t)fx, seq, t);
            continue;
        }
        if (cls == FL_EDGE_LAST) {
            PROF_MARK(10);                  // edges before a "last" one
            const uint64_t a = (q == qlast ? alast : acc_read(c, f, (int)(ent >> 19) * R + L.lr)) & VAL48;
            dispatch(g, c, L, s, f, d, db, (int64_t)(a > fx ? a : fx), seq, t);
            PROF_MARK(11);                  // "last" edge: accumulator read + dispatch
            continue;
        }
        // first dependency to complete: the word holds nothing of this design point,
        // so skip reading it (a DRAM round trip on the critical chain)
        uint64_t a;
        if (f.touch) {
            uint64_t &tw = touch_ref<K>(c, L, R, d >> 6);
            const uint64_t tb = 1ull << (d & 63);
            if (tw & tb) {
                a = (uint64_t)*slot;
            } else {
                tw |= tb;
                a = f.epoch | (rec_indeg(db, f.fold) << 48);
            }
        } else {                // a word of an earlier design point reads as "no dependency completed"
            a = (uint64_t)*slot;
            if ((a >> 58) != (f.epoch >> 58)) a = f.epoch | (rec_indeg(db, f.fold) << 48);
        }
        const uint64_t v = (a & VAL48) > fx ? (a & VAL48) : fx;
        const uint64_t left = ((a >> 48) & 0x3ff) - 1;
        if (left == 0) dispatch(g, c, L, s, f, d, db, (int64_t)v, seq, t);
        else *slot = (int64_t)(f.epoch | (left << 48) | v);
    }
}

constexpr int64_t HS_ALLOC = INT64_MIN;   // head_s once the head's outputs are allocated (it started)

template <int K>
__device__ __forceinline__ void load_head(const Ctx &c, const Lane &L, Rank<K> &s, int R) {
    const int h = F32<K>(Q_RING_HEAD, L.lr);
    if (h < F32<K>(Q_RING_SEEN, L.lr)) {
        const int i = c.ring_inst[h * R + L.lr];
        F32<K>(Q_HEAD_NODE, L.lr) = c.ring_node[h * R + L.lr];
        F32<K>(Q_HEAD_INST, L.lr) = i;
        s.head_s = c.inst_s[i];
        s.head_e = c.inst_e[i];
    } else {
        s.head_e = TINF;
    }
}

// Append to lane lm's comm FIFO.  An entry appended to an empty FIFO is the head: it goes
// straight to the head fields in shared memory, the rest to HBM.
template <int K>
__device__ __forceinline__ void append_ring(const Ctx &c, int lm, int R, int inst, int node) {
    const int slot = F32<K>(Q_RING_TAIL, lm)++;
    if (slot == F32<K>(Q_RING_HEAD, lm)) {
        F32<K>(Q_HEAD_NODE, lm) = node;
        F32<K>(Q_HEAD_INST, lm) = inst;
    } else {
        c.ring_inst[slot * R + lm] = inst;
        c.ring_node[slot * R + lm] = node;
    }
}

// After reservations: pick up comm-FIFO entries appended for this rank.
template <int K>
__device__ __forceinline__ void refresh_ring(const Ctx &c, const Lane &L, Rank<K> &s) {
    const int tail = F32<K>(Q_RING_TAIL, L.lr);
    const int seen = F32<K>(Q_RING_SEEN, L.lr);
    if (tail != seen) {
        F32<K>(Q_RING_SEEN, L.lr) = tail;
        if (s.head_e == TINF) {     // the FIFO was empty: append_ring installed the new head
            const int i = F32<K>(Q_HEAD_INST, L.lr);
            s.head_s = c.inst_s[i];
            s.head_e = c.inst_e[i];
        }
    }
}

template <int K>
__device__ __forceinline__ int64_t next_time(const DevGraph &g, const Ctx &c, const Lane &L, const Rank<K> &s,
                                             int64_t tcur) {
    // (a lean point has no zero-length node: the due set is always drained at the top of a step)
    if (!(lean<K>() && FL_LEAN_STEP) && s.due.head >= 0) return tcur;
    int64_t nt = (!nohost<K>() && s.host_n >= 0) ? F64<K>(F_HOST_E, L.lr) : TINF;
#pragma unroll
    for (int q = 0; q < nstreams<K>(); q++) if (s.occ_n[q] >= 0 && s.occ_e[q] < nt) nt = s.occ_e[q];
    if (s.head_e < nt) nt = s.head_e;
    if (K & 8) {                                  // the earliest end of an in-flight message
        const int64_t e = FM64<K>(MF_E, L.lr);
        nt = e < nt ? e : nt;
    }
    return nt;
}

// Events already scheduled for exactly t join the due set.
template <int K>
__device__ __forceinline__ void gather_due(const DevGraph &g, const Ctx &c, const Lane &L, Rank<K> &s,
                                           int64_t t) {
    const int R = g.R;                      // (a kernel parameter: no shared-memory load)
    if (!nohost<K>() && s.host_n >= 0 && F64<K>(F_HOST_E, L.lr) == t) {
        ms_insert_cp<K, F_DUE_CP, F_DUE_SUM>(s.due, c.due, c.cp, R, L, s.host_n, F64<K>(F_HOST_CP, L.lr));
        s.host_n = -1;
    }
#pragma unroll
    for (int q = 0; q < nstreams<K>(); q++)
        if (s.occ_n[q] >= 0 && s.occ_e[q] == t) {
            const int64_t v = q == 0 ? F64<K>(F_OCC_CP, L.lr) : c.cp[s.occ_n[q] * R + L.lr];
            ms_insert_cp<K, F_DUE_CP, F_DUE_SUM>(s.due, c.due, c.cp, R, L, s.occ_n[q], v);
            s.occ_n[q] = -1;
            if (nstreams<K>() == 1) RF<K>(s, F_OVL, L.lr) += s.commcum - RF<K>(s, F_COMP_A, L.lr);   // comm time under [start, t)
        }
    while (s.head_e == t) {
        const int hn = F32<K>(Q_HEAD_NODE, L.lr), hi = F32<K>(Q_HEAD_INST, L.lr);
        if (s.head_s != HS_ALLOC) { const uint4 hb = rec_b(g, L.nb + hn); RF<K>(s, F_ALLOC, L.lr) += rec_u64(hb.z, hb.w); }  // zero-length: starts now
        // every member of an instance finishes at max over members' critical-path starts + duration
        // (simulator.py:419-428)
        ms_insert_cp<K, F_DUE_CP, F_DUE_SUM>(s.due, c.due, c.cp, R, L, hn, c.inst_cpmax[hi] + c.inst_dur[hi]);
        F32<K>(Q_RING_HEAD, L.lr)++;
        load_head(c, L, s, R);
    }
    if ((K & 8) && FM64<K>(MF_E, L.lr) == t) {   // messages of this rank ending now: their endpoints complete
        int n = QMN<K>(L.lr);
        int64_t me = TINF, msn = TINF, mna = TINF;
        for (int k = 0; k < n;) {
            const int ent = c.mlist[k * R + L.lr];
            const int64_t e = c.mlist_e[k * R + L.lr], st = c.mlist_s[k * R + L.lr];
            if (e == t) {
                const int node = c.mlist_node[k * R + L.lr];
                if (!(ent & MSG_ALLOC)) { const uint4 hb = rec_b(g, L.nb + node); RF<K>(s, F_ALLOC, L.lr) += rec_u64(hb.z, hb.w); }
                ms_insert_cp<K, F_DUE_CP, F_DUE_SUM>(s.due, c.due, c.cp, R, L, node, c.cp[node * R + L.lr] & (int64_t)VAL48);
                if (k != --n) {         // (unordered list: the last entry takes its place)
                    c.mlist[k * R + L.lr] = c.mlist[n * R + L.lr];
                    c.mlist_node[k * R + L.lr] = c.mlist_node[n * R + L.lr];
                    c.mlist_s[k * R + L.lr] = c.mlist_s[n * R + L.lr];
                    c.mlist_e[k * R + L.lr] = c.mlist_e[n * R + L.lr];
                }
                continue;
            }
            me = e < me ? e : me;
            msn = st < msn ? st : msn;
            if (!(ent & MSG_ALLOC)) mna = st < mna ? st : mna;
            k++;
        }
        QMN<K>(L.lr) = n;
        FM64<K>(MF_E, L.lr) = me;
        FM64<K>(MF_S, L.lr) = msn;
        FM64<K>(MF_NA, L.lr) = mna;
    }
}

// Close [tcur, tnew): busy/overlap integration (simulator.py:346-354 as a
// timeline) and the alloc-before-free high-water mark at tcur (:381-393).
template <int K>
__device__ __forceinline__ void advance(const DevGraph &g, const Ctx &c, const Lane &L, Rank<K> &s,
                                        int64_t tcur, int64_t tnew) {
    const int R = g.R;                      // (a kernel parameter: no shared-memory load)
    const bool head = s.head_e != TINF;
    if (head && s.head_s != HS_ALLOC && s.head_s <= tcur) {   // a collective that started by tcur
        const uint4 hb = rec_b(g, L.nb + F32<K>(Q_HEAD_NODE, L.lr));
        RF<K>(s, F_ALLOC, L.lr) += rec_u64(hb.z, hb.w);
        s.head_s = HS_ALLOC;
    }
    bool msg_on = false;            // a message of this rank is on the wire during [tcur, tnew)
    if (K & 8) {
        msg_on = FM64<K>(MF_S, L.lr) <= tcur;     // (TINF when no message is in flight)
        if (FM64<K>(MF_NA, L.lr) <= tcur) {      // a message started: allocate its endpoint's outputs
            const int n = QMN<K>(L.lr);
            int64_t mna = TINF;
            for (int k = 0; k < n; k++) {
                const int ent = c.mlist[k * R + L.lr];
                if (ent & MSG_ALLOC) continue;
                const int64_t st = c.mlist_s[k * R + L.lr];
                if (st <= tcur) {
                    const uint4 hb = rec_b(g, L.nb + c.mlist_node[k * R + L.lr]);
                    RF<K>(s, F_ALLOC, L.lr) += rec_u64(hb.z, hb.w);
                    c.mlist[k * R + L.lr] = ent | MSG_ALLOC;
                } else {
                    mna = st < mna ? st : mna;
                }
            }
            FM64<K>(MF_NA, L.lr) = mna;
        }
    }
    {
        const int64_t at = RF<K>(s, F_ALLOC, L.lr), ft = RF<K>(s, F_FREE, L.lr);
        if (at | ft) {
            const int64_t cur = RF<K>(s, F_CUR, L.lr) + at;
            if (cur > RF<K>(s, F_PEAK, L.lr)) RF<K>(s, F_PEAK, L.lr) = cur;
            RF<K>(s, F_CUR, L.lr) = cur - ft;
            RF<K>(s, F_ALLOC, L.lr) = 0;
            RF<K>(s, F_FREE, L.lr) = 0;
        }
    }
    if (tnew == TINF) return;
    const int64_t dt = tnew - tcur;
    const bool comm_on = (head && s.head_s <= tcur) || msg_on;
    if (comm_on) s.commcum += dt;
    if (nstreams<K>() > 1) {              // overlapping compute streams: integrate the union
        bool comp_on = false;
#pragma unroll
        for (int q = 0; q < nstreams<K>(); q++) comp_on |= s.occ_n[q] >= 0;
        if (comp_on) {
            RF<K>(s, F_COMP, L.lr) += dt;
            if (comm_on) RF<K>(s, F_OVL, L.lr) += dt;
        }
    }
}

__device__ __forceinline__ bool comp_before(const DevGraph &g, const Ctx &c, int a, int b, bool init) {
    // reservation order of instances completed in the same step
    const int64_t la = g.inst_lead_id[a], lb = g.inst_lead_id[b];
    if (init) {
        if (la != lb) return la < lb;
        return g.inst_init_key[a] < g.inst_init_key[b];
    }
    const unsigned long long ka = c.inst_ckey[a] >> 12, kb = c.inst_ckey[b] >> 12;
    if (ka != kb) return ka < kb;
    if (la != lb) return la < lb;
    return (c.inst_ckey[a] & 0xfff) < (c.inst_ckey[b] & 0xfff);
}

// Visit the directed links of a src->dst message in route order
// (topology.py:68-86); ids: switch eg/in of rank index i -> 2i / 2i+1,
// mesh a -> neighbour: 4a + {+col, -col, +row, -row}.
template <typename F>
__device__ __forceinline__ void for_route(const DevGraph &g, int topo, int cols, int si, int di, F &&fn) {
    if (si == di) return;
    if (topo == FL_SWITCH) { fn(2 * si); fn(2 * di + 1); return; }
    const int src = (int)g.rank_value[si], dst = (int)g.rank_value[di];   // (capi.cu: rank ids < 2^27 with messages)
    int r = src / cols, cc = src % cols;
    const int r1 = dst / cols, c1 = dst % cols;
    while (cc != c1) { fn(4 * (r * cols + cc) + (c1 > cc ? 0 : 1)); cc += c1 > cc ? 1 : -1; }
    while (r != r1) { fn(4 * (r * cols + cc) + (r1 > r ? 2 : 3)); r += r1 > r ? 1 : -1; }
}

// topology.py:95-102: per-hop latency plus one serialization, integer ns.
__device__ __forceinline__ int64_t transfer_ns(const DevGraph &g, int topo, int cols, int si, int di, int64_t bytes,
                                               int64_t lat, double beta) {
    if (si == di) return 0;
    int64_t hops = 1;
    if (topo == FL_MESH2D) {
        const int src = (int)g.rank_value[si], dst = (int)g.rank_value[di];
        const int dr = src / cols - dst / cols, dc = src % cols - dst % cols;
        hops = (dr < 0 ? -dr : dr) + (dc < 0 ? -dc : dc);
    }
    return rhu(__dadd_rn((double)(hops * lat), __dmul_rn((double)bytes, beta)));
}

// Message phase (simulator.py:310-327): FIFO per link, a message holds every link on its
// route for the whole transfer, messages are granted in (completing pop, source rank id,
// SEND node id) order.  Only messages that share a link interact, so the phase runs on the
// whole CTA in rounds: each pending message claims its links with an atomicMin of its
// order key, a message that holds every one of its links is the earliest pending user of
// each and is granted (reads and advances their free times), then the claims are released.
// A message is granted only after every earlier message sharing one of its links, so the
// result is the reference's sequential loop; messages on disjoint links (a ring step: every
// rank sends to its neighbour) are granted in one round.
//   key: completing pop (rank << 13 | pop sequence, the reservation's step is common) << 32
//        | the message's static (source rank id, SEND id) order (capi.cu msg_ord)
constexpr int32_t MQ_DONE = 1 << 30;     // mcomplist entry granted in the current round
__device__ __forceinline__ unsigned long long msg_key(const DevGraph &g, const Ctx &c, int m, bool init) {
    const unsigned long long pop = init ? 0ull : (c.msg[m].ckey >> 12) & ((1ull << 27) - 1);
    return (pop << 32) | (uint32_t)g.msg_ord[m];
}

// Rank rr's in-flight summary field (or list length): this CTA's shared memory, or in a
// cluster the owning CTA's, through distributed shared memory (blockDim ranks per CTA).
template <int K, bool CL>
__device__ __forceinline__ int64_t *msg_field(int k, int rr) {
    if constexpr (!CL) return &FM64<K>(k, rr);
    else return cg::this_cluster().map_shared_rank(&FM64<K>(k, rr % (int)blockDim.x), rr / (int)blockDim.x);
}
template <int K, bool CL>
__device__ __forceinline__ int32_t *msg_count(int rr) {
    if constexpr (!CL) return &QMN<K>(rr);
    else return cg::this_cluster().map_shared_rank(&QMN<K>(rr % (int)blockDim.x), rr / (int)blockDim.x);
}

// Grant message m the links of its route (its claims hold all of them): the reservation,
// the endpoints' critical-path values and their in-flight list entries.
template <int K, bool CL>
__device__ __forceinline__ void grant_msg(const DevGraph &g, const DevOut &o, const Ctx &c, int m, int si, int di,
                                          int topo, int cols, int cfg, uint64_t epoch, int64_t lat, double beta) {
    const int R = g.R;
    MsgState &ms = c.msg[m];
    int64_t st = ms.sendt > ms.recvt ? ms.sendt : ms.recvt;
    for_route(g, topo, cols, si, di, [&](int l) { st = c.link_free[l] > st ? c.link_free[l] : st; });
    const int64_t xf = transfer_ns(g, topo, cols, si, di, g.msg_bytes[m], lat, beta), e = st + xf;
    for_route(g, topo, cols, si, di, [&](int l) {
        c.link_free[l] = e;
        const int64_t b0 = c.link_busy[l];
        c.link_busy[l] = (b0 < 0 ? 0 : b0) + (e - st);
    });
    ms.s = st;
    ms.e = e;
    // critical path: a RECV also waits for its SEND plus the wire (simulator.py:430-435, :450-452)
    const int64_t cs = ms.cps_s;
    const int64_t cr = ms.cps_r > cs + xf ? ms.cps_r : cs + xf;
    const int sn = g.msg_send_node[m], dn = g.msg_recv_node[m];
    c.cp_g[sn * R + si] = (int64_t)(epoch | (uint64_t)cs);
    c.cp_g[dn * R + di] = (int64_t)(epoch | (uint64_t)cr);
    record<K>(g, o, cfg, si, sn, st, e);
    record<K>(g, o, cfg, di, dn, st, e);
    for (int side = 0; side < 2; side++) {     // both endpoints' in-flight lists and summaries
        const int rr = side ? di : si;
        const int k2 = atomicAdd(msg_count<K, CL>(rr), 1);
        c.mlist_g[k2 * R + rr] = m;
        c.mlist_node_g[k2 * R + rr] = side ? dn : sn;
        c.mlist_s_g[k2 * R + rr] = st;
        c.mlist_e_g[k2 * R + rr] = e;
        atomicMin(reinterpret_cast<long long *>(msg_field<K, CL>(MF_E, rr)), (long long)e);
        atomicMin(reinterpret_cast<long long *>(msg_field<K, CL>(MF_S, rr)), (long long)st);
        atomicMin(reinterpret_cast<long long *>(msg_field<K, CL>(MF_NA, rr)), (long long)st);
    }
}

template <int K, bool CL>
static __device__ void reserve_msgs(const DevGraph &g, const DevOut &o, const Ctx &c, int nm, bool init, int topo,
                                    int cols, int cfg, uint64_t epoch, int64_t lat, double beta) {
    const int tid = threadIdx.x, bd = blockDim.x;
    unsigned long long *own = c.link_owner;           // KINF between phases
    if (nm <= bd) {
        // the common case, at most one message per thread: its identity stays in registers
        const int m = tid < nm ? c.mcomplist[tid] : -1;
        unsigned long long k = 0;
        int si = 0, di = 0;
        if (m >= 0) { k = msg_key(g, c, m, init); si = g.msg_send_rank[m]; di = g.msg_recv_rank[m]; }
        bool pending = m >= 0;
        for (;;) {
            if (pending) for_route(g, topo, cols, si, di, [&](int l) { atomicMin(&own[l], k); });     // claim
            if (!__syncthreads_or(pending)) break;
            bool mine = pending;
            if (pending) for_route(g, topo, cols, si, di, [&](int l) { mine &= *(volatile unsigned long long *)&own[l] == k; });
            if (mine) grant_msg<K, CL>(g, o, c, m, si, di, topo, cols, cfg, epoch, lat, beta);
            __syncthreads();
            if (pending) for_route(g, topo, cols, si, di, [&](int l) { own[l] = KINF; });            // release
            pending &= !mine;
            __syncthreads();
        }
        return;
    }
    for (;;) {
        int left = 0;
        for (int q = tid; q < nm; q += bd) {           // claim
            const int m = c.mcomplist[q];
            if (m < 0) continue;
            left = 1;
            const unsigned long long k = msg_key(g, c, m, init);
            for_route(g, topo, cols, g.msg_send_rank[m], g.msg_recv_rank[m], [&](int l) { atomicMin(&own[l], k); });
        }
        if (!__syncthreads_or(left)) break;
        for (int q = tid; q < nm; q += bd) {           // grant the messages holding all their links
            const int m = c.mcomplist[q];
            if (m < 0) continue;
            const int si = g.msg_send_rank[m], di = g.msg_recv_rank[m];
            const unsigned long long k = msg_key(g, c, m, init);
            bool mine = true;
            for_route(g, topo, cols, si, di, [&](int l) { mine &= *(volatile unsigned long long *)&own[l] == k; });
            if (!mine) continue;
            grant_msg<K, CL>(g, o, c, m, si, di, topo, cols, cfg, epoch, lat, beta);
            c.mcomplist[q] = m | MQ_DONE;
        }
        __syncthreads();
        for (int q = tid; q < nm; q += bd) {           // release every claim of this round
            const int e = c.mcomplist[q];
            if (e < 0) continue;
            const int m = e & ~MQ_DONE;
            for_route(g, topo, cols, g.msg_send_rank[m], g.msg_recv_rank[m], [&](int l) { own[l] = KINF; });
            if (e & MQ_DONE) c.mcomplist[q] = -1;
        }
        __syncthreads();
    }
}

// Reserve the comm streams of every instance completed in this step, in the
// reference's order (simulator.py:298-309), block- (or cluster-) wide; then the
// step's messages (simulator.py:310-327).  Returns the end of the first reserved
// instance when every reserved instance spanned the world with uniform comm streams
// (then every rank's FIFO changed the same way), else -1.
// (inlined: as a real call the ABI spilled the caller's live registers around it)
template <bool MSG, bool CL, int K>
__device__ __forceinline__ int64_t reserve_n(const DevGraph &g, const DevOut &o, const Ctx &c, Shared &sh, int &par,
                                          int64_t t, bool init, int cfg, uint64_t epoch,
                                          int nc, int nmc, int topo, int cols) {
    // A cluster without messages never rewinds the completion list within a design point:
    // this reservation's entries start at sh.ncons, so no barrier is needed before the
    // counter could be reset (the instance times it writes are per-CTA copies).
    constexpr bool MONO = CL && !MSG;
    int32_t *const cl = c.complist + (MONO ? sh.ncons : 0);
    int64_t efirst = -1;            // end of the first reserved instance ...
    bool allfull = true;            // ... if every one spanned the world with uniform comm streams
    if (nc > 1) {                   // one thread orders the list (shared by the cluster's CTAs)
        if ((!CL || c.lead_cta) && threadIdx.x == 0) {
            for (int a = 1; a < nc; a++) {
                const int x = cl[a];
                int b = a - 1;
                while (b >= 0 && comp_before(g, c, x, cl[b], init)) { cl[b + 1] = cl[b]; b--; }
                cl[b + 1] = x;
            }
        }
        gsync<CL>();
    }
    const int R = g.R, RL = CL ? c.RL : g.R, base = CL ? c.base : 0;
    // While every collective so far spanned all ranks, every comm stream ends at the
    // same time and a full-world reservation needs no reduction (simulator.py:300-303).
    bool uni = sh.cend_uniform;
    int64_t cend = sh.cend_all;
    for (int q = 0; q < nc; q++) {
        const int i = cl[q];
        const int64_t m0 = g.inst_mem_off[i], nm = g.inst_mem_off[i + 1] - m0;
        const int full_node = g.inst_full_node[i];      // >= 0: members are ranks 0..R-1, all at this node
        int64_t s;
        if (full_node >= 0 && uni) {
            s = cend > t ? cend : t;
        } else {
            allfull = false;
            gsync<CL>();            // comm ends written by the previous reservation
            int64_t local = t;
            for (int64_t j = threadIdx.x; j < nm; j += blockDim.x) {
                const int lm = g.inst_mem_rank[m0 + j] - base;
                if (lm < 0 || lm >= RL) continue;       // another CTA's rank
                const int64_t ce = F64<K>(F_COMM_END, lm);
                local = ce > local ? ce : local;
            }
            s = gmax_i64<CL>(local, sh, par);
        }
        const int64_t e = s + c.inst_dur[i];
        if (q == 0) efirst = e;
        if (threadIdx.x == 0) { c.inst_s[i] = s; c.inst_e[i] = e; }      // (each CTA its own copy)
        if (full_node >= 0) {
            for (int lm = threadIdx.x; lm < RL; lm += blockDim.x) {
                const int m = base + lm;
                F64<K>(F_COMM_END, lm) = e;
                append_ring<K>(c, lm, R, i, full_node);
                record<K>(g, o, cfg, m, full_node, s, e);
            }
            uni = true;
            cend = e;
        } else {
            for (int64_t j = threadIdx.x; j < nm; j += blockDim.x) {
                const int m = g.inst_mem_rank[m0 + j], node = g.inst_mem_node[m0 + j];
                const int lm = m - base;
                if (lm < 0 || lm >= RL) continue;
                F64<K>(F_COMM_END, lm) = e;
                append_ring<K>(c, lm, R, i, node);
                record<K>(g, o, cfg, m, node, s, e);
            }
            uni = false;
            gsync<CL>();            // the next reservation reads these comm ends
        }
    }
    if (MONO) __syncthreads();      // this CTA has read sh.cend_* and sh.ncons
    else gsync<CL>();               // every CTA has read the counters and the list
    if (threadIdx.x == 0) {
        sh.cend_uniform = uni;
        sh.cend_all = cend;
        sh.cflag = 0;
        if (MONO) sh.ncons += nc;
    }
    if (!MONO && (!CL || c.lead_cta) && threadIdx.x == 0) { if (CL) *c.ncomp = 0; else sh.ncomp = 0; }
    // Without messages nothing written above is read before the caller's next barrier
    // (its step reduction, or reserve()'s own).  The message phase runs on the (lead) CTA
    // and fills other ranks' in-flight lists, which their own threads then order.
    if (MSG && nmc) {
        if (!CL || c.lead_cta) {
            reserve_msgs<K, CL>(g, o, c, nmc, init, topo, cols, cfg, epoch, sh.mlat, sh.mbeta);
            if (threadIdx.x == 0) { if (CL) *c.nmcomp = 0; else sh.nmcomp = 0; }
        }
        gsync<CL>();
    }
    return allfull && !(MSG && nmc) ? efirst : -1;
}

// Barrier, then reserve whatever completed since the last reservation.
template <bool MSG, bool CL, int K>
__device__ __forceinline__ int64_t reserve(const DevGraph &g, const DevOut &o, const Ctx &c, Shared &sh, int &par,
                                           int64_t t, bool init, int cfg, uint64_t epoch,
                                           int topo, int cols) {
    gsync<CL>();
    const int nc = CL ? *c.ncomp - (MSG ? 0 : sh.ncons) : sh.ncomp, nmc = MSG ? (CL ? *c.nmcomp : sh.nmcomp) : 0;
    return (nc | nmc) ? reserve_n<MSG, CL, K>(g, o, c, sh, par, t, init, cfg, epoch, nc, nmc, topo, cols) : 0;
}

// Critical-path node trace of one completed design point, walked back on the device
// (fl_outputs.trace; the rule of engine.critical_path_trace, restated in
// oracle/pyoracle.py).  Every node's contention-free finish is in its word of c.cp
// (pop_event, f.trace); a node's start is finish - duration for HOST / COMP, the
// instance's critical-path start for a collective member (the union-of-deps join,
// simulator.py:419-428) and the finish itself for SEND / RECV (no duration; a RECV's
// start already includes its SEND plus the wire, simulator.py:450-452).  Runs on one
// CTA (a cluster's lead CTA reads the other CTAs' ranks from the shared slot): warp 0
// resolves ordinary nodes, the whole CTA a collective's union of member dependencies.
static __device__ void trace_walk(const DevGraph &g, const DevOut &o, const Ctx &c, Shared &sh, int &par, int cfg,
                                  int r0, int64_t best) {
    const int R = g.R, tid = threadIdx.x, lane = tid & 31, bd = blockDim.x;
    auto fin = [&](int r, int x) -> int64_t { return __ldcg(c.cp_g + ((size_t)x * R + r)) & (int64_t)VAL48; };
    if (tid < 32) {             // the sink: rank r0's lowest node finishing at the critical path
        const int st = g.rank_struct[r0], nb = g.s_node_off[st], n = g.s_node_off[st + 1] - nb;
        int found = -1;
        for (int x0 = 0; x0 < n && found < 0; x0 += 32) {
            const unsigned b = __ballot_sync(FULL, x0 + lane < n && fin(r0, x0 + lane) == best);
            if (b) found = x0 + __ffs(b) - 1;
        }
        if (tid == 0) { sh.tr_r = r0; sh.tr_x = found; }
    }
    __syncthreads();
    const int64_t cap = o.trace ? o.trace_cap : 0, guard = (int64_t)g.total_nodes * R + g.n_inst + 1;
    int64_t *out = o.trace + (size_t)cfg * cap;
    int64_t len = 0;
    for (;;) {
        const int r = sh.tr_r, x = sh.tr_x;
        if (x < 0 || len >= guard) break;
        if (tid == 0 && len < cap) out[len] = ((int64_t)r << 32) | x;
        len++;
        const int nb = g.s_node_off[g.rank_struct[r]];
        const uint4 rb = rec_b(g, nb + x);
        const int kind = rec_kind(rb);
        __syncthreads();                            // every thread has read sh.tr_*
        if (kind == FL_COLL) {
            const int i = g.rank_coll_inst[r * g.coll_stride + (int)rb.y];
            const int64_t s0 = c.inst_cpmax[i];
            uint64_t k = KINF;
            for (int64_t j = g.inst_mem_off[i] + tid; j < g.inst_mem_off[i + 1]; j += bd) {
                const int rm = g.inst_mem_rank[j];
                const int gm = g.s_node_off[g.rank_struct[rm]] + g.inst_mem_node[j];
                for (int u = g.pred_off[gm]; u < g.pred_off[gm + 1]; u++) {
                    const int pn = g.pred_idx[u];
                    if (fin(rm, pn) == s0) {
                        const uint64_t kk = ((uint64_t)rm << 32) | (uint32_t)pn;
                        k = kk < k ? kk : k;
                    }
                }
            }
            k = block_min_any(k, sh, par);
            if (tid == 0) { sh.tr_r = k == KINF ? 0 : (int)(k >> 32); sh.tr_x = k == KINF ? -1 : (int)(uint32_t)k; }
        } else if (tid < 32) {
            const int64_t fx = fin(r, x);
            const int64_t s0 = kind <= FL_COMP ? fx - dur_of(g, c, nb + x) : fx;
            int kx = 0x7fffffff;
            for (int u = g.pred_off[nb + x] + lane; u < g.pred_off[nb + x + 1]; u += 32) {
                const int pn = g.pred_idx[u];
                if (fin(r, pn) == s0) kx = pn < kx ? pn : kx;
            }
            kx = __reduce_min_sync(FULL, kx);
            if (lane == 0) {
                int nr = r, nx = kx == 0x7fffffff ? -1 : kx;
                if (nx < 0 && kind == FL_RECV) {    // the start was set by the SEND plus the wire
                    const int m = g.rank_p2p_msg[r * g.p2p_stride + (int)rb.y];
                    nr = g.msg_send_rank[m];
                    nx = g.msg_send_node[m];
                }
                sh.tr_r = nr;
                sh.tr_x = nx;
            }
        }
        __syncthreads();
    }
    if (tid == 0) o.trace_len[cfg] = (int32_t)len;
}

// Zero this CTA's ranks' columns of a [rows][R] array (clusters split a point's ranks; `a`
// is the CTA's offset view, column 0 = its first rank).
template <bool CL, typename T>
__device__ __forceinline__ void zero_cols(T *a, size_t rows, int R, int RL) {
    if constexpr (!CL) {
        for (size_t i = threadIdx.x; i < rows * R; i += blockDim.x) a[i] = 0;
    } else {               // (a cluster CTA's columns: RL == blockDim.x except in the last CTA)
        if ((int)threadIdx.x < RL)
            for (size_t w = 0; w < rows; w++) a[w * R + threadIdx.x] = 0;
    }
}

template <int K, bool CL>
#ifndef FL_NARROW_BOUNDS
#define FL_NARROW_BOUNDS 1
#endif
// Narrow-plane variants (<= 256 ranks per CTA) are launched with at most that many threads,
// so their register budget is not the 64 a 1024-thread CTA allows (FL_NARROW_BOUNDS=0: A/B)
__global__ void __launch_bounds__((FL_NARROW_BOUNDS && !CL) ? plane_lanes<K>() : 1024, 1)
    sweep_kernel(const __grid_constant__ DevGraph g, const __grid_constant__ DevPoints p,
                 const __grid_constant__ DevOut o, const __grid_constant__ DevScratch sc) {
    unsigned char *smem = fl_smem;
    Shared &sh = *reinterpret_cast<Shared *>(smem);
    constexpr int KK = K | (CL ? 16 : 0);   // helpers see the cluster variant through K's bit 16
    const int R = g.R;
    const int tid = threadIdx.x, bd = blockDim.x;
    const int CS = CL ? (int)cg::this_cluster().num_blocks() : 1;
    const int crank = CL ? (int)cg::this_cluster().block_rank() : 0;
    const int cid = blockIdx.x / CS, ncl = gridDim.x / CS;     // this cluster, clusters in the grid
    const int base_r = crank * bd;
    // ranks owned by this CTA (a single CTA's block is R rounded up to a warp, so RL = R: a
    // kernel parameter, which `active` tests straight from the constant bank -- a computed RL
    // was spilled and re-loaded from local memory at every step)
    const int RL = CL ? (R - base_r < bd ? R - base_r : bd) : R;
    if (!lean<K>() && p.retry) {    // second pass after a lean launch: leave at once without work
        int mine = 0;               // (every CTA of a cluster reads the same points: a uniform exit)
        for (int q = cid + tid * ncl; q < p.n && !mine; q += bd * ncl) mine = o.status[q] == FL_RETRY;
        if (!__syncthreads_or(mine)) return;
    }

    // ---- carve shared memory and this cluster's scratch slot ----
    // (the pointer table lives in shared memory: it is block-uniform and would
    // otherwise pin ~34 registers per thread)
    __shared__ Ctx c_sh;
    Ctx &c = c_sh;
    if (tid == 0) {
        c.R = R;
        c.RL = RL;
        c.base = base_r;
        unsigned char *base = sc.base + (size_t)cid * sc.slot_bytes;
        const size_t words = (size_t)g.max_words * R;
        uint64_t *gbits = reinterpret_cast<uint64_t *>(base + sc.off_bits) + base_r;   // (offset views)
        c.rdyc = gbits;
        c.rdyh = gbits + words;
        c.due = gbits + 2 * words;
        c.done = sc.done_in_smem ? reinterpret_cast<uint64_t *>(smem + sc.sm_off_done) : gbits + 3 * words;
        c.DR = sc.done_in_smem ? bd : R;
        c.touched = sc.touch_in_smem ? reinterpret_cast<uint64_t *>(smem + sc.sm_off_touch) : gbits + 4 * words;
        c.BR = sc.touch_in_smem ? bd : R;
        c.cp_g = reinterpret_cast<int64_t *>(base + sc.off_cp);
        c.cp = c.cp_g + base_r;
        c.acc = sc.acc_in_smem ? reinterpret_cast<int64_t *>(smem + sc.sm_off_acc)    // (single-CTA points only)
                               : reinterpret_cast<int64_t *>(base + sc.off_acc) + base_r;
        c.ring_inst = reinterpret_cast<int32_t *>(base + sc.off_ring) + base_r;
        c.ring_node = c.ring_inst + (size_t)g.coll_stride * R;    // (offset view)
        c.dur = sc.dur_in_smem ? reinterpret_cast<int64_t *>(smem + sc.sm_off_dur)
                               : reinterpret_cast<int64_t *>(base + sc.off_dur) + (size_t)crank * g.total_nodes;
        unsigned char *ib = sc.inst_in_smem ? smem + sc.sm_off_inst : base + sc.off_inst;
        const int NI = g.n_inst;
        c.inst_dur = reinterpret_cast<int64_t *>(ib);
        c.inst_s = c.inst_dur + NI;
        c.inst_e = c.inst_s + NI;
        c.inst_cpmax = c.inst_e + NI;
        if (CL) {                   // reservation times: one copy per CTA, written and read locally
            c.inst_s = reinterpret_cast<int64_t *>(base + sc.off_inst_se) + (size_t)crank * 2 * NI;
            c.inst_e = c.inst_s + NI;
        }
        c.inst_ckey = reinterpret_cast<unsigned long long *>(c.inst_cpmax + NI);
        c.inst_wait = reinterpret_cast<int32_t *>(c.inst_ckey + NI);
        c.complist = c.inst_wait + NI;
        int *ctr = reinterpret_cast<int *>(base + sc.off_ctr);   // cluster-wide completion counters
        c.ncomp = CL ? ctr : &sh.ncomp;
        c.nmcomp = CL ? ctr + 1 : &sh.nmcomp;
        c.lead_cta = crank == 0;
        const int M = g.n_msg;
        c.msg = reinterpret_cast<MsgState *>(base + sc.off_msg);
        c.link_free = sc.links_in_smem ? reinterpret_cast<int64_t *>(smem + sc.sm_off_links)
                                       : reinterpret_cast<int64_t *>(base + sc.off_links);
        c.link_busy = c.link_free + sc.link_cap;
        c.link_owner = reinterpret_cast<unsigned long long *>(c.link_busy + sc.link_cap);
        c.link_cap = sc.link_cap;
        c.mcomplist = reinterpret_cast<int32_t *>(c.msg + M);
        c.mlist_g = c.mcomplist + M;
        c.mlist_node_g = c.mlist_g + (size_t)g.p2p_stride * R;
        c.mlist_s_g = reinterpret_cast<int64_t *>(base + sc.off_mlist_se);
        c.mlist_e_g = c.mlist_s_g + (size_t)g.p2p_stride * R;
        c.mlist = c.mlist_g + base_r;
        c.mlist_node = c.mlist_node_g + base_r;
        c.mlist_s = c.mlist_s_g + base_r;
        c.mlist_e = c.mlist_e_g + base_r;
    }
    __syncthreads();
    const bool is_leader = crank == 0 && tid == 0;      // writes the point's row
    uint64_t *gbits = c.rdyc;
    const int NI = g.n_inst;

    // (a lean single-CTA variant runs only blocks of exactly R threads: every lane is a rank)
    const bool active = (lean<K>() && !CL && FL_LEAN_FULL) ? true : CL ? tid < RL : tid < g.R;
    Lane L;
    L.r = base_r + tid;             // (inactive lanes never index per-rank state with it)
    L.lr = tid;
    L.br = tid;                     // (shared memory, or the offset HBM view)
    L.dr = tid;
    {
        // kept in shared memory: re-reading them there is cheaper than the two dependent
        // global loads the compiler would otherwise repeat under register pressure
        const int st = active ? g.rank_struct[L.r] : 0;
        F32<K>(Q_NB, tid) = g.s_node_off[st];
        F32<K>(Q_TB, tid) = g.s_tens_off[st];
        F32<K>(Q_MYN, tid) = !active ? 0 : lean<K>() ? g.s_nsink[st] : g.s_node_off[st + 1] - g.s_node_off[st];
        L.nb = F32<K>(Q_NB, tid);
        L.tb = F32<K>(Q_TB, tid);
    }

    int par = 0;
    unsigned xk = 0;                // cluster step exchanges done (cl_step_min)
    // (the previous point's device -- its durations are reused when unchanged -- is kept in shared
    // memory, sh.dev_*: four registers fewer across the event loop)
    if (tid == 0) { sh.ncomp = 0; sh.nmcomp = 0; sh.cflag = 0; sh.have_dur = 0; }
    if (CL && tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sh.xmbar[0])) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&sh.xmbar[1])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (CL && is_leader) { c.ncomp[0] = 0; c.nmcomp[0] = 0; }
    // the global bitmaps are all-zero after a point that ran to completion;
    // clear them once up front and again only after a point that did not
    zero_cols<CL>(gbits, (size_t)g.max_words * 5, R, RL);  // ready/due/done/touched columns
    bool dirty = false;
    // epoch 0 = empty.  With the first-dependency bitmap in shared memory no word is read before
    // this design point wrote it (counted words behind their touched bit, set members and
    // trace finishes written first), so small points skip the table-wide clear
    if (!sc.touch_in_smem) zero_cols<CL>(c.cp, (size_t)g.max_nodes, R, RL);
    gsync<CL>();
    unsigned epoch = 0;
    const int gt = crank * bd + tid, gstride = CS * bd;        // cluster-wide thread index / stride

    for (int cfg = cid; cfg < p.n; cfg += ncl) {
        if (!lean<K>() && p.retry && o.status[cfg] != FL_RETRY) continue;   // (evaluated by the lean pass)
        // ---- cost stage (K1): this point's durations ----
        // (each design-point column is read once: fl_sweep_run may pass them in mapped host memory)
        const int algo = p.algo[cfg], topo = p.topo_kind[cfg];
        const double bwv = p.bw[cfg];
        const int64_t lat = p.latency[cfg];
        const int prows = p.rows[cfg], pcols = p.cols[cfg];
        if (tid == 0) sh.pcols = pcols;
        int bad = 0, zero = 0, cap_bad = 0;
        for (int i = gt; i < NI; i += gstride) {
            int64_t d = coll_time(g, i, algo, topo, bwv, lat, prows, pcols);
            if (d < 0) { bad = 1; d = 0; }
            zero |= d == 0;
            c.inst_dur[i] = d;
            c.inst_cpmax[i] = 0;
            c.inst_ckey[i] = 0ull;
            c.inst_wait[i] = (int32_t)(g.inst_mem_off[i + 1] - g.inst_mem_off[i]);
            if (!CL) { c.inst_s[i] = 0; c.inst_e[i] = 0; }
        }
        if (CL) for (int i = tid; i < NI; i += bd) { c.inst_s[i] = 0; c.inst_e[i] = 0; }   // (per-CTA copies)
        if (K & 8) {                // messages: fresh message and link state
            const double beta = __ddiv_rn(1e9, bwv);
            const int cols = pcols;
            if (topo == FL_MESH2D && (cols <= 0 || 4LL * prows * cols > c.link_cap)) cap_bad = 1;
            // a zero wire time would put events at the reservation's own time (serial mode); the
            // smallest possible one is one hop of the smallest message (transfer_ns is monotone)
            if (g.msg_self || (g.n_msg > 0 && rhu(__dadd_rn((double)lat, __dmul_rn((double)g.msg_min_bytes, beta))) == 0))
                zero = 1;
            if (tid == 0) { sh.mbeta = beta; sh.mlat = lat; }
            for (int m = gt; m < g.n_msg; m += gstride)     // ckey = 0, wait = 2 (one 16-byte store)
                *reinterpret_cast<uint4 *>(&c.msg[m].ckey) = make_uint4(0u, 0u, 2u, 0u);
            if (!CL || crank == 0)  // (only the lead CTA runs the message phase: links may be in its shared memory)
                for (int l = tid; l < c.link_cap; l += bd) { c.link_free[l] = 0; c.link_busy[l] = -1; c.link_owner[l] = KINF; }
            FM64<K>(MF_E, tid) = TINF;
            FM64<K>(MF_S, tid) = TINF;
            FM64<K>(MF_NA, tid) = TINF;
            QMN<K>(tid) = 0;
        }
        const bool recost = p.peak_flops != nullptr;
        const double pk = recost ? p.peak_flops[cfg] : 0.0, ef = recost ? p.efficiency[cfg] : 0.0;
        const bool same_dev = sh.have_dur && pk == sh.dev_pk && ef == sh.dev_ef;   // durations already in place
        int zdur = same_dev ? sh.dev_zdur : 0;   // a zero-duration COMP or non-static HOST could complete at t = 0
        if (!same_dev) for (int n = tid; n < g.total_nodes; n += bd) {
            int64_t d = g.node_dur[n];
            if (recost && g.node_flops[n] >= 0) d = flops_to_ns(g.node_flops[n], pk, ef);
            c.dur[n] = d;
            if (d == 0) {
                const uint4 nb_ = rec_b(g, n);
                zdur |= rec_kind(nb_) == FL_COMP || (rec_kind(nb_) == FL_HOST && !rec_static(nb_));
            }
        }
        if (dirty) zero_cols<CL>(gbits, (size_t)g.max_words * 3, R, RL);
        if (g.needs_done) {
            if (sc.done_in_smem) for (size_t i = tid; i < (size_t)g.max_words * bd; i += bd) c.done[i] = 0;
            else zero_cols<CL>(c.done, (size_t)g.max_words, R, RL);
        }
        if (sc.touch_in_smem) for (size_t i = tid; i < (size_t)g.max_words * bd; i += bd) c.touched[i] = 0;
        if (tid == 0) { sh.cend_all = 0; sh.cend_uniform = 1; sh.ncons = 0; sh.seq_ovf = 0; }
        if (CL && is_leader) *c.ncomp = 0;          // (MONO clusters: the list restarts per point)
#pragma unroll
        for (int k = 0; k < F_N64; k++) F64<K>(k, tid) = 0;
#pragma unroll
        for (int k = 0; k < Q_N32; k++) F32<K>(k, tid) = 0;
        bad = gor<CL>(bad, sh, par);
        cap_bad = gor<CL>(cap_bad, sh, par);
        if (cap_bad) bad = 2;
        zero = gor<CL>(zero, sh, par);
        zdur = gor<CL>(zdur, sh, par);
        if (tid == 0) { sh.have_dur = 1; sh.dev_pk = pk; sh.dev_ef = ef; sh.dev_zdur = zdur; }   // (read after barriers)
        if (bad) {
            if (is_leader) o.status[cfg] = bad == 2 ? FL_ERR_CAPACITY : FL_ERR_UNSUPPORTED_ALGO;
            if (is_leader && o.trace_len) o.trace_len[cfg] = 0;
            dirty = false;
            gsync<CL>();
            continue;
        }
        if (nohost<K>() && (!g.fold_ok || zero || zdur)) {   // left to the general variant's second pass
            if (is_leader) o.status[cfg] = FL_RETRY;
            dirty = false;
            gsync<CL>();
            continue;
        }
        if (++epoch == 64) {       // 6-bit tags wrap: start a fresh accumulator table
            if (!sc.touch_in_smem) zero_cols<CL>(c.cp, (size_t)g.max_nodes, R, RL);
            epoch = 1;
            gsync<CL>();
        }
        Step f;
        f.step = 0;
        f.epoch = (uint64_t)epoch << 58;
        f.init = 1;
        f.fold = nohost<K>() ? 1 : g.fold_ok && !zero && !zdur;   // (lean: points that do not fold were retried)
        f.touch = lean<K>() ? lean_sm<K>() : (bool)sc.touch_in_smem;
        f.acc_sm = lean<K>() ? lean_sm<K>() : (bool)sc.acc_in_smem;
        f.trace = !lean<K>() && o.trace_len != nullptr;

        // ---- per-rank state ----
        Rank<KK> s;
#pragma unroll
        for (int q = 0; q < (regf<KK>() ? F_REGN : 1); q++) s.rf[q] = 0;
        s.due.head = s.rc.head = s.rh.head = -1;
        s.host_n = -1;
        const int ncs = p.compute_streams;
#pragma unroll
        for (int q = 0; q < nstreams<K>(); q++) {
            if constexpr (nstreams<K>() > 1) s.slot[q] = q < ncs ? 0 : TINF;
            s.occ_e[q] = 0;
            s.occ_n[q] = -1;
        }
        s.head_s = 0;
        s.head_e = TINF;
        RF<KK>(s, F_ALLOC, tid) = active ? g.s_init_alloc[g.rank_struct[L.r]] : 0;
        s.commcum = 0;
        s.pop_seq = 0;
        constexpr bool MSG = (K & 8) != 0;

        // ---- t = 0: initial dispatch + start phase (simulator.py:275-277) ----
        if (active) {
            const int st = g.rank_struct[L.r];
            if (f.fold) {
                for (int q = g.s_init_ns_off[st]; q < g.s_init_ns_off[st + 1]; q++) {
                    const int d = g.init_ns[q];
                    dispatch(g, c, L, s, f, d, rec_b(g, L.nb + d), 0, 0, 0);
                }
            } else {
                for (int q = g.s_init_off[st]; q < g.s_init_off[st + 1]; q++) {
                    const int d = g.init_list[q];
                    const uint4 db = rec_b(g, L.nb + d);
                    if (rec_never(db)) continue;
                    dispatch(g, c, L, s, f, d, db, 0, 0, 0);
                }
            }
            start_phase(g, o, c, L, s, f, 0, cfg);
        }
        // (reservations also return their instances' critical-path finishes; every member's
        // pop folds the same value into F_CPMAX, so the row needs only that)
        reserve<MSG, CL, KK>(g, o, c, sh, par, 0, true, cfg, f.epoch, topo, sh.pcols);
        if (active) refresh_ring(c, L, s);
        f.init = 0;
        if (f.fold) {
            // ---- t = 0 host pops, folded.  Every HOST with no dependencies and zero
            // duration starts at t=0 in the initial start phase and completes at t=0
            // (simulator.py:282-287); with no other zero-length node in this design
            // point they are the only t=0 events, popped in id order.  Their effect
            // is (a) counted away in the dependency accumulators (in-degree without
            // static hosts) and (b) the dispatch of nodes waiting only on them,
            // replayed here in (trigger host, position) order, each host's pop
            // followed by its start phase.
            f.step++;
            if (active) {
                const int st = g.rank_struct[L.r];
                s.pop_seq = 0;
                int prev = -1;
                for (int q = g.trig_off[st]; q < g.trig_off[st + 1]; q++) {
                    const int4 tr = g.trig[q];
                    if (tr.x != prev) {
                        if (prev >= 0) start_phase(g, o, c, L, s, f, 0, cfg);
                        if (++s.pop_seq > 8191) sh.seq_ovf = 1;
                        prev = tr.x;
                    }
                    dispatch(g, c, L, s, f, tr.y, rec_b(g, L.nb + tr.y), 0, tr.z, 0);
                }
                if (prev >= 0) start_phase(g, o, c, L, s, f, 0, cfg);
                if (!lean<K>()) F32<K>(Q_DONE, tid) += g.s_nstatic[st];   // (lean: sinks only)
                if (f.trace)        // folded static hosts start and finish at 0 (never popped here)
                    for (int q = g.static_off[st]; q < g.static_off[st + 1]; q++)
                        c.cp[g.static_list[q] * R + L.lr] = (int64_t)f.epoch;
                if (!lean<K>() && o.ev_start)
                    for (int q = g.static_off[st]; q < g.static_off[st + 1]; q++)
                        record<K>(g, o, cfg, L.r, g.static_list[q], 0, 0);
            }
            reserve<MSG, CL, KK>(g, o, c, sh, par, 0, false, cfg, f.epoch, topo, sh.pcols);
            if (active) refresh_ring(c, L, s);
        }
        int64_t tcur = 0;
        bool overflow = false;

        // ---- event loop ----
        const int64_t TCAP = (int64_t)1 << 48;   // 48-bit accumulators; keys pack (t, rank)
#ifdef FL_PROFILE
        if (blockIdx.x == 0 && threadIdx.x == 0) fl_prof_t = clock64();
#endif
        for (;;) {
            PROF_MARK(0);                                   // loop back-edge
            int64_t nt = active ? next_time(g, c, L, s, tcur) : TINF;
            uint64_t key = nt == TINF ? KINF : ((uint64_t)(nt < TCAP ? nt : TCAP) << 14) | (uint64_t)L.r;
            PROF_MARK(1);                                   // next_time + key
            int any = 0;
            uint64_t kmin = CL ? cl_step_min(key, any, sh, par, xk) : gmin_key<CL>(key, sh, par);
            PROF_MARK(2);                                   // step reduction (incl. barrier wait)
            // collectives completed by the previous step's pops: reserve them now (the
            // reduction's barrier made every arrival visible -- in a cluster, the full
            // barrier taken here), then re-derive the next time
            if (CL && any) gsync<CL>();
            const int nc = CL ? (any ? *c.ncomp - (MSG ? 0 : sh.ncons) : 0) : sh.ncomp;
            const int nmc = MSG ? (CL ? (any ? *c.nmcomp : 0) : sh.nmcomp) : 0;
            if (nc | nmc) {
                if ((CL || FL_RS1) && tid == 0) sh.fifo_empty = s.head_e == TINF;   // (identical for every rank when uniform)
                const int64_t ef = reserve_n<MSG, CL, K>(g, o, c, sh, par, tcur, false, cfg, f.epoch, nc, nmc,
                                                         topo, sh.pcols);
                if (active) refresh_ring(c, L, s);
                if ((CL || FL_RS1) && ef >= 0) {
                    // every rank's next event only gained the same new FIFO head (if its FIFO was
                    // empty), so the step minimum follows without another reduction; rank 0 is
                    // the lowest rank holding it
                    if (sh.fifo_empty) {
                        const uint64_t k = (uint64_t)(ef < TCAP ? ef : TCAP) << 14;
                        kmin = k < kmin ? k : kmin;
                    }
                } else {
                    nt = active ? next_time(g, c, L, s, tcur) : TINF;
                    key = nt == TINF ? KINF : ((uint64_t)(nt < TCAP ? nt : TCAP) << 14) | (uint64_t)L.r;
                    kmin = CL ? cl_step_min(key, any, sh, par, xk) : gmin_key<CL>(key, sh, par);
                }
            }
            if (kmin == KINF) break;
            const int64_t t = (int64_t)(kmin >> 14);
            const int rmin = (int)(kmin & 0x3fff);
            // (a lean launch has fewer pops per point than the 25-bit step field holds, and every step pops)
            if (t >= TCAP || (!lean<K>() && f.step >= (1ull << 25) - 2)) { overflow = true; break; }
            PROF_MARK(3);                                   // reservations
            // (a lean point has no zero-length node, so every step lies past the last one)
            if ((lean<K>() && FL_LEAN_STEP) || t > tcur) {
                if (active) advance(g, c, L, s, tcur, t);
                tcur = t;
            }
            f.step++;
            PROF_MARK(4);                                   // advance
            if (nohost<K>() || !zero) {                 // (lean: no serial mode, see above)
                if (active) {
                    gather_due(g, c, L, s, t);
                    PROF_MARK(5);                           // gather_due
                    if (L.r > rmin) start_phase(g, o, c, L, s, f, t, cfg);
                    PROF_MARK(6);                           // tie start phase
                    s.pop_seq = 0;
                    while (s.due.head >= 0) {
                        int64_t fx;
                        const int x = ms_pop_cp<K, F_DUE_CP, F_DUE_SUM>(s.due, c.due, c.cp, R, L, fx, g.max_words);
                        pop_event(g, c, L, s, f, x, fx, t);
                        PROF_MARK(7);                       // pop_event
                        start_phase(g, o, c, L, s, f, t, cfg);
                        PROF_MARK(8);                       // start phase after a pop
                    }
                }
            } else {
                // serial mode: the reference loop verbatim, one pop per iteration
                if (active) gather_due(g, c, L, s, t);
                for (;;) {
                    const uint64_t k2 = (active && s.due.head >= 0) ? (((uint64_t)L.r << 16) | (uint64_t)ms_min(s.due))
                                                                     : KINF;
                    const uint64_t m2 = gmin_key<CL>(k2, sh, par);
                    if (m2 == KINF) break;
                    f.step++;
                    if (active && (int)(m2 >> 16) == L.r) {
                        s.pop_seq = 0;
                        int64_t fx;
                        const int x = ms_pop_cp<K, F_DUE_CP, F_DUE_SUM>(s.due, c.due, c.cp, R, L, fx, g.max_words);
                        pop_event(g, c, L, s, f, x, fx, t);
                    }
                    if (active) start_phase(g, o, c, L, s, f, t, cfg);
                    reserve<MSG, CL, KK>(g, o, c, sh, par, t, false, cfg, f.epoch, topo,
                                                       sh.pcols);
                            if (active) {
                        refresh_ring(c, L, s);
                        gather_due(g, c, L, s, t);
                    }
                }
            }
        }
        if (active) advance(g, c, L, s, tcur, TINF);
#ifdef FL_PROFILE
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&fl_prof[15], 1ull);
        if (blockIdx.x == 0 && threadIdx.x == 0 && cfg + ncl >= p.n) {
            printf("FLPROF points %llu steps(last point) %llu zero %d fold %d", fl_prof[15],
                   (unsigned long long)f.step, zero, f.fold);
            for (int k = 0; k < 15; k++) printf(" s%d %llu", k, fl_prof[k]);
            printf("\n");
        }
#endif

        // ---- row: reductions over ranks (cli.py:336-341) ----
        overflow |= gor<CL>(sh.seq_ovf, sh, par) != 0;
        int dead = active && F32<K>(Q_DONE, tid) != F32<K>(Q_MYN, tid);
        dead = gor<CL>(dead | overflow, sh, par);
        dirty = dead != 0;
        int64_t vals[6] = {0, 0, 0, 0, 0, 0};
        if (active) {
            const int64_t comm = s.commcum, cpx = F64<K>(F_CPMAX, tid);
            vals[0] = F64<K>(F_FIN, tid);
            vals[1] = cpx;
            vals[2] = RF<KK>(s, F_COMP, tid);
            vals[3] = comm;
            vals[4] = comm - RF<KK>(s, F_OVL, tid);
            vals[5] = RF<KK>(s, F_PEAK, tid);
            if (o.rank_stats) {
                int64_t *rs = o.rank_stats + ((size_t)cfg * R + L.r) * 5;
                rs[0] = vals[0]; rs[1] = vals[2]; rs[2] = vals[3]; rs[3] = vals[4]; rs[4] = vals[5];
            }
        }
        int64_t cpbest = 0;
#pragma unroll
        for (int k = 0; k < 6; k++) {
            const int64_t v = gmax_i64<CL>(vals[k], sh, par);
            if (k == 1) cpbest = v;
            if (is_leader) o.rows[(size_t)cfg * 6 + k] = v;
        }
        if (is_leader) o.status[cfg] = overflow ? FL_ERR_CAPACITY : dead ? FL_ERR_DEADLOCK : FL_OK;
        if (!lean<K>() && o.trace_len) {
            // the sink's rank: the lowest one whose largest critical-path finish is the point's
            uint64_t rk = (active && F64<K>(F_CPMAX, tid) == cpbest) ? (uint64_t)L.r : KINF;
            rk = gmin_key<CL>(rk, sh, par);
            gsync<CL>();                                // (cluster: every CTA's finishes visible)
            if (!CL || crank == 0) {
                if (dead || rk == KINF) { if (tid == 0) o.trace_len[cfg] = 0; }
                else trace_walk(g, o, c, sh, par, cfg, (int)rk, cpbest);
            }
        }
        if (o.link_busy && crank == 0)   // SimReport.link_busy_ns (simulator.py:321, :367)
            for (int l = tid; l < o.link_cap; l += bd)
                o.link_busy[(size_t)cfg * o.link_cap + l] = (g.n_msg && l < c.link_cap) ? c.link_busy[l] : -1;
        gsync<CL>();
    }
}

// ------------------------------------------------ standalone critical path

// critical_path (simulator.py:400-460) without the simulation: the longest path
// through the merged multi-rank graph in a host-computed topological order.
// Only needed when the simulation itself deadlocks: a SEND completes in the
// simulation only once its RECV is ready (simulator.py:259-268), a wait the
// contention-free bound does not have.  One thread per design point.
//   vertex v: vkind 0 = (rank va, local node vb), 1 = collective instance va;
//   vsend[v] >= 0 for a RECV: the vertex of its SEND, vmsg[v] the message.
#if FL_COMMON
__global__ void cp_kernel(const __grid_constant__ DevGraph g, const __grid_constant__ DevPoints p, int nv,
                          const int32_t *order, const int32_t *vkind, const int32_t *va, const int32_t *vb,
                          const int32_t *vsend, const int32_t *vmsg, const int32_t *poff, const int32_t *pidx,
                          int64_t *vals, int64_t *starts, int64_t *out, int32_t *status) {
    const int cfg = blockIdx.x * blockDim.x + threadIdx.x;
    if (cfg >= p.n) return;
    int64_t *cv = vals + (size_t)cfg * nv;
    int64_t *sv = starts ? starts + (size_t)cfg * nv : nullptr;   // start times, for the node trace
    const int topo = p.topo_kind[cfg], cols = p.cols[cfg];
    const double beta = __ddiv_rn(1e9, p.bw[cfg]);
    int64_t best = 0;
    int st = FL_OK;
    for (int q = 0; q < nv; q++) {
        const int v = order[q];
        if (v < 0) break;                           // order is padded with -1 past the live vertices
        int64_t x = 0;
        for (int u = poff[v]; u < poff[v + 1]; u++) x = cv[pidx[u]] > x ? cv[pidx[u]] : x;   // :449
        if (vkind[v] == 1) {                        // collective: union of the members' deps (:419-428)
            const int64_t d = coll_time(g, va[v], p.algo[cfg], topo, p.bw[cfg], p.latency[cfg], p.rows[cfg], cols);
            if (d < 0) { st = FL_ERR_UNSUPPORTED_ALGO; break; }
            if (sv) sv[v] = x;
            x += d;
        } else {
            const int gn = g.s_node_off[g.rank_struct[va[v]]] + vb[v];
            if (vsend[v] >= 0) {                    // RECV waits for its SEND plus the wire (:450-452)
                const int m = vmsg[v];
                const int64_t w = cv[vsend[v]] + transfer_ns(g, topo, cols, g.msg_send_rank[m], g.msg_recv_rank[m],
                                                             g.msg_bytes[m], p.latency[cfg], beta);
                x = w > x ? w : x;
            }
            int64_t d = g.node_dur[gn];
            if (p.peak_flops && g.node_flops[gn] >= 0) d = flops_to_ns(g.node_flops[gn], p.peak_flops[cfg], p.efficiency[cfg]);
            if (sv) sv[v] = x;
            if ((g.node_rec[2 * gn + 1].x & 15u) <= FL_COMP) x += d;   // `duration_ns or 0`
        }
        cv[v] = x;
        best = x > best ? x : best;
    }
    out[cfg] = best;
    status[cfg] = st;
}
#endif

// ------------------------------------------------------------ host side

template <int T>
static cudaError_t launch_t(int grid, int block, size_t smem, cudaStream_t st, int cluster, const DevGraph &g,
                            const DevPoints &p, const DevOut &o, const DevScratch &sc) {
    if constexpr (((T >> 5) & 3) != 0) {     // narrow planes: single-CTA design points only
        sweep_kernel<T, false><<<grid, block, smem, st>>>(g, p, o, sc);
        return cudaGetLastError();
    } else {
    if (cluster <= 1) {
        sweep_kernel<T, false><<<grid, block, smem, st>>>(g, p, o, sc);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, sweep_kernel<T, true>, g, p, o, sc);
    }
}

static inline int plane_class(int block) { return block > 256 ? 0 : block > 64 ? 1 : 2; }
static inline int plane_lanes_for(int block) { return block > 256 ? 1024 : block > 64 ? 256 : 64; }

// The variants are compiled in eight translation units (-DFL_BASE = compute streams | 8 with
// messages), each holding its three plane widths and its cluster variant.
#define FL_PART_DECL(B)                                                                                     \
    cudaError_t launch_sweep_b##B(int T, int grid, int block, size_t smem, cudaStream_t st, int cluster,   \
                                  const DevGraph &g, const DevPoints &p, const DevOut &o, const DevScratch &sc); \
    cudaError_t set_smem_b##B(size_t smem);
FL_PART_DECL(1) FL_PART_DECL(2) FL_PART_DECL(4) FL_PART_DECL(9) FL_PART_DECL(10) FL_PART_DECL(12)
FL_PART_DECL(512) FL_PART_DECL(520)

#define FL_PART_DEF(B)                                                                                      \
    cudaError_t launch_sweep_b##B(int T, int grid, int block, size_t smem, cudaStream_t st, int cluster,   \
                                  const DevGraph &g, const DevPoints &p, const DevOut &o, const DevScratch &sc) { \
        switch (T) {                                                                                        \
            case B: return launch_t<B>(grid, block, smem, st, cluster, g, p, o, sc);                        \
            case B + 32: return launch_t<B + 32>(grid, block, smem, st, cluster, g, p, o, sc);              \
            case B + 64: return launch_t<B + 64>(grid, block, smem, st, cluster, g, p, o, sc);              \
            default: return cudaErrorInvalidValue;                                                          \
        }                                                                                                   \
    }                                                                                                       \
    cudaError_t set_smem_b##B(size_t smem) {                                                                \
        cudaError_t e = cudaSuccess;                                                                        \
        const cudaFuncAttribute A = cudaFuncAttributeMaxDynamicSharedMemorySize;                            \
        if (e == cudaSuccess) e = cudaFuncSetAttribute(sweep_kernel<B, false>, A, (int)smem);               \
        if (e == cudaSuccess) e = cudaFuncSetAttribute(sweep_kernel<B + 32, false>, A, (int)smem);          \
        if (e == cudaSuccess) e = cudaFuncSetAttribute(sweep_kernel<B + 64, false>, A, (int)smem);          \
        if (e == cudaSuccess) e = cudaFuncSetAttribute(sweep_kernel<B, true>, A, (int)smem);                \
        if (e == cudaSuccess)                                                                               \
            e = cudaFuncSetAttribute(sweep_kernel<B, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); \
        return e;                                                                                           \
    }

#if FL_BASE == 0 || FL_BASE == 1
FL_PART_DEF(1)
#endif
// Lean variants (lean<K>, "bit 7"), all in the FL_BASE 1 unit: one compute stream, no messages,
// 1024-lane planes (single CTA and cluster) and the narrow planes with the bitmap and slot table
// in shared memory.  A/B (scripts/ab.py, FL_LEAN=0): C3 +5.3%, C2 +4.8%, C4 +4.4-4.7%; the same
// specialization of the message variants gained nothing on the expanded workloads.
#define FL_LEAN_LIST1(X) X(1 + 128) X(1 + 64 + 128 + 256) X(1 + 32 + 128 + 256)
// (the cluster variant of 1 + 128 lives in the FL_BASE 1 unit)
#define FL_LEAN_CLUSTER1 (T == 1 + 128 ? launch_t<1 + 128>(grid, block, smem, st, cluster, g, p, o, sc) : cudaErrorInvalidValue)
#define FL_LEAN_CLUSTER_SMEM1                                                                               \
    if (e == cudaSuccess) e = cudaFuncSetAttribute(sweep_kernel<1 + 128, true>, A, (int)smem);              \
    if (e == cudaSuccess)                                                                                   \
        e = cudaFuncSetAttribute(sweep_kernel<1 + 128, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
#define FL_LEAN_CASE(T) case T: sweep_kernel<T, false><<<grid, block, smem, st>>>(g, p, o, sc); return cudaGetLastError();
#define FL_LEAN_SMEM(T) if (e == cudaSuccess) e = cudaFuncSetAttribute(sweep_kernel<T, false>, A, (int)smem);
#define FL_LEAN_DEF(U)                                                                                      \
    cudaError_t launch_sweep_lean##U(int T, int grid, int block, size_t smem, cudaStream_t st, int cluster,  \
                                     const DevGraph &g, const DevPoints &p, const DevOut &o, const DevScratch &sc) { \
        if (cluster > 1) return FL_LEAN_CLUSTER##U;                                                         \
        switch (T) { FL_LEAN_LIST##U(FL_LEAN_CASE) default: return cudaErrorInvalidValue; }                 \
    }                                                                                                       \
    cudaError_t set_smem_lean##U(size_t smem) {                                                             \
        cudaError_t e = cudaSuccess;                                                                        \
        const cudaFuncAttribute A = cudaFuncAttributeMaxDynamicSharedMemorySize;                            \
        FL_LEAN_LIST##U(FL_LEAN_SMEM)                                                                       \
        FL_LEAN_CLUSTER_SMEM##U                                                                             \
        return e;                                                                                           \
    }
#define FL_LEAN_DECL(U)                                                                                     \
    cudaError_t launch_sweep_lean##U(int T, int grid, int block, size_t smem, cudaStream_t st, int cluster,  \
                                     const DevGraph &g, const DevPoints &p, const DevOut &o, const DevScratch &sc); \
    cudaError_t set_smem_lean##U(size_t smem);
FL_LEAN_DECL(1)
#if FL_BASE == 0 || FL_BASE == 1
FL_LEAN_DEF(1)
#endif
#if FL_BASE == 0 || FL_BASE == 2
FL_PART_DEF(2)
#endif
#if FL_BASE == 0 || FL_BASE == 4
FL_PART_DEF(4)
#endif
#if FL_BASE == 0 || FL_BASE == 9
FL_PART_DEF(9)
#endif
#if FL_BASE == 0 || FL_BASE == 10
FL_PART_DEF(10)
#endif
#if FL_BASE == 0 || FL_BASE == 12
FL_PART_DEF(12)
#endif
#if FL_BASE == 0 || FL_BASE == 512
FL_PART_DEF(512)
#endif
#if FL_BASE == 0 || FL_BASE == 520
FL_PART_DEF(520)
#endif

#if FL_COMMON
cudaError_t launch_sweep(int K, int grid, int block, size_t smem, cudaStream_t st, int cluster, const DevGraph &g,
                         const DevPoints &p0, const DevOut &o, const DevScratch &sc, int *launches,
                         bool defer_retry, bool *deferred) {
    // variant word: compute streams (1, 2, 4; 512: 8) | 8 when the graphs carry SEND/RECV | plane class << 5
    const int B = K | (g.n_msg > 0 ? 8 : 0);
    DevPoints p = p0;
    if (launches) *launches = 1;
    if (deferred) *deferred = false;
    // the lean variant when the run needs none of the branches it drops (bits 7, 8): then the
    // general variant runs a second pass over the points the lean one left (FL_RETRY), which
    // exits at once when there are none
    if (!p0.retry && FL_LEAN && B == 1 && !o.ev_start && !o.trace_len && g.dur_sm_off && sc.touch_in_smem == sc.acc_in_smem &&
        g.fold_ok && !g.dyn_host && (cluster > 1 || !FL_LEAN_FULL || block == g.R) && g.max_nodes <= 8191 &&
        (long long)g.R * g.max_nodes < (1 << 25) - 8) {
        const int pc = cluster > 1 ? 0 : plane_class(block);
        const int TL = B | pc << 5 | 128 | (sc.touch_in_smem ? 256 : 0);
        const unsigned doff = TL == 1 + 128 ? dur_off<1 + 128>() : TL == 1 + 64 + 128 + 256 ? dur_off<1 + 64 + 128 + 256>()
                                                                                           : dur_off<1 + 32 + 128 + 256>();
        if ((TL == 1 + 128 || (cluster <= 1 && (TL == 1 + 64 + 128 + 256 || TL == 1 + 32 + 128 + 256))) &&
            g.dur_sm_off == doff) {
            const cudaError_t e = launch_sweep_lean1(TL, grid, block, smem, st, cluster, g, p, o, sc);
            if (e != cudaSuccess || defer_retry) {
                if (deferred) *deferred = e == cudaSuccess;
                return e;
            }
            p.retry = 1;
            if (launches) *launches = 2;
        }
    }
    const int T = B | (cluster > 1 ? 0 : plane_class(block) << 5);
    switch (B) {
        case 1: return launch_sweep_b1(T, grid, block, smem, st, cluster, g, p, o, sc);
        case 2: return launch_sweep_b2(T, grid, block, smem, st, cluster, g, p, o, sc);
        case 4: return launch_sweep_b4(T, grid, block, smem, st, cluster, g, p, o, sc);
        case 9: return launch_sweep_b9(T, grid, block, smem, st, cluster, g, p, o, sc);
        case 10: return launch_sweep_b10(T, grid, block, smem, st, cluster, g, p, o, sc);
        case 12: return launch_sweep_b12(T, grid, block, smem, st, cluster, g, p, o, sc);
        case 512: return launch_sweep_b512(T, grid, block, smem, st, cluster, g, p, o, sc);
        case 520: return launch_sweep_b520(T, grid, block, smem, st, cluster, g, p, o, sc);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t sweep_occupancy(int block, size_t smem, int cluster, int *occ) {
    if (cluster <= 1) {
        const int pc = plane_class(block);
        return pc == 0 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, sweep_kernel<1, false>, block, smem)
             : pc == 1 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, sweep_kernel<33, false>, block, smem)
                       : cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, sweep_kernel<65, false>, block, smem);
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cluster);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaOccupancyMaxActiveClusters(occ, sweep_kernel<1, true>, &cfg);   // clusters, not blocks
}

cudaError_t sweep_set_smem(size_t smem) {
    cudaError_t e = set_smem_b1(smem);
    if (e == cudaSuccess) e = set_smem_lean1(smem);
    if (e == cudaSuccess) e = set_smem_b2(smem);
    if (e == cudaSuccess) e = set_smem_b4(smem);
    if (e == cudaSuccess) e = set_smem_b9(smem);
    if (e == cudaSuccess) e = set_smem_b10(smem);
    if (e == cudaSuccess) e = set_smem_b12(smem);
    if (e == cudaSuccess) e = set_smem_b512(smem);
    if (e == cudaSuccess) e = set_smem_b520(smem);
    return e;
}

size_t sweep_shared_header_bytes() { return SM_HDR; }
size_t sweep_shared_bytes_per_rank(bool msg) { return 8 * F_N64 + 4 * Q_ALL + (msg ? 8 * MF_N64 + 4 : 0); }   // x plane lanes
int sweep_plane_lanes(int block, int cluster) { return cluster > 1 ? 1024 : plane_lanes_for(block); }

cudaError_t launch_cp(const DevGraph &g, const DevPoints &p, int nv, const int32_t *order, const int32_t *vkind,
                      const int32_t *va, const int32_t *vb, const int32_t *vsend, const int32_t *vmsg,
                      const int32_t *poff, const int32_t *pidx, int64_t *vals, int64_t *starts, int64_t *out,
                      int32_t *status) {
    cp_kernel<<<(p.n + 127) / 128, 128>>>(g, p, nv, order, vkind, va, vb, vsend, vmsg, poff, pidx, vals, starts, out,
                                          status);
    return cudaGetLastError();
}

// Deterministic topological order of each structure (graph.py:282-306: Kahn's
// algorithm, lowest node_id first -- local index order is node_id order) and every
// node's level (longest path from a source, in edges).  One warp per structure: the
// ready set is a bitmap whose lowest set bit is found with ballots; a node's
// successors are released in parallel.  order[s_node_off[s] + k] is the k-th node
// (local index), -1 past the placed ones when the structure has a cycle.
__global__ void topo_kernel(const __grid_constant__ DevGraph g, int32_t *indeg, int32_t *order, int32_t *level) {
    extern __shared__ uint64_t ready[];
    const int s = blockIdx.x, lane = threadIdx.x;
    const int nb = g.s_node_off[s], n = g.s_node_off[s + 1] - nb, W = (n + 63) / 64;
    for (int v = lane; v < n; v += 32) {
        indeg[nb + v] = g.pred_off[nb + v + 1] - g.pred_off[nb + v];
        level[nb + v] = 0;
        order[nb + v] = -1;
    }
    for (int w = lane; w < W; w += 32) {
        uint64_t word = 0;
        for (int b = 0; b < 64 && 64 * w + b < n; b++)
            if (g.pred_off[nb + 64 * w + b + 1] == g.pred_off[nb + 64 * w + b]) word |= 1ull << b;
        ready[w] = word;
    }
    __syncwarp();
    for (int k = 0; k < n; k++) {
        int v = -1;
        for (int w0 = 0; w0 < W && v < 0; w0 += 32) {
            const uint64_t word = w0 + lane < W ? ready[w0 + lane] : 0ull;
            const unsigned bal = __ballot_sync(FULL, word != 0ull);
            if (bal) {
                const int src = __ffs(bal) - 1;
                const uint64_t wv = __shfl_sync(FULL, word, src);
                v = 64 * (w0 + src) + __ffsll((long long)wv) - 1;
            }
        }
        if (v < 0) break;                           // cycle: nothing ready
        __syncwarp();
        if (lane == 0) {
            atomicAnd(reinterpret_cast<unsigned long long *>(&ready[v >> 6]), ~(1ull << (v & 63)));
            order[nb + k] = v;
        }
        __syncwarp();
        const int lv = level[nb + v] + 1;
        for (int q = g.succ_off[nb + v] + lane; q < g.succ_off[nb + v + 1]; q += 32) {
            const int w = g.succ_idx[q];
            atomicMax(&level[nb + w], lv);
            if (atomicSub(&indeg[nb + w], 1) == 1) atomicOr(reinterpret_cast<unsigned long long *>(&ready[w >> 6]),
                                                            1ull << (w & 63));
        }
        __syncwarp();
    }
}

cudaError_t launch_topo(const DevGraph &g, int32_t *indeg_ws, int32_t *order, int32_t *level) {
    const size_t smem = (size_t)g.max_words * 8;
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(topo_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    topo_kernel<<<g.S, 32, smem>>>(g, indeg_ws, order, level);
    return cudaGetLastError();
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
#endif  // FL_COMMON

}  // namespace fl
