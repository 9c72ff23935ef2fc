// engine_internal.h -- device-side views shared by engine.cu and capi.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fl {

// internal status of a point the lean variant left to the general one (never returned)
constexpr int FL_RETRY = 0x7f;
enum { FL_EDGE_COUNTED = 0, FL_EDGE_SINGLE = 1, FL_EDGE_FIRST = 2, FL_EDGE_MID = 3, FL_EDGE_LAST = 4 };

// Device copy of fl_graph_desc (pointers are device pointers).
struct DevGraph {
    int R, S, n_inst, coll_stride, max_nodes, max_words, total_nodes, total_tens, n_succ;
    const int32_t *rank_struct;
    const int32_t *s_node_off, *s_tens_off, *s_init_off, *s_ncoll;
    const int64_t *s_init_alloc;
    const uint8_t *node_kind, *node_flags;
    const int64_t *node_dur, *node_flops, *node_alloc;
    const int32_t *node_coll_ord, *pred_off, *pred_idx, *succ_off, *succ_idx, *free_off, *free_tens, *init_list;
    const int64_t *tens_bytes;
    const int32_t *tens_cons_off, *tens_cons;
    const uint8_t *inst_kind;
    const int32_t *inst_n;
    const int64_t *inst_bytes, *inst_lead_id, *inst_init_key, *inst_mem_off;
    const int32_t *inst_mem_rank, *inst_mem_node, *rank_coll_inst;
    const int32_t *inst_full_node;   // >= 0 when members are ranks 0..R-1 in order, all at this local node
    // derived on upload (capi.cu): packed per-node records and tensor consumer ranges
    const uint4 *node_rec;       // [2 * total_nodes] (engine.cu "Node record")
    const int32_t *mfree_off;    // [total_nodes] first entry in free_tens of a node's shared-tensor frees
    const int2 *tens_rng;        // [total_tens] {first, end} into tens_cons
    // static-host folding (engine.cu "t = 0 host pops")
    int fold_ok;
    int dyn_host;                // some HOST node is not a static host (it can run on the host stream)
    int needs_done;              // some tensor's last consumer is only known at run time
    const int32_t *s_nstatic, *trig_off, *static_off, *static_list;
    const int32_t *s_nsink;      // per structure: nodes without successors, static hosts excluded
    const int4 *trig;            // {trigger host, node, position in the host's dependents, -}
    unsigned dur_sm_off;         // per-point durations in shared memory at this offset (0: HBM, per CTA)
    const int32_t *s_init_ns_off, *init_ns;   // initial dispatch list without static hosts
    const int32_t *succ_ent;     // succ_idx | edge class << 16 (FL_EDGE_*, valid when static hosts are folded)
                                 // | accumulator slot << 19 (FIRST / MID / LAST edges, capi.cu "slots")
    int n_acc;                   // accumulator slots per rank (colouring of the ordered multi-dependency nodes)
    // messages
    const int64_t *rank_value;
    int n_msg, p2p_stride;
    const int32_t *msg_send_rank, *msg_send_node, *msg_recv_rank, *msg_recv_node, *rank_p2p_msg;
    const int64_t *msg_bytes, *msg_send_id;
    const int32_t *msg_ord;      // [M] position in (source rank id, SEND node_id) order (simulator.py:311)
    int msg_self;                // some message has the same source and destination rank (zero wire time)
    int64_t msg_min_bytes;       // smallest message
};

struct DevPoints {
    int n;
    const uint8_t *algo, *topo_kind;
    const double *bw;
    const int64_t *latency;
    const int32_t *rows, *cols;
    const double *peak_flops, *efficiency;
    int compute_streams;
    int retry;                   // second pass after a lean launch: only points whose status is FL_RETRY
};

struct DevOut {
    int32_t *status;
    int64_t *rows, *rank_stats, *ev_start, *ev_end, *link_busy;
    int link_cap;
    int64_t *trace;              // critical-path node trace (flint_b200.h fl_outputs.trace)
    int32_t *trace_len;
    int trace_cap;
};

// Per-CTA scratch: slot_bytes each, laid out at the given byte offsets.
struct DevScratch {
    unsigned char *base;
    size_t slot_bytes, off_bits, off_cp, off_ring, off_dur, off_inst;
    size_t off_acc;              // [n_acc][R] int64: accumulators of statically ordered nodes, by slot
    // dynamic shared-memory layout (bytes from the start of the CTA's smem)
    size_t off_msg;              // message state, per-rank in-flight lists
    size_t off_mlist_se;         // [2][p2p_stride][R] int64: in-flight entries' wire start / end
    size_t off_links;            // link state [3][link_cap]: free-at, busy, message-phase claim (last in the slot: grows per launch)
    size_t off_ctr;              // cluster-wide completion counters
    size_t off_inst_se;          // clusters: per-CTA copies of the instances' reservation start / end
    int link_cap;
    unsigned sm_off_dyn, sm_off_done, sm_off_dur, sm_off_inst, sm_off_touch, sm_off_acc, sm_off_links;
    int done_in_smem, dur_in_smem, inst_in_smem, touch_in_smem, acc_in_smem;
    int links_in_smem;           // the link table is in the (lead) CTA's shared memory (per launch: it grows)
};

// p.retry = 1: only the general variant's second pass (points whose status is FL_RETRY).
// defer_retry: after a lean launch, leave the second pass to the caller (*deferred = true),
// which launches it with p.retry = 1 only if a status it read back is FL_RETRY.
cudaError_t launch_sweep(int K, int grid, int block, size_t smem, cudaStream_t st, int cluster, const DevGraph &g,
                         const DevPoints &p, const DevOut &o, const DevScratch &sc, int *launches,
                         bool defer_retry = false, bool *deferred = nullptr);
cudaError_t sweep_occupancy(int block, size_t smem, int cluster, int *occ);
cudaError_t sweep_set_smem(size_t smem);
size_t sweep_shared_header_bytes();
size_t sweep_shared_bytes_per_rank(bool msg);   // the [field][blockDim] per-rank planes (msg: + message summaries)
int sweep_plane_lanes(int block, int cluster);   // per-rank planes are this many lanes wide
cudaError_t launch_cp(const DevGraph &g, const DevPoints &p, int nv, const int32_t *order, const int32_t *vkind,
                      const int32_t *va, const int32_t *vb, const int32_t *vsend, const int32_t *vmsg,
                      const int32_t *poff, const int32_t *pidx, int64_t *vals, int64_t *starts, int64_t *out,
                      int32_t *status);
cudaError_t launch_topo(const DevGraph &g, int32_t *indeg_ws, int32_t *order, int32_t *level);
cudaError_t launch_cost_only(int n, const uint8_t *kind, const int64_t *size, const int64_t *gn,
                             const uint8_t *algo, const double *alpha, const double *beta,
                             const int32_t *rows, const int32_t *cols, int64_t *out, int32_t *status,
                             int m, const int64_t *flops, const double *peak, const double *eff,
                             int64_t *out_comp);

}  // namespace fl
