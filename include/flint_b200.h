/*
 * flint_b200.h -- C-ABI of the B200 sweep engine (libflint_b200.so).
 *
 * The reference (arxiv 2604.17550 "Flint", package trainsim) is pure Python
 * and has no FFI; its hot path is three Python functions that this ABI
 * replaces for a whole batch of design points at once:
 *
 *   simulate(graphs, topo, opts) -> SimReport     pkg/src/trainsim/simulator.py:203-367
 *   critical_path(graphs, topo, algo) -> int      pkg/src/trainsim/simulator.py:400-460
 *   _sweep_row(task) -> dict (one CSV row)        pkg/src/trainsim/cli.py:319-342
 *
 * plus their cost models analytical_time (collectives.py:251-293) and
 * analytical_duration (traceio.py:163-184).  The binding a maintainer adds on
 * the reference side is ctypes; plain pointers and sizes
 * only, no torch types.
 *
 * Life cycle: fl_graph_create() uploads one compiled set of per-rank graphs
 * (CSR, instance tables) to a device and returns an opaque handle;
 * fl_sweep_run() / fl_sweep_run_device() evaluate any number of design
 * points against it; fl_graph_destroy() frees it.  Handles are independent
 * (no global mutable state besides the thread-local last-error string).
 *
 * Every function returns an FL_* status; per-design-point statuses are
 * written to fl_outputs.status.  The Python layer maps FL_ERR_DEADLOCK,
 * FL_ERR_UNSUPPORTED_ALGO and FL_ERR_INCONSISTENT to the reference's
 * DeadlockError, UnsupportedAlgoTopologyError and InconsistentGroupsError.
 */
#ifndef FLINT_B200_H
#define FLINT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FL_ABI_VERSION 3

enum fl_status {
    FL_OK = 0,
    FL_ERR_INVALID = 1,          /* malformed descriptor / argument            */
    FL_ERR_CUDA = 2,             /* CUDA runtime failure (no GPU, launch, OOM) */
    FL_ERR_DEADLOCK = 3,         /* simulator.py:329-333, :459                 */
    FL_ERR_UNSUPPORTED_ALGO = 4, /* collectives.py:274-282                     */
    FL_ERR_INCONSISTENT = 5,     /* collectives.py:441-449 (host-side compile) */
    FL_ERR_CAPACITY = 6,         /* graph exceeds this build's engine limits   */
    FL_ERR_NOT_RUN = 7           /* row belongs to another GPU's slice         */
};

enum fl_node_kind { FL_HOST = 0, FL_COMP = 1, FL_COLL = 2, FL_SEND = 3, FL_RECV = 4 };
enum fl_coll_kind { FL_ALL_REDUCE = 0, FL_ALL_GATHER = 1, FL_REDUCE_SCATTER = 2 };
enum fl_algo { FL_RING = 0, FL_TREE = 1, FL_MESH_HIER = 2 };
enum fl_topo { FL_SWITCH = 0, FL_MESH2D = 1 };

/* Engine limits of this build. */
#define FL_MAX_NODES_PER_RANK 65535  /* 16-bit local node index (set heads, dependency entries) */
#define FL_MAX_RANKS 16384           /* one thread per rank; > 1024 ranks run on a CTA cluster (<= 16) */
#define FL_MAX_P2P_PER_RANK 65535    /* SEND+RECV nodes per rank graph */

/*
 * A compiled graph set.  Ranks are dense 0..R-1 in ascending rank-value
 * order.  Each rank points at a *structure* (a distinct node list; ranks of
 * a synthesized family all share one).  Node indices inside a structure are
 * 0..N_s-1 in ascending node_id order, so "lowest ready id first"
 * (simulator.py:5-6) is "lowest index first".  Arrays marked [nodes] are
 * concatenated over structures (global node g = s_node_off[s] + local);
 * CSR payloads hold LOCAL indices.
 */
typedef struct {
    int32_t n_ranks;
    const int32_t *rank_struct;       /* [R] */
    const int32_t *rank_graph_pos;    /* [R] position of the rank in the caller's list */

    int32_t n_structs;
    const int32_t *s_node_off;        /* [S+1] */
    const int32_t *s_tens_off;        /* [S+1] */
    const int32_t *s_init_off;        /* [S+1] into init_list */
    const int64_t *s_init_alloc;      /* [S] bytes of tensors with no producer (live from t=0) */
    const int32_t *s_ncoll;           /* [S] collectives per rank of this structure */

    const uint8_t *node_kind;         /* [nodes] fl_node_kind */
    const uint8_t *node_flags;        /* [nodes] bit0: waits on a node that does not exist */
    const int64_t *node_id;           /* [nodes] original node_id (for ordering keys) */
    const int64_t *node_dur;          /* [nodes] duration_ns or 0 (HOST/COMP)  */
    const int64_t *node_flops;        /* [nodes] flops for re-costing, -1: keep node_dur */
    const int64_t *node_alloc;        /* [nodes] bytes of tensors this node produces */
    const int32_t *node_coll_ord;     /* [nodes] k-th COLL in list order, -1 otherwise */
    const int32_t *pred_off;          /* [nodes+1] global positions into pred_idx */
    const int32_t *pred_idx;          /* deduplicated dependencies (local)      */
    const int32_t *succ_off;          /* [nodes+1]                              */
    const int32_t *succ_idx;          /* dependents in the caller's list order  */
    const int32_t *free_off;          /* [nodes+1] tensors this node consumes   */
    const int32_t *free_tens;         /* local tensor indices                   */
    const int32_t *init_list;         /* zero-indegree nodes, list order (local) */

    const int64_t *tens_bytes;        /* [tensors] */
    const int32_t *tens_cons_off;     /* [tensors+1] global positions into tens_cons */
    const int32_t *tens_cons;         /* consumers (local node indices)         */

    int32_t n_inst;                   /* collective instances (collectives.py:419-453) */
    const uint8_t *inst_kind;         /* [I] fl_coll_kind */
    const int32_t *inst_n;            /* [I] group size */
    const int64_t *inst_bytes;        /* [I] comm_bytes of the lead node */
    const int64_t *inst_lead_id;      /* [I] node_id of the lead member (sort key, simulator.py:299) */
    const int64_t *inst_init_key;     /* [I] completion order if it completes at dispatch time 0 */
    const int64_t *inst_mem_off;      /* [I+1] */
    const int32_t *inst_mem_rank;     /* members in group order: rank index */
    const int32_t *inst_mem_node;     /* member node (local index in that rank's structure) */
    int32_t coll_stride;              /* max collectives per rank (row stride below) */
    const int32_t *rank_coll_inst;    /* [R*coll_stride] instance of rank r's k-th COLL */

    /* point-to-point messages (EXPANDED comm mode), matched as simulator.py:177-200 */
    const int64_t *rank_value;        /* [R] the graphs' rank ids (routing, ordering keys) */
    int32_t n_msg;
    const int32_t *msg_send_rank, *msg_send_node;   /* [M] rank index, local node */
    const int32_t *msg_recv_rank, *msg_recv_node;
    const int64_t *msg_bytes;         /* [M] */
    const int64_t *msg_send_id;       /* [M] node_id of the SEND (order key, simulator.py:311) */
    int32_t p2p_stride;               /* max SEND+RECV per rank */
    const int32_t *rank_p2p_msg;      /* [R*p2p_stride] message of rank r's k-th SEND/RECV */
} fl_graph_desc;

/* Design points, structure of arrays, one entry per point. */
typedef struct {
    int32_t n_points;
    const uint8_t *algo;              /* fl_algo */
    const uint8_t *topo_kind;         /* fl_topo */
    const double *bw;                 /* bytes/s; beta = 1e9/bw (topology.py:49) */
    const int64_t *latency;           /* ns (alpha) */
    const int32_t *rows, *cols;       /* mesh shape (MESH_HIER) */
    const double *peak_flops;         /* NULL: keep node_dur; else re-cost COMP from flops */
    const double *efficiency;
    int32_t compute_streams;          /* SimOptions.compute_streams (1..8) */
} fl_points;

/* Results, one row per point: makespan, critical path, max compute busy,
 * max comm busy, max exposed comm, max peak memory (cli.py:336-341). */
typedef struct {
    int32_t *status;                  /* [n] */
    int64_t *rows;                    /* [n*6] */
    int64_t *rank_stats;              /* optional [n*R*5]: finish, compute, comm, exposed, peak */
    int64_t *ev_start, *ev_end;       /* optional [n*R*max_nodes] (record_events) */
    int64_t *link_busy;               /* optional [n*link_cap]; -1 = link never used (SimReport.link_busy_ns) */
    int32_t link_cap;                 /* links per point in link_busy: switch 2*R (eg/in per rank), mesh 4*rows*cols */
    /* optional critical-path node trace per point ("duration_ns and node path"; the
     * reference returns only the length, simulator.py:400-460), walked back on the device from the
     * contention-free finish times the simulation computes.  trace[n*trace_cap]: entries from the
     * sink back to the source, (rank index << 32) | local node index; trace_len[n]: the full path
     * length (entries beyond trace_cap are not stored; 0 for a point that did not complete).
     * Rule (engine.critical_path_trace): sink = largest finish, lowest (rank, node_id) on ties; a
     * node's predecessor = its lowest (rank, node_id) dependency (a collective: over all members'
     * dependencies) whose finish equals the node's start, else a RECV's SEND. */
    int64_t *trace;
    int32_t *trace_len;
    int32_t trace_cap;
} fl_outputs;

typedef struct fl_graph fl_graph;

int fl_version(void);
const char *fl_last_error(void);
int fl_device_count(int32_t *count);

/* Upload + validate; device = CUDA ordinal. */
int fl_graph_create(const fl_graph_desc *desc, int32_t device, fl_graph **out);
int fl_graph_destroy(fl_graph *g);
int32_t fl_graph_max_nodes(const fl_graph *g);

/* Host buffers in and out; synchronous.  Copies are part of the call. */
int fl_sweep_run(fl_graph *g, const fl_points *host_points, fl_outputs *host_out);

/* Device-resident points/outputs; asynchronous on `stream` (cudaStream_t,
 * NULL = legacy default).  *launches receives the number of kernels enqueued. */
int fl_sweep_run_device(fl_graph *g, const fl_points *dev_points, fl_outputs *dev_out,
                        void *stream, int32_t *launches);

/* Contention-free critical path alone (simulator.py:400-460) for host design
 * points, over the merged multi-rank graph given as vertices in topological
 * order (n_vert entries, padded with -1 after the live vertices;
 * vkind 0: rank va's node vb; 1: collective instance va; RECVs carry
 * their SEND's vertex in vsend and the message in vmsg) with predecessor CSR.
 * fl_sweep_run computes the same value as a by-product of the simulation; this
 * entry point serves critical_path() when the simulation itself deadlocks. */
int fl_critical_path(fl_graph *g, const fl_points *host_points, int32_t n_vert, const int32_t *order,
                     const int32_t *vkind, const int32_t *va, const int32_t *vb, const int32_t *vsend,
                     const int32_t *vmsg, const int32_t *pred_off, const int32_t *pred_idx,
                     int64_t *out_cp, int32_t *out_status);

/* fl_critical_path plus every vertex's contention-free finish and start times
 * (out_vals[point * n_vert + vertex] finishes, then out_vals[(n_points + point) * n_vert
 * + vertex] starts; host buffer of 2 * n_points * n_vert), from which the host derives the
 * critical-path node trace ("duration_ns and node path"; the reference
 * implementation returns only the length, simulator.py:400-460). */
int fl_critical_path_values(fl_graph *g, const fl_points *host_points, int32_t n_vert, const int32_t *order,
                            const int32_t *vkind, const int32_t *va, const int32_t *vb, const int32_t *vsend,
                            const int32_t *vmsg, const int32_t *pred_off, const int32_t *pred_idx,
                            int64_t *out_cp, int32_t *out_status, int64_t *out_vals);

/* Deterministic topological order of every structure of the graph set and each node's
 * topological level, computed on the graph's device (replaces graph.py:282-306 topo_order:
 * Kahn's algorithm, lowest node_id first).  out_order[s_node_off[s] + k] = local index of
 * the k-th node of structure s (-1 past the placed nodes when the structure has a cycle ->
 * CyclicGraphError); out_level[global node] = longest path from a zero-indegree node, in
 * edges.  Host buffers of total nodes each; synchronous. */
int fl_topo_order(fl_graph *g, int32_t *out_order, int32_t *out_level);

/* Cost stage alone (K1 parity hook): alpha-beta time of n collectives and
 * flops->ns of m compute nodes, evaluated by the device code path. Host buffers. */
int fl_cost_only(int32_t n, const uint8_t *kind, const int64_t *size_bytes,
                 const int64_t *group_n, const uint8_t *algo, const double *alpha,
                 const double *beta, const int32_t *rows, const int32_t *cols,
                 int64_t *out_ns, int32_t *out_status,
                 int32_t m, const int64_t *flops, const double *peak, const double *eff,
                 int64_t *out_comp_ns);

#ifdef __cplusplus
}
#endif
#endif /* FLINT_B200_H */
