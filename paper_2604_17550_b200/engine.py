"""Reference-facing API over the CUDA engine.

Drop-in replacements for the reference's hot-path functions, same names,
argument meaning and exceptions:

* :func:`simulate` -- ``trainsim.simulate`` (pkg/src/trainsim/simulator.py:203-367)
* :func:`critical_path` -- ``trainsim.critical_path`` (simulator.py:400-460)

plus the batched entry point the reference lacks, :func:`simulate_batch`
(one compiled graph set x N design points -> N sweep rows), and
:class:`Engine`, a graph set resident on one GPU.

Every call runs on the GPU through ``libflint_b200.so``; there is no CPU
path.  Results are bit-identical to the reference (tests/test_gpu_parity.py).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _native
from .costs import CollectiveAlgo
from .errors import (EngineError, FL_ERR_NOT_RUN, FL_OK, raise_for_status)
from .store import GraphSet, check_supported, compile_graphs, desc_arrays

ALGO = {"ring": 0, "tree": 1, "mesh-hier": 2}
ROW_FIELDS = ("makespan_ns", "critical_path_ns", "compute_busy_ns", "comm_busy_ns",
              "exposed_comm_ns", "peak_mem_bytes")


def _ev(x):
    return x.value if hasattr(x, "value") else x


# ------------------------------------------------------------ report types
# (simulator.py:45-106)


@dataclass
class SimOptions:
    algo: CollectiveAlgo = CollectiveAlgo.RING
    compute_streams: int = 1
    comm_streams: int = 1
    record_events: bool = True


@dataclass
class TraceEvent:
    rank: int
    node_id: int
    stream: str
    op_name: str
    start_ns: int
    end_ns: int


@dataclass
class RankStats:
    finish_ns: int = 0
    compute_busy_ns: int = 0
    comm_busy_ns: int = 0
    exposed_comm_ns: int = 0
    peak_mem_bytes: int = 0


@dataclass
class SimReport:
    makespan_ns: int
    ranks: dict
    link_busy_ns: dict = field(default_factory=dict)
    events: list = field(default_factory=list)

    @property
    def exposed_comm_ns(self) -> int:
        return max((s.exposed_comm_ns for s in self.ranks.values()), default=0)

    @property
    def peak_mem_bytes(self) -> int:
        return max((s.peak_mem_bytes for s in self.ranks.values()), default=0)

    def to_doc(self) -> dict:
        return {
            "format_version": "sim-trace/1",
            "makespan_ns": self.makespan_ns,
            "ranks": {str(r): {"finish_ns": s.finish_ns, "compute_busy_ns": s.compute_busy_ns,
                               "comm_busy_ns": s.comm_busy_ns, "exposed_comm_ns": s.exposed_comm_ns,
                               "peak_mem_bytes": s.peak_mem_bytes}
                      for r, s in sorted(self.ranks.items())},
            "links": dict(sorted(self.link_busy_ns.items())),
            "events": [{"rank": e.rank, "node_id": e.node_id, "stream": e.stream, "op": e.op_name,
                        "start_ns": e.start_ns, "end_ns": e.end_ns} for e in self.events],
        }


# ------------------------------------------------------------ design points


@dataclass
class DesignPoints:
    """Structure-of-arrays design points (fl_points)."""
    algo: np.ndarray          # uint8 (ring=0, tree=1, mesh-hier=2)
    topo_kind: np.ndarray     # uint8 (switch=0, mesh=1)
    bw: np.ndarray            # float64 bytes/s
    latency: np.ndarray       # int64 ns
    rows: np.ndarray          # int32
    cols: np.ndarray          # int32
    peak_flops: Optional[np.ndarray] = None   # float64; None keeps each node's duration_ns
    efficiency: Optional[np.ndarray] = None
    compute_streams: int = 1

    def __len__(self) -> int:
        return len(self.bw)

    @classmethod
    def from_topologies(cls, topos, algos, devices=None, compute_streams: int = 1) -> "DesignPoints":
        n = len(topos)
        algos = list(algos) if not isinstance(algos, (str, CollectiveAlgo)) else [algos] * n
        pts = cls(algo=np.asarray([ALGO[_ev(a)] for a in algos], np.uint8),
                  topo_kind=np.asarray([0 if _ev(t.kind) == "switch" else 1 for t in topos], np.uint8),
                  bw=np.asarray([float(t.bw_bytes_per_s) for t in topos], np.float64),
                  latency=np.asarray([int(t.latency_ns) for t in topos], np.int64),
                  rows=np.asarray([int(getattr(t, "rows", 0)) for t in topos], np.int32),
                  cols=np.asarray([int(getattr(t, "cols", 0)) for t in topos], np.int32),
                  compute_streams=compute_streams)
        if devices is not None:
            pts.peak_flops = np.asarray([d.peak_flops for d in devices], np.float64)
            pts.efficiency = np.asarray([d.efficiency for d in devices], np.float64)
        return pts

    def raw(self):
        """The fl_points struct of these columns (validated; rebuilt only when a column object or
        the stream count changed -- in-place edits of the arrays need no rebuild)."""
        key = (self.compute_streams, id(self.algo), id(self.topo_kind), id(self.bw), id(self.latency),
               id(self.rows), id(self.cols), id(self.peak_flops), id(self.efficiency))   # (= _POINT_COLS)
        cached = self.__dict__.get("_raw")
        if cached is None or cached[0] != key:
            n = len(self)
            st = _native.PointsRaw(n, *(_addr(getattr(self, f), t, n, f) for f, t in _POINT_COLS), self.compute_streams)
            self.__dict__["_raw"] = cached = (key, st, [getattr(self, f) for f, _ in _POINT_COLS])
        return cached[1]

    def slice(self, a: int, b: int) -> "DesignPoints":
        f = lambda x: None if x is None else np.ascontiguousarray(x[a:b])
        return DesignPoints(f(self.algo), f(self.topo_kind), f(self.bw), f(self.latency), f(self.rows),
                            f(self.cols), f(self.peak_flops), f(self.efficiency), self.compute_streams)

    def take(self, idx) -> "DesignPoints":
        f = lambda x: None if x is None else np.ascontiguousarray(x[idx])
        return DesignPoints(f(self.algo), f(self.topo_kind), f(self.bw), f(self.latency), f(self.rows),
                            f(self.cols), f(self.peak_flops), f(self.efficiency), self.compute_streams)


def _ptr(a, typ):
    return None if a is None else a.ctypes.data_as(typ)


_POINT_COLS = (("algo", np.uint8), ("topo_kind", np.uint8), ("bw", np.float64), ("latency", np.int64),
               ("rows", np.int32), ("cols", np.int32), ("peak_flops", np.float64), ("efficiency", np.float64))


def _addr(a, dtype=None, n=None, name=""):
    """Raw address of a C-contiguous array for the ABI structs (None -> NULL); with `dtype`, the
    design-point column must have that dtype and n entries (the engine reads it as such)."""
    if a is None:
        return None
    if dtype is not None and (a.dtype != dtype or len(a) != n or not a.flags.c_contiguous):
        raise EngineError(f"DesignPoints.{name} must be a contiguous {np.dtype(dtype).name} array of {n} entries")
    return a.ctypes.data


# ------------------------------------------------------------ engine handle


class Engine:
    """A compiled graph set resident on one GPU (an ``fl_graph`` handle)."""

    def __init__(self, graphs_or_set, device: int = 0):
        self.gs = graphs_or_set if isinstance(graphs_or_set, GraphSet) else compile_graphs(graphs_or_set)
        check_supported(self.gs)
        if self.gs.pair_error:      # an unmatched SEND/RECV channel never runs (simulator.py:177-200)
            from .errors import DeadlockError
            raise DeadlockError(self.gs.pair_error)
        L = _native.lib()
        arrs = desc_arrays(self.gs)
        d = _native.GraphDesc()
        keep = []
        for name, typ in _native.GraphDesc._fields_:
            v = arrs[name]
            if isinstance(v, np.ndarray):
                if v.size == 0:
                    v = np.zeros(1, v.dtype)
                v = np.ascontiguousarray(v)
                keep.append(v)
                setattr(d, name, v.ctypes.data_as(typ))
            else:
                setattr(d, name, v)
        h = C.c_void_p()
        rc = L.fl_graph_create(C.byref(d), device, C.byref(h))
        if rc:
            raise EngineError(f"fl_graph_create: {_native.last_error()} (status {rc})")
        self._h = h
        self.device = device
        self.max_nodes = int(L.fl_graph_max_nodes(h))
        self.units_per_point = self.gs.units()

    def close(self) -> None:
        if getattr(self, "_h", None):
            _native.lib().fl_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def link_cap(self, pts: DesignPoints) -> int:
        """Link-id space of these points: switch eg/in per rank, mesh 4 per position."""
        mesh = pts.topo_kind == 1
        cap = 2 * self.gs.n_ranks
        if mesh.any():
            cap = max(cap, int((4 * pts.rows[mesh].astype(np.int64) * pts.cols[mesh]).max()))
        return cap

    def run(self, pts: DesignPoints, rank_stats: bool = False, events: bool = False,
            links: bool = False, trace_cap: int = 0) -> dict:
        """Evaluate design points from host buffers (copies included).

        ``trace_cap > 0`` also returns each point's critical-path node trace, walked back on
        the device (fl_outputs.trace): ``trace_len[n]`` and ``trace[n, trace_cap]`` with
        entries (rank index << 32 | local node index) from the sink back to the source."""
        n = len(pts)
        R = self.gs.n_ranks
        out = {"status": np.empty(n, np.int32), "rows": np.empty((n, 6), np.int64)}
        if not (links or rank_stats or events or trace_cap > 0):
            # the sweep's common case, on the end-to-end path of every call: a cached fl_outputs
            # with only the two row pointers set (numpy's .ctypes costs ~2 us per array)
            o = self.__dict__.get("_out_rows")
            if o is None:
                o = self.__dict__["_out_rows"] = _native.OutputsRaw(None, None, None, None, None, None, 0, None, None, 0)
            o.status = C.addressof(C.c_char.from_buffer(out["status"]))
            o.rows = C.addressof(C.c_char.from_buffer(out["rows"]))
            rc = _native.lib().fl_sweep_run(self._h, C.addressof(pts.raw()), C.addressof(o))
            if rc:
                raise EngineError(f"fl_sweep_run: {_native.last_error()} (status {rc})")
            return out
        cap = self.link_cap(pts) if links else 0
        if links:
            out["link_busy"] = np.full((n, max(cap, 1)), -1, np.int64)
        if rank_stats:
            out["rank_stats"] = np.zeros((n, R, 5), np.int64)
        if events:
            out["ev_start"] = np.zeros((n, R, self.max_nodes), np.int64)
            out["ev_end"] = np.zeros((n, R, self.max_nodes), np.int64)
        if trace_cap > 0:
            out["trace"] = np.zeros((n, trace_cap), np.int64)
            out["trace_len"] = np.zeros(n, np.int32)
        p = pts.raw()
        o = _native.OutputsRaw(out["status"].ctypes.data, out["rows"].ctypes.data, _addr(out.get("rank_stats")),
                               _addr(out.get("ev_start")), _addr(out.get("ev_end")), _addr(out.get("link_busy")), cap,
                               _addr(out.get("trace")), _addr(out.get("trace_len")), int(trace_cap))
        rc = _native.lib().fl_sweep_run(self._h, C.addressof(p), C.addressof(o))
        if rc:
            raise EngineError(f"fl_sweep_run: {_native.last_error()} (status {rc})")
        return out

    def topo_levels(self):
        """Every structure's deterministic topological order and node levels, computed on the
        device (fl_topo_order; graph.py:282-306).  Returns one ``(order, level)`` pair per
        structure: node ids in Kahn / lowest-id-first order, and {node_id: level} (longest
        path from a zero-indegree node, in edges).  CyclicGraphError for a cyclic structure."""
        from .errors import CyclicGraphError
        total = sum(st.n for st in self.gs.structs)
        order = np.zeros(max(1, total), np.int32)
        level = np.zeros(max(1, total), np.int32)
        rc = _native.lib().fl_topo_order(self._h, order.ctypes.data_as(_native.P32),
                                         level.ctypes.data_as(_native.P32))
        if rc:
            raise EngineError(f"fl_topo_order: {_native.last_error()} (status {rc})")
        out, b = [], 0
        for st in self.gs.structs:
            o, lv = order[b:b + st.n], level[b:b + st.n]
            b += st.n
            if (o < 0).any():
                raise CyclicGraphError("graph has a dependency cycle; no topological order")
            ids = st.node_id
            out.append(([int(ids[k]) for k in o], {int(ids[k]): int(lv[k]) for k in range(st.n)}))
        return out

    def critical_path_only(self, pts: DesignPoints, mg: dict) -> int:
        """fl_critical_path on one design point over a merged graph (store.merged_cp_graph)."""
        p = _native.Points(len(pts), _ptr(pts.algo, _native.PU8), _ptr(pts.topo_kind, _native.PU8),
                           _ptr(pts.bw, _native.PF64), _ptr(pts.latency, _native.P64),
                           _ptr(pts.rows, _native.P32), _ptr(pts.cols, _native.P32),
                           _ptr(pts.peak_flops, _native.PF64), _ptr(pts.efficiency, _native.PF64), 1)
        cp = np.zeros(len(pts), np.int64)
        st = np.zeros(len(pts), np.int32)
        arr = {k: np.ascontiguousarray(v if len(v) else np.zeros(1, np.int32)) for k, v in mg.items() if k != "n_vert"}
        rc = _native.lib().fl_critical_path(self._h, C.byref(p), mg["n_vert"], *(
            _ptr(arr[k], _native.P32) for k in ("order", "vkind", "va", "vb", "vsend", "vmsg", "pred_off", "pred_idx")),
            _ptr(cp, _native.P64), _ptr(st, _native.P32))
        if rc:
            raise EngineError(f"fl_critical_path: {_native.last_error()} (status {rc})")
        raise_for_status(int(st[0]))
        return int(cp[0])

    def run_device(self, dev: dict, stream_ptr: int, n: int, compute_streams: int = 1) -> int:
        """Evaluate design points already resident in device memory.

        ``dev`` maps fl_points field names, and fl_outputs field names prefixed
        with ``out_`` (``out_status``, ``out_rows``, ...), to raw device
        pointers (ints, e.g. ``tensor.data_ptr()``).  Asynchronous on ``stream_ptr``.
        Returns the number of kernels enqueued.
        """
        v = lambda k, t: C.cast(C.c_void_p(dev[k]), t) if dev.get(k) else None
        p = _native.Points(n, v("algo", _native.PU8), v("topo_kind", _native.PU8), v("bw", _native.PF64),
                           v("latency", _native.P64), v("rows", _native.P32), v("cols", _native.P32),
                           v("peak_flops", _native.PF64), v("efficiency", _native.PF64), compute_streams)
        o = _native.Outputs(v("out_status", _native.P32), v("out_rows", _native.P64),
                            v("out_rank_stats", _native.P64), v("out_ev_start", _native.P64),
                            v("out_ev_end", _native.P64), None, 0)
        if not dev.get("out_status") or not dev.get("out_rows"):
            raise EngineError("run_device needs out_status and out_rows device buffers")
        launches = C.c_int32(0)
        rc = _native.lib().fl_sweep_run_device(self._h, C.byref(p), C.byref(o), C.c_void_p(stream_ptr),
                                               C.byref(launches))
        if rc:
            raise EngineError(f"fl_sweep_run_device: {_native.last_error()} (status {rc})")
        return int(launches.value)


# ------------------------------------------------------------ drop-in API


def _single_point(topo, algo, compute_streams=1) -> DesignPoints:
    return DesignPoints.from_topologies([topo], [algo], compute_streams=compute_streams)


def _raise_pair_error(gs: GraphSet, topo, algo) -> None:
    """An unmatched SEND/RECV channel is a DeadlockError, raised by the reference
    only after its collectives were costed (simulator.py:220-228), so an
    undefined algorithm on this topology wins."""
    from .costs import analytical_time
    from .graph import CollectiveKind
    kinds = {0: CollectiveKind.ALL_REDUCE, 1: CollectiveKind.ALL_GATHER, 2: CollectiveKind.REDUCE_SCATTER}
    mesh = (topo.rows, topo.cols) if _ev(topo.kind) == "mesh" else None
    for i in range(gs.n_inst):
        k, n = kinds[int(gs.inst_kind[i])], int(gs.inst_n[i])
        size = int(gs.inst_bytes[i]) * n if k == CollectiveKind.ALL_GATHER else int(gs.inst_bytes[i])
        analytical_time(k, size, n, CollectiveAlgo(_ev(algo)), topo.latency_ns, topo.beta_ns_per_byte, mesh_shape=mesh)
    from .errors import DeadlockError
    raise DeadlockError(gs.pair_error)


def _link_names(gs: GraphSet, topo, busy) -> dict:
    out = {}
    cols = getattr(topo, "cols", 0)
    for l in np.nonzero(busy >= 0)[0]:
        l = int(l)
        if _ev(topo.kind) == "switch":
            out[f"{'eg' if l % 2 == 0 else 'in'}{int(gs.rank_values[l // 2])}"] = int(busy[l])
        else:
            a, d = divmod(l, 4)
            b = a + (1, -1, cols, -cols)[d]
            out[f"{a}->{b}"] = int(busy[l])
    return dict(sorted(out.items()))


def simulate(graphs, topo, opts: Optional[SimOptions] = None, device: int = 0) -> SimReport:
    """Drop-in ``trainsim.simulate`` (simulator.py:203) evaluated on the GPU."""
    opts = opts or SimOptions()
    if opts.compute_streams < 1 or opts.comm_streams < 1:
        raise ValueError("stream counts must be >= 1")
    gs = compile_graphs(graphs)
    if gs.pair_error:
        _raise_pair_error(gs, topo, opts.algo)
    eng = Engine(gs, device)
    try:
        out = eng.run(_single_point(topo, opts.algo, opts.compute_streams), rank_stats=True,
                      events=opts.record_events, links=gs.has_p2p)
    finally:
        eng.close()
    raise_for_status(int(out["status"][0]), "simulation stalled with work remaining"
                     if out["status"][0] == 3 else "")
    ranks = {}
    for r in range(gs.n_ranks):
        s = out["rank_stats"][0, r]
        ranks[int(gs.rank_values[r])] = RankStats(*map(int, s))
    rep = SimReport(makespan_ns=int(out["rows"][0, 0]), ranks=ranks)
    if gs.has_p2p:
        rep.link_busy_ns = _link_names(gs, topo, out["link_busy"][0])
    if opts.record_events:
        stream_of = {0: "host", 1: "compute", 2: "comm", 3: "comm", 4: "comm"}
        evs = []
        for r in range(gs.n_ranks):
            st = gs.structs[gs.rank_struct[r]]
            rv = int(gs.rank_values[r])
            s0, e0 = out["ev_start"][0, r], out["ev_end"][0, r]
            for k, node in enumerate(st.nodes):
                evs.append(TraceEvent(rv, node.node_id, stream_of[int(st.kind[k])], node.op_name,
                                      int(s0[k]), int(e0[k])))
        evs.sort(key=lambda e: (e.start_ns, e.rank, e.node_id))
        rep.events = evs
    # ranks must be reported in the caller's order (dict insertion order of the reference)
    rep.ranks = {int(g.rank): rep.ranks[int(g.rank)] for g in graphs}
    return rep


def critical_path(graphs, topo, algo=CollectiveAlgo.RING, device: int = 0) -> int:
    """Drop-in ``trainsim.critical_path`` (simulator.py:400): contention-free bound."""
    gs = compile_graphs(graphs)
    if gs.pair_error:
        _raise_pair_error(gs, topo, algo)
    eng = Engine(gs, device)
    try:
        pts = _single_point(topo, algo)
        out = eng.run(pts)
        if out["status"][0] == 3 and gs.has_p2p:
            # the simulation deadlocked on a SEND waiting for its RECV (simulator.py:259-268);
            # the contention-free bound has no such wait: relax the merged graph alone
            from .store import merged_cp_graph
            return eng.critical_path_only(pts, merged_cp_graph(gs))
    finally:
        eng.close()
    raise_for_status(int(out["status"][0]), "cyclic cross-rank wait in critical path"
                     if out["status"][0] == 3 else "")
    return int(out["rows"][0, 1])


def critical_path_trace(graphs, topo, algo=CollectiveAlgo.RING, device: int = 0):
    """Critical path with its node trace: ``(length_ns, [(rank, node_id), ...])``.

    SPEC.md:460 defines ``critical_path`` as "duration_ns and node path"; the reference
    implementation returns only the length (simulator.py:400-460), so the path rule is
    this package's, restated in oracle/pyoracle.py:critical_path_trace:

    * the sink is the (rank, node_id) with the largest contention-free finish, the
      lowest (rank, node_id) on ties;
    * a node's predecessor on the path is its lowest (rank, node_id) dependency whose
      finish equals the node's start (a collective member's dependencies are the union
      over its group, simulator.py:419-428); when no dependency does, the start was
      set by a RECV's SEND plus the wire time (simulator.py:430-435, :450-452) and the
      path continues at the SEND; a node whose start no predecessor sets is the source.

    The walk runs on the device inside the sweep kernel (fl_outputs.trace, from the
    finishes the simulation computes); ``trace_paths`` converts any batch of them.  Only a
    graph whose *simulation* deadlocks (a SEND waits for its RECV, simulator.py:259-268,
    while the contention-free bound has no such wait) falls back to the standalone
    critical-path kernel (fl_critical_path_values) and a host walk.
    """
    gs = compile_graphs(graphs)
    if gs.pair_error:
        _raise_pair_error(gs, topo, algo)
    eng = Engine(gs, device)
    try:
        out = eng.run(_single_point(topo, algo), trace_cap=trace_capacity(gs))
    finally:
        eng.close()
    st = int(out["status"][0])
    if st == FL_OK:
        return int(out["rows"][0, 1]), trace_paths(gs, out)[0]
    if st != 3:
        raise_for_status(st)
    return _critical_path_trace_fallback(gs, topo, algo, device)


def trace_capacity(gs: GraphSet) -> int:
    """Entries that always hold a critical-path trace: every (rank, node) once."""
    return int(gs.units()) + 1


def trace_paths(gs: GraphSet, out: dict) -> list:
    """Device traces (Engine.run(..., trace_cap=)) -> per point [(rank, node_id), ...] source first."""
    paths = []
    for k in range(len(out["trace_len"])):
        n = int(out["trace_len"][k])
        if n > out["trace"].shape[1]:
            raise EngineError(f"critical-path trace of {n} nodes exceeds trace_cap {out['trace'].shape[1]}")
        ent = out["trace"][k, :n][::-1]
        ranks, nodes = (ent >> 32).astype(np.int64), (ent & 0xffffffff).astype(np.int64)
        paths.append([(int(gs.rank_values[r]), int(gs.structs[gs.rank_struct[r]].node_id[x]))
                      for r, x in zip(ranks, nodes)])
    return paths


def _critical_path_trace_fallback(gs, topo, algo, device):
    from .store import merged_cp_graph
    mg = merged_cp_graph(gs)
    eng = Engine(gs, device)
    try:
        pts = _single_point(topo, algo)
        p = _native.Points(1, _ptr(pts.algo, _native.PU8), _ptr(pts.topo_kind, _native.PU8),
                           _ptr(pts.bw, _native.PF64), _ptr(pts.latency, _native.P64),
                           _ptr(pts.rows, _native.P32), _ptr(pts.cols, _native.P32),
                           _ptr(pts.peak_flops, _native.PF64), _ptr(pts.efficiency, _native.PF64), 1)
        V = int(mg["n_vert"])
        cp = np.zeros(1, np.int64)
        st = np.zeros(1, np.int32)
        vals = np.zeros(2 * max(V, 1), np.int64)
        arr = {k: np.ascontiguousarray(v if len(v) else np.zeros(1, np.int32)) for k, v in mg.items() if k != "n_vert"}
        rc = _native.lib().fl_critical_path_values(eng._h, C.byref(p), V, *(
            _ptr(arr[k], _native.P32) for k in ("order", "vkind", "va", "vb", "vsend", "vmsg", "pred_off", "pred_idx")),
            _ptr(cp, _native.P64), _ptr(st, _native.P32), _ptr(vals, _native.P64))
        if rc:
            raise EngineError(f"fl_critical_path_values: {_native.last_error()} (status {rc})")
    finally:
        eng.close()
    raise_for_status(int(st[0]))
    finish, start = vals[:V], vals[V:2 * V]
    R = gs.n_ranks
    base = np.zeros(R + 1, np.int64)
    for r in range(R):
        base[r + 1] = base[r] + gs.structs[gs.rank_struct[r]].n
    total = int(base[-1])
    vid = np.arange(total, dtype=np.int64)
    inst_of = np.full(total, -1, np.int64)
    for i in range(gs.n_inst):
        for j in range(int(gs.inst_mem_off[i]), int(gs.inst_mem_off[i + 1])):
            g_ = base[gs.inst_mem_rank[j]] + gs.inst_mem_node[j]
            vid[g_], inst_of[g_] = total + i, i
    send_of = {}
    for m in range(len(gs.msg_bytes) if gs.msg_bytes is not None else 0):
        send_of[int(base[gs.msg_recv_rank[m]] + gs.msg_recv_node[m])] = int(base[gs.msg_send_rank[m]] + gs.msg_send_node[m])
    rank_of = np.repeat(np.arange(R), np.diff(base))
    key = lambda g_: (int(gs.rank_values[rank_of[g_]]), int(gs.structs[gs.rank_struct[rank_of[g_]]].node_id[g_ - base[rank_of[g_]]]))

    def deps(g_):
        r = int(rank_of[g_])
        members = ([int(base[gs.inst_mem_rank[j]] + gs.inst_mem_node[j])
                    for j in range(int(gs.inst_mem_off[inst_of[g_]]), int(gs.inst_mem_off[inst_of[g_] + 1]))]
                   if inst_of[g_] >= 0 else [g_])
        out = []
        for m_ in members:
            rm = int(rank_of[m_])
            st_ = gs.structs[gs.rank_struct[rm]]
            k = m_ - int(base[rm])
            out.extend(int(base[rm]) + int(q) for q in st_.pred_idx[st_.pred_off[k]:st_.pred_off[k + 1]])
        return out

    cand = [g_ for g_ in range(total)]
    if not cand:
        return 0, []
    sink = min(cand, key=lambda g_: (-int(finish[vid[g_]]), key(g_)))
    path = [sink]
    while True:
        cur = path[-1]
        s0 = int(start[vid[cur]])
        hit = [d for d in deps(cur) if int(finish[vid[d]]) == s0]
        if hit:
            path.append(min(hit, key=key))
        elif cur in send_of:
            path.append(send_of[cur])
        else:
            break
    return int(cp[0]), [key(g_) for g_ in reversed(path)]


def simulate_batch(graphs, points: DesignPoints, device: int = 0, engine: Optional[Engine] = None) -> dict:
    """One graph set x N design points -> sweep rows (cli.py:319-342, batched).

    Returns ``{"status": int32[N], field: int64[N] for field in ROW_FIELDS}``;
    rows whose status is not FL_OK carry zeros (see errors.raise_for_status).
    """
    eng = engine or Engine(graphs, device)
    out = eng.run(points)
    res = {"status": out["status"]}
    for k, name in enumerate(ROW_FIELDS):
        res[name] = out["rows"][:, k]
    return res


def topo_orders(graphs, device: int = 0) -> dict:
    """``trainsim.graph.topo_order`` (graph.py:282-306) for every rank of a graph set,
    computed on the GPU: {rank: [node_id, ...]}.  Ranks sharing a structure share its order."""
    eng = Engine(graphs, device)
    try:
        per = eng.topo_levels()
        return {int(eng.gs.rank_values[r]): list(per[int(eng.gs.rank_struct[r])][0])
                for r in range(eng.gs.n_ranks)}
    finally:
        eng.close()


def cost_only(kind, size_bytes, group_n, algo, alpha, beta, rows, cols, flops=None, peak=None, eff=None):
    """K1 on the device: alpha-beta times (collectives.py:251-293) and flops->ns
    (traceio.py:184) for arrays of inputs.  Returns (ns, status, comp_ns)."""
    c = lambda a, t: np.ascontiguousarray(np.asarray(a, dtype=t))
    kind, size_bytes, group_n, algo = c(kind, np.uint8), c(size_bytes, np.int64), c(group_n, np.int64), c(algo, np.uint8)
    alpha, beta, rows, cols = c(alpha, np.float64), c(beta, np.float64), c(rows, np.int32), c(cols, np.int32)
    n = len(kind)
    m = 0 if flops is None else len(flops)
    flops = c(flops if flops is not None else [0], np.int64)
    peak = c(peak if peak is not None else [1.0], np.float64)
    eff = c(eff if eff is not None else [1.0], np.float64)
    out, st, comp = np.zeros(max(n, 1), np.int64), np.zeros(max(n, 1), np.int32), np.zeros(max(m, 1), np.int64)
    rc = _native.lib().fl_cost_only(n, _ptr(kind, _native.PU8), _ptr(size_bytes, _native.P64),
                                    _ptr(group_n, _native.P64), _ptr(algo, _native.PU8),
                                    _ptr(alpha, _native.PF64), _ptr(beta, _native.PF64),
                                    _ptr(rows, _native.P32), _ptr(cols, _native.P32), _ptr(out, _native.P64),
                                    _ptr(st, _native.P32), m, _ptr(flops, _native.P64), _ptr(peak, _native.PF64),
                                    _ptr(eff, _native.PF64), _ptr(comp, _native.P64))
    if rc:
        raise EngineError(f"fl_cost_only: {_native.last_error()} (status {rc})")
    return out[:n], st[:n], comp[:m]
