"""ctypes front end of the CPU parity oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) import this module.  The product package
(paper_2604_17550_b200) never does.

``flatten`` serializes per-rank graphs (the reference's ``trainsim`` objects
or ours -- attributes are read by name) into the flat arrays of
``or_graphs`` in flint_oracle.c without any semantic transformation: node
lists in list order, raw ``dep_ids()`` with duplicates, raw tensor tables.
All interpretation (dedup, id lookup, instance matching) happens in the C
restatement, independently of the product's graph compiler.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "libflint_oracle.so"

KIND = {"HOST": 0, "COMP": 1, "COLL": 2, "SEND": 3, "RECV": 4}
CKIND = {"ALL_REDUCE": 0, "ALL_GATHER": 1, "REDUCE_SCATTER": 2}
ALGO = {"ring": 0, "tree": 1, "mesh-hier": 2}
STATUS_NAMES = {1: "ValueError", 3: "DeadlockError", 4: "UnsupportedAlgoTopologyError",
                5: "InconsistentGroupsError"}


class OracleError(Exception):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.kind = STATUS_NAMES.get(code, str(code))


P = C.POINTER(C.c_int64)
P32 = C.POINTER(C.c_int32)


class OrGraphs(C.Structure):
    _fields_ = [("n_ranks", C.c_int64), ("rank_value", P), ("node_off", P), ("rank_base", P), ("node_id", P),
                ("node_kind", P32), ("node_dur", P), ("dep_off", P), ("dep_ids", P),
                ("in_off", P), ("in_tid", P), ("out_off", P), ("out_tid", P),
                ("coll_kind", P32), ("coll_bytes", P), ("grp_off", P), ("grp_rank", P),
                ("p2p_peer", P), ("p2p_bytes", P), ("p2p_tag", P),
                ("tens_lo", P), ("tens_hi", P), ("tens_id", P), ("tens_bytes", P), ("sv", P)]


class OrConfig(C.Structure):
    _fields_ = [("topo_kind", C.c_int32), ("algo", C.c_int32), ("world_size", C.c_int64),
                ("bw", C.c_double), ("latency", C.c_int64), ("rows", C.c_int64),
                ("cols", C.c_int64), ("compute_streams", C.c_int32), ("comm_streams", C.c_int32)]


class OrSimOut(C.Structure):
    _fields_ = [("makespan", C.c_int64), ("rank_stats", P), ("ev_start", P), ("ev_end", P),
                ("link_busy", P), ("n_links", C.c_int64)]


_lib = None


def build(force: bool = False) -> Path:
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off)."""
    if force or not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < (HERE / "flint_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-C", str(HERE)], check=True, capture_output=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        _lib = C.CDLL(str(LIB_PATH))
        _lib.or_simulate.argtypes = [C.POINTER(OrGraphs), C.POINTER(OrConfig), C.POINTER(OrSimOut), C.c_char_p, C.c_int]
        _lib.or_critical_path.argtypes = [C.POINTER(OrGraphs), C.POINTER(OrConfig), P, C.c_char_p, C.c_int]
        _lib.or_critical_path_ex.argtypes = [C.POINTER(OrGraphs), C.POINTER(OrConfig), P, P, P, P, P,
                                             C.c_char_p, C.c_int]
        _lib.or_analytical_time.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_double, C.c_double,
                                            C.c_int64, C.c_int64, C.POINTER(C.c_int)]
        _lib.or_analytical_time.restype = C.c_int64
        _lib.or_duration_from_flops.argtypes = [C.c_int64, C.c_double, C.c_double]
        _lib.or_duration_from_flops.restype = C.c_int64
    return _lib


def _ev(x):
    return x.value if hasattr(x, "value") else x


def _flatten_nodes(nodes) -> dict:
    node_id, kind, dur, ckind, cbytes, peer, pbytes, tag = ([] for _ in range(8))
    dep, dep_off, ins, in_off, outs, out_off, grp, grp_off = [], [0], [], [0], [], [0], [], [0]
    for n in nodes:
        node_id.append(n.node_id)
        kind.append(KIND[_ev(n.kind)])
        dur.append(-1 if n.duration_ns is None else n.duration_ns)
        dep.extend(n.dep_ids()); dep_off.append(len(dep))
        ins.extend(n.inputs); in_off.append(len(ins))
        outs.extend(n.outputs); out_off.append(len(outs))
        if n.coll is not None:
            ckind.append(CKIND[_ev(n.coll.kind)]); cbytes.append(n.coll.comm_bytes); grp.extend(n.coll.group)
        else:
            ckind.append(-1); cbytes.append(0)
        grp_off.append(len(grp))
        if n.p2p is not None:
            peer.append(n.p2p.peer_rank); pbytes.append(n.p2p.comm_bytes); tag.append(n.p2p.channel_tag)
        else:
            peer.append(-1); pbytes.append(0); tag.append(0)
    i64 = lambda a: np.asarray(a, dtype=np.int64)
    return dict(node_id=i64(node_id), node_kind=np.asarray(kind, np.int32), node_dur=i64(dur),
                dep_off=i64(dep_off), dep_ids=i64(dep), in_off=i64(in_off), in_tid=i64(ins),
                out_off=i64(out_off), out_tid=i64(outs), coll_kind=np.asarray(ckind, np.int32),
                coll_bytes=i64(cbytes), grp_off=i64(grp_off), grp_rank=i64(grp),
                p2p_peer=i64(peer), p2p_bytes=i64(pbytes), p2p_tag=i64(tag))


def flatten(graphs) -> dict:
    """Per-structure node tables plus a per-rank index into them.

    Ranks whose graphs share one node list (by identity, as synth emits,
    synth.py:331-335) share one copy of the node arrays, group lists included,
    and likewise for tensor tables.  The C side maps a flat (rank, position)
    node to its structure node (``SV`` in flint_oracle.c), so memory is
    O(R + structures) instead of O(R x N) -- and O(R x C x R) for full-world
    group lists, which at 8192 ranks would be ~120 GiB."""
    scache: dict = {}
    tcache: dict = {}
    sparts, tparts = [], []
    rank_base, node_count, tens_lo, tens_hi = [], [], [], []
    sbase = tbase = 0
    for g in graphs:
        key = id(g.nodes)
        if key not in scache:
            part = _flatten_nodes(g.nodes)
            scache[key] = (sbase, len(part["node_id"]))
            sparts.append(part)
            sbase += len(part["node_id"])
        b, c = scache[key]
        rank_base.append(b); node_count.append(c)
        tk = id(g.tensors)
        if tk not in tcache:
            items = list(g.tensors.items())
            tcache[tk] = (tbase, tbase + len(items))
            tparts.append((np.asarray([k for k, _ in items], np.int64),
                           np.asarray([t.bytes for _, t in items], np.int64)))
            tbase += len(items)
        lo, hi = tcache[tk]
        tens_lo.append(lo); tens_hi.append(hi)
    i64 = lambda a: np.asarray(a, np.int64)
    out = {"n_ranks": len(graphs), "rank_value": i64([g.rank for g in graphs]),
           "node_off": np.concatenate([[0], np.cumsum(i64(node_count))]).astype(np.int64),
           "rank_base": i64(rank_base), "tens_lo": i64(tens_lo), "tens_hi": i64(tens_hi)}
    for name in ("node_id", "node_kind", "node_dur", "coll_kind", "coll_bytes", "p2p_peer", "p2p_bytes", "p2p_tag"):
        out[name] = np.concatenate([p[name] for p in sparts]) if sparts else np.zeros(0, np.int64)
    for off, val in (("dep_off", "dep_ids"), ("in_off", "in_tid"), ("out_off", "out_tid"), ("grp_off", "grp_rank")):
        vals, offs, base = [], [np.zeros(1, np.int64)], 0
        for p in sparts:
            vals.append(p[val])
            offs.append(p[off][1:] + base)
            base += len(p[val])
        out[val] = np.concatenate(vals) if vals else np.zeros(0, np.int64)
        out[off] = np.concatenate(offs).astype(np.int64)
    out["tens_id"] = np.concatenate([t[0] for t in tparts]) if tparts else np.zeros(0, np.int64)
    out["tens_bytes"] = np.concatenate([t[1] for t in tparts]) if tparts else np.zeros(0, np.int64)
    for k, v in out.items():
        if isinstance(v, np.ndarray):
            out[k] = np.ascontiguousarray(v)
    return out


def structure_index(flat: dict) -> np.ndarray:
    """flat node -> structure node (the C side's SV map)."""
    node_off = flat["node_off"]
    counts = np.diff(node_off)
    rank_of = np.repeat(np.arange(len(counts)), counts)
    return flat["rank_base"][rank_of] + (np.arange(int(node_off[-1])) - node_off[rank_of])


def _struct(flat: dict) -> OrGraphs:
    g = OrGraphs()
    g.n_ranks = flat["n_ranks"]
    for name, typ in OrGraphs._fields_[1:-1]:
        arr = flat[name]
        if len(arr) == 0:
            arr = np.zeros(1, arr.dtype)
            flat[name + "_pad"] = arr
        setattr(g, name, arr.ctypes.data_as(typ))
    return g


def _config(topo, algo, compute_streams=1, comm_streams=1) -> OrConfig:
    c = OrConfig()
    c.topo_kind = 0 if _ev(topo.kind) == "switch" else 1
    c.algo = ALGO[_ev(algo)]
    c.world_size = topo.world_size
    c.bw = float(topo.bw_bytes_per_s)
    c.latency = int(topo.latency_ns)
    c.rows = int(getattr(topo, "rows", 0))
    c.cols = int(getattr(topo, "cols", 0))
    c.compute_streams = compute_streams
    c.comm_streams = comm_streams
    return c


def link_name(topo, link_id: int, rank_values) -> str:
    if _ev(topo.kind) == "switch":
        r = rank_values[link_id // 2]
        return f"eg{r}" if link_id % 2 == 0 else f"in{r}"
    a, d = divmod(link_id, 4)
    cols = topo.cols
    b = a + (1 if d == 0 else -1 if d == 1 else cols if d == 2 else -cols)
    return f"{a}->{b}"


def simulate(graphs, topo, algo="ring", compute_streams=1, comm_streams=1,
             record_events=False, flat=None) -> dict:
    """Returns {makespan_ns, ranks: {rank: {...}}, links: {...}, events?}."""
    flat = flat if flat is not None else flatten(graphs)
    g = _struct(flat)
    cfg = _config(topo, algo, compute_streams, comm_streams)
    nr = flat["n_ranks"]
    total = int(flat["node_off"][-1])
    stats = np.zeros(max(1, nr * 5), np.int64)
    n_links = 2 * nr if cfg.topo_kind == 0 else 4 * cfg.rows * cfg.cols
    links = np.full(max(1, n_links), -1, np.int64)
    out = OrSimOut()
    out.rank_stats = stats.ctypes.data_as(P)
    out.link_busy = links.ctypes.data_as(P)
    out.n_links = n_links
    if record_events:
        st = np.zeros(max(1, total), np.int64); en = np.zeros(max(1, total), np.int64)
        out.ev_start = st.ctypes.data_as(P); out.ev_end = en.ctypes.data_as(P)
    err = C.create_string_buffer(512)
    rc = lib().or_simulate(C.byref(g), C.byref(cfg), C.byref(out), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    ranks = {}
    for i in range(nr):
        s = stats[5 * i: 5 * i + 5]
        ranks[int(flat["rank_value"][i])] = dict(finish_ns=int(s[0]), compute_busy_ns=int(s[1]),
                                                 comm_busy_ns=int(s[2]), exposed_comm_ns=int(s[3]),
                                                 peak_mem_bytes=int(s[4]))
    rv = [int(x) for x in flat["rank_value"]]
    res = {"makespan_ns": int(out.makespan), "ranks": ranks,
           "links": dict(sorted((link_name(topo, k, rv), int(v)) for k, v in enumerate(links[:n_links]) if v >= 0))}
    if record_events:
        res["events"] = (st[:total].copy(), en[:total].copy())
    return res


def critical_path(graphs, topo, algo="ring", flat=None) -> int:
    flat = flat if flat is not None else flatten(graphs)
    g = _struct(flat)
    cfg = _config(topo, algo)
    res = C.c_int64(0)
    err = C.create_string_buffer(512)
    rc = lib().or_critical_path(C.byref(g), C.byref(cfg), C.byref(res), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    return int(res.value)


def critical_path_trace(graphs, topo, algo="ring", flat=None):
    """(length, [(rank, node_id), ...]) -- the node-trace rule documented at
    paper_2604_17550_b200.engine.critical_path_trace, over the C restatement's
    per-node finish/start times (or_critical_path_ex, simulator.py:400-460)."""
    flat = flat if flat is not None else flatten(graphs)
    g = _struct(flat)
    cfg = _config(topo, algo)
    total = int(flat["node_off"][-1])
    fin, start, inst, send = (np.zeros(max(1, total), np.int64) for _ in range(4))
    res = C.c_int64(0)
    err = C.create_string_buffer(512)
    rc = lib().or_critical_path_ex(C.byref(g), C.byref(cfg), C.byref(res), fin.ctypes.data_as(P),
                                   start.ctypes.data_as(P), inst.ctypes.data_as(P), send.ctypes.data_as(P), err, 512)
    if rc:
        raise OracleError(rc, err.value.decode())
    if total == 0:
        return int(res.value), []
    node_off, rank_value = flat["node_off"], flat["rank_value"]
    sv = structure_index(flat)
    node_id = flat["node_id"][sv]
    rank_of = np.repeat(np.arange(len(rank_value)), np.diff(node_off))
    index = {(int(rank_of[v]), int(node_id[v])): v for v in range(total)}
    members = {}
    for v in range(total):
        if inst[v] >= 0:
            members.setdefault(int(inst[v]), []).append(v)
    dep_off, dep_ids = flat["dep_off"], flat["dep_ids"]

    def key(v):
        return int(rank_value[rank_of[v]]), int(node_id[v])

    def deps(v):
        out = set()
        for m in (members[int(inst[v])] if inst[v] >= 0 else [v]):
            r = int(rank_of[m])
            for q in range(int(dep_off[sv[m]]), int(dep_off[sv[m] + 1])):
                out.add(index[(r, int(dep_ids[q]))])
        return out

    v = min(range(total), key=lambda u: (-int(fin[u]), key(u)))
    path = [v]
    while True:
        hit = [d for d in deps(v) if fin[d] == start[v]]
        if hit:
            v = min(hit, key=key)
        elif send[v] >= 0:
            v = int(send[v])
        else:
            break
        path.append(v)
    return int(res.value), [key(u) for u in reversed(path)]


def analytical_time(kind: str, size_bytes: int, n: int, algo: str, alpha: float, beta: float,
                    rows: int = 0, cols: int = 0) -> int:
    st = C.c_int(0)
    v = lib().or_analytical_time(CKIND[kind], size_bytes, n, ALGO[algo], float(alpha), float(beta),
                                 rows, cols, C.byref(st))
    if st.value:
        raise OracleError(st.value, "unsupported algorithm/topology")
    return int(v)


def duration_from_flops(flops: int, peak: float, eff: float) -> int:
    return int(lib().or_duration_from_flops(flops, peak, eff))


def sweep_row(graphs, topo, algo, flat=None) -> dict:
    """What reference cli._sweep_row (cli.py:319-342) returns, minus the labels."""
    flat = flat if flat is not None else flatten(graphs)
    rep = simulate(graphs, topo, algo, flat=flat)
    cp = critical_path(graphs, topo, algo, flat=flat)
    rs = rep["ranks"].values()
    return {"makespan_ns": rep["makespan_ns"], "critical_path_ns": cp,
            "compute_busy_ns": max(s["compute_busy_ns"] for s in rs),
            "comm_busy_ns": max(s["comm_busy_ns"] for s in rs),
            "exposed_comm_ns": max((s["exposed_comm_ns"] for s in rs), default=0),
            "peak_mem_bytes": max((s["peak_mem_bytes"] for s in rs), default=0)}
