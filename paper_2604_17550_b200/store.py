"""Graph store: compile per-rank workload graphs into the engine's CSR form.

Input is a list of per-rank graphs (the reference's ``trainsim`` objects or
ours; attributes are read by name).  Output is a :class:`GraphSet`, the host
image of ``fl_graph_desc`` (include/flint_b200.h), which
:class:`paper_2604_17550_b200.engine.Engine` uploads once per device.

Layout decisions:

* ranks are dense 0..R-1 in ascending rank-value order (the reference's
  event-heap tie order, simulator.py:240) and point at a *structure*; ranks
  whose graphs share the same node list and tensor table (every synthesized
  family, synth.py:331-335) share one structure, so the CSR is stored once;
* inside a structure nodes are re-indexed by ascending node_id, which turns
  the reference's "lowest ready id" heaps into lowest-set-bit searches;
* ``succ`` lists keep the reference's dispatch order (the graph's node-list
  order, simulator.py:214-218), which decides ties between collectives that
  complete in the same pop;
* collective instances are matched across ranks exactly as
  ``collective_instances`` does (collectives.py:419-453).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import DeadlockError, EngineError, InconsistentGroupsError

KIND = {"HOST": 0, "COMP": 1, "COLL": 2, "SEND": 3, "RECV": 4}
CKIND = {"ALL_REDUCE": 0, "ALL_GATHER": 1, "REDUCE_SCATTER": 2}


def _ev(x):
    return x.value if hasattr(x, "value") else x


@dataclass
class Structure:
    """One distinct rank graph, compiled (all arrays local to the structure)."""
    nodes: list                     # original Node objects in ascending-id order
    node_id: np.ndarray
    listpos: np.ndarray
    kind: np.ndarray
    flags: np.ndarray
    dur: np.ndarray
    flops: np.ndarray
    alloc: np.ndarray
    coll_ord: np.ndarray
    pred_off: np.ndarray
    pred_idx: np.ndarray
    succ_off: np.ndarray
    succ_idx: np.ndarray
    free_off: np.ndarray
    free_tens: np.ndarray
    init_list: np.ndarray
    tens_bytes: np.ndarray
    cons_off: np.ndarray
    cons_idx: np.ndarray
    init_alloc: int
    colls: list                     # local indices of COLL nodes in list order
    p2ps: list = field(default_factory=list)   # local indices of SEND/RECV nodes in list order

    @property
    def n(self) -> int:
        return len(self.node_id)


def _csr(lists) -> tuple:
    off = np.zeros(len(lists) + 1, np.int32)
    off[1:] = np.cumsum([len(x) for x in lists]) if lists else []
    flat = np.fromiter((v for x in lists for v in x), np.int32, count=int(off[-1]))
    return off, flat


def compile_structure(nodes, tensors) -> Structure:
    order = sorted(range(len(nodes)), key=lambda i: nodes[i].node_id)
    ids = [nodes[i].node_id for i in order]
    if len(set(ids)) != len(ids):
        raise ValueError("duplicate node_id in a rank graph")
    local = {nid: k for k, nid in enumerate(ids)}
    n = len(ids)
    listpos = np.empty(n, np.int64)
    for k, i in enumerate(order):
        listpos[k] = i
    kind = np.empty(n, np.uint8)
    flags = np.zeros(n, np.uint8)
    dur = np.zeros(n, np.int64)
    flops = np.full(n, -1, np.int64)
    coll_ord = np.full(n, -1, np.int32)
    preds = [None] * n
    succs = [[] for _ in range(n)]
    init = []
    colls = []
    p2ps = []
    for li, node in enumerate(nodes):               # list order: dispatch order of the reference
        k = local[node.node_id]
        kd = KIND[_ev(node.kind)]
        kind[k] = kd
        if kd in (0, 1):
            dur[k] = node.duration_ns or 0
            fl = getattr(node, "flops", None)
            if kd == 1 and fl is not None:
                flops[k] = fl
        elif kd == 2:
            coll_ord[k] = len(colls)
            colls.append(k)
        else:                                       # SEND / RECV: ordinal among this rank's p2p nodes
            coll_ord[k] = len(p2ps)
            p2ps.append(k)
        deps = set(node.dep_ids())
        p = []
        for d in deps:
            if d in local:
                p.append(local[d])
            else:
                flags[k] |= 1                       # waits forever (simulator.py:216, :329-333)
        preds[k] = sorted(p)
        for d in sorted(p):
            succs[d].append(k)
        if not deps:
            init.append(k)
    # tensors (simulator.py:370-393): producer = last node listing it as output
    tids = list(tensors.keys())
    tpos = {t: j for j, t in enumerate(tids)}
    tbytes = np.asarray([tensors[t].bytes for t in tids], np.int64) if tids else np.zeros(0, np.int64)
    producer = {}
    consumers = [[] for _ in tids]
    for node in nodes:
        k = local[node.node_id]
        for t in node.outputs:
            if t in tpos:
                producer[tpos[t]] = k
        for t in node.inputs:
            j = tpos.get(t)
            if j is not None and (not consumers[j] or consumers[j][-1] != k) and k not in consumers[j]:
                consumers[j].append(k)
    alloc = np.zeros(n, np.int64)
    init_alloc = 0
    for j in range(len(tids)):
        if j in producer:
            alloc[producer[j]] += tbytes[j]
        else:
            init_alloc += int(tbytes[j])
    frees = [[] for _ in range(n)]
    for j, cs in enumerate(consumers):
        for k in cs:
            frees[k].append(j)
    pred_off, pred_idx = _csr(preds)
    succ_off, succ_idx = _csr(succs)
    free_off, free_tens = _csr(frees)
    cons_off, cons_idx = _csr(consumers)
    return Structure([nodes[i] for i in order], np.asarray(ids, np.int64), listpos, kind, flags, dur,
                     flops, alloc, coll_ord, pred_off, pred_idx, succ_off, succ_idx, free_off,
                     free_tens, np.asarray(init, np.int32), tbytes, cons_off, cons_idx,
                     int(init_alloc), colls, p2ps)


@dataclass
class GraphSet:
    """Host image of fl_graph_desc for one list of per-rank graphs."""
    rank_values: np.ndarray          # [R] ascending
    rank_graph_pos: np.ndarray       # [R] index into the caller's list
    rank_struct: np.ndarray          # [R]
    structs: list
    inst_kind: np.ndarray
    inst_n: np.ndarray
    inst_bytes: np.ndarray
    inst_lead_id: np.ndarray
    inst_init_key: np.ndarray
    inst_mem_off: np.ndarray
    inst_mem_rank: np.ndarray
    inst_mem_node: np.ndarray
    coll_stride: int
    rank_coll_inst: np.ndarray       # [R, coll_stride]
    has_p2p: bool = False
    # messages (simulator.py:177-200): k-th SEND matched to k-th RECV per (src, dst, tag)
    msg_send_rank: np.ndarray = None
    msg_send_node: np.ndarray = None
    msg_recv_rank: np.ndarray = None
    msg_recv_node: np.ndarray = None
    msg_bytes: np.ndarray = None
    msg_send_id: np.ndarray = None
    p2p_stride: int = 1
    rank_p2p_msg: np.ndarray = None  # [R, p2p_stride]
    pair_error: str = ""             # unmatched channel: DeadlockError once the run starts
    _keep: list = field(default_factory=list)

    @property
    def n_ranks(self) -> int:
        return len(self.rank_values)

    @property
    def n_inst(self) -> int:
        return len(self.inst_kind)

    @property
    def max_nodes(self) -> int:
        return max((s.n for s in self.structs), default=0)

    def units(self) -> int:
        """(rank, node) pairs per design point: the logical work W / point."""
        return int(sum(self.structs[s].n for s in self.rank_struct))


def _zip_is_natural(structs, rank_struct, rank_values, rindex, group, members) -> bool:
    """zip(group, members) pairs rank group[q] with members[q] (members = [lead] + the others in
    group order).  It equals the natural pairing (each rank with its own collective) when every
    members[q] has the node_id of rank group[q]'s own member and the union of the members'
    dependencies, taken at the zipped ranks, is the natural one (critical_path's join,
    simulator.py:419-428)."""
    own = {r: node for r, node in members}
    node = lambda r, n: structs[rank_struct[r]].nodes[n]
    zr = [rindex[v] for v in group]
    if any(node(r, own[r]).node_id != node(mr, mn).node_id for r, (mr, mn) in zip(zr, members)):
        return False
    nat = {(int(rank_values[mr]), d) for mr, mn in members for d in node(mr, mn).dep_ids()}
    zipped = {(int(rank_values[r]), d) for r, (mr, mn) in zip(zr, members) for d in node(mr, mn).dep_ids()}
    return nat == zipped


def _match_instances(gs: "GraphSet", graphs, rank_values, rank_struct, structs):
    """collective_instances (collectives.py:419-453) over compiled structures."""
    R = len(rank_values)
    rindex = {int(v): r for r, v in enumerate(rank_values)}
    ncoll = [len(structs[rank_struct[r]].colls) for r in range(R)]
    stride = max(ncoll, default=0)
    rank_coll_inst = np.full((R, max(stride, 1)), -1, np.int32)

    def spec(r, k):
        st = structs[rank_struct[r]]
        node = st.nodes[st.colls[k]]
        c = node.coll
        return CKIND[_ev(c.kind)], list(c.group), int(c.comm_bytes), st.colls[k], node.node_id

    # fast path: one structure, every collective spans all ranks 0..R-1 in order
    if len(structs) == 1 and list(map(int, rank_values)) == list(range(R)):
        st = structs[0]
        full = list(range(R))
        if all(list(st.nodes[k].coll.group) == full for k in st.colls):
            C = len(st.colls)
            kinds = np.asarray([CKIND[_ev(st.nodes[k].coll.kind)] for k in st.colls], np.uint8)
            byts = np.asarray([st.nodes[k].coll.comm_bytes for k in st.colls], np.int64)
            lead = np.asarray([st.nodes[k].node_id for k in st.colls], np.int64)
            mem_off = np.arange(C + 1, dtype=np.int64) * R
            mem_rank = np.tile(np.arange(R, dtype=np.int32), C)
            mem_node = np.repeat(np.asarray(st.colls, np.int32), R)
            rank_coll_inst[:, :C] = np.arange(C, dtype=np.int32)[None, :]
            pos = np.asarray(gs.rank_graph_pos, np.int64)
            last_pos = int(pos.max()) if R else 0
            init_key = np.asarray([(last_pos << 24) | int(st.listpos[k]) for k in st.colls], np.int64)
            return (kinds, np.full(C, R, np.int32), byts, lead, init_key, mem_off, mem_rank, mem_node,
                    max(stride, 1), rank_coll_inst)

    idx = [0] * R
    kinds, ns, byts, lead, init_key, mem_off, mem_rank, mem_node = [], [], [], [], [], [0], [], []
    while True:
        start = next((r for r in range(R) if idx[r] < ncoll[r]), None)
        if start is None:
            break
        k0, group, nbytes, lnode, lid = spec(start, idx[start])
        members = [(start, lnode)]
        for v in group:
            r = rindex.get(v)
            if r == start:
                continue
            if r is None or idx[r] >= ncoll[r]:
                raise InconsistentGroupsError(f"rank {v} is missing collective #{idx[r] if r is not None else 0} of group {group}")
            ok, og, ob, onode, oid = spec(r, idx[r])
            if ok != k0 or og != group or ob != nbytes:
                raise InconsistentGroupsError(f"rank {v} node {oid} disagrees with rank {rank_values[start]} node {lid}")
            members.append((r, onode))
        if len(members) != len(group):
            raise InconsistentGroupsError(f"collective group {group} lists a rank twice")
        if rindex.get(group[0]) != start and not _zip_is_natural(structs, rank_struct, rank_values, rindex, group,
                                                                   members):
            # the reference pairs zip(group, members) (simulator.py:222-223, :419-425): with the
            # lead listed first that is each rank with its own node; otherwise it is only the same
            # pairing when node ids and the zipped dependency union agree (else the reference
            # fails with a KeyError in simulate or a spurious cycle in critical_path)
            raise InconsistentGroupsError(f"collective group {group} pairs ranks with other ranks' nodes "
                                          f"(zip(group, members), simulator.py:222-223)")
        i = len(kinds)
        kinds.append(k0); ns.append(len(group)); byts.append(nbytes); lead.append(lid)
        key = 0
        for r, node in members:
            st = structs[rank_struct[r]]
            rank_coll_inst[r, st.coll_ord[node]] = i
            key = max(key, (int(gs.rank_graph_pos[r]) << 24) | int(st.listpos[node]))
            mem_rank.append(r); mem_node.append(node)
        init_key.append(key)
        mem_off.append(len(mem_rank))
        for v in group:
            idx[rindex[v]] += 1
    return (np.asarray(kinds, np.uint8), np.asarray(ns, np.int32), np.asarray(byts, np.int64),
            np.asarray(lead, np.int64), np.asarray(init_key, np.int64), np.asarray(mem_off, np.int64),
            np.asarray(mem_rank, np.int32), np.asarray(mem_node, np.int32), max(stride, 1), rank_coll_inst)


def compile_graphs(graphs) -> GraphSet:
    values = [int(g.rank) for g in graphs]
    if len(set(values)) != len(values):
        raise ValueError("duplicate rank in graphs")          # simulator.py:206-207
    order = sorted(range(len(graphs)), key=lambda i: values[i])
    structs, skey, rank_struct = [], {}, []
    for i in order:
        g = graphs[i]
        key = (id(g.nodes), id(g.tensors))
        if key not in skey:
            skey[key] = len(structs)
            structs.append(compile_structure(g.nodes, g.tensors))
        rank_struct.append(skey[key])
    has_p2p = any(int(k) in (3, 4) for s in structs for k in s.kind)
    gs = GraphSet(np.asarray([values[i] for i in order], np.int64), np.asarray(order, np.int32),
                  np.asarray(rank_struct, np.int32), structs, *([None] * 9), None)
    (gs.inst_kind, gs.inst_n, gs.inst_bytes, gs.inst_lead_id, gs.inst_init_key, gs.inst_mem_off,
     gs.inst_mem_rank, gs.inst_mem_node, gs.coll_stride, gs.rank_coll_inst) = _match_instances(
        gs, graphs, gs.rank_values, rank_struct, structs)
    gs.has_p2p = has_p2p
    _pair_messages(gs)
    return gs


def _pair_messages(gs: GraphSet) -> None:
    """_pair_messages (simulator.py:177-200): per channel (src, dst, tag), the k-th
    SEND (by node id) carries the k-th RECV; unequal counts deadlock."""
    R = gs.n_ranks
    stride = max((len(gs.structs[gs.rank_struct[r]].p2ps) for r in range(R)), default=0)
    gs.p2p_stride = max(stride, 1)
    gs.rank_p2p_msg = np.full((R, gs.p2p_stride), -1, np.int32)
    sends, recvs = {}, {}
    for r in range(R):
        st = gs.structs[gs.rank_struct[r]]
        rv = int(gs.rank_values[r])
        for k in st.p2ps:
            node = st.nodes[k]
            p = node.p2p
            if int(st.kind[k]) == 3:
                sends.setdefault((rv, int(p.peer_rank), int(p.channel_tag)), []).append((node.node_id, r, k))
            else:
                recvs.setdefault((int(p.peer_rank), rv, int(p.channel_tag)), []).append((node.node_id, r, k))
    cols = {name: [] for name in ("sr", "sn", "rr", "rn", "by", "sid")}
    for key in sorted(set(sends) | set(recvs)):
        ss, rr = sorted(sends.get(key, [])), sorted(recvs.get(key, []))
        if len(ss) != len(rr):
            # simulate raises this after its collective checks (simulator.py:220-228)
            gs.pair_error = f"channel {key}: {len(ss)} sends but {len(rr)} recvs"
            break
        for (sid, sr, sk), (_, dr, dk) in zip(ss, rr):
            m = len(cols["sr"])
            st_s = gs.structs[gs.rank_struct[sr]]
            cols["sr"].append(sr); cols["sn"].append(sk); cols["rr"].append(dr); cols["rn"].append(dk)
            cols["by"].append(int(st_s.nodes[sk].p2p.comm_bytes)); cols["sid"].append(sid)
            gs.rank_p2p_msg[sr, st_s.coll_ord[sk]] = m
            gs.rank_p2p_msg[dr, gs.structs[gs.rank_struct[dr]].coll_ord[dk]] = m
    i32 = lambda v: np.asarray(v, np.int32)
    gs.msg_send_rank, gs.msg_send_node = i32(cols["sr"]), i32(cols["sn"])
    gs.msg_recv_rank, gs.msg_recv_node = i32(cols["rr"]), i32(cols["rn"])
    gs.msg_bytes = np.asarray(cols["by"], np.int64)
    gs.msg_send_id = np.asarray(cols["sid"], np.int64)


def desc_arrays(gs: GraphSet) -> dict:
    """Concatenate structures into the flat arrays of fl_graph_desc."""
    S = gs.structs
    node_off = np.zeros(len(S) + 1, np.int32)
    node_off[1:] = np.cumsum([s.n for s in S])
    tens_off = np.zeros(len(S) + 1, np.int32)
    tens_off[1:] = np.cumsum([len(s.tens_bytes) for s in S])
    init_off = np.zeros(len(S) + 1, np.int32)
    init_off[1:] = np.cumsum([len(s.init_list) for s in S])

    def cat(name, dtype):
        parts = [getattr(s, name) for s in S]
        return np.ascontiguousarray(np.concatenate(parts).astype(dtype)) if parts else np.zeros(0, dtype)

    def cat_csr(off_name, idx_name):
        offs, idxs, base = [np.zeros(1, np.int32)], [], 0
        for s in S:
            off = getattr(s, off_name)
            offs.append((off[1:] + base).astype(np.int32))
            idxs.append(getattr(s, idx_name))
            base += int(off[-1])
        return (np.ascontiguousarray(np.concatenate(offs)),
                np.ascontiguousarray(np.concatenate(idxs).astype(np.int32)) if idxs else np.zeros(0, np.int32))

    pred_off, pred_idx = cat_csr("pred_off", "pred_idx")
    succ_off, succ_idx = cat_csr("succ_off", "succ_idx")
    free_off, free_tens = cat_csr("free_off", "free_tens")
    cons_off, cons_idx = cat_csr("cons_off", "cons_idx")
    return dict(
        n_ranks=gs.n_ranks, rank_struct=gs.rank_struct.astype(np.int32),
        rank_graph_pos=gs.rank_graph_pos.astype(np.int32),
        n_structs=len(S), s_node_off=node_off, s_tens_off=tens_off, s_init_off=init_off,
        s_init_alloc=np.asarray([s.init_alloc for s in S], np.int64),
        s_ncoll=np.asarray([len(s.colls) for s in S], np.int32),
        node_kind=cat("kind", np.uint8), node_flags=cat("flags", np.uint8), node_id=cat("node_id", np.int64),
        node_dur=cat("dur", np.int64), node_flops=cat("flops", np.int64), node_alloc=cat("alloc", np.int64),
        node_coll_ord=cat("coll_ord", np.int32),
        pred_off=pred_off, pred_idx=pred_idx, succ_off=succ_off, succ_idx=succ_idx,
        free_off=free_off, free_tens=free_tens, init_list=cat("init_list", np.int32),
        tens_bytes=cat("tens_bytes", np.int64), tens_cons_off=cons_off, tens_cons=cons_idx,
        n_inst=gs.n_inst, inst_kind=gs.inst_kind, inst_n=gs.inst_n, inst_bytes=gs.inst_bytes,
        inst_lead_id=gs.inst_lead_id, inst_init_key=gs.inst_init_key, inst_mem_off=gs.inst_mem_off,
        inst_mem_rank=gs.inst_mem_rank, inst_mem_node=gs.inst_mem_node,
        coll_stride=int(gs.coll_stride),
        rank_coll_inst=np.ascontiguousarray(gs.rank_coll_inst.astype(np.int32)),
        rank_value=np.ascontiguousarray(gs.rank_values.astype(np.int64)),
        n_msg=len(gs.msg_bytes), msg_send_rank=gs.msg_send_rank, msg_send_node=gs.msg_send_node,
        msg_recv_rank=gs.msg_recv_rank, msg_recv_node=gs.msg_recv_node, msg_bytes=gs.msg_bytes,
        msg_send_id=gs.msg_send_id, p2p_stride=int(gs.p2p_stride),
        rank_p2p_msg=np.ascontiguousarray(gs.rank_p2p_msg.astype(np.int32)),
    )


def check_supported(gs: GraphSet, max_ranks: int = 16384, max_nodes: int = 65535) -> None:
    if gs.n_ranks > max_ranks:
        raise EngineError(f"{gs.n_ranks} ranks exceed this engine build's {max_ranks} per design point")
    if gs.max_nodes > max_nodes:
        raise EngineError(f"a rank graph has {gs.max_nodes} nodes; this build supports {max_nodes}")


def merged_cp_graph(gs: GraphSet):
    """The graph ``critical_path`` relaxes (simulator.py:408-436), in topological order.

    Vertices: every (rank, node) that is not a collective, plus one vertex per
    collective instance (its members share the union of their dependencies,
    :419-428); a RECV also depends on its SEND (:430-435).  Returns the arrays of
    ``fl_critical_path``, or raises DeadlockError when the merged graph has a
    cycle or a dependency on a missing node (:458-459).
    """
    R = gs.n_ranks
    base = np.zeros(R + 1, np.int64)
    for r in range(R):
        base[r + 1] = base[r] + gs.structs[gs.rank_struct[r]].n
    total = int(base[-1])
    V = total + gs.n_inst
    vid = np.arange(total, dtype=np.int64)            # (rank, node) -> vertex, collectives remapped
    for i in range(gs.n_inst):
        for j in range(int(gs.inst_mem_off[i]), int(gs.inst_mem_off[i + 1])):
            vid[base[gs.inst_mem_rank[j]] + gs.inst_mem_node[j]] = total + i
    preds = [set() for _ in range(V)]
    never = np.zeros(V, bool)
    vkind = np.zeros(V, np.int32)
    va = np.zeros(V, np.int32)
    vb = np.zeros(V, np.int32)
    vsend = np.full(V, -1, np.int32)
    vmsg = np.full(V, -1, np.int32)
    live = np.zeros(V, bool)
    for r in range(R):
        st = gs.structs[gs.rank_struct[r]]
        for k in range(st.n):
            v = int(vid[base[r] + k])
            live[v] = True
            if v < total:
                va[v], vb[v] = r, k
            ps = st.pred_idx[st.pred_off[k]:st.pred_off[k + 1]]
            preds[v].update(int(vid[base[r] + q]) for q in ps)
            if st.flags[k] & 1:
                never[v] = True
    for i in range(gs.n_inst):
        vkind[total + i], va[total + i] = 1, i
    for m in range(len(gs.msg_bytes)):
        s_v = int(vid[base[gs.msg_send_rank[m]] + gs.msg_send_node[m]])
        r_v = int(vid[base[gs.msg_recv_rank[m]] + gs.msg_recv_node[m]])
        preds[r_v].add(s_v)
        vsend[r_v], vmsg[r_v] = s_v, m
    indeg = np.array([len(p) for p in preds], np.int64)
    succ = [[] for _ in range(V)]
    for v in range(V):
        for u in preds[v]:
            succ[u].append(v)
    order = [v for v in range(V) if live[v] and indeg[v] == 0 and not never[v]]
    k = 0
    while k < len(order):
        u = order[k]
        k += 1
        for v in succ[u]:
            indeg[v] -= 1
            if indeg[v] == 0 and not never[v]:
                order.append(v)
    if len(order) != int(live.sum()):
        raise DeadlockError("cyclic cross-rank wait in critical path")
    poff = np.zeros(V + 1, np.int32)
    poff[1:] = np.cumsum([len(p) for p in preds])
    pidx = np.fromiter((u for p in preds for u in sorted(p)), np.int32, count=int(poff[-1]))
    # n_vert entries: vertices of collective members' own (rank, node) slots are unused, -1 pads
    order = np.asarray(order + [-1] * (V - len(order)), np.int32)
    return dict(n_vert=V, order=order, vkind=vkind, va=va, vb=vb, vsend=vsend,
                vmsg=vmsg, pred_off=poff, pred_idx=pidx)
