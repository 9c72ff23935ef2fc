"""Per-rank workload graph values (host side).

Field names and enum values are those of the reference's data model
(``pkg/src/trainsim/graph.py:19-133``) so that graphs built by either package
can be handed to :func:`paper_2604_17550_b200.simulate` unchanged; the engine
only reads attributes (duck typing), it never isinstance-checks.  The device
replica of these graphs is built by :mod:`paper_2604_17550_b200.store`.
"""

from __future__ import annotations

import heapq
import math
from dataclasses import dataclass, field
from enum import Enum
from typing import Optional


class Dtype(Enum):
    F32 = "f32"
    F16 = "f16"
    BF16 = "bf16"
    I64 = "i64"
    I32 = "i32"
    BOOL = "bool"

    @property
    def byte_width(self) -> int:
        return {"f32": 4, "f16": 2, "bf16": 2, "i64": 8, "i32": 4, "bool": 1}[self.value]


class NodeKind(Enum):
    HOST = "HOST"
    COMP = "COMP"
    COLL = "COLL"
    SEND = "SEND"
    RECV = "RECV"


class CollectiveKind(Enum):
    ALL_REDUCE = "ALL_REDUCE"
    ALL_GATHER = "ALL_GATHER"
    REDUCE_SCATTER = "REDUCE_SCATTER"


def tensor_bytes(shape, dtype: Dtype) -> int:
    return math.prod(shape) * dtype.byte_width


@dataclass
class TensorMeta:
    tensor_id: int
    shape: list
    dtype: Dtype
    bytes: int

    @classmethod
    def make(cls, tensor_id: int, shape, dtype: Dtype) -> "TensorMeta":
        return cls(tensor_id, list(shape), dtype, tensor_bytes(shape, dtype))


@dataclass
class CollSpec:
    kind: CollectiveKind
    group: list            # ordered global ranks
    comm_bytes: int        # input bytes (the shard for ALL_GATHER)


@dataclass
class P2pSpec:
    peer_rank: int
    comm_bytes: int
    channel_tag: int


@dataclass
class Node:
    node_id: int
    kind: NodeKind
    op_name: str
    inputs: list = field(default_factory=list)
    outputs: list = field(default_factory=list)
    data_deps: list = field(default_factory=list)
    ctrl_deps: list = field(default_factory=list)   # [(node_id, label)]
    duration_ns: Optional[int] = None
    coll: Optional[CollSpec] = None
    p2p: Optional[P2pSpec] = None
    # not in the reference model: the flop count behind an analytical
    # duration, kept by our graph families so a design point can re-cost the
    # node for another device ("per-op throughput axis").
    flops: Optional[int] = None

    def dep_ids(self) -> list:
        return list(self.data_deps) + [d for d, _ in self.ctrl_deps]


@dataclass
class WorkloadGraph:
    rank: int
    world_size: int
    nodes: list
    tensors: dict
    meta: dict

    def node_map(self) -> dict:
        return {n.node_id: n for n in self.nodes}

    def graph_inputs(self) -> set:
        return set(self.meta.get("graph_inputs", []))


def topo_order(g) -> list:
    """Kahn's order, lowest node id first (reference graph.py:282-306)."""
    from .errors import CyclicGraphError

    ids = {n.node_id for n in g.nodes}
    indeg = dict.fromkeys(ids, 0)
    succ: dict = {i: [] for i in ids}
    for n in g.nodes:
        for d in set(n.dep_ids()):
            if d in ids:
                indeg[n.node_id] += 1
                succ[d].append(n.node_id)
    ready = [i for i, c in indeg.items() if c == 0]
    heapq.heapify(ready)
    out = []
    while ready:
        i = heapq.heappop(ready)
        out.append(i)
        for s in succ[i]:
            indeg[s] -= 1
            if indeg[s] == 0:
                heapq.heappush(ready, s)
    if len(out) != len(ids):
        raise CyclicGraphError("graph has a dependency cycle; no topological order")
    return out


# ------------------------------------------------------------ validation


@dataclass
class Violation:
    """One broken structural rule (reference graph.py:137-150)."""
    rule: str
    detail: str
    node_id: Optional[int] = None
    tensor_id: Optional[int] = None

    def __str__(self) -> str:
        where = [f"node {self.node_id}"] * (self.node_id is not None) + \
                [f"tensor {self.tensor_id}"] * (self.tensor_id is not None)
        return f"[{self.rule}] {' @ '.join(where) or 'graph'}: {self.detail}"


def _kv(x):
    return getattr(x, "value", x)


def _cycle(g, nmap) -> Optional[list]:
    """One dependency cycle, found by an iterative depth-first walk over data and
    control edges in node-list order (reference graph.py:246-279)."""
    state = dict.fromkeys(nmap, 0)          # 0 unvisited, 1 on the path, 2 finished
    parent: dict = {}
    for root in nmap:
        if state[root]:
            continue
        state[root] = 1
        path = [(root, iter(nmap[root].dep_ids()))]
        while path:
            nid, deps = path[-1]
            for d in deps:
                if d not in state or d == nid:
                    continue
                if state[d] == 1:
                    cyc, cur = [d, nid], nid
                    while cur in parent and parent[cur] != d:
                        cur = parent[cur]
                        cyc.append(cur)
                    return cyc[::-1]
                if state[d] == 0:
                    state[d], parent[d] = 1, nid
                    path.append((d, iter(nmap[d].dep_ids())))
                    break
            else:
                state[nid] = 2
                path.pop()
    return None


def validate_graph(g) -> list:
    """Every structural invariant of a rank graph (reference graph.py:153-243)."""
    out = []
    seen = set()
    for n in g.nodes:
        if n.node_id in seen:
            out.append(Violation("duplicate-node-id", "node_id appears twice", node_id=n.node_id))
        seen.add(n.node_id)
    nmap = {n.node_id: n for n in g.nodes}
    ginputs = set(g.meta.get("graph_inputs", []))
    for tid, tm in g.tensors.items():
        if tid != tm.tensor_id:
            out.append(Violation("tensor-id-mismatch", f"table key {tid} != tensor_id {tm.tensor_id}", tensor_id=tid))
        if not tm.shape or min(tm.shape) <= 0:
            out.append(Violation("tensor-shape", f"shape must be non-empty positive ints, got {tm.shape}",
                                 tensor_id=tid))
        elif tm.bytes != math.prod(tm.shape) * Dtype(_kv(tm.dtype)).byte_width:
            want = math.prod(tm.shape) * Dtype(_kv(tm.dtype)).byte_width
            out.append(Violation("tensor-bytes", f"bytes {tm.bytes} != prod(shape)*width {want}", tensor_id=tid))
    prod: dict = {}
    for n in g.nodes:
        for t in n.outputs:
            prod.setdefault(t, []).append(n.node_id)
    out += [Violation("multi-producer", f"produced by nodes {ps}", tensor_id=t) for t, ps in prod.items() if len(ps) > 1]
    for n in g.nodes:
        kind = _kv(n.kind)
        if (n.coll is not None) != (kind == "COLL"):
            out.append(Violation("coll-presence", f"coll attrs on {kind} node", node_id=n.node_id))
        if (n.p2p is not None) != (kind in ("SEND", "RECV")):
            out.append(Violation("p2p-presence", f"p2p attrs on {kind} node", node_id=n.node_id))
        if n.duration_ns is not None:
            if kind != "COMP":
                out.append(Violation("duration-on-non-comp", f"duration on {kind} node", node_id=n.node_id))
            elif n.duration_ns < 0:
                out.append(Violation("negative-duration", f"duration {n.duration_ns}", node_id=n.node_id))
        for d in n.dep_ids():
            if d not in nmap:
                out.append(Violation("dangling-dep", f"dep on missing node {d}", node_id=n.node_id))
            elif d == n.node_id:
                out.append(Violation("self-dep", "node depends on itself", node_id=n.node_id))
        for t in list(n.inputs) + list(n.outputs):
            if t not in g.tensors:
                out.append(Violation("unknown-tensor", f"references tensor {t} not in table", node_id=n.node_id,
                                     tensor_id=t))
        # data deps = producers of the inputs, plus deps on HOST launch twins and
        # on SEND/RECV plan operations
        need = set()
        for t in n.inputs:
            if prod.get(t):
                need.add(prod[t][0])
            elif t not in ginputs and t in g.tensors:
                out.append(Violation("missing-producer", "consumed tensor has no producer and is not a graph input",
                                     node_id=n.node_id, tensor_id=t))
        have = set(n.data_deps)
        out += [Violation("missing-data-dep", f"input producer {m} not in data_deps", node_id=n.node_id)
                for m in sorted(need - have)]
        out += [Violation("spurious-data-dep", f"data_dep {x} is not an input producer", node_id=n.node_id)
                for x in sorted(have - need) if x in nmap and _kv(nmap[x].kind) not in ("HOST", "SEND", "RECV")]
        if n.coll is not None:
            grp = n.coll.group
            if not grp:
                out.append(Violation("empty-group", "collective group is empty", node_id=n.node_id))
            else:
                if g.rank not in grp:
                    out.append(Violation("rank-not-in-group", f"rank {g.rank} not in group {grp}", node_id=n.node_id))
                if any(r < 0 or r >= g.world_size for r in grp):
                    out.append(Violation("group-out-of-range", f"group {grp} outside world {g.world_size}",
                                         node_id=n.node_id))
            if n.coll.comm_bytes < 0:
                out.append(Violation("negative-comm-bytes", str(n.coll.comm_bytes), node_id=n.node_id))
        if n.p2p is not None and (n.p2p.peer_rank == g.rank or not 0 <= n.p2p.peer_rank < g.world_size):
            out.append(Violation("bad-peer", f"peer {n.p2p.peer_rank}", node_id=n.node_id))
    cyc = _cycle(g, nmap)
    if cyc:
        out.append(Violation("cycle", "dependency cycle through nodes " + "->".join(map(str, cyc))))
    return out
