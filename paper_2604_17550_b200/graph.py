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
