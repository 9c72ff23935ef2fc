"""Decode the committed golden fixtures (tests/golden/*.json.gz) into graphs."""

from __future__ import annotations

import gzip
import hashlib
import json
from functools import lru_cache
from pathlib import Path

from paper_2604_17550_b200.graph import (CollectiveKind, CollSpec, Dtype, Node, NodeKind, P2pSpec,
                                         TensorMeta, WorkloadGraph)
from paper_2604_17550_b200.topology import Topology, TopologyKind

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def corpus() -> list:
    with gzip.open(GOLDEN / "corpus.json.gz", "rt") as f:
        return json.load(f)


@lru_cache(maxsize=None)
def synth_fixtures() -> dict:
    with gzip.open(GOLDEN / "synth.json.gz", "rt") as f:
        return json.load(f)


def decode_graphs(case) -> list:
    lists = []
    for nl in case["node_lists"]:
        nodes = []
        for nid, kind, op, ins, outs, dd, cd, dur, coll, p2p in nl:
            nodes.append(Node(nid, NodeKind(kind), op, inputs=list(ins), outputs=list(outs),
                              data_deps=list(dd), ctrl_deps=[tuple(c) for c in cd], duration_ns=dur,
                              coll=CollSpec(CollectiveKind(coll[0]), list(coll[1]), coll[2]) if coll else None,
                              p2p=P2pSpec(*p2p) if p2p else None))
        lists.append(nodes)
    out = []
    for g in case["graphs"]:
        tensors = {t[0]: TensorMeta(t[0], list(t[1]), Dtype(t[2]), t[3]) for t in g["tensors"]}
        out.append(WorkloadGraph(g["rank"], g["world_size"], lists[g["nodes"]], tensors,
                                 {"graph_inputs": g["graph_inputs"]}))
    return out


def decode_topo(t) -> Topology:
    return Topology(TopologyKind(t["kind"]), t["world_size"], float(t["bw"]), int(t["lat"]),
                    t.get("rows", 0), t.get("cols", 0))


def has_p2p(case) -> bool:
    return any(n[1] in ("SEND", "RECV") for nl in case["node_lists"] for n in nl)


def _v(x):
    return getattr(x, "value", x)


def canon(graphs) -> str:
    """sha256 of a graph set's canonical encoding (either package's classes)."""
    enc = []
    for g in graphs:
        nodes = [[n.node_id, _v(n.kind), n.op_name, list(n.inputs), list(n.outputs), list(n.data_deps),
                  [list(c) for c in n.ctrl_deps], n.duration_ns,
                  [_v(n.coll.kind), list(n.coll.group), n.coll.comm_bytes] if n.coll else None,
                  [n.p2p.peer_rank, n.p2p.comm_bytes, n.p2p.channel_tag] if n.p2p else None] for n in g.nodes]
        enc.append([g.rank, g.world_size, nodes, sorted(g.tensors), g.meta.get("passes")])
    return hashlib.sha256(json.dumps(enc, separators=(",", ":")).encode()).hexdigest()


@lru_cache(maxsize=None)
def expand_fixtures() -> dict:
    with gzip.open(GOLDEN / "expand.json.gz", "rt") as f:
        return json.load(f)
