"""Random multi-rank graphs that stress the scheduler's tie rules.

Unlike the reference's random_world_graphs (symmetric ranks, positive
durations), these give every rank its own node list and durations drawn from
a tiny set (0, 5, 10, 15 ns), so equal-time events across ranks -- the
cross-rank start-phase race of SURVEY.md Appendix A.3 -- happen constantly.
They also mix HOST launch twins, zero-duration collectives, collectives
over sub-groups, shuffled node-list order and sparse node ids.
"""

from __future__ import annotations

import random

from paper_2604_17550_b200.graph import (CollectiveKind, CollSpec, Dtype, Node, NodeKind, TensorMeta,
                                         WorkloadGraph)
from paper_2604_17550_b200.topology import Topology

KINDS = [CollectiveKind.ALL_REDUCE, CollectiveKind.ALL_GATHER, CollectiveKind.REDUCE_SCATTER]


def random_graphs(seed: int, max_world: int = 6, max_nodes: int = 24, p_zero: float = 0.25,
                  subgroups: bool = True, shuffle: bool = True, sparse_ids: bool = True, min_world: int = 1):
    rng = random.Random(seed)
    world = rng.randint(min_world, max_world)
    n_inst = rng.randint(0, 4)
    insts = []
    for _ in range(n_inst):
        if subgroups and world > 2 and rng.random() < 0.3:
            lo = rng.randrange(world - 1)
            g = [lo] + sorted(rng.sample(range(lo + 1, world), rng.randint(1, world - lo - 1)))
        else:
            g = list(range(world))
        nbytes = rng.choice([0, 4, 64, 1000, 4096]) if rng.random() < 0.3 else rng.randrange(4, 8192, 4)
        insts.append((rng.choice(KINDS if rng.random() < 0.5 else KINDS[:1]), g, nbytes))
    graphs = []
    for rank in range(world):
        nodes, tensors, produced = [], {}, []
        my = [i for i, (_, g, _) in enumerate(insts) if rank in g]
        n_comp = rng.randint(1, max_nodes)
        slots = sorted(rng.sample(range(n_comp + len(my)), len(my))) if my else []
        nid = 0
        step = lambda: rng.randint(1, 3) if sparse_ids else 1
        inputs = []
        for _ in range(rng.randint(0, 2)):
            t = len(tensors)
            tensors[t] = TensorMeta.make(t, [rng.randint(1, 64)], Dtype.F32)
            inputs.append(t)
        produced.extend((None, t) for t in inputs)
        k_inst = 0
        for pos in range(n_comp + len(my)):
            ins = [t for _, t in rng.sample(produced, min(len(produced), rng.randint(0, 3)))]
            deps = sorted({p for p, t in produced if t in ins and p is not None})
            extra = [p.node_id for p in rng.sample(nodes, min(len(nodes), rng.randint(0, 1)))
                     if p.kind != NodeKind.HOST]
            deps = sorted(set(deps) | set(extra))
            out = len(tensors)
            tensors[out] = TensorMeta.make(out, [rng.randint(1, 256)], Dtype.F32)
            ctrl = []
            if rng.random() < 0.5:
                nodes.append(Node(nid, NodeKind.HOST, "launch"))
                ctrl = [(nid, "launch")]
                nid += step()
            if k_inst < len(my) and pos == slots[k_inst]:
                kind, g, nbytes = insts[my[k_inst]]
                k_inst += 1
                nodes.append(Node(nid, NodeKind.COLL, kind.value.lower(), inputs=ins, outputs=[out],
                                  data_deps=deps, ctrl_deps=ctrl, coll=CollSpec(kind, list(g), nbytes)))
            else:
                d = rng.choice([0, 5, 10, 15]) if rng.random() < p_zero * 2 else rng.choice([5, 10, 15, 20, 40])
                nodes.append(Node(nid, NodeKind.COMP, "work", inputs=ins, outputs=[out], data_deps=deps,
                                  ctrl_deps=ctrl, duration_ns=d))
            produced.append((nid, out))
            nid += step()
        if shuffle and rng.random() < 0.3:
            # keep COLL relative order (instance matching follows list order)
            colls = [n for n in nodes if n.kind == NodeKind.COLL]
            rest = [n for n in nodes if n.kind != NodeKind.COLL]
            rng.shuffle(rest)
            merged, ci = [], 0
            for n in nodes:
                if n.kind == NodeKind.COLL:
                    merged.append(colls[ci]); ci += 1
                else:
                    merged.append(rest.pop())
            nodes = merged
        graphs.append(WorkloadGraph(rank, world, nodes, tensors, {"graph_inputs": inputs}))
    if rng.random() < 0.3:
        rng.shuffle(graphs)
    lat = rng.choice([0, 1, 10, 100])
    bw = rng.choice([1e9, 4e9, 1e12])
    return graphs, Topology.switch(world, bw, lat)


def random_p2p_graphs(seed: int, mesh: bool = False, world: int = 0, n_msgs: int = 10):
    """Ranks exchanging point-to-point messages (expanded comm mode): random
    SEND/RECV pairs on shared channels, interleaved with compute and an
    optional collective; links are contended and some graphs deadlock."""
    from paper_2604_17550_b200.graph import P2pSpec
    rng = random.Random(seed)
    if mesh:
        rows, cols = rng.choice([(1, 2), (2, 2), (2, 3)])
        world = rows * cols
    elif not world:
        world = rng.randint(2, 5)
    msgs = []
    for _ in range(rng.randint(1, n_msgs)):
        a, b = rng.sample(range(world), 2)
        msgs.append((a, b, rng.randint(0, 2), rng.choice([0, 8, 100, 1000, 4096])))
    per_rank = [[] for _ in range(world)]
    for mi, (a, b, tag, nb) in enumerate(msgs):
        per_rank[a].append(("send", mi))
        per_rank[b].append(("recv", mi))
    graphs = []
    for rank in range(world):
        ops = per_rank[rank]
        rng.shuffle(ops)
        nodes, tensors = [], {}
        last = None
        nid = 0
        for kind, mi in ops:
            if rng.random() < 0.6:
                out = len(tensors)
                tensors[out] = TensorMeta.make(out, [rng.randint(1, 64)], Dtype.F32)
                deps = [last] if last is not None and rng.random() < 0.7 else []
                nodes.append(Node(nid, NodeKind.COMP, "work", outputs=[out], data_deps=deps,
                                  duration_ns=rng.choice([0, 5, 10, 40])))
                last = nid
                nid += 1
            a, b, tag, nb = msgs[mi]
            deps = [last] if last is not None and rng.random() < 0.6 else []
            if kind == "send":
                nodes.append(Node(nid, NodeKind.SEND, "send", data_deps=deps, p2p=P2pSpec(b, nb, tag)))
            else:
                out = len(tensors)
                tensors[out] = TensorMeta.make(out, [max(1, nb // 4)], Dtype.F32)
                nodes.append(Node(nid, NodeKind.RECV, "recv", outputs=[out], data_deps=deps, p2p=P2pSpec(a, nb, tag)))
            if rng.random() < 0.5:
                last = nid
            nid += 1
        graphs.append(WorkloadGraph(rank, world, nodes, tensors, {"graph_inputs": []}))
    lat = rng.choice([0, 5, 10])
    bw = rng.choice([1e9, 2e9])
    topo = Topology.mesh2d(rows, cols, bw, lat) if mesh else Topology.switch(world, bw, lat)
    return graphs, topo


def random_spmd_graphs(seed: int, world: int, n_nodes: int = 24, p_coll: float = 0.3, per_rank_dur: bool = True):
    """One random DAG shared by every rank (same node ids, same dependencies), whose
    collectives all span the world -- the structure of data-parallel and FSDP graphs, and
    the one cluster design points reserve without instance state in HBM (engine.cu
    cl_step_clic).  Durations are drawn per rank (0, 5, 10, 15 ns, so ranks complete their
    part of an instance at different steps and many collectives complete together) or shared."""
    rng = random.Random(seed)
    tmpl = []                           # (kind, deps, coll kind, bytes, launch twin)
    for i in range(n_nodes):
        deps = sorted(rng.sample(range(i), min(i, rng.randint(0, 3))))
        if rng.random() < p_coll:
            kind = rng.choice(KINDS if rng.random() < 0.5 else KINDS[:1])
            nbytes = rng.choice([0, 64, 4096, 1 << 20]) if rng.random() < 0.3 else rng.randrange(4, 8192, 4)
            tmpl.append(("coll", deps, kind, nbytes, rng.random() < 0.3))
        else:
            tmpl.append(("comp", deps, None, 0, rng.random() < 0.3))
    shared = [rng.choice([0, 5, 10, 15]) for _ in range(n_nodes)]
    graphs = []
    group = list(range(world))
    for rank in range(world):
        nodes, tensors = [], {}
        ids = {}
        nid = 0
        for i, (kind, deps, ck, nbytes, twin) in enumerate(tmpl):
            ctrl = []
            if twin:
                nodes.append(Node(nid, NodeKind.HOST, "launch"))
                ctrl = [(nid, "launch")]
                nid += 1
            tensors[i] = TensorMeta.make(i, [4], Dtype.F32)
            data = sorted(ids[d] for d in deps)
            ins = list(deps)
            if kind == "coll":
                nodes.append(Node(nid, NodeKind.COLL, ck.value.lower(), inputs=ins, outputs=[i], data_deps=data,
                                  ctrl_deps=ctrl, coll=CollSpec(ck, group, nbytes)))
            else:
                d = rng.choice([0, 5, 10, 15]) if per_rank_dur else shared[i]
                nodes.append(Node(nid, NodeKind.COMP, "work", inputs=ins, outputs=[i], data_deps=data,
                                  ctrl_deps=ctrl, duration_ns=d))
            ids[i] = nid
            nid += 1
        graphs.append(WorkloadGraph(rank, world, nodes, tensors, {"graph_inputs": []}))
    lat = rng.choice([0, 1, 10, 100])
    bw = rng.choice([1e9, 4e9, 1e12])
    return graphs, Topology.switch(world, bw, lat)
