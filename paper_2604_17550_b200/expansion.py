"""EXPANDED comm mode, host side: lower collectives to point-to-point messages.

SURVEY.md 8(f) row 1.  The engine already runs SEND/RECV graphs (the message
phase, per-link FIFO and routes of simulator.py:177-200, :310-327); this
module produces them the way the reference does:

* :func:`expand` -- one collective node -> a per-rank schedule of SEND/RECV
  operations for RING, TREE or MESH_HIER (reference collectives.py:76-240);
* :func:`expand_collectives` -- every collective of a graph set replaced by
  its rank's operations, dependencies rewired (collectives.py:456-537);
* :func:`wire_bytes`, :func:`check_plan`, :func:`dataflow_check` -- the
  reference's accounting and plan checks (collectives.py:296-416).

A schedule is built as one flat list of messages in the reference's emission
order.  A rank's operation list is every message it sends or receives, in
that order, stably sorted by step (collectives.py:237-239), and node ids
follow it.  Parity: tests/test_expand.py compares the expanded graphs and
their simulations with golden fixtures made by the reference.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field
from typing import Optional

from .costs import CollectiveAlgo
from .errors import DeadlockError, InconsistentGroupsError, UnsupportedAlgoTopologyError
from .graph import CollectiveKind, Node, NodeKind, P2pSpec, WorkloadGraph
from .topology import TopologyKind


def _v(x):
    return getattr(x, "value", x)


@dataclass
class PlanOp:
    """One side of a message (collectives.py:50-59)."""
    kind: NodeKind                 # SEND or RECV
    peer: int
    nbytes: int
    chunk: int                     # channel tag
    step: int
    reduce: bool
    slots: tuple


@dataclass
class P2pPlan:
    """A collective lowered to messages (collectives.py:62-73)."""
    kind: CollectiveKind
    algo: CollectiveAlgo
    group: list
    num_slots: int
    ops: dict = field(default_factory=dict)

    def send_count(self, rank: int) -> int:
        return sum(o.kind == NodeKind.SEND for o in self.ops.get(rank, []))

    def bytes_sent(self, rank: int) -> int:
        return sum(o.nbytes for o in self.ops.get(rank, []) if o.kind == NodeKind.SEND)


class _Msgs:
    """Messages in emission order: (src, dst, nbytes, chunk, step, reduce, slots)."""

    def __init__(self):
        self.m = []

    def add(self, src, dst, nbytes, chunk, step, reduce, slots):
        self.m.append((src, dst, nbytes, chunk, step, reduce, slots))

    def plan(self, kind, algo, group, num_slots, ranks) -> P2pPlan:
        ops = {r: [] for r in ranks}
        for src, dst, nb, ch, st, red, sl in self.m:
            ops[src].append(PlanOp(NodeKind.SEND, dst, nb, ch, st, red, sl))
            ops[dst].append(PlanOp(NodeKind.RECV, src, nb, ch, st, red, sl))
        for r in ops:
            ops[r].sort(key=lambda o: o.step)          # stable
        return P2pPlan(kind, algo, list(group), num_slots, ops)


def chunk_sizes(total: int, n: int) -> list:
    """total bytes in n pieces, the remainder spread over the first ones (collectives.py:76-79)."""
    q, r = divmod(total, n)
    return [q + 1] * r + [q] * (n - r)


# ---- RING (collectives.py:88-119): position i sends to i+1 every step

def _ring(ms: _Msgs, group, sizes, step0: int, reduce: bool) -> int:
    n = len(group)
    lag = 1 if reduce else 0           # reduce-scatter trails the all-gather by one chunk
    for s in range(n - 1):
        for i in range(n):
            c = (i - s - lag) % n
            ms.add(group[i], group[(i + 1) % n], sizes[c], c, step0 + s, reduce, (c,))
    return step0 + n - 1


def _ring_plan(kind, group, nbytes) -> P2pPlan:
    ms, n = _Msgs(), len(group)
    if kind == CollectiveKind.ALL_GATHER:
        _ring(ms, group, [nbytes] * n, 0, False)
    else:
        sizes = chunk_sizes(nbytes, n)
        nxt = _ring(ms, group, sizes, 0, True)
        if kind == CollectiveKind.ALL_REDUCE:
            _ring(ms, group, sizes, nxt, False)
    return ms.plan(kind, CollectiveAlgo.RING, group, n, group)


# ---- TREE (collectives.py:122-141): binomial reduce to position 0, mirrored broadcast

def _tree_plan(kind, group, nbytes) -> P2pPlan:
    if kind != CollectiveKind.ALL_REDUCE:
        raise UnsupportedAlgoTopologyError("TREE is defined for ALL_REDUCE only")
    n = len(group)
    rounds = max(1, (n - 1).bit_length())            # ceil(log2 n)
    edges = [(i, i - (1 << d), d) for d in range(rounds) for i in range(n)
             if i % (2 << d) == (1 << d)]
    every = tuple(range(n))
    ms = _Msgs()
    for a, b, d in edges:
        ms.add(group[a], group[b], nbytes, 0, d, True, every)
    for a, b, d in edges[::-1]:
        ms.add(group[b], group[a], nbytes, 0, 2 * rounds - 1 - d, False, every)
    return ms.plan(kind, CollectiveAlgo.TREE, group, n, group)


# ---- MESH_HIER (collectives.py:144-216): rings along rows, then columns, neighbour links only

def _line_reduce(ms: _Msgs, line, owner_slots, owner_bytes, step0: int) -> int:
    """Partials of piece j flow into line[j] from both ends, one hop per step."""
    k = len(line)
    for j in range(k):
        for i in range(j):
            ms.add(line[i], line[i + 1], owner_bytes[j], j, step0 + i, True, owner_slots[j])
        for i in range(k - 1, j, -1):
            ms.add(line[i], line[i - 1], owner_bytes[j], j, step0 + k - 1 - i, True, owner_slots[j])
    return step0 + max(k - 1, 0)


def _line_gather(ms: _Msgs, line, owner_slots, owner_bytes, step0: int) -> int:
    """Piece j spreads from line[j] to both ends, one hop per step."""
    k = len(line)
    for j in range(k):
        for i in range(j, k - 1):
            ms.add(line[i], line[i + 1], owner_bytes[j], j, step0 + i - j, False, owner_slots[j])
        for i in range(j, 0, -1):
            ms.add(line[i], line[i - 1], owner_bytes[j], j, step0 + j - i, False, owner_slots[j])
    return step0 + max(k - 1, 0)


def _mesh_plan(kind, group, nbytes, topo) -> P2pPlan:
    if _v(topo.kind) != TopologyKind.MESH2D.value:
        raise UnsupportedAlgoTopologyError("MESH_HIER requires a MESH2D topology")
    if sorted(group) != list(range(topo.world_size)):
        raise UnsupportedAlgoTopologyError(f"MESH_HIER expects the full mesh as the group, got {group}")
    R, C = topo.rows, topo.cols
    at = lambda r, c: r * C + c
    rows = [[at(r, c) for c in range(C)] for r in range(R)]
    cols = [[at(r, c) for r in range(R)] for c in range(C)]
    ms = _Msgs()
    if kind == CollectiveKind.ALL_GATHER:
        nxt = 0
        for line in rows:
            nxt = max(nxt, _line_gather(ms, line, [(x,) for x in line], [nbytes] * C, 0))
        for line in cols:
            _line_gather(ms, line, [tuple(rw) for rw in rows], [nbytes * C] * R, nxt)
        return ms.plan(kind, CollectiveAlgo.MESH_HIER, group, R * C, range(R * C))
    slot = chunk_sizes(nbytes, R * C)
    stripe = [tuple(cl) for cl in cols]                   # piece c of a row = column c's slots
    stripe_bytes = [sum(slot[s] for s in st) for st in stripe]
    t1 = 0
    for line in rows:
        t1 = max(t1, _line_reduce(ms, line, stripe, stripe_bytes, 0))
    own = [[(x,) for x in cl] for cl in cols]             # column phase: one slot per rank
    own_bytes = [[slot[x] for x in cl] for cl in cols]
    t2 = t1
    for c, line in enumerate(cols):
        t2 = max(t2, _line_reduce(ms, line, own[c], own_bytes[c], t1))
    if kind == CollectiveKind.ALL_REDUCE:
        t3 = t2
        for c, line in enumerate(cols):
            t3 = max(t3, _line_gather(ms, line, own[c], own_bytes[c], t2))
        for line in rows:
            _line_gather(ms, line, stripe, stripe_bytes, t3)
    return ms.plan(kind, CollectiveAlgo.MESH_HIER, group, R * C, range(R * C))


def expand(coll_node, algo, topo) -> P2pPlan:
    """Lower one collective node to per-rank SEND/RECV operations (collectives.py:219-240)."""
    spec = coll_node.coll
    if spec is None:
        raise ValueError(f"node {coll_node.node_id} is not a collective")
    if len(spec.group) < 2:
        raise ValueError(f"collective group must have at least 2 ranks, got {spec.group}")
    kind, a = CollectiveKind(_v(spec.kind)), _v(algo)
    if a == CollectiveAlgo.RING.value:
        return _ring_plan(kind, list(spec.group), spec.comm_bytes)
    if a == CollectiveAlgo.TREE.value:
        return _tree_plan(kind, list(spec.group), spec.comm_bytes)
    if a == CollectiveAlgo.MESH_HIER.value:
        return _mesh_plan(kind, list(spec.group), spec.comm_bytes, topo)
    raise UnsupportedAlgoTopologyError(f"unknown algorithm {algo}")


def wire_bytes(kind, comm_bytes: int, n: int, algo, mesh_shape: Optional[tuple] = None) -> int:
    """Bytes crossing links, summed over the group (collectives.py:296-318)."""
    if n <= 1:
        return 0
    kind, a, s = CollectiveKind(_v(kind)), _v(algo), comm_bytes
    if a == CollectiveAlgo.TREE.value:
        return 2 * (n - 1) * s
    if a == CollectiveAlgo.MESH_HIER.value:
        if not mesh_shape:
            raise UnsupportedAlgoTopologyError("MESH_HIER byte accounting needs the mesh shape")
        r, c = mesh_shape
        row = r * (c - 1) * s
        if kind == CollectiveKind.ALL_GATHER:
            return row * c + c * (r - 1) * r * c * s
        col = c * (r - 1) * (s // c)
        return 2 * row + 2 * col if kind == CollectiveKind.ALL_REDUCE else row + col
    if kind == CollectiveKind.ALL_GATHER:
        return n * (n - 1) * s
    return (2 if kind == CollectiveKind.ALL_REDUCE else 1) * (n - 1) * s


def check_plan(plan: P2pPlan, topo=None) -> list:
    """SEND/RECV pairing per channel, and neighbour-only messages for MESH_HIER (collectives.py:390-416)."""
    chan: dict = {}
    for r, ops in plan.ops.items():
        for o in ops:
            key = (r, o.peer, o.chunk) if o.kind == NodeKind.SEND else (o.peer, r, o.chunk)
            chan.setdefault(key, ([], []))[o.kind != NodeKind.SEND].append(o)
    problems = []
    for key, (ss, rr) in chan.items():
        if len(ss) != len(rr):
            problems.append(f"channel {key}: {len(ss)} sends vs {len(rr)} recvs")
            continue
        problems += [f"channel {key}: mismatched send/recv ({a} vs {b})"
                     for a, b in zip(ss, rr) if a.nbytes != b.nbytes or a.step != b.step]
    if _v(plan.algo) == CollectiveAlgo.MESH_HIER.value and topo is not None:
        mesh = _v(topo.kind) == TopologyKind.MESH2D.value

        def adjacent(a, b):                                  # topology.py:61-66
            if not mesh:
                return a != b
            (r0, c0), (r1, c1) = divmod(a, topo.cols), divmod(b, topo.cols)
            return abs(r0 - r1) + abs(c0 - c1) == 1
        problems += [f"non-adjacent message {r}->{o.peer}" for r, ops in plan.ops.items() for o in ops
                     if not adjacent(r, o.peer)]
    return problems


def dataflow_check(plan: P2pPlan) -> bool:
    """Run the plan on symbolic values and check the collective's postcondition
    (collectives.py:325-387): position p contributes p+1."""
    group, n = plan.group, len(plan.group)
    pos = {r: i for i, r in enumerate(group)}
    gather = plan.kind == CollectiveKind.ALL_GATHER
    val = {r: [(pos[r] + 1 if s == pos[r] else None) if gather else pos[r] + 1 for s in range(plan.num_slots)]
           for r in group}
    done = {r: [False] * len(plan.ops.get(r, [])) for r in group}
    left = sum(map(len, done.values()))
    wire: dict = {}
    while left:
        moved = False
        for r in sorted(plan.ops):
            ops = plan.ops[r]
            for i, o in enumerate(ops):
                if done[r][i] or any(not done[r][j] and ops[j].step < o.step for j in range(len(ops))):
                    continue
                if o.kind == NodeKind.SEND:
                    wire.setdefault((r, o.peer, o.chunk), deque()).append({s: val[r][s] for s in o.slots})
                else:
                    q = wire.get((o.peer, r, o.chunk))
                    if not q:
                        continue
                    for s, x in q.popleft().items():
                        if not o.reduce:
                            val[r][s] = x
                        else:
                            val[r][s] = None if val[r][s] is None or x is None else val[r][s] + x
                done[r][i] = True
                left -= 1
                moved = True
        if not moved:
            stuck = [(r, i) for r in done for i, d in enumerate(done[r]) if not d]
            raise DeadlockError(f"plan stalled with {left} ops pending, e.g. {stuck[:4]}")
    total = n * (n + 1) // 2
    if plan.kind == CollectiveKind.ALL_REDUCE:
        return all(x == total for r in group for x in val[r])
    if gather:
        return all(val[r][s] == s + 1 for r in group for s in range(plan.num_slots))
    return all(val[r][pos[r]] == total for r in group)


def collective_instances(graphs) -> list:
    """k-th COLL of every member rank -> one instance, checked for agreement (collectives.py:419-453)."""
    colls = {g.rank: [n for n in g.nodes if _v(n.kind) == "COLL"] for g in graphs}
    nxt = dict.fromkeys(sorted(colls), 0)
    out = []
    while True:
        lead_rank = next((r for r in nxt if nxt[r] < len(colls[r])), None)
        if lead_rank is None:
            return out
        lead = colls[lead_rank][nxt[lead_rank]]
        members = [lead]
        for r in lead.coll.group:
            if r == lead_rank:
                continue
            if r not in colls or nxt[r] >= len(colls[r]):
                raise InconsistentGroupsError(
                    f"rank {r} is missing collective #{nxt.get(r, 0)} of group {lead.coll.group}")
            o = colls[r][nxt[r]]
            if (_v(o.coll.kind), list(o.coll.group), o.coll.comm_bytes) != \
                    (_v(lead.coll.kind), list(lead.coll.group), lead.coll.comm_bytes):
                raise InconsistentGroupsError(f"rank {r} node {o.node_id} disagrees with rank {lead_rank} "
                                              f"node {lead.node_id}: {o.coll} vs {lead.coll}")
            members.append(o)
        for r in lead.coll.group:
            nxt[r] += 1
        out.append(members)


def expand_collectives(graphs, algo, topo) -> list:
    """Every COLL replaced by its rank's operations of the instance's plan
    (collectives.py:456-537).  The first step's operations inherit the
    collective's inputs and dependencies, each later step depends on the whole
    previous step, and the last operation carries the outputs, waits for its
    own step and stands in for the collective in its dependents."""
    plan_of = {}
    for members in collective_instances(graphs):
        p = expand(members[0], algo, topo)
        for r, m in zip(members[0].coll.group, members):
            plan_of[(r, m.node_id)] = p
    out = []
    for g in graphs:
        ids, span, nid = {}, {}, 0
        for n in g.nodes:
            p = plan_of.get((g.rank, n.node_id)) if _v(n.kind) == "COLL" else None
            cnt = len(p.ops.get(g.rank, [])) if p is not None else 1
            span[n.node_id] = nid
            ids[n.node_id] = nid + cnt - 1           # dependents of a collective wait for its last op
            nid += cnt
        data = lambda deps: sorted({ids[d] for d in deps})
        ctrl = lambda deps: sorted({(ids[d], lbl) for d, lbl in deps})
        nodes = []
        for n in g.nodes:
            p = plan_of.get((g.rank, n.node_id)) if _v(n.kind) == "COLL" else None
            if p is None:
                nodes.append(Node(ids[n.node_id], n.kind, n.op_name, inputs=list(n.inputs), outputs=list(n.outputs),
                                  data_deps=data(n.data_deps), ctrl_deps=ctrl(n.ctrl_deps),
                                  duration_ns=n.duration_ns, coll=n.coll, p2p=n.p2p,
                                  flops=getattr(n, "flops", None)))
                continue
            ops = p.ops.get(g.rank, [])
            b0 = span[n.node_id]
            last = b0 + len(ops) - 1
            layer: dict = {}
            for j, o in enumerate(ops):
                layer.setdefault(o.step, []).append(b0 + j)
            steps = sorted(layer)
            prev = dict(zip(steps[1:], steps))
            for j, o in enumerate(ops):
                me = b0 + j
                if o.step == (steps[0] if steps else 0):
                    dd, cd, ins = data(n.data_deps), ctrl(n.ctrl_deps), list(n.inputs)
                else:
                    dd, cd, ins = sorted(layer[prev[o.step]]), [], []
                outs = []
                if me == last:
                    outs = list(n.outputs)
                    dd = sorted(set(dd).union(x for x in layer[o.step] if x != me))
                kind = NodeKind.SEND if o.kind == NodeKind.SEND else NodeKind.RECV
                nodes.append(Node(me, kind, "send" if kind == NodeKind.SEND else "recv", inputs=ins, outputs=outs,
                                  data_deps=dd, ctrl_deps=cd, p2p=P2pSpec(o.peer, o.nbytes, o.chunk)))
        meta = dict(g.meta)
        meta["passes"] = list(meta.get("passes", [])) + [{"pass": "expand_collectives", "algo": _v(algo)}]
        out.append(WorkloadGraph(g.rank, g.world_size, nodes, dict(g.tensors), meta))
    return out
