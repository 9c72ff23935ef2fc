"""Scheduling rewrites of one rank graph, as sweep axes.

* :func:`reorder_allgather` -- FSDP weight gathers prefetched k layers early
  (reference passes.py:53-110);
* :func:`bucket_allreduce` -- consecutive gradient ALL_REDUCEs fused under a
  byte cap (passes.py:113-212);
* :func:`verify_pass_safety` -- work, dataflow and collective volume kept
  (passes.py:215-277).

Every (pass, parameter) value gives a new graph structure; the engine
evaluates each structure over the design points in one launch
(:func:`paper_2604_17550_b200.sweep.sweep_rows` ``passes=``).  Parity:
tests/test_passes.py against fixtures made by the reference.
"""

from __future__ import annotations

from dataclasses import replace
from typing import Optional

from .errors import UnsupportedComboError
from .graph import CollectiveKind, CollSpec, WorkloadGraph, topo_order, validate_graph

DEFAULT_PREFETCH = 1
DEFAULT_BUCKET_CAP = 25 * 2 ** 20          # 25 MiB
SYNC_LABELS = ("fsdp-sync", "prefetch-gate")


def _v(x):
    return getattr(x, "value", x)


def _is_coll(n, kind: str) -> bool:
    return _v(n.kind) == "COLL" and _v(n.coll.kind) == kind


def _with_pass(g, nodes, entry) -> WorkloadGraph:
    meta = dict(g.meta)
    meta["passes"] = list(meta.get("passes", [])) + [entry]
    return WorkloadGraph(g.rank, g.world_size, nodes, dict(g.tensors), meta)


def ancestor_masks(g) -> dict:
    """node id -> bitset (python int) of its strict ancestors (passes.py:34-43)."""
    nmap = {n.node_id: n for n in g.nodes}
    masks: dict = {}
    for nid in topo_order(g):
        m = 0
        for d in nmap[nid].dep_ids():
            m |= masks[d] | (1 << d)
        masks[nid] = m
    return masks


def _launch_twin(n) -> Optional[int]:
    return next((d for d, lbl in n.ctrl_deps if lbl == "launch"), None)


def reorder_allgather(g, k: int = DEFAULT_PREFETCH):
    """Re-anchor every ALL_GATHER's layer-boundary gate k gathers earlier.

    Gathers of one shard tensor pair up: the first is the forward fetch, the
    rest backward re-fetches.  Within the forward and the backward sequence,
    gather i takes the gate of gather i-k (forward gathers before the start
    lose it, backward ones clamp to the first backward gate), and all gathers
    are chained in issue order with "stream-order" edges."""
    if k < 0:
        raise ValueError("prefetch distance must be non-negative")
    ags = sorted((n for n in g.nodes if _is_coll(n, "ALL_GATHER")), key=lambda n: n.node_id)
    if k == 0 or not ags:
        return g, {"gathers": len(ags), "moved": 0, "k": k}
    shards: dict = {}
    for n in ags:
        shards.setdefault(n.inputs[0], []).append(n)
    fwd = sorted((s[0] for s in shards.values()), key=lambda n: n.node_id)
    bwd = sorted((n for s in shards.values() for n in s[1:]), key=lambda n: n.node_id)
    gate = lambda n: next((d for d, lbl in n.ctrl_deps if lbl in SYNC_LABELS), None)
    nodes = {n.node_id: n for n in g.nodes}
    moved, prev = 0, None
    for seq, clamp in ((fwd, False), (bwd, True)):
        gates = [gate(n) for n in seq]
        for i, n in enumerate(seq):
            j = max(i - k, 0) if clamp else i - k
            new_gate = gates[j] if j >= 0 else None
            ctrl = [(d, lbl) for d, lbl in n.ctrl_deps if lbl not in SYNC_LABELS + ("stream-order",)]
            if new_gate is not None:
                ctrl.append((new_gate, "prefetch-gate"))
            if prev is not None:
                ctrl.append((prev, "stream-order"))
            prev = n.node_id
            moved += new_gate != gates[i]
            nodes[n.node_id] = replace(n, ctrl_deps=ctrl)
    out = _with_pass(g, [nodes[i] for i in sorted(nodes)], {"pass": "reorder_allgather", "k": k})
    return out, {"gathers": len(ags), "moved": moved, "k": k}


def _buckets(ars, masks, cap: int) -> list:
    """Greedy packing in list order: a bucket closes on cap overflow, another
    group, or a member that depends on an earlier member."""
    out, cur, size, members = [], [], 0, 0
    for n in ars:
        b = n.coll.comm_bytes
        if cur and size + b <= cap and n.coll.group == cur[0].coll.group and not masks[n.node_id] & members:
            cur.append(n)
            size += b
        else:
            if cur:
                out.append(cur)
            cur, size, members = [n], b, 0
        members |= 1 << n.node_id
    out.append(cur)
    return out


def bucket_allreduce(g, cap_bytes: int = DEFAULT_BUCKET_CAP):
    """Fuse consecutive ALL_REDUCEs into buckets of at most cap_bytes.

    A bucket becomes one collective (and its launch twin) at the position of
    its last member; the other members and their twins are dropped, and their
    dependents are rewired to the bucket's nodes.  Ids are renumbered densely
    in list order.  Total bytes are conserved."""
    if cap_bytes <= 0:
        raise ValueError("bucket cap must be positive")
    ars = [n for n in g.nodes if _is_coll(n, "ALL_REDUCE")]
    total = sum(n.coll.comm_bytes for n in ars)
    if len(ars) < 2:
        return g, {"buckets": len(ars), "merged": 0, "bytes": total}
    buckets = _buckets(ars, ancestor_masks(g), cap_bytes)
    nmap = {n.node_id: n for n in g.nodes}
    drop: set = set()
    fused: dict = {}        # kept id (last member, its twin) -> (twin node, collective node)
    alias: dict = {}        # dropped id -> (twin id, last member id)
    for mem in buckets:
        if len(mem) < 2:
            continue
        last = mem[-1]
        twin = _launch_twin(last)
        for m in mem[:-1]:
            h = _launch_twin(m)
            drop.add(m.node_id)
            alias[m.node_id] = (twin, last.node_id)
            if h is not None:
                drop.add(h)
                alias[h] = (twin, last.node_id)
        ctrl = sorted({(d, lbl) for m in mem for d, lbl in m.ctrl_deps if lbl != "launch" and d not in drop})
        data = {d for m in mem for d in m.data_deps}
        host = replace(nmap[twin], op_name="all_reduce")
        coll = replace(last, inputs=[t for m in mem for t in m.inputs], outputs=[t for m in mem for t in m.outputs],
                       data_deps=sorted(data - drop), ctrl_deps=[(twin, "launch")] + ctrl,
                       coll=CollSpec(CollectiveKind.ALL_REDUCE, list(last.coll.group),
                                     sum(m.coll.comm_bytes for m in mem)))
        fused[last.node_id] = fused[twin] = (host, coll)
    ids, kept = {}, []
    for n in g.nodes:
        if n.node_id in drop:
            continue
        ids[n.node_id] = len(kept)
        f = fused.get(n.node_id)
        kept.append(n if f is None else f[1] if _v(n.kind) == "COLL" else f[0])
    for old, (h, c) in alias.items():
        ids[old] = ids[h] if _v(nmap[old].kind) == "HOST" else ids[c]
    nodes = [replace(n, node_id=i, data_deps=sorted({ids[d] for d in n.data_deps}),
                     ctrl_deps=sorted({(ids[d], lbl) for d, lbl in n.ctrl_deps})) for i, n in enumerate(kept)]
    out = _with_pass(g, nodes, {"pass": "bucket_allreduce", "cap_bytes": cap_bytes})
    left = sum(_is_coll(n, "ALL_REDUCE") for n in nodes)
    return out, {"buckets": len(buckets), "merged": len(ars) - left, "bytes": total}


def verify_pass_safety(before, after) -> list:
    """Violations of a rewrite: invalid result, changed tensors, changed compute,
    changed collective bytes per kind, or a lost data dependency (passes.py:215-277)."""
    bad = [f"invalid-after: {v}" for v in validate_graph(after)]
    if bad:
        return bad
    if before.tensors != after.tensors:
        bad.append("tensor-table-changed")

    def comp(g):
        return {tuple(n.outputs): (n.op_name, n.duration_ns, tuple(sorted(n.inputs)))
                for n in g.nodes if _v(n.kind) == "COMP"}
    cb, ca = comp(before), comp(after)
    if cb != ca:
        bad += [f"compute-changed: outputs {list(k)}" for k in sorted(set(cb) ^ set(ca))]
        bad += [f"compute-changed: outputs {list(k)}" for k in sorted(set(cb) & set(ca)) if cb[k] != ca[k]]

    def volume(g):
        v: dict = {}
        for n in g.nodes:
            if _v(n.kind) == "COLL":
                v[_v(n.coll.kind)] = v.get(_v(n.coll.kind), 0) + n.coll.comm_bytes
        return v
    if volume(before) != volume(after):
        bad.append(f"collective-bytes-changed: {volume(before)} -> {volume(after)}")
    made_by = {}
    for n in after.nodes:
        for t in n.outputs:
            made_by[t] = n.node_id
    try:
        masks = ancestor_masks(after)
    except Exception as exc:
        bad.append(f"after-not-orderable: {exc}")
        return bad
    bmap = {n.node_id: n for n in before.nodes}
    for v in before.nodes:
        if not v.outputs:
            continue
        iv = made_by.get(v.outputs[0])
        if iv is None:
            bad.append(f"lost-producer: tensor {v.outputs[0]}")
            continue
        for d in v.data_deps:
            u = bmap[d]
            if not u.outputs:
                continue                    # launch twin; its collective is checked
            iu = made_by.get(u.outputs[0])
            if iu is None:
                bad.append(f"lost-producer: tensor {u.outputs[0]}")
            elif iu != iv and not masks[iv] >> iu & 1:
                bad.append(f"lost-dep: node {v.node_id} no longer reaches producer of tensor {u.outputs[0]}")
    return bad


def apply_pass(graphs, spec: str) -> list:
    """A sweep-axis value applied to every rank graph: "none",
    "reorder-allgather:<k>" or "bucket-allreduce:<cap bytes>" (the reference
    CLI's ``pass`` subcommand names, cli.py:109-117)."""
    name, _, arg = spec.partition(":")
    try:
        val = int(arg) if arg else None
    except ValueError:
        raise UnsupportedComboError(f"pass {spec!r}: parameter must be an integer") from None
    if name == "none":
        return list(graphs)
    if name == "reorder-allgather":
        return [reorder_allgather(g, DEFAULT_PREFETCH if val is None else val)[0] for g in graphs]
    if name == "bucket-allreduce":
        return [bucket_allreduce(g, DEFAULT_BUCKET_CAP if val is None else val)[0] for g in graphs]
    raise UnsupportedComboError(f"unknown pass {spec!r} (none, reorder-allgather:<k>, bucket-allreduce:<bytes>)")
