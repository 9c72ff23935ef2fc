"""IR ingestion: captured raw operator exports -> workload graphs.

Restates the reference's ``raw-ir/1`` reader and ``convert``
(pkg/src/trainsim/traceio.py:186-465) with one addition: every analytically
costed COMP node keeps its flop count (``Node.flops``), so a design point can
re-cost the captured graph for another device on the GPU (the engine's
``peak_flops``/``efficiency`` columns) instead of re-ingesting it per point.

Lowering (traceio.py:322-338): a compute call becomes a HOST launch node plus
a COMP node joined by a "launch" control edge; a collective call becomes
HOST + COLL; WAIT vanishes and consumers of the waited tensor depend on both
the HOST and the COLL node; PLACEHOLDERs become graph inputs and OUTPUT
records its dependency sets in meta["graph_outputs"].
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path
from typing import Optional

from .costs import DEFAULT_DEVICE, DeviceSpec, ProfileTable, duration_from_flops, op_flops, parse_dtype
from .errors import FormatError, MissingShapeError, UnknownOperatorError, UnresolvedReferenceError
from .graph import CollectiveKind, CollSpec, Node, NodeKind, TensorMeta, WorkloadGraph, tensor_bytes

RAW_FORMAT_VERSION = "raw-ir/1"
RAW_KINDS = ("PLACEHOLDER", "CALL", "WAIT", "OUTPUT")

# Operator table (the reference ships it as ops_map.json): target -> (op name, flop class)
_COMPUTE_BY_CLASS = {
    "matmul": {"addmm": ["aten.addmm"], "mm": ["aten.mm"], "bmm": ["aten.bmm"], "matmul": ["aten.matmul"],
               "linear": ["aten.linear"]},
    "attention": {"scaled_dot_product_attention": ["aten.scaled_dot_product_attention",
                                                   "aten._scaled_dot_product_flash_attention",
                                                   "aten._scaled_dot_product_efficient_attention"]},
    "elementwise": {"add": ["aten.add", "aten.add_"], "sub": ["aten.sub"], "mul": ["aten.mul"], "div": ["aten.div"],
                    "relu": ["aten.relu", "aten.relu_"], "gelu": ["aten.gelu"], "silu": ["aten.silu"],
                    "sigmoid": ["aten.sigmoid"], "tanh": ["aten.tanh"], "softmax": ["aten.softmax", "aten._softmax"],
                    "layer_norm": ["aten.layer_norm", "aten.native_layer_norm"], "sum": ["aten.sum"],
                    "mean": ["aten.mean"], "threshold_backward": ["aten.threshold_backward"],
                    "gelu_backward": ["aten.gelu_backward"], "silu_backward": ["aten.silu_backward"],
                    "ones_like": ["aten.ones_like"], "zeros_like": ["aten.zeros_like"]},
}
COMPUTE = {t: (op, cls) for cls, ops in _COMPUTE_BY_CLASS.items() for op, ts in ops.items() for t in ts}
_COLL_KINDS = {"all_reduce": ("ALL_REDUCE", ["all_reduce", "all_reduce_"]),
               "all_gather": ("ALL_GATHER", ["all_gather_into_tensor"]),
               "reduce_scatter": ("REDUCE_SCATTER", ["reduce_scatter_tensor"])}
COLLECTIVE = {f"{ns}.{name}": (op, kind)
              for op, (kind, names) in _COLL_KINDS.items() for name in names
              for ns in ("c10d", "c10d_functional", "_c10d_functional")
              if not (ns == "c10d_functional" and name == "all_reduce_")}
ELIDE = {"_operator.getitem"} | {f"aten.{v}" for v in ("_to_copy", "alias", "clone", "detach", "expand", "permute",
                                                        "reshape", "t", "transpose", "view")}


def normalize_target(target: str) -> str:
    """namespace.opname of an operator reference, overload dropped (traceio.py:213-221)."""
    t = target[len("torch.ops."):] if target.startswith("torch.ops.") else target
    parts = t.split(".")
    return ".".join(parts[:2]) if len(parts) >= 2 else t


@dataclass
class RawIrNode:
    name: str
    kind: str
    target: str
    arg_names: list
    tensor_out: Optional[dict] = None     # {"shape": [...], "dtype": tag}
    coll_attrs: Optional[dict] = None     # {"kind": tag, "group": [ranks]}


@dataclass
class RawExport:
    rank: int
    world_size: int
    nodes: list


def parse_raw_export(doc, source: str = "<memory>") -> RawExport:
    """A ``raw-ir/1`` document, checked like traceio.py:256-289."""
    if not isinstance(doc, dict):
        raise FormatError(f"{source}: raw export must be a JSON object")
    if doc.get("format_version") != RAW_FORMAT_VERSION:
        raise FormatError(f"{source}: unknown format_version {doc.get('format_version')!r}")
    try:
        rank, world = int(doc["rank"]), int(doc["world_size"])
    except (KeyError, TypeError, ValueError) as e:
        raise FormatError(f"{source}: bad rank/world_size: {e}") from e
    items = doc.get("nodes")
    if not isinstance(items, list) or not items:
        raise FormatError(f"{source}: node list is empty or missing")
    nodes, seen = [], set()
    for i, nd in enumerate(items):
        try:
            name, kind = str(nd["name"]), str(nd["kind"])
            target, args = str(nd.get("target", "")), [str(a) for a in nd.get("arg_names", [])]
        except (KeyError, TypeError) as e:
            raise FormatError(f"{source}: node {i} malformed: {e}") from e
        if kind not in RAW_KINDS:
            raise FormatError(f"{source}: node {name!r} has unknown kind {kind!r}")
        if name in seen:
            raise FormatError(f"{source}: duplicate node name {name!r}")
        unseen = next((a for a in args if a not in seen), None)
        if unseen is not None:
            raise UnresolvedReferenceError(f"{source}: node {name!r} references unseen name {unseen!r}")
        seen.add(name)
        nodes.append(RawIrNode(name, kind, target, args, nd.get("tensor_out"), nd.get("coll_attrs")))
    return RawExport(rank, world, nodes)


def read_raw_export(path) -> RawExport:
    try:
        doc = json.loads(Path(path).read_text())
    except (OSError, json.JSONDecodeError) as e:
        raise FormatError(f"cannot read raw export {path}: {e}") from e
    return parse_raw_export(doc, source=str(path))


def convert(raw: RawExport, profile: Optional[ProfileTable] = None,
            device: Optional[DeviceSpec] = None) -> WorkloadGraph:
    """Lower one rank's raw operator list to a workload graph (traceio.py:322-465)."""
    dev = device or (profile.device if profile else DEFAULT_DEVICE)
    nodes, tensors = [], {}
    env: dict = {}                 # raw name -> (tensor id or None, dependency node ids)
    waited: dict = {}              # collective output tensor -> (host id, coll id)
    g_in, g_out = [], []
    by_name = {rn.name: rn for rn in raw.nodes}

    def tensor(spec, owner):
        if not spec or "shape" not in spec or "dtype" not in spec:
            raise MissingShapeError(f"node {owner!r} carries no tensor shape")
        tm = TensorMeta.make(len(tensors), [int(d) for d in spec["shape"]] or [1], parse_dtype(str(spec["dtype"])))
        tensors[tm.tensor_id] = tm
        return tm

    def bound(rn):
        names = [a for a in rn.arg_names if env[a][0] is not None]
        return names, [env[a] for a in names]

    def shape_at(name, b):
        # an elided view between producer and use can change the rank: the
        # argument node's own recorded shape wins over the storage's
        spec = by_name[name].tensor_out if name in by_name else None
        if spec and "shape" in spec:
            return [int(d) for d in spec["shape"]] or [1]
        return tensors[b[0]].shape

    def pair(kind, op, ins, outs, deps, **extra):
        host = Node(len(nodes), NodeKind.HOST, op)
        nodes.append(host)
        work = Node(len(nodes), kind, op, inputs=ins, outputs=outs, data_deps=sorted(set(deps)),
                    ctrl_deps=[(host.node_id, "launch")], **extra)
        nodes.append(work)
        return host, work

    for rn in raw.nodes:
        if rn.kind == "PLACEHOLDER":
            tm = tensor(rn.tensor_out, rn.name)
            g_in.append(tm.tensor_id)
            env[rn.name] = (tm.tensor_id, [])
        elif rn.kind == "WAIT":
            _, args = bound(rn)
            if not args:
                raise FormatError(f"WAIT node {rn.name!r} has no tensor argument")
            t, deps = args[0]
            env[rn.name] = (t, list(waited[t]) if t in waited else list(deps))
        elif rn.kind == "OUTPUT":
            g_out += [{"tensor_id": t, "deps": sorted(set(deps))} for t, deps in bound(rn)[1]]
        else:
            target = normalize_target(rn.target)
            names, args = bound(rn)
            if target in ELIDE:
                if not args:
                    raise FormatError(f"elided call {rn.name!r} has no tensor argument")
                env[rn.name] = args[0]
            elif target in ("aten.copy", "aten.copy_"):
                # functionalized in-place write: the value is the source (last
                # argument); the destination's producers keep the ordering
                if not args:
                    raise FormatError(f"copy {rn.name!r} has no tensor argument")
                env[rn.name] = (args[-1][0], sorted({d for _, deps in args for d in deps}))
            elif target in COMPUTE:
                op, cls = COMPUTE[target]
                out = tensor(rn.tensor_out, rn.name)
                shapes = [shape_at(a, b) for a, b in zip(names, args)]
                dur = profile.lookup(op, shapes, out.dtype) if profile else None
                flops = None
                if dur is None:
                    flops = op_flops(cls, shapes, out.shape)
                    dur = duration_from_flops(flops, dev)
                _, comp = pair(NodeKind.COMP, op, [t for t, _ in args], [out.tensor_id],
                               [d for _, deps in args for d in deps], duration_ns=dur, flops=flops)
                env[rn.name] = (out.tensor_id, [comp.node_id])
            elif target in COLLECTIVE:
                op, kind = COLLECTIVE[target]
                if not args:
                    raise FormatError(f"collective {rn.name!r} has no tensor argument")
                attrs = rn.coll_attrs or {}
                if "group" not in attrs:
                    raise FormatError(f"collective {rn.name!r} carries no group ranks")
                if "kind" in attrs and str(attrs["kind"]) != kind:
                    raise FormatError(f"collective {rn.name!r}: coll_attrs kind {attrs['kind']!r} "
                                      f"contradicts target {target!r}")
                out = tensor(rn.tensor_out, rn.name)
                nbytes = tensor_bytes(shape_at(names[0], args[0]), tensors[args[0][0]].dtype)
                host, coll = pair(NodeKind.COLL, op, [t for t, _ in args], [out.tensor_id],
                                  [d for _, deps in args for d in deps],
                                  coll=CollSpec(CollectiveKind(kind), [int(r) for r in attrs["group"]], nbytes))
                waited[out.tensor_id] = (host.node_id, coll.node_id)
                env[rn.name] = (out.tensor_id, [coll.node_id])
            else:
                raise UnknownOperatorError(f"target {rn.target!r} (normalized {target!r}) is not mapped")
    meta = {"source": "capture", "graph_inputs": g_in, "graph_outputs": g_out}
    return WorkloadGraph(raw.rank, raw.world_size, nodes, tensors, meta)
