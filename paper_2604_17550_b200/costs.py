"""Scalar cost-model helpers for graph construction on the host.

The engine never calls these: durations for a design point are computed on
the GPU by the cost stage of the sweep kernel (``csrc/engine.cu``,
``cost_*``), from the raw per-node flops / collective sizes and the design
point's bandwidth, latency, algorithm and device.  These scalar versions exist
because graph construction (the synthesizer, the reference's ``dur()`` at
``pkg/src/trainsim/synth.py:196-200``) bakes a ``duration_ns`` into each
node, exactly as the reference does, and because they are part of the public
API the reference exports.

Arithmetic order follows the reference line by line (fp64, no FMA is possible
in CPython): ``traceio.py:68-70`` (round half up), ``traceio.py:135-184``
(flops, analytical duration), ``collectives.py:243-293`` (alpha-beta forms).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass, field
from enum import Enum
from pathlib import Path
from typing import Optional

from .errors import (FormatError, MissingShapeError, UnknownOperatorError,
                     UnsupportedAlgoTopologyError)
from .graph import CollectiveKind, Dtype


class CollectiveAlgo(Enum):
    RING = "ring"
    TREE = "tree"
    MESH_HIER = "mesh-hier"


def round_half_up_ns(x: float) -> int:
    return int(math.floor(x + 0.5))


@dataclass
class DeviceSpec:
    peak_flops: float
    efficiency: float


DEFAULT_DEVICE = DeviceSpec(peak_flops=1.0e12, efficiency=1.0)


def shape_str(shapes) -> str:
    return "x".join("[" + ",".join(str(d) for d in s) + "]" for s in shapes)


@dataclass
class ProfileTable:
    device: DeviceSpec
    entries: dict = field(default_factory=dict)

    def lookup(self, op: str, shapes, dtype: Dtype) -> Optional[int]:
        return self.entries.get((op, shape_str(shapes), dtype.value))


_DTYPE_ALIASES = {"float32": "f32", "float16": "f16", "bfloat16": "bf16",
                  "int64": "i64", "int32": "i32", "bool": "bool"}


def parse_dtype(tag: str) -> Dtype:
    if tag.startswith("torch."):
        tag = tag[len("torch."):]
    try:
        return Dtype(_DTYPE_ALIASES.get(tag, tag))
    except ValueError:
        raise FormatError(f"unknown dtype tag {tag!r}") from None


def load_profile(path) -> ProfileTable:
    """Measured-kernel profile JSON (reference traceio.py:100-129)."""
    try:
        doc = json.loads(Path(path).read_text())
    except (OSError, json.JSONDecodeError) as e:
        raise FormatError(f"cannot read profile {path}: {e}") from e
    if not isinstance(doc, dict) or "device" not in doc:
        raise FormatError("profile must be an object with a 'device' section")
    try:
        peak = float(doc["device"]["peak_flops"])
        eff = float(doc["device"]["efficiency"])
    except (KeyError, TypeError, ValueError) as e:
        raise FormatError(f"bad device section: {e}") from e
    if peak <= 0:
        raise FormatError(f"peak_flops must be positive, got {peak}")
    if not (0.0 < eff <= 1.0):
        raise FormatError(f"efficiency must be in (0, 1], got {eff}")
    table = ProfileTable(DeviceSpec(peak, eff))
    for i, ent in enumerate(doc.get("entries", [])):
        try:
            key = (str(ent["op"]), str(ent["shape"]), parse_dtype(str(ent["dtype"])).value)
            ns = ent["ns"]
        except KeyError as e:
            raise FormatError(f"profile entry {i} missing {e}") from e
        if not isinstance(ns, int) or ns <= 0:
            raise FormatError(f"profile entry {i}: ns must be a positive integer, got {ns!r}")
        table.entries[key] = ns
    return table


_MM = {"mm", "addmm", "bmm", "matmul", "linear", "baddbmm"}
_ATTN = ("scaled_dot_product_attention", "attention", "sdpa")
_ELEMENTWISE = {
    "add", "sub", "mul", "div", "neg", "relu", "gelu", "silu", "sigmoid", "tanh",
    "exp", "log", "softmax", "_softmax", "log_softmax", "layer_norm", "native_layer_norm",
    "rms_norm", "dropout", "sum", "mean", "ones_like", "zeros_like", "fill", "copy",
    "threshold", "threshold_backward", "embedding", "where", "pow", "rsqrt", "sqrt",
}


def flops_class_of(op_name: str) -> Optional[str]:
    """Op-name bucket used by the analytical fallback (graph.py:319-331)."""
    base = op_name
    for suffix in ("_backward", "_grad"):
        if base.endswith(suffix):
            base = base[: -len(suffix)]
    if any(m in base for m in _ATTN):
        return "attention"
    if base in _MM:
        return "matmul"
    if base in _ELEMENTWISE:
        return "elementwise"
    return None


def op_flops(flops_class: str, in_shapes, out_shape) -> int:
    if flops_class == "matmul":
        mats = [s for s in in_shapes if len(s) >= 2]
        if len(mats) < 2:
            raise MissingShapeError(f"matmul cost needs two 2d+ operands, got {in_shapes}")
        a, b = mats[-2], mats[-1]
        batch = math.prod(a[:-2]) if len(a) > 2 else 1
        return 2 * batch * a[-2] * a[-1] * b[-1]
    if flops_class == "attention":
        four = [s for s in in_shapes if len(s) == 4]
        if not four:
            raise MissingShapeError(f"attention cost needs a 4d input, got {in_shapes}")
        bsz, heads, seq, hd = four[0]
        return 2 * bsz * heads * seq * seq * hd * 2
    if flops_class == "elementwise":
        ref = out_shape if out_shape else (in_shapes[0] if in_shapes else [1])
        return math.prod(ref)
    raise UnknownOperatorError(f"no cost rule for flops class {flops_class!r}")


def duration_from_flops(flops: int, device: DeviceSpec) -> int:
    return round_half_up_ns(flops / (device.peak_flops * device.efficiency) * 1e9)


def analytical_duration(op_name: str, in_shapes, dtype: Dtype, device: DeviceSpec,
                        out_shape=None, flops_class: Optional[str] = None) -> int:
    cls = flops_class or flops_class_of(op_name)
    if cls is None:
        raise UnknownOperatorError(f"no analytical cost model for op {op_name!r}")
    return duration_from_flops(op_flops(cls, in_shapes, out_shape), device)


def _rs(n: int, size: float, a: float, b: float) -> float:
    return (n - 1) * a + (n - 1) / n * size * b


def _ar(n: int, size: float, a: float, b: float) -> float:
    return 2 * (n - 1) * a + 2 * (n - 1) / n * size * b


def analytical_time(kind: CollectiveKind, size_bytes: int, n: int, algo: CollectiveAlgo,
                    alpha_ns: float, beta_ns_per_byte: float, mesh_shape=None) -> int:
    """Alpha-beta collective time in integer ns (collectives.py:251-293)."""
    if n <= 1:
        return 0
    a, b, s = float(alpha_ns), float(beta_ns_per_byte), float(size_bytes)
    kind, algo = CollectiveKind(kind.value), CollectiveAlgo(algo.value)
    if algo == CollectiveAlgo.RING:
        t = _ar(n, s, a, b) if kind == CollectiveKind.ALL_REDUCE else _rs(n, s, a, b)
    elif algo == CollectiveAlgo.TREE:
        if kind != CollectiveKind.ALL_REDUCE:
            raise UnsupportedAlgoTopologyError("TREE is defined for ALL_REDUCE only")
        t = 2 * math.ceil(math.log2(n)) * a + 2 * s * b
    else:
        if not mesh_shape:
            raise UnsupportedAlgoTopologyError("MESH_HIER timing needs the mesh shape")
        rows, cols = mesh_shape
        if rows * cols != n:
            raise UnsupportedAlgoTopologyError(f"mesh {rows}x{cols} does not hold {n} ranks")
        if kind == CollectiveKind.ALL_REDUCE:
            t = _rs(cols, s, a, b) + _ar(rows, s / cols, a, b) + _rs(cols, s, a, b)
        elif kind == CollectiveKind.ALL_GATHER:
            t = _rs(cols, s / rows, a, b) + _rs(rows, s, a, b)
        else:
            t = _rs(cols, s, a, b) + _rs(rows, s / cols, a, b)
    return round_half_up_ns(t)
