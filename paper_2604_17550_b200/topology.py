"""Design-point topology parameters.

Same value semantics as the reference (``pkg/src/trainsim/topology.py``):
``alpha_ns`` is the integer latency, ``beta_ns_per_byte = 1e9 / bw``
(topology.py:47-53), and the spec grammar ``switch:<N>:<bw>:<lat>`` /
``mesh:<R>x<C>:<bw>:<lat>`` with KB/MB/GB/TB and ns/us/ms/s suffixes
(topology.py:105-166).  Spec strings are parsed here on the host so the
parsing semantics (Python ``float`` / ``round``) stay bit-identical; the
engine receives the parsed SoA columns.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum

from .errors import FormatError


class TopologyKind(Enum):
    SWITCH = "switch"
    MESH2D = "mesh"


@dataclass
class Topology:
    kind: TopologyKind
    world_size: int
    bw_bytes_per_s: float
    latency_ns: int
    rows: int = 0
    cols: int = 0

    @classmethod
    def switch(cls, num_ranks: int, nic_bw_bytes_per_s: float, latency_ns: int) -> "Topology":
        if num_ranks < 1:
            raise ValueError("switch needs at least one rank")
        return cls(TopologyKind.SWITCH, num_ranks, float(nic_bw_bytes_per_s), int(latency_ns))

    @classmethod
    def mesh2d(cls, rows: int, cols: int, link_bw_bytes_per_s: float, latency_ns: int) -> "Topology":
        if rows < 1 or cols < 1:
            raise ValueError("mesh needs positive dimensions")
        return cls(TopologyKind.MESH2D, rows * cols, float(link_bw_bytes_per_s),
                   int(latency_ns), rows=rows, cols=cols)

    @property
    def beta_ns_per_byte(self) -> float:
        return 1e9 / self.bw_bytes_per_s

    @property
    def alpha_ns(self) -> int:
        return self.latency_ns

    def coords(self, rank: int):
        return divmod(rank, self.cols)

    def hops(self, src: int, dst: int) -> int:
        if self.kind != TopologyKind.MESH2D:
            return 1
        r0, c0 = self.coords(src)
        r1, c1 = self.coords(dst)
        return abs(r0 - r1) + abs(c0 - c1)

    def route(self, src: int, dst: int) -> list:
        """Directed link names a src->dst message holds (topology.py:68-86)."""
        if src == dst:
            return []
        if self.kind != TopologyKind.MESH2D:
            return [f"eg{src}", f"in{dst}"]
        (r, c), (r1, c1) = self.coords(src), self.coords(dst)
        out = []
        while c != c1:
            c2 = c + (1 if c1 > c else -1)
            out.append(f"{r * self.cols + c}->{r * self.cols + c2}")
            c = c2
        while r != r1:
            r2 = r + (1 if r1 > r else -1)
            out.append(f"{r * self.cols + c}->{r2 * self.cols + c}")
            r = r2
        return out


_BW_UNITS = {"": 1.0, "B": 1.0, "KB": 1e3, "MB": 1e6, "GB": 1e9, "TB": 1e12}
_LAT_UNITS = {"": 1, "ns": 1, "us": 1000, "ms": 1000 * 1000, "s": 1000 * 1000 * 1000}


def _split_unit(token: str, units) -> tuple:
    t = token.strip()
    for unit in sorted(units, key=len, reverse=True):
        if unit and t.endswith(unit):
            return t[: -len(unit)], unit
    return t, ""


def parse_bandwidth(token: str) -> float:
    num, unit = _split_unit(token, _BW_UNITS)
    try:
        val = float(num)
    except ValueError:
        raise FormatError(f"bad bandwidth {token!r}") from None
    if val <= 0:
        raise FormatError(f"bandwidth must be positive, got {token!r}")
    return val * _BW_UNITS[unit]


def parse_latency(token: str) -> int:
    num, unit = _split_unit(token, _LAT_UNITS)
    try:
        val = float(num)
    except ValueError:
        raise FormatError(f"bad latency {token!r}") from None
    if val < 0:
        raise FormatError(f"latency must be non-negative, got {token!r}")
    return int(round(val * _LAT_UNITS[unit]))    # half-to-even, as topology.py:166


def parse_topology(spec: str) -> Topology:
    parts = spec.split(":")
    if len(parts) != 4:
        raise FormatError(f"topology spec {spec!r} must have 4 colon-separated fields")
    kind, size, bw, lat = parts
    if kind == "switch":
        try:
            n = int(size)
        except ValueError:
            raise FormatError(f"bad rank count {size!r} in {spec!r}") from None
        return Topology.switch(n, parse_bandwidth(bw), parse_latency(lat))
    if kind == "mesh":
        dims = size.split("x")
        if len(dims) != 2:
            raise FormatError(f"mesh size must be RxC, got {size!r}")
        try:
            rows, cols = int(dims[0]), int(dims[1])
        except ValueError:
            raise FormatError(f"bad mesh size {size!r}") from None
        return Topology.mesh2d(rows, cols, parse_bandwidth(bw), parse_latency(lat))
    raise FormatError(f"unknown topology kind {kind!r}")
