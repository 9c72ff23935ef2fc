"""Design-space sweeps: design-point grids, the batched sweep driver, GPU sharding.

The reference's driver (``cmd_sweep``/``_sweep_row``, pkg/src/trainsim/cli.py:314-377)
re-synthesizes the graph and runs ``simulate`` + ``critical_path`` for every
design point, optionally across a process pool.  Here one graph structure per
parallel token is compiled once and *all* its design points are evaluated by
one engine launch; rows come back in the reference's product order
(parallel x topology x algo, cli.py:352-353) with the same fields, the same
``speedup_vs_base`` normalization and the same CSV bytes.

Multi-GPU: design points are share-nothing.  Each process
(one per GPU, torchrun) evaluates a contiguous slice of every graph group and
the rows are collected with one ``all_gather_into_tensor`` (NCCL over NVLink on
the GPU box; gloo in the CPU tests) -- the only collective of the path.
"""

from __future__ import annotations

import csv
import dataclasses
import itertools
import math
import time
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .costs import CollectiveAlgo, load_profile
from .engine import ROW_FIELDS, DesignPoints, Engine
from .expansion import expand_collectives
from .passes import apply_pass
from .errors import (EngineError, FL_OK, TrainsimError, UnsupportedAlgoTopologyError,
                     UnsupportedComboError, raise_for_status)
from .synth import PRESETS, FsdpMode, parse_parallel, synth_transformer
from .topology import parse_topology

SWEEP_FIELDS = ["model", "parallel", "fsdp_mode", "algo", "comm_mode", "topology", "world_size",
                "makespan_ns", "critical_path_ns", "compute_busy_ns", "comm_busy_ns",
                "exposed_comm_ns", "peak_mem_bytes", "speedup_vs_base"]     # cli.py:314-316


# ------------------------------------------------------------------ grids


def log_grid(lo: float, hi: float, n: int) -> np.ndarray:
    if n == 1:
        return np.asarray([lo], np.float64)
    return np.exp(np.linspace(math.log(lo), math.log(hi), n))


def latency_grid(lo_ns: float, hi_ns: float, n: int) -> np.ndarray:
    return np.rint(log_grid(lo_ns, hi_ns, n)).astype(np.int64)


@dataclass
class WorkloadPart:
    """One graph family of a workload and the design points evaluated on it.

    ``expand`` = (algo, topology spec): the family is the EXPANDED form of the
    graphs (collectives lowered to SEND/RECV plans, collectives.py:456-537),
    which depends on the algorithm and, for MESH_HIER, the mesh shape."""
    parallel: str
    points: DesignPoints
    labels: list               # (topology kind, algo) per point, for reporting
    expand: Optional[tuple] = None


@dataclass
class Workload:
    """A named BASELINE configuration: graph families x design-point grids.

    A step of the bench evaluates every part (one engine launch per graph
    family); single-family workloads expose ``parallel``/``points`` directly."""
    name: str
    model: str
    parts: list

    @property
    def parallel(self) -> str:
        return self.parts[0].parallel if len(self.parts) == 1 else ",".join(p.parallel for p in self.parts)

    @property
    def points(self) -> DesignPoints:
        assert len(self.parts) == 1, "multi-family workload: use .parts"
        return self.parts[0].points

    @points.setter
    def points(self, pts: DesignPoints) -> None:
        assert len(self.parts) == 1, "multi-family workload: use .parts"
        self.parts[0].points = pts

    def n_points(self) -> int:
        return sum(len(p.points) for p in self.parts)


def _grid(pairs, bws, lats, rows_cols) -> DesignPoints:
    algo, topo, bw, lat, rows, cols = [], [], [], [], [], []
    amap = {"ring": 0, "tree": 1, "mesh-hier": 2}
    for kind, a in pairs:
        for b in bws:
            for l in lats:
                algo.append(amap[a]); topo.append(0 if kind == "switch" else 1)
                bw.append(float(b)); lat.append(int(l))
                r, c = rows_cols if kind == "mesh" else (0, 0)
                rows.append(r); cols.append(c)
    return DesignPoints(np.asarray(algo, np.uint8), np.asarray(topo, np.uint8), np.asarray(bw, np.float64),
                        np.asarray(lat, np.int64), np.asarray(rows, np.int32), np.asarray(cols, np.int32))


def _part(parallel, pairs, bws, lats, rows_cols) -> WorkloadPart:
    return WorkloadPart(parallel, _grid(pairs, bws, lats, rows_cols),
                        [p for p in pairs for _ in range(len(bws) * len(lats))])


def c3_workload() -> Workload:
    """BASELINE config 3: llama-8b-like fsdp:1024, 4096 points =
    {switch:1024 + ring, mesh:32x32 + mesh-hier} x 64 bandwidths in
    [10 GB/s, 1.8 TB/s] x 32 latencies in [100 ns, 20 us] (log-spaced)."""
    pairs = [("switch", "ring"), ("mesh", "mesh-hier")]
    return Workload("c3", "llama-8b-like", [_part("fsdp:1024", pairs, log_grid(10e9, 1.8e12, 64),
                                                  latency_grid(100, 20000, 32), (32, 32))])


def c2_workload() -> Workload:
    """BASELINE config 2: GPT-2 small dp:64, 256 points = {ring, tree} x 16
    bandwidths in [10 GB/s, 1.8 TB/s] x 8 latencies in [100 ns, 10 us]."""
    pairs = [("switch", "ring"), ("switch", "tree")]
    return Workload("c2", "gpt2-small", [_part("dp:64", pairs, log_grid(10e9, 1.8e12, 16),
                                               latency_grid(100, 10000, 8), (0, 0))])


def c4_workload() -> Workload:
    """BASELINE config 4 as SURVEY.md 8(d) defines it: llama-70b-like at 8192
    ranks, 16384 points = {dp:8192 + switch ring, dp:8192 + switch tree,
    dp:8192 + mesh:64x128 mesh-hier, fsdp:8192 + mesh:64x128 mesh-hier} x 64
    bandwidths in [10 GB/s, 1.8 TB/s] x 64 latencies in [100 ns, 20 us].
    Two graph families (dp: 1760 nodes per rank, fsdp: 2080), one engine
    launch each; a design point spans a thread-block cluster (9 CTAs on B200).  The pipeline /
    3-D part of the BASELINE wording is not expressible in the reference
    (synth.py:172-181)."""
    bws, lats = log_grid(10e9, 1.8e12, 64), latency_grid(100, 20000, 64)
    return Workload("c4", "llama-70b-like", [
        _part("dp:8192", [("switch", "ring"), ("switch", "tree"), ("mesh", "mesh-hier")], bws, lats, (64, 128)),
        _part("fsdp:8192", [("mesh", "mesh-hier")], bws, lats, (64, 128))])


def c2x_workload() -> Workload:
    """BASELINE config 2 in EXPANDED comm mode: GPT-2 small
    dp:64 with every all-reduce lowered to its ring or tree SEND/RECV plan and
    replayed on switch:64 links, 256 points = {ring, tree} x 16 bw x 8 latency.
    The expanded graph depends on the algorithm: two families."""
    bws, lats = log_grid(10e9, 1.8e12, 16), latency_grid(100, 10000, 8)
    w = Workload("c2x", "gpt2-small", [
        _part("dp:64", [("switch", "ring")], bws, lats, (0, 0)),
        _part("dp:64", [("switch", "tree")], bws, lats, (0, 0))])
    w.parts[0].expand, w.parts[1].expand = ("ring", "switch:64:50GB:1us"), ("tree", "switch:64:50GB:1us")
    return w


def meshx_workload() -> Workload:
    """The reference's mesh study (acceptance criterion 6, test_acceptance.py:260-276)
    at 8x8: tiny dp:64 on mesh:8x8, collectives expanded to ring and to mesh-hier
    SEND/RECV plans with per-link FIFOs, 256 points = {ring, mesh-hier} x 16 bw x 8
    latency."""
    bws, lats = log_grid(10e9, 1.8e12, 16), latency_grid(100, 10000, 8)
    w = Workload("meshx", "tiny", [
        _part("dp:64", [("mesh", "ring")], bws, lats, (8, 8)),
        _part("dp:64", [("mesh", "mesh-hier")], bws, lats, (8, 8))])
    w.parts[0].expand, w.parts[1].expand = ("ring", "mesh:8x8:50GB:1us"), ("mesh-hier", "mesh:8x8:50GB:1us")
    return w


def part_graphs(w: Workload, part: WorkloadPart):
    from .synth import GPT2_SMALL
    m = GPT2_SMALL if w.model == "gpt2-small" else PRESETS[w.model]
    p = parse_parallel(part.parallel)
    graphs = synth_transformer(m, p, p.degree)
    if part.expand:
        algo, spec = part.expand
        graphs = expand_collectives(graphs, CollectiveAlgo(algo), parse_topology(spec))
    return graphs


def workload_graphs(w: Workload):
    assert len(w.parts) == 1, "multi-family workload: use part_graphs"
    return part_graphs(w, w.parts[0])


# ------------------------------------------------------------- sharding


def shard(n: int, world: int, rank: int) -> tuple:
    """Contiguous, balanced slice [a, b) of n design points for one GPU."""
    base, rem = divmod(n, world)
    a = rank * base + min(rank, rem)
    return a, a + base + (1 if rank < rem else 0)


def gather_rows(local_status, local_rows, n_total: int, world: int, rank: int, device=None):
    """All-gather per-slice results into full [n_total] arrays on every rank.

    Slices are padded to the largest slice so one all_gather_into_tensor moves
    everything (status is packed into column 6 of an int64 [n, 7] block)."""
    import torch
    import torch.distributed as dist
    per = -(-n_total // world)
    block = torch.full((per, 7), -1, dtype=torch.int64, device=device)
    m = len(local_status)
    if m:
        block[:m, :6] = torch.as_tensor(np.asarray(local_rows), dtype=torch.int64, device=device)
        block[:m, 6] = torch.as_tensor(np.asarray(local_status), dtype=torch.int64, device=device)
    out = torch.empty((per * world, 7), dtype=torch.int64, device=device)
    dist.all_gather_into_tensor(out, block)
    out = out.cpu().numpy()
    rows = np.zeros((n_total, 6), np.int64)
    status = np.zeros(n_total, np.int32)
    for r in range(world):
        a, b = shard(n_total, world, r)
        rows[a:b] = out[r * per: r * per + (b - a), :6]
        status[a:b] = out[r * per: r * per + (b - a), 6]
    return status, rows


# --------------------------------------------------------- sweep driver


def sweep_rows(preset: str, parallels, topos, algos, comm_mode: str = "analytical",
               fsdp_mode: str = "delayed", profile_path: Optional[str] = None, device: int = 0,
               passes: Optional[list] = None, devices: Optional[list] = None) -> list:
    """Rows of ``trainsim sweep`` (cli.py:319-358) computed on the GPU.

    Design points that share a graph are evaluated in one engine launch: all
    points of a parallel token in ANALYTICAL mode; in EXPANDED mode the graph
    also depends on the algorithm and, for MESH_HIER, on the mesh shape
    (collectives.py:456-537), so those join the grouping key.

    ``passes`` (an extension; the reference sweeps one graph per parallel
    token) adds a graph-rewrite axis, e.g. ``["none", "reorder-allgather:1",
    "bucket-allreduce:2097152"]`` (passes.apply_pass); rows then carry a
    ``pass`` column and each value is another graph structure.

    ``devices`` spreads every group's design points over several GPUs from this
    one process (contiguous slices, one host thread per GPU; the engine call
    releases the GIL); the rows do not depend on how they are split."""
    if comm_mode not in ("analytical", "expanded"):
        raise UnsupportedComboError(f"unknown comm mode {comm_mode!r}")
    if not parallels or not topos or not algos:
        raise UnsupportedComboError("sweep lists must be non-empty")
    expanded = comm_mode == "expanded"
    profile = load_profile(profile_path) if profile_path else None
    pass_axis = list(passes) if passes else ["none"]
    tasks = [(par, ps, spec, algo) for par in parallels for ps in pass_axis for spec in topos for algo in algos]
    groups: dict = {}
    errors: dict = {}
    parsed = {}
    for i, (par, ps, spec, algo) in enumerate(tasks):
        try:
            topo = parse_topology(spec)
            a = CollectiveAlgo(algo)
        except (TrainsimError, ValueError) as e:
            errors[i] = e
            continue
        parsed[i] = (topo, a)
        key = (par, ps)
        if expanded:
            key += (a.value, topo.kind.value, topo.rows, topo.cols) if a == CollectiveAlgo.MESH_HIER else (a.value,)
        groups.setdefault(key, []).append(i)
    results = {}
    synth_cache: dict = {}
    for key, idxs in groups.items():
        par, ps = key[0], key[1]
        try:
            if par not in synth_cache:
                p = dataclasses.replace(parse_parallel(par), fsdp_mode=FsdpMode(fsdp_mode))
                synth_cache[par] = (p, synth_transformer(PRESETS[preset], p, p.degree, profile=profile))
            p, graphs = synth_cache[par]
            graphs = apply_pass(graphs, ps)
            if expanded:
                topo0, a0 = parsed[idxs[0]]
                graphs = expand_collectives(graphs, a0, topo0)
        except (TrainsimError, ValueError) as e:
            for i in idxs:
                errors[i] = e
            continue
        devs = list(devices) if devices else [device]
        pts = DesignPoints.from_topologies([parsed[i][0] for i in idxs], [parsed[i][1] for i in idxs])
        for (a, b), out in zip(*_run_on_devices(graphs, pts, devs)):
            for j in range(a, b):
                results[idxs[j]] = (int(out["status"][j - a]), out["rows"][j - a], p.degree)
    rows = []
    for i, (par, ps, spec, algo) in enumerate(tasks):  # first failure in task order, like the pool map
        if i in errors:
            raise errors[i]
        st, vals, deg = results[i]
        if st != FL_OK:
            raise_for_status(st, f"design point {par} {spec} {algo}")
        row = {"model": preset, "parallel": par, "fsdp_mode": fsdp_mode, "algo": algo,
               "comm_mode": comm_mode, "topology": spec, "world_size": deg}
        if passes:
            row["pass"] = ps
        row.update({k: int(v) for k, v in zip(ROW_FIELDS, vals)})
        rows.append(row)
    return rows


def _run_on_devices(graphs, pts: DesignPoints, devices: list):
    """Evaluate `pts` split into contiguous slices, one per device, concurrently."""
    from concurrent.futures import ThreadPoolExecutor
    from .store import compile_graphs
    gs = compile_graphs(graphs)
    slices = [shard(len(pts), len(devices), k) for k in range(len(devices))]

    def one(k):
        a, b = slices[k]
        if a == b:
            return {"status": np.zeros(0, np.int32), "rows": np.zeros((0, 6), np.int64)}
        eng = Engine(gs, devices[k])
        try:
            return eng.run(pts.take(np.arange(a, b)))
        finally:
            eng.close()

    if len(devices) == 1:
        return slices, [one(0)]
    with ThreadPoolExecutor(max_workers=len(devices)) as ex:
        return slices, list(ex.map(one, range(len(devices))))


def normalize(rows: list, normalize_to: Optional[str]) -> None:
    """speedup_vs_base exactly as cli.py:360-369."""
    base = {}
    if normalize_to:
        for row in rows:
            if row["parallel"] == normalize_to:
                base[(row["model"], row["topology"], row["algo"], row["comm_mode"], row.get("pass"))] = \
                    row["makespan_ns"]
    for row in rows:
        b = base.get((row["model"], row["topology"], row["algo"], row["comm_mode"], row.get("pass")))
        row["speedup_vs_base"] = f"{b / row['makespan_ns']:.6f}" if b and row["makespan_ns"] else "1.000000"


def write_csv(rows: list, path: str) -> None:
    with open(path, "w", newline="") as f:
        fields = SWEEP_FIELDS
        if rows and "pass" in rows[0]:
            fields = SWEEP_FIELDS[:3] + ["pass"] + SWEEP_FIELDS[3:]
        w = csv.DictWriter(f, fieldnames=fields, lineterminator="\n")
        w.writeheader()
        w.writerows(rows)
