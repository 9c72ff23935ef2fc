"""EXPANDED comm mode at workload scale.

Golden rows: tests/golden/expanded_scale.json, produced by the reference's own
``_sweep_row`` path (tests/golden/make_expanded_golden.py) on design points of the
expanded bench workloads (``sweep.c2x_workload``: GPT-2 small dp:64 ring/tree on
switch:64; ``sweep.meshx_workload``: tiny dp:64 ring/mesh-hier on mesh:8x8) and on
llama-8b-like fsdp:64 ring expanded (12,832 nodes per rank).

CPU: the oracle reproduces every golden row (pins the checker at this scale).
GPU: the engine reproduces every golden row and its per-link busy times, and
agrees with the oracle on a spread of each expanded workload's 256-point grid.
"""

import json
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2604_17550_b200 import expansion as X
from paper_2604_17550_b200 import sweep as S
from paper_2604_17550_b200 import synth
from paper_2604_17550_b200.costs import CollectiveAlgo
from paper_2604_17550_b200.engine import ROW_FIELDS
from paper_2604_17550_b200.topology import Topology, TopologyKind

GOLDEN = json.loads((Path(__file__).parent / "golden" / "expanded_scale.json").read_text())["rows"]
IDS = [f"{g['workload']}-{g['part']}-{g['point']}" for g in GOLDEN]


def _topo(g) -> Topology:
    if g["kind"] == "switch":
        return Topology(TopologyKind.SWITCH, int(g["parallel"].split(":")[1]), g["bw"], g["lat"])
    return Topology(TopologyKind.MESH2D, g["rows"] * g["cols"], g["bw"], g["lat"], g["rows"], g["cols"])


@lru_cache(maxsize=None)
def _graphs(workload: str, part: int):
    if workload == "fsdp64x":
        gs = synth.synth_transformer(synth.PRESETS["llama-8b-like"], synth.parse_parallel("fsdp:64"), 64)
        return X.expand_collectives(gs, CollectiveAlgo.RING, Topology(TopologyKind.SWITCH, 64, 50e9, 1000))
    w = getattr(S, f"{workload}_workload")()
    return S.part_graphs(w, w.parts[part])


@lru_cache(maxsize=None)
def _flat(workload: str, part: int):
    return O.flatten(_graphs(workload, part))


@pytest.mark.parametrize("i", range(len(GOLDEN)), ids=IDS)
def test_oracle_matches_reference_expanded(i):
    g = GOLDEN[i]
    gs = _graphs(g["workload"], g["part"])
    assert len(gs[0].nodes) == g["nodes_per_rank"]
    assert O.sweep_row(gs, _topo(g), g["algo"], flat=_flat(g["workload"], g["part"])) == g["row"]


def test_expanded_workload_points_match_golden_inputs():
    """The golden rows were taken at the workloads' own grid points."""
    for g in GOLDEN:
        if g["workload"] == "fsdp64x":
            continue
        p = getattr(S, f"{g['workload']}_workload")().parts[g["part"]].points
        i = g["point"]
        assert (float(p.bw[i]), int(p.latency[i]), int(p.rows[i]), int(p.cols[i])) == \
            (g["bw"], g["lat"], g["rows"], g["cols"])


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(GOLDEN)), ids=IDS)
def test_engine_matches_reference_expanded(i):
    from paper_2604_17550_b200 import engine as E
    g = GOLDEN[i]
    gs = _graphs(g["workload"], g["part"])
    topo = _topo(g)
    out = E.simulate_batch(gs, E.DesignPoints.from_topologies([topo], [g["algo"]]))
    assert int(out["status"][0]) == 0
    assert {k: int(out[k][0]) for k in ROW_FIELDS} == g["row"]
    rep = E.simulate(gs, topo, E.SimOptions(algo=CollectiveAlgo(g["algo"])))
    assert rep.link_busy_ns == g["link_busy_ns"]


@pytest.mark.gpu
@pytest.mark.parametrize("workload", ["c2x", "meshx"])
def test_engine_expanded_grid_vs_oracle(workload):
    """A spread of 12 points per family of the 256-point expanded grid, one launch per family."""
    from paper_2604_17550_b200 import engine as E
    w = getattr(S, f"{workload}_workload")()
    algos = {0: "ring", 1: "tree", 2: "mesh-hier"}
    for k, part in enumerate(w.parts):
        gs = _graphs(workload, k)
        out = E.simulate_batch(gs, part.points)
        assert (out["status"] == 0).all()
        p = part.points
        for i in np.linspace(0, len(p) - 1, 12).round().astype(int):
            kind = TopologyKind.SWITCH if p.topo_kind[i] == 0 else TopologyKind.MESH2D
            topo = Topology(kind, len(gs), float(p.bw[i]), int(p.latency[i]), int(p.rows[i]), int(p.cols[i]))
            want = O.sweep_row(gs, topo, algos[int(p.algo[i])], flat=_flat(workload, k))
            assert {f: int(out[f][i]) for f in ROW_FIELDS} == want, (workload, k, i)
