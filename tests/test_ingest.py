"""IR ingestion (ingest.py) and BASELINE config 1 vs the reference's own outputs.

Fixtures: tests/golden/ingest.json.gz, made by tests/golden/make_ingest_golden.py
(reference frontend capture of the 8-rank DP MLP + trainsim.convert).
"""

import gzip
import json
from functools import lru_cache

import numpy as np
import pytest

from golden_io import GOLDEN, canon
from oracle import pyoracle as O
from paper_2604_17550_b200 import ingest as I
from paper_2604_17550_b200.costs import DeviceSpec
from paper_2604_17550_b200.errors import TrainsimError
from paper_2604_17550_b200.topology import Topology, parse_topology


@lru_cache(maxsize=None)
def fixtures():
    with gzip.open(GOLDEN / "ingest.json.gz", "rt") as f:
        return json.load(f)


FX = fixtures()
RECS = [("c1_" + k, v) for k, v in FX["c1"].items()] + [(f["name"], f) for f in FX["fixtures"]]


def convert_all(rec, device=None):
    return [I.convert(I.parse_raw_export(d), device=device) for d in rec["raw"]]


@pytest.mark.parametrize("name,rec", RECS, ids=[n for n, _ in RECS])
def test_convert_matches_reference(name, rec):
    dev = DeviceSpec(*rec["device"]) if "device" in rec else None
    if "parse_error" in rec:
        with pytest.raises(TrainsimError) as e:
            I.parse_raw_export(rec["raw"][0])
        assert type(e.value).__name__ == rec["parse_error"]
        return
    try:
        gs = convert_all(rec, dev)
    except TrainsimError as e:
        assert rec.get("error") == type(e).__name__
        return
    assert "error" not in rec
    assert canon(gs) == rec["hash"]
    assert [g.meta for g in gs] == rec["meta"]
    assert [[n.duration_ns for n in g.nodes] for g in gs] == rec["durations"]


def test_flops_retained_recost_equals_reconvert():
    """A graph converted once keeps flops; re-costing them for another device gives
    exactly the durations the reference's convert(device=) computes."""
    from paper_2604_17550_b200.costs import duration_from_flops
    base = next(f for f in FX["fixtures"] if f["name"] == "mm_allreduce")
    dev_rec = next(f for f in FX["fixtures"] if f["name"] == "mm_allreduce_device")
    dev = DeviceSpec(*dev_rec["device"])
    gs = convert_all(base)
    recost = [[duration_from_flops(n.flops, dev) if n.flops is not None else n.duration_ns for n in g.nodes]
              for g in gs]
    assert recost == dev_rec["durations"]


@pytest.mark.parametrize("tag", sorted(FX["c1"]))
def test_oracle_on_c1(tag):
    rec = FX["c1"][tag]
    gs = convert_all(rec)
    topo = parse_topology("switch:8:25GB:1us")
    r = O.simulate(gs, topo, "ring")
    assert {"makespan_ns": r["makespan_ns"], "ranks": {str(k): v for k, v in r["ranks"].items()},
            "links": r["links"]} == rec["sim"]
    assert O.critical_path(gs, topo, "ring") == rec["cp"]


def test_read_raw_export_file(tmp_path):
    p = tmp_path / "r.json"
    p.write_text(json.dumps(FX["c1"]["bwd0"]["raw"][0]))
    assert I.read_raw_export(p).world_size == 8
    (tmp_path / "bad.json").write_text("{")
    with pytest.raises(TrainsimError):
        I.read_raw_export(tmp_path / "bad.json")


@pytest.mark.gpu
@pytest.mark.parametrize("tag", sorted(FX["c1"]))
def test_engine_on_c1(tag):
    """BASELINE config 1: the captured 8-rank DP MLP, one design point."""
    from test_gpu_parity import engine_result
    rec = FX["c1"][tag]
    got = engine_result(convert_all(rec), parse_topology("switch:8:25GB:1us"), "ring", 1, False)
    assert got["sim"] == rec["sim"]
    assert got["cp"] == rec["cp"]


@pytest.mark.gpu
def test_engine_recosts_converted_graph_per_point():
    """Device axis on an ingested graph: one upload, points with different
    (peak_flops, efficiency) equal separate conversions for those devices."""
    from paper_2604_17550_b200.engine import ROW_FIELDS, DesignPoints, simulate_batch
    base = next(f for f in FX["fixtures"] if f["name"] == "mm_allreduce")
    gs = convert_all(base)
    devs = [DeviceSpec(1e12, 1.0), DeviceSpec(3.5e14, 0.55), DeviceSpec(2.25e15, 0.4), DeviceSpec(5e9, 0.9)]
    topo = Topology.switch(2, 25e9, 1000)
    pts = DesignPoints.from_topologies([topo] * len(devs), "ring", devices=devs)
    out = simulate_batch(gs, pts)
    for i, d in enumerate(devs):
        want = O.sweep_row(convert_all(base, d), topo, "ring")
        assert {k: int(out[k][i]) for k in ROW_FIELDS} == want
