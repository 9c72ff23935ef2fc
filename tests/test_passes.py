"""Graph passes (passes.py) vs the reference's own outputs, and as sweep axes.

Fixtures: tests/golden/passes.json.gz, made by tests/golden/make_passes_golden.py
with trainsim imported from /root/reference.  CPU tests pin the rewritten
graphs (canonical hash), the statistics and verify_pass_safety, and run the
CPU oracle on the results; GPU tests run the engine on them.
"""

import gzip
import json
from functools import lru_cache

import pytest

from golden_io import GOLDEN, canon, decode_topo
from oracle import pyoracle as O
from paper_2604_17550_b200 import passes as P
from paper_2604_17550_b200 import synth
from paper_2604_17550_b200.graph import validate_graph
from randgraphs import random_graphs


@lru_cache(maxsize=None)
def fixtures():
    with gzip.open(GOLDEN / "passes.json.gz", "rt") as f:
        return json.load(f)["cases"]


CASES = fixtures()


def source(src):
    if src["kind"] == "synth":
        p = synth.parse_parallel(src["parallel"])
        p.fsdp_mode = synth.FsdpMode(src["fsdp_mode"])
        return synth.synth_transformer(synth.PRESETS[src["preset"]], p, p.degree)
    if src["kind"] == "model":
        m = synth.ModelConfig(name="r", micro_batch=1, **src["model"])
        par = synth.ParallelConfig(synth.Strategy(src["strategy"]), src["degree"], synth.FsdpMode(src["mode"]))
        return synth.synth_transformer(m, par, src["degree"])
    return random_graphs(src["seed"], max_world=5, max_nodes=14)[0]


def rewrite(case):
    name, _, arg = case["pass"].partition(":")
    fn = P.reorder_allgather if name == "reorder-allgather" else P.bucket_allreduce
    gs = source(case["src"])
    res = [fn(g, int(arg)) for g in gs]
    return gs, [r[0] for r in res], [r[1] for r in res]


@pytest.mark.parametrize("i", range(len(CASES)), ids=[c["name"] for c in CASES])
def test_pass_matches_reference(i):
    case = CASES[i]
    try:
        gs, out, stats = rewrite(case)
    except Exception as e:
        assert case.get("error") == type(e).__name__
        return
    assert "error" not in case
    assert stats == case["stats"]
    assert canon(out) == case["hash"]
    assert [P.verify_pass_safety(a, b) for a, b in zip(gs, out)] == case["verify"]


OK = [i for i, c in enumerate(CASES) if "hash" in c]


@pytest.mark.parametrize("i", OK[::3], ids=[CASES[i]["name"] for i in OK[::3]])
def test_oracle_on_rewritten_graphs(i):
    case = CASES[i]
    _, out, _ = rewrite(case)
    topo = decode_topo(case["topo"])
    try:
        r = O.simulate(out, topo, case["algo"])
        got = {"makespan_ns": r["makespan_ns"], "ranks": {str(k): v for k, v in r["ranks"].items()},
               "links": r["links"]}
    except O.OracleError as e:
        got = {"error": e.kind}
    assert got == case["sim"]


def test_validate_graph_flags_broken_graphs():
    gs = source({"kind": "synth", "preset": "tiny", "parallel": "fsdp:4", "fsdp_mode": "delayed"})
    g = gs[0]
    assert validate_graph(g) == []
    import dataclasses
    bad = dataclasses.replace(g, nodes=g.nodes + [dataclasses.replace(g.nodes[-1])])
    assert any(v.rule == "duplicate-node-id" for v in validate_graph(bad))
    first, second = g.nodes[0], g.nodes[1]
    cyc = dataclasses.replace(g, nodes=[dataclasses.replace(first, ctrl_deps=list(first.ctrl_deps) +
                                                            [(second.node_id, "x")])] + g.nodes[1:])
    if first.node_id in second.dep_ids():
        assert any(v.rule == "cycle" for v in validate_graph(cyc))


def test_apply_pass_specs():
    gs = source({"kind": "synth", "preset": "tiny", "parallel": "fsdp:4", "fsdp_mode": "delayed"})
    assert P.apply_pass(gs, "none") == gs
    assert canon(P.apply_pass(gs, "reorder-allgather:2")) == canon([P.reorder_allgather(g, 2)[0] for g in gs])
    from paper_2604_17550_b200.errors import UnsupportedComboError
    with pytest.raises(UnsupportedComboError):
        P.apply_pass(gs, "fuse-everything")
    with pytest.raises(ValueError):
        P.apply_pass(gs, "reorder-allgather:-1")


@pytest.mark.gpu
@pytest.mark.parametrize("i", OK, ids=[CASES[i]["name"] for i in OK])
def test_engine_on_rewritten_graphs(i):
    from test_gpu_parity import engine_result
    case = CASES[i]
    _, out, _ = rewrite(case)
    got = engine_result(out, decode_topo(case["topo"]), case["algo"], 1, False)
    assert got["sim"] == case["sim"]
    assert got["cp"] == case["cp"]


@pytest.mark.gpu
def test_sweep_pass_axis_matches_per_variant_runs(tmp_path):
    """--pass: each value is its own graph structure; rows equal separate runs."""
    from paper_2604_17550_b200 import cli
    from paper_2604_17550_b200.engine import ROW_FIELDS
    from paper_2604_17550_b200.sweep import sweep_rows
    rows = sweep_rows("tiny", ["fsdp:8"], ["switch:8:10GB:1us", "switch:8:100MB:1us"], ["ring"],
                      passes=["none", "reorder-allgather:1", "bucket-allreduce:1000000"])
    assert [r["pass"] for r in rows] == ["none"] * 2 + ["reorder-allgather:1"] * 2 + ["bucket-allreduce:1000000"] * 2
    gs = source({"kind": "synth", "preset": "tiny", "parallel": "fsdp:8", "fsdp_mode": "delayed"})
    for r in rows:
        variant = P.apply_pass(gs, r["pass"])
        want = O.sweep_row(variant, __import__("paper_2604_17550_b200").parse_topology(r["topology"]), "ring")
        assert {k: r[k] for k in ROW_FIELDS} == want
    base = {r["topology"]: r["makespan_ns"] for r in rows if r["pass"] == "none"}
    moved = {r["topology"]: r["makespan_ns"] for r in rows if r["pass"] == "reorder-allgather:1"}
    assert moved["switch:8:10GB:1us"] < base["switch:8:10GB:1us"]     # acceptance 4: prefetch helps at B
    out = tmp_path / "p.csv"
    assert cli.main(["sweep", "--preset", "tiny", "--parallel", "fsdp:8", "--topo", "switch:8:10GB:1us",
                     "--pass", "none,reorder-allgather:2", "--out", str(out)]) == 0
    head = out.read_text().splitlines()[0].split(",")
    assert head[:4] == ["model", "parallel", "fsdp_mode", "pass"]
    assert cli.main(["sweep", "--preset", "tiny", "--parallel", "fsdp:8", "--topo", "switch:8:10GB:1us",
                     "--pass", "unroll:3", "--out", str(out)]) == 1
