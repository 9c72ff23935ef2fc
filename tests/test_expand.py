"""EXPANDED comm mode host side (expansion.py) vs the reference's own outputs.

Fixtures: tests/golden/expand.json.gz, made by tests/golden/make_expand_golden.py
with trainsim imported from /root/reference.  CPU tests pin the plans
(collectives.py:76-416) and the expanded graphs (collectives.py:456-537, by
canonical hash) and run the CPU oracle on the expanded graphs; GPU tests run
the engine on them and the expanded sweep CLI end to end.
"""

import pytest

from golden_io import canon, decode_topo, expand_fixtures
from oracle import pyoracle as O
from paper_2604_17550_b200 import expansion as X
from paper_2604_17550_b200 import synth
from paper_2604_17550_b200.costs import CollectiveAlgo
from paper_2604_17550_b200.graph import CollSpec, CollectiveKind, Node, NodeKind
from randgraphs import random_graphs

FX = expand_fixtures()


def _plan_rec(p):
    topo = decode_topo(p["topo"])
    node = Node(0, NodeKind.COLL, "c", coll=CollSpec(CollectiveKind(p["kind"]), list(p["group"]), p["bytes"]))
    try:
        pl = X.expand(node, CollectiveAlgo(p["algo"]), topo)
    except Exception as e:
        return {"error": type(e).__name__}, None, topo
    return {"ops": {str(r): [[o.kind.value, o.peer, o.nbytes, o.chunk, o.step, o.reduce, list(o.slots)] for o in v]
                    for r, v in pl.ops.items()}, "num_slots": pl.num_slots}, pl, topo


@pytest.mark.parametrize("i", range(len(FX["plans"])))
def test_plan_matches_reference(i):
    p = FX["plans"][i]
    got, pl, topo = _plan_rec(p)
    if "error" in p:
        assert got == {"error": p["error"]}
        return
    assert got == {"ops": p["ops"], "num_slots": p["num_slots"]}
    mesh = (topo.rows, topo.cols) if topo.kind.value == "mesh" else None
    try:
        w = X.wire_bytes(CollectiveKind(p["kind"]), p["bytes"], len(p["group"]), CollectiveAlgo(p["algo"]), mesh)
    except Exception as e:
        w = type(e).__name__
    assert w == p["wire"]
    assert X.dataflow_check(pl) == p["dataflow"]
    assert sorted(X.check_plan(pl, topo)) == sorted(p["check"])


def source_graphs(src):
    if src["kind"] == "synth":
        p = synth.parse_parallel(src["parallel"])
        p.fsdp_mode = synth.FsdpMode(src["fsdp_mode"])
        return synth.synth_transformer(synth.PRESETS[src["preset"]], p, p.degree)
    return random_graphs(src["seed"], max_world=6, max_nodes=12)[0]


def expanded(rec):
    return X.expand_collectives(source_graphs(rec["src"]), CollectiveAlgo(rec["algo"]), decode_topo(rec["topo"]))


GRAPHS = FX["graphs"]


@pytest.mark.parametrize("i", range(len(GRAPHS)), ids=[g["name"] for g in GRAPHS])
def test_expand_collectives_matches_reference(i):
    rec = GRAPHS[i]
    try:
        ex = expanded(rec)
    except Exception as e:
        assert rec.get("error") == type(e).__name__
        return
    assert [len(g.nodes) for g in ex] == rec["nodes"]
    assert canon(ex) == rec["hash"]


SMALL = [i for i, g in enumerate(GRAPHS) if "hash" in g and sum(g["nodes"]) <= 20000]


@pytest.mark.parametrize("i", SMALL, ids=[GRAPHS[i]["name"] for i in SMALL])
def test_oracle_on_expanded_graphs(i):
    """The CPU oracle (test infrastructure) reproduces the reference on expanded graphs."""
    rec = GRAPHS[i]
    gs, topo = expanded(rec), decode_topo(rec["topo"])
    try:
        r = O.simulate(gs, topo, rec["algo"])
        got = {"makespan_ns": r["makespan_ns"], "ranks": {str(k): v for k, v in r["ranks"].items()},
               "links": r["links"]}
    except O.OracleError as e:
        got = {"error": e.kind}
    assert got == rec["sim"]
    try:
        cp = O.critical_path(gs, topo, rec["algo"])
    except O.OracleError as e:
        cp = {"error": e.kind}
    assert cp == rec["cp"]


@pytest.mark.gpu
@pytest.mark.parametrize("i", [i for i, g in enumerate(GRAPHS) if "hash" in g],
                         ids=[g["name"] for g in GRAPHS if "hash" in g])
def test_engine_on_expanded_graphs(i):
    from test_gpu_parity import engine_result
    rec = GRAPHS[i]
    got = engine_result(expanded(rec), decode_topo(rec["topo"]), rec["algo"], 1, False)
    assert got["sim"] == rec["sim"]
    assert got["cp"] == rec["cp"]


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(FX["sweeps"]))
def test_expanded_sweep_cli_byte_identical(name, tmp_path):
    from paper_2604_17550_b200 import cli
    sw = FX["sweeps"][name]
    out = tmp_path / "out.csv"
    assert cli.main(["sweep", *sw["argv"], "--out", str(out)]) == sw["rc"]
    assert out.read_text() == sw["csv"]
