"""Pin the CPU oracle (oracle/flint_oracle.c) to the reference's own outputs.

Every expectation here was produced by the reference implementation
(tests/golden/make_golden.py); the oracle must reproduce simulate's makespan,
per-rank stats, link busy times and full event trace, critical_path, and the
exception class, for every case.  Only after this passes is the oracle used
as the checker of the CUDA engine (tests/test_gpu_parity.py).
"""

import pytest

from golden_io import corpus, decode_graphs, decode_topo, synth_fixtures
from oracle import pyoracle as O
from paper_2604_17550_b200 import synth
from paper_2604_17550_b200.topology import parse_topology

CASES = corpus()


def oracle_result(graphs, topo, algo, cs, ms, events):
    res = {}
    try:
        r = O.simulate(graphs, topo, algo, cs, ms, record_events=events)
        res["sim"] = {"makespan_ns": r["makespan_ns"],
                      "ranks": {str(k): v for k, v in sorted(r["ranks"].items())},
                      "links": r["links"]}
        if events:
            st, en = r["events"]
            evs, k = [], 0
            for g in graphs:
                for n in g.nodes:
                    evs.append((int(st[k]), g.rank, n.node_id, int(en[k])))
                    k += 1
            res["events"] = [[rk, nid, s, e] for s, rk, nid, e in sorted(evs)]
    except O.OracleError as e:
        res["sim"] = {"error": e.kind}
    try:
        res["cp"] = O.critical_path(graphs, topo, algo)
    except O.OracleError as e:
        res["cp"] = {"error": e.kind}
    return res


@pytest.mark.parametrize("idx", range(len(CASES)), ids=[c["name"] for c in CASES])
def test_oracle_matches_reference(idx):
    case = CASES[idx]
    graphs = decode_graphs(case)
    got = oracle_result(graphs, decode_topo(case["topo"]), case["algo"], case["compute_streams"],
                        case["comm_streams"], "events" in case)
    assert got["sim"] == case["sim"]
    assert got["cp"] == case["cp"]
    if "events" in case:
        assert got["events"] == case["events"]


def _family(preset, par, mode):
    p = synth.parse_parallel(par)
    p.fsdp_mode = synth.FsdpMode(mode)
    return synth.synth_transformer(synth.PRESETS[preset], p, p.degree)


@pytest.mark.parametrize("fx", synth_fixtures()["families"],
                         ids=lambda f: f"{f['parallel']}-{f['fsdp_mode']}-{f['topo_spec']}-{f['algo']}")
def test_oracle_synth_families(fx):
    gs = _family(fx["preset"], fx["parallel"], fx["fsdp_mode"])
    got = oracle_result(gs, parse_topology(fx["topo_spec"]), fx["algo"], 1, 1, False)
    assert got["sim"] == fx["sim"]
    assert got["cp"] == fx["cp"]


def _model(name):
    return synth.GPT2_SMALL if name == "gpt2-small" else synth.PRESETS[name]


ROW_KEYS = ("makespan_ns", "critical_path_ns", "compute_busy_ns", "comm_busy_ns", "exposed_comm_ns",
            "peak_mem_bytes")


@pytest.mark.parametrize("row", synth_fixtures()["rows"], ids=lambda r: f"{r['model']}-{r['parallel']}-{r['topo_spec']}-{r['algo']}")
def test_oracle_sweep_rows(row):
    p = synth.parse_parallel(row["parallel"])
    gs = synth.synth_transformer(_model(row["model"]), p, p.degree)
    got = O.sweep_row(gs, parse_topology(row["topo_spec"]), row["algo"])
    assert {k: got[k] for k in ROW_KEYS} == {k: row[k] for k in ROW_KEYS}


@pytest.mark.parametrize("row", synth_fixtures()["c3_r1024"], ids=lambda r: f"{r['spec']}-{r['algo']}")
def test_oracle_c3_north_star_points(row):
    """llama-8b-like fsdp:1024 -- the BASELINE config-3 graph at full size."""
    gs = synth.synth_transformer(synth.PRESETS["llama-8b-like"], synth.ParallelConfig(synth.Strategy.FSDP, 1024), 1024)
    got = O.sweep_row(gs, parse_topology(row["spec"]), row["algo"])
    assert {k: got[k] for k in ROW_KEYS} == {k: row[k] for k in ROW_KEYS}


def test_critical_path_trace_is_a_tight_chain():
    """The oracle's node trace: a dependency chain whose finishes add up to the length
    (each step's start is its predecessor's finish, or a SEND's finish plus the wire)."""
    from oracle import pyoracle as O
    from paper_2604_17550_b200 import synth
    from paper_2604_17550_b200.topology import parse_topology
    gs = synth.synth_transformer(synth.PRESETS["tiny"], synth.ParallelConfig(synth.Strategy.FSDP, 8), 8)
    for spec, algo in [("switch:8:25GB:2us", "ring"), ("mesh:2x4:100GB:1us", "mesh-hier")]:
        topo = parse_topology(spec)
        length, path = O.critical_path_trace(gs, topo, algo)
        assert length == O.critical_path(gs, topo, algo)
        nodes = {(g.rank, n.node_id): n for g in gs for n in g.nodes}
        for (ra, a), (rb, b) in zip(path, path[1:]):
            nb = nodes[(rb, b)]
            same_rank_dep = ra == rb and a in set(nb.dep_ids())
            coll_dep = nb.coll is not None and ra in nb.coll.group
            assert same_rank_dep or coll_dep, ((ra, a), (rb, b))
