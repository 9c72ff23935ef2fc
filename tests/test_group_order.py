"""Collectives whose group does not list the lead rank first (store.py).

The reference pairs zip(group, members) (pkg/src/trainsim/simulator.py:222-223,
:419-425).  Golden cases from the reference itself (tests/golden/group_order.json,
tests/golden/make_group_order_golden.py): where it simulates a permuted group
(node ids agree across ranks), the oracle and the engine reproduce its makespan,
per-rank stats and critical path; where its zip pairing breaks (simulate raises
KeyError), both raise InconsistentGroupsError instead -- the documented deviation.
"""

import json
from pathlib import Path

import pytest

from oracle import pyoracle as O
from paper_2604_17550_b200.errors import InconsistentGroupsError
from paper_2604_17550_b200.graph import CollSpec, CollectiveKind, Node, NodeKind, WorkloadGraph
from paper_2604_17550_b200.topology import Topology, TopologyKind

CASES = json.loads((Path(__file__).parent / "golden" / "group_order.json").read_text())["cases"]


def graphs(c):
    out = []
    for r, nodes in enumerate(c["ranks"]):
        out.append(WorkloadGraph(r, c["world"], [
            Node(d["id"], NodeKind(d["kind"]), "n", data_deps=list(d["deps"]), duration_ns=d["dur"],
                 coll=CollSpec(CollectiveKind.ALL_REDUCE, list(d["group"]), d["bytes"]) if d["group"] else None)
            for d in nodes], {}, {}))
    return out


def topo(c):
    return Topology(TopologyKind.SWITCH, c["world"], 1e9, 100)


def want(c):
    if "error" in c["sim"]:
        assert c["sim"]["error"] == "KeyError"
        return "InconsistentGroupsError"
    return c["sim"]["makespan_ns"], c["sim"]["ranks"], c["cp"]


@pytest.mark.parametrize("i", range(len(CASES)))
def test_oracle_group_order(i):
    c = CASES[i]
    gs = graphs(c)
    try:
        r = O.simulate(gs, topo(c), "ring")
        got = (r["makespan_ns"], {str(k): [v["finish_ns"], v["compute_busy_ns"], v["comm_busy_ns"],
                                            v["exposed_comm_ns"], v["peak_mem_bytes"]] for k, v in r["ranks"].items()},
               O.critical_path(gs, topo(c), "ring"))
    except O.OracleError as e:
        got = e.kind
    assert got == want(c)


@pytest.mark.gpu
@pytest.mark.parametrize("i", range(len(CASES)))
def test_engine_group_order(i):
    from paper_2604_17550_b200 import engine as E
    c = CASES[i]
    gs = graphs(c)
    try:
        rep = E.simulate(gs, topo(c))
        got = (rep.makespan_ns, {str(k): [v.finish_ns, v.compute_busy_ns, v.comm_busy_ns, v.exposed_comm_ns,
                                          v.peak_mem_bytes] for k, v in rep.ranks.items()},
               E.critical_path(gs, topo(c)))
    except InconsistentGroupsError:
        got = "InconsistentGroupsError"
    assert got == want(c)
