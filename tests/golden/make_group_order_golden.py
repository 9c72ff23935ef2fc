"""Golden cases for collectives whose group does not list the lead rank first.

Run in the build container (the reference is mounted read-only there):

    python tests/golden/make_group_order_golden.py    # writes tests/golden/group_order.json

The reference pairs zip(group, members) (pkg/src/trainsim/simulator.py:222-223 and
:419-425, members = [lead] + the others in group order).  For a permuted group that
is still each rank with its own collective when the node ids agree across ranks
(SPMD graphs), and then simulate / critical_path behave as for the ascending group.
When they do not agree, simulate fails with a KeyError and critical_path may join the
wrong dependencies.  Each case records what trainsim (imported from
/root/reference/pkg/src) returns, or the exception class it raises.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF / "src"))

import trainsim as T  # noqa: E402

OUT = HERE / "group_order.json"


def case(seed: int) -> dict:
    rng = random.Random(seed)
    world = rng.randint(2, 5)
    n_coll = rng.randint(1, 3)
    perms, sizes = [], []
    for _ in range(n_coll):
        g = list(range(world))
        rng.shuffle(g)
        perms.append(g)
        sizes.append(rng.choice([100, 4000]))
    ids_agree = seed % 4 != 3          # every fourth case: collective node ids differ across ranks
    deps_agree = seed % 5 != 4         # every fifth: the collectives' dependencies differ across ranks
    spec = {"world": world, "groups": perms, "ids_agree": ids_agree, "deps_agree": deps_agree, "ranks": []}
    for r in range(world):
        nodes, nid = [], 0
        prev = None
        for k in range(n_coll):
            c0 = T.Node(nid, T.NodeKind.COMP, "c", duration_ns=rng.randint(1, 40) + (r * 3 if seed % 2 else 0),
                        data_deps=[prev] if prev is not None else [])
            nodes.append(c0)
            nid += 1
            extra = []
            if not deps_agree and r % 2 == 1:
                c1 = T.Node(nid, T.NodeKind.COMP, "x", duration_ns=5)
                nodes.append(c1)
                extra = [nid]
                nid += 1
            cid = nid + (r if not ids_agree else 0) * 1000
            nodes.append(T.Node(cid, T.NodeKind.COLL, "ar", data_deps=[c0.node_id] + extra,
                                coll=T.CollSpec(T.CollectiveKind.ALL_REDUCE, perms[k], sizes[k])))
            nid += 1
            prev = cid
        nodes.append(T.Node(nid + 5000, T.NodeKind.COMP, "tail", duration_ns=7, data_deps=[prev]))
        spec["ranks"].append([{"id": n.node_id, "kind": n.kind.value, "dur": n.duration_ns, "deps": list(n.data_deps),
                               "group": n.coll.group if n.coll else None,
                               "bytes": n.coll.comm_bytes if n.coll else 0} for n in nodes])
    graphs = [T.WorkloadGraph(r, world, [T.Node(d["id"], T.NodeKind(d["kind"]), "n", data_deps=d["deps"],
                                                 duration_ns=d["dur"],
                                                 coll=T.CollSpec(T.CollectiveKind.ALL_REDUCE, d["group"], d["bytes"])
                                                 if d["group"] else None) for d in spec["ranks"][r]], {}, {})
              for r in range(world)]
    topo = T.Topology.switch(world, 1e9, 100)
    try:
        rep = T.simulate(graphs, topo)
        spec["sim"] = {"makespan_ns": rep.makespan_ns,
                       "ranks": {str(r): [s.finish_ns, s.compute_busy_ns, s.comm_busy_ns, s.exposed_comm_ns,
                                          s.peak_mem_bytes] for r, s in sorted(rep.ranks.items())}}
    except Exception as e:          # noqa: BLE001 -- the reference's KeyError is recorded as such
        spec["sim"] = {"error": type(e).__name__}
    try:
        spec["cp"] = T.critical_path(graphs, topo)
    except Exception as e:          # noqa: BLE001
        spec["cp"] = {"error": type(e).__name__}
    return spec


def main():
    cases = [case(s) for s in range(60)]
    OUT.write_text(json.dumps({"source": "trainsim (reference), tests/golden/make_group_order_golden.py",
                               "cases": cases}) + "\n")
    print(f"wrote {len(cases)} cases to {OUT}")


if __name__ == "__main__":
    main()
