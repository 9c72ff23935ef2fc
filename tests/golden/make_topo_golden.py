"""Golden topological orders from the reference's own ``topo_order`` (graph.py:282-306).

    python tests/golden/make_topo_golden.py        # writes tests/golden/topo.json

Imports ``trainsim`` read-only from /root/reference/pkg/src and records, per
graph, the order ``trainsim.graph.topo_order`` returns for:
* every distinct rank graph of the golden corpus (tests/golden/corpus.json.gz:
  hand schedules, random world / rank graphs, the race witness), decoded with
  tests/golden_io.py -- the reference function reads only node ids and dep_ids;
* 300 random DAGs whose node ids are a random permutation of the topological
  positions (so lowest-id-first genuinely reorders), with ctrl deps, duplicate
  and missing deps, and some cycles (``random_dags`` below; the fixture stores
  each graph's (id, data_deps, ctrl_deps) so the GPU box rebuilds it);
* rank 0 of the BASELINE graph families C1 (captured MLP, tests/golden/ingest
  fixture), C2 (GPT-2 small dp:64), C3 (llama-8b-like fsdp:1024) and C4
  (llama-70b-like dp:8192 / fsdp:8192), synthesized by the reference itself.
"""
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parents[1]))

import trainsim as T                                   # noqa: E402
from trainsim.graph import topo_order                  # noqa: E402
from golden_io import corpus, decode_graphs            # noqa: E402


def random_dags(count=300):
    import random
    dags = []
    for seed in range(count):
        rng = random.Random(7000 + seed)
        n = rng.randint(1, 400 if seed % 10 == 0 else 60)
        ids = rng.sample(range(3 * n + 5), n)               # id of topological position k
        nodes = []
        for k in range(n):
            deps = [ids[j] for j in rng.sample(range(k), min(k, rng.randint(0, 4)))]
            if deps and rng.random() < 0.2:
                deps.append(deps[0])                        # duplicate dep
            ctrl = [ids[j] for j in rng.sample(range(k), min(k, rng.randint(0, 2)))]
            if rng.random() < 0.05:
                deps.append(10 ** 6 + k)                    # dep on a missing node (ignored)
            nodes.append([ids[k], deps, ctrl])
        if n > 2 and seed % 25 == 24:                       # a back edge: cycle
            a, b = rng.sample(range(n), 2)
            lo, hi = min(a, b), max(a, b)
            nodes[lo][1].append(ids[hi])
        rng.shuffle(nodes)                                  # list order independent of ids
        dags.append(nodes)
    return dags


def dag_graph(nodes):
    """Our graph objects for a stored DAG: COMP nodes of 10 ns (the order reads only ids/deps)."""
    from paper_2604_17550_b200.graph import Node, NodeKind, WorkloadGraph
    return WorkloadGraph(0, 1, [Node(i, NodeKind.COMP, "work", data_deps=list(d),
                                     ctrl_deps=[(c, "ctrl") for c in cl], duration_ns=10) for i, d, cl in nodes],
                         {}, {"graph_inputs": []})


def main():
    out = {"corpus": {}, "synth": {}, "dags": []}
    for nodes in random_dags():
        try:
            order = topo_order(dag_graph(nodes))
        except T.TrainsimError as e:
            order = type(e).__name__
        out["dags"].append({"nodes": nodes, "order": order})
    for case in corpus():
        try:
            gs = decode_graphs(case)
        except Exception:
            continue
        seen = {}
        for g in gs:
            if id(g.nodes) in seen:
                continue
            try:
                seen[id(g.nodes)] = (g.rank, topo_order(g))
            except T.TrainsimError as e:
                seen[id(g.nodes)] = (g.rank, type(e).__name__)
        out["corpus"][case["name"]] = {str(r): o for r, o in seen.values()}
    import gzip
    from trainsim.traceio import convert, parse_raw_export
    with gzip.open(HERE / "ingest.json.gz", "rt") as f:
        c1 = json.load(f)["c1"]
    for k, rec in sorted(c1.items()):                 # BASELINE config 1: the captured MLP, per rank 0
        out["synth"][f"C1_{k}"] = topo_order(convert(parse_raw_export(rec["raw"][0])))
    from trainsim.synth import PRESETS, ModelConfig, ParallelConfig, synth_transformer
    gpt2 = ModelConfig(12, 768, 12, ffn_mult=4, seq_len=1024, micro_batch=1, dtype=T.Dtype.BF16, name="gpt2-small")
    for name, m, par in (("C2", gpt2, "dp:64"), ("C3", PRESETS["llama-8b-like"], "fsdp:1024"),
                         ("C4dp", PRESETS["llama-70b-like"], "dp:8192"),
                         ("C4fsdp", PRESETS["llama-70b-like"], "fsdp:8192")):
        p = T.parse_parallel(par)
        gs = synth_transformer(m, ParallelConfig(p.strategy, p.degree), p.degree)
        out["synth"][name] = topo_order(gs[0])
    (HERE / "topo.json").write_text(json.dumps(out, separators=(",", ":")) + "\n")
    print("corpus graphs:", sum(len(v) for v in out["corpus"].values()), "synth:", len(out["synth"]),
          "dags:", len(out["dags"]), "non-identity:", sum(isinstance(d["order"], list) and d["order"] != sorted(d["order"])
                                                        for d in out["dags"]))


if __name__ == "__main__":
    main()
