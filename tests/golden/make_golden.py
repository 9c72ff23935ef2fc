"""Generate the golden corpus from the reference implementation itself.

Run in the build container, where the reference is mounted read-only:

    python tests/golden/make_golden.py            # writes tests/golden/*.json.gz

It imports ``trainsim`` from /root/reference/pkg/src (never copies it) and
records, for every case, the inputs and what the reference returns:
``simulate(...).to_doc()`` minus events, ``critical_path(...)``, or the
exception class name.  The GPU box has no /root/reference; tests there read
only these committed fixtures.

Cases (reference file:line of the generators):
  * hand schedules of the acceptance gate (pkg/tests/test_acceptance.py:84-179)
    and of test_simulator.py:24-249;
  * random_world_graphs seeds 0..299 (ring and tree) and random_rank_graph
    seeds 0..199 (1 and 2 compute streams) (pkg/tests/conftest.py:87-130);
  * expanded (SEND/RECV) versions of random_world_graphs 0..39;
  * the cross-rank race witness, worlds 1..4;
  * synthesized families (tiny dp/fsdp/tp x delayed/none x 2,4,8 ranks) on
    switch and mesh topologies, recorded by generator arguments because
    tests/test_synth_parity.py pins our generator to the reference's;
  * sweep rows for GPT-2 dp:64 and llama-8b-like fsdp:64 design points.
"""

from __future__ import annotations

import gzip
import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))

import trainsim as T  # noqa: E402
from conftest import GraphBuilder, random_rank_graph, random_world_graphs  # noqa: E402

OUT = Path(__file__).resolve().parent


def enc_graphs(graphs) -> dict:
    lists, index, out = [], {}, []
    for g in graphs:
        key = id(g.nodes)
        if key not in index:
            index[key] = len(lists)
            lists.append([[n.node_id, n.kind.value, n.op_name, list(n.inputs), list(n.outputs),
                           list(n.data_deps), [list(c) for c in n.ctrl_deps], n.duration_ns,
                           [n.coll.kind.value, list(n.coll.group), n.coll.comm_bytes] if n.coll else None,
                           [n.p2p.peer_rank, n.p2p.comm_bytes, n.p2p.channel_tag] if n.p2p else None]
                          for n in g.nodes])
        out.append({"rank": g.rank, "world_size": g.world_size, "nodes": index[key],
                    "tensors": [[t.tensor_id, list(t.shape), t.dtype.value, t.bytes] for t in g.tensors.values()],
                    "graph_inputs": list(g.meta.get("graph_inputs", []))})
    return {"node_lists": lists, "graphs": out}


def enc_topo(t) -> dict:
    return {"kind": t.kind.value, "world_size": t.world_size, "bw": t.bw_bytes_per_s,
            "lat": t.latency_ns, "rows": t.rows, "cols": t.cols}


def run(graphs, topo, algo="ring", cs=1, ms=1) -> dict:
    res = {}
    try:
        rep = T.simulate(graphs, topo, T.SimOptions(algo=T.CollectiveAlgo(algo), compute_streams=cs,
                                                      comm_streams=ms, record_events=True))
        doc = rep.to_doc()
        res["sim"] = {"makespan_ns": doc["makespan_ns"], "ranks": doc["ranks"], "links": doc["links"]}
        res["events"] = [[e["rank"], e["node_id"], e["start_ns"], e["end_ns"]] for e in doc["events"]]
    except T.TrainsimError as e:
        res["sim"] = {"error": type(e).__name__}
    except ValueError as e:
        res["sim"] = {"error": "ValueError"}
    try:
        res["cp"] = T.critical_path(graphs, topo, T.CollectiveAlgo(algo))
    except T.TrainsimError as e:
        res["cp"] = {"error": type(e).__name__}
    return res


def case(name, graphs, topo, algo="ring", cs=1, ms=1, keep_events=True) -> dict:
    r = run(graphs, topo, algo, cs, ms)
    if not keep_events:
        r.pop("events", None)
    return {"name": name, **enc_graphs(graphs), "topo": enc_topo(topo), "algo": algo,
            "compute_streams": cs, "comm_streams": ms, **r}


def hand_cases() -> list:
    sw = T.Topology.switch(2, 1e9, 10)
    AR, AG = T.CollectiveKind.ALL_REDUCE, T.CollectiveKind.ALL_GATHER
    out = []

    def one(fn):
        b = GraphBuilder()
        fn(b)
        return [b.build()]

    out.append(case("single", one(lambda b: b.comp(100)), sw))

    def chain(b):
        a = b.comp(10); c = b.comp(20, inputs=[b.out_of(a)], deps=[a]); b.comp(30, inputs=[b.out_of(c)], deps=[c])
    out.append(case("chain", one(chain), sw))

    def indep(b):
        b.comp(50); b.comp(70)
    out.append(case("indep_1s", one(indep), sw))
    out.append(case("indep_2s", one(indep), sw, cs=2))

    def host_pair(b):
        h = b.host(); c = b.comp(40); b.nodes[c].ctrl_deps = [(h, "launch")]
    out.append(case("host_pair", one(host_pair), sw))

    def diamond(b):
        a = b.comp(10); t = b.out_of(a)
        x = b.comp(20, inputs=[t], deps=[a]); y = b.comp(30, inputs=[t], deps=[a])
        b.comp(40, inputs=[b.out_of(x), b.out_of(y)], deps=[x, y])
    out.append(case("diamond_1s", one(diamond), sw))
    out.append(case("diamond_2s", one(diamond), sw, cs=2))
    out.append(case("diamond_4s", one(diamond), sw, cs=4))

    def two_rank_ar(d0, d1, nbytes):
        gs = []
        for rank, d in enumerate((d0, d1)):
            b = GraphBuilder(rank=rank, world_size=2)
            c = b.comp(d)
            b.coll(AR, nbytes, [0, 1], inputs=[b.out_of(c)], deps=[c])
            gs.append(b.build())
        return gs
    out.append(case("two_rank_ar", two_rank_ar(50, 80, 1000), sw))

    gs = []
    for rank in range(4):
        b = GraphBuilder(rank=rank, world_size=4)
        b.coll(AG, 256, [0, 1, 2, 3])
        gs.append(b.build())
    out.append(case("allgather4", gs, T.Topology.switch(4, 1e9, 10)))
    out.append(case("allgather4_mesh", gs, T.Topology.mesh2d(2, 2, 1e9, 10), "mesh-hier"))
    out.append(case("allgather4_tree", gs, T.Topology.switch(4, 1e9, 10), "tree"))

    def chained(extra_indep):
        gs = []
        for rank in range(2):
            b = GraphBuilder(rank=rank, world_size=2)
            if extra_indep:
                ca = b.comp(10); cb = b.comp(30)
                b.coll(AR, 100, [0, 1], inputs=[b.out_of(ca)], deps=[ca])
                b.coll(AR, 200, [0, 1], inputs=[b.out_of(cb)], deps=[cb])
            else:
                c = b.comp(10)
                a1 = b.coll(AR, 100, [0, 1], inputs=[b.out_of(c)], deps=[c])
                b.coll(AR, 200, [0, 1], inputs=[b.out_of(a1)], deps=[a1])
            gs.append(b.build())
        return gs
    out.append(case("chained_ars", chained(False), sw))
    out.append(case("queued_ars", chained(True), sw))

    def p2p(tags, topo=sw):
        b0 = GraphBuilder(rank=0, world_size=2); b1 = GraphBuilder(rank=1, world_size=2)
        for tag in tags:
            b0.send(1, 1000, tag=tag); b1.recv(0, 1000, tag=tag)
        return [b0.build(), b1.build()]
    out.append(case("p2p", p2p((0,)), sw))
    out.append(case("link_fifo", p2p((0, 1)), sw))
    bs = [GraphBuilder(rank=r, world_size=4) for r in range(4)]
    bs[0].send(3, 1000); bs[3].recv(0, 1000)
    out.append(case("mesh_hop", [b.build() for b in bs], T.Topology.mesh2d(2, 2, 1e9, 10)))
    b0 = GraphBuilder(rank=0, world_size=2); b0.send(1, 100)
    out.append(case("unmatched_send", [b0.build(), GraphBuilder(rank=1, world_size=2).build()], sw))

    def cycle(b):
        a = b.comp(10); c = b.comp(10, deps=[a]); b.nodes[a].data_deps = [c]
    out.append(case("cycle", one(cycle), sw))

    gs = []
    for rank in range(2):
        b = GraphBuilder(rank=rank, world_size=2)
        a = b.comp(50); b.comp(50)
        b.coll(AR, 100, [0, 1], inputs=[b.out_of(a)], deps=[a])
        gs.append(b.build())
    out.append(case("exposed_partial", gs, T.Topology.switch(2, 1e9, 0)))

    def peak1(b):
        t_a = b.input_tensor([25]); c1 = b.comp(10, inputs=[t_a], out_shape=[25])
        b.comp(10, inputs=[b.out_of(c1)], deps=[c1], out_shape=[25])
    out.append(case("peak_mem_1", one(peak1), sw))

    def peak2(b):
        t_a = b.input_tensor([25]); c1 = b.comp(10, inputs=[t_a], out_shape=[50])
        c2 = b.comp(10, inputs=[b.out_of(c1)], deps=[c1], out_shape=[25])
        b.comp(10, inputs=[b.out_of(c2)], deps=[c2], out_shape=[25])
    out.append(case("peak_mem_2", one(peak2), sw))

    # collective edge cases: size-1 group (zero duration), zero latency and bytes,
    # inconsistent groups, TREE on a gather, MESH_HIER without a mesh
    b = GraphBuilder(rank=0, world_size=1)
    c = b.comp(10); b.coll(AR, 64, [0], inputs=[b.out_of(c)], deps=[c]); b.comp(5)
    out.append(case("group_of_one", [b.build()], T.Topology.switch(1, 1e9, 10)))
    gs = []
    for rank in range(3):
        b = GraphBuilder(rank=rank, world_size=3)
        c = b.comp(10 + rank)
        a = b.coll(AR, 0, [0, 1, 2], inputs=[b.out_of(c)], deps=[c])
        b.comp(7, inputs=[b.out_of(a)], deps=[a]); b.comp(3)
        gs.append(b.build())
    out.append(case("zero_cost_ar", gs, T.Topology.switch(3, 1e12, 0)))
    gs = []
    for rank in range(2):
        b = GraphBuilder(rank=rank, world_size=2)
        b.coll(AR, 100 + rank, [0, 1])
        gs.append(b.build())
    out.append(case("inconsistent", gs, sw))
    out.append(case("tree_on_gather", [g for g in case_graphs_ag()], T.Topology.switch(2, 1e9, 10), "tree"))
    out.append(case("meshhier_on_switch", two_rank_ar(5, 5, 100), sw, "mesh-hier"))
    return out


def case_graphs_ag():
    gs = []
    for rank in range(2):
        b = GraphBuilder(rank=rank, world_size=2)
        b.coll(T.CollectiveKind.ALL_GATHER, 128, [0, 1])
        gs.append(b.build())
    return gs


def witness(world, coll):
    gs = []
    for r in range(world):
        b = GraphBuilder(rank=r, world_size=world)
        c0 = b.comp(15); c1 = b.comp(5, inputs=[b.out_of(c0)], deps=[c0]); b.comp(7)
        if coll:
            b.coll(T.CollectiveKind.ALL_REDUCE, 1000, list(range(world)), inputs=[b.out_of(c1)], deps=[c1])
        gs.append(b.build())
    return gs


def main():
    cases = hand_cases()
    for w in (1, 2, 3, 4):
        for coll in (False, True):
            cases.append(case(f"witness_w{w}_{'ar' if coll else 'plain'}", witness(w, coll), T.Topology.switch(w, 1e9, 10)))
    for seed in range(300):
        gs = random_world_graphs(seed)
        topo = T.Topology.switch(gs[0].world_size, 1e9, 10)
        cases.append(case(f"world_{seed}_ring", gs, topo))
        cases.append(case(f"world_{seed}_tree", gs, topo, "tree", keep_events=False))
        if seed < 40:
            ex = T.expand_collectives(gs, T.CollectiveAlgo.RING, topo)
            cases.append(case(f"world_{seed}_expanded", ex, topo, keep_events=False))
    for seed in range(200):
        g = random_rank_graph(seed)
        topo = T.Topology.switch(1, 1e9, 10)
        cases.append(case(f"rank_{seed}_1s", [g], topo))
        cases.append(case(f"rank_{seed}_2s", [g], topo, cs=2, keep_events=False))
    with gzip.open(OUT / "corpus.json.gz", "wt") as f:
        json.dump(cases, f, separators=(",", ":"))
    print("corpus cases:", len(cases))

    # synthesized families, recorded by generator arguments
    from trainsim.synth import PRESETS, FsdpMode, ParallelConfig, Strategy, synth_transformer
    synth = []
    for strat in ("dp", "fsdp", "tp"):
        for mode in ("delayed", "none"):
            if strat != "fsdp" and mode == "none":
                continue
            for deg in (2, 4, 8):
                if strat == "tp" and deg == 8:
                    continue
                gs = synth_transformer(PRESETS["tiny"], ParallelConfig(Strategy(strat), deg, FsdpMode(mode)), deg)
                specs = [(f"switch:{deg}:25GB:2us", "ring"), (f"switch:{deg}:400GB:100ns", "ring"),
                         (f"mesh:2x{deg // 2}:50GB:1us", "mesh-hier")]
                if strat != "fsdp":
                    specs.append((f"switch:{deg}:100GB:500ns", "tree"))
                for spec, algo in specs:
                    topo = T.parse_topology(spec)
                    r = run(gs, topo, algo)
                    r.pop("events", None)
                    synth.append({"preset": "tiny", "parallel": f"{strat}:{deg}", "fsdp_mode": mode,
                                  "topo_spec": spec, "algo": algo, **r})
    # bigger families: sweep rows only
    rows = []
    from trainsim.synth import ModelConfig
    gpt2 = ModelConfig(12, 768, 12, ffn_mult=4, seq_len=1024, micro_batch=1, dtype=T.Dtype.BF16, name="gpt2-small")
    for model_name, m, par in (("gpt2-small", gpt2, "dp:64"), ("llama-8b-like", PRESETS["llama-8b-like"], "fsdp:64"),
                               ("llama-8b-like", PRESETS["llama-8b-like"], "dp:16"),
                               ("llama-8b-like", PRESETS["llama-8b-like"], "tp:8")):
        p = T.parse_parallel(par)
        gs = synth_transformer(m, ParallelConfig(p.strategy, p.degree), p.degree)
        R = p.degree
        specs = [(f"switch:{R}:10GB:100ns", "ring"), (f"switch:{R}:1800GB:10us", "ring"),
                 (f"switch:{R}:50GB:2us", "ring")]
        if p.strategy.value != "fsdp":
            specs.append((f"switch:{R}:80GB:300ns", "tree"))
        side = {64: (8, 8), 16: (4, 4), 8: (2, 4)}[R]
        specs.append((f"mesh:{side[0]}x{side[1]}:100GB:500ns", "mesh-hier"))
        for spec, algo in specs:
            topo = T.parse_topology(spec)
            rep = T.simulate(gs, topo, T.SimOptions(algo=T.CollectiveAlgo(algo), record_events=False))
            cp = T.critical_path(gs, topo, T.CollectiveAlgo(algo))
            rows.append({"model": model_name, "parallel": par, "topo_spec": spec, "algo": algo,
                         "makespan_ns": rep.makespan_ns, "critical_path_ns": cp,
                         "compute_busy_ns": max(s.compute_busy_ns for s in rep.ranks.values()),
                         "comm_busy_ns": max(s.comm_busy_ns for s in rep.ranks.values()),
                         "exposed_comm_ns": rep.exposed_comm_ns, "peak_mem_bytes": rep.peak_mem_bytes})
    # C3 points at the north-star size, measured with the reference here (13-15 min each)
    c3 = [json.loads(l) for l in open(OUT / "c3_r1024.jsonl") if l.strip()]
    with gzip.open(OUT / "synth.json.gz", "wt") as f:
        json.dump({"families": synth, "rows": rows, "c3_r1024": c3}, f, separators=(",", ":"))
    print("synth cases:", len(synth), "rows:", len(rows), "c3:", len(c3))


SWEEPS = {
    "sweep_tiny_dp_tp.csv": ["--preset", "tiny", "--parallel", "dp:4,dp:8,tp:4",
                             "--topo", "switch:8:25GB:2us,switch:8:100GB:500ns",
                             "--algo", "ring,tree", "--normalize-to", "dp:4"],
    "sweep_tiny_fsdp_mesh.csv": ["--preset", "tiny", "--parallel", "fsdp:8",
                                 "--topo", "mesh:2x4:50GB:1us,mesh:2x4:400GB:100ns",
                                 "--algo", "ring,mesh-hier", "--fsdp-mode", "none"],
}


def sweeps():
    """Reference CLI sweeps (cli.py:345-377), kept byte-for-byte."""
    from trainsim.cli import main as ref_main
    for name, args in SWEEPS.items():
        assert ref_main(["sweep", *args, "--out", str(OUT / name)]) == 0
    (OUT / "sweeps.json").write_text(json.dumps(SWEEPS, indent=1) + "\n")


if __name__ == "__main__":
    main()
    sweeps()
