"""Small engine runs for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool memcheck python scripts/sanitize.py [analytical|p2p|cluster|cluster9|cluster_p2p|lean|streams8]

Every case is also checked against the CPU oracle, so a run that the sanitizer
passes is a correct one.  Sizes are kept small: racecheck replays shared-memory
accesses of every thread.
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import pyoracle as O  # noqa: E402
from paper_2604_17550_b200 import engine as E  # noqa: E402
from paper_2604_17550_b200 import synth  # noqa: E402
from paper_2604_17550_b200.topology import parse_topology  # noqa: E402


def check(gs, specs):
    topos = [parse_topology(s) for s, _ in specs]
    out = E.simulate_batch(gs, E.DesignPoints.from_topologies(topos, [a for _, a in specs]))
    flat = O.flatten(gs)
    for i, (topo, (_, algo)) in enumerate(zip(topos, specs)):
        want = O.sweep_row(gs, topo, algo, flat=flat)
        got = {k: int(out[k][i]) for k in E.ROW_FIELDS}
        assert int(out["status"][i]) == 0 and got == want, (specs[i], got, want)


def main(case: str) -> None:
    if case == "analytical":
        gs = synth.synth_transformer(synth.PRESETS["tiny"], synth.ParallelConfig(synth.Strategy.FSDP, 8), 8)
        check(gs, [("switch:8:25GB:2us", "ring"), ("mesh:2x4:50GB:1us", "mesh-hier")])
        gs = synth.synth_transformer(synth.PRESETS["tiny"], synth.ParallelConfig(synth.Strategy.DP, 64), 64)
        check(gs, [("switch:64:25GB:2us", "ring"), ("switch:64:100GB:1us", "tree")])
        # event traces, per-rank stats and the device-side critical-path trace
        eng = E.Engine(gs)
        pts = E.DesignPoints.from_topologies([parse_topology("switch:64:25GB:2us")], ["ring"])
        eng.run(pts, rank_stats=True, events=True, trace_cap=64)
        eng.topo_levels()
        eng.close()
    elif case == "p2p":
        from paper_2604_17550_b200 import expansion as X
        from paper_2604_17550_b200.costs import CollectiveAlgo
        gs = synth.synth_transformer(synth.PRESETS["tiny"], synth.ParallelConfig(synth.Strategy.DP, 16), 16)
        for spec, algo in [("switch:16:25GB:2us", "ring"), ("switch:16:25GB:2us", "tree"),
                           ("mesh:4x4:50GB:1us", "ring"), ("mesh:4x4:50GB:1us", "mesh-hier")]:
            ex = X.expand_collectives(gs, CollectiveAlgo(algo), parse_topology(spec))
            check(ex, [(spec, algo)])
            E.simulate(ex, parse_topology(spec), E.SimOptions(algo=CollectiveAlgo(algo), record_events=True))
    elif case == "cluster":
        gs = synth.synth_transformer(synth.PRESETS["tiny"], synth.ParallelConfig(synth.Strategy.DP, 2048), 2048)
        check(gs, [("switch:2048:100GB:1us", "ring"), ("mesh:32x64:400GB:100ns", "mesh-hier")])
    elif case == "lean":             # lean variants (1024 lanes, 64 lanes) and the second pass
        import numpy as np
        for deg in (1024, 64):
            gs = synth.synth_transformer(synth.PRESETS["tiny"], synth.ParallelConfig(synth.Strategy.FSDP, deg), deg)
            check(gs, [(f"switch:{deg}:25GB:2us", "ring"), (f"switch:{deg}:400GB:1us", "ring")])
            topos = [parse_topology(f"switch:{deg}:25GB:2us")] * 2
            pts = E.DesignPoints.from_topologies(topos, ["ring", "ring"])
            pts.peak_flops = np.array([1e12, 1e30])      # the second point cannot fold: second pass
            pts.efficiency = np.array([0.5, 0.5])
            out = E.simulate_batch(gs, pts)
            assert (out["status"] == 0).all(), out["status"]
    elif case == "cluster9":          # 8192 ranks: 9 CTAs of 911 ranks (blocks of 928 threads)
        gs = synth.synth_transformer(synth.PRESETS["tiny"], synth.ParallelConfig(synth.Strategy.DP, 8192), 8192)
        check(gs, [("switch:8192:100GB:1us", "ring"), ("mesh:64x128:400GB:100ns", "mesh-hier")])
    elif case == "cluster_p2p":       # messages on a cluster of 4 CTAs of 600 ranks (DSMEM summaries)
        import os
        os.environ["FL_CLUSTER_CTAS"] = "4"
        from randgraphs import random_p2p_graphs
        gs, topo = random_p2p_graphs(40_004, world=2400, n_msgs=2000)
        want = O.simulate(gs, topo, "ring", 1, 1)
        got = E.simulate(gs, topo, E.SimOptions())
        assert got.makespan_ns == want["makespan_ns"], (got.makespan_ns, want["makespan_ns"])
    elif case == "streams8":          # the 8-stream variant (compute_streams 5-8), one CTA and a cluster
        from randgraphs import random_graphs, random_spmd_graphs
        for seed in (1, 7, 11):
            gs, topo = random_graphs(seed, max_nodes=32)
            for cs in (5, 8):
                try:
                    want = O.simulate(gs, topo, "ring", cs, 1)["makespan_ns"]
                except O.OracleError as e:
                    want = e.kind
                try:
                    got = E.simulate(gs, topo, E.SimOptions(compute_streams=cs)).makespan_ns
                except Exception as e:
                    got = type(e).__name__
                assert got == want, (seed, cs, got, want)
        gs, topo = random_spmd_graphs(60_000, 1100, n_nodes=12, per_rank_dur=True)
        want = O.simulate(gs, topo, "ring", 7, 1)["makespan_ns"]
        got = E.simulate(gs, topo, E.SimOptions(compute_streams=7)).makespan_ns
        assert got == want, (got, want)
    else:
        raise SystemExit(f"unknown case {case}")
    print(f"sanitize case {case}: ok")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "analytical")
