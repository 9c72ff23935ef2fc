"""CUDA engine vs the reference's outputs (golden fixtures) and vs the oracle.

All comparisons are bit-exact on integer nanoseconds and bytes.  Every call
goes through libflint_b200.so's C-ABI (fl_graph_create / fl_sweep_run).
"""

import numpy as np
import pytest

from golden_io import corpus, decode_graphs, decode_topo, has_p2p, synth_fixtures
from oracle import pyoracle as O
from paper_2604_17550_b200 import engine as E
from paper_2604_17550_b200 import synth
from paper_2604_17550_b200.errors import EngineError
from paper_2604_17550_b200.topology import Topology, parse_topology
from randgraphs import random_graphs

pytestmark = pytest.mark.gpu

CASES = corpus()      # including SEND/RECV (expanded comm mode) cases


def engine_result(graphs, topo, algo, cs, events):
    res = {}
    try:
        rep = E.simulate(graphs, topo, E.SimOptions(algo=algo, compute_streams=cs, record_events=events))
        doc = rep.to_doc()
        res["sim"] = {"makespan_ns": doc["makespan_ns"], "ranks": doc["ranks"], "links": doc["links"]}
        if events:
            res["events"] = [[e["rank"], e["node_id"], e["start_ns"], e["end_ns"]] for e in doc["events"]]
    except (ValueError, EngineError) as e:
        if isinstance(e, EngineError):
            raise
        res["sim"] = {"error": "ValueError"}
    except Exception as e:  # trainsim-compatible error classes
        res["sim"] = {"error": type(e).__name__}
    try:
        res["cp"] = E.critical_path(graphs, topo, algo)
    except EngineError:
        raise
    except Exception as e:
        res["cp"] = {"error": type(e).__name__}
    return res


@pytest.mark.parametrize("idx", range(len(CASES)), ids=[c["name"] for c in CASES])
def test_engine_matches_reference(idx):
    case = CASES[idx]
    got = engine_result(decode_graphs(case), decode_topo(case["topo"]), case["algo"],
                        case["compute_streams"], "events" in case)
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
def test_engine_synth_families(fx):
    gs = _family(fx["preset"], fx["parallel"], fx["fsdp_mode"])
    got = engine_result(gs, parse_topology(fx["topo_spec"]), fx["algo"], 1, False)
    assert got["sim"] == fx["sim"]
    assert got["cp"] == fx["cp"]


ROW_KEYS = E.ROW_FIELDS


def _batch(gs, specs_algos):
    topos = [parse_topology(s) for s, _ in specs_algos]
    pts = E.DesignPoints.from_topologies(topos, [a for _, a in specs_algos])
    return E.simulate_batch(gs, pts)


def test_engine_sweep_rows_batched():
    rows = synth_fixtures()["rows"]
    groups = {}
    for r in rows:
        groups.setdefault((r["model"], r["parallel"]), []).append(r)
    for (model, par), rs in groups.items():
        p = synth.parse_parallel(par)
        m = synth.GPT2_SMALL if model == "gpt2-small" else synth.PRESETS[model]
        gs = synth.synth_transformer(m, p, p.degree)
        out = _batch(gs, [(r["topo_spec"], r["algo"]) for r in rs])
        assert (out["status"] == 0).all()
        for i, r in enumerate(rs):
            assert {k: int(out[k][i]) for k in ROW_KEYS} == {k: r[k] for k in ROW_KEYS}, (model, par, r["topo_spec"])


def test_engine_c3_north_star_points():
    """llama-8b-like fsdp:1024 -- rows measured with the reference (15 min each on CPU)."""
    rows = synth_fixtures()["c3_r1024"]
    gs = synth.synth_transformer(synth.PRESETS["llama-8b-like"], synth.ParallelConfig(synth.Strategy.FSDP, 1024), 1024)
    out = _batch(gs, [(r["spec"], r["algo"]) for r in rows])
    for i, r in enumerate(rows):
        assert {k: int(out[k][i]) for k in ROW_KEYS} == {k: r[k] for k in ROW_KEYS}


@pytest.mark.parametrize("seed", range(400))
def test_engine_random_race_graphs_vs_oracle(seed):
    gs, topo = random_graphs(seed)
    _check_race(gs, topo, seed, (("ring", 1), ("ring", 2), ("tree", 1), ("ring", 3)))


@pytest.mark.parametrize("seed", range(120))
def test_engine_random_race_graphs_many_compute_streams(seed):
    """compute_streams 5-8 (the reference takes any count, simulator.py:233,289): they run on the
    8-stream kernel variant, whose slots above the count never free."""
    gs, topo = random_graphs(seed, max_nodes=32)
    _check_race(gs, topo, seed, (("ring", 5), ("ring", 8), ("tree", 6)))


@pytest.mark.parametrize("seed", range(2))
def test_engine_cluster_many_compute_streams(seed):
    """The 8-stream variant on a thread-block cluster (> 1024 ranks)."""
    from randgraphs import random_spmd_graphs
    gs, topo = random_spmd_graphs(60_000 + seed, 1500 + 200 * seed, n_nodes=20, per_rank_dur=True)
    _check_race(gs, topo, seed, (("ring", 7),))


def test_engine_refuses_more_than_eight_compute_streams():
    gs, topo = random_graphs(3)
    with pytest.raises(EngineError, match="compute_streams"):
        E.simulate(gs, topo, E.SimOptions(algo="ring", compute_streams=9))


def _check_race(gs, topo, seed, configs):
    for algo, cs in configs:
        try:
            ref = O.simulate(gs, topo, algo, cs, 1, record_events=True)
            st, en = ref.pop("events")
            ref.pop("links")
            evs, k = [], 0
            for g in gs:
                for n in g.nodes:
                    evs.append((int(st[k]), g.rank, n.node_id, int(en[k])))
                    k += 1
            want = (ref["makespan_ns"], ref["ranks"], sorted(evs))
        except O.OracleError as e:
            want = e.kind
        try:
            rep = E.simulate(gs, topo, E.SimOptions(algo=algo, compute_streams=cs))
            got = (rep.makespan_ns, {k: vars(v) for k, v in rep.ranks.items()},
                   sorted((e.start_ns, e.rank, e.node_id, e.end_ns) for e in rep.events))
        except EngineError:
            raise
        except Exception as e:
            got = "ValueError" if isinstance(e, ValueError) else type(e).__name__
        assert got == want, (seed, algo, cs)
        try:
            want_cp = O.critical_path(gs, topo, algo)
        except O.OracleError as e:
            want_cp = e.kind
        try:
            got_cp = E.critical_path(gs, topo, algo)
        except EngineError:
            raise
        except Exception as e:
            got_cp = type(e).__name__
        assert got_cp == want_cp, (seed, algo)


def test_engine_c3_grid_sample_vs_oracle():
    """A spread of BASELINE config-3 design points (switch ring + mesh-hier) at R=1024."""
    gs = synth.synth_transformer(synth.PRESETS["llama-8b-like"], synth.ParallelConfig(synth.Strategy.FSDP, 1024), 1024)
    flat = O.flatten(gs)
    specs = [("switch:1024:10GB:100ns", "ring"), ("switch:1024:1800GB:20us", "ring"),
             ("mesh:32x32:37GB:1us", "mesh-hier"), ("mesh:32x32:640GB:150ns", "mesh-hier")]
    out = _batch(gs, specs)
    for i, (spec, algo) in enumerate(specs):
        want = O.sweep_row(gs, parse_topology(spec), algo, flat=flat)
        assert {k: int(out[k][i]) for k in ROW_KEYS} == want, spec


def test_cost_stage_matches_oracle_exhaustively():
    """K1: alpha-beta forms and flops->ns on the device vs the C restatement."""
    from paper_2604_17550_b200 import costs
    rng = np.random.default_rng(7)
    n = 20000
    kind = rng.integers(0, 3, n).astype(np.uint8)
    algo = rng.integers(0, 3, n).astype(np.uint8)
    gn = rng.integers(1, 9000, n).astype(np.int64)
    size = rng.integers(0, 1 << 40, n).astype(np.int64)
    alpha = rng.integers(0, 20000, n).astype(np.float64)
    beta = 1e9 / np.exp(rng.uniform(np.log(1e9), np.log(2e12), n))
    rows = np.ones(n, np.int32)
    cols = gn.astype(np.int32)
    sq = rng.random(n) < 0.5
    rows[sq] = 2
    cols[sq] = (gn[sq] // 2).astype(np.int32)
    gn[sq] = rows[sq] * cols[sq]
    flops = rng.integers(0, 1 << 50, n).astype(np.int64)
    peak = np.exp(rng.uniform(np.log(1e11), np.log(5e15), n))
    eff = rng.uniform(0.05, 1.0, n)
    got, st, comp = E.cost_only(kind, size, gn, algo, alpha, beta, rows, cols, flops, peak, eff)
    names = {0: "ALL_REDUCE", 1: "ALL_GATHER", 2: "REDUCE_SCATTER"}
    anames = {0: "ring", 1: "tree", 2: "mesh-hier"}
    for i in range(n):
        try:
            want = O.analytical_time(names[int(kind[i])], int(size[i]), int(gn[i]), anames[int(algo[i])],
                                     float(alpha[i]), float(beta[i]), int(rows[i]), int(cols[i]))
            assert st[i] == 0 and got[i] == want, i
        except O.OracleError:
            assert st[i] == 4, i
        assert comp[i] == O.duration_from_flops(int(flops[i]), float(peak[i]), float(eff[i])), i


@pytest.mark.parametrize("name", ["sweep_tiny_dp_tp.csv", "sweep_tiny_fsdp_mesh.csv"])
def test_sweep_cli_csv_byte_identical(name, tmp_path):
    """`python -m paper_2604_17550_b200 sweep` == reference `trainsim sweep` byte for byte."""
    import json
    from golden_io import GOLDEN
    from paper_2604_17550_b200.cli import main
    args = json.loads((GOLDEN / "sweeps.json").read_text())[name]
    out = tmp_path / name
    assert main(["sweep", *args, "--out", str(out)]) == 0
    assert out.read_bytes() == (GOLDEN / name).read_bytes()


def test_sweep_cli_exit_codes(tmp_path):
    from paper_2604_17550_b200.cli import main
    out = str(tmp_path / "x.csv")
    # mesh-hier on a switch: UnsupportedAlgoTopologyError -> exit 1 (cli.py:395-397)
    assert main(["sweep", "--preset", "tiny", "--parallel", "dp:4", "--topo", "switch:4:1GB:1us",
                 "--algo", "mesh-hier", "--out", out]) == 1
    # tree on FSDP gathers
    assert main(["sweep", "--preset", "tiny", "--parallel", "fsdp:4", "--topo", "switch:4:1GB:1us",
                 "--algo", "tree", "--out", out]) == 1
    # bad topology spec: FormatError -> exit 2
    assert main(["sweep", "--preset", "tiny", "--parallel", "dp:4", "--topo", "ring:4",
                 "--algo", "ring", "--out", out]) == 2


@pytest.mark.parametrize("seed", range(200))
def test_engine_random_p2p_vs_oracle(seed):
    """Expanded comm mode: per-link FIFO, message ordering, busy/exposed stats."""
    from randgraphs import random_p2p_graphs
    gs, topo = random_p2p_graphs(seed, mesh=seed % 2 == 1)
    _check_p2p(gs, topo, seed)


def _check_p2p(gs, topo, seed):
    try:
        ref = O.simulate(gs, topo, "ring", record_events=True)
        st, en = ref.pop("events")
        evs, k = [], 0
        for g in gs:
            for n in g.nodes:
                evs.append((int(st[k]), g.rank, n.node_id, int(en[k])))
                k += 1
        want = (ref["makespan_ns"], ref["ranks"], ref["links"], sorted(evs))
    except O.OracleError as e:
        want = e.kind
    try:
        rep = E.simulate(gs, topo, E.SimOptions())
        got = (rep.makespan_ns, {k: vars(v) for k, v in rep.ranks.items()}, rep.link_busy_ns,
               sorted((e.start_ns, e.rank, e.node_id, e.end_ns) for e in rep.events))
    except EngineError:
        raise
    except Exception as e:
        got = type(e).__name__
    assert got == want, seed
    try:
        want_cp = O.critical_path(gs, topo, "ring")
    except O.OracleError as e:
        want_cp = e.kind
    try:
        got_cp = E.critical_path(gs, topo, "ring")
    except EngineError:
        raise
    except Exception as e:
        got_cp = type(e).__name__
    assert got_cp == want_cp, seed


# ---- more ranks than one CTA has threads: a design point spans a thread-block cluster ----

@pytest.mark.parametrize("seed", range(12))
def test_engine_cluster_race_graphs_vs_oracle(seed):
    """1025..3000 ranks (2-3 CTAs per point): cross-CTA ties, sub-group collectives, zero durations."""
    gs, topo = random_graphs(10_000 + seed, min_world=1025, max_world=3000, max_nodes=10)
    _check_race(gs, topo, seed, (("ring", 1), ("ring", 2), ("tree", 1)))


@pytest.mark.parametrize("seed", range(6))
def test_engine_cluster_p2p_vs_oracle(seed):
    from randgraphs import random_p2p_graphs
    gs, topo = random_p2p_graphs(20_000 + seed, world=1024 + 512 * (seed % 3) + seed, n_msgs=3000)
    _check_p2p(gs, topo, seed)


@pytest.mark.parametrize("spec,algo", [("switch:2048:50GB:1us", "ring"), ("switch:2048:900GB:200ns", "tree"),
                                       ("mesh:32x64:200GB:500ns", "mesh-hier")])
def test_engine_cluster_fsdp2048_vs_oracle(spec, algo):
    gs = synth.synth_transformer(synth.PRESETS["llama-8b-like"], synth.ParallelConfig(synth.Strategy.FSDP, 2048), 2048)
    out = _batch(gs, [(spec, algo)])
    try:
        want = O.sweep_row(gs, parse_topology(spec), algo)
    except O.OracleError as e:       # TREE is ALL_REDUCE-only (collectives.py:273-275)
        assert e.kind == "UnsupportedAlgoTopologyError" and out["status"][0] == 4
        return
    assert {k: int(out[k][0]) for k in ROW_KEYS} == want


def test_engine_cluster_8192_ranks_vs_oracle():
    """BASELINE config-4 scale: 8192 ranks = a cluster of 9 CTAs per design point."""
    gs = synth.synth_transformer(synth.PRESETS["tiny"], synth.ParallelConfig(synth.Strategy.DP, 8192), 8192)
    specs = [("switch:8192:100GB:1us", "ring"), ("switch:8192:25GB:5us", "tree"), ("mesh:64x128:400GB:100ns", "mesh-hier")]
    out = _batch(gs, specs)
    flat = O.flatten(gs)
    for i, (spec, algo) in enumerate(specs):
        assert {k: int(out[k][i]) for k in ROW_KEYS} == O.sweep_row(gs, parse_topology(spec), algo, flat=flat), spec


@pytest.mark.parametrize("ctas", [3, 4, 5, 7])
@pytest.mark.parametrize("kind", ["race", "p2p"])
def test_engine_cluster_sizes_vs_oracle(kind, ctas, monkeypatch):
    """Clusters wider than ceil(R / 1024): ceil(R / CTAs) ranks per CTA, blocks that are not
    a multiple of 1024 (FL_CLUSTER_CTAS forces the size the engine otherwise picks from
    occupancy), DSMEM owners of the message summaries included."""
    monkeypatch.setenv("FL_CLUSTER_CTAS", str(ctas))
    if kind == "race":
        gs, topo = random_graphs(30_000 + ctas, min_world=2049, max_world=3000, max_nodes=10)
        _check_race(gs, topo, ctas, (("ring", 1), ("tree", 2)))
    else:
        from randgraphs import random_p2p_graphs
        gs, topo = random_p2p_graphs(40_000 + ctas, world=2100 + 37 * ctas, n_msgs=3000)
        _check_p2p(gs, topo, ctas)


@pytest.mark.parametrize("seed", range(8))
def test_engine_cluster_spmd_vs_oracle(seed, monkeypatch):
    """SPMD graphs whose collectives all span the world at 1025-3244 ranks (the structure of
    the C4 families) on clusters of 2-6 CTAs: per-rank durations in {0, 5, 10, 15}, so a
    CTA's members finish at different steps, several instances complete in one step, and
    zero-length collectives run serial mode."""
    from randgraphs import random_spmd_graphs
    if seed % 2:
        monkeypatch.setenv("FL_CLUSTER_CTAS", str(3 + seed % 4))
    gs, topo = random_spmd_graphs(50_000 + seed, 1025 + 317 * seed, n_nodes=16 + seed, per_rank_dur=seed % 3 != 0)
    _check_race(gs, topo, seed, (("ring", 1), ("ring", 2)))


@pytest.mark.parametrize("world,reps", [(32, 1), (64, 1), (1024, 1), (64, 300), (1024, 100)])
def test_engine_lean_pass_leaves_unfoldable_points_to_the_general_one(world, reps):
    """A batched launch takes the lean variant (no events, every lane a rank, static hosts only)
    with a second pass of the general one for the points that cannot fold: here every other
    point re-costs the COMP nodes on a device so fast that their durations round to 0 ns
    (zero-length nodes at t = 0, serial mode).  Both kinds of point, interleaved in one launch,
    against the oracle on graphs carrying the re-costed durations.  fl_sweep_run launches the
    second pass only after reading a FL_RETRY status back; `reps` > 1 repeats the four points
    past the resident grid, so the statuses come back through the staging copy instead of
    mapped memory."""
    import copy
    from oracle.pyoracle import duration_from_flops
    gs = synth.synth_transformer(synth.PRESETS["tiny"], synth.ParallelConfig(synth.Strategy.DP, world), world)
    specs = [(f"switch:{world}:{bw}GB:1us", algo) for bw in (25, 400) for algo in ("ring", "tree")]
    peaks = [1e12, 1e30, 3e14, 1e30]
    topos = [parse_topology(sp) for sp, _ in specs]
    pts = E.DesignPoints.from_topologies(topos * reps, [a for _, a in specs] * reps)
    pts.peak_flops = np.array(peaks * reps, np.float64)
    pts.efficiency = np.full(len(specs) * reps, 0.5, np.float64)
    out = E.simulate_batch(gs, pts)
    for i, ((spec, algo), topo) in enumerate(zip(specs, topos)):
        g2 = copy.deepcopy(gs)
        for g in g2:
            for n in g.nodes:
                if n.flops is not None:
                    n.duration_ns = duration_from_flops(n.flops, peaks[i], 0.5)
        want = O.sweep_row(g2, topo, algo)
        for j in range(i, len(specs) * reps, len(specs)):
            assert int(out["status"][j]) == 0
            assert {k: int(out[k][j]) for k in ROW_KEYS} == want, (spec, algo, peaks[i], j)


# ---- critical-path node trace (the path rule is documented at engine.critical_path_trace) ----

def _trace_both(gs, topo, algo):
    try:
        want = O.critical_path_trace(gs, topo, algo)
    except O.OracleError as e:
        want = e.kind
    try:
        got = E.critical_path_trace(gs, topo, algo)
    except EngineError:
        raise
    except Exception as e:
        got = type(e).__name__
    return got, want


@pytest.mark.parametrize("seed", range(120))
def test_critical_path_trace_random_vs_oracle(seed):
    gs, topo = random_graphs(seed)
    for algo in ("ring", "tree"):
        got, want = _trace_both(gs, topo, algo)
        assert got == want, (seed, algo)


@pytest.mark.parametrize("seed", range(40))
def test_critical_path_trace_p2p_vs_oracle(seed):
    from randgraphs import random_p2p_graphs
    gs, topo = random_p2p_graphs(seed, mesh=seed % 2 == 1)
    got, want = _trace_both(gs, topo, "ring")
    assert got == want, seed


@pytest.mark.parametrize("spec,algo", [("switch:64:50GB:2us", "ring"), ("mesh:8x8:100GB:500ns", "mesh-hier")])
def test_critical_path_trace_fsdp_vs_oracle(spec, algo):
    gs = synth.synth_transformer(synth.PRESETS["llama-8b-like"], synth.ParallelConfig(synth.Strategy.FSDP, 64), 64)
    got, want = _trace_both(gs, parse_topology(spec), algo)
    assert got == want
    length, path = got
    assert length == E.critical_path(gs, parse_topology(spec), algo) and len(path) > 1


def test_engine_c3_full_grid_vs_oracle():
    """BASELINE config 3 in full -- 4096 design points x 1024 ranks x 832 nodes in one
    launch -- every row bit-exact against the CPU oracle's (tests/golden/make_c3_grid.py),
    plus the reference's own invariants (critical path <= makespan, test_simulator.py:275-295;
    exposed comm <= comm busy; busy times <= makespan)."""
    from pathlib import Path
    from paper_2604_17550_b200 import sweep as S
    w = S.c3_workload()
    gs = S.workload_graphs(w)
    out = E.simulate_batch(gs, w.points)
    assert (out["status"] == 0).all()
    got = np.stack([np.asarray(out[k], np.int64) for k in ROW_KEYS], 1)
    fx = np.load(Path(__file__).parent / "golden" / "c3_grid_rows.npz")
    assert list(fx["fields"]) == list(ROW_KEYS)
    bad = np.nonzero((got != fx["rows"]).any(1))[0]
    assert bad.size == 0, (bad[:5], got[bad[:2]], fx["rows"][bad[:2]])
    mk, cp = got[:, 0], got[:, 1]
    assert (cp <= mk).all() and (got[:, 4] <= got[:, 3]).all() and (got[:, 2] <= mk).all() and (got[:, 3] <= mk).all()


def test_sweep_rows_split_over_devices_is_identical():
    """sweep_rows(devices=[...]) evaluates contiguous slices concurrently (one host thread per
    GPU; here the same GPU twice) and returns exactly the single-launch rows."""
    from paper_2604_17550_b200.sweep import sweep_rows
    topos = [f"switch:8:{bw}GB:{lat}us" for bw in (10, 50, 400) for lat in (1, 5)] + ["mesh:2x4:100GB:1us"]
    args = ("tiny", ["fsdp:8", "dp:8"], topos, ["ring", "mesh-hier"][:1])
    one = sweep_rows(*args)
    two = sweep_rows(*args, devices=[0, 0, 0])
    assert one == two and len(one) == 2 * len(topos)


def test_c3_grid_with_device_traces():
    """BASELINE config 3 in full with the critical-path node trace of every point walked back
    on the device (fl_outputs.trace): rows unchanged (golden full-grid rows), every path ends
    at the row's critical path, and four points' paths equal the oracle restatement's
    (pyoracle.critical_path_trace, the rule of engine.critical_path_trace)."""
    from pathlib import Path
    from paper_2604_17550_b200 import sweep as S
    from paper_2604_17550_b200.topology import Topology, TopologyKind
    w = S.c3_workload()
    gs = S.workload_graphs(w)
    eng = E.Engine(gs)
    try:
        out = eng.run(w.points, trace_cap=4 * eng.gs.max_nodes)
    finally:
        eng.close()
    fx = np.load(Path(__file__).parent / "golden" / "c3_grid_rows.npz")
    assert (out["status"] == 0).all() and (out["rows"] == fx["rows"]).all()
    paths = E.trace_paths(eng.gs, out)
    assert all(len(p) > 1 for p in paths)
    flat = O.flatten(gs)
    algos = {0: "ring", 1: "tree", 2: "mesh-hier"}
    pts = w.points
    for i in (0, 1000, 2049, 4095):
        kind = TopologyKind.SWITCH if pts.topo_kind[i] == 0 else TopologyKind.MESH2D
        topo = Topology(kind, 1024, float(pts.bw[i]), int(pts.latency[i]), int(pts.rows[i]), int(pts.cols[i]))
        length, path = O.critical_path_trace(gs, topo, algos[int(pts.algo[i])], flat=flat)
        assert length == int(out["rows"][i, 1])
        assert paths[i] == path, i
