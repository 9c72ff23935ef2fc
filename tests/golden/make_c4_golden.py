"""Golden rows for BASELINE config 4 (llama-70b-like at 8192 ranks).

Run in the build container, where the reference is mounted read-only:

    python tests/golden/make_c4_golden.py          # writes tests/golden/c4_golden.json

Two fixtures, both committed:

* ``family`` -- rows the REFERENCE itself (``trainsim``, imported read-only from
  /root/reference/pkg/src, never copied) returns for the C4 graph family at
  reduced world sizes R in {16, 64, 256}: every (strategy, algorithm) pair of
  the C4 grid -- dp ring, dp tree, dp mesh-hier, fsdp mesh-hier -- plus fsdp
  ring, on bandwidth/latency corners of the C4 grid.  These pin the oracle and
  the engine on the 70B graphs (synth.py:164-335, collectives.py:251-293).
  At R = 8192 the reference is infeasible (critical_path is O(R^2) set unions,
  simulator.py:419-428; ~20 GB and 11 min already at R = 1024).
* ``grid`` -- rows of the C4 grid itself at R = 8192 (8 design points per
  family, 32 in total, indices into ``sweep.c4_workload()``'s parts) computed
  by the CPU oracle (oracle/flint_oracle.c), which ``family`` pins to the
  reference on the same graph family.  ~40 s and ~2.3 GB per point.
"""

from __future__ import annotations

import json
import multiprocessing as mp
import sys
import time
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
REF = Path("/root/reference/pkg/src")
OUT = HERE / "c4_golden.json"

ROW = ("makespan_ns", "critical_path_ns", "compute_busy_ns", "comm_busy_ns", "exposed_comm_ns", "peak_mem_bytes")
MESH = {16: "4x4", 64: "8x8", 256: "8x32"}
CORNERS = [("10GB", "100ns"), ("1800GB", "20us"), ("120GB", "1500ns")]


def family_cases():
    cases = []
    for R in (16, 64, 256):
        corners = CORNERS if R < 256 else CORNERS[:2]
        for par, kind, algo in (("dp", "switch", "ring"), ("dp", "switch", "tree"), ("dp", "mesh", "mesh-hier"),
                                ("fsdp", "mesh", "mesh-hier"), ("fsdp", "switch", "ring")):
            for bw, lat in corners:
                shape = str(R) if kind == "switch" else MESH[R]
                cases.append((f"{par}:{R}", f"{kind}:{shape}:{bw}:{lat}", algo))
    return cases


def ref_row(case):
    sys.path.insert(0, str(REF))
    import trainsim as T
    from trainsim.synth import PRESETS, ParallelConfig, synth_transformer
    par, spec, algo = case
    p = T.parse_parallel(par)
    gs = synth_transformer(PRESETS["llama-70b-like"], ParallelConfig(p.strategy, p.degree), p.degree)
    topo = T.parse_topology(spec)
    t0 = time.time()
    rep = T.simulate(gs, topo, T.SimOptions(algo=T.CollectiveAlgo(algo)))
    cp = T.critical_path(gs, topo, T.CollectiveAlgo(algo))
    row = {"parallel": par, "topo_spec": spec, "algo": algo,
           "makespan_ns": rep.makespan_ns, "critical_path_ns": cp,
           "compute_busy_ns": max(s.compute_busy_ns for s in rep.ranks.values()),
           "comm_busy_ns": max(s.comm_busy_ns for s in rep.ranks.values()),
           "exposed_comm_ns": rep.exposed_comm_ns, "peak_mem_bytes": rep.peak_mem_bytes}
    print(f"ref {par} {spec} {algo}: {time.time() - t0:.1f} s", flush=True)
    return row


def grid_indices():
    """8 points per family of the 64 x 64 (bw, latency) sub-grid: corners, edges, interior."""
    ij = [(0, 0), (63, 63), (0, 63), (63, 0), (21, 42), (42, 10), (37, 37), (5, 58)]
    return [i * 64 + j for i, j in ij]


def grid_row(job):
    sys.path.insert(0, str(ROOT))
    from oracle import pyoracle as O
    from paper_2604_17550_b200 import sweep as S
    from paper_2604_17550_b200.topology import Topology, TopologyKind
    part_idx, point = job
    w = S.c4_workload()
    part = w.parts[part_idx]
    gs = S.part_graphs(w, part)
    pts = part.points
    kind = TopologyKind.SWITCH if pts.topo_kind[point] == 0 else TopologyKind.MESH2D
    topo = Topology(kind, len(gs), float(pts.bw[point]), int(pts.latency[point]), int(pts.rows[point]),
                    int(pts.cols[point]))
    algo = {0: "ring", 1: "tree", 2: "mesh-hier"}[int(pts.algo[point])]
    t0 = time.time()
    row = O.sweep_row(gs, topo, algo)
    print(f"oracle part {part_idx} point {point}: {time.time() - t0:.1f} s", flush=True)
    return {"part": part_idx, "parallel": part.parallel, "point": point, "algo": algo, **row}


def main():
    ctx = mp.get_context("fork")
    sys.path.insert(0, str(ROOT))
    from paper_2604_17550_b200 import sweep as S
    w = S.c4_workload()
    # families: dp part holds {ring, tree, mesh-hier} x 4096, fsdp part {mesh-hier} x 4096
    jobs = [(0, k * 4096 + i) for k in range(3) for i in grid_indices()] + [(1, i) for i in grid_indices()]
    assert all(j[1] < len(w.parts[j[0]].points) for j in jobs)
    with ctx.Pool(8) as pool:
        fam = pool.map(ref_row, family_cases(), chunksize=1)
    with ctx.Pool(6) as pool:                        # ~2.3 GB each
        grid = pool.map(grid_row, jobs, chunksize=1)
    OUT.write_text(json.dumps({"family": fam, "grid": grid}, indent=0) + "\n")
    print("family rows:", len(fam), "grid rows:", len(grid))


if __name__ == "__main__":
    main()
