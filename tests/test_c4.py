"""BASELINE config 4 (llama-70b-like at 8192 ranks) pinned end to end.

tests/golden/c4_golden.json (tests/golden/make_c4_golden.py):
* ``family``: rows the reference itself returns on the C4 graph family
  (llama-70b-like dp and fsdp, synth.py:164-335) at R in {16, 64, 256} for
  every (strategy, algorithm) pair of the C4 grid plus fsdp ring
  (collectives.py:251-293);
* ``grid``: 32 rows of the C4 grid itself at R = 8192 (8 per family) from the
  CPU oracle, which ``family`` pins to the reference on the same graphs.

CPU: the oracle reproduces every ``family`` row.  GPU (-m gpu): the engine
reproduces every ``family`` row and every ``grid`` row bit-exactly, the 8192-
rank rows through the cluster-of-CTAs kernel in one launch per family.
"""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import pyoracle as O
from paper_2604_17550_b200 import synth
from paper_2604_17550_b200.topology import parse_topology

FIX = json.loads((Path(__file__).parent / "golden" / "c4_golden.json").read_text())
ROW = ("makespan_ns", "critical_path_ns", "compute_busy_ns", "comm_busy_ns", "exposed_comm_ns", "peak_mem_bytes")
_GRAPHS: dict = {}


def graphs(par):
    if par not in _GRAPHS:
        p = synth.parse_parallel(par)
        _GRAPHS[par] = synth.synth_transformer(synth.PRESETS["llama-70b-like"], p, p.degree)
    return _GRAPHS[par]


def _fam_ids():
    return [f"{r['parallel']}-{r['topo_spec']}-{r['algo']}" for r in FIX["family"]]


def test_fixture_covers_the_c4_grid_pairs():
    pairs = {(r["parallel"].split(":")[0], r["topo_spec"].split(":")[0], r["algo"]) for r in FIX["family"]}
    assert {("dp", "switch", "ring"), ("dp", "switch", "tree"), ("dp", "mesh", "mesh-hier"),
            ("fsdp", "mesh", "mesh-hier")} <= pairs
    fams = {(r["part"], r["algo"]) for r in FIX["grid"]}
    assert fams == {(0, "ring"), (0, "tree"), (0, "mesh-hier"), (1, "mesh-hier")}
    assert len(FIX["grid"]) >= 16


@pytest.mark.parametrize("row", FIX["family"], ids=_fam_ids())
def test_oracle_matches_reference_on_70b_family(row):
    got = O.sweep_row(graphs(row["parallel"]), parse_topology(row["topo_spec"]), row["algo"])
    assert got == {k: row[k] for k in ROW}


@pytest.mark.gpu
def test_engine_matches_reference_on_70b_family():
    from paper_2604_17550_b200 import engine as E
    by_par: dict = {}
    for r in FIX["family"]:
        by_par.setdefault(r["parallel"], []).append(r)
    for par, rows in by_par.items():
        topos = [parse_topology(r["topo_spec"]) for r in rows]
        out = E.simulate_batch(graphs(par), E.DesignPoints.from_topologies(topos, [r["algo"] for r in rows]))
        for i, r in enumerate(rows):
            assert int(out["status"][i]) == 0
            assert {k: int(out[k][i]) for k in ROW} == {k: r[k] for k in ROW}, (par, r["topo_spec"], r["algo"])


@pytest.mark.gpu
def test_engine_c4_grid_rows_at_8192_ranks():
    """The C4 grid's own design points at 8192 ranks (9-CTA clusters), both families."""
    from paper_2604_17550_b200 import engine as E
    from paper_2604_17550_b200 import sweep as S
    w = S.c4_workload()
    for k, part in enumerate(w.parts):
        rows = [r for r in FIX["grid"] if r["part"] == k]
        idx = np.asarray([r["point"] for r in rows], np.int64)
        out = E.simulate_batch(graphs(part.parallel), part.points.take(idx))
        for i, r in enumerate(rows):
            assert int(out["status"][i]) == 0
            got = {f: int(out[f][i]) for f in ROW}
            assert got == {f: r[f] for f in ROW}, (part.parallel, r["point"], r["algo"])
            assert got["critical_path_ns"] <= got["makespan_ns"]
