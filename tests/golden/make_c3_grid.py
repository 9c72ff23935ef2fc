"""Full BASELINE config-3 grid through the CPU oracle -> tests/golden/c3_grid_rows.npz.

4096 design points x R = 1024 (llama-8b-like fsdp:1024), every sweep-row field, computed
by oracle/flint_oracle.c (pinned to the reference: tests/test_oracle_golden.py, and the
two R = 1024 points of c3_r1024.jsonl measured with trainsim itself).  The GPU test
tests/test_gpu_parity.py::test_engine_c3_full_grid_vs_oracle compares a whole C3 sweep
against it, bit for bit.  Takes ~1 s per point per core:

    python tests/golden/make_c3_grid.py [threads]
"""
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import pyoracle as O                                   # noqa: E402
from paper_2604_17550_b200 import sweep as S                       # noqa: E402
from paper_2604_17550_b200.engine import ROW_FIELDS                # noqa: E402
from paper_2604_17550_b200.topology import Topology, TopologyKind  # noqa: E402


def main():
    threads = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    O.build()
    w = S.c3_workload()
    gs = S.workload_graphs(w)
    flat = O.flatten(gs)
    pts = w.points
    algos = {0: "ring", 1: "tree", 2: "mesh-hier"}

    def one(i):
        kind = TopologyKind.SWITCH if pts.topo_kind[i] == 0 else TopologyKind.MESH2D
        topo = Topology(kind, len(gs), float(pts.bw[i]), int(pts.latency[i]), int(pts.rows[i]), int(pts.cols[i]))
        r = O.sweep_row(gs, topo, algos[int(pts.algo[i])], flat=flat)
        return [r[k] for k in ROW_FIELDS]

    t0 = time.time()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        rows = np.array(list(ex.map(one, range(len(pts)))), np.int64)
    np.savez_compressed(Path(__file__).with_name("c3_grid_rows.npz"), rows=rows, fields=np.array(ROW_FIELDS))
    print(f"{len(rows)} points in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
