import sys, collections
sys.path.insert(0, ".")
import numpy as np
from paper_2604_17550_b200 import sweep as S
from paper_2604_17550_b200.engine import Engine
w = S.c3_workload(); gs = S.workload_graphs(w); eng = Engine(gs)
pts = w.points
for recost in (False, True):
    if recost:
        pts.peak_flops = np.full(len(pts), 1e12); pts.efficiency = np.full(len(pts), 1.0)
    for sub in (pts.slice(0, 8), pts.slice(2048, 2056), pts):
        out = eng.run(sub)
        c = collections.Counter(out["status"].tolist())
        print("recost", recost, "n", len(sub), dict(c), out["rows"][:2].tolist(), flush=True)
