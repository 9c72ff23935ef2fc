"""Development probe: where the C2 end-to-end time goes (fl_sweep_run host path vs kernel).

    python scripts/e2e_probe.py [c2|c3] [reps]
"""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2604_17550_b200 import _native, sweep as S                      # noqa: E402
from paper_2604_17550_b200.engine import DesignPoints, Engine               # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
w = {"c2": S.c2_workload, "c3": S.c3_workload}[wl]()
part = w.parts[0]
graphs = S.part_graphs(w, part)
pts = part.points
eng = Engine(graphs, device=0)
pin = {k: torch.as_tensor(np.ascontiguousarray(getattr(pts, k))).pin_memory().numpy()
       for k in ("algo", "topo_kind", "bw", "latency", "rows", "cols")}
hp = DesignPoints(pin["algo"], pin["topo_kind"], pin["bw"], pin["latency"], pin["rows"], pin["cols"], None, None)
for _ in range(20):
    eng.run(hp)
torch.cuda.synchronize()


def timeit(fn, n=reps):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e6, np.min(ts) * 1e6


print("Engine.run (python + fl_sweep_run)   median/min us: %.1f / %.1f" % timeit(lambda: eng.run(hp)))
n = len(hp)
st, rows = np.empty(n, np.int32), np.empty((n, 6), np.int64)
p = hp.raw()
o = _native.OutputsRaw(st.ctypes.data, rows.ctypes.data, None, None, None, None, 0, None, None, 0)
L = _native.lib()
print("fl_sweep_run only (ctypes)           median/min us: %.1f / %.1f" %
      timeit(lambda: L.fl_sweep_run(eng._h, C.addressof(p), C.addressof(o))))
# kernel alone, CUDA events, inputs on the device
dev = torch.device("cuda:0")
d_in = {k: torch.as_tensor(v).to(dev) for k, v in pin.items()}
d_st = torch.zeros(n, dtype=torch.int32, device=dev)
d_rows = torch.zeros((n, 6), dtype=torch.int64, device=dev)
ptrs = {k: t.data_ptr() for k, t in d_in.items()}
ptrs.update(out_status=d_st.data_ptr(), out_rows=d_rows.data_ptr())
stream = torch.cuda.current_stream(dev)
ks = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    eng.run_device(ptrs, stream.cuda_stream, n)
    e1.record(stream)
    torch.cuda.synchronize()
    ks.append(e0.elapsed_time(e1) * 1e3)
print("kernel (events, device inputs)        median/min us: %.1f / %.1f" % (np.median(ks), np.min(ks)))
print("run_device + synchronize (wall)       median/min us: %.1f / %.1f" %
      timeit(lambda: (eng.run_device(ptrs, stream.cuda_stream, n), torch.cuda.synchronize())))
# as bench.py times it: a 256 MiB L2 flush and a synchronize before every step
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def flushed(fn):
    ts = []
    for _ in range(reps // 4):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e6, np.min(ts) * 1e6


print("Engine.run after flush + sync         median/min us: %.1f / %.1f" % flushed(lambda: eng.run(hp)))
ks = []
for _ in range(reps // 4):
    flush.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    eng.run_device(ptrs, stream.cuda_stream, n)
    e1.record(stream)
    torch.cuda.synchronize()
    ks.append(e0.elapsed_time(e1) * 1e3)
print("kernel after flush (events)           median/min us: %.1f / %.1f" % (np.median(ks), np.min(ks)))
hp2 = DesignPoints(pin["algo"], pin["topo_kind"], pin["bw"], pin["latency"], pin["rows"], pin["cols"],
                   torch.full((n,), 1e12, dtype=torch.float64).pin_memory().numpy(),
                   torch.full((n,), 1.0, dtype=torch.float64).pin_memory().numpy())
print("Engine.run + peak/eff, flush + sync   median/min us: %.1f / %.1f" % flushed(lambda: eng.run(hp2)))
import gc
gc.disable()
print("  same, GC off                        median/min us: %.1f / %.1f" % flushed(lambda: eng.run(hp2)))
gc.enable()
