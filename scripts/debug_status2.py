import sys, collections
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2604_17550_b200 import sweep as S
from paper_2604_17550_b200.engine import Engine
w = S.c3_workload(); gs = S.workload_graphs(w); eng = Engine(gs)
pts = w.points; n = len(pts)
pts.peak_flops = np.full(n, 1e12); pts.efficiency = np.full(n, 1.0)
dev = torch.device("cuda", 0)
cols = {"algo": pts.algo, "topo_kind": pts.topo_kind, "bw": pts.bw, "latency": pts.latency, "rows": pts.rows, "cols": pts.cols, "peak_flops": pts.peak_flops, "efficiency": pts.efficiency}
d_in = {k: torch.as_tensor(np.ascontiguousarray(v)).to(dev) for k, v in cols.items()}
for k, t in d_in.items(): print(k, t.dtype, t.shape, t[:2].tolist(), t[2048:2050].tolist())
st = torch.zeros(n, dtype=torch.int32, device=dev); rows = torch.zeros((n, 6), dtype=torch.int64, device=dev)
ptrs = {k: t.data_ptr() for k, t in d_in.items()}; ptrs.update(status=st.data_ptr(), rows=rows.data_ptr())
s = torch.cuda.current_stream(dev)
for it in range(3):
    eng.run_device(ptrs, s.cuda_stream, n); torch.cuda.synchronize()
    stc = st.cpu().numpy()
    print("iter", it, collections.Counter(stc.tolist()), np.nonzero(stc)[0][:10], rows.cpu().numpy()[:1].tolist(), flush=True)
