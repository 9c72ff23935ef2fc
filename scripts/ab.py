"""A/B timing of engine builds (development tool, not part of the product).

    python scripts/ab.py build NAME [-DFLAG ...]      # here: nvcc into paper_2604_17550_b200/_build/ab_NAME.so
    python scripts/ab.py run [--workload c3] [--points N] [--reps K] NAME ...   # on the GPU box

`run` times every variant on the same evenly spaced subset of the workload's
design points (CUDA events around the launch, L2 flushed before each rep) in
its own process, and checks every variant's rows and status bit-for-bit
against the first one.  NAME "base" is the default in-tree library.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
BUILD = ROOT / "paper_2604_17550_b200" / "_build"


def lib_path(name):
    return str(BUILD / "libflint_b200.so") if name == "base" else str(BUILD / f"ab_{name}.so")


def child(name, workload, points, reps):
    import numpy as np
    import torch
    from paper_2604_17550_b200 import sweep as S
    from paper_2604_17550_b200.engine import Engine
    ranks = 0
    if ":" in workload:                 # e.g. c3:512 -- the C3 grid on fsdp:512 (scaling probes)
        workload, ranks = workload.split(":")[0], int(workload.split(":")[1])
    part = {"c4dp": 0, "c4fsdp": 1}.get(workload, 0)     # one family of the C4 grid
    if "." in workload:                 # e.g. c2x.1 -- family 1 of a multi-family workload
        workload, part = workload.split(".")[0], int(workload.split(".")[1])
    w = {"c3": S.c3_workload, "c2": S.c2_workload, "c4dp": S.c4_workload, "c4fsdp": S.c4_workload,
         "c2x": S.c2x_workload, "meshx": S.meshx_workload}[workload]()
    w.parts = [w.parts[part]]
    if ranks:
        w.parts[0].parallel = f"fsdp:{ranks}"
        side = int(round(ranks ** 0.5))
        while ranks % side:
            side -= 1
        w.points.rows[:] = np.where(w.points.rows > 0, side, 0)
        w.points.cols[:] = np.where(w.points.cols > 0, ranks // side, 0)
    if os.environ.get("AB_FSDP_NONE"):      # the same grid on the fsdp NONE family (counted dependencies)
        from paper_2604_17550_b200 import synth as SY
        p = SY.parse_parallel(w.parallel)
        graphs = SY.synth_transformer(SY.PRESETS[w.model], SY.ParallelConfig(p.strategy, p.degree, SY.FsdpMode.NONE),
                                      p.degree)
    else:
        graphs = S.workload_graphs(w)
    n_all = len(w.points)
    if points and points < n_all:
        w.points = w.points.take(np.linspace(0, n_all - 1, points).round().astype(np.int64))
    pts = w.points
    n = len(pts)
    pts.peak_flops = np.full(n, 1.0e12)
    pts.efficiency = np.full(n, 1.0)
    eng = Engine(graphs, device=0)
    dev = torch.device("cuda:0")
    cols = {"algo": pts.algo, "topo_kind": pts.topo_kind, "bw": pts.bw, "latency": pts.latency, "rows": pts.rows,
            "cols": pts.cols, "peak_flops": pts.peak_flops, "efficiency": pts.efficiency}
    d_in = {k: torch.as_tensor(np.ascontiguousarray(v)).to(dev) for k, v in cols.items()}
    st = torch.zeros(n, dtype=torch.int32, device=dev)
    rows = torch.zeros((n, 6), dtype=torch.int64, device=dev)
    ptrs = {k: t.data_ptr() for k, t in d_in.items()}
    ptrs.update(out_status=st.data_ptr(), out_rows=rows.data_ptr())
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(2):
        eng.run_device(ptrs, stream.cuda_stream, n)
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        eng.run_device(ptrs, stream.cuda_stream, n)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    out = Path(f"/tmp/ab_rows_{name}.npy")
    np.save(out, np.concatenate([rows.cpu().numpy(), st.cpu().numpy()[:, None].astype(np.int64)], axis=1))
    units = n * eng.gs.units()
    print(json.dumps({"name": name, "ms": sorted(ms)[len(ms) // 2], "ms_all": ms, "points": n,
                      "units_per_s": units / (sorted(ms)[len(ms) // 2] / 1e3)}))


def main():
    mode = sys.argv[1]
    if mode == "build":
        from paper_2604_17550_b200 import _native
        name, flags = sys.argv[2], [f[2:] if f.startswith("-D") else f for f in sys.argv[3:]]
        BUILD.mkdir(exist_ok=True)
        err = _native.build_variant(Path(lib_path(name)), flags, verbose=True)
        lines = err.splitlines()
        for i, l in enumerate(lines):
            if "sweep_kernelILi1ELb0" in l and "Function properties" in l:
                print(name, lines[i + 1].strip(), "|", lines[i + 2].strip())
        return
    if mode == "child":
        child(sys.argv[2], sys.argv[3], int(sys.argv[4]), int(sys.argv[5]))
        return
    import argparse
    import numpy as np
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+")
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--points", type=int, default=1184)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args(sys.argv[2:])
    res, ref = [], None
    for name in a.names:
        env = dict(os.environ, FLINT_B200_LIB=lib_path(name))
        p = subprocess.run([sys.executable, __file__, "child", name, a.workload, str(a.points), str(a.reps)],
                           env=env, capture_output=True, text=True, timeout=1800)
        line = [l for l in p.stdout.splitlines() if l.startswith("{")]
        if p.returncode or not line:
            print(f"{name}: FAILED rc={p.returncode}\n{p.stderr[-2000:]}", flush=True)
            continue
        r = json.loads(line[-1])
        got = np.load(f"/tmp/ab_rows_{name}.npy")
        if ref is None:
            ref = got
            r["match"] = "ref"
        else:
            r["match"] = bool((got == ref).all())
        res.append(r)
        print(json.dumps(r), flush=True)
    base = res[0]["ms"] if res else 0
    for r in res:
        print(f"{r['name']:24s} {r['ms']:9.3f} ms  x{base / r['ms']:.3f}  match={r['match']}")


if __name__ == "__main__":
    main()
