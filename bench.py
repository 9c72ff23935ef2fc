#!/usr/bin/env python
"""Benchmark of the hot path: batched design-point evaluation of a workload graph.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c3|c2]

One *step* = one engine launch evaluating every design point of the
workload (BASELINE config 3 by default: llama-8b-like fsdp:1024, 4096 points,
851,968 (rank, node) pairs per point) -- simulate + critical_path + the
per-point reductions of cli._sweep_row for all of them.  Under torchrun each
process drives one GPU; the job is weak-scaled: GPU k evaluates the C3 grid
for compute-efficiency variant k (k = 0 is exactly C3), and the rows are
all-gathered over NCCL at the end of every step.

Prints one JSON line (rank 0): `value` = (rank, node, design point) triples
per second over all GPUs with inputs resident in HBM, `e2e` = the same
through the public host-buffer API (copies included), `roofline` for the
sweep kernel, `cpu_baseline` = the CPU oracle (oracle/flint_oracle.c) timed
on a bounded sample of the same workload.  `--impl reference` times that CPU
implementation alone with every host thread (the reference arm).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "graph-node×design-point evaluations/sec at 1/2/4/8 B200; % HBM roofline"
UNIT = "graph-node×design-point evaluations/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------- clocks


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                self.out = ""
        return False

    def summary(self):
        if not self.proc or not getattr(self, "out", ""):
            return None
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for row in csv.reader(io.StringIO(self.out)):
            if len(row) < 9:
                continue
            try:
                sm.append(float(row[1])); mx = max(mx, float(row[2]))
            except ValueError:
                continue
            for name, v in zip(names, row[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------ workload


def load_workload(name: str):
    from paper_2604_17550_b200 import sweep as S
    w = {"c3": S.c3_workload, "c2": S.c2_workload, "c4": S.c4_workload}[name]()
    graphs = S.workload_graphs(w)
    return w, graphs


def workload_desc(w, gs) -> dict:
    st = gs.structs[0]
    return {"workload": {"c3": "BASELINE config 3: llama-8b-like FSDP (delayed) graph at 1024 ranks, 4096 design "
                               "points = {switch:1024+ring, mesh:32x32+mesh-hier} x 64 bw [10GB/s,1.8TB/s] x "
                               "32 latency [100ns,20us]",
                         "c2": "BASELINE config 2: GPT-2 small dp:64, 256 design points = {ring, tree} x 16 bw "
                               "[10GB/s,1.8TB/s] x 8 latency [100ns,10us]",
                         "c4": "BASELINE config 4 scale: llama-70b-like FSDP graph at 8192 ranks (clusters of 8 "
                               "CTAs per design point), design points from {switch:8192+ring, mesh:64x128+"
                               "mesh-hier} x 128 bw [10GB/s,1.8TB/s] x 64 latency [100ns,20us]"}[w.name],
            "model": w.model, "parallel": w.parallel, "ranks": gs.n_ranks, "nodes_per_rank": st.n,
            "edges_per_rank": int(st.pred_off[-1]), "points_per_gpu": len(w.points),
            "units_per_point": gs.units()}


def bytes_per_unit(gs) -> float:
    """B = 8 (4 + 2 E/N) algorithmic bytes per (rank, node, point)."""
    st = gs.structs[0]
    return 8.0 * (4.0 + 2.0 * int(st.pred_off[-1]) / st.n)


def measured_peak_hbm():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except (KeyError, ValueError):
            pass
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def profiled_traffic(workload: str):
    p = ROOT / "profiles" / f"traffic_{workload}.json"
    if p.exists():
        try:
            return json.loads(p.read_text())
        except ValueError:
            return None
    return None


# ------------------------------------------------------------ CPU oracle


def oracle_sample(gs_graphs, w, idxs, threads: int):
    """Run the CPU oracle on design points `idxs` with `threads` threads; returns seconds."""
    from concurrent.futures import ThreadPoolExecutor
    from oracle import pyoracle as O
    from paper_2604_17550_b200.topology import Topology, TopologyKind
    flat = getattr(oracle_sample, "_flat", None)
    if flat is None or getattr(oracle_sample, "_key", None) != id(gs_graphs):
        flat = O.flatten(gs_graphs)
        oracle_sample._flat, oracle_sample._key = flat, id(gs_graphs)
    pts = w.points
    algos = {0: "ring", 1: "tree", 2: "mesh-hier"}
    R = len(gs_graphs)

    def one(i):
        kind = TopologyKind.SWITCH if pts.topo_kind[i] == 0 else TopologyKind.MESH2D
        topo = Topology(kind, R, float(pts.bw[i]), int(pts.latency[i]), int(pts.rows[i]), int(pts.cols[i]))
        return O.sweep_row(gs_graphs, topo, algos[int(pts.algo[i])], flat=flat)

    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=threads) as ex:
        rows = list(ex.map(one, idxs))
    return time.perf_counter() - t0, rows


def run_reference(args):
    """The reference arm: the CPU implementation of the path on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import pyoracle as O
    O.build()
    w, graphs = load_workload(args.workload)
    from paper_2604_17550_b200.store import compile_graphs
    gs = compile_graphs(graphs)
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    n = len(w.points)
    stride = max(1, n // (threads * (args.steps + args.warmup) + 1))
    order = [(k * stride) % n for k in range(threads * (args.steps + args.warmup))]
    times = []
    for s in range(args.warmup + args.steps):
        dt, _ = oracle_sample(graphs, w, order[s * threads:(s + 1) * threads], threads)
        if s >= args.warmup:
            times.append(dt)
    units = threads * gs.units()
    step_s = sum(times) / len(times)
    value = units / step_s
    sample = (f"{threads} design points per step (one per host thread) of the {args.workload.upper()} grid, "
              f"every {stride}th point; oracle/flint_oracle.c (C restatement of simulate+critical_path, "
              f"pinned to the reference) per point")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": workload_desc(w, gs),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                             "cpu_model": _cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _cpu_model() -> str:
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ------------------------------------------------------------ our arm


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (the engine has no CPU path)")
    # FLINT_BENCH_SHARE_GPU=1 (development only): every rank on the visible GPUs modulo their
    # count, gloo for the result gather -- exercises the multi-rank logic on a 1-GPU box
    share = os.environ.get("FLINT_BENCH_SHARE_GPU") == "1"
    if share:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cdev = torch.device("cpu") if share else dev       # where the collectives' tensors live
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    from paper_2604_17550_b200 import sweep as S
    from paper_2604_17550_b200.engine import Engine
    w, graphs = load_workload(args.workload)
    if args.points:
        w.points = w.points.take(np.linspace(0, len(w.points) - 1, args.points).round().astype(np.int64))
    eng = Engine(graphs, device=local)
    gs = eng.gs
    n = len(w.points)
    units_step = n * gs.units()                        # per GPU, W_sched == W (no rank collapse)
    pts = w.points
    # weak scaling: GPU k re-costs compute for efficiency 1 - 0.05 k (k = 0 reproduces C3 exactly)
    pts.peak_flops = np.full(n, 1.0e12, np.float64)
    pts.efficiency = np.full(n, 1.0 - 0.05 * rank, np.float64)

    cols = {"algo": (pts.algo, torch.uint8), "topo_kind": (pts.topo_kind, torch.uint8), "bw": (pts.bw, torch.float64),
            "latency": (pts.latency, torch.int64), "rows": (pts.rows, torch.int32), "cols": (pts.cols, torch.int32),
            "peak_flops": (pts.peak_flops, torch.float64), "efficiency": (pts.efficiency, torch.float64)}
    d_in = {k: torch.as_tensor(np.ascontiguousarray(v)).to(dev) for k, (v, _) in cols.items()}
    d_status = torch.zeros(n, dtype=torch.int32, device=dev)
    d_rows = torch.zeros((n, 6), dtype=torch.int64, device=dev)
    ptrs = {k: t.data_ptr() for k, t in d_in.items()}
    ptrs.update(out_status=d_status.data_ptr(), out_rows=d_rows.data_ptr())
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)       # > L2 (126 MB)
    per = -(-n * world // world)
    gather_out = torch.empty((n * world, 7), dtype=torch.int64, device=cdev) if world > 1 else None
    gather_in = torch.empty((n, 7), dtype=torch.int64, device=cdev) if world > 1 else None

    def step():
        k = eng.run_device(ptrs, stream.cuda_stream, n)
        return k

    def gather():
        if world > 1:
            gather_in[:, :6].copy_(d_rows)
            gather_in[:, 6].copy_(d_status)
            dist.all_gather_into_tensor(gather_out, gather_in)

    for _ in range(args.warmup):
        step(); gather()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    launches = 0
    k_ms, s_ms = [], []
    with ClockSampler(local) as clocks:
        for _ in range(args.steps):
            flush.zero_()
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            launches += step()
            e1.record(stream)
            gather()
            e2.record(stream)
            torch.cuda.synchronize()
            k_ms.append(e0.elapsed_time(e1))
            s_ms.append(e0.elapsed_time(e2))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    total_ms = sum(s_ms)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = world * units_step / (ms_per_step / 1e3)
    status = d_status.cpu().numpy()
    if (status != 0).any():
        raise SystemExit(f"engine returned non-OK status for {(status != 0).sum()} points")

    # ---- e2e: public host-buffer API (fl_sweep_run), pinned host SoA, rows back to host ----
    pin = {k: torch.as_tensor(np.ascontiguousarray(v)).pin_memory().numpy() for k, (v, _) in cols.items()}
    from paper_2604_17550_b200.engine import DesignPoints
    hp = DesignPoints(pin["algo"], pin["topo_kind"], pin["bw"], pin["latency"], pin["rows"], pin["cols"],
                      pin["peak_flops"], pin["efficiency"])
    for _ in range(max(1, args.warmup)):
        eng.run(hp)
    e2e_s = []
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = eng.run(hp)
        if world > 1:
            S.gather_rows(out["status"], out["rows"], n * world, world, rank, device=cdev)
        e2e_s.append(time.perf_counter() - t0)
    e2e_step = sum(e2e_s) / len(e2e_s)
    if world > 1:
        t = torch.tensor([e2e_step], dtype=torch.float64, device=cdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_step = float(t.item())
    h2d = sum(v.nbytes for v in pin.values())
    d2h = out["status"].nbytes + out["rows"].nbytes

    kernel_ms = sum(k_ms) / len(k_ms)
    bpu = bytes_per_unit(gs)
    peak, peak_src = measured_peak_hbm()
    achieved = bpu * units_step / (kernel_ms / 1e3) / 1e9
    traffic = profiled_traffic(args.workload) if not args.points else None   # (captured on the full grid)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic.get("dram_bytes_per_launch") if traffic else None,
                "peak_source": peak_src, "kernel": "fl::sweep_kernel<1>",
                "kernel_ms": kernel_ms, "algorithmic_bytes_per_unit": bpu,
                "units_per_launch": units_step}

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {**workload_desc(w, gs), "parallelism": f"dp{world} over design points",
                       "l2": "flushed before every timed step (256 MiB memset)",
                       "w_sched_equals_w": True},
            "roofline": roofline,
            "e2e": {"value": world * units_step / e2e_step, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": launches, "clocks": clocks.summary()}

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import pyoracle as O
        O.build()
        idxs = list(range(0, n, max(1, n // args.cpu_points)))[: args.cpu_points]
        dt, rows = oracle_sample(graphs, w, idxs, 1)
        got = d_rows.cpu().numpy()
        if pts.efficiency[0] == 1.0:
            from paper_2604_17550_b200.engine import ROW_FIELDS
            for i, r in zip(idxs, rows):
                assert [int(x) for x in got[i]] == [r[k] for k in ROW_FIELDS], f"GPU/oracle mismatch at point {i}"
        line["cpu_baseline"] = {"value": len(idxs) * gs.units() / dt, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"{len(idxs)} of the {n} design points (every {n // len(idxs)}th), "
                                          f"single thread, oracle/flint_oracle.c; rows checked equal to the GPU's",
                                "seconds": dt, "cpu_model": _cpu_model()}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=["c3", "c2", "c4"], default="c3")
    ap.add_argument("--points", type=int, default=0, help="evaluate an evenly spaced subset of the grid")
    ap.add_argument("--cpu-points", type=int, default=6)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        log("note: W >= 3 warm-up steps are required by the bench contract; raising to 3")
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
