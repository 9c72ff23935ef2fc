"""Time and record one C3 design point (llama-8b-like fsdp:1024) with the reference.

Usage: python tests/golden/c3_reference_point.py <topology spec> <algo> >> tests/golden/c3_r1024.jsonl
Takes ~15 min and ~20 GB RSS (critical_path). Build container only (needs /root/reference).
"""
import sys, json, time
sys.path.insert(0, "/root/reference/pkg/src")
from trainsim import *
from trainsim.synth import PRESETS, ParallelConfig, Strategy, FsdpMode, synth_transformer
from trainsim.simulator import simulate, critical_path, SimOptions
from trainsim.topology import parse_topology
from trainsim.collectives import CollectiveAlgo
spec, algo = sys.argv[1], sys.argv[2]
R = 1024
gs = synth_transformer(PRESETS["llama-8b-like"], ParallelConfig(Strategy.FSDP, R), R)
topo = parse_topology(spec)
t0 = time.time()
rep = simulate(gs, topo, SimOptions(algo=CollectiveAlgo(algo), record_events=False))
t1 = time.time()
cp = critical_path(gs, topo, CollectiveAlgo(algo))
t2 = time.time()
out = dict(spec=spec, algo=algo, R=R, makespan_ns=rep.makespan_ns, critical_path_ns=cp,
  compute_busy_ns=max(s.compute_busy_ns for s in rep.ranks.values()),
  comm_busy_ns=max(s.comm_busy_ns for s in rep.ranks.values()),
  exposed_comm_ns=rep.exposed_comm_ns, peak_mem_bytes=rep.peak_mem_bytes,
  distinct_rank_stats=len({(s.finish_ns,s.compute_busy_ns,s.comm_busy_ns,s.exposed_comm_ns,s.peak_mem_bytes) for s in rep.ranks.values()}),
  sim_s=t1-t0, cp_s=t2-t1)
print(json.dumps(out))
