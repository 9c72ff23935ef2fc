"""Golden fixtures for IR ingestion and BASELINE config 1, made by the reference.

Run in the build container (the reference is mounted read-only there):

    python tests/golden/make_ingest_golden.py     # writes tests/golden/ingest.json.gz

* C1: the reference frontend (pkg/frontend, fxcapture)
  captures its test MLP Linear(16,32)->ReLU->Linear(32,8) under a fake
  8-rank process group on the meta device (pkg/frontend/tests/test_capture.py:
  45-78); the raw exports are stored, converted with trainsim.convert
  (traceio.py:322-465) and simulated on switch:8:25GB:1us, ring.
* The reference's own raw fixtures (pkg/tests/fixtures/raw_*.json) and
  malformed variants of them, with what convert / parse_raw_export return.
"""

from __future__ import annotations

import copy
import gzip
import json
import sys
import tempfile
from pathlib import Path

REF = Path("/root/reference/pkg")
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "frontend" / "src"))
sys.path.insert(0, str(REF / "frontend" / "tests"))
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent))

import trainsim as T  # noqa: E402
from trainsim import traceio as TI  # noqa: E402

from golden_io import canon  # noqa: E402
from make_expand_golden import run  # noqa: E402


def convert_rec(docs, device=None):
    rec = {"raw": docs}
    try:
        gs = [TI.convert(TI.parse_raw_export(d), device=device) for d in docs]
    except T.TrainsimError as e:
        rec["error"] = type(e).__name__
        return rec, None
    rec["hash"] = canon(gs)
    rec["meta"] = [g.meta for g in gs]
    rec["durations"] = [[n.duration_ns for n in g.nodes] for g in gs]
    return rec, gs


def main():
    import test_capture as TCAP
    out = {"c1": {}, "fixtures": []}
    with tempfile.TemporaryDirectory() as tmp:
        for r in range(8):
            cfg = TCAP.CaptureConfig(output_dir=tmp, rank=r, world_size=8)
            with TCAP.fake_group(r, 8):
                import torch
                with torch.device("meta"):
                    model = TCAP.Mlp()
                step = torch.compile(TCAP.dp_step(model), backend=TCAP.register_backend(cfg), fullgraph=True,
                                     dynamic=False)
                loss = step(torch.randn(4, 16, device="meta"))
                loss.backward()
        for tag in ("fwd0", "bwd0"):
            docs = [json.loads((Path(tmp) / f"capture_{tag}_rank{r}.json").read_text()) for r in range(8)]
            rec, gs = convert_rec(docs)
            topo = T.parse_topology("switch:8:25GB:1us")
            rec.update(run(gs, topo, "ring"))
            out["c1"][tag] = rec
    raw0 = json.loads((REF / "tests" / "fixtures" / "raw_mm_allreduce_rank0.json").read_text())
    raw1 = json.loads((REF / "tests" / "fixtures" / "raw_mm_allreduce_rank1.json").read_text())
    rec, gs = convert_rec([raw0, raw1])
    rec.update(run(gs, T.Topology.switch(2, 25e9, 1000), "ring"))
    out["fixtures"].append({"name": "mm_allreduce", **rec})
    rec, _ = convert_rec([raw0, raw1], device=T.DeviceSpec(3.5e14, 0.55))
    out["fixtures"].append({"name": "mm_allreduce_device", "device": [3.5e14, 0.55], **rec})
    # malformed variants: each must fail the way the reference fails
    def variant(name, fn):
        d = copy.deepcopy(raw0)
        fn(d)
        try:
            TI.parse_raw_export(d)
        except T.TrainsimError as e:
            out["fixtures"].append({"name": name, "raw": [d], "parse_error": type(e).__name__})
            return
        r, _ = convert_rec([d])
        out["fixtures"].append({"name": name, **r})
    variant("bad_version", lambda d: d.update(format_version="raw-ir/0"))
    variant("no_nodes", lambda d: d.update(nodes=[]))
    variant("dup_name", lambda d: d["nodes"].append(copy.deepcopy(d["nodes"][0])))
    variant("unseen_arg", lambda d: d["nodes"][1]["arg_names"].append("nope"))
    variant("bad_kind", lambda d: d["nodes"][0].update(kind="LOOP"))
    variant("unmapped", lambda d: [n.update(target="aten.fft") for n in d["nodes"] if n["kind"] == "CALL"][:1])
    variant("no_shape", lambda d: [n.update(tensor_out=None) for n in d["nodes"] if n["kind"] == "CALL"][:1])
    variant("bad_dtype", lambda d: [n["tensor_out"].update(dtype="torch.complex64") for n in d["nodes"]
                                    if n.get("tensor_out")][:1])
    variant("no_group", lambda d: [n.update(coll_attrs={"kind": "ALL_REDUCE"}) for n in d["nodes"]
                                   if n.get("coll_attrs")])
    variant("kind_clash", lambda d: [n["coll_attrs"].update(kind="ALL_GATHER") for n in d["nodes"]
                                     if n.get("coll_attrs")])
    with gzip.open(HERE / "ingest.json.gz", "wt") as f:
        json.dump(out, f, separators=(",", ":"))
    print({k: (v.get("sim"), v.get("cp")) for k, v in out["c1"].items()})
    print([(f["name"], f.get("error") or f.get("parse_error") or "ok") for f in out["fixtures"]])


if __name__ == "__main__":
    main()
