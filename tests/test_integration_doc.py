"""INTEGRATION.md's ctypes stub, executed as written (the doc must stay runnable)."""
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2604_17550_b200 import engine as E
from paper_2604_17550_b200 import synth
from paper_2604_17550_b200.topology import parse_topology

ROOT = Path(__file__).resolve().parent.parent


def _stub_source():
    text = (ROOT / "INTEGRATION.md").read_text()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    src = next(b for b in blocks if "def sweep_rows" in b)
    return src.replace("/path/to/paper_2604_17550_b200/_build/libflint_b200.so",
                       str(ROOT / "paper_2604_17550_b200" / "_build" / "libflint_b200.so"))


def test_stub_parses():
    compile(_stub_source(), "INTEGRATION.md", "exec")


@pytest.mark.gpu
def test_stub_matches_simulate_batch():
    ns = {}
    exec(compile(_stub_source(), "INTEGRATION.md", "exec"), ns)
    gs = synth.synth_transformer(synth.PRESETS["tiny"], synth.ParallelConfig(synth.Strategy.FSDP, 8), 8)
    topos = [parse_topology(s) for s in ("switch:8:25GB:2us", "switch:8:400GB:100ns", "switch:8:10GB:10us")]
    algo = E.CollectiveAlgo.RING
    status, rows = ns["sweep_rows"](gs, topos, algo)
    want = E.simulate_batch(gs, E.DesignPoints.from_topologies(topos, ["ring"] * 3))
    assert (status == 0).all()
    assert (rows == np.stack([want[k] for k in E.ROW_FIELDS], 1)).all()
