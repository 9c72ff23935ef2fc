"""bench.py's multi-rank path through the real engine (one GPU shared by 2 ranks).

`python bench.py --gpus 2` re-launches itself under torch.distributed.run; each
rank evaluates its contiguous slice of the grid (sweep.shard) and the rows are
all-gathered inside the timed step.  FLINT_BENCH_SHARE_GPU=1 puts both ranks on
the one visible GPU (gloo for the gather), so the strong-scaled split and the
gather run through the engine on a 1-GPU box; the rows must equal N=1's.
Reference: share-nothing design points, pkg/src/trainsim/cli.py:352-358.
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent

pytestmark = pytest.mark.gpu


def _bench(tmp_path, gpus, workload, points, tag):
    out = tmp_path / f"rows_{tag}.npz"
    env = dict(os.environ, FLINT_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", str(gpus), "--workload", workload,
           "--points", str(points), "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--dump-rows", str(out)]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    line = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][-1])
    return line, np.load(out)


@pytest.mark.parametrize("workload,points", [("c3", 96), ("c2", 256)])
def test_bench_two_ranks_equal_one(tmp_path, workload, points):
    one, r1 = _bench(tmp_path, 1, workload, points, "n1")
    two, r2 = _bench(tmp_path, 2, workload, points, "n2")
    assert one["n_gpus"] == 1 and two["n_gpus"] == 2 and two["scaling"] == "strong"
    assert one["config"]["units_per_step"] == two["config"]["units_per_step"]
    assert sorted(r1.files) == sorted(r2.files)
    for k in r1.files:
        assert np.array_equal(r1[k], r2[k]), k
    assert (r1["status0"] == 0).all() and len(r1["rows0"]) == points
