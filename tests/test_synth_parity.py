"""Our graph families vs the reference generator, node for node (build container only)."""

import sys

import pytest

from conftest import REFERENCE_SRC
from paper_2604_17550_b200 import synth as ms

pytestmark = pytest.mark.reference


def _ref():
    sys.path.insert(0, str(REFERENCE_SRC))
    from trainsim import synth as rs
    return rs


def canon(gs):
    out = []
    for g in gs[:2] + gs[-1:]:
        nodes = [(n.node_id, n.kind.value, n.op_name, list(n.inputs), list(n.outputs), list(n.data_deps),
                  [tuple(c) for c in n.ctrl_deps], n.duration_ns,
                  (n.coll.kind.value, list(n.coll.group), n.coll.comm_bytes) if n.coll else None) for n in g.nodes]
        tens = sorted((k, v.tensor_id, list(v.shape), v.dtype.value, v.bytes) for k, v in g.tensors.items())
        out.append((g.rank, g.world_size, nodes, tens, g.meta))
    return out


@pytest.mark.parametrize("preset", ["tiny", "llama-8b-like", "llama-70b-like"])
@pytest.mark.parametrize("strat", ["dp", "fsdp", "tp"])
@pytest.mark.parametrize("mode", ["delayed", "none"])
@pytest.mark.parametrize("deg", [2, 4, 8])
def test_synth_matches_reference(preset, strat, mode, deg):
    rs = _ref()
    def build(mod):
        try:
            return canon(mod.synth_transformer(mod.PRESETS[preset],
                                               mod.ParallelConfig(mod.Strategy(strat), deg, mod.FsdpMode(mode)), deg))
        except Exception as e:
            return type(e).__name__
    assert build(ms) == build(rs)


@pytest.mark.parametrize("strat", ["dp", "fsdp"])
def test_synth_matches_reference_c4_scale(strat):
    """The BASELINE config-4 graphs themselves: llama-70b-like at 8192 ranks."""
    rs = _ref()
    def build(mod):
        gs = mod.synth_transformer(mod.PRESETS["llama-70b-like"], mod.ParallelConfig(mod.Strategy(strat), 8192), 8192)
        assert len(gs) == 8192 and all(g.nodes is gs[0].nodes for g in gs)   # one shared node list
        return canon(gs)
    assert build(ms) == build(rs)


def test_flops_recost_reproduces_baked_durations():
    """Every COMP node's flops re-costed on the default device gives its duration_ns."""
    from paper_2604_17550_b200.costs import DEFAULT_DEVICE, duration_from_flops
    gs = ms.synth_transformer(ms.PRESETS["llama-8b-like"], ms.ParallelConfig(ms.Strategy.FSDP, 8), 8)
    comps = [n for n in gs[0].nodes if n.kind.value == "COMP"]
    assert comps and all(n.flops is not None for n in comps)
    assert all(duration_from_flops(n.flops, DEFAULT_DEVICE) == n.duration_ns for n in comps)
