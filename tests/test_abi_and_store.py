"""CPU-only checks of the boundary: the C-ABI library and the graph compiler."""

import re
from pathlib import Path

import numpy as np
import pytest

from paper_2604_17550_b200 import _native, synth
from paper_2604_17550_b200.store import compile_graphs, desc_arrays
from paper_2604_17550_b200.errors import InconsistentGroupsError

ROOT = Path(__file__).resolve().parent.parent


def header_functions():
    text = (ROOT / "include" / "flint_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|const char \*)\s*\*?\s*(fl_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    lib = _native.lib()       # builds in-tree with nvcc if needed; loads without a GPU
    names = header_functions()
    assert set(names) == set(_native.EXPORTED)
    for name in names:
        assert hasattr(lib, name), name
    assert lib.fl_version() == _native._header_abi_version()


def test_library_is_sm100a_only():
    import subprocess
    res = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB)], capture_output=True, text=True)
    arches = set(re.findall(r"sm_\d+a?", res.stdout))
    assert arches == {"sm_100a"}, res.stdout


def test_compile_c3_structure_shared_once():
    R = 64
    gs = synth.synth_transformer(synth.PRESETS["llama-8b-like"], synth.ParallelConfig(synth.Strategy.FSDP, R), R)
    cs = compile_graphs(gs)
    assert len(cs.structs) == 1 and cs.n_ranks == R
    st = cs.structs[0]
    assert st.n == 832 and len(st.colls) == 96 and cs.n_inst == 96
    assert int(st.pred_off[-1]) == 1596            # E, deduplicated
    assert cs.units() == R * 832
    d = desc_arrays(cs)
    assert d["inst_mem_off"][-1] == 96 * R
    assert (d["rank_coll_inst"] == np.arange(96)[None, :]).all()
    # ids ascend with index; node list order is id order for synthesized graphs
    assert (np.diff(st.node_id) > 0).all() and (st.listpos == np.arange(832)).all()


def test_compile_rejects_inconsistent_groups():
    from golden_io import corpus, decode_graphs
    case = next(c for c in corpus() if c["name"] == "inconsistent")
    with pytest.raises(InconsistentGroupsError):
        compile_graphs(decode_graphs(case))


def test_compile_rejects_duplicate_ranks():
    gs = synth.synth_transformer(synth.PRESETS["tiny"], synth.ParallelConfig(synth.Strategy.DP, 2), 2)
    gs[1].rank = 0
    with pytest.raises(ValueError):
        compile_graphs(gs)


def test_engine_refuses_unmatched_channel_with_deadlock_error():
    """A SEND without its RECV (simulator.py:177-200): the batched engine raises the
    reference's DeadlockError before any launch instead of returning rows."""
    from paper_2604_17550_b200.engine import Engine
    from paper_2604_17550_b200.errors import DeadlockError
    from paper_2604_17550_b200.graph import Node, NodeKind, P2pSpec, WorkloadGraph
    g0 = WorkloadGraph(0, 2, [Node(0, NodeKind.SEND, "send", p2p=P2pSpec(1, 64, 7))], {}, {"graph_inputs": []})
    g1 = WorkloadGraph(1, 2, [Node(0, NodeKind.HOST, "idle")], {}, {"graph_inputs": []})
    with pytest.raises(DeadlockError):
        Engine([g0, g1])
