"""Host cost helpers: reference known answers and agreement with the oracle."""

import itertools

import pytest

from oracle import pyoracle as O
from paper_2604_17550_b200.costs import (DEFAULT_DEVICE, CollectiveAlgo, DeviceSpec, analytical_duration,
                                         analytical_time, round_half_up_ns)
from paper_2604_17550_b200.errors import UnsupportedAlgoTopologyError
from paper_2604_17550_b200.graph import CollectiveKind, Dtype

AR, AG, RS = CollectiveKind.ALL_REDUCE, CollectiveKind.ALL_GATHER, CollectiveKind.REDUCE_SCATTER
RING, TREE, MESH = CollectiveAlgo.RING, CollectiveAlgo.TREE, CollectiveAlgo.MESH_HIER


def test_known_answers_from_reference_tests():
    # pkg/tests/test_collectives.py:126-162 (alpha 10, beta 1)
    assert analytical_time(AR, 1000, 4, RING, 10, 1.0) == 1560
    assert analytical_time(AG, 1000, 4, RING, 10, 1.0) == 780
    assert analytical_time(RS, 1000, 4, RING, 10, 1.0) == 780
    assert analytical_time(AR, 1000, 5, TREE, 10, 1.0) == 2060
    assert analytical_time(AR, 1000, 4, MESH, 10, 1.0, mesh_shape=(2, 2)) == 1540
    assert analytical_time(AR, 1000, 1, RING, 10, 1.0) == 0
    # traceio.py durations (pkg/tests/test_traceio.py:74-85)
    assert round_half_up_ns(132.5) == 133 and round_half_up_ns(0.49) == 0
    assert analytical_duration("mm", [[64, 64], [64, 64]], Dtype.F32, DEFAULT_DEVICE) == 524
    with pytest.raises(UnsupportedAlgoTopologyError):
        analytical_time(AG, 10, 4, TREE, 1, 1.0)
    with pytest.raises(UnsupportedAlgoTopologyError):
        analytical_time(AR, 10, 4, MESH, 1, 1.0, mesh_shape=(3, 3))


@pytest.mark.parametrize("kind,algo", list(itertools.product([AR, AG, RS], [RING, TREE, MESH])))
def test_host_costs_agree_with_oracle(kind, algo):
    for n, size, alpha, bw in itertools.product([1, 2, 3, 4, 6, 64, 1024, 8192], [0, 1, 999, 1 << 33],
                                                [0, 7, 2000], [1e9, 3.3e10, 1.8e12]):
        rows, cols = (2, n // 2) if n % 2 == 0 else (1, n)
        try:
            want = O.analytical_time(kind.value, size, n, algo.value, alpha, 1e9 / bw, rows, cols)
        except O.OracleError:
            want = "err"
        try:
            got = analytical_time(kind, size, n, algo, alpha, 1e9 / bw, mesh_shape=(rows, cols))
        except UnsupportedAlgoTopologyError:
            got = "err"
        assert got == want
