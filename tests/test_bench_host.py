"""Host-side logic of bench.py that must agree with the oracle (no GPU): the resident-row rule of
`--resident` (C2) and the shard shapes used at N > 1."""
import os
import sys

import pytest

import oracle

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


@pytest.mark.parametrize("model", sorted(bench.MODELS))
@pytest.mark.parametrize("r", [0.0, 0.1, 0.25, 0.37, 0.5, 0.9, 1.0])
@pytest.mark.parametrize("world", [1, 2, 8])
def test_resident_rows_match_oracle(model, r, world):
    bench.set_model(model)
    for name in bench.NAMES:
        N = bench.SHAPES[name][0] // world
        if N % 128:
            continue
        assert bench.resident_rows(r, N) == oracle.resident_rows(r, N, 128), (name, N)


def test_c5_resident_rows_worked_values():
    """OPT-175B shard of 8 at r = 0.1 -> fc1 640 of 6144, fc2 128 of 1536."""
    assert bench.resident_rows(0.1, 49152 // 8) == 640
    assert bench.resident_rows(0.1, 12288 // 8) == 128
