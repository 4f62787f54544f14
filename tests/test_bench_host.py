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


def test_percentile_matches_numpy_linear():
    import numpy as np
    rng = np.random.default_rng(3)
    for n in (1, 2, 7, 20, 64):
        v = sorted(rng.standard_normal(n).tolist())
        for q in (0, 10, 50, 90, 100):
            assert abs(bench.pct(v, q) - float(np.percentile(v, q))) <= 1e-12


def test_reference_arm_small_sample_runs():
    """--impl reference on a cut-down model (OPT-6.7B shapes, one layer per step): one JSON line with the
    oracle's timing; ms_per_step is the step's own time, value the per-token scaling."""
    import json
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--model", "opt-6.7b", "--steps", "1",
                        "--warmup", "3", "--ref-layers", "1"], capture_output=True, text=True, cwd=root, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["unit"] == "ms/token" and d["cpu_baseline"]["kind"] == "oracle"
    assert abs(d["value"] - d["ms_per_step"] * 32) <= 0.1 * 32 + 1e-6
