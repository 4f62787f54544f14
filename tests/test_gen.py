"""Harness generator: the C and numpy implementations produce identical bits."""
import math

import numpy as np
import pytest

from harness import gen


@pytest.mark.parametrize("seed,tid,a", [(1164, 0, math.sqrt(3.0)), (1165, (3 << 8) | (2 << 4), 0.02),
                                        (0, 1, 0.1), (2**63 + 5, 2**40, 7.5)])
def test_c_matches_numpy_first_1e4(seed, tid, a):
    c = gen.uniform_bf16(seed, tid, 10_000, a)
    p = gen.uniform_bf16_np(seed, tid, 10_000, a)
    assert np.array_equal(c, p)


def test_int_mode_matches_and_range():
    c = gen.int_bf16(7, 9, 10_000, 16)
    p = gen.int_bf16_np(7, 9, 10_000, 16)
    assert np.array_equal(c, p)
    v = gen.bf16_bits_to_f32(c)
    assert v.min() == -16 and v.max() == 16 and np.all(v == np.round(v))


def test_offset_slices_are_consistent():
    full = gen.uniform_bf16(11, 3, 5000, 1.0)
    part = gen.uniform_bf16(11, 3, 1000, 1.0, offset=2500)
    assert np.array_equal(full[2500:3500], part)


def test_multithreaded_equals_single():
    n = (1 << 20) + 12345
    a = gen.uniform_bf16(5, 5, n, 1.0, nthreads=1)
    b = gen.uniform_bf16(5, 5, n, 1.0, nthreads=8)
    assert np.array_equal(a, b)


def test_scales_give_unit_variance():
    v = gen.bf16_bits_to_f32(gen.uniform_bf16(1, 2, 200_000, gen.X_SCALE)).astype(np.float64)
    assert abs(v.var() - 1.0) < 0.02 and abs(v.mean()) < 0.01
    K = 4096
    w = gen.bf16_bits_to_f32(gen.uniform_bf16(1, 3, 200_000, gen.w_scale(K))).astype(np.float64)
    assert abs(w.var() * K - 1.0) < 0.02


def test_bf16_roundtrip_rne():
    f = np.array([1.0, 1.0 + 2**-8, 1.0 + 3 * 2**-8, -2.5, 3.0e-3], dtype=np.float32)
    b = gen.f32_to_bf16_bits(f)
    back = gen.bf16_bits_to_f32(b)
    assert back[0] == 1.0 and back[1] == 1.0 and back[2] == 1.0 + 2**-6 and back[3] == -2.5
