"""Pins for oracle.linear / split_linear.

Each test ties the oracle to something other than itself: numpy float64
matmul (a library routine), closed forms (identity, permutation, zero weight),
exact integer arithmetic, or brute force over every split.
"""
import itertools

import numpy as np
import pytest

import oracle
from harness import gen


def _rand(B, N, K, seed=3, integer=0, bias=True):
    return gen.linear_inputs(seed, 0, "fc1", B, N, K, bias=bias, integer=integer)


@pytest.mark.parametrize("B,N,K", [(1, 3072, 768), (8, 64, 1000), (3, 130, 257), (2, 1, 1)])
def test_matches_numpy_float64_matmul(B, N, K):
    x, W, b = _rand(B, N, K)
    y = oracle.linear(x, W, b)
    ref = oracle.linear_np(x, W, b)
    # fp64 summation-order difference only: bound ~ K * eps * sum|x w|
    assert np.allclose(y, ref, rtol=0, atol=1e-12 * max(1, K))


def test_transpose_would_fail():
    """A transposed W (a plausible mistake) is caught by the numpy pin."""
    x, W, _ = _rand(2, 48, 48, bias=False)
    y = oracle.linear(x, W)
    wrong = oracle.bf16_to_f64(x) @ oracle.bf16_to_f64(W)
    assert not np.allclose(y, wrong, atol=1e-6)


def test_small_integer_inputs_exact():
    """|x|,|w| <= 16 and K <= 256: every partial sum is an exact integer."""
    x, W, b = _rand(4, 96, 256, integer=16)
    y = oracle.linear(x, W, b)
    xi = oracle.bf16_to_f64(x).astype(np.int64)
    Wi = oracle.bf16_to_f64(W).astype(np.int64)
    bi = b.astype(np.int64)
    exact = np.array([[sum(int(xi[r, k]) * int(Wi[n, k]) for k in range(256)) + int(bi[n])
                       for n in range(96)] for r in range(4)], dtype=np.float64)
    assert np.array_equal(y, exact)


def test_identity_weight_returns_x():
    K = 256
    x, _, _ = _rand(3, K, K, bias=False)
    eye = np.zeros((K, K), dtype=np.uint16)
    eye[np.arange(K), np.arange(K)] = 0x3F80  # bf16 1.0
    y = oracle.linear(x, eye)
    assert np.array_equal(y, oracle.bf16_to_f64(x))


def test_one_hot_permutation():
    K, N = 200, 150
    rng = np.random.default_rng(0)
    perm = rng.integers(0, K, size=N)
    x, _, _ = _rand(2, N, K, bias=False)
    W = np.zeros((N, K), dtype=np.uint16)
    W[np.arange(N), perm] = 0x3F80
    y = oracle.linear(x, W)
    assert np.array_equal(y, oracle.bf16_to_f64(x)[:, perm])


def test_zero_weight_gives_bias():
    x, W, b = _rand(2, 64, 128)
    W[:] = 0
    y = oracle.linear(x, W, b)
    assert np.array_equal(y, np.broadcast_to(b.astype(np.float64), y.shape))


def test_rows_and_threads_do_not_change_bits():
    x, W, b = _rand(5, 333, 321)
    y1 = oracle.linear(x, W, b, nthreads=1)
    y4 = oracle.linear(x, W, b, nthreads=4)
    assert np.array_equal(y1, y4)
    rows = np.array([0, 7, 332, 100, 100])
    ys = oracle.linear_rows(x, W, rows, b, nthreads=3)
    assert np.array_equal(ys, y1[:, rows])


def test_split_invariance_brute_force_tiny():
    """c2.2 + c4: every (n_res, n_str) with G=1 on a tiny matrix is bit-identical."""
    N, K = 9, 13
    x, W, b = _rand(2, N, K, seed=17)
    y = oracle.linear(x, W, b)
    for n_res in range(N + 1):
        for n_str in range(N - n_res + 1):
            assert np.array_equal(oracle.split_linear(x, W, b, n_res, n_str), y)


def test_alpha_extremes_reduce_to_single_lane():
    """alpha=0 -> all host rows on the CPU lane; alpha=1 -> all streamed (c4 special cases)."""
    N, K = 512, 64
    x, W, b = _rand(1, N, K)
    for a, expect in ((0.0, (0, 0, N)), (1.0, (0, N, 0))):
        assert oracle.partition(N, 0, a, 128) == expect
        n_res, n_str, _ = expect
        assert np.array_equal(oracle.split_linear(x, W, b, n_res, n_str), oracle.linear(x, W, b))


def test_gather_shards_is_global_column_order():
    B, N, K, P = 3, 512, 64, 4
    x, W, b = _rand(B, N, K)
    y = oracle.linear(x, W, b)
    shards = []
    for p in range(P):
        r0, r1 = oracle.shard(N, P, p, 128)
        shards.append(oracle.linear(x, W[r0:r1], b[r0:r1]))
    assert np.array_equal(oracle.gather_shards(shards, B), y)


def test_tolerance_definition():
    ok, worst = oracle.within_tol([1.0, 200.0], [1.0099, 201.9])
    assert ok and worst < 1
    ok, _ = oracle.within_tol([0.0], [0.0101])
    assert not ok
