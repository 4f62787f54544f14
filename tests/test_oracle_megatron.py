"""Pins for the oracle's Megatron pairing (reading R32).

Column-parallel QKV / fc1 and row-parallel O / fc2 compute the same layer as the unsharded one; only
the order of the fp64 sums changes.  Checked against: exact integer arithmetic (brute force on small
integer-valued operands, where every fp64 sum is exact whatever its order), numpy float64 matmul of the
unsharded operands, the unsharded oracle layer (itself pinned to torch float64 in test_oracle_layer),
and the index sets the sharding must produce.
"""
import numpy as np
import pytest

import oracle
from harness import gen


@pytest.mark.parametrize("H,P", [(1024, 8), (512, 4), (256, 2), (128, 1)])
def test_megatron_qkv_rows_partition_the_fused_weight(H, P):
    rows = [oracle.megatron_qkv_rows(H, P, p, 128) for p in range(P)]
    allr = np.concatenate(rows)
    assert np.array_equal(np.sort(allr), np.arange(3 * H))            # disjoint, complete
    for p, r in enumerate(rows):
        lo, hi = p * H // P, (p + 1) * H // P
        Hl = H // P
        assert np.array_equal(r[:Hl], np.arange(lo, hi))               # q of its heads
        assert np.array_equal(r[Hl:2 * Hl], H + np.arange(lo, hi))     # k
        assert np.array_equal(r[2 * Hl:], 2 * H + np.arange(lo, hi))   # v: feeds its O columns


def _int_bf16(rng, shape, lo, hi):
    """Small integers as bf16 bit patterns (exact)."""
    v = rng.integers(lo, hi, size=shape).astype(np.float64)
    return oracle.round_to_bf16(v), v


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_linear_rowpar_exact_on_integers(P):
    """Brute force: integer operands keep every fp64 partial and sum exact, so the row-parallel
    result equals Python-integer arithmetic exactly, bias included once."""
    rng = np.random.default_rng(P)
    B, N, Kp = 2, 5, 6
    K = Kp * P
    xb, xv = _int_bf16(rng, (B, K), -9, 10)
    Wb, Wv = _int_bf16(rng, (N, K), -9, 10)
    bias = rng.integers(-50, 50, size=N).astype(np.float64)
    parts_x = [xb[:, p * Kp:(p + 1) * Kp] for p in range(P)]
    parts_W = [np.ascontiguousarray(Wb[:, p * Kp:(p + 1) * Kp]) for p in range(P)]
    y = oracle.linear_rowpar(parts_x, parts_W, bias)
    for b in range(B):
        for n in range(N):
            exact = sum(int(xv[b, k]) * int(Wv[n, k]) for k in range(K)) + int(bias[n])
            assert y[b, n] == exact


@pytest.mark.parametrize("P", [2, 4, 8])
def test_linear_rowpar_equals_numpy_full_matmul(P):
    B, N, K = 3, 256, 1024
    x, W, b = gen.linear_inputs(5, 0, "fc2", B, N, K)
    ref = oracle.bf16_to_f64(x) @ oracle.bf16_to_f64(W).T + b
    parts = [oracle.shard_k(K, P, p, 128) for p in range(P)]
    y = oracle.linear_rowpar([x[:, a:c] for a, c in parts], [np.ascontiguousarray(W[:, a:c]) for a, c in parts], b)
    scale = oracle.bf16_to_f64(x).__abs__() @ oracle.bf16_to_f64(W).__abs__().T + np.abs(b)
    assert np.all(np.abs(y - ref) <= 1e-13 * scale)
    # a dropped or doubled shard, or the bias added per rank, moves it far outside that bound
    y_drop = oracle.linear_rowpar([x[:, a:c] for a, c in parts[1:]],
                                  [np.ascontiguousarray(W[:, a:c]) for a, c in parts[1:]], b)
    assert not np.all(np.abs(y_drop - ref) <= 1e-6 * scale)


def _layer_weights(seed, H, F):
    shapes = {"qkv": (3 * H, H), "o": (H, H), "fc1": (F, H), "fc2": (H, F)}
    Wd, bd = {}, {}
    for name, (N, K) in shapes.items():
        _, Wd[name], bd[name] = gen.linear_inputs(seed, 0, name, 1, N, K)
    return Wd, bd


def test_megatron_layer_p1_is_the_layer_bit_for_bit():
    H, F = 128, 512
    Wd, bd = _layer_weights(3, H, F)
    h = gen.uniform_bf16(4, 9, 2 * H, 1.0).reshape(2, H)
    full, mg = oracle.layer(h, Wd, bd, H), oracle.megatron_layer(h, Wd, bd, H, 1)
    for key in ("a", "y_qkv", "v", "y_o", "h1", "a2", "y_fc1", "u", "y_fc2", "out"):
        assert np.array_equal(full[key], mg[key]), key


@pytest.mark.parametrize("P", [2, 4, 8])
def test_megatron_layer_matches_the_unsharded_layer(P):
    """Same layer, sums regrouped: fp64 outputs agree to ~1e-13 relative, and every bf16 storage point
    (a, v, h1, a2, u, out) agrees except where an fp64 difference of that size straddles a rounding
    boundary (at most one bf16 ulp, in a vanishing fraction of elements)."""
    H, F, B = 1024, 4096, 2
    Wd, bd = _layer_weights(11, H, F)
    h = gen.uniform_bf16(12, 9, B * H, 1.0).reshape(B, H)
    full, mg = oracle.layer(h, Wd, bd, H), oracle.megatron_layer(h, Wd, bd, H, P)
    for key in ("y_qkv", "y_o", "y_fc1", "y_fc2"):
        assert np.allclose(mg[key], full[key], rtol=1e-12, atol=1e-12), key
    for key in ("a", "v", "h1", "a2", "u", "out"):
        a, b = oracle.bf16_to_f64(mg[key]), oracle.bf16_to_f64(full[key])
        diff = a != b
        assert diff.mean() < 1e-3, key
        if diff.any():
            assert np.all(np.abs(a - b)[diff] <= 2.0 ** -7 * np.maximum(np.abs(b[diff]), 2.0 ** -126)), key
    # the per-rank pieces are the column slices of the full tensors
    Hl = H // P
    for p in range(P):
        assert np.array_equal(mg["v_p"][p], full["v"][:, p * Hl:(p + 1) * Hl])
        r0, r1 = oracle.shard(F, P, p, 128)
        assert np.array_equal(mg["y_fc1_p"][p], full["y_fc1"][:, r0:r1])
