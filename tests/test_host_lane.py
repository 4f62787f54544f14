"""CPU lane through the C ABI on a host-only context: parity with
the fp64 oracle, exactness on small integers, every ISA path, ragged shapes."""
import os

import numpy as np
import pytest

import oracle
from harness import gen
from paper_2403_01164_b200 import hg

TOL_NOTE = "elementwise |y - y_ref| <= 1e-2 * max(1, |y_ref|) (BJ:5)"


@pytest.fixture(scope="module")
def ctx():
    c = hg.Context(-1, cpu_threads=4)
    yield c
    c.close()


def _run(ctx, B, N, K, seed=1, integer=0, bias=True):
    x, W, b = gen.linear_inputs(seed, 0, "fc1", B, N, K, bias=bias, integer=integer)
    y = np.full((B, N), np.nan, np.float32)
    ctx.hg_host_gemv(x, B, N, K, W, b, y)
    return x, W, b, y


@pytest.mark.parametrize("B", range(1, 9))
@pytest.mark.parametrize("N,K", [(1, 8), (37, 768), (130, 1000), (64, 4104)])
def test_parity(ctx, B, N, K):
    x, W, b, y = _run(ctx, B, N, K)
    ok, worst = oracle.within_tol(y, oracle.linear(x, W, b))
    assert ok, (TOL_NOTE, worst)


@pytest.mark.parametrize("B", [1, 4, 8])
def test_small_integers_bit_exact(ctx, B):
    x, W, b, y = _run(ctx, B, 96, 256, integer=16)
    assert np.array_equal(y.astype(np.float64), oracle.linear(x, W, b))


def test_no_bias_and_zero_rows(ctx):
    x, W, b, y = _run(ctx, 2, 50, 64, bias=False)
    assert oracle.within_tol(y, oracle.linear(x, W))[0]
    y0 = np.zeros((2, 0), np.float32)
    ctx.hg_host_gemv(x, 2, 0, 64, W, None, y0)


def test_deterministic_across_thread_counts():
    x, W, b = gen.linear_inputs(3, 0, "fc2", 3, 777, 1024)
    ys = []
    for t in (1, 3, 8):
        with hg.Context(-1, cpu_threads=t) as c:
            y = np.zeros((3, 777), np.float32)
            c.hg_host_gemv(x, 3, 777, 1024, W, b, y)
            ys.append(y)
    assert np.array_equal(ys[0], ys[1]) and np.array_equal(ys[0], ys[2])


@pytest.mark.parametrize("isa", ["avx2", "scalar"])
def test_fallback_isas(isa, monkeypatch):
    monkeypatch.setenv("HG_HOST_ISA", isa)
    assert hg.hg_host_isa() == isa
    with hg.Context(-1, cpu_threads=2) as c:
        for B in (1, 5):
            x, W, b = gen.linear_inputs(4, 0, "o", B, 70, 264)
            y = np.zeros((B, 70), np.float32)
            c.hg_host_gemv(x, B, 70, 264, W, b, y)
            assert oracle.within_tol(y, oracle.linear(x, W, b))[0]
            xi, Wi, bi = gen.linear_inputs(4, 0, "o", B, 70, 256, integer=16)
            c.hg_host_gemv(xi, B, 70, 256, Wi, bi, y[:, :70])
            assert np.array_equal(y.astype(np.float64), oracle.linear(xi, Wi, bi))


def test_bad_shapes(ctx):
    x = np.zeros((1, 12), np.uint16)
    W = np.zeros((4, 12), np.uint16)
    y = np.zeros((1, 4), np.float32)
    with pytest.raises(hg.HgError) as e:
        ctx.hg_host_gemv(x, 1, 4, 12, W, None, y)
    assert e.value.status == hg.HG_EALIGN
    with pytest.raises(hg.HgError) as e:
        ctx.hg_host_gemv(x, 9, 4, 8, W, None, y)
    assert e.value.status == hg.HG_EINVAL


@pytest.mark.parametrize("B", [4, 8])
def test_amx_lane_matches_oracle(B, monkeypatch):
    """Batches >= 4 use AMX tiles when the host has them (HG_AMX_MIN_BATCH); rows not a multiple of
    16 fall back to AVX-512 for the tail.  Tolerance parity with the fp64 oracle either way."""
    monkeypatch.setenv("HG_AMX_MIN_BATCH", "4")
    x, W, b = gen.linear_inputs(44, 0, "fc1", B, 1000, 4096)
    y = np.zeros((B, 1000), np.float32)
    with hg.Context(-1, cpu_threads=3) as c:
        c.hg_host_gemv(x, B, 1000, 4096, W, b, y)
    ok, worst = oracle.within_tol(y, oracle.linear(x, W, b))
    assert ok, worst
