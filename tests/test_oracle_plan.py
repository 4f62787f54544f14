"""Pins for the oracle's cost model (Eqs. 4-9) and integer partition.

Pins: exact rationals solving Eq. (4) directly (fractions.Fraction), the worked
values in tests/golden/alpha_closed_forms.txt, algebraic identities the paper
states (the two forms of Eq. 5, T' = W/V turning Eq. 7 into Eq. 6), limits, and
brute-force properties of the partition.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "alpha_closed_forms.txt")


def _golden():
    rows = []
    for line in open(GOLDEN):
        line = line.split("#")[0].strip()
        if line:
            m, vc, vg, vm, num, den = line.split()
            rows.append((m, float(vc), float(vg), float(vm), Fraction(int(num), int(den))))
    return rows


@pytest.mark.parametrize("row", _golden())
def test_golden_closed_forms(row):
    mode, vc, vg, vm, exact = row
    a = oracle.alpha_eq5(vc, vg, vm) if mode == "exact" else oracle.alpha_eq6(vc, vm)
    assert abs(a - float(exact)) <= 2e-16 * float(exact) * 4


def test_eq5_solves_eq4_in_exact_rationals():
    """Eq. (5) is the solution of Eq. (4): check with Fractions on random integer rates."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        vc, vg, vm = (Fraction(int(v)) for v in rng.integers(1, 10**6, size=3))
        a = 1 / (vc / vm + vc / vg + 1)            # Eq. (5) second form, exact
        W = Fraction(1)
        assert (1 - a) * W / vc == a * W / vg + a * W / vm      # Eq. (4) exactly
        a_first = vg * vm / (vc * vg + vc * vm + vm * vg)      # Eq. (5) first form, exact
        assert a == a_first
        # the float oracle agrees with the exact value
        af = oracle.alpha_eq5(float(vc), float(vg), float(vm))
        assert abs(af - float(a)) <= 4e-16


def test_two_forms_of_eq5_agree_in_float():
    rng = np.random.default_rng(2)
    for vc, vg, vm in 10.0 ** rng.uniform(6, 13, size=(500, 3)):
        a1 = oracle.alpha_eq5(vc, vg, vm)
        a2 = oracle.alpha_eq5_first_form(vc, vg, vm)
        assert abs(a1 - a2) <= 1e-15 * a1 * 4


def test_alpha_properties():
    rng = np.random.default_rng(3)
    for vc, vg, vm in 10.0 ** rng.uniform(6, 13, size=(1000, 3)):
        a = oracle.alpha_eq5(vc, vg, vm)
        assert 0.0 < a < 1.0
        # scale invariance (dimensionless)
        assert abs(oracle.alpha_eq5(7 * vc, 7 * vg, 7 * vm) - a) <= 1e-15
        # faster CPU -> smaller alpha; faster link -> larger alpha
        assert oracle.alpha_eq5(2 * vc, vg, vm) < a
        assert oracle.alpha_eq5(vc, vg, 2 * vm) > a
        # dropping the GPU term (Eq. 6) removes a positive denominator term
        assert oracle.alpha_eq5(vc, vg, vm) < oracle.alpha_eq6(vc, vm)


def test_limits():
    assert oracle.alpha_eq5(1e30, 1e12, 5e10) < 1e-15           # infinitely fast CPU -> 0
    assert oracle.alpha_eq5(1e11, math.inf, math.inf) == 1.0      # free link + GPU -> 1
    assert oracle.alpha_eq5(1e11, math.inf, 1e11) == 0.5


def test_eq7_with_whole_times_equals_eq6():
    """V -> 1/T' ; with T'_X = W/V_X Eq. (7) is Eq. (6)."""
    rng = np.random.default_rng(4)
    for vc, vm, W in zip(*(10.0 ** rng.uniform(6, 12, size=(3, 300)))):
        assert abs(oracle.alpha_eq7(W / vc, W / vm) - oracle.alpha_eq6(vc, vm)) <= 1e-15


def test_eq9_reduces():
    """pinning free (pre-pinned weights, reading R7) -> Eq. (7); pin-bound -> pin lane."""
    assert oracle.alpha_eq9(3.0, 0.0, 1.0) == oracle.alpha_eq7(3.0, 1.0) == 0.75
    assert oracle.alpha_eq9(3.0, 2.0, 1.0) == oracle.alpha_eq7(3.0, 2.0) == 0.6


def test_balanced_time_illustrative():
    """c2.4 worked value: W = 411,041,792 B (OPT-30B fc1), Vm=55 GB/s, Vc=100 GB/s, Vg=6.5 TB/s."""
    W, vc, vg, vm = 411_041_792.0, 100e9, 6.5e12, 55e9
    a = oracle.alpha_eq5(vc, vg, vm)
    assert abs(a - 715 / 2026) < 1e-15 and round(a, 5) == 0.35291
    T = oracle.balanced_time(W, vc, vg, vm)
    assert abs(T - (1 - a) * W / vc) <= 1e-15 * T * 8            # CPU lane time at alpha
    assert abs(T - (a * W / vg + a * W / vm)) <= 1e-15 * T * 8    # GPU + transfer lane
    assert round(T * 1e3, 3) == 2.660


# ---------------------------------------------------------------- partition
def test_partition_dyadic_alpha_matches_exact_round_half_up():
    """alpha = i/64 makes alpha*m exact: n_str/G must be floor(alpha*m + 1/2) in rationals."""
    for N, G in ((3072, 128), (28672, 128), (40, 1), (64, 4)):
        for n_res in range(0, N + 1, max(G, N // 7 // G * G)):
            m = (N - n_res) // G
            prev = -1
            for i in range(65):
                a = i / 64
                r, s, c = oracle.partition(N, n_res, a, G)
                exact = math.floor(Fraction(i, 64) * m + Fraction(1, 2))
                assert (r, s, c) == (n_res, G * exact, N - n_res - G * exact)
                assert s >= prev
                prev = s


def test_partition_random_alpha_nearest_granule():
    rng = np.random.default_rng(5)
    for _ in range(3000):
        G = int(rng.choice([1, 2, 8, 128]))
        N = G * int(rng.integers(1, 400))
        n_res = G * int(rng.integers(0, N // G + 1))
        a = float(rng.random())
        r, s, c = oracle.partition(N, n_res, a, G)
        m = (N - n_res) // G
        assert r + s + c == N and s % G == 0 and c % G == 0 and s >= 0 and c >= 0
        assert abs(s / G - a * m) <= 0.5 + 1e-9


def test_partition_rejects_bad_input():
    for args in ((100, 0, 0.5, 128), (256, 64, 0.5, 128), (256, 0, 1.5, 128), (256, 0, -0.1, 128),
                 (256, 384, 0.5, 128), (256, 0, float("nan"), 128)):
        with pytest.raises(ValueError):
            oracle.partition(*args)


def test_chunks_cover_and_respect_size():
    for K in (768, 4096, 7168, 28672, 49152):
        for cb in (1, 1 << 20, 8 << 20, 64 << 20):
            C = oracle.chunk_rows(K, 128, cb)
            assert C % 128 == 0 and C >= 128
            assert C == 128 or C * K * 2 <= cb
            assert (C + 128) * K * 2 > cb or C == 128 and 128 * K * 2 > cb or C * K * 2 <= cb
            for n_res, n_str in ((0, 0), (0, 128), (256, 28672 - 256), (128, 5 * C + 128)):
                ch = oracle.chunks(n_res, n_str, C)
                assert len(ch) == -(-n_str // C)
                pos = n_res
                for i, (a, b) in enumerate(ch):
                    assert a == pos and b > a and b - a <= C
                    if i < len(ch) - 1:
                        assert b - a == C
                    pos = b
                assert pos == n_res + n_str


def test_chunk_rows_known_values():
    """8 MiB target -> C=512 rows at K=7168, 128 rows at K=28672/49152."""
    assert oracle.chunk_rows(7168, 128, 8 << 20) == 512
    assert oracle.chunk_rows(28672, 128, 8 << 20) == 128
    assert oracle.chunk_rows(49152, 128, 8 << 20) == 128


def test_resident_rows_and_shards():
    assert oracle.resident_rows(0.1, 6144, 128) == 640      # SURVEY: C5 fc1 shard
    assert oracle.resident_rows(0.1, 1536, 128) == 128      # C5 fc2 shard
    assert oracle.resident_rows(0.5, 12288, 128) == 6144
    N, P = 28672, 8
    covered = []
    for p in range(P):
        a, b = oracle.shard(N, P, p, 128)
        assert b - a == N // P
        covered += list(range(a, b))
    assert covered == list(range(N))
    with pytest.raises(ValueError):
        oracle.shard(768, 8, 0, 128)


def test_alpha_sweep_values_c4():
    """OPT-30B fc1 (N=28672) alpha=0.1..1.0 -> n_str list."""
    got = [oracle.partition(28672, 0, i / 10, 128)[1] for i in range(1, 11)]
    assert got == [2816, 5760, 8576, 11520, 14336, 17152, 20096, 22912, 25856, 28672]
    assert oracle.partition(3072, 0, 0.5, 128) == (0, 1536, 1536)


def test_plan_fields():
    rates = dict(v_cpu=100e9, v_gpu=6.5e12, v_link=55e9, v_pin=math.inf,
                 b_hbm=6.5e12, b_link=55e9, b_cpu=100e9)
    N, K = 28672, 7168
    p = oracle.plan(rates, N, K, 1, 0, oracle.EXACT, 0.0, 128, 8 << 20)
    assert p["n_res"] + p["n_str"] + p["n_cpu"] == N
    assert p["alpha_req"] == oracle.alpha_eq5(100e9, 6.5e12, 55e9)
    assert p["n_str"] == oracle.partition(N, 0, p["alpha_req"], 128)[1]
    assert p["n_chunks"] == -(-p["n_str"] // p["chunk_rows"])
    row = 2 * K
    assert p["t_cpu"] == row * p["n_cpu"] / 100e9
    assert p["t_roof"] == max(p["t_hbm"], row * p["n_str"] / 55e9, row * p["n_cpu"] / 100e9)
    # near balance the pipelined prediction is close to the closed-form optimum
    T = oracle.balanced_time(2.0 * K * N, 100e9, 6.5e12, 55e9)
    assert abs(p["t_eq4"] - T) / T < 0.01
    # alpha = 0 with r = 0: everything on the CPU lane; roofline = host bytes / b_cpu
    p0 = oracle.plan(rates, N, K, 1, 0, oracle.FIXED, 0.0, 128, 8 << 20)
    assert p0["n_str"] == 0 and p0["n_chunks"] == 0 and p0["t_roof"] == 2.0 * K * N / 100e9
    # fully resident: alpha irrelevant, roofline = HBM read of W once
    pr = oracle.plan(rates, N, K, 1, N, oracle.EXACT, 0.0, 128, 8 << 20)
    assert pr["n_str"] == pr["n_cpu"] == 0 and pr["alpha_eff"] == 0.0
    assert pr["t_roof"] == 2.0 * K * N / 6.5e12
    # async mode with pre-pinned weights (v_pin = inf) equals Eq. (7)
    pa = oracle.plan(rates, N, K, 1, 0, oracle.ASYNC, 0.0, 128, 8 << 20)
    pt = oracle.plan(rates, N, K, 1, 0, oracle.TPRIME, 0.0, 128, 8 << 20)
    assert pa["alpha_req"] == pt["alpha_req"]
