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


# ---------------------------------------------------------------------------------------------
# Hand-worked pins of plan()'s time fields.  Every number below is worked by
# hand in the comments, not recomputed with the oracle's formula.
# ---------------------------------------------------------------------------------------------
def _rates(**kw):
    r = dict(v_cpu=1.0, v_gpu=1.0, v_link=1.0, v_pin=math.inf, b_hbm=1.0, b_link=1.0, b_cpu=1.0)
    r.update(kw)
    return r


def test_plan_t_eq4_spec_hand_schedule():
    """S:447-448 hand schedule with the pin lane free (weights pre-pinned, reading R7): one module,
    t_cpu = 4, t_trans = 2, t_gpu = 0.1 -> period max(4, 2 + 0.1) = 4; with t_cpu = 2 -> 2.1.
    Realised as N = 256 rows of K = 8 (16 B per row), G = 128, alpha = 0.5 -> 128 streamed rows and
    128 CPU rows = 2048 B each: v_cpu = 2048/4 = 512 B/s, v_link = 2048/2 = 1024 B/s,
    v_gpu = 2048/0.1 = 20480 B/s."""
    p = oracle.plan(_rates(v_cpu=512.0, v_link=1024.0, v_gpu=20480.0), 256, 8, 1, 0, oracle.FIXED, 0.5, 128, 1)
    assert (p["n_str"], p["n_cpu"]) == (128, 128)
    assert p["t_cpu"] == 4.0 and p["t_link"] == 2.0
    assert abs(p["t_eq4"] - 4.0) <= 1e-12
    p = oracle.plan(_rates(v_cpu=1024.0, v_link=1024.0, v_gpu=20480.0), 256, 8, 1, 0, oracle.FIXED, 0.5, 128, 1)
    assert abs(p["t_eq4"] - 2.1) <= 1e-12


def test_plan_t_pred_and_t_hbm_hand_worked():
    """N = 1152 rows of K = 64 (row = 128 B), n_res = 128, alpha = 0.75, G = 128:
    m = (1152-128)/128 = 8, g_str = floor(0.75*8 + 0.5) = 6 -> n_str = 768, n_cpu = 256.
    chunk_bytes = 49152 -> C = 128*max(1, floor(49152/(128*64*2))) = 128*3 = 384 rows -> chunks
    [128, 512) and [512, 896): 2 chunks, the last of 384 rows.
    Rates: v_link = 98304 -> t_link = 768*128/98304 = 1.0; v_gpu = 491520 -> GEMV of the last chunk
    t_tail = 384*128/491520 = 0.1, GEMV of all GPU rows t_gpu = 896*128/491520 = 0.2333...;
    v_cpu = 32768 -> t_cpu = 256*128/32768 = 1.0.
    t_pred (pipelined) = max(1.0, 1.0 + 0.1, 0.2333) = 1.1.
    t_eq4 (serial, Eq. (4): streamed GEMV after the whole transfer) = max(1.0, 1.0 + 768*128/491520 = 1.2) = 1.2.
    t_hbm: resident 128*128 = 16384 B read once + streamed 768*128 = 98304 B written by the copy engine
    and read by the SMs = 196608 B -> 212992 B; b_hbm = 212992 -> t_hbm = 1.0 (without the doubling it
    would be 114688/212992 = 0.538).  t_roof = max(1.0, 98304/196608 = 0.5, 32768/65536 = 0.5) = 1.0."""
    r = _rates(v_cpu=32768.0, v_link=98304.0, v_gpu=491520.0, b_hbm=212992.0, b_link=196608.0, b_cpu=65536.0)
    p = oracle.plan(r, 1152, 64, 1, 128, oracle.FIXED, 0.75, 128, 49152)
    assert (p["n_res"], p["n_str"], p["n_cpu"], p["chunk_rows"], p["n_chunks"]) == (128, 768, 256, 384, 2)
    assert abs(p["t_pred"] - 1.1) <= 1e-12
    assert abs(p["t_eq4"] - 1.2) <= 1e-12
    assert abs(p["t_gpu"] - 896 * 128 / 491520) <= 1e-15 and abs(p["t_gpu"] - 0.23333333333333334) <= 1e-12
    assert p["t_hbm"] == 1.0 and p["t_roof"] == 1.0


def test_strategy_periods_spec_and_paper():
    """Fig. 5 strategies, steady-state period per module.  S:448: pinned-blocking
    3.1 vs hybrid 2.1 at t_cpu=2, t_pin=1, t_trans=2, t_gpu=0.1; hybrid 4 at t_cpu=4.  At
    t_cpu=4 the pinned-blocking period is 1 + max(4, 2.1) = 5 under P:225 ("the pinning memory
    blocks both communication and CPU computation"), not S:447's max(4, 3.1) = 4 (reading R27)."""
    per = oracle.strategy_period
    assert per("hybrid", 4, 1, 2, 0.1) == 4
    assert abs(per("hybrid", 2, 1, 2, 0.1) - 2.1) <= 1e-12
    assert abs(per("pinned_blocking", 2, 1, 2, 0.1) - 3.1) <= 1e-12
    assert per("pinned_blocking", 4, 1, 2, 0.1) == 5
    # naive (Fig. 5a): no pin lane, the transfer runs at the pageable rate (t_trans given as such)
    # beside the CPU lane, plus the activation hop on the CPU side
    assert abs(per("naive", 2, 0, 3, 0.1, t_act=0.05) - 3.1) <= 1e-12
    assert abs(per("naive", 4, 0, 3, 0.1, t_act=0.05) - 4.05) <= 1e-12
    # v_pin = inf (t_pin = 0): hybrid == pinned-blocking (S: compare_strategies, "pin free")
    assert per("hybrid", 3, 0, 2, 0.5) == per("pinned_blocking", 3, 0, 2, 0.5) == 3
    # ranking at equal lane times: hybrid <= pinned-blocking
    import random
    rnd = random.Random(5)
    for _ in range(1000):
        t = [rnd.uniform(0, 5) for _ in range(4)]
        assert per("hybrid", *t) <= per("pinned_blocking", *t)
    with pytest.raises(ValueError):
        per("other", 1, 1, 1, 1)
