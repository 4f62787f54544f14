"""Pins of oracle.schedule, the heterogeneous module scheduler (Sec. 4.5), and parity
of the library's hg_schedule with it (pure host function: no GPU needed)."""
import random
from fractions import Fraction

import pytest

import oracle
from paper_2403_01164_b200 import hg

G = 128


def test_zero_budget_places_nothing():
    mods = [(256, 64, 1.0), (512, 128, 3.0)]
    assert oracle.schedule(mods, 0, G) == ([0, 0], 0)


def test_budget_covering_everything_places_everything():
    mods = [(256, 64, 1.0), (512, 128, 3.0), (128, 8, 0.1)]
    total = sum(2 * n * k for n, k, _ in mods)
    for partial in (True, False):
        assert oracle.schedule(mods, total, G, partial) == ([256, 512, 128], total)
        assert oracle.schedule(mods, total + 12345, G, partial) == ([256, 512, 128], total)


def test_gain_is_time_per_byte_not_time_or_time_per_row():
    """Three modules ranked differently by t, by t/N and by t/(N*K) (Eq. 13): only the last
    ranking is the paper's.  A: t=4 over 2*256*512 B (g=1/65536); B: t=3 over 2*256*64 B
    (g=3/32768, best); C: t=2 over 2*128*32 B (g=1/4096 ... highest).  Worked by hand:
    order C, B, A; budget = C + B + 10 rows of A."""
    A, B, C = (256, 512, 4.0), (256, 64, 3.0), (128, 32, 2.0)
    bytes_ = [2 * n * k for n, k, _ in (A, B, C)]
    budget = bytes_[2] + bytes_[1] + 2 * 512 * 130  # 130 rows of A -> 128 after the granule floor
    n_res, used = oracle.schedule([A, B, C], budget, G, True)
    assert n_res == [128, 256, 128]
    assert used == bytes_[2] + bytes_[1] + 2 * 512 * 128
    # without partial placement A is passed over
    assert oracle.schedule([A, B, C], budget, G, False) == ([0, 256, 128], bytes_[2] + bytes_[1])


def test_skip_then_smaller_module_fits():
    """Greedy order is by gain; a module that does not fit is passed over and a later, smaller
    one with lower gain still gets placed (allow_partial=False)."""
    big, small = (1024, 1024, 10.0), (128, 64, 0.01)  # g(big)=10/2^21 > g(small)=0.01/2^14
    assert Fraction(10.0) / (2 * 1024 * 1024) > Fraction(0.01) / (2 * 128 * 64)
    n_res, used = oracle.schedule([big, small], 2 * 128 * 64, G, False)
    assert n_res == [0, 128] and used == 2 * 128 * 64


def test_equal_gains_fill_in_index_order():
    """t proportional to bytes (one CPU rate for every module): all gains equal, so modules are
    placed in index order -- layer by layer, as P:288 describes."""
    mods = [(256 * (1 + i % 3), 64 * (1 + i % 2), 1e-9 * 2 * 256 * (1 + i % 3) * 64 * (1 + i % 2))
            for i in range(12)]
    gains = {Fraction(t) / (2 * n * k) for n, k, t in mods}
    budget = sum(2 * n * k for n, k, _ in mods[:5]) + 2 * mods[5][1] * 128
    n_res, _ = oracle.schedule(mods, budget, G, True)
    if len(gains) == 1:
        assert n_res[:5] == [m[0] for m in mods[:5]] and n_res[5] == 128 and n_res[6:] == [0] * 6


def test_invariants_random():
    rng = random.Random(3)
    for _ in range(300):
        mods = [(G * rng.randint(0, 8), 8 * rng.randint(1, 64), rng.random()) for _ in range(rng.randint(1, 9))]
        budget = rng.randint(0, sum(2 * n * k for n, k, _ in mods) + 10)
        for partial in (True, False):
            n_res, used = oracle.schedule(mods, budget, G, partial)
            assert used == sum(2 * r * k for r, (n, k, _) in zip(n_res, mods)) <= budget
            assert all(r % G == 0 and 0 <= r <= n for r, (n, _, _) in zip(n_res, mods))
            if not partial:
                assert all(r in (0, n) for r, (n, _, _) in zip(n_res, mods))
            partial_mods = [i for i, (r, (n, _, _)) in enumerate(zip(n_res, mods)) if 0 < r < n]
            assert len(partial_mods) <= (1 if partial else 0)


@pytest.mark.parametrize("seed", range(4))
def test_hg_schedule_equals_oracle(seed):
    rng = random.Random(100 + seed)
    for _ in range(250):
        n = rng.randint(0, 12)
        mods = []
        for _ in range(n):
            N, K = G * rng.randint(0, 20), 8 * rng.randint(1, 4000)
            t = rng.choice([rng.random() * 1e-3, 2 * N * K * 1e-11, 0.0])
            mods.append((N, K, t))
        total = sum(2 * a * b for a, b, _ in mods)
        budget = rng.choice([0, total, total + 1, rng.randint(0, total + 1)])
        for partial in (True, False):
            assert hg.hg_schedule(mods, budget, G, partial) == oracle.schedule(mods, budget, G, partial)


def test_hg_schedule_errors():
    with pytest.raises(hg.HgError):
        hg.hg_schedule([(100, 64, 1.0)], 1 << 20, G)  # N % G
    with pytest.raises(hg.HgError):
        hg.hg_schedule([(128, 64, -1.0)], 1 << 20, G)
    with pytest.raises(hg.HgError):
        hg.hg_schedule([(128, 64, 1.0)], -1, G)


# ---------------------------------------------------------------------------------------------
# Row-granular variant (reading R31): one resident fraction r for every module
# ---------------------------------------------------------------------------------------------
def test_schedule_rows_hand_worked():
    """Two modules (N, K) = (256, 8), (512, 8), G = 128: m = 2 and 4 granules, 2 K G = 2048 B per
    granule.  Budget 4096 B -> at most 2 granules: r = 0.25 gives floor(0.5 + 0.5) = 1 and
    floor(1.0 + 0.5) = 1 granule (feasible); the next change point is r = 0.375 where the second
    module reaches floor(1.5 + 0.5) = 2 (3 granules, infeasible) -> (128, 128), 4096 B used."""
    mods = [(256, 8, 1.0), (512, 8, 5.0)]
    assert oracle.schedule_rows(mods, 4096, 128) == ([128, 128], 4096)
    # budget 2047 B: not even one granule -> nothing; the whole weight -> everything
    assert oracle.schedule_rows(mods, 2047, 128) == ([0, 0], 0)
    assert oracle.schedule_rows(mods, 2 * 8 * 768, 128) == ([256, 512], 2 * 8 * 768)
    # 3 granules: r = 0.375 -> (1, 2) granules
    assert oracle.schedule_rows(mods, 3 * 2048, 128) == ([128, 256], 3 * 2048)


def test_schedule_rows_brute_force():
    """Against a brute-force scan of r on a fine grid plus every candidate's neighbours: no r in
    [0, 1] with a feasible vector beats the returned one (component-wise it is the maximum)."""
    rng = random.Random(9)
    for _ in range(60):
        G = rng.choice([1, 2, 4])
        mods = [(G * rng.randint(0, 12), rng.randint(1, 9), 1.0) for _ in range(rng.randint(1, 5))]
        total = sum(2 * K * N for N, K, _ in mods)
        budget = rng.randint(0, total + 5)
        got, used = oracle.schedule_rows(mods, budget, G)
        assert used <= budget
        for i in range(2001):
            r = i / 2000
            v = [oracle.resident_rows(r, N, G) for N, _, _ in mods]
            if sum(2 * K * n for (N, K, _), n in zip(mods, v)) <= budget:
                assert all(a <= b for a, b in zip(v, got)), (mods, budget, r, v, got)


def test_hg_schedule_rows_matches_oracle_exactly():
    rng = random.Random(19)
    for _ in range(300):
        G = rng.choice([1, 8, 128])
        mods = [(G * rng.randint(0, 40), rng.choice([8, 64, 7168]), 0.0) for _ in range(rng.randint(0, 8))]
        total = sum(2 * K * N for N, K, _ in mods)
        budget = rng.randint(0, total + 100) if rng.random() < 0.9 else total
        assert hg.hg_schedule_rows(mods, budget, G) == oracle.schedule_rows(mods, budget, G), (mods, budget, G)
    for r in (0.0, 0.1, 0.25, 0.37, 0.5, 0.999, 1.0):
        for N in (0, 128, 640, 28672):
            assert hg.hg_resident_rows(r, N, 128) == oracle.resident_rows(r, N, 128)


def test_hg_module_tcpu_host_only():
    """T-bar_CPU on a host-only context: positive, and (1 - alpha) times the whole module."""
    import numpy as np
    from harness import gen
    N, K = 512, 256
    W = gen.uniform_bf16(3, 7, N * K, 0.1).reshape(N, K)
    with hg.Context(-1, cpu_threads=2) as c:
        t0, rate = c.hg_module_tcpu(W, N, K, 1, 0.0)
        assert t0 > 0 and rate > 0 and abs(t0 - 2 * N * K / rate) <= 1e-12 * t0
        t5, rate5 = c.hg_module_tcpu(W, N, K, 1, 0.5)
        assert abs(t5 - 0.5 * 2 * N * K / rate5) <= 1e-12 * t5
        with pytest.raises(hg.HgError):
            c.hg_module_tcpu(W, N, K, 1, 1.5)
