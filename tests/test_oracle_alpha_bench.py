"""Pins for the oracle's alpha-benchmark refinement.

Pins: analytic roots of linear lane models (F_CPU = (1-a)c, F_COM = a k -> c/(c+k),
the closed form of Eq. (4) with the GPU term dropped), recovery of Eq. (5)'s alpha
from noiseless analytic samples, the pin lane dominating, identical curves, and
the clamp when no root lies in the window (SPEC S:161-163, S:172-174 examples).
"""
import math

import numpy as np
import pytest

import oracle


def test_window_sampling():
    pts = oracle.alpha_window(0.3, 0.1, 0.02)
    assert len(pts) == 11 and abs(pts[0] - 0.2) < 1e-15 and abs(pts[-1] - 0.4) < 1e-12
    assert oracle.alpha_window(0.05, 0.1, 0.02)[0] == 0.0      # clipped at 0
    assert oracle.alpha_window(0.97, 0.1, 0.02)[-1] == 1.0     # clipped at 1


def test_linear_lanes_root_is_c_over_c_plus_k():
    """F_CPU=(1-a)*3, F_COM=a*1, seed 0.7, gamma 0.2 -> a = 0.75."""
    a = oracle.alpha_window(0.7, 0.2, 0.02)
    tc = [(1 - x) * 3.0 for x in a]
    tm = [x * 1.0 for x in a]
    for deg in (1, 2, 3):
        ab, clamped = oracle.alpha_bench_solve(a, tc, tm, deg, a[0], a[-1], 0.7)
        assert not clamped and abs(ab - 0.75) < 1e-9


def test_recovers_eq4_balance_from_analytic_samples():
    """Analytic lane times of Eq. (4): t_cpu=(1-a)W/Vc, t_com=aW/Vg+aW/Vm -> root = Eq. (5)."""
    W, vc, vg, vm = 411e6, 170e9, 5e12, 55e9
    seed = oracle.alpha_eq6(vc, vm)
    a = oracle.alpha_window(seed, 0.1, 0.02)
    tc = [(1 - x) * W / vc for x in a]
    tm = [x * W / vg + x * W / vm for x in a]
    ab, clamped = oracle.alpha_bench_solve(a, tc, tm, 2, a[0], a[-1], seed)
    assert not clamped and abs(ab - oracle.alpha_eq5(vc, vg, vm)) < 1e-9


def test_quadratic_lane_model():
    """Mildly nonlinear lanes: the fitted quadratics reproduce the exact root."""
    a = oracle.alpha_window(0.4, 0.1, 0.01)
    tc = [2.0 - 2.5 * x + 0.5 * x * x for x in a]
    tm = [0.2 + 2.0 * x + 0.3 * x * x for x in a]
    ab, clamped = oracle.alpha_bench_solve(a, tc, tm, 2, a[0], a[-1], 0.4)
    # 0.2 x^2 - 4.5 x + 1.8 = 0
    root = (4.5 - math.sqrt(4.5 ** 2 - 4 * 0.2 * 1.8)) / (2 * 0.2)
    assert not clamped and abs(ab - root) < 1e-9


def test_pin_lane_dominates():
    """F_COM = max(F_PIN, F_TRANS): a pin lane above the transfer lane moves the root."""
    a = oracle.alpha_window(0.5, 0.2, 0.02)
    tc = [(1 - x) * 2.0 for x in a]
    tt = [x * 1.0 for x in a]
    tp = [x * 2.0 for x in a]
    ab, _ = oracle.alpha_bench_solve(a, tc, tt, 1, a[0], a[-1], 0.5, t_pin=tp)
    assert abs(ab - 0.5) < 1e-9                        # (1-a)2 = 2a
    ab2, _ = oracle.alpha_bench_solve(a, tc, tt, 1, a[0], a[-1], 0.5)
    assert abs(ab2 - 2.0 / 3.0) < 1e-9                 # (1-a)2 = a


def test_identical_curves_return_seed_and_no_root_clamps():
    a = oracle.alpha_window(0.3, 0.1, 0.02)
    t = [1.0 + x for x in a]
    assert oracle.alpha_bench_solve(a, t, t, 1, a[0], a[-1], 0.3) == (0.3, False)
    tc = [5.0 - x for x in a]                          # CPU slower everywhere in the window
    tm = [x for x in a]
    ab, clamped = oracle.alpha_bench_solve(a, tc, tm, 1, a[0], a[-1], 0.3)
    assert clamped and ab == a[-1]


def test_noisy_samples_stay_near_truth():
    rng = np.random.default_rng(0)
    a = oracle.alpha_window(0.25, 0.1, 0.02)
    tc = [(1 - x) * 4.0 * (1 + 0.002 * rng.standard_normal()) for x in a]
    tm = [x * 12.0 * (1 + 0.002 * rng.standard_normal()) for x in a]
    ab, clamped = oracle.alpha_bench_solve(a, tc, tm, 2, a[0], a[-1], 0.25)
    assert not clamped and abs(ab - 0.25) < 0.01
