"""Oracle pins for the opportunistic evaluator trigger sweep (P:218-235,
Eq. 8; reading L19): closed-form trigger times on
constant, periodic and sinusoidal carbon-intensity traces."""
import math

import numpy as np
import pytest

import oracle


def sweep(k2, kmax, dt=1.0, betas=(0.028,), thetas=(0.5,), grace=6.0, F=3, e=1.0, pue=1.0):
    k2 = np.asarray(k2, float)
    R = 1 if k2.ndim == 1 else k2.shape[0]
    T = k2.shape[-1]
    return oracle.evaluator_sweep(k2.ravel(), np.atleast_1d(np.asarray(kmax, float)), T, dt, betas, thetas,
                                  grace, F, e, pue)


def test_eq8_factor_halves_in_a_day():
    # beta = 0.028 "halves the urgency-adjusted carbon intensity ... after a 24-hour lapse";
    # S:337-338 (48 h factor 0.2608, SURVEY erratum): the iterated factor d^n equals e^{-beta n dt}
    d = math.exp(-0.028)
    f = 1.0
    for _ in range(24):
        f = f * d
    assert f == pytest.approx(math.exp(-0.028 * 24), rel=1e-13)
    assert f == pytest.approx(0.51075, abs=1e-3)
    for _ in range(24):
        f = f * d
    assert f == pytest.approx(0.260800, abs=1e-5)


def test_constant_intensity_fallback_fires_every_19_hours():
    """k2 = 400 constant, historical max 500, threshold 50%, beta 0.028/h, grace 6 h,
    fallback F = 3 (S:347's example, corrected in SURVEY 4): k' = 400 e^{-0.028 t} < 250
    first at t = 17 h (t > ln(1.6)/0.028 = 16.79), then two more samples: fire at 19 h, and
    the same again after every evaluation.  With no fallback a strictly decreasing k' never
    has a local minimum, so nothing fires (why Fig. 4(b) needs the fallback)."""
    T = 100
    o = sweep(np.full(T, 400.0), 500.0, e=0.25, pue=1.2)[0, 0, 0]
    fires = [19, 38, 57, 76, 95]
    assert o[0] == len(fires)
    assert o[1] == pytest.approx(len(fires) * 400 * 1.2 * 0.25, rel=1e-15)
    assert o[2] == 19.0 and o[3] == 400.0 * len(fires)
    o = sweep(np.full(T, 400.0), 500.0, F=0)[0, 0, 0]
    assert o[0] == 0 and o[2] == T


def test_grace_period_makes_it_periodic():
    # threshold never binding, F = 1: fire at the first sample once the grace period has elapsed
    for grace, dt, period in ((6.0, 1.0, 6), (5.5, 1.0, 6), (2.0, 1.0 / 12, 24), (0.0, 1.0, 1)):
        T = 200
        o = sweep(np.full(T, 100.0), 100.0, dt=dt, thetas=(10.0,), grace=grace, F=1)[0, 0, 0]
        assert o[0] == (T - 1) // period
        assert o[2] == pytest.approx(max(period, T - period * ((T - 1) // period)) * dt)


def test_local_minimum_fires_the_sample_after_each_trough():
    # beta = 0 (k' = k2), diurnal sinusoid with troughs at 18 + 24m: fire at 19 + 24m
    T = 24 * 5
    t = np.arange(T)
    k2 = 300.0 + 200.0 * np.sin(2 * np.pi * t / 24)
    o = sweep(k2, 500.0, betas=(0.0,), thetas=(1.0,), grace=12.0, F=0)[0, 0, 0]
    fires = [19 + 24 * m for m in range(5)]
    assert o[0] == len(fires)
    assert o[3] == pytest.approx(sum(k2[f] for f in fires), rel=1e-15)
    assert o[2] == 24.0
    # a 30 h grace period: 19 is too early (trace start = last evaluation), then 43 fires,
    # 67 is 24 h later (too early), 91 fires, 115 too early -> gaps 43, 48, 29
    o = sweep(k2, 500.0, betas=(0.0,), thetas=(1.0,), grace=30.0, F=0)[0, 0, 0]
    assert o[0] == 2 and o[2] == 48.0 and o[3] == pytest.approx(k2[43] + k2[91], rel=1e-15)


def test_threshold_below_the_trace_never_fires():
    T = 500
    k2 = np.linspace(200.0, 400.0, T)
    o = sweep(k2, 400.0, betas=(0.0,), thetas=(0.4,), grace=1.0, F=1)[0, 0, 0]
    assert o[0] == 0 and o[1] == 0 and o[2] == T


def test_configs_are_independent():
    rng = np.random.default_rng(3)
    k2 = rng.uniform(50, 500, size=(3, 400))
    kmax = k2.max(axis=1)
    betas, thetas = (0.0, 0.01, 0.028, 0.1), (0.3, 0.5, 0.8)
    full = sweep(k2, kmax, betas=betas, thetas=thetas)
    for r in range(3):
        for b, be in enumerate(betas):
            for h, th in enumerate(thetas):
                one = sweep(k2[r], kmax[r], betas=(be,), thetas=(th,))[0, 0, 0]
                np.testing.assert_array_equal(full[r, b, h], one)
                assert full[r, b, h, 2] >= 6.0 or full[r, b, h, 0] == 0
