"""Oracle pins for NEXT-1's q update per evaluation epoch ("a timely
update to the q^T vector", P:243 500 samples; reading L24):
the evaluations fire exactly where the pinned evaluator sweep fires (count
and the sum of k2 at them), the estimate is the empirical preference rate
of the latent best levels of the sampled requests -- recomputed here with
synth's independent numpy Philox and a numpy inverse CDF -- it stays
constant between evaluations, equals q_true before any sample, and
concentrates around q_true; the closed loop uses each interval's epoch q."""
import dataclasses

import numpy as np
import pytest

import oracle
import synth


def _numpy_pref_levels(q, seed, g_lo, g_hi):
    """l* of requests [g_lo, g_hi): Philox4x32-10 stream 2 (synth's numpy
    implementation), word g & 3, inverse CDF of q with 2^32-scaled
    thresholds and the saturation clamp (a4/a6 written out in numpy)."""
    g = np.arange(g_lo, g_hi, dtype=np.uint64)
    blk = g >> np.uint64(2)
    words = np.stack(synth.philox4x32_10(blk & np.uint64(0xFFFFFFFF), blk >> np.uint64(32), 2, 0,
                                         seed & 0xFFFFFFFF, seed >> 32))
    u = words[(g & np.uint64(3)).astype(np.int64), np.arange(len(g))].astype(np.float64)
    n = len(q)
    cum, T, ml = 0.0, [], n - 1
    for i in range(n - 1):
        cum = cum + q[i]
        t = min(np.ceil(cum * 2.0**32), 2.0**32)
        T.append(t)
        if t == 2.0**32 and ml == n - 1:
            ml = i
    L = np.zeros(len(g), np.int64)
    for t in T:
        L += (u >= t)
    return np.minimum(L, ml)


def _cfg(name="C2", **kw):
    w = synth.make_workload(name, **kw)
    return w, dict(dt=1.0 if w.prob.T <= 8760 else 1 / 12, beta=0.028, theta=0.5, grace=6.0, fallback=3)


@pytest.mark.parametrize("sample", [500, 37])
def test_fires_and_estimates(sample):
    w, c = _cfg("C2", n_requests=40_000, n_intervals=240)
    P = w.prob
    q_true = np.asarray(P.q)
    q, fired = oracle.evaluation_q(P.k0, P.kmax, P.T, c["dt"], c["beta"], c["theta"], c["grace"], c["fallback"],
                                   q_true, w.cost.seed, w.spec.seg_offsets, sample)
    sweep = oracle.evaluator_sweep(P.k0, P.kmax, P.T, c["dt"], [c["beta"]], [c["theta"]], c["grace"],
                                   c["fallback"], 0.2778, P.pue)
    off = w.spec.seg_offsets
    for r in range(P.R):
        fr = fired[r * P.T:(r + 1) * P.T]
        assert fr[0] == 1
        assert fr[1:].sum() == sweep[r, 0, 0, 0]                               # the pinned sweep's count
        acc = 0.0   # the sweep sums k2 at its evaluations sequentially
        for v in np.asarray(P.k0)[r * P.T + np.nonzero(fr[1:])[0] + 1]:
            acc += float(v)
        assert acc == sweep[r, 0, 0, 3]
        cur = q_true[r].copy()
        for t in range(P.T):
            s = r * P.T + t
            if fr[t]:
                end, begin = off[s], max(off[r * P.T], off[s] - sample)
                if end > begin:
                    lv = _numpy_pref_levels(q_true[r], w.cost.seed, begin, end)
                    cur = np.bincount(lv, minlength=P.n) / (end - begin)
            np.testing.assert_array_equal(q[s], cur)


def test_estimates_concentrate():
    w, c = _cfg("C2", n_requests=400_000, n_intervals=480)
    P = w.prob
    q, fired = oracle.evaluation_q(P.k0, P.kmax, P.T, c["dt"], c["beta"], c["theta"], c["grace"], c["fallback"],
                                   np.asarray(P.q), w.cost.seed, w.spec.seg_offsets, 500)
    for r in range(P.R):
        rows = q[r * P.T:(r + 1) * P.T][fired[r * P.T:(r + 1) * P.T] == 1][1:]   # epochs with 500 samples
        assert len(rows) > 3
        for i, qi in enumerate(np.asarray(P.q)[r]):
            assert np.all(np.abs(rows[:, i] - qi) <= 5 * np.sqrt(qi * (1 - qi) / 500))
        np.testing.assert_allclose(rows.sum(axis=1), 1.0, rtol=0, atol=1e-12)


def test_closed_loop_uses_epoch_q():
    w = synth.make_workload("C3", n_requests=6_000, n_intervals=36, n_regions=2)
    sh = synth.shard(w.spec, 1, 0)
    toks, fl = synth.host_trace(w.spec, sh)
    P = w.prob
    q_const = np.repeat(np.asarray(P.q), P.T, axis=0)
    base = oracle.closed_loop(P, w.cost, 50, w.spec.seg_offsets, toks, fl)
    same = oracle.closed_loop(P, w.cost, 50, w.spec.seg_offsets, toks, fl, q_seg=q_const)
    for k in ("x", "cnt", "tok", "carbon", "profile"):
        np.testing.assert_array_equal(base[k], same[k])
    q, fired = oracle.evaluation_q(P.k0, P.kmax, P.T, 1 / 12, 0.028, 0.5, 2.0, 3, np.asarray(P.q), w.cost.seed,
                                   w.spec.seg_offsets, 200)
    cl = oracle.closed_loop(P, w.cost, 50, w.spec.seg_offsets, toks, fl, q_seg=q)
    # every interval's LP is the one of its profile and its epoch's q
    X = P.X
    for cell in range(0, P.R * P.T * X, 5):
        s = cell // X
        r = s // P.T
        one = dataclasses.replace(P, R=1, T=1, X=1, k0=P.k0[s:s + 1], kmin=P.kmin[r:r + 1], kmax=P.kmax[r:r + 1],
                                  xi=P.xi[cell % X:cell % X + 1], e=cl["profile"][cell, 0][None],
                                  p=cl["profile"][cell, 1][None], q=q[s][None])
        np.testing.assert_array_equal(cl["x"][cell], oracle.solve_cells(one)["x"][0])
