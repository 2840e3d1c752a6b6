"""Oracle pins for closed-loop profiles (reading
L20): the replay equals the open-loop replay wherever the mixes agree, the
first interval uses the priors, and the profile of every later interval is
the mean over exactly the right window (W >= all requests: every earlier
request of the level; W = 1: the last one), checked by brute force."""
import numpy as np
import pytest

import oracle
import synth


def _w(name="C1", **kw):
    w = synth.make_workload(name, **kw)
    sh = synth.shard(w.spec, 1, 0)
    toks, fl = synth.host_trace(w.spec, sh)
    return w, toks, fl


def _open(w, toks, fl):
    S = w.prob.R * w.prob.T
    off = w.spec.seg_offsets
    return oracle.simulate(w.prob, w.cost, np.arange(S), off[:-1], np.diff(off), off[:-1], toks, fl)


@pytest.mark.parametrize("W", [1, 5, 1000, 10**7])
def test_replay_matches_open_loop_where_mixes_agree(W):
    w, toks, fl = _w("C2", n_requests=30_000, n_intervals=40)
    cl = oracle.closed_loop(w.prob, w.cost, W, w.spec.seg_offsets, toks, fl)
    op = oracle.solve_cells(w.prob)
    sim = _open(w, toks, fl)
    same = np.all(cl["x"] == op["x"], axis=1)
    assert same.any()
    X, NC, n = w.prob.X, w.cost.n_classes, w.prob.n
    cnt = sim["cnt"].reshape(-1, NC, n)
    tok = sim["tok"].reshape(-1, NC, n)
    np.testing.assert_array_equal(cl["cnt"][same], cnt[same])
    np.testing.assert_array_equal(cl["tok"][same], tok[same])
    for k in ("energy", "time", "carbon", "quality"):
        np.testing.assert_array_equal(cl[k][same], sim[k].reshape(-1)[same])
    # conservation: every valid request is counted once per cell
    m = np.diff(w.spec.seg_offsets)
    np.testing.assert_array_equal(cl["cnt"].reshape(-1, X, NC * n).sum(axis=2), np.repeat(m, X).reshape(-1, X))


def test_priors_then_windows():
    w, toks, fl = _w("C1")
    n, T = w.prob.n, w.prob.T
    big = oracle.closed_loop(w.prob, w.cost, 10**7, w.spec.seg_offsets, toks, fl)
    one = oracle.closed_loop(w.prob, w.cost, 1, w.spec.seg_offsets, toks, fl)
    e0, p0 = w.prob.e[0], w.prob.p[0]
    np.testing.assert_array_equal(big["profile"][0, 0], e0)
    np.testing.assert_array_equal(big["profile"][0, 1], p0)
    ef, et, pf, pt = (np.asarray(a)[0] for a in (w.cost.ef, w.cost.et, w.cost.pf, w.cost.pt))
    # W unbounded: the mean over every earlier request of the level (single class)
    cnt = big["cnt"][:, 0, :].astype(np.float64)
    tok = big["tok"][:, 0, :].astype(np.float64)
    for t in range(1, T):
        for L in range(n):
            m, k = cnt[:t, L].sum(), tok[:t, L].sum()
            want_e = e0[L] if m == 0 else (m * ef[L] + k * et[L]) / m
            want_p = p0[L] if m == 0 else (m * pf[L] + k * pt[L]) / m
            assert big["profile"][t, 0, L] == pytest.approx(want_e, rel=1e-15)
            assert big["profile"][t, 1, L] == pytest.approx(want_p, rel=1e-15)
    # W = 1: the last request run at the level, from a brute-force replay of the levels
    off = w.spec.seg_offsets
    last = [None] * n
    for t in range(T):
        for L in range(n):
            if last[L] is None:
                assert one["profile"][t, 0, L] == e0[L]
            else:
                assert one["profile"][t, 0, L] == pytest.approx(ef[L] + et[L] * last[L], rel=1e-15)
                assert one["profile"][t, 1, L] == pytest.approx(pf[L] + pt[L] * last[L], rel=1e-15)
        if one["cell_status"][t] != 0:
            continue
        for g in range(off[t], off[t + 1]):
            Lg = oracle.select_level(one["x"][t], oracle.draw_word(w.cost.seed, g), bool(fl[g] & 1))
            last[Lg] = int(toks[Lg, g])


# --------------------------------------------------------------------------
# Brute-force window pins for 1 < W < infinity: a plain
# replay that keeps, per (chain, level), the literal list of the last W
# (class, tokens) entries in a collections.deque(maxlen=W) and recomputes the
# mean Eq. 1 energy / time from scratch, entry by entry, before every
# interval ("average ... for recent requests at each level"; SPEC.md
# level_profiles S:193-201).  It shares nothing with the oracle's ring /
# running-sum bookkeeping: a wrong eviction (newest instead of oldest) or a
# decrement of the incoming request's class instead of the evicted one's
# changes the mean and fails here.

import collections
import dataclasses


def _brute_profiles(w, toks, fl, cl, W):
    n, R, T, X = w.prob.n, w.prob.R, w.prob.T, w.prob.X
    ef, et, pf, pt = (np.asarray(a, dtype=np.float64) for a in (w.cost.ef, w.cost.et, w.cost.pf, w.cost.pt))
    off = w.spec.seg_offsets
    NC = w.cost.n_classes
    for r in range(R):
        for j in range(X):
            win = [collections.deque(maxlen=W) for _ in range(n)]
            for t in range(T):
                s = r * T + t
                cell = s * X + j
                for L in range(n):
                    if not win[L]:
                        assert cl["profile"][cell, 0, L] == w.prob.e[r][L]
                        assert cl["profile"][cell, 1, L] == w.prob.p[r][L]
                        continue
                    eE = sum(ef[c][L] + et[c][L] * k for c, k in win[L]) / len(win[L])
                    eT = sum(pf[c][L] + pt[c][L] * k for c, k in win[L]) / len(win[L])
                    assert cl["profile"][cell, 0, L] == pytest.approx(eE, rel=1e-12), (r, j, t, L)
                    assert cl["profile"][cell, 1, L] == pytest.approx(eT, rel=1e-12), (r, j, t, L)
                # the interval's LP with exactly that profile is the one the oracle solved
                e_b = np.array([w.prob.e[r][L] if not win[L] else
                                sum(ef[c][L] + et[c][L] * k for c, k in win[L]) / len(win[L]) for L in range(n)])
                p_b = np.array([w.prob.p[r][L] if not win[L] else
                                sum(pf[c][L] + pt[c][L] * k for c, k in win[L]) / len(win[L]) for L in range(n)])
                one = dataclasses.replace(w.prob, R=1, T=1, X=1, k0=w.prob.k0[s:s + 1], kmin=w.prob.kmin[r:r + 1],
                                          kmax=w.prob.kmax[r:r + 1], xi=w.prob.xi[j:j + 1], e=e_b[None],
                                          p=p_b[None], q=np.asarray(w.prob.q)[r:r + 1])
                ref = oracle.solve_cells(one)
                np.testing.assert_allclose(cl["x"][cell], ref["x"][0], rtol=0, atol=1e-12)
                if cl["cell_status"][cell] != 0:
                    continue
                for g in range(off[s], off[s + 1]):
                    f = int(fl[g]) if fl is not None else 0
                    c = (f >> 1) & 3
                    if c >= NC:
                        continue
                    Lg = oracle.select_level(cl["x"][cell], oracle.draw_word(w.cost.seed, g), bool(f & 1))
                    win[Lg].append((c, int(toks[Lg, g])))


@pytest.mark.parametrize("W", [2, 3, 17])
@pytest.mark.parametrize("name,NC", [("C3", 2), ("C1", 1)])
def test_window_brute_force(W, name, NC):
    if name == "C3":
        w, toks, fl = _w("C3", n_requests=4_000, n_intervals=30, n_regions=2)
    else:
        w, toks, fl = _w("C1")
    assert w.cost.n_classes == NC
    cl = oracle.closed_loop(w.prob, w.cost, W, w.spec.seg_offsets, toks, fl)
    _brute_profiles(w, toks, fl, cl, W)


def test_window_brute_force_four_classes():
    """NC = 4 with flags: classes drawn from the flag bits; the window mixes
    classes whose (ef, et) differ, so evicting the wrong class shifts the mean."""
    w, toks, fl = _w("C3", n_requests=3_000, n_intervals=24, n_regions=1)
    rng = np.random.default_rng(7)
    fl = ((rng.integers(0, 4, size=fl.size) << 1) | (rng.random(fl.size) < 0.05)).astype(np.uint8)
    ef = np.array(w.cost.ef, dtype=np.float64).copy()
    et = np.array(w.cost.et, dtype=np.float64).copy()
    pf = np.array(w.cost.pf, dtype=np.float64).copy()
    pt = np.array(w.cost.pt, dtype=np.float64).copy()
    for c in range(4):
        ef[c] = ef[0] * (1.0 + 0.3 * c)
        et[c] = et[0] * (1.0 + 0.2 * c)
        pf[c] = pf[0] * (1.0 + 0.1 * c)
        pt[c] = pt[0] * (1.0 + 0.25 * c)
    w = dataclasses.replace(w, cost=dataclasses.replace(w.cost, n_classes=4, ef=ef, et=et, pf=pf, pt=pt))
    for W in (2, 7, 50):
        cl = oracle.closed_loop(w.prob, w.cost, W, w.spec.seg_offsets, toks, fl)
        _brute_profiles(w, toks, fl, cl, W)


def test_spec_w2_example():
    """"level 1 entries with energies [1,3] kWh, W=2 -> e_1 = 2".
    One region, two intervals, pure-L1 optimum in interval 0 (L1 has the
    highest q and the lowest prior cost); E = tok kWh at L1 (ef = 0, et = 1).
    Interval 0 runs three requests at L1 with tokens [5, 1, 3]: the W = 2
    window then holds the last two, [1, 3] -> e_1 = 2 (evicting the newest
    would leave [5, 3] -> 4; W = 3 gives 3)."""
    n = 3
    prob = synth.Problem(n=n, R=1, T=2, X=1, k0=np.array([100.0, 100.0]), kmin=np.array([50.0]),
                         kmax=np.array([150.0]), xi=np.array([0.1]), e=np.array([[3.0, 1.0, 2.0]]),
                         p=np.zeros((1, n)), q=np.array([[0.3, 0.4, 0.3]]), profile_per_interval=0,
                         k1=0.0, pue=1.0)
    ef = np.zeros((4, 8)); et = np.zeros((4, 8)); pf = np.zeros((4, 8)); pt = np.zeros((4, 8))
    ef[0, :n] = [3.0, 0.0, 2.0]
    et[0, 1] = 1.0
    cost = synth.CostModel(seed=1234, n_classes=1, ef=ef, et=et, pf=pf, pt=pt)
    off = np.array([0, 3, 4], np.int64)
    toks = np.zeros((n, 8), np.uint16)
    toks[1, :4] = [5, 1, 3, 2]
    for W, want in ((2, 2.0), (3, 3.0), (1, 3.0)):
        cl = oracle.closed_loop(prob, cost, W, off, toks, None)
        np.testing.assert_array_equal(cl["x"][0], [0.0, 1.0, 0.0])
        assert cl["cnt"][0, 0, 1] == 3
        assert cl["profile"][1, 0, 1] == want
        # levels that never ran keep the priors (S:201 cold start)
        assert cl["profile"][1, 0, 0] == 3.0 and cl["profile"][1, 0, 2] == 2.0
