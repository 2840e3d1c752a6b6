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
