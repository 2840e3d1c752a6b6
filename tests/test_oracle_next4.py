"""Oracle pins for NEXT-4: the normalized preference score
(SPEC S:462-470 worked values), the latent best level (
reading L21), the head-to-head outcome against Base (reading L22), the
per-request outputs of Fig. eval2 and the Oracle scheme (
reading L23).  Each is checked against something other than itself: the
paper's worked numbers, an independent Philox (synth's numpy one), binomial
frequencies, plain-Python replays, and exhaustive enumeration of every
assignment on tiny instances."""
import dataclasses
import itertools

import numpy as np
import pytest

import oracle
import synth


# ---- P:377 normalized preference --------------------------------------------

def test_normalized_preference_worked_values():
    assert oracle.normalized_preference(0.48) == pytest.approx(0.923, abs=1e-3)    # P:377 "92.3%"
    assert oracle.normalized_preference(0.487) == pytest.approx(0.9493, abs=1e-3)
    assert oracle.normalized_preference(0.5) == 1.0                                 # parity
    assert oracle.normalized_preference(0.0) == 0.0
    assert oracle.normalized_preference(1.0) == float("inf")
    ws = np.linspace(0.0, 0.99, 100)
    v = [oracle.normalized_preference(w) for w in ws]
    assert all(b > a for a, b in zip(v, v[1:]))


# ---- reading L21: latent best level --------------------------------------------

def test_pref_word_is_philox_stream_2():
    seed = 0x5350524F5554 + 3
    g = np.array([0, 1, 2, 3, 4, 5, 2**32 + 7, 2**33 + 1, 123456789], np.uint64)
    blk = g >> np.uint64(2)
    words = synth.philox4x32_10(blk & np.uint64(0xFFFFFFFF), blk >> np.uint64(32), 2, 0,
                                seed & 0xFFFFFFFF, seed >> 32)
    want = np.stack(words)[(g & np.uint64(3)).astype(np.int64), np.arange(len(g))]
    got = [oracle.pref_word(seed, int(x)) for x in g]
    np.testing.assert_array_equal(got, want)
    # a different stream from the selection draw (stream 0)
    assert any(oracle.pref_word(seed, int(x)) != oracle.draw_word(seed, int(x)) for x in g)


@pytest.mark.parametrize("q", [[0.5, 0.3, 0.2], [0.34, 0.36, 0.30], [0.1, 0.0, 0.9], [0.25, 0.25, 0.25, 0.25]])
def test_pref_level_frequencies(q):
    seed, M = 99, 60_000
    lv = np.array([oracle.pref_level(q, seed, g) for g in range(M)])
    for i, qi in enumerate(q):
        f = np.mean(lv == i)
        assert abs(f - qi) <= 5 * np.sqrt(max(qi * (1 - qi), 1e-12) / M) + 1e-12, (i, f, qi)


def test_pref_level_degenerate():
    for k in range(3):
        q = [0.0, 0.0, 0.0]
        q[k] = 1.0
        assert all(oracle.pref_level(q, 5, g) == k for g in range(500))


# ---- reading L22: head-to-head against Base -------------------------------------

def test_head_to_head_table():
    for L, ls in itertools.product(range(4), range(4)):
        win, loss = oracle.head_to_head(L, ls)
        if L == 0:
            assert (win, loss) == (0, 0)              # identical responses: a tie
        elif ls == L:
            assert (win, loss) == (1, 0)
        elif ls == 0:
            assert (win, loss) == (0, 1)
        else:
            assert (win, loss) == (0, 0)              # the best level is a third one


def _small(name="C1", **kw):
    w = synth.make_workload(name, **kw)
    sh = synth.shard(w.spec, 1, 0)
    toks, fl = synth.host_trace(w.spec, sh)
    return w, toks, fl


def _replay_levels(w, x, s, fl):
    off = w.spec.seg_offsets
    out = []
    for g in range(off[s], off[s + 1]):
        f = int(fl[g]) if fl is not None else 0
        out.append((g, f, oracle.select_level(x, oracle.draw_word(w.cost.seed, g), bool(f & 1))))
    return out


def test_preference_stats_replay():
    w, toks, fl = _small("C2", n_requests=4_000, n_intervals=8)
    st = oracle.preference(w.prob, w.cost, w.spec.seg_offsets, fl)
    cells = oracle.solve_cells(w.prob)
    X = w.prob.X
    for cell in range(0, w.prob.R * w.prob.T * X, 7):
        s, j = divmod(cell, X)
        q = np.asarray(w.prob.q)[s // w.prob.T]
        hits = wins = losses = 0
        for g, f, L in _replay_levels(w, cells["x"][cell], s, fl):
            ls = oracle.pref_level(q, w.cost.seed, g)
            hits += L == ls
            wins += L != 0 and ls == L
            losses += L != 0 and ls == 0
        assert tuple(st[cell]) == (hits, wins, losses)


def test_base_like_cell_scores_one():
    """xi = 0 with a unique-max q0 forces pure L0: every comparison
    with Base is a tie, w = 1/2, score 1."""
    w, toks, fl = _small("C1")
    prob = dataclasses.replace(w.prob, xi=np.array([0.0]))
    st = oracle.preference(prob, w.cost, w.spec.seg_offsets, fl)
    assert np.all(st[:, 1] == 0) and np.all(st[:, 2] == 0)
    m = np.diff(w.spec.seg_offsets)
    wfrac = (st[:, 1] + (m - st[:, 1] - st[:, 2]) / 2) / m
    assert np.allclose([oracle.normalized_preference(x) for x in wfrac], 1.0)


# ---- P:425 per-request outputs ----------------------------------------------------

def test_request_outputs_replay_and_totals():
    w, toks, fl = _small("C2", n_requests=3_000, n_intervals=6)
    j = 1
    ro = oracle.request_outputs(w.prob, w.cost, w.spec.seg_offsets, toks, fl, j=j)
    cells = oracle.solve_cells(w.prob)
    S = w.prob.R * w.prob.T
    off = w.spec.seg_offsets
    sim = oracle.simulate(w.prob, w.cost, np.arange(S), off[:-1], np.diff(off), off[:-1], toks, fl)
    ef, et, pf, pt = (np.asarray(a) for a in (w.cost.ef, w.cost.et, w.cost.pf, w.cost.pt))
    X = w.prob.X
    for s in range(S):
        kp = w.prob.k0[s] * w.prob.pue
        csum = 0.0
        for g, f, L in _replay_levels(w, cells["x"][s * X + j], s, fl):
            c = (f >> 1) & 3
            assert ro["level"][g] == L
            el = ef[c, L] + et[c, L] * float(toks[L, g])
            pl = pf[c, L] + pt[c, L] * float(toks[L, g])
            e0 = ef[c, 0] + et[c, 0] * float(toks[0, g])
            p0 = pf[c, 0] + pt[c, 0] * float(toks[0, g])
            assert ro["carbon"][g] == kp * el + w.prob.k1 * pl
            assert ro["base"][g] == kp * e0 + w.prob.k1 * p0
            assert ro["ratio"][g] == ro["carbon"][g] / ro["base"][g]
            csum += ro["carbon"][g]
        # the per-request carbons add up (in request order) to the cell total (S:485 conservation)
        assert csum == sim["carbon"][s, j]
    assert np.all(ro["ratio"][ro["level"] == 0] == 1.0)


# ---- reading L23: the Oracle scheme -----------------------------------------------

def _tiny_oracle_problem(seed=3, m=(5, 6, 4), xis=(0.0, 0.4, 1.0)):
    rng = np.random.default_rng(seed)
    n, T = 3, len(m)
    prob = synth.Problem(n=n, R=1, T=T, X=len(xis), k0=rng.uniform(50, 450, T), kmin=np.array([40.0]),
                         kmax=np.array([460.0]), xi=np.array(xis), e=np.zeros((1, n)), p=np.zeros((1, n)),
                         q=np.array([[0.45, 0.35, 0.20]]), profile_per_interval=0, k1=9.5e-4, pue=1.2)
    ef = np.zeros((4, 8)); et = np.zeros((4, 8)); pf = np.zeros((4, 8)); pt = np.zeros((4, 8))
    ef[0, :n] = [2e-6, 1.9e-6, 1.8e-6]; et[0, :n] = [1e-7, 1.1e-7, 1.2e-7]
    pf[0, :n] = 0.01; pt[0, :n] = 0.0016
    cost = synth.CostModel(seed=seed + 11, n_classes=1, ef=ef, et=et, pf=pf, pt=pt)
    off = np.concatenate([[0], np.cumsum(m)]).astype(np.int64)
    N = int(off[-1])
    toks = rng.integers(1, 400, size=(n, max(8, N))).astype(np.uint16)
    toks[1] = np.minimum(toks[1], toks[0]); toks[2] = np.minimum(toks[2], toks[1])
    fl = np.zeros(max(8, N), np.uint8)
    fl[rng.random(max(8, N)) < 0.15] |= 1          # opted-out users
    return prob, cost, off, toks, fl


def _carbon(prob, cost, s, g, L, toks):
    kp = prob.k0[s] * prob.pue
    t = float(toks[L, g])
    return kp * (cost.ef[0][L] + cost.et[0][L] * t) + prob.k1 * (cost.pf[0][L] + cost.pt[0][L] * t)


@pytest.mark.parametrize("seed", [3, 4, 5, 6])
def test_oracle_scheme_exhaustive(seed):
    """Every assignment of every (<= 6-request) segment: the oracle's carbon
    is the minimum over the assignments meeting the realised-quality floor."""
    prob, cost, off, toks, fl = _tiny_oracle_problem(seed)
    out = oracle.oracle_scheme(prob, cost, off, toks, fl)
    n, X = prob.n, prob.X
    for s in range(prob.T):
        gs = list(range(off[s], off[s + 1]))
        ls = [oracle.pref_level(prob.q[0], cost.seed, g) for g in gs]
        m = len(gs)
        for j in range(X):
            b = oracle.quality_lower_bound(prob.k0[s], prob.kmin[0], prob.kmax[0], prob.xi[j], prob.q[0][0])
            k = int(np.ceil(b * m))
            best = None
            for assign in itertools.product(range(n), repeat=m):
                if any(fl[g] & 1 and L != 0 for g, L in zip(gs, assign)):
                    continue
                if sum(L == l for L, l in zip(assign, ls)) < k:
                    continue
                c = sum(_carbon(prob, cost, s, g, L, toks) for g, L in zip(gs, assign))
                best = c if best is None else min(best, c)
            cell = s * X + j
            assert out["status"][cell] == 0
            assert out["carbon"][cell] == pytest.approx(best, rel=1e-12)
            assert out["stats"][cell][0] >= k
            assert out["cnt"][cell].sum() == m


def test_oracle_scheme_bounds_and_monotone():
    w, toks, fl = _small("C2", n_requests=6_000, n_intervals=12)
    prob = dataclasses.replace(w.prob, xi=np.array([0.0, 0.05, 0.1, 0.2, 0.5, 1.0]))
    out = oracle.oracle_scheme(prob, w.cost, w.spec.seg_offsets, toks, fl)
    X, NC, n = prob.X, w.cost.n_classes, prob.n
    off = w.spec.seg_offsets
    ef, et, pf, pt = (np.asarray(a) for a in (w.cost.ef, w.cost.et, w.cost.pf, w.cost.pt))
    for s in range(prob.R * prob.T):
        q = np.asarray(prob.q)[s // prob.T]
        kp = prob.k0[s] * prob.pue
        cmin = cbest = 0.0
        for g in range(off[s], off[s + 1]):
            c = (int(fl[g]) >> 1) & 3
            C = [kp * (ef[c, L] + et[c, L] * float(toks[L, g])) + prob.k1 * (pf[c, L] + pt[c, L] * float(toks[L, g]))
                 for L in range(n)]
            pinned = int(fl[g]) & 1
            cmin += C[0] if pinned else min(C)
            cbest += C[0] if pinned else C[oracle.pref_level(q, w.cost.seed, g)]
        cs = out["carbon"][s * X:(s + 1) * X]
        assert np.all(cs >= cmin * (1 - 1e-12)) and np.all(cs <= cbest * (1 + 1e-12))
        assert np.all(np.diff(cs) <= 0)                    # relaxing xi never costs carbon
        assert np.all(out["status"][s * X:(s + 1) * X] == 0)
