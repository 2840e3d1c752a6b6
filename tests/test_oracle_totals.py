"""Pins of the oracle's trace replay and group totals (CPU only).

Against: an independent Python replay of tiny traces (exact rational sums,
selection draws from synth's separately-KAT-pinned Philox), special cases
with closed forms (xi = 0 => Base, uniform q => cheapest level, k0 = kmin),
conservation laws, binomial level frequencies and thread invariance.
"""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth


def tiny_workload(n=3, R=2, T=3, X=2, N=60, NC=2, flags=True, seed=5, xi=(0.1, 0.4)):
    w = synth.make_workload("C2", n_requests=N, n_intervals=T, n_regions=R, xi=np.array(xi), seed_offset=seed)
    prob = w.prob
    if n != 3:
        raise NotImplementedError
    spec = w.spec
    spec.n_classes = NC
    spec.has_flags = flags
    spec.pin_thresh = 2_000_000 if flags else 0          # ~12% pinned: exercises P:240
    spec.q0_table = np.stack([synth.q0_table(250.0), synth.q0_table(220.0)])[:NC]
    ef, et, pf, pt = synth.cost_coefficients(NC, n)
    cost = synth.CostModel(seed=0xABCDEF0123 + seed, n_classes=NC, ef=ef, et=et, pf=pf, pt=pt)
    return prob, cost, spec


def run_all(prob, cost, spec, levels=False, threads=4):
    sh = synth.shard(spec, 1, 0)
    toks, flags = synth.host_trace(spec, sh)
    S = prob.R * prob.T
    seg_id = np.arange(S)
    req_begin = sh.seg_offsets[:-1]
    seg_m = np.diff(sh.seg_offsets)
    g0 = sh.first_request + req_begin
    sim = oracle.simulate(prob, cost, seg_id, req_begin, seg_m, g0, toks, flags, levels=levels, threads=threads)
    return sh, toks, flags, sim


def _draw(seed, g):
    blk = g >> 2
    out = synth.philox4x32_10(np.uint64(blk & 0xFFFFFFFF), np.uint64(blk >> 32), 0, 0,
                              seed & 0xFFFFFFFF, seed >> 32)
    return int(out[g & 3])


def test_tiny_trace_vs_independent_replay():
    prob, cost, spec = tiny_workload()
    sh, toks, flags, sim = run_all(prob, cost, spec, levels=True)
    cells = oracle.solve_cells(prob)
    n, X, NC = prob.n, prob.X, cost.n_classes
    for s in range(prob.R * prob.T):
        r = s // prob.T
        a, b = sh.seg_offsets[s], sh.seg_offsets[s + 1]
        kp = Fraction(prob.k0[s]) * Fraction(prob.pue)
        for j in range(X):
            cell = s * X + j
            x = cells["x"][cell]
            cum = [sum((Fraction(v) for v in x[:i + 1]), Fraction(0)) for i in range(n - 1)]
            E = Fraction(0); Tm = Fraction(0); Cg = Fraction(0); Q = Fraction(0)
            cnt = np.zeros((NC, n), np.int64); tok = np.zeros((NC, n), np.int64)
            for ri in range(a, b):
                g = sh.first_request + ri
                w = _draw(cost.seed, g)
                f = int(flags[ri])
                pinned, c = f & 1, (f >> 1) & 3
                if pinned:
                    L = 0
                else:
                    u = Fraction(w, 2**32)
                    L = next((i for i in range(n - 1) if u < cum[i]), n - 1)
                assert sim["levels"][j, ri] == L
                t = int(toks[L, ri])
                e = Fraction(cost.ef[c, L]) + Fraction(cost.et[c, L]) * t
                p = Fraction(cost.pf[c, L]) + Fraction(cost.pt[c, L]) * t
                E += e; Tm += p; Cg += kp * e + Fraction(prob.k1) * p
                Q += Fraction(prob.q[r, L])
                cnt[c, L] += 1; tok[c, L] += t
            np.testing.assert_array_equal(sim["cnt"][s, j], cnt)
            np.testing.assert_array_equal(sim["tok"][s, j], tok)
            for got, want in ((sim["energy"][s, j], E), (sim["time"][s, j], Tm),
                              (sim["carbon"][s, j], Cg), (sim["quality"][s, j], Q)):
                assert got == pytest.approx(float(want), rel=1e-13, abs=1e-300)


def test_xi_zero_equals_base():
    # S:442 / S:484: xi = 0 with a unique-max q0 forces L0 => every cell's
    # totals equal the Base counterfactual; savings 0
    prob, cost, spec = tiny_workload(xi=(0.0,), N=400)
    sh, toks, flags, sim = run_all(prob, cost, spec)
    assert np.all(prob.q[:, 0] > prob.q[:, 1:].max(axis=1))
    for s in range(prob.R * prob.T):
        assert np.all(sim["cnt"][s, 0, :, 1:] == 0)
        np.testing.assert_array_equal(sim["cnt"][s, 0, :, 0], sim["seg_count"][s])
        assert sim["energy"][s, 0] == sim["seg_base"][s, 0]
        assert sim["time"][s, 0] == sim["seg_base"][s, 1]
        assert sim["carbon"][s, 0] == sim["seg_base"][s, 2]
        assert sim["quality"][s, 0] == sim["seg_base"][s, 3]


def test_uniform_q_selects_cheapest_level():
    # q uniform => pure cheapest level; pinned requests stay at L0
    prob, cost, spec = tiny_workload(N=500)
    prob.q[:] = 1.0 / 3.0
    sh, toks, flags, sim = run_all(prob, cost, spec)
    cells = oracle.solve_cells(prob)
    for s in range(prob.R * prob.T):
        c = oracle.cost_vector(prob.k0[s], prob.pue, prob.k1, prob.e[s // prob.T], prob.p[s // prob.T])
        L = int(np.argmin(c))
        for j in range(prob.X):
            assert cells["vertex"][s * prob.X + j] == L
            for cls in range(cost.n_classes):
                want = np.zeros(prob.n, np.uint64)
                want[L] += sim["seg_count"][s, cls] - sim["seg_pinned"][s, cls]
                want[0] += sim["seg_pinned"][s, cls]
                np.testing.assert_array_equal(sim["cnt"][s, j, cls], want)


def test_kmin_interval_forces_q0():
    prob, cost, spec = tiny_workload()
    prob.k0[:] = np.repeat(prob.kmin, prob.T)
    cells = oracle.solve_cells(prob)
    q0 = np.repeat(prob.q[:, 0], prob.T * prob.X)
    np.testing.assert_array_equal(cells["q_lb"], q0)


def test_conservation_and_closed_form():
    prob, cost, spec = tiny_workload(N=3000)
    sh, toks, flags, sim = run_all(prob, cost, spec)
    cells = oracle.solve_cells(prob)
    n = prob.n
    for s in range(prob.R * prob.T):
        a, b = sh.seg_offsets[s], sh.seg_offsets[s + 1]
        assert int(sim["seg_count"][s].sum()) == b - a
        for i in range(n):
            assert int(sim["seg_tok"][s, :, i].sum()) == int(toks[i, a:b].sum())
        kp = prob.k0[s] * prob.pue
        for j in range(prob.X):
            cnt, tok = sim["cnt"][s, j].astype(np.int64), sim["tok"][s, j].astype(np.int64)
            np.testing.assert_array_equal(cnt.sum(axis=1), sim["seg_count"][s].astype(np.int64))
            # Eq. 1 summed per request equals its closed form in the integer stats
            E = math.fsum(float(Fraction(cost.ef[c, L]) * int(cnt[c, L]) + Fraction(cost.et[c, L]) * int(tok[c, L]))
                          for c in range(cost.n_classes) for L in range(n))
            Tm = math.fsum(float(Fraction(cost.pf[c, L]) * int(cnt[c, L]) + Fraction(cost.pt[c, L]) * int(tok[c, L]))
                           for c in range(cost.n_classes) for L in range(n))
            assert sim["energy"][s, j] == pytest.approx(E, rel=1e-12)
            assert sim["time"][s, j] == pytest.approx(Tm, rel=1e-12)
            assert sim["carbon"][s, j] == pytest.approx(kp * E + prob.k1 * Tm, rel=1e-12)
            Q = math.fsum(float(prob.q[s // prob.T, L]) * int(cnt[:, L].sum()) for L in range(n))
            assert sim["quality"][s, j] == pytest.approx(Q, rel=1e-12)


def test_level_frequencies_binomial():
    # the realised mix follows x: binomial 5 sigma per level
    prob, cost, spec = tiny_workload(R=1, T=1, X=2, N=200_000, flags=False, NC=1)
    prob.kmin[:] = 100.0; prob.kmax[:] = 500.0; prob.k0[:] = 450.0
    sh, toks, flags, sim = run_all(prob, cost, spec)
    cells = oracle.solve_cells(prob)
    m = int(sim["seg_count"][0].sum())
    for j in range(prob.X):
        x = cells["x"][j]
        assert np.count_nonzero(x) == 2          # a mixed policy, not a pure level
        got = sim["cnt"][0, j, 0].astype(np.float64)
        sd = np.sqrt(m * x * (1 - x)) + 1e-9
        assert np.all(np.abs(got - m * x) <= 5 * sd + 1), (got, m * x)


def test_thread_invariance_and_bad_class():
    prob, cost, spec = tiny_workload(N=2000)
    sh, toks, flags, sim1 = run_all(prob, cost, spec, threads=1)
    _, _, _, sim8 = run_all(prob, cost, spec, threads=8)
    for k in ("cnt", "tok", "energy", "time", "carbon", "quality", "seg_count", "seg_base"):
        np.testing.assert_array_equal(sim1[k], sim8[k])
    # class index >= n_classes: request skipped and counted
    flags2 = flags.copy()
    flags2[sh.seg_offsets[0]] = (3 << 1)
    S = prob.R * prob.T
    out = oracle.simulate(prob, cost, np.arange(S), sh.seg_offsets[:-1], np.diff(sh.seg_offsets),
                          sh.first_request + sh.seg_offsets[:-1], toks, flags2)
    assert out["bad_requests"] == 1
    assert int(out["seg_count"].sum()) == int(sim1["seg_count"].sum()) - 1


def test_reduce_conservation():
    prob, cost, spec = tiny_workload(N=5000)
    sh, toks, flags, sim = run_all(prob, cost, spec)
    cells = oracle.solve_cells(prob)
    S = prob.R * prob.T
    G = oracle.reduce(prob, cost.n_classes, 0, S, cells, sim)
    n, X, R, T = prob.n, prob.X, prob.R, prob.T
    for r in range(R):
        for j in range(X):
            segs = range(r * T, (r + 1) * T)
            g = G[r, j]
            assert g[0] == sum(int(sim["seg_count"][s].sum()) for s in segs)
            assert g[1] == sum(int(sim["seg_pinned"][s].sum()) for s in segs)
            assert g[2] == pytest.approx(math.fsum(sim["energy"][s, j] for s in segs), rel=1e-14)
            assert g[4] == pytest.approx(math.fsum(sim["carbon"][s, j] for s in segs), rel=1e-14)
            assert g[8] == pytest.approx(math.fsum(sim["seg_base"][s, 2] for s in segs), rel=1e-14)
            for L in range(n):
                assert g[11 + L] == sum(int(sim["cnt"][s, j, :, L].sum()) for s in segs)
                assert g[11 + n + L] == sum(int(sim["tok"][s, j, :, L].sum()) for s in segs)
            exp = math.fsum(float(sim["seg_count"][s].sum()) * cells["objective"][s * X + j] for s in segs)
            assert g[10] == pytest.approx(exp, rel=1e-14)
    np.testing.assert_allclose(G[R], G[:R].sum(axis=0), rtol=1e-14)
    # counts per level add up to requests
    np.testing.assert_array_equal(G[:, :, 11:11 + n].sum(axis=2), G[:, :, 0])
