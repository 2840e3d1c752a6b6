"""Pins of the CPU oracle against things other than itself (CPU only).

Each test pins one oracle function to the paper's / SPEC's worked examples,
known-answer vectors, exact rational arithmetic, the paper's own solver
(HiGHS dual simplex, via SciPy), a simplex grid, closed forms or
invariants -- chosen so a dropped term, a wrong sign/index or a transposed
operand fails at least one of them.
"""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
from conftest import hexint

# ----------------------------------------------------------------- Philox


def test_philox_known_answers(golden):
    for case in golden["philox4x32_10_kat"]["cases"]:
        ctr = [hexint(v) for v in case["ctr"]]
        key = [hexint(v) for v in case["key"]]
        out = oracle.philox4x32_10(ctr, key)
        assert [int(v) for v in out] == [hexint(v) for v in case["out"]]


def test_draw_word_counter_layout(golden):
    # a5: key = (seed lo, seed hi), ctr = (g>>2 lo, g>>2 hi, 0, 0), word g&3.
    # With seed 0 and g in 0..3 the words are the first KAT vector's output.
    kat = [hexint(v) for v in golden["philox4x32_10_kat"]["cases"][0]["out"]]
    assert [oracle.draw_word(0, g) for g in range(4)] == kat
    # key words = (seed lo32, seed hi32); counter words 0-1 = (g>>2 lo32,
    # g>>2 hi32); words 2-3 are zero on stream 0.  Compare with the raw call.
    seed = 0x299F31D0A4093822
    blk = 0x05A308D3243F6A88          # g = 4*blk + k must fit in 64 bits
    raw = oracle.philox4x32_10([blk & 0xFFFFFFFF, blk >> 32, 0, 0], [seed & 0xFFFFFFFF, seed >> 32])
    for k in range(4):
        assert oracle.draw_word(seed, blk * 4 + k) == int(raw[k])


# ------------------------------------------------------------- Eqs. 1-3


def test_request_footprint_examples(golden):
    for c in golden["request_footprint"]["cases"]:
        kp = c["k0"] * c["pue"]
        got = oracle.request_carbon(kp, c["k1"], c["energy_kwh"], c["time_s"])
        assert got == pytest.approx(c["carbon_g"], rel=1e-15, abs=1e-18), c["cite"]


def test_request_footprint_linearity():
    # S:69 footprint(aE,T) - footprint(0,T) = a (footprint(E,T) - footprint(0,T))
    rng = np.random.default_rng(1)
    for _ in range(200):
        kp, k1, E, T, a = rng.uniform(0, 600), rng.uniform(0, 1e-3), rng.uniform(0, 1e-3), rng.uniform(0, 5), rng.uniform(0, 10)
        f0 = oracle.request_carbon(kp, k1, 0.0, T)
        lhs = oracle.request_carbon(kp, k1, a * E, T) - f0
        rhs = a * (oracle.request_carbon(kp, k1, E, T) - f0)
        assert lhs == pytest.approx(rhs, rel=1e-12, abs=1e-15)
        assert oracle.request_carbon(kp, k1, E, T) >= k1 * T


def test_quality_lower_bound_examples(golden):
    for c in golden["quality_lower_bound"]["cases"]:
        got = oracle.quality_lower_bound(c["k0"], c["kmin"], c["kmax"], c["xi"], c["q0"])
        assert got == pytest.approx(c["b"], rel=2e-16, abs=0), c["cite"]


def test_quality_lower_bound_closed_form_and_clamp():
    rng = np.random.default_rng(2)
    for _ in range(500):
        kmin = rng.uniform(0, 200); kmax = kmin + rng.uniform(1, 500)
        xi, q0 = rng.uniform(0, 1), rng.uniform(0, 1)
        # boundaries: b(kmin) = q0, b(kmax) = (1 - xi) q0 exactly
        assert oracle.quality_lower_bound(kmin, kmin, kmax, xi, q0) == q0
        assert oracle.quality_lower_bound(kmax, kmin, kmax, xi, q0) == (1.0 - xi) * q0
        # clamp outside [kmin, kmax] (reading L3)
        assert oracle.quality_lower_bound(kmin - 50, kmin, kmax, xi, q0) == q0
        assert oracle.quality_lower_bound(kmax + 50, kmin, kmax, xi, q0) == (1.0 - xi) * q0
        # exact rational value of Eq. 3 inside the range
        k0 = rng.uniform(kmin, kmax)
        exact = (1 - (Fraction(k0) - Fraction(kmin)) / (Fraction(kmax) - Fraction(kmin)) * Fraction(xi)) * Fraction(q0)
        assert oracle.quality_lower_bound(k0, kmin, kmax, xi, q0) == pytest.approx(float(exact), rel=1e-15, abs=1e-300)
        # monotone: raising k0 never raises b
        k0b = rng.uniform(k0, kmax)
        assert oracle.quality_lower_bound(k0b, kmin, kmax, xi, q0) <= oracle.quality_lower_bound(k0, kmin, kmax, xi, q0)
    # degenerate kmax == kmin: fraction defined as 0
    assert oracle.quality_lower_bound(77.0, 77.0, 77.0, 0.3, 0.6) == 0.6


def test_cost_vector_examples(golden):
    for c in golden["cost_vector"]["cases"]:
        got = oracle.cost_vector(c["k0"], c["pue"], c["k1"], c["e"], c["p"])
        np.testing.assert_allclose(got, c["c"], rtol=3e-16, atol=0, err_msg=c["cite"])


def test_cost_vector_terms_separately():
    # operational and embodied terms each appear with the right factor
    e = np.array([0.02, 0.01, 0.005]); p = np.array([3.0, 2.0, 1.0])
    c_op = oracle.cost_vector(200.0, 1.2, 0.0, e, p)
    np.testing.assert_allclose(c_op, 200.0 * 1.2 * e, rtol=3e-16)
    c_em = oracle.cost_vector(0.0, 1.2, 0.004, e, p)
    np.testing.assert_allclose(c_em, 0.004 * p, rtol=3e-16)
    c = oracle.cost_vector(200.0, 1.2, 0.004, e, p)
    np.testing.assert_allclose(c, c_op + c_em, rtol=3e-16)


# ------------------------------------------------------------- the LP


def _vertex_id(n, support):
    if len(support) == 1:
        return support[0]
    i, j = sorted(support)
    return n + [pair for pair in itertools.combinations(range(n), 2)].index((i, j))


def test_lp_worked_examples(golden):
    for c in golden["solve_lp"]["cases"]:
        x, obj, vid, st = oracle.solve_lp(c["c"], c["q"], c["b"])
        assert st == 0
        np.testing.assert_allclose(x, c["x"], rtol=0, atol=1e-15, err_msg=c["cite"])
        assert obj == pytest.approx(c["objective"], rel=1e-15), c["cite"]
        n = len(c["c"])
        kind, idx = c["vertex"].split("(")
        support = [int(v) for v in idx.rstrip(")").split(",")]
        assert vid == _vertex_id(n, support), c["cite"]


def _exact_lp(c, q, b):
    """Exact-rational vertex brute force: every feasible basic solution of
    {x >= 0, sum x = 1, q.x >= b}: pure e_i with q_i >= b, and for each pair
    the point of the edge with q.x = b."""
    n = len(c)
    C = [Fraction(v) for v in c]; Q = [Fraction(v) for v in q]; B = Fraction(b)
    best = None
    for i in range(n):
        if Q[i] >= B:
            val = C[i]
            if best is None or val < best:
                best = val
    for i, j in itertools.combinations(range(n), 2):
        if Q[i] == Q[j]:
            continue
        t = (B - Q[j]) / (Q[i] - Q[j])          # weight on i
        if 0 <= t <= 1:
            val = t * C[i] + (1 - t) * C[j]
            if best is None or val < best:
                best = val
    return best


def _random_instance(rng, n):
    c = rng.uniform(0, 3, n)
    q = rng.uniform(0, 1, n)
    if rng.random() < 0.2:                         # ties in q / c
        q[rng.integers(n)] = q[0]
    if rng.random() < 0.2:
        c[rng.integers(n)] = c[rng.integers(n)]
    b = rng.uniform(0, q.max())
    return c, q, b


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8])
def test_lp_vs_exact_rationals(n):
    rng = np.random.default_rng(100 + n)
    for _ in range(400):
        c, q, b = _random_instance(rng, n)
        x, obj, vid, st = oracle.solve_lp(c, q, b)
        exact = _exact_lp(c, q, b)
        assert st == 0 and exact is not None
        assert abs(Fraction(obj) - exact) <= Fraction(1, 10**15) * max(abs(exact), Fraction(1, 10**300)) + Fraction(1, 10**300)
        # the chosen x itself attains the objective (no transposed operands)
        xf = [Fraction(v) for v in x]
        val = sum(Fraction(ci) * xi for ci, xi in zip(c, xf))
        assert abs(val - exact) <= Fraction(4, 10**15) * max(abs(exact), 1)


def test_lp_vs_highs_dual_simplex():
    from scipy.optimize import linprog
    rng = np.random.default_rng(7)
    worst = 0.0
    for n in (2, 3, 4, 5, 8):
        for _ in range(150):
            c, q, b = _random_instance(rng, n)
            x, obj, vid, st = oracle.solve_lp(c, q, b)
            res = linprog(c, A_ub=-q[None, :], b_ub=[-b], A_eq=np.ones((1, n)), b_eq=[1.0],
                          bounds=[(0, 1)] * n, method="highs-ds")
            assert res.status == 0
            err = abs(obj - res.fun) / max(abs(res.fun), 1e-12)
            worst = max(worst, err)
            assert err <= 1e-12, (c, q, b, obj, res.fun)
    assert worst <= 1e-12


def test_lp_vs_simplex_grid():
    # LP <= grid <= LP + step*(max c - min c): rounding the edge weight of the
    # higher-q end up to the grid keeps feasibility (SPEC S:286's "1e-6" is
    # not a valid bound).
    rng = np.random.default_rng(9)
    steps = 1000
    i1, i2 = np.meshgrid(np.arange(steps + 1), np.arange(steps + 1), indexing="ij")
    mask = i1 + i2 <= steps
    X = np.stack([i1[mask], i2[mask], steps - i1[mask] - i2[mask]], axis=1) / steps
    for _ in range(30):
        c, q, b = _random_instance(rng, 3)
        x, obj, vid, st = oracle.solve_lp(c, q, b)
        feas = X @ q >= b - 1e-12
        grid = (X[feas] @ c).min()
        assert obj <= grid + 1e-12
        assert grid <= obj + (1.0 / steps) * (c.max() - c.min()) + 1e-12


def test_lp_invariants():
    rng = np.random.default_rng(11)
    for _ in range(3000):
        n = int(rng.integers(1, 9))
        c, q, b = _random_instance(rng, n)
        x, obj, vid, st = oracle.solve_lp(c, q, b)
        assert st == 0
        assert np.all(x >= 0.0)                       # x >= 0 exactly
        s = 0.0
        for v in x:
            s = s + v
        assert s == 1.0                               # sum x = 1 exactly (SURVEY 8c proof)
        assert float(np.dot(q, x)) >= b - 1e-15      # quality floor (Eq. 5)
        assert np.count_nonzero(x) <= 2              # basic solution
        # floor inactive => minimum-carbon level (north_star invariant)
        cmin = c.min()
        cand = [i for i in range(n) if c[i] == cmin and q[i] >= b]
        if cand:
            m = cand[0]
            assert vid == m and x[m] == 1.0 and obj == cmin


def test_lp_carbon_nonincreasing_in_xi():
    # relaxing xi (larger paper xi) lowers b, so the optimum never rises
    rng = np.random.default_rng(13)
    xis = np.arange(64) / 63.0
    for _ in range(300):
        n = int(rng.integers(2, 6))
        e = rng.uniform(1e-6, 3e-5, n); p = rng.uniform(0.05, 0.5, n)
        q = rng.dirichlet(np.ones(n))
        kmin = rng.uniform(5, 150); kmax = kmin + rng.uniform(100, 600); k0 = rng.uniform(kmin, kmax)
        c = oracle.cost_vector(k0, 1.2, 9.5e-4, e, p)
        prev = math.inf
        for xi in xis:
            b = oracle.quality_lower_bound(k0, kmin, kmax, xi, q[0])
            _, obj, _, st = oracle.solve_lp(c, q, b)
            assert st == 0
            assert obj <= prev
            prev = obj


def test_lp_scale_invariance():
    # S:288 scaling c by a positive power of two leaves the support unchanged
    rng = np.random.default_rng(17)
    for _ in range(500):
        n = int(rng.integers(2, 7))
        c, q, b = _random_instance(rng, n)
        x1, o1, v1, _ = oracle.solve_lp(c, q, b)
        x2, o2, v2, _ = oracle.solve_lp(c * 4.0, q, b)
        assert v1 == v2 and o2 == 4.0 * o1
        np.testing.assert_array_equal(x1, x2)


def test_lp_infeasible_is_reported():
    x, obj, vid, st = oracle.solve_lp([1.0, 2.0], [0.3, 0.4], 0.5)
    assert st == 2 and vid == 255 and math.isnan(obj)


# ------------------------------------------------------ thresholds / selector


def test_selector_worked_examples(golden):
    s = golden["selector"]
    T, ml = oracle.thresholds(s["x"])
    assert [int(v) for v in T] == s["thresholds"] and ml == s["max_level"]
    for c in s["cases"]:
        assert c["w"] == math.floor(c["u"] * 2**32)          # u = w 2^-32
        assert oracle.select_level(s["x"], c["w"]) == c["level"], c["cite"]
        assert oracle.select_level(s["x"], c["w"], pinned=True) == 0


def test_thresholds_exact_definition():
    # T_i = min(ceil(cum_i 2^32), 2^32) with cum_i the sequential fp64 sum:
    # compare with exact rational ceil of the same fp64 partial sums.
    rng = np.random.default_rng(19)
    for _ in range(2000):
        n = int(rng.integers(1, 9))
        c, q, b = _random_instance(rng, n)
        x, *_ = oracle.solve_lp(c, q, b)
        T, ml = oracle.thresholds(x)
        cum = 0.0
        want = []
        for i in range(n - 1):
            cum = cum + x[i]
            want.append(min(math.ceil(Fraction(cum) * 2**32), 2**32))
        assert [int(v) for v in T] == want
        sat = [i for i, t in enumerate(want) if t == 2**32]
        assert ml == (sat[0] if sat else n - 1)


def test_selector_threshold_form_equivalence():
    # the saturated-u32 + max_level form used by the kernel equals the
    # inverse-CDF definition, on random, degenerate and +-1 boundary words
    rng = np.random.default_rng(23)
    for _ in range(300):
        n = int(rng.integers(1, 9))
        c, q, b = _random_instance(rng, n)
        x, *_ = oracle.solve_lp(c, q, b)
        if rng.random() < 0.1:
            x = np.zeros(n); x[rng.integers(n)] = 1.0
        T, ml = oracle.thresholds(x)
        T32 = [min(int(t), 0xFFFFFFFF) for t in T]
        words = list(rng.integers(0, 2**32, 20)) + [0, 1, 2**32 - 1, 2**31]
        for t in T32:
            words += [max(t - 1, 0), t, min(t + 1, 2**32 - 1)]
        for w in words:
            w = int(w)
            cnt = sum(1 for t in T32 if w >= t)
            assert oracle.select_level(x, w) == min(cnt, ml)


def test_selector_frequencies_evenly_spaced():
    # frequencies over evenly spaced u match x within 1e-3
    x = [0.5, 0.3, 0.2]
    N = 200_000
    counts = np.zeros(3)
    for k in range(N):
        w = (k * 2**32) // N
        counts[oracle.select_level(x, w)] += 1
    np.testing.assert_allclose(counts / N, x, atol=1e-3)


def test_selector_degenerate_policies():
    for n in range(1, 9):
        for k in range(n):
            x = np.zeros(n); x[k] = 1.0
            for w in (0, 1, 2**31, 2**32 - 1):
                assert oracle.select_level(x, w) == k


def test_normalized_preference_context(golden):
    # w/(1-w): context pin for reading L15
    for c in golden["normalized_preference"]["cases"]:
        assert c["w"] / (1 - c["w"]) == pytest.approx(c["score"], abs=c["tol"]), c["cite"]
