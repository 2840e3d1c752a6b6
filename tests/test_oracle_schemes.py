"""Oracle pins for the competing schemes of the evaluation (
SURVEY 8(f) NEXT-3): CO2_Opt's argmin, the Sprout_Sta simplex grid and its
selection rule -- each checked against something other than the oracle's
own code (brute force in Python, stars-and-bars counts, the LP with its
quality constraint removed, worked examples)."""
import dataclasses
import itertools
import math

import numpy as np
import pytest

import oracle
import synth


def test_co2opt_worked_example_and_ties():
    # CO2Opt with c = [3, 1.5, 1] -> 2 ("lowest carbon footprint")
    assert oracle.co2opt_level([3.0, 1.5, 1.0]) == 2
    assert oracle.co2opt_level([1.0, 1.0, 2.0]) == 0      # reading L17: ties to the lowest index
    assert oracle.co2opt_level([2.0, 1.0, 1.0]) == 1
    assert oracle.co2opt_level([5.0]) == 0


def test_co2opt_is_the_lp_without_its_quality_floor():
    """Dropping constraint (5) (b = 0 <= q.x always) leaves min c.x over the
    simplex, attained at the cheapest pure level: the LP solver and the argmin
    agree, and both equal a brute-force minimum."""
    rng = np.random.default_rng(11)
    for _ in range(2000):
        n = int(rng.integers(1, 9))
        c = rng.choice([0.5, 1.0, 1.5, 2.0], n) if rng.random() < 0.3 else rng.random(n)
        q = rng.random(n)
        m = oracle.co2opt_level(c)
        assert m == min(range(n), key=lambda i: (c[i], i))
        x, obj, vid, st = oracle.solve_lp(c, q, 0.0)
        assert st == 0 and vid == m and obj == c[m]


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5])
def test_grid_is_the_simplex_lattice_in_stated_order(n):
    for D in (1, 2, 3, 5, 20 if n <= 3 else 6):
        pts = [k for k in itertools.product(range(D, -1, -1), repeat=n) if sum(k) == D]   # k_0 desc, then k_1 desc
        assert oracle.grid_size(n, D) == len(pts) == math.comb(D + n - 1, n - 1)
        for j, k in enumerate(pts):
            x = oracle.grid_point(n, D, j)
            np.testing.assert_array_equal(x, np.array(k, float) / D)
        with pytest.raises(IndexError):
            oracle.grid_point(n, D, len(pts))
    # grid step 1 -> the candidates are the pure levels only
    assert [tuple(oracle.grid_point(n, 1, j)) for j in range(n)] == [tuple(np.eye(n)[i]) for i in range(n)]


def _static_problem(w, D):
    G = oracle.grid_size(w.prob.n, D)
    return dataclasses.replace(w.prob, X=G, xi=np.zeros(G)), G


def _small_workload():
    return synth.make_workload("C2", n_requests=20000, n_intervals=48)


def test_scheme_cells():
    w = _small_workload()
    prob = w.prob
    co2 = oracle.solve_cells(prob, scheme=oracle.SCHEME_CO2_OPT)
    sp = oracle.solve_cells(prob)
    S = prob.R * prob.T
    for s in range(S):
        r = s // prob.T
        c = oracle.cost_vector(prob.k0[s], prob.pue, prob.k1, prob.e[r], prob.p[r])
        for j in range(prob.X):
            cell = s * prob.X + j
            m = min(range(prob.n), key=lambda i: (c[i], i))
            np.testing.assert_array_equal(co2["x"][cell], np.eye(prob.n)[m])
            assert co2["vertex"][cell] == m and co2["objective"][cell] == c[m]
            assert co2["q_lb"][cell] == prob.q[r][m]
            # the unconstrained optimum is never dearer than the Sprout LP's (P:368 vs P:197)
            assert co2["objective"][cell] <= sp["objective"][cell]
    D = 4
    sprob, G = _static_problem(w, D)
    st = oracle.solve_cells(sprob, scheme=oracle.SCHEME_STATIC_GRID, grid_den=D)
    for s in range(0, S, 7):
        r = s // prob.T
        c = oracle.cost_vector(prob.k0[s], prob.pue, prob.k1, prob.e[r], prob.p[r])
        for j in range(G):
            cell = s * G + j
            x = oracle.grid_point(prob.n, D, j)
            np.testing.assert_array_equal(st["x"][cell], x)
            assert st["cell_status"][cell] == 0
            assert st["objective"][cell] == pytest.approx(float(np.dot(c, x)), rel=1e-15)
            assert st["q_lb"][cell] == pytest.approx(float(np.dot(prob.q[r], x)), rel=1e-15)
            T, ml = oracle.thresholds(x)
            np.testing.assert_array_equal(st["threshold"][cell], T)
            nz = np.flatnonzero(x)
            assert st["vertex"][cell] == (nz[0] if len(nz) == 1 else 254)
    with pytest.raises(ValueError):
        oracle.solve_cells(sprob, scheme=oracle.SCHEME_STATIC_GRID, grid_den=D + 1)   # G mismatch


def test_select_static_brute_force():
    """The Sprout_Sta choice equals a brute-force scan of the sweep's totals
    (floor: Eq. 3 at the mean intensity, via the pinned quality_lower_bound)."""
    w = _small_workload()
    D = 5
    sprob, G = _static_problem(w, D)
    sh = synth.shard(w.spec, 1, 0)
    toks, flags = synth.host_trace(w.spec, sh)
    seg = np.arange(sprob.R * sprob.T)
    sim = oracle.simulate(sprob, w.cost, seg, sh.seg_offsets[:-1], np.diff(sh.seg_offsets),
                          sh.first_request + sh.seg_offsets[:-1], toks, flags,
                          scheme=oracle.SCHEME_STATIC_GRID, grid_den=D)
    cells = oracle.solve_cells(sprob, scheme=oracle.SCHEME_STATIC_GRID, grid_den=D)
    group = oracle.reduce(sprob, w.cost.n_classes, 0, sprob.R * sprob.T, cells, sim)
    n, K = sprob.n, 11 + 2 * sprob.n
    for xi in (0.0, 0.1, 0.5, 1.0):
        choice, x = oracle.select_static(sprob, xi, D, group)
        for r in range(sprob.R):
            kbar = math.fsum(sprob.k0[r * sprob.T:(r + 1) * sprob.T]) / sprob.T
            b = oracle.quality_lower_bound(kbar, sprob.kmin[r], sprob.kmax[r], xi, sprob.q[r][0])
            feas = []
            for g in range(G):
                S_ = group[r, g]
                Q = sum(S_[11 + L] * sprob.q[r][L] for L in range(n))
                if Q >= b * S_[0] * (1 + 1e-12):
                    feas.append(g)
                elif Q >= b * S_[0] * (1 - 1e-12):
                    feas.append(g)    # boundary: rounding-order dependent, accepted either way
            assert 0 in feas                               # pure L0 always meets the floor
            assert choice[r] in feas
            best = min(group[r, g, 4] for g in feas)
            assert group[r, choice[r], 4] <= best * (1 + 1e-12)
            np.testing.assert_array_equal(x[r], oracle.grid_point(n, D, int(choice[r])))
        if xi == 0.0:
            # xi = 0: the floor is q0 itself, so only mixes as good as pure L0 qualify
            for r in range(sprob.R):
                S_ = group[r, choice[r]]
                assert sum(S_[11 + L] * sprob.q[r][L] for L in range(n)) >= S_[0] * sprob.q[r][0] * (1 - 1e-12)
