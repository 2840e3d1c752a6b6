"""The C-ABI library loads and exports every symbol include/sprout.h declares;
host-side validation rejects bad arguments before touching a device (CPU)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sprout.h")
LIB = os.path.join(ROOT, "paper_2403_12900_b200", "libsprout.so")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sprout_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2403_12900_b200 import build
        build.build()
    return C.CDLL(LIB)


def test_header_declares_the_hot_path():
    fns = declared_functions()
    for name in ("sprout_solve_directives", "sprout_simulate_trace", "sprout_reduce_totals"):
        assert name in fns


def test_every_declared_symbol_is_exported(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_binding_covers_every_export():
    from paper_2403_12900_b200 import sprout as S
    assert sorted(S.EXPORTS) == declared_functions()


def test_struct_layouts_match_header():
    from paper_2403_12900_b200 import sprout as S
    # field offsets implied by the C declarations (LP64)
    assert C.sizeof(S.LpProblem) == 4 + 4 + 8 + 4 + 4 + 7 * 8 + 8 + 8 + 8 + 8
    assert S.LpProblem.n_intervals.offset == 8 and S.LpProblem.k0.offset == 24
    assert C.sizeof(S.CostModel) == 16 + 4 * 4 * 8 * 8
    assert S.CostModel.ef.offset == 16
    assert C.sizeof(S.Trace) == 48 and C.sizeof(S.CellTotals) == 11 * 8
    assert C.sizeof(S.TraceGenerator) == 8 + 8 + 8 + 4 + 4 + 4 + 4 + 8 + 8


def test_status_strings(lib):
    lib.sprout_status_string.restype = C.c_char_p
    assert lib.sprout_status_string(0) == b"ok"
    assert lib.sprout_status_string(1) == b"invalid argument"
    lib.sprout_group_stat_count.restype = C.c_int32
    assert lib.sprout_group_stat_count(3) == 17


def _problem(S, **kw):
    d = dict(n_levels=3, n_regions=1, n_intervals=2, n_xi=1, profile_per_interval=0,
             k0=16, k0_min=16, k0_max=16, xi=16, e=16, p=16, q=16, k1=0.001, pue=1.2,
             first_segment=0, n_segments=2)
    d.update(kw)
    return S.LpProblem(*[d[f[0]] for f in S.LpProblem._fields_])


@pytest.mark.parametrize("field,value", [("n_levels", 0), ("n_levels", 9), ("n_regions", 0), ("n_xi", 0),
                                         ("n_xi", 5000), ("pue", 0.9), ("pue", float("nan")), ("k1", -1.0),
                                         ("n_segments", 3), ("first_segment", -1), ("k0", None)])
def test_host_validation_rejects_without_device(field, value):
    from paper_2403_12900_b200 import sprout as S
    P = _problem(S, **{field: value})
    sol = S.LpSolution(16, 16, 16, 16, 16, 16, 16)
    st = S._lib.sprout_solve_directives(C.byref(P), C.byref(sol), None)
    assert st == 1
    assert S._lib.sprout_workspace_bytes(C.byref(P), None) == 0


def test_trace_validation_rejects_without_device():
    from paper_2403_12900_b200 import sprout as S
    P = _problem(S)
    sol = S.LpSolution(16, 16, 16, 16, 16, 16, 16)
    cost = S.CostModel(); cost.n_classes = 1
    tot = S.CellTotals(*([16] * 11))
    for tr in (S.Trace(10, 4, 16, 16, 16, None),       # first_request not a multiple of 8
               S.Trace(10, 0, 16, 16, 12, None),       # pitch not a multiple of 8
               S.Trace(20, 0, 16, 16, 16, None),       # pitch < n_requests
               S.Trace(10, 0, 16, 18, 16, None),       # misaligned tokens
               S.Trace(10, 0, None, 16, 16, None)):    # no offsets
        st = S._lib.sprout_simulate_trace(C.byref(P), C.byref(sol), C.byref(tr), C.byref(cost), C.byref(tot),
                                          None, 256, 1 << 20, None)
        assert st == 1
    cost.n_classes = 5
    st = S._lib.sprout_simulate_trace(C.byref(P), C.byref(sol), C.byref(S.Trace(10, 0, 16, 16, 16, None)),
                                      C.byref(cost), C.byref(tot), None, 256, 1 << 20, None)
    assert st == 1


def test_workspace_size_monotone():
    from paper_2403_12900_b200 import sprout as S
    a = S._lib.sprout_workspace_bytes(C.byref(_problem(S, n_segments=1)), None)
    b = S._lib.sprout_workspace_bytes(C.byref(_problem(S, n_segments=2)), None)
    c = S._lib.sprout_workspace_bytes(C.byref(_problem(S, n_xi=64, n_segments=2)), None)
    assert 0 < a <= b < c


def test_static_grid_size_closed_form():
    """sprout_static_grid_size = C(D + n - 1, n - 1) (stars and bars), -1 past SPROUT_MAX_XI."""
    import math
    from paper_2403_12900_b200 import sprout as S
    for n in range(1, 9):
        for D in range(1, 40):
            g = math.comb(D + n - 1, n - 1)
            assert S.static_grid_size(n, D) == (g if g <= S.MAX_XI else -1), (n, D)
    assert S.static_grid_size(0, 5) == -1 and S.static_grid_size(3, 0) == -1


def test_scheme_validation_rejects_without_device():
    from paper_2403_12900_b200 import sprout as S
    sol = S.LpSolution(16, 16, 16, 16, 16, 16, 16)
    P = _problem(S)
    assert S._lib.sprout_solve_scheme(C.byref(P), 7, 0, C.byref(sol), None) == 1          # unknown scheme
    assert S._lib.sprout_solve_scheme(C.byref(P), 2, 0, C.byref(sol), None) == 1          # grid_den < 1
    assert S._lib.sprout_solve_scheme(C.byref(P), 2, 20, C.byref(sol), None) == 1         # n_xi != 231
    assert S._lib.sprout_solve_scheme(C.byref(_problem(S, pue=0.5)), 1, 0, C.byref(sol), None) == 1
    G = _problem(S, n_xi=231)
    assert S._lib.sprout_select_static(C.byref(G), 20, 1.5, 16, 16, 16, None) == 1       # xi > 1
    assert S._lib.sprout_select_static(C.byref(G), 19, 0.1, 16, 16, 16, None) == 1       # wrong grid
    assert S._lib.sprout_select_static(C.byref(G), 20, 0.1, None, 16, 16, None) == 1     # NULL totals
    assert S._lib.sprout_select_static(C.byref(_problem(S, n_xi=231, profile_per_interval=1)), 20, 0.1,
                                       16, 16, 16, None) == 1


def test_evaluator_validation_rejects_without_device():
    from paper_2403_12900_b200 import sprout as S
    b = (C.c_double * 2)(0.028, 0.0)
    t = (C.c_double * 2)(0.5, 0.3)

    def P(**kw):
        d = dict(n_regions=1, n_beta=2, n_intervals=24, interval_hours=1.0, k2=16, k2_max=16,
                 beta=C.addressof(b), n_theta=2, fallback=3, theta=C.addressof(t), grace_hours=6.0,
                 eval_kwh=0.28, pue=1.2)
        d.update(kw)
        return S.EvaluatorProblem(*[d[f[0]] for f in S.EvaluatorProblem._fields_])
    for kw in (dict(n_regions=0), dict(n_beta=0), dict(n_beta=65), dict(n_theta=0), dict(interval_hours=0.0),
               dict(grace_hours=-1.0), dict(fallback=-1), dict(pue=0.9), dict(eval_kwh=float("nan")),
               dict(k2=None), dict(beta=None)):
        assert S._lib.sprout_evaluator_sweep(C.byref(P(**kw)), 16, None) == 1, kw
    bad = (C.c_double * 2)(-0.1, 0.0)
    assert S._lib.sprout_evaluator_sweep(C.byref(P(beta=C.addressof(bad))), 16, None) == 1
