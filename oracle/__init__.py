"""CPU oracle for the Sprout hot path -- TEST INFRASTRUCTURE ONLY.

Plain, slow, independent implementation of arXiv 2403.12900's directive
optimiser (Eqs. 2-7), directive selector and carbon
accounting (Eq. 1), written in C (``sprout_oracle.c``, fp64,
-ffp-contract=off) and loaded here with ctypes.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  It
shares nothing with ``paper_2403_12900_b200`` and never imports it; its inputs
come from ``synth`` (seeded input generation, none of the method's
arithmetic) or from literals in the tests.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sprout_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math", "-pthread"]


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C11, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            _lib = _bind(C.CDLL(build()))
    return _lib


_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)
_u32p = C.POINTER(C.c_uint32)
_u16p = C.POINTER(C.c_uint16)
_u8p = C.POINTER(C.c_uint8)
_ip = C.POINTER(C.c_int)


def _bind(L):
    L.orc_philox4x32_10.argtypes = [_u32p, _u32p, _u32p]
    L.orc_philox4x32_10.restype = None
    L.orc_draw_word.argtypes = [C.c_uint64, C.c_uint64]
    L.orc_draw_word.restype = C.c_uint32
    L.orc_quality_lower_bound.argtypes = [C.c_double] * 5
    L.orc_quality_lower_bound.restype = C.c_double
    L.orc_cost_vector.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, _dp, _dp, _dp]
    L.orc_cost_vector.restype = None
    L.orc_request_carbon.argtypes = [C.c_double] * 4
    L.orc_request_carbon.restype = C.c_double
    L.orc_solve_lp.argtypes = [C.c_int, _dp, _dp, C.c_double, _dp, _dp, _ip]
    L.orc_solve_lp.restype = C.c_int
    L.orc_thresholds.argtypes = [C.c_int, _dp, _u64p, _ip]
    L.orc_thresholds.restype = None
    L.orc_select_level.argtypes = [C.c_int, _dp, C.c_uint32, C.c_int]
    L.orc_select_level.restype = C.c_int
    L.orc_solve_cells.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                  C.c_int, C.c_double, C.c_double, C.c_int64, C.c_int64,
                                  _dp, _dp, _dp, _u8p, _u64p, _u8p, _u8p]
    L.orc_solve_cells.restype = C.c_int
    L.orc_simulate.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                               C.c_int, C.c_double, C.c_double,
                               C.c_uint64, C.c_int, _dp, _dp, _dp, _dp,
                               C.c_int64, _i64p, _i64p, _i64p, _u64p,
                               _u16p, C.c_int64, _u8p,
                               _u64p, _u64p, _dp, _dp, _dp, _dp,
                               _u64p, _u64p, _u64p, _dp, _u8p, C.c_int, _i64p]
    L.orc_simulate.restype = C.c_int
    L.orc_reduce.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int64, C.c_int64,
                             _u8p, _dp, _u64p, _u64p, _dp, _dp, _dp, _dp, _u64p, _u64p, _dp, _dp]
    L.orc_reduce.restype = C.c_int
    L.orc_solve_cells_scheme.argtypes = L.orc_solve_cells.argtypes + [C.c_int, C.c_int]
    L.orc_solve_cells_scheme.restype = C.c_int
    L.orc_simulate_scheme.argtypes = L.orc_simulate.argtypes + [C.c_int, C.c_int]
    L.orc_simulate_scheme.restype = C.c_int
    L.orc_co2opt_level.argtypes = [C.c_int, _dp]
    L.orc_co2opt_level.restype = C.c_int
    L.orc_grid_size.argtypes = [C.c_int, C.c_int]
    L.orc_grid_size.restype = C.c_int64
    L.orc_grid_point.argtypes = [C.c_int, C.c_int, C.c_int64, _dp]
    L.orc_grid_point.restype = C.c_int
    L.orc_select_static.argtypes = [C.c_int, C.c_int, C.c_int64, _dp, _dp, _dp, _dp, C.c_double, C.c_int,
                                    C.c_int64, _dp, C.POINTER(C.c_int32), _dp]
    L.orc_select_static.restype = C.c_int
    L.orc_evaluator_sweep.argtypes = [C.c_int, C.c_int64, C.c_double, _dp, _dp, C.c_int, _dp, C.c_int, _dp,
                                      C.c_double, C.c_int, C.c_double, C.c_double, _dp]
    L.orc_evaluator_sweep.restype = C.c_int
    L.orc_closed_loop.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                  C.c_double, C.c_double, C.c_uint64, C.c_int, _dp, _dp, _dp, _dp, C.c_int, _dp,
                                  _i64p, _u16p, C.c_int64, _u8p, _dp, _u64p, _u8p, _dp, _dp, _u64p, _u64p, _dp, _dp,
                                  _dp, _dp]
    L.orc_closed_loop.restype = C.c_int
    L.orc_evaluation_q.argtypes = [C.c_int, C.c_int64, C.c_double, _dp, _dp, C.c_double, C.c_double, C.c_double,
                                   C.c_int, C.c_int, _dp, C.c_uint64, _i64p, C.c_int, _dp, _u8p]
    L.orc_evaluation_q.restype = C.c_int
    L.orc_pref_word.argtypes = [C.c_uint64, C.c_uint64]
    L.orc_pref_word.restype = C.c_uint32
    L.orc_pref_level.argtypes = [C.c_int, _dp, C.c_uint64, C.c_uint64]
    L.orc_pref_level.restype = C.c_int
    L.orc_normalized_preference.argtypes = [C.c_double]
    L.orc_normalized_preference.restype = C.c_double
    L.orc_head_to_head.argtypes = [C.c_int, C.c_int, _ip, _ip]
    L.orc_head_to_head.restype = None
    L.orc_preference.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                 C.c_int, C.c_double, C.c_double, C.c_uint64, C.c_int, _i64p, _u64p, _u8p, C.c_int,
                                 C.c_int, _u64p]
    L.orc_preference.restype = C.c_int
    L.orc_request_outputs.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                      C.c_int, C.c_double, C.c_double, C.c_uint64, C.c_int, _dp, _dp, _dp, _dp,
                                      _i64p, _u64p, _u16p, C.c_int64, _u8p, C.c_int, C.c_int, C.c_int,
                                      _u8p, _dp, _dp, _dp, _u8p]
    L.orc_request_outputs.restype = C.c_int
    L.orc_oracle_scheme.argtypes = [C.c_int, C.c_int, C.c_int64, C.c_int, _dp, _dp, _dp, _dp, _dp, C.c_int,
                                    C.c_double, C.c_double, C.c_uint64, C.c_int, _dp, _dp, _dp, _dp,
                                    _i64p, _u64p, _u16p, C.c_int64, _u8p, _u64p, _u64p, _dp, _dp, _dp, _dp, _u64p,
                                    _u8p]
    L.orc_oracle_scheme.restype = C.c_int
    return L


def _p(a, t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# --------------------------------------------------------------------------
# scalar / small-vector entry points (one call per definition in the paper)

def philox4x32_10(ctr, key):
    c = np.ascontiguousarray(np.asarray(ctr, dtype=np.uint32))
    k = np.ascontiguousarray(np.asarray(key, dtype=np.uint32))
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_p(c, _u32p), _p(k, _u32p), _p(out, _u32p))
    return out


def draw_word(seed: int, g: int) -> int:
    return int(lib().orc_draw_word(seed, g))


def quality_lower_bound(k0, kmin, kmax, xi, q0) -> float:
    return lib().orc_quality_lower_bound(k0, kmin, kmax, xi, q0)


def cost_vector(k0, pue, k1, e, p):
    e = _f64(e); p = _f64(p)
    c = np.zeros(len(e))
    lib().orc_cost_vector(len(e), k0, pue, k1, _p(e, _dp), _p(p, _dp), _p(c, _dp))
    return c


def request_carbon(kp, k1, energy_kwh, time_s) -> float:
    return lib().orc_request_carbon(kp, k1, energy_kwh, time_s)


def solve_lp(c, q, b):
    """Returns (x, objective, vertex_id, status)."""
    c = _f64(c); q = _f64(q)
    n = len(c)
    x = np.zeros(n)
    obj = C.c_double(0.0)
    vid = C.c_int(0)
    st = lib().orc_solve_lp(n, _p(c, _dp), _p(q, _dp), float(b), _p(x, _dp), C.byref(obj), C.byref(vid))
    return x, obj.value, vid.value, st


def thresholds(x):
    """Returns (T as uint64 values up to 2**32, max_level)."""
    x = _f64(x)
    n = len(x)
    T = np.zeros(max(n - 1, 1), np.uint64)
    ml = C.c_int(0)
    lib().orc_thresholds(n, _p(x, _dp), _p(T, _u64p), C.byref(ml))
    return T[: n - 1], ml.value


def select_level(x, w: int, pinned: bool = False) -> int:
    x = _f64(x)
    return int(lib().orc_select_level(len(x), _p(x, _dp), int(w) & 0xFFFFFFFF, int(bool(pinned))))


# competing schemes: scheme ids as in the C-ABI
SCHEME_SPROUT, SCHEME_CO2_OPT, SCHEME_STATIC_GRID = 0, 1, 2


def co2opt_level(c) -> int:
    c = _f64(c)
    return int(lib().orc_co2opt_level(len(c), _p(c, _dp)))


def grid_size(n: int, D: int) -> int:
    return int(lib().orc_grid_size(n, D))


def grid_point(n: int, D: int, j: int):
    x = np.zeros(n)
    if lib().orc_grid_point(n, D, j, _p(x, _dp)) != 0:
        raise IndexError(j)
    return x


def select_static(prob, xi: float, grid_den: int, group):
    """Sprout_Sta choice per region from a sweep's group totals [R+1][G][K]."""
    n, R, T = prob.n, prob.R, prob.T
    assert not prob.profile_per_interval
    G = group.shape[1]
    group = np.ascontiguousarray(group, np.float64)
    choice = np.zeros(R, np.int32)
    x = np.zeros((R, n))
    st = lib().orc_select_static(n, R, int(T), _p(_f64(prob.k0), _dp), _p(_f64(prob.kmin), _dp),
                                 _p(_f64(prob.kmax), _dp), _p(_f64(prob.q), _dp), float(xi), int(grid_den),
                                 int(G), _p(group, _dp), choice.ctypes.data_as(C.POINTER(C.c_int32)), _p(x, _dp))
    if st != 0:
        raise ValueError("oracle select_static: invalid argument")
    return choice, x


# --------------------------------------------------------------------------
# whole-problem entry points.  `prob` is a synth.Problem, `cost` a
# synth.CostModel (plain containers of numpy arrays).

def _prob_args(prob):
    return (int(prob.n), int(prob.R), int(prob.T), int(prob.X),
            _p(prob.k0, _dp), _p(prob.kmin, _dp), _p(prob.kmax, _dp), _p(prob.xi, _dp),
            _p(prob.e, _dp), _p(prob.p, _dp), _p(prob.q, _dp), int(prob.profile_per_interval),
            float(prob.k1), float(prob.pue))


def solve_cells(prob, first_segment: int = 0, n_segments: int | None = None, scheme: int = 0, grid_den: int = 0):
    if n_segments is None:
        n_segments = prob.R * prob.T - first_segment
    n, X = prob.n, prob.X
    cells = n_segments * X
    out = dict(
        x=np.zeros((cells, n)), objective=np.zeros(cells), q_lb=np.zeros(cells),
        vertex=np.zeros(cells, np.uint8), threshold=np.zeros((cells, max(n - 1, 1)), np.uint64),
        max_level=np.zeros(cells, np.uint8), cell_status=np.zeros(cells, np.uint8))
    a = _prob_args(prob)
    st = lib().orc_solve_cells_scheme(*a, int(first_segment), int(n_segments),
                                      _p(out["x"], _dp), _p(out["objective"], _dp), _p(out["q_lb"], _dp),
                                      _p(out["vertex"], _u8p), _p(out["threshold"], _u64p),
                                      _p(out["max_level"], _u8p), _p(out["cell_status"], _u8p),
                                      int(scheme), int(grid_den))
    if st != 0:
        raise ValueError(f"oracle solve_cells: invalid argument (status {st})")
    out["threshold"] = out["threshold"][:, : n - 1]
    return out


def simulate(prob, cost, seg_id, req_begin, seg_m, g0, tokens, flags=None,
             levels: bool = False, threads: int | None = None, scheme: int = 0, grid_den: int = 0):
    """Replay the requests of the listed segments.

    seg_id[k]   global segment index r*T + t
    req_begin[k] index of the segment's first request in `tokens`/`flags`
    seg_m[k]    number of requests of the segment
    g0[k]       global request index of that first request (Philox counter)
    tokens      uint16 [n][pitch];  flags uint8 [pitch] or None
    """
    n, X, NC = prob.n, prob.X, cost.n_classes
    seg_id = np.ascontiguousarray(seg_id, dtype=np.int64)
    req_begin = np.ascontiguousarray(req_begin, dtype=np.int64)
    seg_m = np.ascontiguousarray(seg_m, dtype=np.int64)
    g0 = np.ascontiguousarray(g0, dtype=np.uint64)
    tokens = np.ascontiguousarray(tokens, dtype=np.uint16)
    assert tokens.ndim == 2 and tokens.shape[0] >= n
    pitch = tokens.shape[1]
    if flags is not None:
        flags = np.ascontiguousarray(flags, dtype=np.uint8)
        assert flags.shape[0] >= pitch or flags.shape[0] == pitch
    k = len(seg_id)
    out = dict(
        cnt=np.zeros((k, X, NC, n), np.uint64), tok=np.zeros((k, X, NC, n), np.uint64),
        energy=np.zeros((k, X)), time=np.zeros((k, X)), carbon=np.zeros((k, X)), quality=np.zeros((k, X)),
        seg_count=np.zeros((k, NC), np.uint64), seg_pinned=np.zeros((k, NC), np.uint64),
        seg_tok=np.zeros((k, NC, n), np.uint64), seg_base=np.zeros((k, 4)))
    lv = np.full((X, pitch), 0xFF, np.uint8) if levels else None
    bad = C.c_int64(0)
    if threads is None:
        threads = os.cpu_count() or 1
    ef = _f64(cost.ef); et = _f64(cost.et); pf = _f64(cost.pf); pt = _f64(cost.pt)
    st = lib().orc_simulate_scheme(*_prob_args(prob), C.c_uint64(int(cost.seed)), int(NC),
                            _p(ef, _dp), _p(et, _dp), _p(pf, _dp), _p(pt, _dp),
                            int(k), _p(seg_id, _i64p), _p(req_begin, _i64p), _p(seg_m, _i64p), _p(g0, _u64p),
                            _p(tokens, _u16p), int(pitch), _p(flags, _u8p),
                            _p(out["cnt"], _u64p), _p(out["tok"], _u64p), _p(out["energy"], _dp),
                            _p(out["time"], _dp), _p(out["carbon"], _dp), _p(out["quality"], _dp),
                            _p(out["seg_count"], _u64p), _p(out["seg_pinned"], _u64p),
                            _p(out["seg_tok"], _u64p), _p(out["seg_base"], _dp),
                            _p(lv, _u8p), int(threads), C.byref(bad), int(scheme), int(grid_den))
    if st != 0:
        raise ValueError(f"oracle simulate: invalid argument (status {st})")
    out["bad_requests"] = bad.value
    if levels:
        out["levels"] = lv
    return out


def reduce(prob, n_classes, first_segment, n_segments, cells, sim):
    """Group totals [R+1][X][K] (last row = global) from this oracle's own
    solve_cells() and simulate() results over ALL local segments."""
    n, R, X = prob.n, prob.R, prob.X
    K = 11 + 2 * n
    out = np.zeros((R + 1, X, K))
    cs = np.ascontiguousarray(cells["cell_status"], np.uint8)
    obj = np.ascontiguousarray(cells["objective"], np.float64)
    st = lib().orc_reduce(n, R, int(prob.T), X, int(n_classes), int(first_segment), int(n_segments),
                          _p(cs, _u8p), _p(obj, _dp), _p(sim["cnt"], _u64p), _p(sim["tok"], _u64p),
                          _p(sim["energy"], _dp), _p(sim["time"], _dp), _p(sim["carbon"], _dp),
                          _p(sim["quality"], _dp), _p(sim["seg_count"], _u64p),
                          _p(sim["seg_pinned"], _u64p), _p(sim["seg_base"], _dp), _p(out, _dp))
    assert st == 0
    return out


def evaluator_sweep(k2, k2max, T: int, dt: float, betas, thetas, grace: float, fallback: int,
                    eval_kwh: float, pue: float):
    """Opportunistic evaluator trigger sweep (Eq. 8): out[R][B][H][4]."""
    k2 = _f64(k2); k2max = _f64(k2max); betas = _f64(betas); thetas = _f64(thetas)
    R = len(k2max)
    assert k2.size == R * T
    out = np.zeros((R, len(betas), len(thetas), 4))
    st = lib().orc_evaluator_sweep(R, int(T), float(dt), _p(k2, _dp), _p(k2max, _dp), len(betas), _p(betas, _dp),
                                   len(thetas), _p(thetas, _dp), float(grace), int(fallback), float(eval_kwh),
                                   float(pue), _p(out, _dp))
    if st != 0:
        raise ValueError("oracle evaluator_sweep: invalid argument")
    return out


def closed_loop(prob, cost, window: int, seg_offsets, tokens, flags=None, q_seg=None):
    """Closed-loop profiles (NEXT-1): per (region, xi) chain, the LP of
    each interval uses the mean E and T of the last `window` requests run at
    each level.  Requests are global: tokens [n][pitch] indexed by the global
    request index, seg_offsets [R*T+1] global."""
    n, R, T, X, NC = prob.n, prob.R, prob.T, prob.X, cost.n_classes
    assert not prob.profile_per_interval
    tokens = np.ascontiguousarray(tokens, dtype=np.uint16)
    off = np.ascontiguousarray(seg_offsets, dtype=np.int64)
    fl = None if flags is None else np.ascontiguousarray(flags, dtype=np.uint8)
    cells = R * T * X
    out = dict(x=np.zeros((cells, n)), threshold=np.zeros((cells, max(n - 1, 1)), np.uint64),
               cell_status=np.zeros(cells, np.uint8), objective=np.zeros(cells), profile=np.zeros((cells, 2, n)),
               cnt=np.zeros((cells, NC, n), np.uint64),
               tok=np.zeros((cells, NC, n), np.uint64), energy=np.zeros(cells), time=np.zeros(cells),
               carbon=np.zeros(cells), quality=np.zeros(cells))
    ef = _f64(cost.ef); et = _f64(cost.et); pf = _f64(cost.pf); pt = _f64(cost.pt)
    st = lib().orc_closed_loop(n, R, int(T), X, _p(_f64(prob.k0), _dp), _p(_f64(prob.kmin), _dp),
                               _p(_f64(prob.kmax), _dp), _p(_f64(prob.xi), _dp), _p(_f64(prob.e), _dp),
                               _p(_f64(prob.p), _dp), _p(_f64(prob.q), _dp), float(prob.k1), float(prob.pue),
                               C.c_uint64(int(cost.seed)), NC, _p(ef, _dp), _p(et, _dp), _p(pf, _dp), _p(pt, _dp),
                               int(window), _p(None if q_seg is None else _f64(q_seg), _dp),
                               _p(off, _i64p), _p(tokens, _u16p), tokens.shape[1], _p(fl, _u8p),
                               _p(out["x"], _dp), _p(out["threshold"], _u64p), _p(out["cell_status"], _u8p),
                               _p(out["objective"], _dp), _p(out["profile"], _dp), _p(out["cnt"], _u64p), _p(out["tok"], _u64p), _p(out["energy"], _dp),
                               _p(out["time"], _dp), _p(out["carbon"], _dp), _p(out["quality"], _dp))
    if st != 0:
        raise ValueError("oracle closed_loop: invalid argument")
    out["threshold"] = out["threshold"][:, : n - 1]
    return out


# --------------------------------------------------------------------------
# NEXT-4: latent preference, head-to-head preference, per-request outputs,
# the Oracle scheme (readings L21-L23)

def pref_word(seed: int, g: int) -> int:
    return int(lib().orc_pref_word(C.c_uint64(int(seed)), C.c_uint64(int(g))))


def pref_level(q, seed: int, g: int) -> int:
    q = _f64(q)
    return int(lib().orc_pref_level(len(q), _p(q, _dp), C.c_uint64(int(seed)), C.c_uint64(int(g))))


def normalized_preference(w: float) -> float:
    """w / (1 - w) for the scheme's head-to-head win fraction w."""
    return float(lib().orc_normalized_preference(float(w)))


def head_to_head(L: int, lstar: int):
    win, loss = C.c_int(0), C.c_int(0)
    lib().orc_head_to_head(int(L), int(lstar), C.byref(win), C.byref(loss))
    return win.value, loss.value


def _problem_args(prob):
    return (prob.n, prob.R, int(prob.T), prob.X, _p(_f64(prob.k0), _dp), _p(_f64(prob.kmin), _dp),
            _p(_f64(prob.kmax), _dp), _p(_f64(prob.xi), _dp), _p(_f64(prob.e), _dp), _p(_f64(prob.p), _dp),
            _p(_f64(prob.q), _dp), int(prob.profile_per_interval), float(prob.k1), float(prob.pue))


def _g0(g0):
    return None if g0 is None else np.ascontiguousarray(g0, dtype=np.uint64)


def preference(prob, cost, seg_offsets, flags=None, scheme: int = 0, grid_den: int = 0, g0=None):
    """Per cell [R*T*X][3]: hits (L = l*), wins, losses against Base (reading L22).
    g0: per segment, the global index of its first request (default: seg_offsets)."""
    keep = [_f64(a) for a in (prob.k0, prob.kmin, prob.kmax, prob.xi, prob.e, prob.p, prob.q)]
    off = np.ascontiguousarray(seg_offsets, dtype=np.int64)
    fl = None if flags is None else np.ascontiguousarray(flags, dtype=np.uint8)
    out = np.zeros((prob.R * prob.T * prob.X, 3), np.uint64)
    gb = _g0(g0)
    st = lib().orc_preference(*_problem_args(prob), C.c_uint64(int(cost.seed)), int(cost.n_classes),
                              _p(off, _i64p), _p(gb, _u64p), _p(fl, _u8p), int(scheme), int(grid_den), _p(out, _u64p))
    del keep
    if st != 0:
        raise ValueError("oracle preference: invalid argument")
    return out


def request_outputs(prob, cost, seg_offsets, tokens, flags=None, j: int = 0, scheme: int = 0, grid_den: int = 0,
                    g0=None):
    """Per request of cell column j: level, carbon, Base carbon, ratio (Fig. eval2), l*."""
    off = np.ascontiguousarray(seg_offsets, dtype=np.int64)
    tokens = np.ascontiguousarray(tokens, dtype=np.uint16)
    fl = None if flags is None else np.ascontiguousarray(flags, dtype=np.uint8)
    N = int(off[-1])
    out = dict(level=np.zeros(N, np.uint8), carbon=np.zeros(N), base=np.zeros(N), ratio=np.zeros(N),
               pref=np.zeros(N, np.uint8))
    ef, et, pf, pt = (_f64(a) for a in (cost.ef, cost.et, cost.pf, cost.pt))
    st = lib().orc_request_outputs(*_problem_args(prob), C.c_uint64(int(cost.seed)), int(cost.n_classes),
                                   _p(ef, _dp), _p(et, _dp), _p(pf, _dp), _p(pt, _dp), _p(off, _i64p),
                                   _p(_g0(g0), _u64p), _p(tokens, _u16p), tokens.shape[1], _p(fl, _u8p), int(scheme), int(grid_den),
                                   int(j), _p(out["level"], _u8p), _p(out["carbon"], _dp), _p(out["base"], _dp),
                                   _p(out["ratio"], _dp), _p(out["pref"], _u8p))
    if st != 0:
        raise ValueError("oracle request_outputs: invalid argument")
    return out


def oracle_scheme(prob, cost, seg_offsets, tokens, flags=None, g0=None):
    """The Oracle scheme (reading L23), per cell: cnt/tok [NC][n],
    energy/time/carbon/quality sums, stats (hits, wins, losses), status."""
    n, R, T, X, NC = prob.n, prob.R, int(prob.T), prob.X, cost.n_classes
    off = np.ascontiguousarray(seg_offsets, dtype=np.int64)
    tokens = np.ascontiguousarray(tokens, dtype=np.uint16)
    fl = None if flags is None else np.ascontiguousarray(flags, dtype=np.uint8)
    cells = R * T * X
    out = dict(cnt=np.zeros((cells, NC, n), np.uint64), tok=np.zeros((cells, NC, n), np.uint64),
               energy=np.zeros(cells), time=np.zeros(cells), carbon=np.zeros(cells), quality=np.zeros(cells),
               stats=np.zeros((cells, 3), np.uint64), status=np.zeros(cells, np.uint8))
    ef, et, pf, pt = (_f64(a) for a in (cost.ef, cost.et, cost.pf, cost.pt))
    st = lib().orc_oracle_scheme(n, R, T, X, _p(_f64(prob.k0), _dp), _p(_f64(prob.kmin), _dp),
                                 _p(_f64(prob.kmax), _dp), _p(_f64(prob.xi), _dp), _p(_f64(prob.q), _dp),
                                 int(prob.profile_per_interval), float(prob.k1), float(prob.pue),
                                 C.c_uint64(int(cost.seed)), NC, _p(ef, _dp), _p(et, _dp), _p(pf, _dp), _p(pt, _dp),
                                 _p(off, _i64p), _p(_g0(g0), _u64p), _p(tokens, _u16p), tokens.shape[1],
                                 _p(fl, _u8p), _p(out["cnt"], _u64p), _p(out["tok"], _u64p), _p(out["energy"], _dp),
                                 _p(out["time"], _dp), _p(out["carbon"], _dp), _p(out["quality"], _dp),
                                 _p(out["stats"], _u64p), _p(out["status"], _u8p))
    if st != 0:
        raise ValueError("oracle oracle_scheme: invalid argument")
    return out


def evaluation_q(k2, k2max, T: int, dt: float, beta: float, theta: float, grace: float, fallback: int, q_true,
                 seed: int, seg_offsets, sample: int = 500):
    """NEXT-1 q update (reading L24): (q per interval [R*T][n], fired [R*T])."""
    k2 = _f64(k2); k2max = _f64(k2max); q_true = _f64(q_true)
    R = len(k2max)
    n = q_true.shape[-1]
    off = np.ascontiguousarray(seg_offsets, dtype=np.int64)
    q_out = np.zeros((R * T, n)); fired = np.zeros(R * T, np.uint8)
    st = lib().orc_evaluation_q(R, int(T), float(dt), _p(k2, _dp), _p(k2max, _dp), float(beta), float(theta),
                                float(grace), int(fallback), int(n), _p(q_true, _dp), C.c_uint64(int(seed)),
                                _p(off, _i64p), int(sample), _p(q_out, _dp), _p(fired, _u8p))
    if st != 0:
        raise ValueError("oracle evaluation_q: invalid argument")
    return q_out, fired
