"""Thin ctypes binding of libsprout.so (include/sprout.h): argument
marshalling only.  Every step of the hot path runs in the CUDA kernels behind
the C ABI; torch provides device memory, streams and process groups.

The library is required: importing this module raises if libsprout.so is
missing (no CPU fallback exists), and every call raises SproutError on a
non-OK status.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
from typing import Optional

import numpy as np
import torch

# SPROUT_LIB_NAME selects another in-tree build of the same library (A/B
# timing of kernel variants during development); default libsprout.so.
_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ.get("SPROUT_LIB_NAME", "libsprout.so"))
if not os.path.exists(_LIB_PATH):
    raise ImportError(f"{_LIB_PATH} is missing: build it with `python -m paper_2403_12900_b200.build` "
                      "(there is no CPU fallback)")
_lib = C.CDLL(_LIB_PATH)

MAX_LEVELS = 8
MAX_CLASSES = 4
MAX_XI = 4096
CELL_OK, CELL_INVALID, CELL_INFEASIBLE = 0, 1, 2
TRACE_BAD_CLASS, TRACE_BAD_OFFSETS, TRACE_TOO_LONG, TRACE_SLOW_PATH = 0x1, 0x2, 0x4, 0x100

STATUS = {0: "SPROUT_OK", 1: "SPROUT_ERR_INVALID_ARGUMENT", 2: "SPROUT_ERR_INFEASIBLE",
          3: "SPROUT_ERR_OVERFLOW", 4: "SPROUT_ERR_CUDA", 5: "SPROUT_ERR_INVALID_CELL"}


class SproutError(RuntimeError):
    def __init__(self, fn: str, status: int):
        self.status = status
        super().__init__(f"{fn}: {STATUS.get(status, status)} ({_lib.sprout_status_string(status).decode()})")


_vp = C.c_void_p


class LpProblem(C.Structure):
    _fields_ = [("n_levels", C.c_int32), ("n_regions", C.c_int32), ("n_intervals", C.c_int64),
                ("n_xi", C.c_int32), ("profile_per_interval", C.c_int32),
                ("k0", _vp), ("k0_min", _vp), ("k0_max", _vp), ("xi", _vp), ("e", _vp), ("p", _vp), ("q", _vp),
                ("k1", C.c_double), ("pue", C.c_double), ("first_segment", C.c_int64), ("n_segments", C.c_int64)]


class LpSolution(C.Structure):
    _fields_ = [("x", _vp), ("objective", _vp), ("q_lb", _vp), ("vertex", _vp), ("threshold", _vp),
                ("max_level", _vp), ("cell_status", _vp)]


class Trace(C.Structure):
    _fields_ = [("n_requests", C.c_int64), ("first_request", C.c_uint64), ("seg_offsets", _vp),
                ("tokens", _vp), ("plane_pitch", C.c_int64), ("flags", _vp)]


class CostModel(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n_classes", C.c_int32), ("reserved", C.c_int32),
                ("ef", (C.c_double * MAX_LEVELS) * MAX_CLASSES), ("et", (C.c_double * MAX_LEVELS) * MAX_CLASSES),
                ("pf", (C.c_double * MAX_LEVELS) * MAX_CLASSES), ("pt", (C.c_double * MAX_LEVELS) * MAX_CLASSES)]


class CellTotals(C.Structure):
    _fields_ = [("cnt", _vp), ("tok", _vp), ("energy_kwh", _vp), ("time_s", _vp), ("carbon_g", _vp),
                ("quality", _vp), ("seg_count", _vp), ("seg_pinned", _vp), ("seg_tok", _vp), ("seg_base", _vp),
                ("trace_status", _vp)]


class TraceGenerator(C.Structure):
    _fields_ = [("gen_seed", C.c_uint64), ("first_request", C.c_uint64), ("n_requests", C.c_int64),
                ("n_levels", C.c_int32), ("n_classes", C.c_int32), ("pin_thresh", C.c_uint32),
                ("reserved", C.c_uint32), ("q0_table", _vp), ("ratio_table", _vp)]


_P = C.POINTER
_lib.sprout_solve_directives.argtypes = [_P(LpProblem), _P(LpSolution), _vp]
_lib.sprout_workspace_bytes.argtypes = [_P(LpProblem), _P(Trace)]
_lib.sprout_workspace_bytes.restype = C.c_size_t
_lib.sprout_simulate_trace.argtypes = [_P(LpProblem), _P(LpSolution), _P(Trace), _P(CostModel), _P(CellTotals),
                                       _vp, _vp, C.c_size_t, _vp]
_lib.sprout_group_stat_count.argtypes = [C.c_int32]
_lib.sprout_group_stat_count.restype = C.c_int32
_lib.sprout_reduce_workspace_bytes.argtypes = [_P(LpProblem)]
_lib.sprout_reduce_workspace_bytes.restype = C.c_size_t
_lib.sprout_reduce_totals.argtypes = [_P(LpProblem), _P(LpSolution), _P(CellTotals), C.c_int32, _vp, _vp,
                                      C.c_size_t, _vp]
_lib.sprout_check_cells.argtypes = [_P(LpProblem), _P(LpSolution), _vp]
_lib.sprout_sweep_workspace_bytes.argtypes = [_P(LpProblem), _P(Trace), C.c_int32]
_lib.sprout_sweep_workspace_bytes.restype = C.c_size_t
_lib.sprout_sweep_host.argtypes = [_P(LpProblem), _P(Trace), _P(CostModel), _vp, _vp, _vp, C.c_size_t, _vp]
_lib.sprout_generate_trace.argtypes = [_P(TraceGenerator), _vp, C.c_int64, _vp, _vp]
_lib.sprout_last_launch_count.restype = C.c_int32
_lib.sprout_status_string.argtypes = [C.c_int]
_lib.sprout_status_string.restype = C.c_char_p
_lib.sprout_simulate_trace_bounded.argtypes = [_P(LpProblem), _P(LpSolution), _P(Trace), _P(CostModel),
                                               _P(CellTotals), _vp, C.c_int32, _vp, C.c_size_t, _vp]
class EvaluatorProblem(C.Structure):
    _fields_ = [("n_regions", C.c_int32), ("n_beta", C.c_int32), ("n_intervals", C.c_int64),
                ("interval_hours", C.c_double), ("k2", _vp), ("k2_max", _vp), ("beta", _vp),
                ("n_theta", C.c_int32), ("fallback", C.c_int32), ("theta", _vp), ("grace_hours", C.c_double),
                ("eval_kwh", C.c_double), ("pue", C.c_double)]


_lib.sprout_evaluator_sweep.argtypes = [_P(EvaluatorProblem), _vp, _vp]
_lib.sprout_simulate_closed_loop.argtypes = [_P(LpProblem), C.c_int32, _P(Trace), _P(CostModel), _P(LpSolution),
                                             _P(CellTotals), _vp, _vp, C.c_size_t, _vp]
_lib.sprout_solve_scheme.argtypes = [_P(LpProblem), C.c_int32, C.c_int32, _P(LpSolution), _vp]
_lib.sprout_static_grid_size.argtypes = [C.c_int32, C.c_int32]
_lib.sprout_static_grid_size.restype = C.c_int64
_lib.sprout_select_static.argtypes = [_P(LpProblem), C.c_int32, C.c_double, _vp, _vp, _vp, _vp]
for _fn in ("sprout_solve_directives", "sprout_simulate_trace", "sprout_reduce_totals", "sprout_check_cells",
            "sprout_sweep_host", "sprout_generate_trace", "sprout_solve_scheme", "sprout_select_static",
            "sprout_simulate_trace_bounded", "sprout_evaluator_sweep", "sprout_simulate_closed_loop"):
    getattr(_lib, _fn).restype = C.c_int

EXPORTS = ["sprout_solve_directives", "sprout_workspace_bytes", "sprout_simulate_trace", "sprout_group_stat_count",
           "sprout_reduce_workspace_bytes", "sprout_reduce_totals", "sprout_check_cells",
           "sprout_sweep_workspace_bytes", "sprout_sweep_host", "sprout_generate_trace",
           "sprout_last_launch_count", "sprout_status_string", "sprout_solve_scheme", "sprout_static_grid_size",
           "sprout_select_static", "sprout_simulate_trace_bounded", "sprout_evaluator_sweep",
           "sprout_simulate_closed_loop", "sprout_request_outputs", "sprout_preference_stats",
           "sprout_normalized_preference", "sprout_oracle_scheme_workspace_bytes",
           "sprout_simulate_oracle_scheme", "sprout_evaluation_q", "sprout_simulate_closed_loop_q",
           "sprout_cell_totals_fp64"]

# competing schemes, include/sprout.h SPROUT_SCHEME_*
SCHEME_SPROUT, SCHEME_CO2_OPT, SCHEME_STATIC_GRID = 0, 1, 2
VERTEX_GRID = 254


def _check(fn: str, st: int):
    if st != 0:
        raise SproutError(fn, st)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else t.data_ptr()


def _stream(stream) -> Optional[int]:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


# --------------------------------------------------------------------------
# device-side bundles (torch tensors kept alive alongside the C structs)

@dataclasses.dataclass
class DeviceProblem:
    n: int
    R: int
    T: int
    X: int
    k0: torch.Tensor
    kmin: torch.Tensor
    kmax: torch.Tensor
    xi: torch.Tensor
    e: torch.Tensor
    p: torch.Tensor
    q: torch.Tensor
    profile_per_interval: int
    k1: float
    pue: float
    first_segment: int
    n_segments: int

    @classmethod
    def from_host(cls, prob, device, first_segment: int = 0, n_segments: Optional[int] = None) -> "DeviceProblem":
        """`prob` is any object with the synth.Problem attributes."""
        f64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, np.float64)).to(device)
        if n_segments is None:
            n_segments = prob.R * prob.T - first_segment
        return cls(prob.n, prob.R, prob.T, prob.X, f64(prob.k0), f64(prob.kmin), f64(prob.kmax), f64(prob.xi),
                   f64(prob.e), f64(prob.p), f64(prob.q), int(prob.profile_per_interval), float(prob.k1),
                   float(prob.pue), int(first_segment), int(n_segments))

    @property
    def cells(self) -> int:
        return self.n_segments * self.X

    def c(self) -> LpProblem:
        return LpProblem(self.n, self.R, self.T, self.X, self.profile_per_interval, _ptr(self.k0), _ptr(self.kmin),
                         _ptr(self.kmax), _ptr(self.xi), _ptr(self.e), _ptr(self.p), _ptr(self.q), self.k1,
                         self.pue, self.first_segment, self.n_segments)


@dataclasses.dataclass
class Solution:
    x: torch.Tensor
    objective: torch.Tensor
    q_lb: torch.Tensor
    vertex: torch.Tensor
    threshold: Optional[torch.Tensor]
    max_level: torch.Tensor
    cell_status: torch.Tensor

    @classmethod
    def empty(cls, prob: DeviceProblem) -> "Solution":
        dev, cells, n = prob.k0.device, prob.cells, prob.n
        return cls(torch.empty((cells, n), dtype=torch.float64, device=dev),
                   torch.empty(cells, dtype=torch.float64, device=dev),
                   torch.empty(cells, dtype=torch.float64, device=dev),
                   torch.empty(cells, dtype=torch.uint8, device=dev),
                   torch.empty((cells, n - 1), dtype=torch.int32, device=dev) if n > 1 else None,
                   torch.empty(cells, dtype=torch.uint8, device=dev),
                   torch.empty(cells, dtype=torch.uint8, device=dev))

    def c(self) -> LpSolution:
        return LpSolution(_ptr(self.x), _ptr(self.objective), _ptr(self.q_lb), _ptr(self.vertex),
                          _ptr(self.threshold), _ptr(self.max_level), _ptr(self.cell_status))

    def thresholds_u32(self) -> np.ndarray:
        return self.threshold.cpu().numpy().view(np.uint32) if self.threshold is not None else np.zeros((0, 0), np.uint32)


@dataclasses.dataclass
class DeviceTrace:
    n_requests: int
    first_request: int
    seg_offsets: torch.Tensor      # int64 [n_segments+1]
    tokens: torch.Tensor           # int16 view of uint16 [n][pitch]
    flags: Optional[torch.Tensor]  # uint8 [pitch]

    @property
    def pitch(self) -> int:
        return self.tokens.shape[1]

    def c(self) -> Trace:
        return Trace(self.n_requests, self.first_request, _ptr(self.seg_offsets), _ptr(self.tokens), self.pitch,
                     _ptr(self.flags))


@dataclasses.dataclass
class Totals:
    cnt: torch.Tensor
    tok: torch.Tensor
    energy: torch.Tensor
    time: torch.Tensor
    carbon: torch.Tensor
    quality: torch.Tensor
    seg_count: torch.Tensor
    seg_pinned: torch.Tensor
    seg_tok: torch.Tensor
    seg_base: torch.Tensor
    trace_status: torch.Tensor

    @classmethod
    def empty(cls, prob: DeviceProblem, n_classes: int) -> "Totals":
        dev, cells, n, S = prob.k0.device, prob.cells, prob.n, prob.n_segments
        i64 = lambda *s: torch.zeros(s, dtype=torch.int64, device=dev)
        f64 = lambda *s: torch.zeros(s, dtype=torch.float64, device=dev)
        return cls(i64(cells, n_classes, n), i64(cells, n_classes, n), f64(cells), f64(cells), f64(cells),
                   f64(cells), i64(S, n_classes), i64(S, n_classes), i64(S, n_classes, n), f64(S, 4),
                   torch.zeros(1, dtype=torch.int32, device=dev))

    def c(self) -> CellTotals:
        return CellTotals(*[_ptr(getattr(self, f.name)) for f in dataclasses.fields(self)])


def cost_model(cost) -> CostModel:
    """From any object with the synth.CostModel attributes."""
    cm = CostModel()
    cm.seed = int(cost.seed) & 0xFFFFFFFFFFFFFFFF
    cm.n_classes = int(cost.n_classes)
    for name in ("ef", "et", "pf", "pt"):
        arr = np.asarray(getattr(cost, name), np.float64)
        dst = getattr(cm, name)
        for c in range(MAX_CLASSES):
            for L in range(MAX_LEVELS):
                dst[c][L] = float(arr[c, L]) if c < arr.shape[0] and L < arr.shape[1] else 0.0
    return cm


# --------------------------------------------------------------------------
# the C-ABI entry points, same names

def solve_directives(prob: DeviceProblem, sol: Solution, stream=None) -> None:
    p, s = prob.c(), sol.c()
    _check("sprout_solve_directives", _lib.sprout_solve_directives(C.byref(p), C.byref(s), _stream(stream)))


def workspace_bytes(prob: DeviceProblem, trace: DeviceTrace) -> int:
    p, t = prob.c(), trace.c()
    return int(_lib.sprout_workspace_bytes(C.byref(p), C.byref(t)))


def simulate_trace(prob: DeviceProblem, sol: Solution, trace: DeviceTrace, cost: CostModel, totals: Totals,
                   workspace: torch.Tensor, levels_out: Optional[torch.Tensor] = None, stream=None) -> None:
    p, s, t, tt = prob.c(), sol.c(), trace.c(), totals.c()
    _check("sprout_simulate_trace",
           _lib.sprout_simulate_trace(C.byref(p), C.byref(s), C.byref(t), C.byref(cost), C.byref(tt),
                                      _ptr(levels_out), _ptr(workspace), workspace.numel() * workspace.element_size(),
                                      _stream(stream)))


def simulate_trace_bounded(prob: DeviceProblem, sol: Solution, trace: DeviceTrace, cost: CostModel, totals: Totals,
                           max_breakpoints: int, workspace: torch.Tensor, levels_out: Optional[torch.Tensor] = None,
                           stream=None) -> None:
    p, s, t, tt = prob.c(), sol.c(), trace.c(), totals.c()
    _check("sprout_simulate_trace_bounded",
           _lib.sprout_simulate_trace_bounded(C.byref(p), C.byref(s), C.byref(t), C.byref(cost), C.byref(tt),
                                              _ptr(levels_out), int(max_breakpoints), _ptr(workspace),
                                              workspace.numel() * workspace.element_size(), _stream(stream)))


def group_stat_count(n_levels: int) -> int:
    return int(_lib.sprout_group_stat_count(n_levels))


def reduce_workspace_bytes(prob: DeviceProblem) -> int:
    p = prob.c()
    return int(_lib.sprout_reduce_workspace_bytes(C.byref(p)))


def reduce_totals(prob: DeviceProblem, sol: Solution, totals: Totals, n_classes: int, group_totals: torch.Tensor,
                  workspace: torch.Tensor, stream=None) -> None:
    p, s, tt = prob.c(), sol.c(), totals.c()
    _check("sprout_reduce_totals",
           _lib.sprout_reduce_totals(C.byref(p), C.byref(s), C.byref(tt), int(n_classes), _ptr(group_totals),
                                     _ptr(workspace), workspace.numel() * workspace.element_size(), _stream(stream)))


def solve_scheme(prob: DeviceProblem, scheme: int, grid_den: int, sol: Solution, stream=None) -> None:
    p, s = prob.c(), sol.c()
    _check("sprout_solve_scheme",
           _lib.sprout_solve_scheme(C.byref(p), int(scheme), int(grid_den), C.byref(s), _stream(stream)))


def static_grid_size(n_levels: int, grid_den: int) -> int:
    return int(_lib.sprout_static_grid_size(int(n_levels), int(grid_den)))


def select_static(prob: DeviceProblem, grid_den: int, xi: float, group_totals: torch.Tensor, choice: torch.Tensor,
                  x: torch.Tensor, stream=None) -> None:
    p = prob.c()
    _check("sprout_select_static",
           _lib.sprout_select_static(C.byref(p), int(grid_den), float(xi), _ptr(group_totals), _ptr(choice),
                                     _ptr(x), _stream(stream)))


def evaluator_sweep(k2: torch.Tensor, k2_max: torch.Tensor, n_intervals: int, interval_hours: float, betas,
                    thetas, grace_hours: float, fallback: int, eval_kwh: float, pue: float, out: torch.Tensor,
                    stream=None) -> None:
    """Opportunistic evaluator trigger sweep (Eq. 8); out [R][len(betas)][len(thetas)][4] fp64 device."""
    b = np.ascontiguousarray(betas, np.float64)
    t = np.ascontiguousarray(thetas, np.float64)
    P = EvaluatorProblem(int(k2_max.numel()), len(b), int(n_intervals), float(interval_hours), _ptr(k2),
                         _ptr(k2_max), b.ctypes.data, len(t), int(fallback), t.ctypes.data, float(grace_hours),
                         float(eval_kwh), float(pue))
    _check("sprout_evaluator_sweep", _lib.sprout_evaluator_sweep(C.byref(P), _ptr(out), _stream(stream)))


def simulate_closed_loop(prob: DeviceProblem, window: int, trace: DeviceTrace, cost: CostModel, sol: Solution,
                         totals: Totals, ws: torch.Tensor, profile_out: Optional[torch.Tensor] = None,
                         stream=None) -> None:
    p, t, s, tt = prob.c(), trace.c(), sol.c(), totals.c()
    _check("sprout_simulate_closed_loop",
           _lib.sprout_simulate_closed_loop(C.byref(p), int(window), C.byref(t), C.byref(cost), C.byref(s),
                                            C.byref(tt), _ptr(profile_out), _ptr(ws), ws.numel(), _stream(stream)))


_lib.sprout_cell_totals_fp64.argtypes = [_P(LpProblem), _P(LpSolution), _P(Trace), _P(CostModel), _vp, _vp, _vp,
                                         _vp, _vp]
_lib.sprout_cell_totals_fp64.restype = C.c_int


def cell_totals_fp64(prob: DeviceProblem, sol: Solution, trace: DeviceTrace, cost: CostModel, stream=None) -> dict:
    """Per-request fp64 accounting (cross-check of the closed form): energy, time, carbon, quality per cell."""
    out = {k: torch.zeros(prob.cells, dtype=torch.float64, device=trace.tokens.device)
           for k in ("energy", "time", "carbon", "quality")}
    p, s, t = prob.c(), sol.c(), trace.c()
    _check("sprout_cell_totals_fp64",
           _lib.sprout_cell_totals_fp64(C.byref(p), C.byref(s), C.byref(t), C.byref(cost), _ptr(out["energy"]),
                                        _ptr(out["time"]), _ptr(out["carbon"]), _ptr(out["quality"]),
                                        _stream(stream)))
    return out


def check_cells(prob: DeviceProblem, sol: Solution, stream=None) -> int:
    p, s = prob.c(), sol.c()
    return int(_lib.sprout_check_cells(C.byref(p), C.byref(s), _stream(stream)))


def sweep_workspace_bytes(prob_host: LpProblem, trace_host: Trace, n_classes: int) -> int:
    return int(_lib.sprout_sweep_workspace_bytes(C.byref(prob_host), C.byref(trace_host), int(n_classes)))


def sweep_host(prob_host: LpProblem, trace_host: Trace, cost: CostModel, out_host: np.ndarray,
               status_host: np.ndarray, workspace: torch.Tensor, stream=None) -> None:
    """End-to-end with HOST buffers (pointers inside prob_host/trace_host are host addresses)."""
    _check("sprout_sweep_host",
           _lib.sprout_sweep_host(C.byref(prob_host), C.byref(trace_host), C.byref(cost),
                                  out_host.ctypes.data, status_host.ctypes.data, _ptr(workspace),
                                  workspace.numel() * workspace.element_size(), _stream(stream)))


def generate_trace(gen: TraceGenerator, tokens: torch.Tensor, flags: Optional[torch.Tensor], stream=None) -> None:
    _check("sprout_generate_trace",
           _lib.sprout_generate_trace(C.byref(gen), _ptr(tokens), tokens.shape[1], _ptr(flags), _stream(stream)))


def last_launch_count() -> int:
    return int(_lib.sprout_last_launch_count())


def status_string(status: int) -> str:
    return _lib.sprout_status_string(status).decode()


def workspace(nbytes: int, device) -> torch.Tensor:
    """A 256-byte aligned device byte buffer (torch's allocator aligns to 512)."""
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


# NEXT-4: per-request outputs, head-to-head preference statistics (readings L21, L22)
_lib.sprout_request_outputs.argtypes = [_P(LpProblem), _P(LpSolution), _P(Trace), _P(CostModel), C.c_int32,
                                        _vp, _vp, _vp, _vp, _vp, _vp]
_lib.sprout_preference_stats.argtypes = [_P(LpProblem), _P(LpSolution), _P(Trace), _P(CostModel), _vp, _vp]
_lib.sprout_normalized_preference.argtypes = [C.c_double]
_lib.sprout_normalized_preference.restype = C.c_double


def request_outputs(prob: DeviceProblem, sol: Solution, trace: DeviceTrace, cost: CostModel, xi_index: int,
                    level_out: torch.Tensor, carbon_out: torch.Tensor, base_out: torch.Tensor,
                    ratio_out: torch.Tensor, pref_out: Optional[torch.Tensor] = None, stream=None) -> None:
    p, s, t = prob.c(), sol.c(), trace.c()
    _check("sprout_request_outputs",
           _lib.sprout_request_outputs(C.byref(p), C.byref(s), C.byref(t), C.byref(cost), int(xi_index),
                                       _ptr(level_out), _ptr(carbon_out), _ptr(base_out), _ptr(ratio_out),
                                       _ptr(pref_out), _stream(stream)))


def preference_stats(prob: DeviceProblem, sol: Solution, trace: DeviceTrace, cost: CostModel, stats: torch.Tensor,
                     stream=None) -> None:
    p, s, t = prob.c(), sol.c(), trace.c()
    _check("sprout_preference_stats",
           _lib.sprout_preference_stats(C.byref(p), C.byref(s), C.byref(t), C.byref(cost), _ptr(stats),
                                        _stream(stream)))


def normalized_preference(w: float) -> float:
    return float(_lib.sprout_normalized_preference(float(w)))


_lib.sprout_oracle_scheme_workspace_bytes.argtypes = [_P(LpProblem), C.c_int64]
_lib.sprout_oracle_scheme_workspace_bytes.restype = C.c_size_t
_lib.sprout_simulate_oracle_scheme.argtypes = [_P(LpProblem), _P(Trace), _P(CostModel), C.c_int64, _P(CellTotals),
                                               _vp, _vp, _vp, C.c_size_t, _vp]


def oracle_scheme_workspace_bytes(prob: DeviceProblem, max_segment_requests: int) -> int:
    p = prob.c()
    return int(_lib.sprout_oracle_scheme_workspace_bytes(C.byref(p), int(max_segment_requests)))


def simulate_oracle_scheme(prob: DeviceProblem, trace: DeviceTrace, cost: CostModel, max_segment_requests: int,
                           totals: Totals, stats: torch.Tensor, cell_status: torch.Tensor, workspace: torch.Tensor,
                           stream=None) -> None:
    p, t, tt = prob.c(), trace.c(), totals.c()
    _check("sprout_simulate_oracle_scheme",
           _lib.sprout_simulate_oracle_scheme(C.byref(p), C.byref(t), C.byref(cost), int(max_segment_requests),
                                              C.byref(tt), _ptr(stats), _ptr(cell_status), _ptr(workspace),
                                              workspace.numel() * workspace.element_size(), _stream(stream)))


# NEXT-1: q per evaluation epoch (reading L24) and the closed loop with it
_lib.sprout_evaluation_q.argtypes = [_P(EvaluatorProblem), _P(LpProblem), _P(Trace), _P(CostModel), C.c_int32,
                                     _vp, _vp, _vp]
_lib.sprout_simulate_closed_loop_q.argtypes = [_P(LpProblem), C.c_int32, _vp, _P(Trace), _P(CostModel),
                                               _P(LpSolution), _P(CellTotals), _vp, _vp, C.c_size_t, _vp]


def evaluation_q(prob: DeviceProblem, trace: DeviceTrace, cost: CostModel, k2: torch.Tensor, k2_max: torch.Tensor,
                 interval_hours: float, beta: float, theta: float, grace_hours: float, fallback: int, sample: int,
                 q_out: torch.Tensor, fired_out: torch.Tensor, stream=None) -> None:
    b = np.array([beta], np.float64)
    t = np.array([theta], np.float64)
    E = EvaluatorProblem(int(k2_max.numel()), 1, int(prob.T), float(interval_hours), _ptr(k2), _ptr(k2_max),
                         b.ctypes.data, 1, int(fallback), t.ctypes.data, float(grace_hours), 0.0, 1.0)
    p, tr = prob.c(), trace.c()
    _check("sprout_evaluation_q",
           _lib.sprout_evaluation_q(C.byref(E), C.byref(p), C.byref(tr), C.byref(cost), int(sample), _ptr(q_out),
                                    _ptr(fired_out), _stream(stream)))


def simulate_closed_loop_q(prob: DeviceProblem, window: int, q_interval: Optional[torch.Tensor], trace: DeviceTrace,
                           cost: CostModel, sol: Solution, totals: Totals, ws: torch.Tensor,
                           profile_out: Optional[torch.Tensor] = None, stream=None) -> None:
    p, t, s, tt = prob.c(), trace.c(), sol.c(), totals.c()
    _check("sprout_simulate_closed_loop_q",
           _lib.sprout_simulate_closed_loop_q(C.byref(p), int(window), _ptr(q_interval), C.byref(t), C.byref(cost),
                                              C.byref(s), C.byref(tt), _ptr(profile_out), _ptr(ws), ws.numel(),
                                              _stream(stream)))
