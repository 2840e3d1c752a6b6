"""Device-side orchestration of one rank's sweep: allocate the C-ABI
buffers as torch tensors, put the trace on the device (uploaded from the host
or generated in place by the harness-only generator kernel), and call the
three hot-path entry points.  Marshalling only -- no arithmetic of the method.

Inputs are duck-typed (any objects with the attributes of synth.Problem,
synth.CostModel, synth.TraceSpec and synth.Shard), so the product package does
not depend on the input generator.
"""
from __future__ import annotations

from typing import Optional

import numpy as np
import torch

from . import sprout as S


def _pitch(n_requests: int) -> int:
    return max(8, ((n_requests + 7) // 8) * 8)


class Sweep:
    """One rank's slice: segments [shard.first_segment, +n_segments) and the
    local requests [shard.first_request, +n_requests)."""

    def __init__(self, prob, cost, shard, device, spec=None, tokens: Optional[np.ndarray] = None,
                 flags: Optional[np.ndarray] = None, has_flags: Optional[bool] = None, scheme: int = 0,
                 grid_den: int = 0):
        self.device = torch.device(device)
        self.scheme, self.grid_den = int(scheme), int(grid_den)
        self.prob_host = prob
        self.dp = S.DeviceProblem.from_host(prob, self.device, shard.first_segment, shard.n_segments)
        self.sol = S.Solution.empty(self.dp)
        self.cost = S.cost_model(cost)
        self.n_classes = int(cost.n_classes)
        self.totals = S.Totals.empty(self.dp, self.n_classes)
        n = prob.n
        pitch = _pitch(shard.n_requests)
        seg = torch.as_tensor(np.ascontiguousarray(shard.seg_offsets, np.int64)).to(self.device)
        if tokens is not None:
            tok = np.zeros((n, pitch), np.uint16)
            tok[:, :tokens.shape[1]] = tokens[:, :pitch]
            tok_t = torch.from_numpy(tok.view(np.int16)).to(self.device)
            fl_t = None
            if flags is not None:
                fl = np.zeros(pitch, np.uint8)
                fl[:flags.shape[0]] = flags[:pitch]
                fl_t = torch.from_numpy(fl).to(self.device)
        else:
            assert spec is not None, "need a TraceSpec to generate the trace on the device"
            use_flags = spec.has_flags if has_flags is None else has_flags
            tok_t = torch.empty((n, pitch), dtype=torch.int16, device=self.device)
            fl_t = torch.empty(pitch, dtype=torch.uint8, device=self.device) if use_flags else None
            self.generate(spec, shard, tok_t, fl_t)
        self.trace = S.DeviceTrace(shard.n_requests, shard.first_request, seg, tok_t, fl_t)
        self.ws = S.workspace(S.workspace_bytes(self.dp, self.trace), self.device)
        self.rws = S.workspace(S.reduce_workspace_bytes(self.dp), self.device)
        K = S.group_stat_count(n)
        self.group = torch.zeros((prob.R + 1, prob.X, K), dtype=torch.float64, device=self.device)
        self.levels = None

    def generate(self, spec, shard, tok_t, fl_t, stream=None):
        q0 = torch.from_numpy(np.ascontiguousarray(spec.q0_table, np.uint16).view(np.int16)).to(self.device)
        rt = torch.from_numpy(np.ascontiguousarray(spec.ratio_table, np.uint16).view(np.int16)).to(self.device)
        self._gen_tables = (q0, rt)
        gen = S.TraceGenerator(int(spec.gen_seed) & 0xFFFFFFFFFFFFFFFF, int(shard.first_request),
                               int(shard.n_requests), int(spec.n_levels), int(spec.n_classes),
                               int(spec.pin_thresh) if fl_t is not None else 0, 0, q0.data_ptr(), rt.data_ptr())
        S.generate_trace(gen, tok_t, fl_t, stream)

    # the three hot-path steps
    def solve(self, stream=None):
        if self.scheme == S.SCHEME_SPROUT:
            S.solve_directives(self.dp, self.sol, stream)
        else:
            S.solve_scheme(self.dp, self.scheme, self.grid_den, self.sol, stream)

    def select_static(self, xi: float, stream=None):
        """Sprout_Sta choice per region from this sweep's group totals (all
        regions' segments must be local, or the totals all-reduced first)."""
        assert self.scheme == S.SCHEME_STATIC_GRID
        R, n = self.prob_host.R, self.prob_host.n
        choice = torch.zeros(R, dtype=torch.int32, device=self.device)
        x = torch.zeros((R, n), dtype=torch.float64, device=self.device)
        S.select_static(self.dp, self.grid_den, xi, self.group, choice, x, stream)
        return choice, x

    def simulate(self, levels: bool = False, stream=None):
        lv = None
        if levels:
            if self.levels is None:
                self.levels = torch.full((self.dp.X, self.trace.pitch), 0xFF, dtype=torch.uint8, device=self.device)
            lv = self.levels
        if self.scheme == S.SCHEME_STATIC_GRID:   # <= 2(D-1) distinct breakpoints per segment
            S.simulate_trace_bounded(self.dp, self.sol, self.trace, self.cost, self.totals,
                                     max(1, 2 * (self.grid_den - 1)), self.ws, lv, stream)
        else:
            S.simulate_trace(self.dp, self.sol, self.trace, self.cost, self.totals, self.ws, lv, stream)

    def closed_loop(self, window: int, profile: bool = False, q_interval: Optional[torch.Tensor] = None, stream=None):
        """Closed-loop profiles (NEXT-1): steps 1-2 as a causal scan per
        (region, xi) chain; writes the solution and every totals field
        (cells and segments), so reduce() can follow directly.  q_interval
        [R*T][n]: the q of every interval's evaluation epoch (evaluation_q)."""
        prof = None
        if profile:
            prof = torch.zeros((self.dp.cells, 2, self.prob_host.n), dtype=torch.float64, device=self.device)
        S.simulate_closed_loop_q(self.dp, window, q_interval, self.trace, self.cost, self.sol, self.totals, self.ws,
                                 prof, stream)
        return prof

    def evaluation_q(self, interval_hours: float, beta: float, theta: float, grace_hours: float, fallback: int,
                     sample: int = 500, stream=None):
        """NEXT-1: q per evaluation epoch (reading L24) -> (q [R*T][n], fired [R*T])."""
        P = self.prob_host
        k2 = self.dp.k0
        q = torch.zeros((P.R * P.T, P.n), dtype=torch.float64, device=self.device)
        fired = torch.zeros(P.R * P.T, dtype=torch.uint8, device=self.device)
        S.evaluation_q(self.dp, self.trace, self.cost, k2, self.dp.kmax, interval_hours, beta, theta, grace_hours,
                       fallback, sample, q, fired, stream)
        return q, fired

    def request_outputs(self, xi_index: int, stream=None) -> dict:
        """NEXT-4: per-request level, carbon, Base carbon, ratio and latent best level of one xi column."""
        N, dev = self.trace.n_requests, self.device
        out = dict(level=torch.empty(N, dtype=torch.uint8, device=dev), carbon=torch.empty(N, dtype=torch.float64, device=dev),
                   base=torch.empty(N, dtype=torch.float64, device=dev), ratio=torch.empty(N, dtype=torch.float64, device=dev),
                   pref=torch.empty(N, dtype=torch.uint8, device=dev))
        S.request_outputs(self.dp, self.sol, self.trace, self.cost, xi_index, out["level"], out["carbon"],
                          out["base"], out["ratio"], out["pref"], stream)
        return out

    def preference_stats(self, stream=None) -> torch.Tensor:
        """NEXT-4: per cell (hits, wins, losses) against Base."""
        st = torch.zeros((self.dp.cells, 3), dtype=torch.int64, device=self.device)
        S.preference_stats(self.dp, self.sol, self.trace, self.cost, st, stream)
        return st

    def oracle_scheme(self, stream=None) -> dict:
        """NEXT-4: the Oracle scheme into self.totals; returns stats and cell status."""
        seg = self.trace.seg_offsets
        cap = int((seg[1:] - seg[:-1]).max().item()) if seg.numel() > 1 else 0
        if getattr(self, "_or_ws", None) is None or self._or_cap < cap:
            self._or_cap = cap
            self._or_ws = S.workspace(S.oracle_scheme_workspace_bytes(self.dp, cap), self.device)
        st = torch.zeros((self.dp.cells, 3), dtype=torch.int64, device=self.device)
        cs = torch.zeros(self.dp.cells, dtype=torch.uint8, device=self.device)
        S.simulate_oracle_scheme(self.dp, self.trace, self.cost, self._or_cap, self.totals, st, cs, self._or_ws, stream)
        return dict(stats=st, cell_status=cs)

    def reduce(self, stream=None):
        S.reduce_totals(self.dp, self.sol, self.totals, self.n_classes, self.group, self.rws, stream)

    def step(self, stream=None):
        self.solve(stream)
        self.simulate(False, stream)
        self.reduce(stream)

    def capture(self, fn=None) -> "torch.cuda.CUDAGraph":
        """Capture one step (default: solve -> simulate -> reduce; or `fn`, e.g.
        one that adds the all-reduce) into a CUDA graph: the library launches
        only asynchronous work on the given stream and allocates nothing, so
        every later replay re-runs the whole step with one launch from the
        host.  Buffers stay the ones of this Sweep."""
        fn = fn or self.step
        side = torch.cuda.Stream(self.device)
        side.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(side):   # warm the lazy state (function attributes) outside the capture
            fn()
        torch.cuda.current_stream(self.device).wait_stream(side)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        return g

    # host views (for tests)
    def host(self) -> dict:
        t = self.totals
        out = {k: getattr(t, k).cpu().numpy() for k in ("energy", "time", "carbon", "quality", "seg_base")}
        for k in ("cnt", "tok", "seg_count", "seg_pinned", "seg_tok"):
            out[k] = getattr(t, k).cpu().numpy().view(np.uint64)
        out["trace_status"] = int(t.trace_status.cpu().numpy().view(np.uint32)[0])
        sol = self.sol
        out["x"] = sol.x.cpu().numpy()
        out["objective"] = sol.objective.cpu().numpy()
        out["q_lb"] = sol.q_lb.cpu().numpy()
        out["vertex"] = sol.vertex.cpu().numpy()
        out["threshold"] = sol.thresholds_u32()
        out["max_level"] = sol.max_level.cpu().numpy()
        out["cell_status"] = sol.cell_status.cpu().numpy()
        out["group"] = self.group.cpu().numpy()
        if self.levels is not None:
            out["levels"] = self.levels.cpu().numpy()
        return out

    def trace_host(self):
        tok = self.trace.tokens.cpu().numpy().view(np.uint16)
        fl = self.trace.flags.cpu().numpy() if self.trace.flags is not None else None
        return tok, fl
