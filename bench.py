#!/usr/bin/env python3
"""Benchmark of the Sprout hot path (solve -> simulate -> reduce [-> NCCL
allreduce]) on synthetic BASELINE.json workloads.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl sprout|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Prints ONE JSON line (rank 0).  A "step" is one pass of the whole hot path
over the workload: every LP cell solved, every request of the trace streamed
and assigned in every xi cell of its segment, group totals reduced (and
all-reduced across ranks).  Inputs are resident in HBM before timing
(`value`); `e2e` re-measures the same metric through the host-buffer C-ABI
call (sprout_sweep_host) with the H2D copy of the trace and the D2H of the
totals inside the timed region.  `--impl reference` times the CPU oracle
(the only reference this paper-only tier has) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "requests simulated/s and LP cells/s at 1/2/4/8 B200; % of HBM peak"
UNIT = "requests/s"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def workload_desc(w, scheme="sprout"):
    P = w.prob
    cells = {"sprout": "xi", "co2opt": "CO2_Opt cell", "static": "static grid points", "oracle": "xi (Oracle scheme)"}[scheme]
    return (f"{w.name}: {P.R} regions x {P.T} CI intervals x {P.X} {cells} x {P.n} directive levels, "
            f"{w.N:,} requests, {w.cost.n_classes} model class(es), flags={'yes' if w.spec.has_flags else 'no'}")


def algorithmic_bytes(w, sh):
    """Bytes the method must move in one sprout_simulate_trace launch
    (DESIGN.md 'Roofline'): the token planes (+flags) once, the segment
    offsets, k0, every cell's thresholds/max_level/status, and the per-cell
    and per-segment outputs."""
    P = w.prob
    n, X, NC = P.n, P.X, w.cost.n_classes
    S = sh.n_segments
    C = S * X
    N = int(sh.seg_offsets[-1] - sh.seg_offsets[0])
    f = 1 if w.spec.has_flags else 0
    b = N * (2 * n + f)                              # trace
    b += 8 * (S + 1) + 8 * S                         # seg_offsets, k0
    b += C * (4 * (n - 1) + 1 + 1)                   # thresholds, max_level, cell_status
    b += C * (NC * n * 16 + 32)                      # cnt, tok, energy/time/carbon/quality
    b += S * (NC * (2 + n) * 8 + 32)                 # segment stats + Base
    return b


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0])); mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------- CPU oracle


def oracle_sample_run(w, seg_ids, threads, scheme=0, grid_den=0):
    """Oracle on a set of whole segments of the workload (LP + replay),
    tokens regenerated on the host (generation not timed)."""
    import oracle
    parts, begins, ms, g0s = [], [], [], []
    pos = 0
    off = w.spec.seg_offsets
    flags_parts = []
    for s in seg_ids:
        a, b = int(off[s]), int(off[s + 1])
        t, f = synth.gen_tokens(w.spec, a, b)
        parts.append(t); flags_parts.append(f)
        begins.append(pos); ms.append(b - a); g0s.append(a); pos += b - a
    toks = np.concatenate(parts, axis=1) if parts else np.zeros((w.prob.n, 0), np.uint16)
    flags = np.concatenate(flags_parts) if w.spec.has_flags and parts else None
    t0 = time.perf_counter()
    oracle.simulate(w.prob, w.cost, np.asarray(seg_ids), np.array(begins), np.array(ms),
                    np.array(g0s, np.uint64), toks, flags, threads=threads, scheme=scheme, grid_den=grid_den)
    dt = time.perf_counter() - t0
    return pos, len(seg_ids), dt


def oracle_baseline(w, target_s=12.0, scheme=0, grid_den=0):
    """cpu_baseline: the oracle as it stands on the host cores, on a bounded,
    deterministic segment sample of the same workload (calibrated to
    ~target_s of CPU time)."""
    import oracle
    oracle.build()
    threads = os.cpu_count() or 1
    S = w.prob.R * w.prob.T
    off = w.spec.seg_offsets
    m = np.diff(off)
    # calibration on a few segments
    ids = synth.sample_segments(w.spec, 0, S, every=max(1, S // max(threads, 8)))[: max(threads, 8)]
    req, _, dt = oracle_sample_run(w, ids, threads, scheme, grid_den)
    rate = req / max(dt, 1e-6)
    want = int(rate * target_s)
    every = max(1, int(np.ceil(w.N / max(want, 1))))
    ids = synth.sample_segments(w.spec, 0, S, every=every)
    req, nseg, dt = oracle_sample_run(w, ids, threads, scheme, grid_den)
    # one thread: the first segments of the same sample, ~target_s / 4 of CPU
    n1 = max(1, int(len(ids) * min(1.0, (target_s / 4) / max(dt * threads, 1e-6))))
    req1, nseg1, dt1 = oracle_sample_run(w, ids[:n1], 1, scheme, grid_den)
    return {"value": req / dt, "unit": UNIT, "cores": threads, "kind": "oracle",
            "sample": f"{nseg} whole segments (every {every}th + first/last/largest) = {req:,} requests x "
                      f"{w.prob.X} xi cells, LP solves included, token generation excluded; {dt:.2f} s",
            "lp_cells_per_s": nseg * w.prob.X / dt,
            "one_thread": {"value": req1 / dt1, "unit": UNIT, "cores": 1,
                           "sample": f"the first {nseg1} segments of that sample = {req1:,} requests; {dt1:.2f} s"}}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = scheme_workload(args)
    scheme, grid_den = SCHEMES[args.scheme], args.grid_den
    import oracle
    oracle.build()
    threads = os.cpu_count() or 1
    S = w.prob.R * w.prob.T
    # each step: a bounded sample sized to ~2 s of host time
    ids = synth.sample_segments(w.spec, 0, S, every=max(1, S // 64))[:64]
    req, _, dt = oracle_sample_run(w, ids, threads, scheme, grid_den)
    rate = req / max(dt, 1e-6)
    every = max(1, int(np.ceil(w.N / max(int(rate * 2.0), 1))))
    ids = synth.sample_segments(w.spec, 0, S, every=every)
    for _ in range(args.warmup):
        oracle_sample_run(w, ids, threads, scheme, grid_den)
    times, reqs = [], 0
    for _ in range(args.steps):
        r, nseg, dt = oracle_sample_run(w, ids, threads, scheme, grid_den)
        times.append(dt); reqs += r
    total = sum(times)
    value = reqs / total
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64/u32",
            "data": "synthetic", "config": {"workload": workload_desc(w, args.scheme), "config": w.name,
                                            "scheme": args.scheme, "sample_segments": int(len(ids))},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "oracle",
                             "sample": f"{len(ids)} whole segments per step (every {every}th + first/last/largest), "
                                       f"{reqs // max(args.steps, 1):,} requests per step"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---------------------------------------------------------------- GPU arm


SCHEMES = {"sprout": 0, "co2opt": 1, "static": 2, "oracle": 3}   # oracle: NEXT-4's Oracle scheme


def scheme_workload(args):
    """The config's workload for the chosen scheme: Sprout keeps
    its xi cells; CO2_Opt has one cell per segment; the Sprout_Sta sweep one
    cell per point of the simplex grid of step 1/grid_den."""
    import dataclasses
    import math
    w = synth.make_workload(args.config)
    if args.scheme in ("sprout", "oracle"):
        return w
    X = 1 if args.scheme == "co2opt" else math.comb(args.grid_den + w.prob.n - 1, w.prob.n - 1)
    prob = dataclasses.replace(w.prob, X=X, xi=np.zeros(X))
    return dataclasses.replace(w, prob=prob, description=w.description + f" [{args.scheme}]")


def run_evaluator(args):
    """The opportunistic evaluator trigger sweep (Eq. 8; NEXT-2) on
    the config's CI traces: 64 urgencies x 64 thresholds per region, one
    sequential scan per configuration (one thread each)."""
    import torch
    from paper_2403_12900_b200 import sprout as S
    w = synth.make_workload(args.config, n_requests=1000)
    P = w.prob
    dt = 1.0 / 12 if args.config == "C3" else 1.0
    dev = torch.device("cuda", 0)
    betas, thetas = np.linspace(0.0, 0.1, 64), np.linspace(0.05, 1.0, 64)
    k2 = torch.as_tensor(P.k0, dtype=torch.float64, device=dev)
    kmax = torch.as_tensor(P.kmax, dtype=torch.float64, device=dev)
    out = torch.zeros((P.R, 64, 64, 4), dtype=torch.float64, device=dev)
    run = lambda: S.evaluator_sweep(k2, kmax, P.T, dt, betas, thetas, 6.0, 3, 0.2778, P.pue, out)
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    cfg = P.R * 64 * 64
    print(json.dumps({"metric": "evaluator trigger sweep: configuration-intervals/s", "value": cfg * P.T / (ms * 1e-3),
                      "unit": "config-intervals/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
                      "ms_per_step": ms, "higher_is_better": True, "dtype": "f64", "data": "synthetic",
                      "config": {"workload": f"{w.name} CI traces: {P.R} regions x {P.T} intervals x 64 beta x 64 "
                                             f"theta, grace 6 h, fallback 3", "configs": cfg},
                      "evaluations_total": float(out[..., 0].sum().item())}))


def run_sprout(args):
    import torch
    import torch.distributed as dist
    from paper_2403_12900_b200 import sprout as S
    from paper_2403_12900_b200.collective import allreduce_totals, max_over_ranks
    from paper_2403_12900_b200.runner import Sweep

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")

    # SPROUT_BENCH_SHARE_GPU=1 (functional test of the N > 1 path on a one-GPU box only: every
    # rank on device local % count, gloo; its timings are not a measurement)
    share = os.environ.get("SPROUT_BENCH_SHARE_GPU") == "1"
    if share:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    w = scheme_workload(args)
    scheme = SCHEMES[args.scheme]
    # closed-loop chains are per region: ranks take whole regions; otherwise request-balanced segments
    sh = synth.shard_regions(w.spec, w.prob.T, world, rank) if args.closed_loop else synth.shard(w.spec, world, rank)
    oracle_scheme = args.scheme == "oracle"
    sw = Sweep(w.prob, w.cost, sh, dev, spec=w.spec, scheme=0 if oracle_scheme else scheme, grid_den=args.grid_den)
    if oracle_scheme:   # the Sprout LP once: every cell's status for the reduction (the Oracle has no mix)
        sw.solve()
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    trace_bytes = sw.trace.tokens.numel() * 2 + (sw.trace.flags.numel() if sw.trace.flags is not None else 0)
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = trace_bytes < 4 * l2 or args.flush_l2
    flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if flush else None

    launches = [0]

    def step(ev=None):
        if not args.closed_loop and not oracle_scheme:   # the closed-loop scan solves every interval's LP itself
            sw.solve(); launches[0] += S.last_launch_count()
        if ev is not None:
            ev[0].record(stream)
        if args.closed_loop:
            qi = None
            if args.q_update:   # NEXT-1: q per evaluation epoch (Eq. 8 trigger, 500 samples; reading L24)
                qi, _ = sw.evaluation_q(24.0 / (w.prob.T / 365), 0.028, 0.5, 6.0, 3, 500); launches[0] += 1
            sw.closed_loop(args.closed_loop, q_interval=qi); launches[0] += S.last_launch_count()
        elif oracle_scheme:
            sw.oracle_scheme(); launches[0] += S.last_launch_count()
        else:
            sw.simulate(); launches[0] += S.last_launch_count()
        if ev is not None:
            ev[1].record(stream)
        sw.reduce(); launches[0] += S.last_launch_count()
        allreduce_totals(sw.group)      # the path's one exchange step (NCCL over NVLink for N > 1)
        if scheme == S.SCHEME_STATIC_GRID:
            sw.select_static(args.static_xi); launches[0] += S.last_launch_count()

    for _ in range(args.warmup):
        if flush:
            flush_buf.zero_()
        step()
    torch.cuda.synchronize()
    graph = None
    # one GPU, the Sprout step: CUDA-graph replay by default (--no-graph for eager launches)
    if args.graph is None:
        args.graph = world == 1 and scheme == S.SCHEME_SPROUT and not args.closed_loop and not oracle_scheme
    if args.graph:   # the whole step (all its launches + the all-reduce) as one CUDA graph replay
        graph = sw.capture(step)
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches[0] = 0
    sim_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for k in range(args.steps):
            if flush:
                flush_buf.zero_()       # L2 flush between steps (outside the per-step events)
            step_ev[k][0].record(stream)
            if graph is not None:
                graph.replay()
            else:
                step(sim_ev[k])
            step_ev[k][1].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in step_ev]
    if graph is not None:   # the simulate launch alone, eagerly, for the roofline
        for k in range(args.steps):
            if flush:
                flush_buf.zero_()
            step(sim_ev[k])
        torch.cuda.synchronize()
    sim_ms = [a.elapsed_time(b) for a, b in sim_ev]
    total_ms = max_over_ranks(sum(step_ms), dev)
    ms_per_step = total_ms / args.steps

    # LP cells/s: the solve kernel alone
    lp_ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    lp_ev[0].record(stream)
    for _ in range(args.steps):
        sw.solve()
    lp_ev[1].record(stream)
    torch.cuda.synchronize()
    lp_ms = max_over_ranks(lp_ev[0].elapsed_time(lp_ev[1]) / args.steps, dev)

    status = int(sw.totals.trace_status.item())
    g = sw.group.cpu().numpy()

    # cross-check after the timed steps: the fp64 per-request accounting mode (Eq. 1 per
    # request, fp64 warp-shuffle / block tree sums) against the streaming kernel's closed
    # form, every cell of the full workload (sprout_cell_totals_fp64)
    fp64_check = {}
    if args.fp64_check and scheme == S.SCHEME_SPROUT and not args.closed_loop and not oracle_scheme:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        f64 = S.cell_totals_fp64(sw.dp, sw.sol, sw.trace, sw.cost)
        e1.record(stream)
        torch.cuda.synchronize()
        t = sw.totals
        diffs = {}
        for k, ref in (("energy", t.energy), ("time", t.time), ("carbon", t.carbon), ("quality", t.quality)):
            den = torch.clamp(ref.abs(), min=1e-300)
            diffs[k] = float(((f64[k] - ref).abs() / den).max().item()) if ref.numel() else 0.0
        fp64_check = {"fp64_per_request_max_rel_diff": max(diffs.values()) if diffs else 0.0,
                      "fp64_per_request_ms": e0.elapsed_time(e1)}

    # NEXT-4 reporting (untimed by the step; each kernel timed on its own)
    extras = {}
    if args.preference and not args.closed_loop:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if oracle_scheme:
            e0.record(stream); st = sw.oracle_scheme()["stats"]; e1.record(stream)
        else:
            e0.record(stream); st = sw.preference_stats(); e1.record(stream)
        torch.cuda.synchronize()
        st = st.view(sh.n_segments, w.prob.X, 3).sum(dim=0).double().cpu().numpy()
        m = float(w.N)
        pick = sorted({0, w.prob.X // 2, w.prob.X - 1})
        extras["preference"] = {
            "reading": "L22: head-to-head vs Base, ties half; score = w/(1-w) (P:377)",
            "kernel_ms": e0.elapsed_time(e1),
            "by_xi": [{"xi": float(w.prob.xi[j]), "hit_rate": st[j, 0] / m,
                       "w": (st[j, 1] + (m - st[j, 1] - st[j, 2]) / 2) / m,
                       "normalized_preference": S.normalized_preference((st[j, 1] + (m - st[j, 1] - st[j, 2]) / 2) / m)}
                      for j in pick]}
    if args.request_cdf >= 0 and not args.closed_loop and not oracle_scheme:
        j = min(args.request_cdf, w.prob.X - 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream); ro = sw.request_outputs(j); e1.record(stream)
        torch.cuda.synchronize()
        r = ro["ratio"]
        r = r[~torch.isnan(r)]
        edges = [0.1 * k for k in range(1, 11)]
        extras["request_cdf"] = {"xi": float(w.prob.xi[j]), "kernel_ms": e0.elapsed_time(e1),
                                 "requests": int(r.numel()),
                                 "fraction_at_or_below": {f"{x:.1f}": float((r <= x).double().mean().item()) for x in edges}}
        del ro, r

    # e2e: the host-buffer C-ABI call (H2D of the trace + D2H of the totals timed)
    e2e = None
    if not args.no_e2e and scheme == S.SCHEME_SPROUT and not args.closed_loop:
        e2e = run_e2e(args, w, sh, sw, dev, world)

    # the roofline's bytes and time over the job (collectives: every rank, before rank 0 reports):
    # per-GPU average = all ranks' algorithmic bytes over the slowest rank's simulate time
    alg = algorithmic_bytes(w, sh)
    if args.closed_loop:   # the trace once (the chains of a region share it) + every interval's LP outputs
        P = w.prob
        alg = algorithmic_bytes(w, sh) + sh.n_segments * P.X * (P.n * 8 + 8 + 8)
    sim_job_ms = (statistics.mean(sim_ms), statistics.median(sim_ms))
    if world > 1:
        t = torch.tensor([float(alg)], dtype=torch.float64, device=dev)
        dist.all_reduce(t)
        alg = float(t.item()) / world
        sim_job_ms = (max_over_ranks(sim_job_ms[0], dev), max_over_ranks(sim_job_ms[1], dev))

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = peaks()
    sim_avg_ms, sim_med_ms = sim_job_ms
    achieved = alg / (sim_avg_ms * 1e-3) / 1e9
    traffic = None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):   # ncu DRAM bytes per launch, keyed by the measured (config, scheme, mode, GPUs)
        key = f"{w.name}/{args.scheme}/{'closed' if args.closed_loop else 'open'}/{world}"
        traffic = json.load(open(tf)).get(key, {}).get("dram_bytes_per_launch")
    cpu = None
    if not args.no_cpu_baseline and world == 1 and not args.closed_loop and not oracle_scheme:
        cpu = oracle_baseline(w, args.cpu_seconds, scheme, args.grid_den)
    N = w.N
    line = {
        "metric": METRIC, "value": N / (ms_per_step * 1e-3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "ms_per_step_median": statistics.median(step_ms), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64/u32", "data": "synthetic",
        "config": {"workload": workload_desc(w, args.scheme) + (f" [closed loop, window {args.closed_loop}"
                                                                   f"{', q per evaluation epoch' if args.q_update else ''}]"
                                                                   if args.closed_loop else ""),
                   "config": w.name, "scheme": args.scheme, "closed_loop_window": args.closed_loop, "requests": N,
                   "lp_cells": w.prob.C,
                   "parallelism": f"segments sharded over {world} GPU(s), one NCCL allreduce of group totals",
                   "cuda_graph": bool(args.graph),
                   "l2": ("flushed (256 MB memset) between steps" if flush else
                          f"inputs larger than L2 (trace {trace_bytes / 1e9:.2f} GB/GPU > L2 {l2 / 1e6:.0f} MB)")},
        "lp_cells_per_s": w.prob.C / (lp_ms * 1e-3),
        "request_cells_per_s": N * w.prob.X / (ms_per_step * 1e-3),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "kernel": ("sprout_simulate_closed_loop (one CTA per group of xi chains "
                                                    "of a region)" if args.closed_loop else
                                                    "sprout_simulate_oracle_scheme (one CTA per segment: per-request "
                                                    "costs, radix sort by extra carbon)" if oracle_scheme
                                                    else "sprout_simulate_trace (prep + trace_kernel, CUDA events)"),
                     "algorithmic_bytes_per_launch": alg, "launch_ms": sim_avg_ms, "launch_ms_median": sim_med_ms,
                     "frac_median": alg / (sim_med_ms * 1e-3) / 1e9 / peak, "peak_source": peak_src},
        "clocks": clk.summary(),
        "gpu_launches": launches[0],
        "e2e": e2e,
        "cpu_baseline": cpu,
        "trace_status": status,
        **extras,
        "check": {"requests_counted": float(g[-1, 0, 0]),
                  "carbon_saving_xi_max": float(1 - g[-1, -1, 4] / g[-1, -1, 8]) if g[-1, -1, 8] > 0 else None,
                  **fp64_check},
    }
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, w, sh, sw, dev, world):
    import ctypes as C
    import torch
    import torch.distributed as dist
    from paper_2403_12900_b200 import sprout as S
    from paper_2403_12900_b200.collective import allreduce_totals, max_over_ranks

    P = w.prob
    tok_dev = sw.trace.tokens
    tok_host = torch.empty(tok_dev.shape, dtype=tok_dev.dtype, pin_memory=True)
    tok_host.copy_(tok_dev)
    fl_host = None
    if sw.trace.flags is not None:
        fl_host = torch.empty(sw.trace.flags.shape, dtype=torch.uint8, pin_memory=True)
        fl_host.copy_(sw.trace.flags)
    keep = []

    def pinned(a, dt):
        t = torch.from_numpy(np.ascontiguousarray(a, dt)).pin_memory()
        keep.append(t)
        return t.data_ptr()

    lp = S.LpProblem(P.n, P.R, P.T, P.X, P.profile_per_interval, pinned(P.k0, np.float64),
                     pinned(P.kmin, np.float64), pinned(P.kmax, np.float64), pinned(P.xi, np.float64),
                     pinned(P.e, np.float64), pinned(P.p, np.float64), pinned(P.q, np.float64), P.k1, P.pue,
                     sh.first_segment, sh.n_segments)
    tr = S.Trace(sh.n_requests, sh.first_request, pinned(sh.seg_offsets, np.int64), tok_host.data_ptr(),
                 tok_dev.shape[1], fl_host.data_ptr() if fl_host is not None else None)
    cm = S.cost_model(w.cost)
    ws = S.workspace(S.sweep_workspace_bytes(lp, tr, w.cost.n_classes), dev)
    out = torch.zeros((P.R + 1) * P.X * S.group_stat_count(P.n), dtype=torch.float64).pin_memory().numpy()
    st = torch.zeros(1, dtype=torch.int32).pin_memory().numpy()
    stream = torch.cuda.current_stream()
    steps = max(3, min(args.steps, args.e2e_steps))
    for _ in range(2):
        S.sweep_host(lp, tr, cm, out, st, ws)
    if world > 1:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(steps):
        S.sweep_host(lp, tr, cm, out, st, ws)
        if world > 1:
            g = torch.from_numpy(out).to(dev)
            allreduce_totals(g)
            out[:] = g.cpu().numpy()
    ev1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / steps, dev)
    h2d = (tok_host.numel() * 2 + (fl_host.numel() if fl_host is not None else 0) + (sh.n_segments + 1) * 8
           + P.k0.size * 8 + (P.e.size + P.p.size + P.q.size + P.xi.size + 2 * P.R) * 8)
    d2h = out.size * 8 + 4
    del ws
    return {"value": w.N / (ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": ms, "steps": steps, "api": "sprout_sweep_host (C ABI, pinned host buffers)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4", choices=synth.CONFIGS)
    ap.add_argument("--impl", default="sprout", choices=["sprout", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--flush-l2", action="store_true")
    ap.add_argument("--scheme", default="sprout", choices=sorted(SCHEMES),
                    help="competing scheme of P:364-373 (co2opt, static = the Sprout_Sta grid sweep)")
    ap.add_argument("--grid-den", type=int, default=20, help="static grid step 1/D (Sprout_Sta sweep)")
    ap.add_argument("--static-xi", type=float, default=0.1, help="xi of the Sprout_Sta quality floor")
    ap.add_argument("--closed-loop", type=int, default=0, metavar="W",
                    help="closed-loop profiles (NEXT-1): window of W requests per level; 0 = open loop")
    ap.add_argument("--graph", dest="graph", action="store_true", default=None,
                    help="replay the step as one captured CUDA graph (runner.Sweep.capture); "
                         "the default on one GPU for the Sprout step")
    ap.add_argument("--no-graph", dest="graph", action="store_false", help="eager launches")
    ap.add_argument("--no-fp64-check", dest="fp64_check", action="store_false",
                    help="skip the after-the-run fp64 per-request cross-check of every cell")
    ap.add_argument("--q-update", action="store_true",
                    help="with --closed-loop: q updated per evaluation epoch (NEXT-1, reading L24) inside each step")
    ap.add_argument("--preference", action="store_true",
                    help="NEXT-4: head-to-head preference vs Base per xi (reading L22, P:377) after the timed steps")
    ap.add_argument("--request-cdf", type=int, default=-1, metavar="J",
                    help="NEXT-4: per-request carbon / Base of xi column J (Fig. eval2 CDF points) after the timed steps")
    ap.add_argument("--evaluator", action="store_true",
                    help="time the opportunistic evaluator trigger sweep (Eq. 8) instead of the hot path")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.evaluator:
        run_evaluator(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_sprout(args)


if __name__ == "__main__":
    main()
