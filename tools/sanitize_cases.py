"""Small invocations of every kernel of the library, for compute-sanitizer
(memcheck / racecheck / synccheck): the trace kernel (histogram path, C2
shape with flags and 3 xi), the one-cell kernel (C1, C3 shape), the closed
loop (+ q per epoch), the NEXT-4 kernels, the competing schemes, the
evaluator sweep, the grouped one-cell kernel (short segments, with and
without verify mode) and the fp64 per-request accounting mode.  Usage: compute-sanitizer --tool T python tools/sanitize_cases.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2403_12900_b200 import sprout as S
from paper_2403_12900_b200.runner import Sweep

DEV = "cuda:0"


def run(name, **kw):
    w = synth.make_workload(name, **kw)
    sh = synth.shard(w.spec, 1, 0)
    toks, fl = synth.host_trace(w.spec, sh)
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=fl)
    sw.solve(); sw.simulate(levels=True); sw.simulate(); sw.reduce()
    S.cell_totals_fp64(sw.dp, sw.sol, sw.trace, sw.cost)
    sw.preference_stats(); sw.request_outputs(0); sw.oracle_scheme()
    q, _ = sw.evaluation_q(24.0 / (w.prob.T / 365) if w.prob.T >= 365 else 1.0, 0.028, 0.5, 6.0, 3, 100)
    sw.closed_loop(20, profile=True, q_interval=q); sw.reduce()
    torch.cuda.synchronize()
    st = int(sw.totals.trace_status.item())
    print(name, kw, "trace_status", st)


run("C1")
run("C2", n_requests=20_000, n_intervals=24)
run("C3", n_requests=12_000, n_intervals=48, n_regions=2)
run("C4", n_requests=60_000, n_intervals=6, n_regions=2)
# competing schemes and the evaluator sweep
w = synth.make_workload("C2", n_requests=10_000, n_intervals=24)
sh = synth.shard(w.spec, 1, 0)
toks, fl = synth.host_trace(w.spec, sh)
for scheme, den in ((S.SCHEME_CO2_OPT, 0), (S.SCHEME_STATIC_GRID, 6)):
    import dataclasses
    X = 1 if scheme == S.SCHEME_CO2_OPT else S.static_grid_size(w.prob.n, den)
    prob = dataclasses.replace(w.prob, X=X, xi=np.zeros(X))
    sw = Sweep(prob, w.cost, sh, DEV, tokens=toks, flags=fl, scheme=scheme, grid_den=den)
    sw.solve(); sw.simulate(); sw.reduce()
    if scheme == S.SCHEME_STATIC_GRID:
        sw.select_static(0.1)
    torch.cuda.synchronize()
    print("scheme", scheme, "ok")
k2 = torch.as_tensor(np.asarray(w.prob.k0)).to(DEV)
k2m = torch.as_tensor(np.asarray(w.prob.kmax)).to(DEV)
out = torch.zeros((w.prob.R, 4, 4, 4), dtype=torch.float64, device=DEV)
S.evaluator_sweep(k2, k2m, w.prob.T, 1.0, [0.0, 0.01, 0.028, 0.1], [0.3, 0.5, 0.7, 1.0], 6.0, 3, 0.2778, 1.2, out)
torch.cuda.synchronize()
print("evaluator ok")
