"""Runs every Sweep entry point at the API's limits (xi count up to
SPROUT_MAX_XI, 8 levels, 4 classes with flags, windows up to the shared-memory
bound, ragged and empty intervals) and reports CUDA errors; no oracle."""
import os
import sys
import traceback

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import synth  # noqa: E402
from paper_2403_12900_b200 import sprout as S  # noqa: E402
from paper_2403_12900_b200.runner import Sweep  # noqa: E402
from test_gpu_parity import _custom  # noqa: E402

CASES = [dict(n=3, X=4096), dict(n=8, X=4096), dict(n=8, X=64, NC=4, flags=True), dict(n=2, X=4096, NC=4, flags=True),
         dict(n=5, X=1000, NC=3, flags=True), dict(n=1, X=4096)]


def run(case):
    w = _custom(N=20_000, T=5, R=2, **case)
    off = w.spec.seg_offsets
    m = np.diff(off); m[::3] = 0; off[1:] = np.cumsum(m)
    sh = synth.shard(w.spec, 1, 0)
    toks, fl = synth.host_trace(w.spec, sh)
    sw = Sweep(w.prob, w.cost, sh, "cuda:0", tokens=toks, flags=fl)
    steps = [("solve", lambda: sw.solve()), ("simulate+levels", lambda: sw.simulate(levels=True)),
             ("reduce", lambda: sw.reduce()),
             ("closed_loop W=1", lambda: sw.closed_loop(1)),
             ("closed_loop Wmax", lambda: sw.closed_loop(min(4096, (96 * 1024) // (4 * case["n"])))),
             ("evaluation_q", lambda: sw.evaluation_q(1.0, 0.028, 0.5, 6.0, 0, 500)),
             ("request_outputs", lambda: (sw.solve(), sw.request_outputs(case["X"] - 1))),
             ("preference_stats", lambda: sw.preference_stats()),
             ("oracle_scheme", lambda: sw.oracle_scheme())]
    for name, fn in steps:
        try:
            fn()
            torch.cuda.synchronize()
            print(f"  {name}: ok", flush=True)
        except Exception as e:  # noqa: BLE001
            print(f"  {name}: FAIL {e}", flush=True)
            if "CUDA" in str(e):
                traceback.print_exc(limit=1)


for c in CASES:
    print(c, flush=True)
    try:
        run(c)
    except Exception as e:  # noqa: BLE001
        print("  setup FAIL", e, flush=True)
