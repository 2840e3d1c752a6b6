"""Closed-loop wave experiment: C4 (5 regions x 8760 intervals, 10^9 requests,
W = 1000) with the first X of the 64 xi values, X chosen around the 296
resident chain slots of one B200 (148 SMs x 2 CTAs).  Prints ms per
closed-loop call (chain kernel + the streaming simulate) per X.
Usage: python tools/cl_tail.py [X ...]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2403_12900_b200.runner import Sweep  # noqa: E402


def main():
    xs = [int(v) for v in sys.argv[1:]] or [29, 59, 64]
    dev = torch.device("cuda", 0)
    for X in xs:
        w = synth.make_workload("C4", xi=np.arange(64)[:X] / 63.0)
        sh = synth.shard_regions(w.spec, w.prob.T, 1, 0)
        sw = Sweep(w.prob, w.cost, sh, dev, spec=w.spec)
        sw.closed_loop(1000)
        torch.cuda.synchronize()
        ts = []
        for _ in range(2):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            sw.closed_loop(1000)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"X={X} chains={5 * X} ms={min(ts):.2f} ({', '.join(f'{t:.2f}' for t in ts)})", flush=True)
        del sw
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
