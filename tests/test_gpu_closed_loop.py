"""GPU parity of closed-loop profiles (NEXT-1; reading L20) through
the C ABI vs the oracle: the profiles each interval used, the LP solution and
the integer statistics bit-exact; fp64 totals within 1e-9."""
import numpy as np
import pytest
import torch

import oracle
import synth
from parity_util import FP_RTOL

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2403_12900_b200 import sprout as S
    from paper_2403_12900_b200.runner import Sweep

DEV = "cuda:0"


@pytest.mark.parametrize("name,kw,W", [("C1", {}, 1), ("C1", {}, 7), ("C2", dict(n_requests=60_000, n_intervals=48), 1000),
                                       ("C3", dict(n_requests=40_000, n_intervals=96), 50),
                                       ("C5", dict(n_requests=50_000, n_intervals=24, n_regions=3), 300),
                                       ("C4", dict(n_requests=80_000, n_intervals=24), 4096)])
def test_closed_loop_parity(name, kw, W):
    w = synth.make_workload(name, **kw)
    sh = synth.shard(w.spec, 1, 0)
    toks, fl = synth.host_trace(w.spec, sh)
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=fl)
    prof = sw.closed_loop(W, profile=True)
    torch.cuda.synchronize()
    got = sw.host()
    want = oracle.closed_loop(w.prob, w.cost, W, w.spec.seg_offsets, toks, fl)
    NC, n = w.cost.n_classes, w.prob.n
    np.testing.assert_array_equal(prof.cpu().numpy().view(np.uint64), want["profile"].view(np.uint64))
    np.testing.assert_array_equal(got["x"].view(np.uint64), want["x"].view(np.uint64))
    np.testing.assert_array_equal(got["cell_status"], want["cell_status"])
    if n > 1:
        np.testing.assert_array_equal(got["threshold"].astype(np.uint64), np.minimum(want["threshold"], 0xFFFFFFFF))
    np.testing.assert_array_equal(got["cnt"].reshape(-1, NC, n), want["cnt"])
    np.testing.assert_array_equal(got["tok"].reshape(-1, NC, n), want["tok"])
    for k in ("energy", "time", "carbon", "quality"):
        np.testing.assert_allclose(got[k].reshape(-1), want[k], rtol=FP_RTOL, atol=0, err_msg=k)
    assert got["trace_status"] == 0


@pytest.mark.parametrize("world", [2, 3])
def test_closed_loop_region_shards(world):
    """Chains are per region, so ranks can take whole regions: every rank's
    cells equal the single-device run's (oracle) cells bit for bit."""
    w = synth.make_workload("C2", n_requests=50_000, n_intervals=48)
    want = oracle.closed_loop(w.prob, w.cost, 200, w.spec.seg_offsets, *synth.host_trace(w.spec, synth.shard(w.spec, 1, 0)))
    X, NC, n = w.prob.X, w.cost.n_classes, w.prob.n
    for rank in range(world):
        sh = synth.shard_regions(w.spec, w.prob.T, world, rank)
        if sh.n_segments == 0:
            continue
        toks, fl = synth.host_trace(w.spec, sh)
        sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=fl)
        prof = sw.closed_loop(200, profile=True)
        torch.cuda.synchronize()
        got = sw.host()
        lo, hi = sh.first_segment * X, (sh.first_segment + sh.n_segments) * X
        np.testing.assert_array_equal(prof.cpu().numpy().view(np.uint64), want["profile"][lo:hi].view(np.uint64))
        np.testing.assert_array_equal(got["x"].view(np.uint64), want["x"][lo:hi].view(np.uint64))
        np.testing.assert_array_equal(got["cnt"].reshape(-1, NC, n), want["cnt"][lo:hi])
        np.testing.assert_array_equal(got["tok"].reshape(-1, NC, n), want["tok"][lo:hi])
        np.testing.assert_allclose(got["carbon"].reshape(-1), want["carbon"][lo:hi], rtol=FP_RTOL, atol=0)
