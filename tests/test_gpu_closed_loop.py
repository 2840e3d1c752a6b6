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


@pytest.mark.parametrize("name,kw,W", [("C2", dict(n_requests=60_000, n_intervals=48), 200),
                                       ("C3", dict(n_requests=30_000, n_intervals=72, n_regions=2), 50),
                                       ("C4", dict(n_requests=120_000, n_intervals=24, n_regions=2), 1000)])
def test_closed_loop_then_reduce(name, kw, W):
    """The closed-loop step alone gives complete totals:
    segment statistics and the Base counterfactual equal the open-loop
    oracle's (they do not depend on the scheme), and reduce() over the
    closed-loop cells equals oracle.reduce over the oracle's closed-loop cells."""
    w = synth.make_workload(name, **kw)
    sh = synth.shard(w.spec, 1, 0)
    toks, fl = synth.host_trace(w.spec, sh)
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=fl)
    sw.closed_loop(W)
    sw.reduce()
    torch.cuda.synchronize()
    got = sw.host()
    cl = oracle.closed_loop(w.prob, w.cost, W, w.spec.seg_offsets, toks, fl)
    S_ = w.prob.R * w.prob.T
    off = w.spec.seg_offsets
    sim = oracle.simulate(w.prob, w.cost, np.arange(S_), off[:-1], np.diff(off), off[:-1], toks, fl)
    np.testing.assert_array_equal(got["seg_count"].reshape(sim["seg_count"].shape), sim["seg_count"])
    np.testing.assert_array_equal(got["seg_pinned"].reshape(sim["seg_pinned"].shape), sim["seg_pinned"])
    np.testing.assert_array_equal(got["seg_tok"].reshape(sim["seg_tok"].shape), sim["seg_tok"])
    np.testing.assert_allclose(got["seg_base"].reshape(sim["seg_base"].shape), sim["seg_base"], rtol=FP_RTOL, atol=0)
    np.testing.assert_array_equal(got["objective"].view(np.uint64), cl["objective"].view(np.uint64))
    X, NC, n = w.prob.X, w.cost.n_classes, w.prob.n
    cells = dict(cell_status=cl["cell_status"], objective=cl["objective"])
    simc = dict(cnt=cl["cnt"].reshape(S_, X, NC, n), tok=cl["tok"].reshape(S_, X, NC, n),
                energy=cl["energy"].reshape(S_, X), time=cl["time"].reshape(S_, X),
                carbon=cl["carbon"].reshape(S_, X), quality=cl["quality"].reshape(S_, X),
                seg_count=sim["seg_count"], seg_pinned=sim["seg_pinned"], seg_base=sim["seg_base"])
    simc = {k: np.ascontiguousarray(v) for k, v in simc.items()}
    G = oracle.reduce(w.prob, NC, 0, S_, cells, simc)
    np.testing.assert_allclose(got["group"], G, rtol=FP_RTOL, atol=0)
    assert got["group"][-1, 0, 0] == w.N   # every request counted (group stat 0)
    assert got["trace_status"] == 0


def test_closed_loop_bad_offsets():
    """Invalid offsets are flagged and the interval skipped: its
    cells and segment fields are zero and nothing enters the windows, as in
    sprout_simulate_trace."""
    w = synth.make_workload("C2", n_requests=20_000, n_intervals=24)
    sh = synth.shard(w.spec, 1, 0)
    toks, fl = synth.host_trace(w.spec, sh)
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=fl)
    bad = sh.seg_offsets.copy()
    T = w.prob.T
    bad[5] = sh.n_requests + 100    # segment 4 ends past the trace, segment 5 starts there
    sw.trace.seg_offsets.copy_(torch.as_tensor(bad))
    sw.closed_loop(50)
    sw.reduce()
    torch.cuda.synchronize()
    got = sw.host()
    assert got["trace_status"] & S.TRACE_BAD_OFFSETS
    X, NC, n = w.prob.X, w.cost.n_classes, w.prob.n
    cnt = got["cnt"].reshape(-1, X, NC, n)
    assert cnt[4].sum() == 0 and cnt[5].sum() == 0
    assert got["seg_count"].reshape(-1, NC)[4].sum() == 0
    assert np.all(got["carbon"].reshape(-1, X)[4] == 0)
    # other regions are untouched: region 1 equals the oracle run on the good offsets
    want = oracle.closed_loop(w.prob, w.cost, 50, w.spec.seg_offsets, toks, fl)
    lo, hi = T * X, 2 * T * X
    np.testing.assert_array_equal(got["cnt"].reshape(-1, NC, n)[lo:hi], want["cnt"][lo:hi])


@pytest.mark.parametrize("name,kw,dt,grace,sample", [("C2", dict(n_requests=60_000, n_intervals=240), 1.0, 6.0, 500),
                                                     ("C3", dict(n_requests=40_000, n_intervals=288, n_regions=2),
                                                      1 / 12, 2.0, 500),
                                                     ("C4", dict(n_requests=200_000, n_intervals=96), 1.0, 6.0, 37)])
def test_evaluation_q_and_closed_loop_q(name, kw, dt, grace, sample):
    """NEXT-1's q update (reading L24): every interval's epoch q and the
    evaluation flags bit-exact; the closed loop with those q bit-exact."""
    w = synth.make_workload(name, **kw)
    sh = synth.shard(w.spec, 1, 0)
    toks, fl = synth.host_trace(w.spec, sh)
    P = w.prob
    sw = Sweep(P, w.cost, sh, DEV, tokens=toks, flags=fl)
    q, fired = sw.evaluation_q(dt, 0.028, 0.5, grace, 3, sample)
    prof = sw.closed_loop(100, profile=True, q_interval=q)
    torch.cuda.synchronize()
    got = sw.host()
    wq, wf = oracle.evaluation_q(P.k0, P.kmax, P.T, dt, 0.028, 0.5, grace, 3, np.asarray(P.q), w.cost.seed,
                                 w.spec.seg_offsets, sample)
    np.testing.assert_array_equal(fired.cpu().numpy(), wf)
    np.testing.assert_array_equal(q.cpu().numpy().view(np.uint64), wq.view(np.uint64))
    want = oracle.closed_loop(P, w.cost, 100, w.spec.seg_offsets, toks, fl, q_seg=wq)
    NC, n = w.cost.n_classes, P.n
    np.testing.assert_array_equal(prof.cpu().numpy().view(np.uint64), want["profile"].view(np.uint64))
    np.testing.assert_array_equal(got["x"].view(np.uint64), want["x"].view(np.uint64))
    np.testing.assert_array_equal(got["cnt"].reshape(-1, NC, n), want["cnt"])
    np.testing.assert_allclose(got["quality"].reshape(-1), want["quality"], rtol=FP_RTOL, atol=0)
    np.testing.assert_allclose(got["carbon"].reshape(-1), want["carbon"], rtol=FP_RTOL, atol=0)


@pytest.mark.parametrize("n,NC,flags,W", [(1, 1, False, 3), (8, 1, False, 40), (4, 4, True, 25), (2, 3, True, 1),
                                            (3, 1, True, 25), (2, 1, False, 2000), (4, 1, True, 700)])
def test_closed_loop_levels_classes_ragged(n, NC, flags, W):
    """The chain kernel's other template instances (n = 1, n = 8, four
    classes, flags with one class, large windows) on ragged intervals: empty
    ones, single requests, and one longer than several scan pieces."""
    from test_gpu_parity import _custom
    w = _custom(n=n, X=3, NC=NC, flags=flags, N=30_000, T=30, R=2, xi=[0.0, 0.35, 1.0])
    off = w.spec.seg_offsets
    m = np.diff(off)
    m[::5] = 0
    m[3] = 1
    m[8] = 9000
    off[1:] = np.cumsum(m)
    sh = synth.shard(w.spec, 1, 0)
    toks, fl = synth.host_trace(w.spec, sh)
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=fl)
    prof = sw.closed_loop(W, profile=True)
    torch.cuda.synchronize()
    got = sw.host()
    want = oracle.closed_loop(w.prob, w.cost, W, w.spec.seg_offsets, toks, fl)
    np.testing.assert_array_equal(prof.cpu().numpy().view(np.uint64), want["profile"].view(np.uint64))
    np.testing.assert_array_equal(got["x"].view(np.uint64), want["x"].view(np.uint64))
    np.testing.assert_array_equal(got["cnt"].reshape(-1, NC, n), want["cnt"])
    np.testing.assert_array_equal(got["tok"].reshape(-1, NC, n), want["tok"])
    for k in ("energy", "time", "carbon", "quality"):
        np.testing.assert_allclose(got[k].reshape(-1), want[k], rtol=FP_RTOL, atol=0, err_msg=k)


@pytest.mark.parametrize("X,N,T,NC,flags", [(2100, 3000, 4, 1, False), (37, 400_000, 6, 1, False),
                                             (5, 300_000, 5, 2, True)])
def test_closed_loop_chain_schedule(X, N, T, NC, flags):
    """The chain schedule is scheduling only: with more chains than the rank
    kernel orders (R*X > 4000: index order) and with long intervals (the
    512-thread chains, longest first), every output still equals the oracle's."""
    from test_gpu_parity import _custom
    w = _custom(X=X, R=2, T=T, N=N, NC=NC, flags=flags)
    sh = synth.shard(w.spec, 1, 0)
    toks, fl = synth.host_trace(w.spec, sh)
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=fl)
    prof = sw.closed_loop(50, profile=True)
    torch.cuda.synchronize()
    got = sw.host()
    want = oracle.closed_loop(w.prob, w.cost, 50, w.spec.seg_offsets, toks, fl)
    np.testing.assert_array_equal(prof.cpu().numpy().view(np.uint64), want["profile"].view(np.uint64))
    np.testing.assert_array_equal(got["x"].view(np.uint64), want["x"].view(np.uint64))
    np.testing.assert_array_equal(got["cnt"].reshape(want["cnt"].shape), want["cnt"])
    np.testing.assert_allclose(got["carbon"].reshape(-1), want["carbon"], rtol=FP_RTOL, atol=0)
