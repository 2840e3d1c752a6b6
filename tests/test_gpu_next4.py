"""GPU parity of NEXT-4 through the C ABI vs the oracle (readings L21-L23):
per-request levels, latent best levels bit-exact and carbon / Base carbon /
ratio bit-exact (same operation order, no FMA); per-cell head-to-head
statistics bit-exact."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2403_12900_b200 import sprout as S
    from paper_2403_12900_b200.runner import Sweep

DEV = "cuda:0"


def _sweep(name, **kw):
    w = synth.make_workload(name, **kw)
    sh = synth.shard(w.spec, 1, 0)
    toks, fl = synth.host_trace(w.spec, sh)
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=fl)
    sw.solve()
    return w, sh, toks, fl, sw


@pytest.mark.parametrize("name,kw,j", [("C1", {}, 0), ("C2", dict(n_requests=40_000, n_intervals=48), 2),
                                       ("C3", dict(n_requests=30_000, n_intervals=96), 0),
                                       ("C4", dict(n_requests=200_000, n_intervals=24), 37),
                                       ("C5", dict(n_requests=40_000, n_intervals=24, n_regions=4), 0)])
def test_request_outputs_bit_exact(name, kw, j):
    w, sh, toks, fl, sw = _sweep(name, **kw)
    got = {k: v.cpu().numpy() for k, v in sw.request_outputs(j).items()}
    want = oracle.request_outputs(w.prob, w.cost, w.spec.seg_offsets, toks, fl, j=j)
    np.testing.assert_array_equal(got["level"], want["level"])
    np.testing.assert_array_equal(got["pref"], want["pref"])
    for k in ("carbon", "base", "ratio"):
        np.testing.assert_array_equal(got[k].view(np.uint64), want[k].view(np.uint64), err_msg=k)


@pytest.mark.parametrize("name,kw", [("C1", {}), ("C2", dict(n_requests=40_000, n_intervals=48)),
                                     ("C3", dict(n_requests=30_000, n_intervals=96)),
                                     ("C4", dict(n_requests=150_000, n_intervals=12))])
def test_preference_stats_bit_exact(name, kw):
    w, sh, toks, fl, sw = _sweep(name, **kw)
    got = sw.preference_stats().cpu().numpy().view(np.uint64)
    want = oracle.preference(w.prob, w.cost, w.spec.seg_offsets, fl)
    np.testing.assert_array_equal(got, want)


def test_normalized_preference_host():
    assert S.normalized_preference(0.48) == pytest.approx(0.923, abs=1e-3)
    assert S.normalized_preference(0.5) == 1.0
    assert S.normalized_preference(1.0) == float("inf")


@pytest.mark.parametrize("name,kw", [("C1", {}), ("C2", dict(n_requests=40_000, n_intervals=48)),
                                     ("C3", dict(n_requests=30_000, n_intervals=96)),
                                     ("C4", dict(n_requests=300_000, n_intervals=12)),
                                     ("C5", dict(n_requests=30_000, n_intervals=24, n_regions=4))])
def test_oracle_scheme_parity(name, kw):
    w, sh, toks, fl, sw = _sweep(name, **kw)
    res = sw.oracle_scheme()
    torch.cuda.synchronize()
    got = sw.host()
    want = oracle.oracle_scheme(w.prob, w.cost, w.spec.seg_offsets, toks, fl)
    NC, n = w.cost.n_classes, w.prob.n
    np.testing.assert_array_equal(res["cell_status"].cpu().numpy(), want["status"])
    np.testing.assert_array_equal(res["stats"].cpu().numpy().view(np.uint64), want["stats"])
    np.testing.assert_array_equal(got["cnt"].reshape(-1, NC, n), want["cnt"])
    np.testing.assert_array_equal(got["tok"].reshape(-1, NC, n), want["tok"])
    for k in ("energy", "time", "carbon", "quality"):
        np.testing.assert_allclose(got[k].reshape(-1), want[k], rtol=1e-9, atol=0, err_msg=k)
    S_ = w.prob.R * w.prob.T
    off = w.spec.seg_offsets
    sim = oracle.simulate(w.prob, w.cost, np.arange(S_), off[:-1], np.diff(off), off[:-1], toks, fl)
    np.testing.assert_array_equal(got["seg_count"].reshape(sim["seg_count"].shape), sim["seg_count"])
    np.testing.assert_allclose(got["seg_base"].reshape(sim["seg_base"].shape), sim["seg_base"], rtol=1e-9, atol=0)
    assert got["trace_status"] == 0


def test_oracle_scheme_too_long_segment_flagged():
    w, sh, toks, fl, sw = _sweep("C2", n_requests=20_000, n_intervals=24)
    cap = 50   # shorter than most segments
    ws = S.workspace(S.oracle_scheme_workspace_bytes(sw.dp, cap), sw.device)
    st = torch.zeros((sw.dp.cells, 3), dtype=torch.int64, device=sw.device)
    cs = torch.zeros(sw.dp.cells, dtype=torch.uint8, device=sw.device)
    S.simulate_oracle_scheme(sw.dp, sw.trace, sw.cost, cap, sw.totals, st, cs, ws)
    torch.cuda.synchronize()
    got = sw.host()
    assert got["trace_status"] & S.TRACE_TOO_LONG
    m = np.diff(sh.seg_offsets)
    long_ = np.repeat(m > cap, w.prob.X)
    assert np.all(got["cnt"].reshape(len(long_), -1)[long_].sum(axis=1) == 0)


def _sample_subproblem(w, ids):
    """The sampled segments as a compact problem (one 'region' per segment,
    T = 1) with their requests regenerated on the host; g0 = each segment's
    global first request (the Philox counters)."""
    import dataclasses
    P = w.prob
    regs = np.asarray(ids) // P.T
    sub = dataclasses.replace(P, R=len(ids), T=1, k0=np.asarray(P.k0)[ids], kmin=np.asarray(P.kmin)[regs],
                              kmax=np.asarray(P.kmax)[regs], e=np.asarray(P.e)[regs], p=np.asarray(P.p)[regs],
                              q=np.asarray(P.q)[regs])
    parts, fparts, off = [], [], [0]
    for s in ids:
        a, b = int(w.spec.seg_offsets[s]), int(w.spec.seg_offsets[s + 1])
        t, f = synth.gen_tokens(w.spec, a, b)
        parts.append(t); fparts.append(f); off.append(off[-1] + b - a)
    toks = np.concatenate(parts, axis=1)
    fl = np.concatenate(fparts) if w.spec.has_flags else None
    return sub, np.array(off, np.int64), toks, fl, np.asarray(w.spec.seg_offsets)[ids].astype(np.uint64)


def test_next4_full_size_c4_sampled():
    """C4 at full size (10^9 requests generated on the GPU): the Oracle scheme,
    the head-to-head statistics and one xi column's per-request outputs on a
    deterministic sample of segments (every 997th + first/last/largest)
    against the oracle run on those segments alone."""
    w = synth.make_workload("C4")
    sh = synth.shard(w.spec, 1, 0)
    sw = Sweep(w.prob, w.cost, sh, DEV, spec=w.spec)
    sw.solve()
    pref = sw.preference_stats().cpu().numpy().view(np.uint64)
    j = 40
    ro = sw.request_outputs(j)
    orr = sw.oracle_scheme()
    torch.cuda.synchronize()
    got = sw.host()
    assert got["trace_status"] == 0
    ids = synth.sample_segments(w.spec, 0, sh.n_segments, every=997)
    sub, off, toks, fl, g0 = _sample_subproblem(w, ids)
    X, NC, n = w.prob.X, w.cost.n_classes, w.prob.n
    cidx = (np.asarray(ids)[:, None] * X + np.arange(X)[None, :]).reshape(-1)
    # head-to-head statistics
    want = oracle.preference(sub, w.cost, off, fl, g0=g0)
    np.testing.assert_array_equal(pref[cidx], want)
    # per-request outputs of column j
    wr = oracle.request_outputs(sub, w.cost, off, toks, fl, j=j, g0=g0)
    for k, (s, a0) in enumerate(zip(ids, off[:-1])):
        a, b = int(w.spec.seg_offsets[s]), int(w.spec.seg_offsets[s + 1])
        sl = slice(a, b)
        np.testing.assert_array_equal(ro["level"][sl].cpu().numpy(), wr["level"][a0:a0 + b - a])
        np.testing.assert_array_equal(ro["pref"][sl].cpu().numpy(), wr["pref"][a0:a0 + b - a])
        np.testing.assert_array_equal(ro["ratio"][sl].cpu().numpy().view(np.uint64),
                                      wr["ratio"][a0:a0 + b - a].view(np.uint64))
    # the Oracle scheme
    wo = oracle.oracle_scheme(sub, w.cost, off, toks, fl, g0=g0)
    np.testing.assert_array_equal(orr["cell_status"].cpu().numpy()[cidx], wo["status"])
    np.testing.assert_array_equal(orr["stats"].cpu().numpy().view(np.uint64)[cidx], wo["stats"])
    np.testing.assert_array_equal(got["cnt"].reshape(-1, NC, n)[cidx], wo["cnt"])
    np.testing.assert_array_equal(got["tok"].reshape(-1, NC, n)[cidx], wo["tok"])
    np.testing.assert_allclose(got["carbon"].reshape(-1)[cidx], wo["carbon"], rtol=1e-9, atol=0)
