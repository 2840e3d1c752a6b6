"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same
seeded inputs.  Bit-exact: LP vertices, x, objective, thresholds, per-request
levels, integer counts/tokens.  fp64 totals within 1e-9 relative."""
import numpy as np
import pytest
import torch

import oracle
import synth
from parity_util import FP_RTOL, compare_cells, compare_sim, oracle_shard

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2403_12900_b200 import sprout as S
    from paper_2403_12900_b200.runner import Sweep

DEV = "cuda:0"


def run_full(w, levels=True, world=1, rank=0, tokens_from_host=True):
    sh = synth.shard(w.spec, world, rank)
    toks, flags = synth.host_trace(w.spec, sh)
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=flags) if tokens_from_host else \
        Sweep(w.prob, w.cost, sh, DEV, spec=w.spec)
    sw.solve()
    sw.simulate(levels=levels)
    sw.reduce()
    torch.cuda.synchronize()
    return sh, toks, flags, sw.host()


def check_full(w, levels=True):
    sh, toks, flags, got = run_full(w, levels)
    cells = oracle.solve_cells(w.prob)
    compare_cells(got, cells)
    sim = oracle_shard(w, sh, toks, flags, levels=levels)
    compare_sim(got, sim, w.prob.X, w.cost.n_classes, w.prob.n)
    if levels:
        np.testing.assert_array_equal(got["levels"][:, sh.seg_offsets[0]:sh.n_requests],
                                      sim["levels"][:, sh.seg_offsets[0]:sh.n_requests])
    G = oracle.reduce(w.prob, w.cost.n_classes, 0, w.prob.R * w.prob.T, cells, sim)
    np.testing.assert_allclose(got["group"], G, rtol=FP_RTOL, atol=1e-300)
    assert got["trace_status"] & ~S.TRACE_SLOW_PATH == 0
    return got, sim


# ---------------------------------------------------------------- configs


def test_c1_full():
    check_full(synth.make_workload("C1"))


def test_c2_full():
    check_full(synth.make_workload("C2"))


def test_c3_shape_reduced():
    # 5-min intervals, two model classes, opted-out users
    check_full(synth.make_workload("C3", n_requests=2_000_000, n_intervals=2016))


def test_c4_shape_reduced():
    # 64 xi per segment: up to 65 breakpoints, the wide histogram
    got, sim = check_full(synth.make_workload("C4", n_requests=3_000_000, n_intervals=96), levels=True)
    assert (got["trace_status"] & S.TRACE_SLOW_PATH) == 0


def test_c5_shape_reduced():
    check_full(synth.make_workload("C5", n_requests=2_000_000, n_intervals=48, n_regions=12))


# ---------------------------------------------------------------- the LP alone


def _random_problem(rng, n, S_, invalid_frac=0.02):
    R, T = 1, S_
    X = 3
    prob = synth.Problem(
        n=n, R=R, T=T, X=X, k0=rng.uniform(0, 600, R * T), kmin=np.array([50.0]), kmax=np.array([450.0]),
        xi=np.array([0.0, rng.uniform(0, 1), 1.0]), e=rng.uniform(0, 3e-5, (R * T, n)),
        p=rng.uniform(0, 0.5, (R * T, n)), q=rng.uniform(0, 1, (R * T, n)), profile_per_interval=1,
        k1=9.5e-4, pue=1.2)
    # ties, degenerate rows, invalid rows
    tie = rng.random(R * T) < 0.05
    prob.q[tie, -1] = prob.q[tie, 0]
    same = rng.random(R * T) < 0.05
    prob.e[same, :] = prob.e[same, :1]
    prob.p[same, :] = prob.p[same, :1]
    bad = rng.random(R * T) < invalid_frac
    which = rng.integers(0, 4, R * T)
    prob.q[bad & (which == 0), 0] = 1.5
    prob.e[bad & (which == 1), -1] = -1.0
    prob.p[bad & (which == 2), 0] = np.nan
    prob.k0[bad & (which == 3)] = np.inf
    return prob


@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 8])
def test_lp_random_instances_bit_exact(n):
    rng = np.random.default_rng(1000 + n)
    prob = _random_problem(rng, n, 20_000)
    dp = S.DeviceProblem.from_host(prob, DEV)
    sol = S.Solution.empty(dp)
    S.solve_directives(dp, sol)
    torch.cuda.synchronize()
    got = {"x": sol.x.cpu().numpy(), "objective": sol.objective.cpu().numpy(), "q_lb": sol.q_lb.cpu().numpy(),
           "vertex": sol.vertex.cpu().numpy(), "threshold": sol.thresholds_u32(),
           "max_level": sol.max_level.cpu().numpy(), "cell_status": sol.cell_status.cpu().numpy()}
    cells = oracle.solve_cells(prob)
    compare_cells(got, cells)
    assert (cells["cell_status"] == 1).any()
    st = S.check_cells(dp, sol)
    assert st == 5          # SPROUT_ERR_INVALID_CELL


# ---------------------------------------------------------------- edge cases


def _custom(n=3, X=4, R=2, T=7, N=5000, NC=1, flags=False, seed=3, xi=None):
    w = synth.make_workload("C2", n_requests=N, n_intervals=T, n_regions=R,
                            xi=np.array(xi if xi is not None else np.linspace(0.0, 1.0, X)), seed_offset=seed)
    if n != 3:
        ratios = [1.0 / (i + 1) for i in range(n)]
        w.spec.n_levels = n
        w.spec.ratio_table = synth.ratio_table(ratios)
        ef, et, pf, pt = synth.cost_coefficients(NC, n)
        e, p = synth.profiles(w.spec, ef, et, pf, pt)
        w.prob.n = n
        w.prob.e = np.tile(e, (R, 1)); w.prob.p = np.tile(p, (R, 1))
        rng = np.random.default_rng(seed)
        w.prob.q = rng.dirichlet(np.full(n, 2.0), size=R)
        w.cost.ef, w.cost.et, w.cost.pf, w.cost.pt = ef, et, pf, pt
    w.spec.n_classes = NC
    w.spec.q0_table = np.stack([synth.q0_table(250.0 - 20 * c) for c in range(NC)])
    w.spec.has_flags = flags
    w.spec.pin_thresh = 1_000_000 if flags else 0
    w.cost.n_classes = NC
    ef, et, pf, pt = synth.cost_coefficients(NC, n)
    w.cost.ef, w.cost.et, w.cost.pf, w.cost.pt = ef, et, pf, pt
    return w


@pytest.mark.parametrize("n,X,NC,flags", [(1, 3, 1, False), (2, 5, 2, True), (4, 7, 3, True),
                                          (8, 4, 4, True), (6, 33, 1, False), (3, 200, 1, False)])
def test_levels_classes_flags(n, X, NC, flags):
    w = _custom(n=n, X=X, NC=NC, flags=flags, N=20_000, T=13, R=3)
    check_full(w)


def test_empty_and_ragged_segments():
    w = _custom(N=3000, T=50, R=2)
    off = w.spec.seg_offsets
    m = np.diff(off)
    m[::3] = 0                    # every third segment empty
    m[5] = 1                      # single-request segment
    m[7] = 4000                   # a long one
    off[1:] = np.cumsum(m)
    check_full(w)


@pytest.mark.parametrize("n,X,N,T", [(3, 4, 4000, 5),       # short segments: search mode
                                     (3, 40, 90_000, 4),    # bucket-table (LUT) mode, n = 3
                                     (5, 12, 60_000, 4),    # LUT mode, two word pairs per row
                                     (8, 10, 40_000, 4)])   # LUT mode, n = 8
def test_large_tokens_take_careful_path(n, X, N, T):
    # tokens >= 4096 cannot take the packed 16/20-bit fast path: the group is
    # reverted and added through the 64-bit accumulators (every row layout)
    w = _custom(n=n, X=X, N=N, T=T, R=1)
    sh = synth.shard(w.spec, 1, 0)
    toks, flags = synth.host_trace(w.spec, sh)
    rng = np.random.default_rng(5)
    for lo, hi in ((32768, 65536), (4096, 8192)):
        idx = rng.integers(0, sh.n_requests, 200)
        toks[rng.integers(0, n, 200), idx] = rng.integers(lo, hi, 200)
    toks[:, 17] = 65535
    toks[:, sh.n_requests - 1] = 40000          # a tail request
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=flags)
    sw.step()
    sw.simulate(levels=True)
    torch.cuda.synchronize()
    got = sw.host()
    sim = oracle_shard(w, sh, toks, flags, levels=True)
    compare_sim(got, sim, w.prob.X, 1, n)
    np.testing.assert_array_equal(got["levels"][:, :sh.n_requests], sim["levels"][:, :sh.n_requests])


def test_count_spill_single_bin():
    # xi = 0 => every cell pure L0 => one bin; 2M requests in one segment
    # overflow the 16-bit count field many times over (spill path)
    w = _custom(N=2_000_000, T=1, R=1, xi=[0.0])
    check_full(w, levels=False)


def test_wide_kernel_spills_long_segment():
    # n = 3, one class, no flags, X > 1: trace_wide_kernel.  One 2M-request
    # segment with two bins (xi = 0 is pure L0, xi = 1 has one breakpoint):
    # every lane's rows pass their guard bits many times (64-bit spill scratch)
    w = _custom(N=2_000_000, T=1, R=1, xi=[0.0, 1.0])
    got, _ = check_full(w, levels=False)
    assert (got["trace_status"] & S.TRACE_SLOW_PATH) == 0


def test_wide_kernel_crowded_keys_and_bad_offsets():
    # many xi values with nearly equal mixes put several keys in one bucket
    # (the trap row and its repair), ragged/empty segments, head and tail
    # requests outside whole groups; then non-monotone offsets are skipped
    w = _custom(N=400_000, T=9, R=2, X=96, xi=np.concatenate([np.linspace(0.0, 1.0, 48),
                                                            np.linspace(0.40, 0.4001, 48)]))
    off = w.spec.seg_offsets
    m = np.diff(off)
    m[3] = 0
    m[4] = 13
    m[5] += 7
    off[1:] = np.cumsum(m)
    check_full(w, levels=True)
    sh = synth.shard(w.spec, 1, 0)
    toks, flags = synth.host_trace(w.spec, sh)
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=flags)
    sw.solve()
    bad = sw.trace.seg_offsets.clone(); bad[6] = bad[7] + 1
    sw.trace.seg_offsets = bad
    sw.simulate()
    torch.cuda.synchronize()
    got = sw.host()
    assert got["trace_status"] & S.TRACE_BAD_OFFSETS
    assert not got["cnt"].reshape(-1, w.prob.X, 3)[6].any()


def test_arbitrary_thresholds_slow_path():
    # user-supplied thresholds with more distinct breakpoints than the fast
    # path holds (kcap = X+1): the generic per-cell path, still exact
    w = _custom(n=4, X=6, N=30_000, T=6, R=2)
    sh = synth.shard(w.spec, 1, 0)
    toks, flags = synth.host_trace(w.spec, sh)
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=flags)
    sw.solve()
    torch.cuda.synchronize()
    rng = np.random.default_rng(9)
    cells = sw.dp.cells
    thr = np.sort(rng.integers(1, 2**32, (cells, 3), dtype=np.uint64), axis=1).astype(np.uint32)
    thr[: cells // 2] = thr[: cells // 2][:, ::-1]      # also non-monotone thresholds
    ml = rng.integers(0, 4, cells).astype(np.uint8)
    sw.sol.threshold.copy_(torch.from_numpy(thr.view(np.int32)))
    sw.sol.max_level.copy_(torch.from_numpy(ml))
    sw.simulate(levels=True)
    sw.reduce()
    torch.cuda.synchronize()
    got = sw.host()
    assert got["trace_status"] & S.TRACE_SLOW_PATH
    # expected: count-and-clamp rule evaluated here from the same draws (oracle Philox)
    lv = got["levels"]
    for s in range(sh.n_segments):
        a, b = sh.seg_offsets[s], sh.seg_offsets[s + 1]
        for r in range(a, min(b, a + 40)):
            wd = oracle.draw_word(w.cost.seed, sh.first_request + r)
            for j in range(w.prob.X):
                c = s * w.prob.X + j
                L = min(int((wd >= thr[c].astype(np.uint64)).sum()), int(ml[c]))
                assert lv[j, r] == L
    # counts consistent with the levels
    cnt = got["cnt"].reshape(sh.n_segments, w.prob.X, 1, 4)
    for s in range(sh.n_segments):
        a, b = sh.seg_offsets[s], sh.seg_offsets[s + 1]
        for j in range(w.prob.X):
            np.testing.assert_array_equal(cnt[s, j, 0], np.bincount(lv[j, a:b], minlength=4)[:4])


@pytest.mark.parametrize("n,X", [(3, 2100), (2, 4096), (3, 4096)])
def test_large_xi_generic_path(n, X):
    """Up to SPROUT_MAX_XI xi values: more thresholds per segment than the
    per-warp breakpoint merge takes (n = 3, X > 2048) run the generic
    per-cell path, whose prep pass needs no sort buffer; n = 2, X = 4096 is
    the largest merge.  Cells and totals equal the oracle's."""
    w = _custom(n=n, X=X, N=6000, T=3, R=1)
    sh = synth.shard(w.spec, 1, 0)
    toks, flags = synth.host_trace(w.spec, sh)
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=flags)
    sw.solve()
    sw.simulate()
    torch.cuda.synchronize()
    got = sw.host()
    compare_cells(got, oracle.solve_cells(w.prob))
    compare_sim(got, oracle_shard(w, sh, toks, flags), X, 1, n)


def test_bad_class_and_bad_offsets_flagged():
    w = _custom(N=5000, T=6, R=1, NC=2, flags=True)
    sh = synth.shard(w.spec, 1, 0)
    toks, flags = synth.host_trace(w.spec, sh)
    flags[sh.seg_offsets[2]] = 3 << 1               # class 3 >= n_classes
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=flags)
    sw.step()
    torch.cuda.synchronize()
    got = sw.host()
    assert got["trace_status"] & S.TRACE_BAD_CLASS
    sim = oracle_shard(w, sh, toks, flags)
    assert sim["bad_requests"] == 1
    compare_sim(got, sim, w.prob.X, 2, 3)
    # non-monotone offsets: that segment is skipped and flagged
    seg = sw.trace.seg_offsets.clone()
    bad = seg.clone(); bad[3] = bad[4] + 1
    sw.trace.seg_offsets = bad
    sw.simulate()
    torch.cuda.synchronize()
    got = sw.host()
    assert got["trace_status"] & S.TRACE_BAD_OFFSETS


def test_host_validation_errors():
    w = _custom(N=100, T=2, R=1)
    sh = synth.shard(w.spec, 1, 0)
    toks, flags = synth.host_trace(w.spec, sh)
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=flags)
    bad = S.DeviceTrace(sh.n_requests, 4, sw.trace.seg_offsets, sw.trace.tokens, None)   # first_request % 8
    with pytest.raises(S.SproutError) as ei:
        S.simulate_trace(sw.dp, sw.sol, bad, sw.cost, sw.totals, sw.ws)
    assert ei.value.status == 1
    small = S.workspace(256, DEV)
    with pytest.raises(S.SproutError):
        S.simulate_trace(sw.dp, sw.sol, sw.trace, sw.cost, sw.totals, small[:10])


# ---------------------------------------------------------------- sharding


@pytest.mark.parametrize("world", [2, 4, 8])
def test_partition_invariance(world):
    w = synth.make_workload("C2", n_requests=400_000, n_intervals=500)
    _, _, _, full = run_full(w, levels=False)
    X, n, NC = w.prob.X, w.prob.n, w.cost.n_classes
    acc = np.zeros_like(full["group"])
    for rank in range(world):
        sh, _, _, part = run_full(w, levels=False, world=world, rank=rank)
        lo, hi = sh.first_segment, sh.first_segment + sh.n_segments
        np.testing.assert_array_equal(part["cnt"], full["cnt"].reshape(-1, X * NC * n)[lo:hi].reshape(part["cnt"].shape))
        np.testing.assert_array_equal(part["tok"], full["tok"].reshape(-1, X * NC * n)[lo:hi].reshape(part["tok"].shape))
        np.testing.assert_array_equal(part["carbon"], full["carbon"].reshape(-1, X)[lo:hi].reshape(-1))
        acc += part["group"]
    np.testing.assert_allclose(acc, full["group"], rtol=1e-12)
    # integer statistics are exact under the sum
    np.testing.assert_array_equal(acc[..., 0], full["group"][..., 0])
    np.testing.assert_array_equal(acc[..., 11:], full["group"][..., 11:])


# ---------------------------------------------------------------- generator, e2e


def test_device_generator_matches_host_generator():
    for name, kw in (("C3", dict(n_requests=3_000_000, n_intervals=2016)), ("C5", dict(n_requests=10**6, n_intervals=24, n_regions=4))):
        w = synth.make_workload(name, **kw)
        for world, rank in ((1, 0), (3, 1)):
            sh = synth.shard(w.spec, world, rank)
            sw = Sweep(w.prob, w.cost, sh, DEV, spec=w.spec)
            torch.cuda.synchronize()
            tok, fl = sw.trace_host()
            t2, f2 = synth.host_trace(w.spec, sh)
            np.testing.assert_array_equal(tok, t2)
            if w.spec.has_flags:
                np.testing.assert_array_equal(fl, f2)


def test_sweep_host_matches_device_path():
    import ctypes as C
    w = synth.make_workload("C2", n_requests=200_000, n_intervals=300)
    sh, toks, flags, got = run_full(w, levels=False)
    P = w.prob
    keep = []
    def hp(a, dt):
        a = np.ascontiguousarray(a, dt)
        keep.append(a)
        return a.ctypes.data
    lp = S.LpProblem(P.n, P.R, P.T, P.X, P.profile_per_interval, hp(P.k0, np.float64), hp(P.kmin, np.float64),
                     hp(P.kmax, np.float64), hp(P.xi, np.float64), hp(P.e, np.float64), hp(P.p, np.float64),
                     hp(P.q, np.float64), P.k1, P.pue, 0, P.R * P.T)
    tr = S.Trace(sh.n_requests, sh.first_request, hp(sh.seg_offsets, np.int64), hp(toks, np.uint16),
                 toks.shape[1], hp(flags, np.uint8))
    nb = S.sweep_workspace_bytes(lp, tr, w.cost.n_classes)
    ws = S.workspace(nb, DEV)
    out = np.zeros(got["group"].shape)
    st = np.zeros(1, np.uint32)
    S.sweep_host(lp, tr, S.cost_model(w.cost), out, st, ws)
    np.testing.assert_array_equal(out, got["group"])
    assert st[0] == 0


@pytest.mark.slow
@pytest.mark.parametrize("name,every", [("C4", 997), ("C3", 4999), ("C5", 99991)])
def test_full_size_sampled(name, every):
    """BASELINE configs at full size, generated on the GPU in the bench's
    launch configuration (C4: 10^9 requests, the histogram kernel; C3: 10^8
    requests in 525,600 five-minute segments with two classes and opted-out
    users, and C5: 10^10 requests, 256 regions, n = 5 -- both the one-cell
    kernel); the oracle replays a deterministic sample of segments
    (every k-th + first/last/largest) regenerated on the host from global
    request indices."""
    w = synth.make_workload(name)
    sh = synth.shard(w.spec, 1, 0)
    sw = Sweep(w.prob, w.cost, sh, DEV, spec=w.spec)
    sw.step()
    torch.cuda.synchronize()
    got = sw.host()
    assert got["trace_status"] == 0
    ids = synth.sample_segments(w.spec, 0, sh.n_segments, every=every)
    X = w.prob.X
    cells = oracle.solve_cells(w.prob)
    compare_cells(got, cells)
    # regenerate only the sampled segments' requests on the host
    parts, fparts, begins, ms, g0s = [], [], [], [], []
    pos = 0
    for s in ids:
        a, b = int(w.spec.seg_offsets[s]), int(w.spec.seg_offsets[s + 1])
        t, f = synth.gen_tokens(w.spec, a, b)
        parts.append(t); fparts.append(f); begins.append(pos); ms.append(b - a); g0s.append(a); pos += b - a
    toks = np.concatenate(parts, axis=1)
    flags = np.concatenate(fparts) if w.spec.has_flags else None
    sim = oracle.simulate(w.prob, w.cost, ids, np.array(begins), np.array(ms), np.array(g0s, np.uint64), toks, flags)
    compare_sim(got, sim, X, w.cost.n_classes, w.prob.n, loc=ids)
    # conservation on the full run
    G = got["group"]
    n = w.prob.n
    assert G[-1, 0, 0] == w.N
    np.testing.assert_array_equal(G[-1, :, 11:11 + n].sum(axis=1), G[-1, :, 0])


# ---------------------------------------------------------------- one cell per segment (trace_x1.cu)


@pytest.mark.parametrize("n,NC,flags", [(1, 1, False), (2, 2, True), (3, 1, True), (3, 2, False), (4, 2, True),
                                        (4, 1, False), (5, 1, False), (6, 1, True), (8, 1, False)])
def test_x1_register_path(n, NC, flags):
    """X = 1 (n <= 4 with <= 2 classes, n <= 8 with one): the register path;
    ragged and empty segments, a long segment and tokens >= 4096 included."""
    w = _custom(n=n, X=1, NC=NC, flags=flags, N=40_000, T=40, R=2, xi=[0.3])
    off = w.spec.seg_offsets
    m = np.diff(off)
    m[::7] = 0
    m[3] = 1
    m[5] = 3
    m[9] = 9000
    off[1:] = np.cumsum(m)
    sh = synth.shard(w.spec, 1, 0)
    toks, fl = synth.host_trace(w.spec, sh)
    rng = np.random.default_rng(n)
    idx = rng.integers(0, sh.n_requests, 300)
    toks[rng.integers(0, n, 300), idx] = rng.integers(4096, 65536, 300)
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=fl)
    sw.step()
    sw.simulate(levels=True)
    torch.cuda.synchronize()
    got = sw.host()
    cells = oracle.solve_cells(w.prob)
    compare_cells(got, cells)
    sim = oracle_shard(w, sh, toks, fl, levels=True)
    compare_sim(got, sim, 1, NC, n)
    np.testing.assert_array_equal(got["levels"][:, :sh.n_requests], sim["levels"][:, :sh.n_requests])
    G = oracle.reduce(w.prob, NC, 0, w.prob.R * w.prob.T, cells, sim)
    np.testing.assert_allclose(got["group"], G, rtol=FP_RTOL, atol=1e-300)


def test_x1_bad_class_invalid_cell_bad_offsets():
    w = _custom(N=6000, T=8, R=1, NC=2, flags=True, X=1, xi=[0.2])
    sh = synth.shard(w.spec, 1, 0)
    toks, flags = synth.host_trace(w.spec, sh)
    flags[sh.seg_offsets[2] + 1] = 3 << 1             # class 3 >= n_classes: skipped, flagged
    w.prob.k0 = w.prob.k0.copy()
    w.prob.k0[4] = -1.0                               # invalid cell: totals 0, segment stats still counted
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=flags)
    sw.step()
    torch.cuda.synchronize()
    got = sw.host()
    assert got["trace_status"] & S.TRACE_BAD_CLASS
    assert got["cell_status"][4] == S.CELL_INVALID
    sim = oracle_shard(w, sh, toks, flags)
    assert sim["bad_requests"] == 1
    compare_sim(got, sim, 1, 2, 3)
    bad = sw.trace.seg_offsets.clone(); bad[3] = bad[4] + 1
    sw.trace.seg_offsets = bad
    sw.simulate()
    torch.cuda.synchronize()
    got = sw.host()
    assert got["trace_status"] & S.TRACE_BAD_OFFSETS
    assert got["seg_count"].reshape(-1, 2)[3].sum() == 0


def test_x1_long_segment_folds():
    # 5M requests in one segment: three 2^21-request folds of the 32-bit lane sums
    w = _custom(N=5_000_000, T=1, R=1, X=1, xi=[0.5])
    check_full(w, levels=False)


@pytest.mark.parametrize("xi", [0.0, 1.0])
def test_x1_pure_mix_skips_draws(xi):
    # xi = 0: pure L0 (no draw needed); xi = 1 at high intensity: a pure or an edge mix per segment
    w = _custom(n=5, X=1, N=60_000, T=30, R=2, xi=[xi])
    check_full(w)


@pytest.mark.parametrize("world", [1, 3])
def test_graph_captured_step_matches_eager(world):
    """The step captured in a CUDA graph (runner.Sweep.capture) and replayed
    gives the eager step's results bit for bit, per shard (partition
    invariance holds through the graph)."""
    w = synth.make_workload("C4", n_requests=300_000, n_intervals=24)
    for rank in range(world):
        sh = synth.shard(w.spec, world, rank)
        eager = Sweep(w.prob, w.cost, sh, DEV, spec=w.spec)
        eager.step()
        torch.cuda.synchronize()
        want = eager.host()
        sw = Sweep(w.prob, w.cost, sh, DEV, spec=w.spec)
        g = sw.capture()
        for k in ("cnt", "tok", "carbon", "energy"):
            getattr(sw.totals, k).zero_()
        g.replay(); g.replay()
        torch.cuda.synchronize()
        got = sw.host()
        for k in ("cnt", "tok", "seg_count", "seg_tok"):
            np.testing.assert_array_equal(got[k], want[k], err_msg=k)
        for k in ("energy", "time", "carbon", "quality", "group"):
            np.testing.assert_array_equal(got[k].view(np.uint64), want[k].view(np.uint64), err_msg=k)


@pytest.mark.parametrize("name,kw", [("C2", dict(n_requests=200_000, n_intervals=48)),
                                     ("C3", dict(n_requests=400_000, n_intervals=288)),
                                     ("C4", dict(n_requests=1_000_000, n_intervals=48)),
                                     ("C5", dict(n_requests=300_000, n_intervals=24, n_regions=6))])
def test_fp64_per_request_mode_matches_closed_form(name, kw):
    # Eq. 1 per request in fp64 + warp-shuffle / block tree sums (sprout_cell_totals_fp64)
    # against the streaming kernel's closed form from exact integer statistics, and the
    # oracle's sequential per-request fp64 sums: both within 1e-12 relative
    w = synth.make_workload(name, **kw)
    sh, toks, flags, got = run_full(w, levels=False)
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=flags)
    sw.solve()
    f64 = S.cell_totals_fp64(sw.dp, sw.sol, sw.trace, sw.cost)
    torch.cuda.synchronize()
    sim = oracle_shard(w, sh, toks, flags)
    X = w.prob.X
    for k in ("energy", "time", "carbon", "quality"):
        v = f64[k].cpu().numpy()
        np.testing.assert_allclose(v, got[k].reshape(-1), rtol=1e-12, atol=1e-300, err_msg=k)
        np.testing.assert_allclose(v, sim[k].reshape(-1), rtol=1e-12, atol=1e-300, err_msg=k)


@pytest.mark.parametrize("n,NC,flags", [(3, 2, True), (2, 1, False)])
def test_x1_grouped_kernel_long_segment_chunks(n, NC, flags):
    """Short segments on average take the grouped one-cell kernel (4 segments
    per warp); one segment longer than a lane group's 2^19-request fold chunk
    forces several folds while its group's neighbours finish early."""
    w = _custom(n=n, X=1, NC=NC, flags=flags, N=1_500_000, T=900, R=2, xi=[0.4])
    off = w.spec.seg_offsets
    m = np.diff(off)
    m[:] = 100
    m[::11] = 0
    m[17] = 1_200_000
    m[18] = 5
    off[1:] = np.cumsum(m)
    assert off[-1] <= 1024 * len(m)
    check_full(w)


@pytest.mark.parametrize("n", [2, 3, 5, 8])
def test_x1_timed_path_with_clamps(n):
    """One class, no flags, long segments, without verify mode (the timed
    one-cell path exactly as bench runs it), then with max_level clamps below
    n - 1 in a third of the cells: counts against the a6 rule recounted here
    from the oracle's draws."""
    w = _custom(n=n, X=1, NC=1, flags=False, N=400_000, T=12, R=3, xi=[0.25])
    check_full(w, levels=False)
    sh = synth.shard(w.spec, 1, 0)
    toks, flags = synth.host_trace(w.spec, sh)
    sw = Sweep(w.prob, w.cost, sh, DEV, tokens=toks, flags=flags)
    sw.solve()
    torch.cuda.synchronize()
    # clamps: max_level below n - 1 in some cells (thresholds unchanged)
    ml = sw.sol.max_level.clone()
    ml[::3] = torch.clamp(ml[::3] - 1, min=0)
    sw.sol.max_level.copy_(ml)
    sw.simulate()
    torch.cuda.synchronize()
    got = sw.host()
    sim_lv = oracle_shard(w, sh, toks, flags, levels=False)
    # expected: the a6 rule from the same draws with the clamped max_level, counted here
    thr = sw.sol.thresholds_u32().reshape(-1, max(n - 1, 1)).astype(np.uint64)
    mlh = ml.cpu().numpy()
    cnt = got["cnt"].reshape(-1, n)
    for sidx in range(0, sh.n_segments, 5):
        a_, b_ = sh.seg_offsets[sidx], sh.seg_offsets[sidx + 1]
        wd = np.array([oracle.draw_word(w.cost.seed, sh.first_request + r) for r in range(a_, b_)], dtype=np.uint64)
        lv = np.minimum((wd[:, None] >= thr[sidx][None, :]).sum(axis=1), mlh[sidx]) if n > 1 else np.zeros(len(wd), int)
        np.testing.assert_array_equal(cnt[sidx], np.bincount(lv, minlength=n)[:n])
