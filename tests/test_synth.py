"""The seeded input generator (CPU only)."""
import numpy as np
import pytest

import synth
from conftest import hexint


def test_numpy_philox_known_answers(golden):
    for case in golden["philox4x32_10_kat"]["cases"]:
        ctr = [hexint(v) for v in case["ctr"]]
        key = [hexint(v) for v in case["key"]]
        out = synth.philox4x32_10(*[np.uint64(c) for c in ctr], key[0], key[1])
        assert [int(v) for v in out] == [hexint(v) for v in case["out"]]


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_configs_shapes_and_bounds(name, golden):
    w = synth.make_workload(name)
    P, spec = w.prob, w.spec
    assert P.k0.shape == (P.R * P.T,) and spec.seg_offsets.shape == (P.R * P.T + 1,)
    assert spec.N == {"C1": 10**3, "C2": 10**6, "C3": 10**8, "C4": 10**9, "C5": 10**10}[name]
    assert np.all(np.diff(spec.seg_offsets) >= 0)
    k = P.k0.reshape(P.R, P.T)
    np.testing.assert_array_equal(k.min(axis=1), P.kmin)       # attained exactly
    np.testing.assert_array_equal(k.max(axis=1), P.kmax)
    if name in ("C2", "C3", "C4"):
        for r, reg in enumerate(synth.REGIONS):                 # Table II
            assert (P.kmin[r], P.kmax[r]) == tuple(golden["table2_bounds"][reg])
    assert np.all((P.xi >= 0) & (P.xi <= 1))
    np.testing.assert_allclose(P.q.sum(axis=1), 1.0, rtol=1e-12)
    assert np.all(np.diff(P.e[0]) < 0) and np.all(np.diff(P.p[0]) < 0)   # directives cut cost


def test_generator_range_consistency_and_ranges():
    w = synth.make_workload("C3", n_requests=10**5, n_intervals=288)
    spec = w.spec
    a, _ = synth.gen_tokens(spec, 1000, 5000)
    b1, f1 = synth.gen_tokens(spec, 1000, 2345)
    b2, f2 = synth.gen_tokens(spec, 2345, 5000)
    np.testing.assert_array_equal(a, np.concatenate([b1, b2], axis=1))
    t, f = synth.gen_tokens(spec, 0, 200_000)
    assert t.min() >= 1 and t.max() <= 4095
    assert t[1].mean() < t[0].mean() / 2.5 and t[2].mean() < t[1].mean()
    cls = (f >> 1) & 3
    assert abs(cls.mean() - 0.5) < 0.01                          # 7B/13B 50/50
    assert abs((f & 1).mean() - 0.01) < 0.002                    # ~1% pinned
    mu = synth.level_means(spec)
    for c in range(2):
        for i in range(3):
            assert t[i][cls == c].mean() == pytest.approx(mu[c, i], rel=0.02)


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_plan(world):
    w = synth.make_workload("C2")
    spec = w.spec
    shards = [synth.shard(spec, world, r) for r in range(world)]
    assert shards[0].first_segment == 0
    tot = 0
    for k, sh in enumerate(shards):
        assert sh.first_request % 8 == 0
        if k + 1 < world:
            assert sh.first_segment + sh.n_segments == shards[k + 1].first_segment
        glob = spec.seg_offsets[sh.first_segment:sh.first_segment + sh.n_segments + 1]
        np.testing.assert_array_equal(sh.seg_offsets + sh.first_request, glob)
        assert 0 <= sh.seg_offsets[0] < 8 and sh.seg_offsets[-1] == sh.n_requests
        tot += sh.n_segments
    assert tot == w.prob.R * w.prob.T
    loads = [int(sh.seg_offsets[-1] - sh.seg_offsets[0]) for sh in shards]
    assert sum(loads) == spec.N
    assert max(loads) - min(loads) <= 2 * int(np.diff(spec.seg_offsets).max()) + 1
