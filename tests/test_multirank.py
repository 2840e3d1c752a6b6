"""The N>1 path on CPU: world_size-2 gloo process groups (127.0.0.1).

Each rank takes its contiguous segment shard (synth.shard), computes its
group totals -- here with the oracle, the CUDA path's stand-in on a box
without a GPU -- and the ranks combine them with the package's collective
(paper_2403_12900_b200.collective).  The result must equal the single-process
totals: integer statistics exactly, fp64 within 1e-12."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2403_12900_b200.collective import allreduce_totals, max_over_ranks


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_totals(w, world, rank):
    P = w.prob
    sh = synth.shard(w.spec, world, rank)
    cells = oracle.solve_cells(P, sh.first_segment, sh.n_segments)
    toks, flags = synth.host_trace(w.spec, sh)
    segs = np.arange(sh.first_segment, sh.first_segment + sh.n_segments)
    loc = segs - sh.first_segment
    sim = oracle.simulate(P, w.cost, segs, sh.seg_offsets[loc], np.diff(sh.seg_offsets),
                          sh.first_request + sh.seg_offsets[loc], toks, flags, threads=1)
    return oracle.reduce(P, w.cost.n_classes, sh.first_segment, sh.n_segments, cells, sim)


def _worker(rank, world, port, name, kw, deterministic, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = synth.make_workload(name, **kw)
        g = torch.from_numpy(_rank_totals(w, world, rank))
        allreduce_totals(g, deterministic=deterministic)
        t = max_over_ranks(1.0 + rank, "cpu")
        if rank == 0:
            np.save(out, g.numpy())
            np.save(out + ".max.npy", np.array([t]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("deterministic", [False, True])
@pytest.mark.parametrize("name,kw", [("C2", dict(n_requests=60_000, n_intervals=96)),
                                     ("C3", dict(n_requests=50_000, n_intervals=288))])
def test_two_rank_totals_equal_single_process(tmp_path, name, kw, deterministic):
    world = 2
    out = str(tmp_path / "g.npy")
    mp.spawn(_worker, args=(world, _free_port(), name, kw, deterministic, out), nprocs=world, join=True)
    got = np.load(out)
    w = synth.make_workload(name, **kw)
    want = _rank_totals(w, 1, 0)
    n = w.prob.n
    # integer statistics: requests, opted-out, per-level counts and tokens -- exact
    for k in [0, 1] + list(range(11, 11 + 2 * n)):
        np.testing.assert_array_equal(got[..., k], want[..., k])
    np.testing.assert_allclose(got, want, rtol=1e-12, atol=0)
    assert float(np.load(out + ".max.npy")[0]) == float(world)


def test_shards_partition_segments_and_requests():
    w = synth.make_workload("C2", n_requests=60_000, n_intervals=96)
    for world in (2, 3, 8):
        shards = [synth.shard(w.spec, world, r) for r in range(world)]
        assert shards[0].first_segment == 0
        for a, b in zip(shards, shards[1:]):
            assert a.first_segment + a.n_segments == b.first_segment
        assert shards[-1].first_segment + shards[-1].n_segments == w.prob.R * w.prob.T
        # every request belongs to exactly one rank's segments
        total = sum(int(s.seg_offsets[-1] - s.seg_offsets[0]) for s in shards)
        assert total == w.N


def _static_worker(rank, world, port, D, xi, out):
    import dataclasses
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = synth.make_workload("C2", n_requests=40_000, n_intervals=48)
        G = oracle.grid_size(w.prob.n, D)
        prob = dataclasses.replace(w.prob, X=G, xi=np.zeros(G))
        sh = synth.shard(w.spec, world, rank)
        cells = oracle.solve_cells(prob, sh.first_segment, sh.n_segments, scheme=oracle.SCHEME_STATIC_GRID,
                                   grid_den=D)
        toks, flags = synth.host_trace(w.spec, sh)
        segs = np.arange(sh.first_segment, sh.first_segment + sh.n_segments)
        loc = segs - sh.first_segment
        sim = oracle.simulate(prob, w.cost, segs, sh.seg_offsets[loc], np.diff(sh.seg_offsets),
                              sh.first_request + sh.seg_offsets[loc], toks, flags, threads=1,
                              scheme=oracle.SCHEME_STATIC_GRID, grid_den=D)
        g = torch.from_numpy(oracle.reduce(prob, w.cost.n_classes, sh.first_segment, sh.n_segments, cells, sim))
        allreduce_totals(g, deterministic=True)
        choice, _ = oracle.select_static(prob, xi, D, g.numpy())     # every rank, identical totals
        gathered = [torch.zeros_like(torch.from_numpy(choice)) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(choice))
        if rank == 0:
            np.save(out, torch.stack(gathered).numpy())
            np.save(out + ".g.npy", g.numpy())
    finally:
        dist.destroy_process_group()


def test_two_rank_static_choice():
    """Sprout_Sta across ranks (SURVEY 8(e) + NEXT-3): the choice is taken
    after the all-reduce, so every rank picks the same static mix, and it is
    the single-process choice (or an equal-carbon near-tie)."""
    import tempfile
    D, xi = 5, 0.1
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "c.npy")
        mp.spawn(_static_worker, args=(2, _free_port(), D, xi, out), nprocs=2, join=True)
        ch = np.load(out)
        g2 = np.load(out + ".g.npy")
    assert (ch[0] == ch[1]).all()
    import dataclasses
    w = synth.make_workload("C2", n_requests=40_000, n_intervals=48)
    G = oracle.grid_size(w.prob.n, D)
    prob = dataclasses.replace(w.prob, X=G, xi=np.zeros(G))
    sh = synth.shard(w.spec, 1, 0)
    cells = oracle.solve_cells(prob, scheme=oracle.SCHEME_STATIC_GRID, grid_den=D)
    toks, flags = synth.host_trace(w.spec, sh)
    S = prob.R * prob.T
    sim = oracle.simulate(prob, w.cost, np.arange(S), sh.seg_offsets[:-1], np.diff(sh.seg_offsets),
                          sh.first_request + sh.seg_offsets[:-1], toks, flags, scheme=oracle.SCHEME_STATIC_GRID,
                          grid_den=D)
    g1 = oracle.reduce(prob, w.cost.n_classes, 0, S, cells, sim)
    c1, _ = oracle.select_static(prob, xi, D, g1)
    for r in range(prob.R):
        assert c1[r] == ch[0][r] or g1[r, c1[r], 4] == pytest.approx(g1[r, ch[0][r], 4], rel=1e-12)
