"""Helpers shared by the GPU parity tests: run the CUDA path through the C ABI
and the oracle on the same seeded inputs, compare element by element."""
import numpy as np

import oracle
import synth

FP_RTOL = 1e-9        # north_star: fp64 totals within 1e-9 relative


def oracle_shard(w, sh, toks, flags, seg_ids=None, levels=False, threads=None):
    """Oracle per-cell/segment results for (a subset of) a shard's segments."""
    if seg_ids is None:
        seg_ids = np.arange(sh.first_segment, sh.first_segment + sh.n_segments)
    loc = seg_ids - sh.first_segment
    req_begin = sh.seg_offsets[loc]
    seg_m = sh.seg_offsets[loc + 1] - sh.seg_offsets[loc]
    g0 = sh.first_request + req_begin
    return oracle.simulate(w.prob, w.cost, seg_ids, req_begin, seg_m, g0, toks, flags, levels=levels,
                           threads=threads)


def compare_cells(got, cells, lo=0, hi=None):
    """LP outputs, bit-exact."""
    hi = len(cells["vertex"]) if hi is None else hi
    np.testing.assert_array_equal(got["cell_status"][lo:hi], cells["cell_status"])
    np.testing.assert_array_equal(got["vertex"][lo:hi], cells["vertex"])
    np.testing.assert_array_equal(got["x"][lo:hi].view(np.uint64), cells["x"].view(np.uint64))
    np.testing.assert_array_equal(got["objective"][lo:hi].view(np.uint64), cells["objective"].view(np.uint64))
    np.testing.assert_array_equal(got["q_lb"][lo:hi].view(np.uint64), cells["q_lb"].view(np.uint64))
    np.testing.assert_array_equal(got["max_level"][lo:hi], cells["max_level"])
    if cells["threshold"].shape[1]:
        np.testing.assert_array_equal(got["threshold"][lo:hi].astype(np.uint64),
                                      np.minimum(cells["threshold"], 0xFFFFFFFF))


def compare_sim(got, sim, X, NC, n, loc=None):
    """Trace replay: integer statistics bit-exact, fp64 within FP_RTOL."""
    S_all = got["seg_count"].shape[0]
    if loc is None:
        loc = np.arange(S_all)
    cnt = got["cnt"].reshape(S_all, X, NC, n)[loc]
    tok = got["tok"].reshape(S_all, X, NC, n)[loc]
    np.testing.assert_array_equal(cnt, sim["cnt"])
    np.testing.assert_array_equal(tok, sim["tok"])
    np.testing.assert_array_equal(got["seg_count"].reshape(S_all, NC)[loc], sim["seg_count"])
    np.testing.assert_array_equal(got["seg_pinned"].reshape(S_all, NC)[loc], sim["seg_pinned"])
    np.testing.assert_array_equal(got["seg_tok"].reshape(S_all, NC, n)[loc], sim["seg_tok"])
    for k_got, k_or in (("energy", "energy"), ("time", "time"), ("carbon", "carbon"), ("quality", "quality")):
        np.testing.assert_allclose(got[k_got].reshape(S_all, X)[loc], sim[k_or], rtol=FP_RTOL, atol=0, err_msg=k_got)
    np.testing.assert_allclose(got["seg_base"].reshape(S_all, 4)[loc], sim["seg_base"], rtol=FP_RTOL, atol=0)
