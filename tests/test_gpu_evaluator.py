"""GPU parity of the opportunistic evaluator trigger sweep (Eq. 8,
P:218-235; reading L19) through the C ABI vs the oracle: every output
bit-exact (the decay factor is evaluated once on the host by both sides;
everything else is IEEE multiplies and comparisons in the same order)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

if torch.cuda.is_available():
    from paper_2403_12900_b200 import sprout as S

DEV = "cuda:0"


def _run(k2, kmax, T, dt, betas, thetas, grace, F, e=0.2778, pue=1.2):
    R = len(kmax)
    out = torch.zeros((R, len(betas), len(thetas), 4), dtype=torch.float64, device=DEV)
    S.evaluator_sweep(torch.as_tensor(k2, dtype=torch.float64, device=DEV),
                      torch.as_tensor(kmax, dtype=torch.float64, device=DEV), T, dt, betas, thetas, grace, F, e,
                      pue, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    want = oracle.evaluator_sweep(k2, kmax, T, dt, betas, thetas, grace, F, e, pue)
    np.testing.assert_array_equal(got.view(np.uint64), want.view(np.uint64))
    return got


@pytest.mark.parametrize("name,dt", [("C2", 1.0), ("C3", 1.0 / 12), ("C1", 1.0)])
def test_evaluator_parity_on_config_traces(name, dt):
    w = synth.make_workload(name, n_requests=1000) if name != "C1" else synth.make_workload("C1")
    P = w.prob
    betas = np.linspace(0.0, 0.1, 16)
    thetas = np.linspace(0.1, 1.0, 12)
    for grace, F in ((6.0, 3), (0.0, 0), (24.0, 1)):
        got = _run(P.k0, P.kmax, P.T, dt, betas, thetas, grace, F)
        assert (got[..., 0] >= 0).all()


def test_evaluator_parity_stress_shapes():
    rng = np.random.default_rng(5)
    R, T = 7, 3001
    k2 = rng.uniform(5, 600, size=R * T)
    kmax = k2.reshape(R, T).max(axis=1)
    betas = rng.uniform(0, 0.2, 64)
    thetas = rng.uniform(0, 1.2, 64)
    got = _run(k2, kmax, T, 0.25, betas, thetas, 3.0, 4)
    assert got[..., 0].sum() > 0
    _run(k2[:R], kmax, 1, 1.0, betas[:3], thetas[:2], 0.0, 1)     # T = 1: nothing to scan
