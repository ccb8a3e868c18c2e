"""Fused ensemble statistics of fixed-step Tsit5 final states (-m gpu): the
solve kernel reduces each warp's final states to a (count, mean, M2) partial in
its epilogue instead of a second pass over the stored states (DESIGN §5,
a12). Checked against (1) the two-pass reduction over the stored states
(ens_ensemble_stats), (2) plain fp64 mean / unbiased variance of the oracle's
final states, on ragged sizes (partial warps, partial blocks), with trajectories
that diverge at t0 (stored u0 kept if finite, NaN u0 excluded) or overflow later
(non-finite final state excluded)."""
import numpy as np
import pytest
import torch

import oracle
import paper_2304_06835_b200 as ens
from synth.inputs import make_inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("N", [1, 31, 65, 1000, 4097])
def test_fused_stats_match_two_pass_and_oracle(dtype, N):
    u0, p = make_inputs("lorenz", "random10", N, seed=11, dtype=dtype)
    if N > 40:
        u0[0, 7] = np.nan      # f(u0) non-finite, stored u0 non-finite: excluded
        p[1, 20] = 1e38 if dtype == "f32" else 1e300   # f(u0) overflows, stored u0 finite: counted
        u0[1, 33] = 1e30 if dtype == "f32" else 1e200  # overflows during the solve: excluded
    dev = torch.device("cuda:0")
    U0, P = torch.from_numpy(u0).to(dev), torch.from_numpy(p).to(dev)
    sol = ens.solve("lorenz", "tsit5", U0, P, (0.0, 1.0), 1e-3, stats=True)
    two = ens.ensemble_stats(sol.u.unsqueeze(0))
    torch.cuda.synchronize()
    st, st2 = sol.stats.cpu().numpy()[0], two.cpu().numpy()[0]
    np.testing.assert_array_equal(st[:, 0], st2[:, 0])
    np.testing.assert_allclose(st[:, 1], st2[:, 1], rtol=1e-13, atol=0)
    np.testing.assert_allclose(st[:, 2], st2[:, 2], rtol=1e-11, atol=1e-300)
    o, orc, _, _ = oracle.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, dtype=dtype)
    final = o[-1] if o.ndim == 3 else o
    x = np.where(np.isfinite(final), final, np.nan).astype(np.float64)
    cnt = np.isfinite(x).sum(1)
    np.testing.assert_array_equal(st[:, 0], cnt)
    mean = np.nanmean(x, 1)
    np.testing.assert_allclose(st[:, 1], mean, rtol=1e-12 if dtype == "f64" else 1e-6)
    if N > 1:
        var = np.nanvar(x, 1, ddof=1)
        np.testing.assert_allclose(st[:, 2] / (st[:, 0] - 1), var, rtol=1e-10 if dtype == "f64" else 1e-5)


def test_fused_stats_full_size_headline():
    """The bench's launch configuration: N = 10^7 fp32, fused vs two-pass statistics."""
    N = 10**7
    u0, p = ens.generate_inputs("lorenz", "rho_sweep", N, dtype=torch.float32)
    sol = ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, stats=True)
    two = ens.ensemble_stats(sol.u.unsqueeze(0))
    torch.cuda.synchronize()
    st, st2 = sol.stats.cpu().numpy()[0], two.cpu().numpy()[0]
    np.testing.assert_array_equal(st[:, 0], np.full(3, N))
    np.testing.assert_allclose(st[:, 1], st2[:, 1], rtol=1e-12)
    np.testing.assert_allclose(st[:, 2], st2[:, 2], rtol=1e-10)
