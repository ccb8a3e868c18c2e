"""Statistics over more than 65,535 (save point, component) rows (-m gpu): the
row-indexed reduction kernels stride over rows beyond the 65,535 limit of
gridDim.y (a12). Checked against a plain fp64 reduction of the
stored states."""
import numpy as np
import pytest

from synth.inputs import make_inputs
from tests.helpers import gpu

pytestmark = pytest.mark.gpu


def _plain(x):
    x = x.astype(np.float64)
    return x.mean(-1), x.var(-1, ddof=1)


def test_ensemble_stats_many_rows():
    import torch

    import paper_2304_06835_b200 as ens
    rows, N = 70_001, 97
    x = torch.randn(rows, N, dtype=torch.float64, device="cuda")
    st = ens.ensemble_stats(x).cpu().numpy()
    m, v = _plain(x.cpu().numpy())
    assert (st[:, 0] == N).all()
    np.testing.assert_allclose(st[:, 1], m, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(st[:, 2] / (N - 1), v, rtol=1e-12)


def test_solve_stats_with_22k_save_points():
    """want_stats on a Lorenz solve with k = 22,001 save points (66,003 rows)."""
    N = 64
    u0, p = make_inputs("lorenz", "random10", N, seed=1, dtype="f64")
    sa = np.linspace(0.0, 1.0, 22_001)
    g, rc, na, nr, st = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-5, saveat=sa, stats=True)
    assert (rc == 0).all()
    m, v = _plain(g)
    assert (st[..., 0] == N).all()
    np.testing.assert_allclose(st[..., 1], m, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(st[..., 2] / (N - 1), v, rtol=1e-10, atol=1e-20)
