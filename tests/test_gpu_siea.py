"""GPU ↔ oracle parity for the weak-order-2 SDE scheme (GPUSIEA; DESIGN R19)."""
import math

import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs
from tests.helpers import gpu, traj_relerr

pytestmark = pytest.mark.gpu
TOL = {"f32": 1e-5, "f64": 1e-12}


@pytest.mark.parametrize("model", ["gbm", "lorenz_sde_add", "lorenz_sde_mul"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_siea_parity(model, dtype):
    N = 900
    u0, p = make_inputs(model, "const", N, dtype=dtype)
    sa = np.linspace(0.0, 1.0, 6)
    g, rc, na, _, st = gpu(model, "siea", u0, p, (0.0, 1.0), 1e-2, seed=0x51EA, saveat=sa, stats=True)
    o, orc, *_ = oracle.solve(model, "siea", u0, p, (0.0, 1.0), 1e-2, dtype=dtype, p_broadcast=True, seed=0x51EA,
                              saveat=sa)
    np.testing.assert_array_equal(rc, orc)
    assert traj_relerr(g, o).max() <= TOL[dtype]
    mean, var, _ = oracle.stats(g)
    np.testing.assert_allclose(st[..., 1], mean, rtol=1e-12, atol=1e-300)


def test_siea_gbm_moments_on_gpu():
    """10^6 GBM paths: sample mean/variance within 4 SE of the scheme's exact discrete moments."""
    X0, r, V, T, h = 0.1, 1.5, 0.1, 1.0, 0.05
    N = 10**6
    A, B, C = 1 + r * h + r * r * h * h / 2, V * (1 + r * h), V * V / 2
    n = round(T / h)
    E = X0 * A**n
    var = X0**2 * (A * A + B * B * h + 2 * C * C * h * h) ** n - E**2
    u0 = np.full((3, N), X0)
    _, rc, _, _, st = gpu("gbm", "siea", u0, np.array([r, V]), (0.0, T), h, seed=99, stats=True, store_states=False)
    m, M2, c = st[0, :, 1], st[0, :, 2], st[0, :, 0]
    assert (c == N).all()
    assert np.all(np.abs(m - E) < 4 * math.sqrt(var / N))
    assert np.all(np.abs(M2 / (N - 1) / var - 1) < 4 * math.sqrt(2 / N))
