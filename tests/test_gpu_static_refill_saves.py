"""Saving adaptive solves on ensembles of several waves: the static mapping
(the written-out loop kernels of Rosenbrock23 and Tsit5, the lane kernels of
Rodas4/5 and Vern7/9) and the refill scheduler (a8) must agree bit for bit,
including lanes that fail (Diverged at t0, MaxIters part-way: NaN-filled rows)
and a ragged last warp (-m gpu). (Written for the warp-staged save experiment,
DESIGN §5; kept as the large-ensemble static-vs-refill check.)"""
import numpy as np
import pytest

from synth.inputs import make_inputs
from tests.helpers import gpu

pytestmark = pytest.mark.gpu

N = 4 * 148 * 256 + 77          # several waves, ragged last warp


def _pair(model, alg, u0, p, tspan, dt, **kw):
    a = gpu(model, alg, u0, p, tspan, dt, refill=False, **kw)
    b = gpu(model, alg, u0, p, tspan, dt, refill=True, **kw)
    return a, b


@pytest.mark.parametrize("alg", ["rosenbrock23", "rodas5", "rodas4"])
def test_staged_saves_robertson(alg):
    u0, p = make_inputs("robertson", "random10", N, seed=0xC3, dtype="f64")
    u0[0, 5] = np.nan                      # Diverged at t0 (NaN rows after the t0 save)
    u0[0, 40000] = np.nan
    sa = np.linspace(0.0, 1e5, 100)
    a, b = _pair("robertson", alg, u0, p, (0.0, 1e5), 1e-4, adaptive=True, abstol=1e-8, reltol=1e-8, saveat=sa)
    for x, y in zip(a[:4], b[:4]):
        np.testing.assert_array_equal(x, y)
    assert a[1][5] == 3 and np.isnan(a[0][1:, :, 5]).all()
    # a cap that stops some lanes part-way: MaxIters with NaN-filled remaining rows
    a, b = _pair("robertson", alg, u0, p, (0.0, 1e5), 1e-4, adaptive=True, abstol=1e-8, reltol=1e-8, saveat=sa,
                 max_steps=120)
    for x, y in zip(a[:4], b[:4]):
        np.testing.assert_array_equal(x, y)
    assert (a[1] == 1).any()


@pytest.mark.parametrize("alg,dtype", [("tsit5", "f64"), ("tsit5", "f32"), ("vern7", "f64"), ("vern9", "f64")])
def test_staged_saves_lorenz(alg, dtype):
    u0, p = make_inputs("lorenz", "random10", N, seed=0xC1, dtype=dtype)
    u0[1, 1000] = np.inf
    sa = np.linspace(0.0, 1.0, 41)
    tol = 1e-8 if dtype == "f64" else 1e-5
    a, b = _pair("lorenz", alg, u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=tol, reltol=tol, saveat=sa)
    for x, y in zip(a[:4], b[:4]):
        np.testing.assert_array_equal(x, y)
