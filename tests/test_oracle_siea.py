"""Weak-order-2 SDE scheme (GPUSIEA; DESIGN R19) pins (-m "not gpu").

For GBM dX = rX dt + VX dW the scheme's step is X_{n+1} = X_n·M with
M = A + B ΔW + C (ΔW² − h), A = 1 + rh + r²h²/2, B = V(1 + rh), C = V²/2
(derived by hand from the scheme's definition), so the discrete moments are
closed forms: E = X0·A^N, E[X²] = X0²·(A² + B²h + 2C²h²)^N."""
import math

import numpy as np
import pytest

import oracle


@pytest.mark.parametrize("h", [0.1, 0.025])
def test_siea_gbm_exact_discrete_moments(h):
    X0, r, V, T = 0.1, 1.5, 0.1, 1.0
    N = round(T / h)
    A, B, C = 1 + r * h + r * r * h * h / 2, V * (1 + r * h), V * V / 2
    E = X0 * A**N
    var = X0**2 * (A * A + B * B * h + 2 * C * C * h * h) ** N - E**2
    out, rc, na, _ = oracle.solve("gbm", "siea", np.full((3, 12000), X0), [r, V], (0, T), h, p_broadcast=True,
                                  seed=17)
    assert (rc == 0).all() and (na == N).all()
    x = out[0].ravel()
    assert abs(x.mean() - E) < 4 * math.sqrt(var / x.size)
    assert abs(x.var(ddof=1) / var - 1) < 4 * math.sqrt(2 / x.size)


def test_siea_weak_order_two_in_the_mean():
    """The mean bias X0·|A^N − e^{rT}| shrinks like h² (EM's like h): the
    scheme's drift part reproduces e^{rh} to second order."""
    X0, r, V, T = 0.1, 1.5, 0.0, 1.0
    errs = []
    for h in [0.1, 0.05, 0.025]:
        out, *_ = oracle.solve("gbm", "siea", np.full((3, 1), X0), [r, V], (0, T), h, p_broadcast=True)
        errs.append(abs(out[0, 0, 0] - X0 * math.exp(r * T)))
        N = round(T / h)
        assert abs(out[0, 0, 0] - X0 * (1 + r * h + r * r * h * h / 2) ** N) < 1e-14   # V = 0: Heun's method
    slopes = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all((slopes > 1.8) & (slopes < 2.2)), slopes


def test_siea_additive_noise_is_stochastic_heun():
    """Additive noise (b constant): the ΔW² term vanishes and the scheme is
    u + ½(a(u + a h + b ΔW) + a(u)) h + b ΔW; with s = 0 it is Heun on Lorenz."""
    u0 = np.array([[1.0], [0.0], [0.0]])
    a, *_ = oracle.solve("lorenz_sde_add", "siea", u0, [10, 28, 8 / 3, 0.0], (0, 1), 1e-3, p_broadcast=True)
    u = u0[:, 0].copy()
    f = lambda y: np.array([10 * (y[1] - y[0]), y[0] * (28 - y[2]) - y[1], y[0] * y[1] - 8 / 3 * y[2]])
    for _ in range(1000):
        k1 = f(u)
        u = u + 0.5 * (f(u + 1e-3 * k1) + k1) * 1e-3
    np.testing.assert_allclose(a[0, :, 0], u, rtol=1e-10)
