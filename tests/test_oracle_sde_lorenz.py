"""Pins for the stochastic Lorenz models of BASELINE config 4 (DESIGN R9):
over many independent paths from one fixed state, one EM step's increment has
mean h·f(u) (the Lorenz drift) and per-component variance b_j²·h with
b_j = s (additive) or b_j = s·u_j (multiplicative), components uncorrelated
(diagonal noise) — checked against the sample moments, not the oracle's code."""
import numpy as np
import pytest

import oracle


@pytest.mark.parametrize("model", ["lorenz_sde_add", "lorenz_sde_mul"])
def test_one_step_increment_moments(model):
    u = np.array([1.5, -2.0, 20.0])
    p = np.array([10.0, 28.0, 8.0 / 3.0, 0.1])
    N, h = 40000, 1e-3
    out, *_ = oracle.solve(model, "em", np.tile(u[:, None], (1, N)), p, (0, h), h, seed=21, p_broadcast=True)
    d = out[0] - u[:, None]
    drift = np.array([p[0] * (u[1] - u[0]), u[0] * (p[1] - u[2]) - u[1], u[0] * u[1] - p[2] * u[2]])
    b = np.full(3, p[3]) if model == "lorenz_sde_add" else p[3] * u
    var = b**2 * h
    se = np.sqrt(var / N)
    assert np.all(np.abs(d.mean(1) - h * drift) < 5 * se), (d.mean(1), h * drift)
    assert np.all(np.abs(d.var(1, ddof=1) / var - 1) < 5 * np.sqrt(2 / N))
    c = np.corrcoef(d)
    assert np.abs(c - np.eye(3)).max() < 5 / np.sqrt(N)


def test_zero_noise_scale_is_deterministic_euler():
    """s = 0: both models reduce to the explicit Euler method of the Lorenz ODE."""
    u0 = np.array([[1.0], [0.0], [0.0]])
    for model in ["lorenz_sde_add", "lorenz_sde_mul"]:
        out, *_ = oracle.solve(model, "em", u0, np.array([10.0, 28.0, 8.0 / 3.0, 0.0]), (0, 0.1), 1e-3, seed=5,
                               p_broadcast=True)
        u = u0[:, 0].copy()
        for _ in range(100):
            f = np.array([10.0 * (u[1] - u[0]), u[0] * (28.0 - u[2]) - u[1], u[0] * u[1] - (8.0 / 3.0) * u[2]])
            u = u + 1e-3 * f
        np.testing.assert_allclose(out[0, :, 0], u, rtol=1e-12)
