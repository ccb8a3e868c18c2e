"""Event handling pins (-m "not gpu"): the bouncing ball.

Under constant gravity the flight between bounces is a parabola, which Tsit5
integrates exactly up to rounding, so the event times and the state at tf have
a closed form: dropped from rest at x0, first impact at t1 = √(2x0/g), impact k
at t_k = t_{k−1} + 2 e^{k−1} t1, rebound speed e^k g t1 (DESIGN R18)."""
import math

import numpy as np
import pytest

import oracle


def closed_form(x0, g, e, tf):
    t1 = math.sqrt(2 * x0 / g)
    if tf < t1:
        return x0 - 0.5 * g * tf * tf, -g * tf
    tk, k = t1, 1
    while tk + 2 * e**k * t1 <= tf:
        tk += 2 * e**k * t1
        k += 1
    v = e**k * g * t1
    d = tf - tk
    return v * d - 0.5 * g * d * d, v - g * d


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-9), ("f32", 2e-4)])
def test_bouncing_ball_closed_form(dtype, tol):
    rng = np.random.default_rng(4)
    N = 64
    g = rng.uniform(8.8, 10.8, N)
    e = rng.uniform(0.77, 0.93, N)
    p = np.stack([g, e])
    u0 = np.stack([np.full(N, 50.0), np.zeros(N)])
    out, rc, na, nr = oracle.solve("ball", "tsit5", u0, p, (0, 15), 0.1, dtype=dtype, adaptive=True,
                                   abstol=1e-10 if dtype == "f64" else 1e-6, reltol=1e-10 if dtype == "f64" else 1e-6)
    assert (rc == 0).all()
    pf = p.astype(np.float32).astype(np.float64) if dtype == "f32" else p
    for i in range(N):
        x, v = closed_form(50.0, pf[0, i], pf[1, i], 15.0)
        scale = 50.0 if dtype == "f32" else max(1.0, abs(x))
        assert abs(out[0, 0, i] - x) <= tol * scale and abs(out[0, 1, i] - v) <= tol * max(1.0, abs(v)) * 10, i


def test_ball_saveat_and_event_state():
    """saveat before, across and after impacts; heights never drop below the
    bisection resolution; the first impact time matches √(2x0/g)."""
    x0, g, e = 50.0, 9.8, 0.85
    sa = np.linspace(0, 15, 301)
    out, rc, *_ = oracle.solve("ball", "tsit5", [[x0], [0.0]], [[g], [e]], (0, 15), 0.1, adaptive=True,
                               abstol=1e-10, reltol=1e-10, saveat=sa)
    assert rc[0] == 0
    x = out[:, 0, 0]
    assert x.min() > -1e-9
    for t, xv in zip(sa, x):
        assert abs(xv - closed_form(x0, g, e, t)[0]) < 1e-8
