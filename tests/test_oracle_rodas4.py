"""Pins for the oracle's Rodas4 (GPURodas4; NEXT-2; DESIGN R20).

The paper names the method but prints no tableau; the oracle carries Hairer &
Wanner's RODAS coefficients in W-form. These tests check them against the
Rosenbrock order conditions (order 4, embedded order 3, dense output order 3),
L-stability, the closed-form stability function of one step, measured
convergence orders, linear invariants and the literature reference solutions
of the stiff suite.
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest

import oracle

GOLD = Path(__file__).parent / "golden"


def gold(name):
    return json.loads((GOLD / name).read_text())


def _standard_form():
    """W-form (a, c, m, γ) → standard Rosenbrock form (α, Γ):
    Γ⁻¹ = diag(1/γ) − C, α = A Γ, weights b = m Γ (Hairer & Wanner IV.7)."""
    g, A, C, D = oracle.rodas4_tableau()
    Gi = np.diag(np.full(6, 1 / g)) - C
    G = np.linalg.inv(Gi)
    alpha = A @ G
    m = np.concatenate([A[5, :5], [1.0]])        # u_new = Y6 + k6 (stiffly accurate)
    me = np.concatenate([A[5, :5], [0.0]])       # embedded solution Y6
    return g, alpha, G, m, me, D


def _residuals(b, alpha, G, order, theta=1.0):
    """Rosenbrock order conditions with β̂ = α + Γ (diagonal included), for a
    step of length θh: Σ_t b·Φ_t = θ^ρ(t)/γ(t) (trees up to `order`)."""
    bh = alpha + G
    a = alpha.sum(1)
    bp = bh.sum(1)
    r = [b.sum() - theta, b @ bp - theta**2 / 2]
    if order >= 3:
        r += [b @ a**2 - theta**3 / 3, b @ bh @ bp - theta**3 / 6]
    if order >= 4:
        r += [b @ a**3 - theta**4 / 4, b @ (a * (alpha @ bp)) - theta**4 / 8,
              b @ bh @ (a**2) - theta**4 / 12, b @ bh @ bh @ bp - theta**4 / 24]
    return np.array(r)


def test_rodas4_order_conditions():
    """Order 4 (8 trees), embedded order 3 (4 trees), γ = 1/4, stage times
    c = (0, 0.386, 0.21, 0.63, 1, 1)."""
    g, alpha, G, m, me, D = _standard_form()
    assert g == 0.25
    assert np.abs(_residuals(m @ G, alpha, G, 4)).max() < 1e-13
    assert np.abs(_residuals(me @ G, alpha, G, 3)).max() < 1e-13
    # the embedded method is genuinely of order 3 only (its 4th-order residuals are not zero)
    assert np.abs(_residuals(me @ G, alpha, G, 4)).max() > 1e-3
    np.testing.assert_allclose(alpha.sum(1), [0, 0.386, 0.21, 0.63, 1, 1], atol=1e-14)


@pytest.mark.parametrize("theta", [0.2, 0.5, 0.8])
def test_rodas4_dense_output_conditions(theta):
    """Continuous extension weights w(θ) = θ m + θ(1−θ)(D2 + θ D3) satisfy the
    order-3 conditions for a step of length θh."""
    g, alpha, G, m, me, D = _standard_form()
    D2 = np.concatenate([D[0], [0.0]])
    D3 = np.concatenate([D[1], [0.0]])
    w = theta * m + theta * (1 - theta) * (D2 + theta * D3)
    assert np.abs(_residuals(w @ G, alpha, G, 3, theta)).max() < 1e-13


def _R(z):
    g, alpha, G, m, me, D = _standard_form()
    bh = alpha + G
    return 1 + z * (m @ G) @ np.linalg.solve(np.eye(6) - z * bh, np.ones(6))


def test_rodas4_stability_function_and_L_stability():
    """One step on u' = −λu returns R(−λh) of the tableau; R(−∞) = 0 (L-stable,
    P:322 'stiff'); R(z) ≈ e^z to O(z^5)."""
    for z in [-0.01, -0.1, -1.0, -10.0, -1e3, -1e6]:
        out, rc, *_ = oracle.solve("expdecay", "rodas4", [[1.0]], [[-z]], (0, 1), 1.0)
        assert rc[0] == 0
        R = out[0, 0, 0]
        assert abs(R - _R(z)) <= 1e-13 * max(1.0, abs(R)) + 1e-16, (z, R, _R(z))
    assert abs(_R(-1e12)) < 1e-10
    for z in [-0.1, -0.05]:
        assert abs(_R(z) - math.exp(z)) < 0.02 * abs(z) ** 5


def test_rodas4_convergence_order():
    """Order 4 on the linear harmonic oscillator (closed form) and on the
    nonlinear Lorenz system (reference: Tsit5 at h = 1e-5, itself pinned)."""
    errs = []
    for k in range(3, 7):
        out, *_ = oracle.solve("harmonic", "rodas4", [[1.0], [0.0]], [[1.0]], (0, 2), 2.0**-k)
        errs.append(np.abs(out[0, :, 0] - [math.cos(2), -math.sin(2)]).max())
    s = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all((s > 3.6) & (s < 4.6)), s
    u0, p = [[1.0], [0.0], [0.0]], [[10.0], [28.0], [8 / 3]]
    ref, *_ = oracle.solve("lorenz", "tsit5", u0, p, (0, 0.5), 1e-5)
    errs = []
    for k in range(6, 10):
        out, *_ = oracle.solve("lorenz", "rodas4", u0, p, (0, 0.5), 2.0**-k)
        errs.append(np.abs(out[0, :, 0] - ref[0, :, 0]).max())
    s = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all((s > 3.5) & (s < 4.7)), s


def test_rodas4_dense_output_accuracy_and_endpoints():
    """θ = 1 reproduces the step value bit-exactly; between grid points the
    interpolant converges with the method's order (local h^4, dense order 3)."""
    tau = np.array([0.25, 0.5, 0.6, 1.0])
    out, *_ = oracle.solve("harmonic", "rodas4", [[1.0], [0.0]], [[1.0]], (0, 1), 0.5, saveat=tau)
    fin, *_ = oracle.solve("harmonic", "rodas4", [[1.0], [0.0]], [[1.0]], (0, 0.5), 0.5)
    np.testing.assert_array_equal(out[1, :, 0], fin[0, :, 0])
    sa = np.array([0.3333, 0.7777, 1.4141])
    exact = np.stack([np.cos(sa), -np.sin(sa)], 1)
    errs = []
    for dt in [0.1, 0.05, 0.025]:
        out, *_ = oracle.solve("harmonic", "rodas4", [[1.0], [0.0]], [[1.0]], (0, 1.5), dt, saveat=sa)
        errs.append(np.abs(out[:, :, 0] - exact).max())
    s = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(s > 3.3), s


def test_rodas4_robertson_reference_and_invariant():
    """P:668-679 Robertson: literature values at t = 40 and 1e5; an exact-J
    Rosenbrock method preserves Σy = 1 to rounding."""
    g = gold("robertson_reference.json")
    u0 = [[1.0], [0.0], [0.0]]
    p = [[0.04], [3e7], [1e4]]
    out, rc, na, nr = oracle.solve("robertson", "rodas4", u0, p, (0, 40), 1e-4, adaptive=True,
                                   abstol=1e-10, reltol=1e-10)
    assert rc[0] == 0
    np.testing.assert_allclose(out[0, :, 0], g["t40"], rtol=1e-6)
    sa = np.linspace(0, 1e5, 100)
    out, rc, na, nr = oracle.solve("robertson", "rodas4", u0, p, (0, 1e5), 1e-4, adaptive=True,
                                   abstol=1e-8, reltol=1e-8, saveat=sa)
    assert rc[0] == 0 and na[0] < 3000
    assert np.abs(out[:, :, 0].sum(1) - 1).max() <= 1e-12
    np.testing.assert_allclose(out[-1, :, 0], g["t1e5"], rtol=2e-3)


def test_rodas4_stiff_suite_references():
    """P:733-844 OREGO / HIRES / POLLU against the IVP test-set references; the
    4th-order method reaches them in far fewer steps than Rosenbrock23."""
    from synth.inputs import make_inputs
    g = gold("stiff_references.json")
    for model, tol, bound in [("hires", 1e-10, 2e-6), ("pollu", 1e-10, 1e-6), ("orego", 1e-9, 1e-4)]:
        u0, p = make_inputs(model, "const", 1)
        if model == "pollu":
            u0[8, 0] = g["pollu"]["y9_0"]
        kw = dict(adaptive=True, abstol=tol, reltol=tol, p_broadcast=True)
        out, rc, na, nr = oracle.solve(model, "rodas4", u0, p, (0, g[model]["tf"]), 1e-6, **kw)
        assert rc[0] == 0
        ref = np.array(g[model]["y"])
        big = np.abs(ref) > 1e-10
        rel = np.abs(out[0, :, 0] - ref)[big] / np.abs(ref[big])
        assert rel.max() < bound, (model, rel.max())
        _, _, na23, _ = oracle.solve(model, "rosenbrock23", u0, p, (0, g[model]["tf"]), 1e-6, **kw)
        assert na[0] < na23[0] / 3, (model, na[0], na23[0])


def test_rodas4_hires_invariant_and_controller():
    """HIRES y7 + y8 = 0.0057 is preserved; the PI controller uses the p = 4
    rule β1 = 7/(10p), β2 = 2/(5p) (DESIGN R2)."""
    from synth.inputs import make_inputs
    u0, p = make_inputs("hires", "random10", 3, seed=5)
    sa = np.linspace(0, 321.8122, 50)
    out, rc, *_ = oracle.solve("hires", "rodas4", u0, p, (0, 321.8122), 1e-6, adaptive=True, abstol=1e-8,
                               reltol=1e-8, saveat=sa)
    assert (rc == 0).all()
    assert np.abs(out[:, 6, :] + out[:, 7, :] - 0.0057).max() < 1e-15
    c = oracle.controller("rodas4")
    assert c["beta1"] == 7 / 40 and c["beta2"] == 2 / 20


def test_rodas4_adaptive_tolerance_proportionality():
    """Global error at the end of an adaptive Lorenz run falls with the tolerance."""
    u0, p = [[1.0], [0.0], [0.0]], [[10.0], [28.0], [8 / 3]]
    ref, *_ = oracle.solve("lorenz", "tsit5", u0, p, (0, 1.0), 1e-5)
    errs = []
    for tol in [1e-5, 1e-7, 1e-9]:
        out, rc, *_ = oracle.solve("lorenz", "rodas4", u0, p, (0, 1.0), 1e-3, adaptive=True, abstol=tol, reltol=tol)
        assert rc[0] == 0
        errs.append(np.abs(out[0, :, 0] - ref[0, :, 0]).max() / np.abs(ref[0, :, 0]).max())
    assert errs[0] > errs[1] > errs[2] and errs[2] < 1e-6, errs


def test_rodas4_full_bseries_order():
    """Every rooted tree up to order 5 through the general Rosenbrock B-series
    recursion (tests/order_conditions.py): main order exactly 4, embedded 3."""
    from tests.order_conditions import rosenbrock_residuals
    g, A, C, D = oracle.rodas4_tableau()
    m = np.concatenate([A[5, :5], [1.0]])
    me = np.concatenate([A[5, :5], [0.0]])
    r = rosenbrock_residuals(A, C, g, m, 5)
    assert max(r[k] for k in range(1, 5)) < 1e-13 and r[5] > 1e-4, r
    r = rosenbrock_residuals(A, C, g, me, 4)
    assert max(r[k] for k in range(1, 4)) < 1e-13 and r[4] > 1e-3, r
