"""Pins for the oracle's Vern7 (GPUVern7; NEXT-1; DESIGN R21).

The tableau is checked against Butcher's rooted-tree order conditions
(tests/order_conditions.py) (all 85 trees of order ≤ 7 for b, all 37 of order ≤ 6 for the
embedded b̂ = b − b̃), the embedded scale against the structural zeros
b̂8 = b̂9 = 0 of Verner's 7(6) design (the order conditions leave one free
scale; one zero fixes it and the other must then vanish too), against measured
convergence orders on a closed-form and a nonlinear problem, and the saveat
rule against plain runs to the same end time (the dense output itself, R24:
tests/test_oracle_dense_output.py).
"""
import math

import numpy as np

import oracle
from tests.order_conditions import rk_max_residual


def _max_residual(b, A, order):
    return rk_max_residual(b, A, order)


def test_vern7_order_conditions():
    """b: order exactly 7 (85 conditions < 1e-13, order 8 violated); b̂: order
    exactly 6; row sums Σ_j a_ij = c_i; b̂2 = b̂3 = b2 = b3 = 0."""
    c, A, b, bt = oracle.vern7_tableau()
    np.testing.assert_allclose(A.sum(1), c, atol=2e-14)
    for k in range(1, 8):
        assert _max_residual(b, A, k) < 1e-13, k
    assert _max_residual(b, A, 8) > 1e-6
    bh = b - bt
    for k in range(1, 7):
        assert _max_residual(bh, A, k) < 1e-13, k
    assert _max_residual(bh, A, 7) > 1e-5
    assert b[1] == b[2] == bt[1] == bt[2] == 0.0


def test_vern7_embedded_scale_structural_zeros():
    """The embedded pair uses stage 10 (f at the new solution) in place of stages
    8 and 9: b̂8 = b̂9 = 0. The order-6 conditions fix b̂ − b up to one scale, so the
    two zeros are one condition plus an independent check (DESIGN R21). A wrong
    scale (round 1 typed b̂1 = 0.044063…, an error estimate 21 % too large) leaves
    b̂8 = 0.063, b̂9 = −0.017."""
    c, A, b, bt = oracle.vern7_tableau()
    bh = b - bt
    assert abs(bh[7]) < 1e-15 and abs(bh[8]) < 1e-15, (bh[7], bh[8])
    assert bt[9] != 0.0 and b[9] == 0.0
    # the scale is not a free choice any more: rescaling the estimate breaks the zeros
    for s in [0.9, 1.1]:
        bhs = b - s * bt
        assert abs(bhs[7]) > 1e-3 and abs(bhs[8]) > 1e-4


def test_vern7_stability_polynomial():
    """One step on u' = λu returns R(hλ) = 1 + z bᵀ(I − zA)⁻¹1 of the tableau,
    which agrees with e^z through z^7."""
    c, A, b, bt = oracle.vern7_tableau()
    for z in [-0.05, -0.3, -1.0, -2.5]:
        R = 1 + z * b @ np.linalg.solve(np.eye(10) - z * A, np.ones(10))
        out, rc, *_ = oracle.solve("expdecay", "vern7", [[1.0]], [[-z]], (0, 1), 1.0)
        assert rc[0] == 0
        assert abs(out[0, 0, 0] - R) <= 2e-14 * max(1, abs(R)), (z, out[0, 0, 0], R)   # |a_ij| up to 187
        if abs(z) <= 0.3:
            assert abs(R - math.exp(z)) < abs(z) ** 8 / math.factorial(8) * 5


def test_vern7_convergence_order():
    """Order 7 on the harmonic oscillator (closed form) and Lorenz (reference:
    Tsit5 at h = 2e-5, itself pinned to order 5)."""
    errs = []
    for h in [0.4, 0.2, 0.1]:
        out, *_ = oracle.solve("harmonic", "vern7", [[1.0], [0.0]], [[1.0]], (0, 8), h)
        errs.append(np.abs(out[0, :, 0] - [math.cos(8), -math.sin(8)]).max())
    s = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all((s > 6.3) & (s < 7.8)), (s, errs)
    u0, p = [[1.0], [0.0], [0.0]], [[10.0], [28.0], [8 / 3]]
    ref, *_ = oracle.solve("lorenz", "tsit5", u0, p, (0, 1.0), 2e-5)
    errs = []
    for h in [0.02, 0.01, 0.005]:
        out, *_ = oracle.solve("lorenz", "vern7", u0, p, (0, 1.0), h)
        errs.append(np.abs(out[0, :, 0] - ref[0, :, 0]).max())
    s = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all((s > 6.0) & (s < 8.0)), (s, errs)


def test_vern7_embedded_error_estimate_order():
    """The local error estimate scales like h^7 (embedded order 6): the
    adaptive controller's accepted-step count grows like tol^(-1/7)."""
    u0, p = [[1.0], [0.0], [0.0]], [[10.0], [28.0], [8 / 3]]
    counts = []
    for tol in [1e-6, 1e-8, 1e-10, 1e-12]:
        out, rc, na, nr = oracle.solve("lorenz", "vern7", u0, p, (0, 1.0), 1e-3, adaptive=True, abstol=tol,
                                       reltol=tol)
        assert rc[0] == 0
        counts.append(na[0])
    r = np.log10(np.array(counts[1:]) / np.array(counts[:-1])) / 2.0   # per decade of tol
    assert np.all((r > 1 / 7 - 0.06) & (r < 1 / 7 + 0.08)), (counts, r)


def test_vern7_adaptive_accuracy_and_efficiency():
    """At tol 1e-10 Vern7 reaches the reference with far fewer steps than Tsit5."""
    u0, p = [[1.0], [0.0], [0.0]], [[10.0], [28.0], [8 / 3]]
    ref, *_ = oracle.solve("lorenz", "tsit5", u0, p, (0, 1.0), 2e-5)
    out, rc, na, nr = oracle.solve("lorenz", "vern7", u0, p, (0, 1.0), 1e-3, adaptive=True, abstol=1e-10,
                                   reltol=1e-10)
    _, _, nat, _ = oracle.solve("lorenz", "tsit5", u0, p, (0, 1.0), 1e-3, adaptive=True, abstol=1e-10,
                                reltol=1e-10)
    assert rc[0] == 0
    assert np.abs(out[0, :, 0] - ref[0, :, 0]).max() / np.abs(ref[0, :, 0]).max() < 1e-8
    assert na[0] < nat[0] / 2, (na[0], nat[0])


def test_vern7_saveat_rule():
    """Adaptive saves (R24: interior τ by a shortened step from the step's
    start): the saved values match the closed form to the tolerance, τ = t0
    stores u0, and a single save at τ = tf equals the plain run's final state."""
    sa = np.array([0.0, 0.37, 1.0, 2.2, 3.0])
    out, rc, na, nr = oracle.solve("harmonic", "vern7", [[1.0], [0.0]], [[1.0]], (0, 3.0), 0.1, adaptive=True,
                                   abstol=1e-12, reltol=1e-12, saveat=sa)
    assert rc[0] == 0
    exact = np.stack([np.cos(sa), -np.sin(sa)], 1)
    assert np.abs(out[:, :, 0] - exact).max() < 1e-10
    np.testing.assert_array_equal(out[0, :, 0], [1.0, 0.0])
    fin, *_ = oracle.solve("harmonic", "vern7", [[1.0], [0.0]], [[1.0]], (0, 3.0), 0.1, adaptive=True,
                           abstol=1e-12, reltol=1e-12, saveat=[3.0])
    single, *_ = oracle.solve("harmonic", "vern7", [[1.0], [0.0]], [[1.0]], (0, 3.0), 0.1, adaptive=True,
                              abstol=1e-12, reltol=1e-12)
    np.testing.assert_array_equal(fin[0, :, 0], single[0, :, 0])


def test_vern7_fixed_grid_saves():
    """Fixed step: saves on grid points equal the state after that many steps."""
    sa = np.array([0.0, 0.5, 1.0])
    out, *_ = oracle.solve("lorenz", "vern7", [[1.0], [0.0], [0.0]], [[10.0], [28.0], [8 / 3]], (0, 1.0), 0.01,
                           saveat=sa)
    half, *_ = oracle.solve("lorenz", "vern7", [[1.0], [0.0], [0.0]], [[10.0], [28.0], [8 / 3]], (0, 0.5), 0.01)
    # (the shorter run's last step is (0.5 − 49·0.01) = 0.01 + 9e-18: equal up to rounding)
    np.testing.assert_allclose(out[1, :, 0], half[0, :, 0], rtol=1e-14)
    np.testing.assert_array_equal(out[0, :, 0], [1.0, 0.0, 0.0])


def test_vern7_controller_constants():
    c = oracle.controller("vern7")
    assert c["beta1"] == 7 / 70 and c["beta2"] == 2 / 35
