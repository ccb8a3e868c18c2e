"""Pins for the oracle's Vern9 (GPUVern9; NEXT-1; DESIGN R21).

Butcher's rooted-tree conditions (tests/order_conditions.py): b of order
exactly 9 (all 486 trees of order ≤ 9), b̂ = b − b̃ of order exactly 8; the
embedded scale (fixed by the published b̂1) is pinned independently by the
emergent b̂14 = b̂15 = 0 of Verner's design; plus the stability polynomial of
one step, measured order 9 and efficiency against Vern7.
"""
import math

import numpy as np

import oracle
from tests.order_conditions import rk_max_residual


def test_vern9_order_conditions():
    c, A, b, bt = oracle.vern9_tableau()
    np.testing.assert_allclose(A.sum(1), c, atol=2e-14)
    for k in range(1, 10):
        assert rk_max_residual(b, A, k) < 1e-13, k
    assert rk_max_residual(b, A, 10) > 1e-7
    bh = b - bt
    for k in range(1, 9):
        assert rk_max_residual(bh, A, k) < 1e-13, k
    assert rk_max_residual(bh, A, 9) > 1e-6
    assert (b[1:7] == 0).all() and (bt[1:7] == 0).all() and b[15] == 0
    # the one-parameter family of order-8 embedded weights with b̂14 = 0 also has
    # b̂15 = 0 (an independent check of the scale) and the published b̂1
    assert abs(bh[13]) < 1e-15 and abs(bh[14]) < 1e-13
    assert abs(bh[0] - 0.01996996514886773) < 5e-14


def test_vern9_stability_polynomial():
    c, A, b, bt = oracle.vern9_tableau()
    for z in [-0.05, -0.4, -1.5, -3.0]:
        R = 1 + z * b @ np.linalg.solve(np.eye(16) - z * A, np.ones(16))
        out, rc, *_ = oracle.solve("expdecay", "vern9", [[1.0]], [[-z]], (0, 1), 1.0)
        assert rc[0] == 0
        assert abs(out[0, 0, 0] - R) <= 2e-14 * max(1, abs(R)), (z, out[0, 0, 0], R)
        if abs(z) <= 0.4:
            assert abs(R - math.exp(z)) < abs(z) ** 10 / math.factorial(10) * 5


def test_vern9_convergence_order():
    errs = []
    for h in [0.8, 0.4, 0.2]:
        out, *_ = oracle.solve("harmonic", "vern9", [[1.0], [0.0]], [[1.0]], (0, 8), h)
        errs.append(np.abs(out[0, :, 0] - [math.cos(8), -math.sin(8)]).max())
    s = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all((s > 8.5) & (s < 10.2)), (s, errs)
    # nonlinear (Lorenz): high order, well above Vern7's 7 (reference: Tsit5, h = 2e-5)
    u0, p = [[1.0], [0.0], [0.0]], [[10.0], [28.0], [8 / 3]]
    ref, *_ = oracle.solve("lorenz", "tsit5", u0, p, (0, 1.0), 2e-5)
    e = [np.abs(oracle.solve("lorenz", "vern9", u0, p, (0, 1.0), h)[0][0, :, 0] - ref[0, :, 0]).max()
         for h in [0.04, 0.02]]
    assert 8.0 < math.log2(e[0] / e[1]) < 12.5, e


def test_vern9_adaptive_efficiency_and_accuracy():
    u0, p = [[1.0], [0.0], [0.0]], [[10.0], [28.0], [8 / 3]]
    ref, *_ = oracle.solve("lorenz", "tsit5", u0, p, (0, 1.0), 2e-5)
    counts = []
    for tol in [1e-6, 1e-8, 1e-10, 1e-12]:
        out, rc, na, nr = oracle.solve("lorenz", "vern9", u0, p, (0, 1.0), 1e-3, adaptive=True, abstol=tol,
                                       reltol=tol)
        assert rc[0] == 0
        counts.append(na[0])
        if tol == 1e-10:
            assert np.abs(out[0, :, 0] - ref[0, :, 0]).max() / np.abs(ref[0, :, 0]).max() < 1e-9
            _, _, na7, _ = oracle.solve("lorenz", "vern7", u0, p, (0, 1.0), 1e-3, adaptive=True, abstol=tol,
                                        reltol=tol)
            assert na[0] < na7[0] * 0.6, (na[0], na7[0])
    r = np.log10(np.array(counts[1:]) / np.array(counts[:-1])) / 2.0
    assert np.all((r > 1 / 9 - 0.05) & (r < 1 / 9 + 0.05)), (counts, r)
    c = oracle.controller("vern9")
    assert c["beta1"] == 7 / 90 and c["beta2"] == 2 / 45
