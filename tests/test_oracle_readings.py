"""Pins of the oracle's Rosenbrock23 error estimate, and what the R1 / R2 / R8
evaluation forms change (-m "not gpu").

1. The Rosenbrock23 embedded estimate E = h/6 (k1 − 2 k2 + k3) (P:124-138 form,
   Shampine–Reichelt ode23s cited at P:321; DESIGN R10) is the difference between
   the embedded 3rd-order solution and u_new, so to leading order it is MINUS the
   true local error of u_new ("embedded estimate within 0.1 % at
   z = −0.01; local error ratio 7.96 on halving"). Checked against the closed
   form e^z on u' = λu and against a DOP853 reference step on Lorenz; a flipped k3
   sign, a mistyped e32 or d, or a wrong 1/6 each fail one of them.

2. Readings R1 (Tsit5 stage sums as u + Σ (h·a_ij) k_j, the products rounded to T,
   instead of u + h·Σ a_ij k_j), R2 (PI controller in the exponent domain with polynomial log2 / exp2,
   instead of libm pow) and R8 (Box–Muller with a polynomial log2 and sincospi,
   instead of libm log / sin / cos) are evaluation forms chosen so that oracle and
   kernel round identically. The oracle's test-only plain mode evaluates them
   literally (the printed stage sum; P:120 with pow; libm Box–Muller). These tests run the BASELINE
   ensembles in both modes and check that the readings change nothing the north
   star measures: fp64 step counts and final states (C1 at 1e-8 / 1e-10, C3),
   fp32 adaptive final states within the solutions' own global error (C2), and
   EM paths, fixed-step states within the fixed-step bars. Measured agreement is
   recorded in DESIGN R1 / R2 / R8.
"""
import math

import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs


# ------------------------------------------------- Rosenbrock23 estimate ----
def _ros23_expdecay(z):
    """One step of u' = −λu from u = 1 with λ = 1, h = −z: (u_new, E, true local error)."""
    un, E = oracle.ros23_step("expdecay", [1.0], [1.0], 0.0, -z)
    return un[0], E[0], un[0] - math.exp(z)


def test_ros23_error_estimate_linear_closed_form():
    """At z = hλ = −0.01, E = −(u_new − e^z) within 0.1 %."""
    un, E, err = _ros23_expdecay(-0.01)
    assert abs(E / -err - 1.0) <= 1e-3, (E, err)
    # also for growth (z > 0) and a smaller step: the ratio tends to 1 as O(z)
    for z, tol in [(0.01, 1e-3), (-0.002, 2e-4)]:
        _, E, err = _ros23_expdecay(z)
        assert abs(E / -err - 1.0) <= tol, (z, E, err)


def test_ros23_local_error_order_on_halving():
    """Local error of the order-2 solution ∝ h³: ratio ≈ 8 on halving (7.96 at
    z = −0.01), and the estimate halves the same way."""
    _, E1, err1 = _ros23_expdecay(-0.01)
    _, E2, err2 = _ros23_expdecay(-0.005)
    assert 7.7 <= err1 / err2 <= 8.3, err1 / err2
    assert 7.7 <= E1 / E2 <= 8.3, E1 / E2


def test_ros23_error_estimate_lorenz_vs_reference_step():
    """Nonlinear system with the exact Jacobian: E matches the true local error
    of u_new (from a DOP853 reference of the same step) to 0.1 % of its size."""
    from scipy.integrate import solve_ivp
    p = np.array([10.0, 28.0, 8.0 / 3.0])
    u = np.array([1.0, 2.0, 3.0])

    def f(t, y):
        return [p[0] * (y[1] - y[0]), y[0] * (p[1] - y[2]) - y[1], y[0] * y[1] - p[2] * y[2]]

    for h in [2e-4, 1e-4]:
        un, E = oracle.ros23_step("lorenz", u, p, 0.0, h)
        ex = solve_ivp(f, (0.0, h), u, method="DOP853", rtol=2.3e-14, atol=1e-18).y[:, -1]
        err = un - ex
        assert np.abs(E + err).max() <= 2e-3 * np.abs(err).max(), (h, E, err)


# ----------------------------------------------- R2 / R8 plain cross-check --
def _both_modes(model, alg, u0, p, tspan, dt, **kw):
    res = {}
    try:
        for plain in (False, True):
            oracle.set_plain(plain)
            res[plain] = oracle.solve(model, alg, u0, p, tspan, dt, **kw)
    finally:
        oracle.set_plain(False)
    return res[False], res[True]


def _relerr(a, b):
    """Per-trajectory ∞-norm relative error (DESIGN §3 last bullet)."""
    return np.abs(a - b).max(axis=(0, 1)) / np.abs(b).max(axis=(0, 1))


def test_plain_mode_switches_and_restores():
    """The plain mode really changes the evaluation (not bit-identical) and the
    default is restored."""
    u0, p = make_inputs("lorenz", "random10", 64, seed=0xC1, dtype="f64")
    canon, plain = _both_modes("lorenz", "tsit5", u0, p, (0, 1), 1e-3, dtype="f64", adaptive=True,
                               abstol=1e-8, reltol=1e-8)
    assert not np.array_equal(canon[0], plain[0])
    again = oracle.solve("lorenz", "tsit5", u0, p, (0, 1), 1e-3, dtype="f64", adaptive=True, abstol=1e-8,
                         reltol=1e-8)
    assert np.array_equal(again[0], canon[0])
    z0 = oracle.normals(0xC4, 3, 0, 8, dtype="f64")
    with oracle.plain_mode():
        z1 = oracle.normals(0xC4, 3, 0, 8, dtype="f64")
    assert not np.array_equal(z0, z1) and np.abs(z0 - z1).max() < 1e-14


@pytest.mark.parametrize("tol", [1e-8, 1e-10])
def test_r2_reading_fp64_c1(tol):
    """C1 (Lorenz, N = 1024, random p ±10 %, fp64): the exponent-domain controller
    and the literal pow controller take identical step counts on ≥ 99.9 % of the
    trajectories and final states agree within 1e-8 (the north-star fp64 bars)."""
    u0, p = make_inputs("lorenz", "random10", 1024, seed=0xC1, dtype="f64")
    (a, _, na_a, nr_a), (b, _, na_b, nr_b) = _both_modes("lorenz", "tsit5", u0, p, (0, 1), 1e-3, dtype="f64",
                                                        adaptive=True, abstol=tol, reltol=tol)
    same = ((na_a == na_b) & (nr_a == nr_b)).mean()
    rel = _relerr(a, b)
    print(f"R2 C1 tol {tol:g}: identical counts {same:.4f}, max rel {rel.max():.2e}")
    assert same >= 0.999
    assert rel.max() <= 1e-8


def test_r2_reading_fp64_c3_rosenbrock23():
    """C3 (Robertson, Rosenbrock23, fp64, 1e-8, 100 saves): same bars as C1."""
    u0, p = make_inputs("robertson", "random10", 256, seed=0xC3, dtype="f64")
    sa = np.linspace(0.0, 1e5, 100)
    (a, _, na_a, nr_a), (b, _, na_b, nr_b) = _both_modes("robertson", "rosenbrock23", u0, p, (0, 1e5), 1e-4,
                                                        dtype="f64", adaptive=True, abstol=1e-8, reltol=1e-8,
                                                        saveat=sa)
    same = ((na_a == na_b) & (nr_a == nr_b)).mean()
    rel = _relerr(a, b)
    print(f"R2 C3: identical counts {same:.4f}, max rel {rel.max():.2e}")
    assert same >= 0.999 and rel.max() <= 1e-8


def test_r2_reading_fp32_c2_adaptive():
    """C2 adaptive (Lorenz ρ sweep, fp32, 1e-6). In fp32 at this tolerance the
    error estimate E ≈ tol·|u| sits a few ulps of |u| above rounding noise, so any
    one-ulp change of h re-routes the step sequence: identical counts are a
    property of bit-identical arithmetic only, not of the method (measured: ≈61 %
    identical between the two controller forms). What the reading must not change
    is the solution: the two final states differ by no more than the larger of
    their own global errors against a tight fp64 reference."""
    N = 4096
    u0, p = make_inputs("lorenz", "rho_sweep", N, dtype="f32")
    (a, *_), (b, *_) = _both_modes("lorenz", "tsit5", u0, p, (0, 1), 1e-3, dtype="f32", adaptive=True,
                                   abstol=1e-6, reltol=1e-6)
    ref, *_ = oracle.solve("lorenz", "tsit5", u0.astype(np.float64), p.astype(np.float64), (0, 1), 1e-3,
                           dtype="f64", adaptive=True, abstol=1e-12, reltol=1e-12)
    ga = _relerr(a.astype(np.float64), ref)
    gb = _relerr(b.astype(np.float64), ref)
    d = _relerr(a.astype(np.float64), b.astype(np.float64))
    print(f"R2 C2a fp32: global err canon {ga.max():.2e} plain {gb.max():.2e}; canon-vs-plain {d.max():.2e}")
    assert d.max() <= max(ga.max(), gb.max())
    assert np.quantile(d, 0.99) <= 1e-5


@pytest.mark.parametrize("dtype,ulps", [("f32", 16), ("f64", 16)])
def test_r8_reading_normals(dtype, ulps):
    """R8: the polynomial Box–Muller normals equal the libm ones within a few ulp
    (relative to max(|Z|, 1)) over 3·10^4 draws."""
    a = oracle.normals(0xC4, 11, 0, 10000, dtype=dtype)
    with oracle.plain_mode():
        b = oracle.normals(0xC4, 11, 0, 10000, dtype=dtype)
    eps = np.finfo(a.dtype).eps
    dev = (np.abs(a.astype(np.float64) - b) / np.maximum(np.abs(b), 1.0)).max() / eps
    print(f"R8 {dtype}: max deviation {dev:.1f} ulp")
    assert dev <= ulps


@pytest.mark.parametrize("model", ["lorenz_sde_add", "lorenz_sde_mul"])
@pytest.mark.parametrize("dtype,tol", [("f32", 1e-5), ("f64", 1e-12)])
def test_r8_reading_em_paths(model, dtype, tol):
    """C4 stochastic Lorenz EM paths (1000 steps): the two Box–Muller forms give
    the same paths within the fixed-step parity bars of the north star."""
    u0, p = make_inputs(model, "const", 256, dtype=dtype)
    (a, *_), (b, *_) = _both_modes(model, "em", u0, p, (0, 1), 1e-3, dtype=dtype, p_broadcast=True, seed=0xC4)
    rel = _relerr(a.astype(np.float64), b.astype(np.float64))
    print(f"R8 EM {model} {dtype}: max rel {rel.max():.2e}")
    assert rel.max() <= tol


@pytest.mark.parametrize("recipe,seed", [("rho_sweep", 0), ("random10", 0xC5)])
@pytest.mark.parametrize("dtype,bar", [("f64", 1e-12), ("f32", 1e-5)])
def test_r1_reading_fixed_step(recipe, seed, dtype, bar):
    """R1 vs the stage sum as printed (y = u + h·Σ a_ij k_j), fixed dt = 1e-3 on the
    C2 / C5 ensembles: the two forms agree within the north star's fixed-step parity
    bars (fp64 1e-12, fp32 1e-5); measured 1.4e-14 / 9.2e-6. Against a tight fp64
    reference both are equally accurate in fp64 (6.0e-12); in fp32 the rounded
    products h·a_ij perturb the tableau (6e-8 relative), so R1's fp32 global error
    is larger (1.0e-5 vs 3.2e-6 on the ρ sweep) — recorded in DESIGN R1."""
    u0, p = make_inputs("lorenz", recipe, 2048, seed=seed, dtype=dtype, N_total=2048)
    (a, *_), (b, *_) = _both_modes("lorenz", "tsit5", u0, p, (0, 1), 1e-3, dtype=dtype)
    rel = _relerr(a.astype(np.float64), b.astype(np.float64))
    ref, *_ = oracle.solve("lorenz", "tsit5", u0.astype(np.float64), p.astype(np.float64), (0, 1), 1e-3,
                           dtype="f64", adaptive=True, abstol=1e-13, reltol=1e-13)
    ea = _relerr(a.astype(np.float64), ref).max()
    eb = _relerr(b.astype(np.float64), ref).max()
    print(f"R1 {recipe} {dtype}: canon-vs-plain {rel.max():.2e}; error canon {ea:.2e} plain {eb:.2e}")
    assert rel.max() <= bar
    if dtype == "f64":
        assert ea <= 1.01 * eb + 1e-14
    else:
        assert ea <= 5 * eb and ea <= 2e-5
