"""GPU ↔ oracle parity of the dense output of Vern7 / Vern9 / Rodas5 / Rodas5P
(DESIGN R24: a save point inside a step stores one step of the method from the
step's start) through the C ABI (-m gpu), and the property R24 exists for: the
GPU's adaptive step sequence does not depend on saveat."""
import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs
from tests.helpers import check_adaptive, check_fixed, gpu

pytestmark = pytest.mark.gpu

CASES = {   # alg: (model, recipe, seed, tspan, dt0, tol)
    "vern7": ("lorenz", "random10", 0xD7, (0.0, 1.0), 1e-3, 1e-10),
    "vern9": ("lorenz", "random10", 0xD9, (0.0, 1.0), 1e-3, 1e-10),
    "rodas5": ("robertson", "random10", 0xD5, (0.0, 1e3), 1e-4, 1e-8),
    "rodas5p": ("robertson", "random10", 0xDF, (0.0, 1e3), 1e-4, 1e-8),
}


@pytest.mark.parametrize("refill", [False, True])
@pytest.mark.parametrize("alg", list(CASES))
def test_dense_adaptive_parity_and_saveat_independence(alg, refill):
    model, recipe, seed, tspan, dt0, tol = CASES[alg]
    N = 1537
    u0, p = make_inputs(model, recipe, N, seed=seed, dtype="f64")
    sa = np.linspace(tspan[0], tspan[1], 41)
    sa[1:-1] += 0.37 * (sa[1] - sa[0]) * np.sin(np.arange(1, 40))   # irregular interior points
    sa = np.sort(sa)
    kw = dict(adaptive=True, abstol=tol, reltol=tol)
    g, rc, na, nr, _ = gpu(model, alg, u0, p, tspan, dt0, saveat=sa, refill=refill, **kw)
    o, orc, ona, onr = oracle.solve(model, alg, u0, p, tspan, dt0, dtype="f64", saveat=sa, **kw)
    np.testing.assert_array_equal(rc, orc)
    check_adaptive(g, o, (na, nr), (ona, onr), tol=1e-8)
    gf, rcf, naf, nrf, _ = gpu(model, alg, u0, p, tspan, dt0, refill=refill, **kw)
    np.testing.assert_array_equal(na, naf)
    np.testing.assert_array_equal(nr, nrf)
    np.testing.assert_array_equal(g[-1], gf[0])      # τ = tf: the final state, bit for bit


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("alg", list(CASES))
def test_dense_fixed_offgrid_parity(alg, dtype):
    model = "harmonic" if alg.startswith("vern") else "robertson"
    if dtype == "f32" and alg.startswith("rodas"):
        model = "harmonic"
    tf, dt = (4.0, 0.05) if model == "harmonic" else (10.0, 0.01)
    N = 1029
    u0, p = make_inputs(model, "random10", N, seed=0xDE, dtype=dtype)
    sa = np.array([0.0, 0.3 * dt, 0.31 * tf, 0.5 * tf, 0.5 * tf + 0.77 * dt, tf - 0.01 * dt, tf])
    g, rc, na, _, _ = gpu(model, alg, u0, p, (0.0, tf), dt, saveat=sa)
    o, orc, ona, _ = oracle.solve(model, alg, u0, p, (0.0, tf), dt, dtype=dtype, saveat=sa)
    np.testing.assert_array_equal(rc, orc)
    np.testing.assert_array_equal(na, ona)
    check_fixed(g, o, {"f32": 1e-5, "f64": 1e-12}[dtype])


@pytest.mark.parametrize("alg", list(CASES))
def test_dense_adaptive_f32(alg):
    """fp32 adaptive runs with interior save points: parity at the fp32 bars
    (tests/helpers.check_adaptive: identical step counts on ≥ 99.9 %, rounding-level
    agreement where they match, re-routed trajectories as accurate as the
    oracle's own against an fp64 reference) and saveat-independent GPU step counts."""
    model, recipe, seed, tspan, dt0, _ = CASES[alg]
    N = 1031
    u0, p = make_inputs(model, recipe, N, seed=seed + 1, dtype="f32")
    sa = np.sort(np.concatenate([[tspan[0], tspan[1]], tspan[0] + (tspan[1] - tspan[0]) *
                                 np.array([0.013, 0.2, 0.37, 0.5, 0.81])]))
    kw = dict(adaptive=True, abstol=1e-5, reltol=1e-5)
    g, rc, na, nr, _ = gpu(model, alg, u0, p, tspan, dt0, saveat=sa, **kw)
    o, orc, ona, onr = oracle.solve(model, alg, u0, p, tspan, dt0, dtype="f32", saveat=sa, **kw)
    ref, *_ = oracle.solve(model, alg, u0.astype(np.float64), p.astype(np.float64), tspan, dt0, dtype="f64",
                           saveat=sa, adaptive=True, abstol=1e-9, reltol=1e-9)
    np.testing.assert_array_equal(rc, orc)
    check_adaptive(g, o, (na, nr), (ona, onr), tol=1e-2, tol_same=1e-5, ref=ref)
    _, _, naf, nrf, _ = gpu(model, alg, u0, p, tspan, dt0, **kw)
    np.testing.assert_array_equal(na, naf)
    np.testing.assert_array_equal(nr, nrf)
