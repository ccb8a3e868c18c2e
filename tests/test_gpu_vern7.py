"""GPU ↔ oracle parity for Vern7 (GPUVern7; NEXT-1; DESIGN R21)
through the C ABI (-m gpu). Bars of BASELINE.json north_star: fixed step rel ≤
1e-12 (fp64) / 1e-5 (fp32); adaptive fp64 at 1e-10: final rel ≤ 1e-8 and
identical accepted-step counts on ≥ 99.9 % of trajectories."""
import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs
from tests.helpers import check_adaptive, check_fixed, gpu, traj_relerr

pytestmark = pytest.mark.gpu

TOL_FIXED = {"f32": 1e-5, "f64": 1e-12}


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("model,recipe,tf,dt", [("lorenz", "rho_sweep", 1.0, 1e-3), ("lorenz", "random10", 1.0, 0.01),
                                                ("harmonic", "random10", 4.0, 0.05)])
def test_vern7_fixed_parity(model, recipe, tf, dt, dtype):
    N = 2051
    u0, p = make_inputs(model, recipe, N, seed=0x77, dtype=dtype)
    nsteps = int(round(tf / dt))
    sa = np.array([0.0, dt * (nsteps // 3), dt * (nsteps // 2), tf])      # grid points (R21)
    g, rc, na, nr, _ = gpu(model, "vern7", u0, p, (0.0, tf), dt, saveat=sa)
    o, orc, ona, _ = oracle.solve(model, "vern7", u0, p, (0.0, tf), dt, dtype=dtype, saveat=sa)
    np.testing.assert_array_equal(rc, orc)
    np.testing.assert_array_equal(na, ona)
    check_fixed(g, o, TOL_FIXED[dtype])


@pytest.mark.parametrize("refill", [False, True])
def test_vern7_adaptive_tight_tolerance(refill):
    """north_star adaptive bar (fp64, abstol = reltol = 1e-10) with interior
    save points (dense output by a shortened step, DESIGN R24)."""
    N = 1029
    u0, p = make_inputs("lorenz", "random10", N, seed=0xC1, dtype="f64")
    sa = np.array([0.0, 0.25, 0.5, 0.8125, 1.0])
    g, rc, na, nr, _ = gpu("lorenz", "vern7", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-10, reltol=1e-10,
                           saveat=sa, refill=refill)
    o, orc, ona, onr = oracle.solve("lorenz", "vern7", u0, p, (0.0, 1.0), 1e-3, dtype="f64", adaptive=True,
                                    abstol=1e-10, reltol=1e-10, saveat=sa)
    np.testing.assert_array_equal(rc, orc)
    check_adaptive(g, o, (na, nr), (ona, onr), tol=1e-8)


def test_vern7_adaptive_final_only_and_f32():
    N = 777
    u0, p = make_inputs("lorenz", "random10", N, seed=5, dtype="f64")
    g, rc, na, nr, _ = gpu("lorenz", "vern7", u0, p, (0.0, 2.0), 1e-3, adaptive=True, abstol=1e-8, reltol=1e-8)
    o, orc, ona, onr = oracle.solve("lorenz", "vern7", u0, p, (0.0, 2.0), 1e-3, dtype="f64", adaptive=True,
                                    abstol=1e-8, reltol=1e-8)
    check_adaptive(g, o, (na, nr), (ona, onr), tol=1e-8)
    u0, p = make_inputs("lorenz", "random10", N, seed=6, dtype="f32")
    g, rc, na, nr, _ = gpu("lorenz", "vern7", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-5, reltol=1e-5)
    o, orc, ona, onr = oracle.solve("lorenz", "vern7", u0, p, (0.0, 1.0), 1e-3, dtype="f32", adaptive=True,
                                    abstol=1e-5, reltol=1e-5)
    # fp32 at 1e-5: rounding-level agreement where the step counts match; any re-routed
    # trajectory must be as accurate as the oracle's own (tests/helpers.check_adaptive)
    ref, *_ = oracle.solve("lorenz", "vern7", u0.astype(np.float64), p.astype(np.float64), (0.0, 1.0), 1e-3,
                           dtype="f64", adaptive=True, abstol=1e-11, reltol=1e-11)
    check_adaptive(g, o, (na, nr), (ona, onr), tol=1e-2, tol_same=1e-5, ref=ref)


def test_vern7_ragged_single_and_offgrid_saveat():
    """Ragged / single-trajectory launches, and fixed-step saves between grid
    points (R24: one Vern7 step of length τ − t_s from the step's start)."""
    for N in [1, 257]:
        u0, p = make_inputs("harmonic", "random10", N, seed=3, dtype="f64")
        g, rc, *_ = gpu("harmonic", "vern7", u0, p, (0.0, 3.0), 0.1, adaptive=True, abstol=1e-9, reltol=1e-9,
                        saveat=[1.0, 2.5])
        o, orc, *_ = oracle.solve("harmonic", "vern7", u0, p, (0.0, 3.0), 0.1, dtype="f64", adaptive=True,
                                  abstol=1e-9, reltol=1e-9, saveat=[1.0, 2.5])
        np.testing.assert_array_equal(rc, orc)
        assert traj_relerr(g, o).max() <= 1e-8
    for dtype in ["f64", "f32"]:
        u0, p = make_inputs("lorenz", "random10", 333, seed=8, dtype=dtype)
        sa = [0.0, 0.005, 0.1234, 0.5, 0.7777, 1.0]
        g, rc, na, *_ = gpu("lorenz", "vern7", u0, p, (0.0, 1.0), 0.01, saveat=sa)
        o, orc, ona, _ = oracle.solve("lorenz", "vern7", u0, p, (0.0, 1.0), 0.01, dtype=dtype, saveat=sa)
        np.testing.assert_array_equal(rc, orc)
        np.testing.assert_array_equal(na, ona)
        check_fixed(g, o, TOL_FIXED[dtype])
