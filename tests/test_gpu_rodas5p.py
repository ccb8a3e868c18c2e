"""GPU ↔ oracle parity for Rodas5P (GPURodas5P, NEXT-2; DESIGN R23) through the C ABI (-m gpu):
fixed step rel ≤ 1e-12 (fp64) / 1e-5 (fp32); adaptive fp64 rel ≤ 1e-8 with
identical step counts on ≥ 99.9 % of trajectories."""
import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs
from tests.helpers import check_adaptive, check_fixed, gpu, traj_relerr

pytestmark = pytest.mark.gpu

TOL_FIXED = {"f32": 1e-5, "f64": 1e-12}


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("model,tf,dt", [("lorenz", 1.0, 1e-3), ("robertson", 1.0, 1e-3), ("hires", 10.0, 0.01)])
def test_rodas5p_fixed_parity(model, tf, dt, dtype):
    N = 1027
    u0, p = make_inputs(model, "random10", N, seed=0x55, dtype=dtype)
    ns = int(round(tf / dt))
    sa = np.array([0.0, dt * (ns // 4), tf])
    g, rc, na, nr, _ = gpu(model, "rodas5p", u0, p, (0.0, tf), dt, saveat=sa)
    o, orc, ona, _ = oracle.solve(model, "rodas5p", u0, p, (0.0, tf), dt, dtype=dtype, saveat=sa)
    np.testing.assert_array_equal(rc, orc)
    np.testing.assert_array_equal(na, ona)
    check_fixed(g, o, TOL_FIXED[dtype])


@pytest.mark.parametrize("refill", [False, True])
def test_rodas5p_robertson_c3_shape(refill):
    N = 1030
    u0, p = make_inputs("robertson", "random10", N, seed=0xC3, dtype="f64")
    sa = np.linspace(0.0, 1e5, 100)
    g, rc, na, nr, _ = gpu("robertson", "rodas5p", u0, p, (0.0, 1e5), 1e-4, adaptive=True, abstol=1e-8,
                           reltol=1e-8, saveat=sa, refill=refill)
    o, orc, ona, onr = oracle.solve("robertson", "rodas5p", u0, p, (0.0, 1e5), 1e-4, dtype="f64", adaptive=True,
                                    abstol=1e-8, reltol=1e-8, saveat=sa)
    assert (rc == 0).all() and (orc == 0).all()
    check_adaptive(g, o, (na, nr), (ona, onr), tol=1e-8)
    assert np.abs(g.sum(1) - 1).max() <= 1e-12


@pytest.mark.parametrize("model,tf,N", [("orego", 30.0, 300), ("hires", 321.8122, 500), ("pollu", 60.0, 300)])
def test_rodas5p_stiff_suite_parity(model, tf, N):
    u0, p = make_inputs(model, "random10", N, seed=0x57, dtype="f64")
    sa = np.linspace(0.0, tf, 7)
    g, rc, na, nr, _ = gpu(model, "rodas5p", u0, p, (0.0, tf), 1e-6, adaptive=True, abstol=1e-8, reltol=1e-8,
                           saveat=sa)
    o, orc, ona, onr = oracle.solve(model, "rodas5p", u0, p, (0.0, tf), 1e-6, dtype="f64", adaptive=True,
                                    abstol=1e-8, reltol=1e-8, saveat=sa)
    np.testing.assert_array_equal(rc, orc)
    assert (rc == 0).mean() > 0.99
    check_adaptive(g, o, (na, nr), (ona, onr), tol=1e-8)


def test_rodas5p_tight_tolerance_and_ragged():
    for N in [1, 777]:
        u0, p = make_inputs("lorenz", "random10", N, seed=0xC1, dtype="f64")
        g, rc, na, nr, _ = gpu("lorenz", "rodas5p", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-10,
                               reltol=1e-10)
        o, orc, ona, onr = oracle.solve("lorenz", "rodas5p", u0, p, (0.0, 1.0), 1e-3, dtype="f64", adaptive=True,
                                        abstol=1e-10, reltol=1e-10)
        np.testing.assert_array_equal(rc, orc)
        check_adaptive(g, o, (na, nr), (ona, onr), tol=1e-8)
