"""GPU ↔ oracle parity for Vern9 (GPUVern9; NEXT-1; DESIGN R21)
through the C ABI (-m gpu), same bars as Vern7."""
import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs
from tests.helpers import gpu, traj_relerr

pytestmark = pytest.mark.gpu

TOL_FIXED = {"f32": 1e-5, "f64": 1e-12}


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("model,tf,dt", [("lorenz", 1.0, 0.01), ("harmonic", 4.0, 0.1)])
def test_vern9_fixed_parity(model, tf, dt, dtype):
    N = 2051
    u0, p = make_inputs(model, "random10", N, seed=0x99, dtype=dtype)
    ns = int(round(tf / dt))
    sa = np.array([0.0, dt * (ns // 3), tf])
    g, rc, na, nr, _ = gpu(model, "vern9", u0, p, (0.0, tf), dt, saveat=sa)
    o, orc, ona, _ = oracle.solve(model, "vern9", u0, p, (0.0, tf), dt, dtype=dtype, saveat=sa)
    np.testing.assert_array_equal(rc, orc)
    np.testing.assert_array_equal(na, ona)
    assert traj_relerr(g, o).max() <= TOL_FIXED[dtype]
    assert (g == o).mean() >= 0.99


@pytest.mark.parametrize("refill", [False, True])
def test_vern9_adaptive_tight_tolerance(refill):
    N = 1029
    u0, p = make_inputs("lorenz", "random10", N, seed=0xC1, dtype="f64")
    sa = np.array([0.0, 0.3, 0.65, 1.0])
    g, rc, na, nr, _ = gpu("lorenz", "vern9", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-10, reltol=1e-10,
                           saveat=sa, refill=refill)
    o, orc, ona, onr = oracle.solve("lorenz", "vern9", u0, p, (0.0, 1.0), 1e-3, dtype="f64", adaptive=True,
                                    abstol=1e-10, reltol=1e-10, saveat=sa)
    np.testing.assert_array_equal(rc, orc)
    same = (na == ona) & (nr == onr)
    assert same.mean() >= 0.999, same.mean()
    assert traj_relerr(g[..., same], o[..., same]).max() <= 1e-8


def test_vern9_ragged_and_f32():
    u0, p = make_inputs("lorenz", "random10", 1, seed=2, dtype="f64")
    g, rc, na, nr, _ = gpu("lorenz", "vern9", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-9, reltol=1e-9)
    o, orc, ona, onr = oracle.solve("lorenz", "vern9", u0, p, (0.0, 1.0), 1e-3, dtype="f64", adaptive=True,
                                    abstol=1e-9, reltol=1e-9)
    assert traj_relerr(g, o).max() <= 1e-8
    u0, p = make_inputs("lorenz", "random10", 333, seed=6, dtype="f32")
    g, rc, na, *_ = gpu("lorenz", "vern9", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-5, reltol=1e-5)
    o, orc, ona, _ = oracle.solve("lorenz", "vern9", u0, p, (0.0, 1.0), 1e-3, dtype="f32", adaptive=True,
                                  abstol=1e-5, reltol=1e-5)
    same = na == ona
    assert same.mean() >= 0.99
    assert traj_relerr(g[..., same], o[..., same]).max() <= 1e-3
