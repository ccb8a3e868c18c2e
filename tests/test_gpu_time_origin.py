"""Nonzero time origin and a non-integer step count (-m gpu): every ODE solver on
tspan = (2.5, 3.7) with dt = 0.07 (17 full steps + a shorter last step, DESIGN
R3) and save points inside, on and between grid points, against the oracle."""
import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs
from tests.helpers import check_adaptive, check_fixed, gpu, traj_relerr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("alg", ["tsit5", "vern7", "vern9", "rosenbrock23", "rodas4", "rodas5"])
@pytest.mark.parametrize("adaptive", [False, True])
def test_shifted_tspan(alg, adaptive):
    N = 300
    u0, p = make_inputs("lorenz", "random10", N, seed=17, dtype="f64")
    t0, tf, dt = 2.5, 3.7, 0.07
    grid_only = alg in ("vern7", "vern9", "rodas5") and not adaptive     # R21: fixed-step saves on the grid
    sa = np.array([t0, t0 + 5 * dt, t0 + 11 * dt, tf]) if grid_only else np.array([t0, 2.61, t0 + 5 * dt, 3.333, tf])
    kw = dict(adaptive=adaptive, abstol=1e-9, reltol=1e-9)
    g, rc, na, nr, _ = gpu("lorenz", alg, u0, p, (t0, tf), dt, saveat=sa, **kw)
    o, orc, ona, onr = oracle.solve("lorenz", alg, u0, p, (t0, tf), dt, dtype="f64", saveat=sa, **kw)
    np.testing.assert_array_equal(rc, orc)
    if not adaptive:
        assert (na == 18).all() and (ona == 18).all()
    check_adaptive(g, o, (na, nr), (ona, onr), tol=(1e-12 if not adaptive else 1e-8))
