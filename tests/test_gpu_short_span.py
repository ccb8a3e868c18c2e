"""Degenerate time spans (-m gpu): a span shorter than dt (fixed step: one step
of h_last = tf − t0, DESIGN R3; adaptive: the first step truncated to land on
tf, R5) and a span of exactly one dt, for every ODE algorithm, fp64 and fp32,
against the oracle through the C ABI."""
import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs
from tests.helpers import gpu, traj_relerr

pytestmark = pytest.mark.gpu

ALGS = ["tsit5", "vern7", "vern9", "rosenbrock23", "rodas4", "rodas5", "rodas5p"]


@pytest.mark.parametrize("alg", ALGS)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("span,dt", [(0.003, 0.01), (0.01, 0.01)])
def test_short_span(alg, dtype, span, dt):
    N = 97
    u0, p = make_inputs("lorenz", "random10", N, seed=7, dtype=dtype)
    tol = 1e-12 if dtype == "f64" else 1e-5
    for kw in [dict(), dict(adaptive=True, abstol=1e-8 if dtype == "f64" else 1e-5,
                            reltol=1e-8 if dtype == "f64" else 1e-5)]:
        g, rc, na, nr, _ = gpu("lorenz", alg, u0, p, (0.5, 0.5 + span), dt, **kw)
        o, orc, ona, onr = oracle.solve("lorenz", alg, u0, p, (0.5, 0.5 + span), dt, dtype=dtype, **kw)
        np.testing.assert_array_equal(rc, orc)
        np.testing.assert_array_equal(na, ona)
        np.testing.assert_array_equal(nr, onr)
        if not kw:
            assert (na == 1).all()
        assert traj_relerr(g, o).max() <= tol
