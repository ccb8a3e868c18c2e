"""The fp32 static adaptive Tsit5 kernel with component pairs on FFMA2 / FMUL2
(tsit5.cuh::tsit5_static_pair_kernel) for every pair layout —
n = 2 (one pair), n = 3 (a pair and a scalar tail), n = 8 (four pairs) — with and
without saves, including failing lanes (Diverged at t0, overflow, MaxIters):
bit for bit equal to the oracle and to the scalar lane kernel the refill
scheduler runs (-m gpu)."""
import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs
from tests.helpers import check_adaptive, gpu

pytestmark = pytest.mark.gpu

CASES = [("harmonic", (0.0, 4.0), 1e-5), ("lorenz", (0.0, 1.0), 1e-5), ("orego", (0.0, 1.0), 1e-4),
         ("hires", (0.0, 0.05), 1e-4)]


@pytest.mark.parametrize("save", [False, True])
@pytest.mark.parametrize("model,tspan,tol", CASES)
def test_pair_kernel_parity(model, tspan, tol, save):
    N = 1000
    u0, p = make_inputs(model, "random10", N, seed=0x2A, dtype="f32")
    u0[0, 3] = np.nan                         # Diverged before any step
    u0[:, 500] = 3e38                         # huge state: overflows (or not) identically on both sides
    sa = np.linspace(tspan[0], tspan[1], 9)[[0, 1, 3, 6, 8]] if save else None
    kw = dict(adaptive=True, abstol=tol, reltol=tol, saveat=sa, max_steps=20000)
    g, rc, na, nr, _ = gpu(model, "tsit5", u0, p, tspan, 1e-3, **kw)
    o, orc, ona, onr = oracle.solve(model, "tsit5", u0, p, tspan, 1e-3, dtype="f32", **kw)
    np.testing.assert_array_equal(rc, orc)
    assert rc[3] == 3
    check_adaptive(g, o, (na, nr), (ona, onr), tol=1e-5, same_min=1.0)
    gr, rcr, nar, nrr, _ = gpu(model, "tsit5", u0, p, tspan, 1e-3, refill=True, **kw)   # scalar lane kernel
    np.testing.assert_array_equal(rc, rcr)
    np.testing.assert_array_equal(na, nar)
    np.testing.assert_array_equal(nr, nrr)
    np.testing.assert_array_equal(g, gr)


def test_pair_kernel_max_steps():
    u0, p = make_inputs("lorenz", "random10", 257, seed=3, dtype="f32")
    kw = dict(adaptive=True, abstol=1e-6, reltol=1e-6, max_steps=9)
    g, rc, na, nr, _ = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, **kw)
    o, orc, ona, onr = oracle.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, dtype="f32", **kw)
    assert (rc == 1).all() and ((na + nr) == 9).all()
    np.testing.assert_array_equal(na, ona)
    np.testing.assert_array_equal(g, o)
