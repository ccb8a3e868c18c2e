"""Group kernels (group.cuh: G lanes per trajectory for the Rodas methods on
HIRES / POLLU) against the one-thread-per-trajectory lane kernels the refill
scheduler runs: bit for bit, with saves (Rodas4's interpolant, the R24 dense
output of Rodas5 / Rodas5P), a lane that diverges at t0, a MaxIters cap and a
ragged ensemble; and against the oracle (-m gpu)."""
import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs
from tests.helpers import check_adaptive, gpu

pytestmark = pytest.mark.gpu

TF = {"hires": 321.8122, "pollu": 60.0}


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("alg", ["rodas4", "rodas5", "rodas5p"])
@pytest.mark.parametrize("model", ["hires", "pollu"])
def test_group_equals_lane_kernel(model, alg, dtype):
    if model == "pollu" and dtype == "f32":
        pytest.skip("POLLU: fp64 only")
    N = 677
    u0, p = make_inputs(model, "random10", N, seed=0x6A, dtype=dtype)
    u0[0, 5] = np.nan
    tf = TF[model]
    tol = 1e-8 if dtype == "f64" else 1e-4
    sa = np.array([0.0, 0.013 * tf, 0.25 * tf, 0.5 * tf, tf])
    for kw in [dict(saveat=sa), dict(), dict(max_steps=40)]:
        a = gpu(model, alg, u0, p, (0.0, tf), 1e-6, adaptive=True, abstol=tol, reltol=tol, **kw)
        b = gpu(model, alg, u0, p, (0.0, tf), 1e-6, adaptive=True, abstol=tol, reltol=tol, refill=True, **kw)
        for x, y in zip(a[:4], b[:4]):
            np.testing.assert_array_equal(x, y)
        assert a[1][5] == 3
        if "max_steps" in kw:
            assert (a[1][np.arange(N) != 5] == 1).all()


@pytest.mark.parametrize("alg", ["rodas4", "rodas5p"])
@pytest.mark.parametrize("model", ["hires", "pollu"])
def test_group_oracle_parity(model, alg):
    N = 130
    u0, p = make_inputs(model, "random10", N, seed=0x6B, dtype="f64")
    tf = TF[model]
    sa = np.array([0.0, 0.5 * tf, tf])
    kw = dict(adaptive=True, abstol=1e-8, reltol=1e-8, saveat=sa)
    g, rc, na, nr, _ = gpu(model, alg, u0, p, (0.0, tf), 1e-6, **kw)
    o, orc, ona, onr = oracle.solve(model, alg, u0, p, (0.0, tf), 1e-6, dtype="f64", **kw)
    np.testing.assert_array_equal(rc, orc)
    check_adaptive(g, o, (na, nr), (ona, onr), tol=1e-8, same_min=1.0)
