"""GPU ↔ oracle parity for event handling (bouncing ball; DESIGN R18)."""
import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs
from tests.helpers import check_adaptive, check_fixed, gpu, traj_relerr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-10), ("f32", 1e-6)])
@pytest.mark.parametrize("refill", [False, True])
def test_bouncing_ball_parity(dtype, tol, refill):
    N = 1000
    u0, p = make_inputs("ball", "random10", N, seed=21, dtype=dtype)
    sa = np.linspace(0.0, 15.0, 61)
    g, rc, na, nr, _ = gpu("ball", "tsit5", u0, p, (0.0, 15.0), 0.1, adaptive=True, abstol=tol, reltol=tol,
                           saveat=sa, refill=refill)
    o, orc, ona, onr = oracle.solve("ball", "tsit5", u0, p, (0.0, 15.0), 0.1, dtype=dtype, adaptive=True,
                                    abstol=tol, reltol=tol, saveat=sa)
    np.testing.assert_array_equal(rc, orc)
    check_adaptive(g, o, (na, nr), (ona, onr), tol=(1e-9 if dtype == "f64" else 1e-4))


def test_ball_requires_adaptive_tsit5():
    import torch

    import paper_2304_06835_b200 as ens
    u0, p = make_inputs("ball", "const", 4, dtype="f64")
    U, P = torch.from_numpy(u0).cuda(), torch.from_numpy(p).cuda()
    for alg, kw in [("tsit5", {}), ("rosenbrock23", dict(adaptive=True, abstol=1e-6))]:
        with pytest.raises(ens.EnsError) as e:
            ens.solve("ball", alg, U, P, (0.0, 1.0), 1e-2, **kw)
        assert e.value.status == 8
