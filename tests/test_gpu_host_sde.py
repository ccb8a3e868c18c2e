"""ensemble_solve_host on the SDE solvers (-m gpu): chunked H2D / solve / D2H must
give the same bits as one device-resident ensemble_solve call — every chunk keys
its Philox counters on global trajectory indices (DESIGN R10) — and both match
the oracle within the north_star fixed-step tolerance."""
import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs
from tests.helpers import gpu, traj_relerr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("model,alg,dtype", [("lorenz_sde_add", "em", "f32"), ("crn", "em", "f64"),
                                             ("gbm", "siea", "f64")])
def test_solve_host_sde_matches_device(model, alg, dtype):
    import torch

    import paper_2304_06835_b200 as ens
    N, off = 5003, 4242
    recipe = "grid" if model == "crn" else "random10"
    kw = dict(N_total=10**6, index_offset=off) if model == "crn" else {}
    u0, p = make_inputs(model, recipe, N, seed=11, dtype=dtype, **kw)
    tf, dt = (10.0, 0.1) if model == "crn" else (1.0, 1e-2)
    sa = np.linspace(0.0, tf, 6)
    U = torch.from_numpy(u0).pin_memory()
    P = torch.from_numpy(p).pin_memory()
    uh, rch, _ = ens.solve_host(model, alg, U, P, (0.0, tf), dt, saveat=sa, n_chunks=7, seed=0xABC,
                                index_offset=off)
    g, rc, *_ = gpu(model, alg, u0, p, (0.0, tf), dt, saveat=sa, seed=0xABC, index_offset=off)
    np.testing.assert_array_equal(uh.numpy(), g)
    np.testing.assert_array_equal(rch.numpy(), rc)
    # a sample of trajectories from the last chunk against the oracle
    idx = np.arange(N - 300, N)
    o, orc, *_ = oracle.solve(model, alg, u0[:, idx], p[:, idx] if p.ndim == 2 else p, (0.0, tf), dt, dtype=dtype,
                              seed=0xABC, saveat=sa, gidx=off + idx)
    np.testing.assert_array_equal(rch.numpy()[idx], orc)
    ok = orc == 0
    tol = 1e-5 if dtype == "f32" else 1e-12
    assert traj_relerr(uh.numpy()[..., idx][..., ok], o[..., ok]).max() <= tol


def test_solve_host_sde_rejects_off_grid_saveat():
    """EM saves on grid points only (DESIGN R11); the host path checks before any copy."""
    import torch

    import paper_2304_06835_b200 as ens
    u0, p = make_inputs("gbm", "random10", 64, dtype="f64")
    with pytest.raises(ens.EnsError):
        ens.solve_host("gbm", "em", torch.from_numpy(u0), torch.from_numpy(p), (0.0, 1.0), 0.1, n_chunks=2,
                       saveat=[0.05])
