"""Save paths of the fixed-step Tsit5 kernel (-m gpu): grid-only saves streamed
by bulk copies from shared memory (full blocks), the per-thread fallback
(ragged last block, odd leading dimension, misaligned host chunks), and
interpolated saves — all against the oracle, with a diverged trajectory inside
a full block (its rows must be NaN after t0)."""
import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs
from tests.helpers import check_fixed, gpu, traj_relerr

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-5, "f64": 1e-12}


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("N", [3000, 3001, 4096])
def test_grid_saves_bulk_and_fallback(dtype, N):
    u0, p = make_inputs("lorenz", "rho_sweep", N, dtype=dtype)
    u0[0, 700] = np.nan                       # diverged lane in a full block
    sa = np.concatenate([[0.0], np.arange(1, 101) * 1e-2])   # every 10th step of dt = 1e-3, incl. tf
    sa[-1] = 1.0
    g, rc, na, nr, _ = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, saveat=sa)
    o, orc, ona, _ = oracle.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, dtype=dtype, saveat=sa)
    np.testing.assert_array_equal(rc, orc)
    assert rc[700] == 3 and np.isnan(g[1:, :, 700]).all()
    ok = rc == 0
    check_fixed(g[..., ok], o[..., ok], TOL[dtype])


def test_grid_saves_every_step_and_host_chunks():
    import torch

    import paper_2304_06835_b200 as ens
    N = 5000
    u0, p = make_inputs("lorenz", "random10", N, seed=4, dtype="f32")
    sa = np.arange(0, 1001) * 1e-3
    sa[-1] = 1.0
    g, rc, *_ = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, saveat=sa)
    idx = np.array([0, 1, 511, 512, 2047, 4999])
    o, *_ = oracle.solve("lorenz", "tsit5", u0[:, idx], p[:, idx], (0.0, 1.0), 1e-3, dtype="f32", saveat=sa)
    assert traj_relerr(g[..., idx], o).max() <= 1e-5
    # host path: chunk starts at odd offsets (misaligned rows → per-thread stores)
    U = torch.from_numpy(u0).pin_memory(); P = torch.from_numpy(p).pin_memory()
    uh, rch, _ = ens.solve_host("lorenz", "tsit5", U, P, (0.0, 1.0), 1e-3, saveat=sa, n_chunks=7)
    np.testing.assert_array_equal(uh.numpy(), g)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_interpolated_saves(dtype):
    N = 2600
    u0, p = make_inputs("lorenz", "random10", N, seed=9, dtype=dtype)
    sa = np.array([0.0, 0.0005, 0.12345, 0.5, 0.77777, 1.0])
    g, rc, *_ = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, saveat=sa)
    o, orc, *_ = oracle.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, dtype=dtype, saveat=sa)
    np.testing.assert_array_equal(rc, orc)
    assert traj_relerr(g, o).max() <= TOL[dtype]


def test_bulk_save_path():
    """The cp.async.bulk save path (off by default, ens_options.bulk_saves = 1):
    grid saves equal the default path bit for bit, with a diverged lane in a full block."""
    import torch

    import paper_2304_06835_b200 as ens
    for dt, name in [(torch.float32, "f32"), (torch.float64, "f64")]:
        u0, p = make_inputs("lorenz", "rho_sweep", 3001, dtype=name)
        u0[0, 700] = np.nan
        sa = np.concatenate([[0.0], np.arange(1, 101) * 1e-2]); sa[-1] = 1.0
        U, P = torch.from_numpy(u0).cuda(), torch.from_numpy(p).cuda()
        a = ens.solve("lorenz", "tsit5", U, P, (0.0, 1.0), 1e-3, saveat=sa).u.cpu().numpy()
        b = ens.solve("lorenz", "tsit5", U, P, (0.0, 1.0), 1e-3, saveat=sa, bulk_saves=True).u.cpu().numpy()
        np.testing.assert_array_equal(a, b)
