"""Full-size BASELINE configurations on the GPU (-m gpu): every config at the
size BASELINE.json quotes, inputs from the on-device generator, launched the
way bench.py / tools/bench_configs.py launch them; parity on sampled
trajectories the oracle computes one by one, plus properties that hold at any
size (retcodes, invariants, statistics against a plain reduction of the stored
states)."""
import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs
from tests.helpers import check_adaptive, check_fixed, sample_indices, traj_relerr

pytestmark = pytest.mark.gpu


def _take(x, idx):
    import torch
    return x[..., torch.from_numpy(idx).to(x.device)].cpu().numpy()


def _inputs_at(model, recipe, idx, N_total, **kw):
    """Host inputs of the trajectories `idx` of an N_total ensemble (each is a
    function of (seed, global index) only), without building all N_total."""
    parts = [make_inputs(model, recipe, 1, index_offset=int(i), N_total=N_total, **kw) for i in idx]
    return np.concatenate([a for a, _ in parts], 1), np.concatenate([b for _, b in parts], 1)


def test_c2_adaptive_full_size_sampled():
    """C2 adaptive: Lorenz ρ sweep fp32, N = 10^7, abstol = reltol = 1e-6."""
    import torch

    import paper_2304_06835_b200 as ens
    N = 10**7
    u0, p = ens.generate_inputs("lorenz", "rho_sweep", N, dtype=torch.float32, N_total=N)
    sol = ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-6, reltol=1e-6)
    assert (sol.retcode == 0).all().item()
    idx = sample_indices(N, head=512, tail=512, stride_count=1024)
    u0h, ph = _inputs_at("lorenz", "rho_sweep", idx, N, dtype="f32")
    o, orc, ona, onr = oracle.solve("lorenz", "tsit5", u0h, ph, (0.0, 1.0), 1e-3, dtype="f32",
                                    adaptive=True, abstol=1e-6, reltol=1e-6)
    ref, *_ = oracle.solve("lorenz", "tsit5", u0h.astype(np.float64), ph.astype(np.float64), (0.0, 1.0), 1e-3,
                           dtype="f64", adaptive=True, abstol=1e-12, reltol=1e-12)
    check_adaptive(_take(sol.u, idx)[None], o,
                   (_take(sol.n_accept, idx), _take(sol.n_reject, idx)), (ona, onr), tol=1e-4, tol_same=1e-5, ref=ref)


@pytest.mark.parametrize("alg", ["rosenbrock23", "rodas5", "rodas5p"])
def test_c3_full_size_sampled(alg):
    """C3: Robertson ±10 % rates, fp64, N = 10^6, tol 1e-8, h0 = 1e-4, 100 save
    points over [0, 1e5] (2.4 GB of states)."""
    import torch

    import paper_2304_06835_b200 as ens
    N = 10**6
    u0, p = ens.generate_inputs("robertson", "random10", N, dtype=torch.float64, seed=0xC3)
    sa = np.linspace(0.0, 1e5, 100)
    sol = ens.solve("robertson", alg, u0, p, (0.0, 1e5), 1e-4, adaptive=True, abstol=1e-8, reltol=1e-8, saveat=sa)
    assert (sol.retcode == 0).all().item()
    # Σy = 1 at every save point of every trajectory (exact-J Rosenbrock invariant)
    dev = (sol.u.sum(1) - 1).abs().max().item()
    assert dev <= 1e-12, dev
    idx = sample_indices(N, head=256, tail=256, stride_count=1024)
    u0h, ph = _inputs_at("robertson", "random10", idx, N, seed=0xC3, dtype="f64")
    o, orc, ona, onr = oracle.solve("robertson", alg, u0h, ph, (0.0, 1e5), 1e-4, dtype="f64",
                                    adaptive=True, abstol=1e-8, reltol=1e-8, saveat=sa)
    check_adaptive(_take(sol.u, idx), o,
                   (_take(sol.n_accept, idx), _take(sol.n_reject, idx)), (ona, onr), tol=1e-8)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_c4_full_size_stats_and_samples(dtype):
    """C4: stochastic Lorenz (additive), N = 10^6, EM dt = 1e-3, 11 save points:
    the fused per-block statistics equal a plain fp64 reduction of the stored
    states, and sampled paths equal the oracle's (same Philox stream)."""
    import torch

    import paper_2304_06835_b200 as ens
    N = 10**6
    T = torch.float32 if dtype == "f32" else torch.float64
    u0, p = ens.generate_inputs("lorenz_sde_add", "const", N, dtype=T)
    sa = np.linspace(0.0, 1.0, 11)
    sol = ens.solve("lorenz_sde_add", "em", u0, p, (0.0, 1.0), 1e-3, seed=0xC4, saveat=sa, stats=True)
    assert (sol.retcode == 0).all().item()
    st = sol.stats.cpu().numpy()
    x = sol.u.double()
    mean = x.mean(-1).cpu().numpy()
    var = x.var(-1, unbiased=True).cpu().numpy()
    np.testing.assert_array_equal(st[..., 0], N)
    np.testing.assert_allclose(st[..., 1], mean, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(st[..., 2] / (N - 1), var, rtol=1e-10, atol=1e-14)
    idx = sample_indices(N, head=128, tail=128, stride_count=256)
    u0h, ph = make_inputs("lorenz_sde_add", "const", N, dtype=dtype)
    o, *_ = oracle.solve("lorenz_sde_add", "em", u0h[:, idx], ph, (0.0, 1.0), 1e-3, dtype=dtype, p_broadcast=True,
                         seed=0xC4, saveat=sa, gidx=idx)
    check_fixed(_take(sol.u, idx), o, 1e-5 if dtype == "f32" else 1e-12)


def test_c5_single_gpu_full_size_sampled():
    """C5 on one GPU: Lorenz fp32 fixed dt = 1e-3, random ±10 % p, N = 10^8
    (the multi-GPU run shards exactly this ensemble)."""
    import torch

    import paper_2304_06835_b200 as ens
    N = 10**8
    u0, p = ens.generate_inputs("lorenz", "random10", N, dtype=torch.float32, seed=0xC5)
    sol = ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3)
    assert (sol.retcode == 0).all().item() and (sol.n_accept == 1000).all().item()
    idx = np.unique(np.concatenate([np.arange(64), N - 1 - np.arange(64),
                                    np.random.default_rng(5).choice(N, 384, replace=False)]))
    u0h, ph = _inputs_at("lorenz", "random10", idx, N, seed=0xC5, dtype="f32")
    o, *_ = oracle.solve("lorenz", "tsit5", u0h, ph, (0.0, 1.0), 1e-3, dtype="f32")
    check_fixed(_take(sol.u, idx)[None], o, 1e-5)
