"""GPU ↔ oracle parity through the C ABI (-m gpu).

Tolerances (BASELINE.json north_star): fixed step rel ≤ 1e-12 (fp64), ≤ 1e-5
(fp32); adaptive fp64 at abstol=reltol=1e-10: final-state rel ≤ 1e-8 and
identical accepted-step counts on ≥ 99.9 % of trajectories; Philox words
bit-exact. Relative error is per trajectory, ∞-norm-wise (helpers.traj_relerr).
Sizes span several 256-thread blocks plus a ragged tail.
"""
import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs
from tests.helpers import check_adaptive, check_fixed, gpu, sample_indices, traj_relerr

pytestmark = pytest.mark.gpu

TOL_FIXED = {"f32": 1e-5, "f64": 1e-12}


# ------------------------------------------------------------ Tsit5 fixed --
@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("recipe", ["rho_sweep", "random10"])
def test_tsit5_fixed_lorenz(dtype, recipe):
    """C2 shape: Lorenz, dt=1e-3 on [0,1] → 1000 steps."""
    N = 4099
    u0, p = make_inputs("lorenz", recipe, N, seed=0xC2, dtype=dtype)
    g, rc, na, nr, _ = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3)
    o, orc, ona, _ = oracle.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, dtype=dtype)
    assert (rc == 0).all() and (orc == 0).all()
    assert (na == 1000).all() and (ona == 1000).all() and (nr == 0).all()
    # canonical operation order on both sides → expected bit-exact
    check_fixed(g, o, TOL_FIXED[dtype])


@pytest.mark.parametrize("model,u0v,pv", [("expdecay", [1.0], [1.3]), ("harmonic", [1.0, 0.0], [2.25])])
@pytest.mark.parametrize("alg", ["tsit5", "rosenbrock23"])
def test_fixed_closed_form_models(model, u0v, pv, alg):
    N = 300
    u0 = np.tile(np.array(u0v)[:, None], (1, N))
    p = np.tile(np.array(pv)[:, None], (1, N)) * np.linspace(0.5, 2.0, N)[None, :]
    sa = [0.0, 0.1234, 0.5, 0.9]
    for dtype in ["f32", "f64"]:
        uu, pp = u0.astype(np.float32 if dtype == "f32" else np.float64), p.astype(
            np.float32 if dtype == "f32" else np.float64)
        g, rc, na, _, _ = gpu(model, alg, uu, pp, (0.0, 1.0), 0.05, saveat=sa)
        o, orc, ona, _ = oracle.solve(model, alg, uu, pp, (0.0, 1.0), 0.05, dtype=dtype, saveat=sa)
        assert (rc == orc).all() and (na == ona).all()
        assert traj_relerr(g, o).max() <= TOL_FIXED[dtype]


def test_tsit5_fixed_saveat_every_step_window():
    """Dense saveat (every 10th step + off-grid points) through the interpolant, fp32 and fp64."""
    N = 1000
    sa = np.concatenate([np.arange(0, 1.0 + 1e-12, 0.01), [0.12345, 0.5555]])
    sa = np.unique(np.clip(sa, 0, 1))
    for dtype in ["f32", "f64"]:
        u0, p = make_inputs("lorenz", "random10", N, seed=5, dtype=dtype)
        g, rc, *_ = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, saveat=sa)
        o, orc, *_ = oracle.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, dtype=dtype, saveat=sa)
        assert traj_relerr(g, o).max() <= TOL_FIXED[dtype]


# --------------------------------------------------------- Tsit5 adaptive --
@pytest.mark.parametrize("tol", [1e-10, 1e-8])
@pytest.mark.parametrize("refill", [False, True])
def test_tsit5_adaptive_lorenz_f64(tol, refill):
    """C1 (N=1024, random p ±10 %, fp64) at 1e-8 and the parity tolerance 1e-10."""
    N = 1024
    u0, p = make_inputs("lorenz", "random10", N, seed=0xC1, dtype="f64")
    g, rc, na, nr, _ = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=tol, reltol=tol,
                           refill=refill)
    o, orc, ona, onr = oracle.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, dtype="f64", adaptive=True,
                                    abstol=tol, reltol=tol)
    assert (rc == 0).all() and (orc == 0).all()
    check_adaptive(g, o, (na, nr), (ona, onr), tol=1e-8)


def test_tsit5_adaptive_saveat_f64():
    N = 700
    u0, p = make_inputs("lorenz", "random10", N, seed=0xC1, dtype="f64")
    sa = np.linspace(0.0, 1.0, 11)
    g, rc, na, nr, _ = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-10, reltol=1e-10,
                           saveat=sa)
    o, orc, ona, onr = oracle.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, dtype="f64", adaptive=True,
                                    abstol=1e-10, reltol=1e-10, saveat=sa)
    check_adaptive(g, o, (na, nr), (ona, onr), tol=1e-8)
    np.testing.assert_array_equal(g[0], u0)     # τ = t0 saves u0


def fp64_reference(model, alg, u0, p, tspan, dt, tol=1e-12, **kw):
    """Tight fp64 oracle solution of fp32 inputs (accuracy reference for fp32 adaptive parity)."""
    ref, *_ = oracle.solve(model, alg, u0.astype(np.float64), p.astype(np.float64), tspan, dt, dtype="f64",
                           adaptive=True, abstol=tol, reltol=tol, **kw)
    return ref


def test_tsit5_adaptive_f32_sweep():
    """C2 adaptive (fp32, abstol=reltol=1e-6, ρ sweep): identical step counts on
    ≥ 99.9 % (same controller arithmetic, DESIGN R2), rounding-level agreement
    where they match, and every trajectory within 1e-4 (≈ 2× the fp32 solutions'
    own global error against an fp64 1e-12 reference, 5e-5 at this size)."""
    N = 4099
    u0, p = make_inputs("lorenz", "rho_sweep", N, dtype="f32")
    g, rc, na, nr, _ = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-6, reltol=1e-6)
    o, orc, ona, onr = oracle.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, dtype="f32", adaptive=True,
                                    abstol=1e-6, reltol=1e-6)
    assert (rc == orc).all()
    ref = fp64_reference("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3)
    check_adaptive(g, o, (na, nr), (ona, onr), tol=1e-4, tol_same=1e-5, ref=ref)


def test_refill_is_bitwise_static():
    """a8: the warp refill scheduler changes only which lane runs a trajectory."""
    N = 3000
    u0, p = make_inputs("lorenz", "random10", N, seed=11, dtype="f32")
    a = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-6, reltol=1e-6, refill=False)
    b = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-6, reltol=1e-6, refill=True)
    for x, y in zip(a[:4], b[:4]):
        np.testing.assert_array_equal(x, y)
    u0, p = make_inputs("robertson", "random10", 600, seed=3, dtype="f64")
    a = gpu("robertson", "rosenbrock23", u0, p, (0.0, 1e5), 1e-4, adaptive=True, abstol=1e-8, reltol=1e-8,
            refill=False)
    b = gpu("robertson", "rosenbrock23", u0, p, (0.0, 1e5), 1e-4, adaptive=True, abstol=1e-8, reltol=1e-8,
            refill=True)
    for x, y in zip(a[:4], b[:4]):
        np.testing.assert_array_equal(x, y)


# ------------------------------------------------------------ Rosenbrock23 --
@pytest.mark.parametrize("refill", [False, True])
def test_ros23_robertson_c3_shape(refill):
    """C3 shape: Robertson, ±10 % rates, fp64, tol 1e-8, h0=1e-4, saveat 100 points."""
    N = 1030
    u0, p = make_inputs("robertson", "random10", N, seed=0xC3, dtype="f64")
    sa = np.linspace(0.0, 1e5, 100)
    g, rc, na, nr, _ = gpu("robertson", "rosenbrock23", u0, p, (0.0, 1e5), 1e-4, adaptive=True, abstol=1e-8,
                           reltol=1e-8, saveat=sa, refill=refill)
    o, orc, ona, onr = oracle.solve("robertson", "rosenbrock23", u0, p, (0.0, 1e5), 1e-4, dtype="f64",
                                    adaptive=True, abstol=1e-8, reltol=1e-8, saveat=sa)
    assert (rc == 0).all() and (orc == 0).all()
    check_adaptive(g, o, (na, nr), (ona, onr), tol=1e-8)
    assert np.abs(g.sum(1) - 1).max() <= 1e-12     # Σy = 1 (linear invariant)


def test_ros23_adaptive_lorenz_f32():
    N = 513
    u0, p = make_inputs("lorenz", "random10", N, seed=9, dtype="f32")
    g, rc, na, nr, _ = gpu("lorenz", "rosenbrock23", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-5,
                           reltol=1e-5)
    o, orc, ona, onr = oracle.solve("lorenz", "rosenbrock23", u0, p, (0.0, 1.0), 1e-3, dtype="f32", adaptive=True,
                                    abstol=1e-5, reltol=1e-5)
    ref = fp64_reference("lorenz", "rosenbrock23", u0, p, (0.0, 1.0), 1e-3, tol=1e-11)
    check_adaptive(g, o, (na, nr), (ona, onr), tol=1e-2, tol_same=1e-5,
                   ref=ref)


# ------------------------------------------------------------------ EM / SDE --
@pytest.mark.parametrize("model", ["lorenz_sde_add", "lorenz_sde_mul", "gbm"])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_em_parity_and_stats(model, dtype):
    """C4 shape: shared p, dt=1e-3, 11 save points, ensemble mean/var."""
    N = 1000
    u0, p = make_inputs(model, "const", N, dtype=dtype)
    sa = np.linspace(0.0, 1.0, 11)
    g, rc, na, _, st = gpu(model, "em", u0, p, (0.0, 1.0), 1e-3, seed=0xC4, saveat=sa, stats=True)
    o, orc, ona, _ = oracle.solve(model, "em", u0, p, (0.0, 1.0), 1e-3, dtype=dtype, p_broadcast=True,
                                  seed=0xC4, saveat=sa)
    assert (rc == orc).all() and (na == 1000).all()
    # fixed-step tolerance of the north star; the normals are specified to the bit (R8)
    check_fixed(g, o, TOL_FIXED[dtype])
    # fused statistics = definition applied to the GPU's own states (exact-arithmetic bound)
    mean, var, cnt = oracle.stats(g)
    np.testing.assert_allclose(st[..., 1], mean, rtol=1e-13, atol=1e-300)
    np.testing.assert_allclose(st[..., 2] / (st[..., 0] - 1), var, rtol=1e-12, atol=1e-300)
    assert (st[..., 0] == N).all()


def test_em_stats_only_no_states():
    N = 5000
    u0, p = make_inputs("gbm", "const", N, dtype="f64")
    _, rc, na, _, st = gpu("gbm", "em", u0, p, (0.0, 1.0), 1e-3, seed=1, stats=True, store_states=False)
    g, *_ = gpu("gbm", "em", u0, p, (0.0, 1.0), 1e-3, seed=1)
    mean, var, _ = oracle.stats(g)
    np.testing.assert_allclose(st[0, :, 1], mean[0], rtol=1e-13)
    np.testing.assert_allclose(st[0, :, 2] / (N - 1), var[0], rtol=1e-12)
    # exact discrete EM moments (tests/test_oracle_pins): E_h = X0(1+rh)^N
    E_h = 0.1 * (1 + 1.5e-3) ** 1000
    se = np.sqrt(var[0] / N)
    assert np.all(np.abs(mean[0] - E_h) < 5 * se)


def test_philox_words_bitexact():
    import torch

    import paper_2304_06835_b200 as ens
    import json
    from pathlib import Path
    kat = json.loads((Path(__file__).parent / "golden" / "philox_kat.json").read_text())["vectors"]
    ctr = np.array([[int(x, 16) for x in v["ctr"]] for v in kat], dtype=np.uint32)
    key = np.array([[int(x, 16) for x in v["key"]] for v in kat], dtype=np.uint32)
    out = ens.philox4x32_10(torch.from_numpy(ctr.view(np.int32)).cuda(), torch.from_numpy(key.view(np.int32)).cuda())
    got = out.cpu().numpy().view(np.uint32)
    want = np.array([[int(x, 16) for x in v["out"]] for v in kat], dtype=np.uint32)
    np.testing.assert_array_equal(got, want)
    # the EM noise stream: words and normals bit-exact (DESIGN R8)
    N, S = 70, 5
    for dt, npd in [(torch.float32, np.float32), (torch.float64, np.float64)]:
        words, z = ens.sde_noise(N, S, seed=0xDEADBEEF12345, dtype=dt, step0=17, index_offset=1 << 33)
        words = words.cpu().numpy().view(np.uint32); z = z.cpu().numpy()
        per = 4 if dt == torch.float32 else 2
        c0 = 3 * 17 // per                          # the stream's calls covering steps 17..21 (R8)
        assert words.shape[0] == -(-(3 * (17 + S)) // per) - c0
        for i in [0, 1, 33, 69]:
            g = (1 << 33) + i
            for c in range(words.shape[0]):
                cc = c0 + c
                ref = oracle.philox([cc & 0xFFFFFFFF, g & 0xFFFFFFFF, g >> 32, cc >> 32],
                                    [0xDEADBEEF12345 & 0xFFFFFFFF, 0xDEADBEEF12345 >> 32])
                np.testing.assert_array_equal(words[c, :, i], ref)
            zr = oracle.normals(0xDEADBEEF12345, g, 17, S, "f32" if dt == torch.float32 else "f64")
            np.testing.assert_array_equal(z[:, :, i], zr.astype(npd))


# ------------------------------------------------------------------ inputs --
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_generate_inputs_bitwise(dtype):
    import torch

    import paper_2304_06835_b200 as ens
    tdt = torch.float32 if dtype == "f32" else torch.float64
    for model, recipe, kw in [("lorenz", "random10", dict(seed=0xC5, index_offset=12345)),
                              ("robertson", "random10", dict(seed=0xC3)),
                              ("lorenz", "rho_sweep", dict(index_offset=1000, N_total=10**7)),
                              ("lorenz", "random10", dict(seed=7, chunk_len=64, chunk_stride=256, index_offset=64))]:
        N = 1777
        u0g, pg = ens.generate_inputs(model, recipe, N, dtype=tdt, **kw)
        u0h, ph = make_inputs(model, recipe, N, dtype=dtype, **kw)
        np.testing.assert_array_equal(u0g.cpu().numpy(), u0h)
        np.testing.assert_array_equal(pg.cpu().numpy(), ph)


# ----------------------------------------------------------- failure paths --
def test_retcodes_and_isolation():
    u0, p = make_inputs("lorenz", "random10", 300, seed=1, dtype="f64")
    u0[0, 7] = np.nan
    u0[1, 100] = 1e300      # overflows in the first step → non-finite q → rejects → DtLessThanMin
    for adaptive in [False, True]:
        g, rc, na, nr, _ = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, adaptive=adaptive, abstol=1e-8,
                               reltol=1e-8)
        o, orc, ona, onr = oracle.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, dtype="f64", adaptive=adaptive,
                                        abstol=1e-8, reltol=1e-8)
        np.testing.assert_array_equal(rc, orc)
        assert rc[7] == 3 and rc[100] != 0 and (np.delete(rc, [7, 100]) == 0).all()
        ok = rc == 0
        assert traj_relerr(g[..., ok], o[..., ok]).max() <= 1e-8
    g, rc, na, nr, _ = gpu("lorenz", "tsit5", u0[:, :5], p[:, :5], (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-8,
                           reltol=1e-8, max_steps=20)
    assert (rc[[0, 1, 2, 3, 4]] == 1).all() and ((na + nr) == 20).all()


@pytest.mark.parametrize("N", [1, 2, 3, 513, 1025])
def test_paired_fp32_kernels_ragged(N):
    """The fp32 fixed-step kernel carries two trajectories per thread (FFMA2 pairs):
    odd N leaves a dead partner lane and a diverged lane sits next to a live
    partner; results must equal the oracle."""
    u0, p = make_inputs("lorenz", "random10", N, seed=N + 7, dtype="f32")
    u0[0, N // 2] = np.nan                         # a diverged lane next to a live partner
    g, rc, na, nr, _ = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3)
    o, orc, ona, onr = oracle.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, dtype="f32")
    np.testing.assert_array_equal(rc, orc)
    np.testing.assert_array_equal(na, ona)
    ok = rc == 0
    if ok.any():
        assert traj_relerr(g[..., ok], o[..., ok]).max() <= TOL_FIXED["f32"]
    np.testing.assert_array_equal(g[..., ~ok], o[..., ~ok])     # diverged lane keeps u0


@pytest.mark.parametrize("saves,stats", [(False, False), (True, False), (False, True), (True, True)])
def test_fp32_pair_lane_diverged_at_t0_even_index(saves, stats):
    """Finite u0 with a non-finite f(u0) (σ·(y2 − y1) overflows in fp32) at an EVEN
    index, the first lane of an FFMA2 pair: Diverged with no step, the stored final
    state is u0 (saves after t0 are NaN), and the fused statistics count u0 for it
    (R6) — the partner lane's integration must not overwrite it."""
    N = 130
    u0, p = make_inputs("lorenz", "random10", N, seed=3, dtype="f32")
    for i in (0, 64, 128):
        u0[:, i] = (3e38, -3e38, 0.0)
    sa = [0.0, 0.25, 1.0] if saves else None
    g, rc, na, nr, st = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, saveat=sa, stats=stats)
    o, orc, ona, onr = oracle.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, dtype="f32", saveat=sa)
    np.testing.assert_array_equal(rc, orc)
    assert (rc[[0, 64, 128]] == 3).all() and (na[[0, 64, 128]] == 0).all()
    np.testing.assert_array_equal(na, ona)
    bad = np.zeros(N, bool); bad[[0, 64, 128]] = True
    np.testing.assert_array_equal(g[..., bad], o[..., bad])      # u0 / NaN saves, bit for bit
    check_fixed(g[..., ~bad], o[..., ~bad], TOL_FIXED["f32"])
    if stats:
        mean, var, cnt = oracle.stats(g)
        np.testing.assert_allclose(st[..., 1], mean, rtol=1e-12)
        np.testing.assert_allclose(st[..., 2] / (st[..., 0] - 1), var, rtol=1e-10)


@pytest.mark.parametrize("N", [1, 31, 32, 33, 255, 257])
def test_small_and_ragged_sizes(N):
    u0, p = make_inputs("lorenz", "random10", N, seed=N, dtype="f64")
    for kw in [dict(), dict(adaptive=True, abstol=1e-8, reltol=1e-8), dict(adaptive=True, abstol=1e-8, reltol=1e-8,
                                                                         refill=True)]:
        g, rc, na, *_ = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, **kw)
        o, orc, ona, _ = oracle.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, dtype="f64",
                                      **{k: v for k, v in kw.items() if k != "refill"})
        assert traj_relerr(g, o).max() <= 1e-8 and (na == ona).all()


def test_validation_errors_on_device():
    import torch

    import paper_2304_06835_b200 as ens
    u0, p = make_inputs("lorenz", "random10", 64, dtype="f32")
    U, P = torch.from_numpy(u0).cuda(), torch.from_numpy(p).cuda()
    cases = [(dict(model="lorenz", alg="em"), 2), (dict(model="lorenz", alg="tsit5", tspan=(1.0, 0.0)), 5),
             (dict(model="lorenz", alg="tsit5", adaptive=True, abstol=0.0), 4),
             (dict(model="lorenz", alg="tsit5", saveat=[0.5, 0.2]), 6)]
    for kw, status in cases:
        kw = dict(kw)
        model, alg = kw.pop("model"), kw.pop("alg")
        tspan = kw.pop("tspan", (0.0, 1.0))
        with pytest.raises(ens.EnsError) as e:
            ens.solve(model, alg, U, P, tspan, 1e-3, **kw)
        assert e.value.status == status


# ------------------------------------------------ full size, sampled parity --
def test_full_size_sampled_parity_bench_config():
    """BASELINE configs[1] headline point at full size in bench.py's launch
    configuration: Lorenz Tsit5 fixed dt=1e-3, fp32, N=10^7 ρ sweep, inputs from
    the on-device generator; sampled trajectories vs the oracle one by one."""
    import torch

    import paper_2304_06835_b200 as ens
    N = 10**7
    u0, p = ens.generate_inputs("lorenz", "rho_sweep", N, dtype=torch.float32, N_total=N)
    sol = ens.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3)
    idx = sample_indices(N, head=1024, tail=1024, stride_count=2048)
    g = sol.u[:, torch.from_numpy(idx).cuda()].cpu().numpy()[None]
    assert (sol.retcode == 0).all().item() and (sol.n_accept == 1000).all().item()
    u0h, ph = make_inputs("lorenz", "rho_sweep", N, dtype="f32")
    o, *_ = oracle.solve("lorenz", "tsit5", u0h[:, idx], ph[:, idx], (0.0, 1.0), 1e-3, dtype="f32")
    check_fixed(g, o, 1e-5)
    assert np.isfinite(sol.u.cpu().numpy()).all()


def test_solve_host_matches_device():
    import torch

    import paper_2304_06835_b200 as ens
    N = 10007
    u0, p = make_inputs("lorenz", "random10", N, seed=4, dtype="f32")
    U = torch.from_numpy(u0).pin_memory(); P = torch.from_numpy(p).pin_memory()
    uh, rch, _ = ens.solve_host("lorenz", "tsit5", U, P, (0.0, 1.0), 1e-3, n_chunks=5)
    g, rc, *_ = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3)
    np.testing.assert_array_equal(uh.numpy(), g[0])
    np.testing.assert_array_equal(rch.numpy(), rc)
    uh, rch, _ = ens.solve_host("lorenz", "tsit5", U, P, (0.0, 1.0), 1e-3, n_chunks=3, adaptive=True, abstol=1e-6,
                                reltol=1e-6, refill=True)
    g, rc, *_ = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-6, reltol=1e-6)
    np.testing.assert_array_equal(uh.numpy(), g[0])


@pytest.mark.parametrize("n_chunks", [8, 16])
def test_solve_host_ramped_chunks_match_device(n_chunks):
    """Large N: ramped chunk sizes (1, 2, 4, 8, …, 8, 4, 2, 1) on two compute streams, fixed and
    adaptive (static), fp32 and an SDE (index offsets per chunk key the Philox stream)."""
    import torch

    import paper_2304_06835_b200 as ens
    N = 140_001
    u0, p = make_inputs("lorenz", "random10", N, seed=5, dtype="f32")
    U = torch.from_numpy(u0).pin_memory(); P = torch.from_numpy(p).pin_memory()
    for kw in [{}, dict(adaptive=True, abstol=1e-6, reltol=1e-6)]:
        uh, rch, _ = ens.solve_host("lorenz", "tsit5", U, P, (0.0, 1.0), 1e-3, n_chunks=n_chunks, **kw)
        g, rc, *_ = gpu("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-3, **kw)
        np.testing.assert_array_equal(uh.numpy(), g[0])
        np.testing.assert_array_equal(rch.numpy(), rc)
    us, ps = make_inputs("lorenz_sde_add", "const", N, dtype="f32")
    Us = torch.from_numpy(us).pin_memory(); Ps = torch.from_numpy(ps).pin_memory()
    uh, rch, _ = ens.solve_host("lorenz_sde_add", "em", Us, Ps, (0.0, 0.1), 1e-3, n_chunks=n_chunks, seed=0xC4)
    g, rc, *_ = gpu("lorenz_sde_add", "em", us, ps, (0.0, 0.1), 1e-3, seed=0xC4)
    np.testing.assert_array_equal(uh.numpy(), g[0])


# ------------------------------------------------------------ CRN (NEXT-3) --
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_crn_em_parity_and_stats(dtype):
    """σ-factor CRN SDE: 4 states, 8 Wiener processes (non-diagonal
    noise), grid parameters over Table 5 (10^6-point grid, a 1500-trajectory
    window of it), dt = 0.1 as in P:725 over [0, 100], saveat every 10."""
    N, off = 1500, 123456
    u0, p = make_inputs("crn", "grid", N, dtype=dtype, N_total=10**6, index_offset=off)
    sa = np.linspace(0.0, 100.0, 11)
    g, rc, na, _, st = gpu("crn", "em", u0, p, (0.0, 100.0), 0.1, seed=0x5EED, saveat=sa, stats=True,
                           index_offset=off)
    o, orc, ona, _ = oracle.solve("crn", "em", u0, p, (0.0, 100.0), 0.1, dtype=dtype, seed=0x5EED, saveat=sa,
                                  gidx=np.arange(off, off + N))
    np.testing.assert_array_equal(rc, orc)
    assert (na == 1000).all()
    ok = rc == 0
    assert ok.mean() > 0.99
    assert traj_relerr(g[..., ok], o[..., ok]).max() <= TOL_FIXED[dtype]
    mean, var, _ = oracle.stats(g)
    np.testing.assert_allclose(st[..., 1], mean, rtol=1e-12, atol=1e-300)


def test_crn_inputs_and_noise_bitwise():
    import torch

    import paper_2304_06835_b200 as ens
    for dt, name in [(torch.float32, "f32"), (torch.float64, "f64")]:
        u0g, pg = ens.generate_inputs("crn", "grid", 3000, dtype=dt, N_total=10**6, index_offset=777)
        u0h, ph = make_inputs("crn", "grid", 3000, dtype=name, N_total=10**6, index_offset=777)
        np.testing.assert_array_equal(u0g.cpu().numpy(), u0h)
        np.testing.assert_array_equal(pg.cpu().numpy(), ph)
        w, z = ens.sde_noise(40, 3, seed=99, dtype=dt, step0=5, index_offset=1000, nw=8)
        z = z.cpu().numpy()
        for i in [0, 17, 39]:
            zr = oracle.normals(99, 1000 + i, 5, 3, name, nw=8)
            np.testing.assert_array_equal(z[:, :, i], zr)
