"""Pins for the oracle's dense output of Vern7 / Vern9 / Rodas5 / Rodas5P
(DESIGN R24: a save point τ inside an accepted step [t, t + h] stores one step
of the same method from (t, u) of length τ − t; τ = t + h stores u_new).

The paper gives these methods "lazy" 7th / 9th-order interpolants
and Rodas5P a "fourth-order stiff-aware interpolation"; their extra
coefficients are not recoverable offline, so R24 keeps what those schemes are
for — saved values at the method's own order, computed only for steps that
contain a save point, with a step sequence that does not depend on saveat.
Pinned here against things other than the oracle's own code path:
  * the definition: a fixed-step save at an off-grid τ equals the fixed-step
    run that ends at τ (whose last step is the same shortened step);
  * the order: global errors at off-grid save points of the harmonic
    oscillator (closed form) fall like dt^p (p = 7, 9, 5, 5) — a lower-order
    interpolant (Hermite, linear) would show up as a smaller slope;
  * saveat-independence: with and without save points the adaptive solver
    takes the identical accepted / rejected steps and ends in the identical
    state (round 2 clipped steps onto save points, which changed both).
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest

import oracle

ALGS = {"vern7": 7, "vern9": 9, "rodas5": 5, "rodas5p": 5}
HARM = dict(u0=[[1.0], [0.0]], p=[[1.0]])
ROB = json.loads((Path(__file__).parent / "golden" / "robertson_reference.json").read_text())


def _exact(ts):
    ts = np.asarray(ts, np.float64)
    return np.stack([np.cos(ts), -np.sin(ts)], 1)   # u'' = −u, u(0) = 1, u'(0) = 0


@pytest.mark.parametrize("alg", list(ALGS))
def test_offgrid_save_is_the_shortened_step(alg):
    """Fixed dt = 0.1 on [0, 1]: τ = 0.537 lies inside step 5 (0.5 → 0.6); its
    saved value is the state of the fixed-step run on [0, 0.537] (five steps of
    0.1, then one of 0.037 — the same shortened step from (0.5, u_5))."""
    taus = [0.0, 0.237, 0.5, 0.537, 0.999, 1.0]
    out, rc, na, _ = oracle.solve("harmonic", alg, HARM["u0"], HARM["p"], (0.0, 1.0), 0.1, saveat=taus)
    assert rc[0] == 0 and na[0] == 10
    np.testing.assert_array_equal(out[0, :, 0], [1.0, 0.0])
    for j, tau in enumerate(taus[1:], 1):
        ref, rrc, *_ = oracle.solve("harmonic", alg, HARM["u0"], HARM["p"], (0.0, tau), 0.1)
        assert rrc[0] == 0
        np.testing.assert_allclose(out[j, :, 0], ref[0, :, 0], rtol=1e-14, atol=1e-15, err_msg=f"{alg} τ={tau}")
    fin, *_ = oracle.solve("harmonic", alg, HARM["u0"], HARM["p"], (0.0, 1.0), 0.1)
    np.testing.assert_array_equal(out[-1, :, 0], fin[0, :, 0])


@pytest.mark.parametrize("alg", list(ALGS))
def test_dense_output_order(alg):
    """Off-grid save points τ = (j + 0.37)·dt-ish over [0, 4]: the max error
    against the closed form falls like dt^p."""
    p = ALGS[alg]
    taus = np.array([0.137, 0.911, 1.553, 2.718, 3.333])
    hs = {7: [0.4, 0.2, 0.1], 9: [0.8, 0.4, 0.2], 5: [0.1, 0.05, 0.025]}[p]
    errs = []
    for h in hs:
        out, rc, *_ = oracle.solve("harmonic", alg, HARM["u0"], HARM["p"], (0.0, 4.0), h, saveat=taus)
        assert rc[0] == 0
        errs.append(np.abs(out[:, :, 0] - _exact(taus)).max())
    s = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all((s > p - 0.8) & (s < p + 1.2)), (alg, s, errs)


@pytest.mark.parametrize("alg", list(ALGS))
def test_step_sequence_independent_of_saveat(alg):
    """Adaptive runs with 37 interior save points and without any take the same
    steps: identical n_accept / n_reject, identical final state (stored at
    τ = tf), and every saved value within the tolerance of the closed form."""
    taus = np.linspace(0.0, 6.0, 39)
    kw = dict(adaptive=True, abstol=1e-10, reltol=1e-10)
    out, rc, na, nr = oracle.solve("harmonic", alg, HARM["u0"], HARM["p"], (0.0, 6.0), 0.01, saveat=taus, **kw)
    fin, frc, fna, fnr = oracle.solve("harmonic", alg, HARM["u0"], HARM["p"], (0.0, 6.0), 0.01, **kw)
    assert rc[0] == frc[0] == 0
    assert (na[0], nr[0]) == (fna[0], fnr[0]), (alg, na[0], nr[0], fna[0], fnr[0])
    np.testing.assert_array_equal(out[-1, :, 0], fin[0, :, 0])
    assert np.abs(out[:, :, 0] - _exact(taus)).max() < 1e-8


@pytest.mark.parametrize("alg", ["vern7", "vern9"])
def test_lorenz_saves_independent_and_accurate(alg):
    """Nonlinear check: Lorenz at tol 1e-10 with save points every 0.01 — the
    step counts equal the run without saves and the saved values agree with a
    fine fixed-step Tsit5 reference (itself pinned to order 5) to 1e-8."""
    u0, p = [[1.0], [0.0], [0.0]], [[10.0], [28.0], [8 / 3]]
    taus = np.round(np.arange(0, 101) * 0.01, 12)
    kw = dict(adaptive=True, abstol=1e-10, reltol=1e-10)
    out, rc, na, nr = oracle.solve("lorenz", alg, u0, p, (0.0, 1.0), 1e-3, saveat=taus, **kw)
    _, _, fna, fnr = oracle.solve("lorenz", alg, u0, p, (0.0, 1.0), 1e-3, **kw)
    assert rc[0] == 0 and (na[0], nr[0]) == (fna[0], fnr[0])
    ref, *_ = oracle.solve("lorenz", "tsit5", u0, p, (0.0, 1.0), 1e-5, saveat=taus)
    scale = np.abs(ref[:, :, 0]).max()
    assert np.abs(out[:, :, 0] - ref[:, :, 0]).max() / scale < 1e-8


def test_rodas5_stiff_dense_output():
    """Stiff (Robertson, tol 1e-8): dense saves keep the conservation law
    Σy = 1 and stay within the IVP-test-set tolerance of the reference values at
    τ = 40 (Hairer–Wanner) while the step counts match the run without saves."""
    u0, p = [[1.0], [0.0], [0.0]], [[0.04], [3e7], [1e4]]
    taus = np.array([0.0, 0.4, 4.0, 40.0, 400.0])
    kw = dict(adaptive=True, abstol=1e-8, reltol=1e-8)
    for alg in ["rodas5", "rodas5p"]:
        out, rc, na, nr = oracle.solve("robertson", alg, u0, p, (0.0, 400.0), 1e-4, saveat=taus, **kw)
        _, _, fna, fnr = oracle.solve("robertson", alg, u0, p, (0.0, 400.0), 1e-4, **kw)
        assert rc[0] == 0 and (na[0], nr[0]) == (fna[0], fnr[0])
        assert np.abs(out[:, :, 0].sum(1) - 1.0).max() < 1e-10
        y40 = np.array(ROB["t40"])   # Hairer–Wanner reference (tests/golden/robertson_reference.json)
        assert np.abs(out[3, :, 0] - y40).max() / np.abs(y40) .max() < 1e-6
        assert math.isfinite(out[1, 1, 0])


@pytest.mark.parametrize("alg", list(ALGS))
def test_tiny_and_end_offsets(alg):
    """A save point a hair after a grid point (τ − t_s = 1e-13) stores a step of
    that length — u_s to within 1e-12 — and one a hair before the next grid point
    agrees with u_{s+1} to the local error of the method (fixed dt = 0.1)."""
    taus = [0.5, 0.5 + 1e-13, 0.6 - 1e-13, 0.6]
    out, rc, *_ = oracle.solve("harmonic", alg, HARM["u0"], HARM["p"], (0.0, 1.0), 0.1, saveat=taus)
    assert rc[0] == 0
    np.testing.assert_allclose(out[1, :, 0], out[0, :, 0], rtol=0, atol=1e-12)
    np.testing.assert_allclose(out[2, :, 0], out[3, :, 0], rtol=0, atol=1e-11)
    assert np.abs(out[:, :, 0] - _exact(taus)).max() < 1e-6
