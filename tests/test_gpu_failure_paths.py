"""Failure paths of every ODE solver on the GPU against the oracle (-m gpu):
a NaN initial state (Diverged before any step), an overflowing trajectory,
the attempted-step cap (MaxIters), and isolation — the other trajectories of
the same launch are unaffected (DESIGN R6, R10)."""
import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs
from tests.helpers import gpu, traj_relerr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("alg", ["tsit5", "vern7", "vern9", "rosenbrock23", "rodas4", "rodas5"])
@pytest.mark.parametrize("adaptive", [False, True])
def test_retcodes_match_oracle(alg, adaptive):
    u0, p = make_inputs("lorenz", "random10", 300, seed=1, dtype="f64")
    u0[0, 7] = np.nan                 # f(u0) non-finite → Diverged, no step
    u0[1, 100] = 1e300                # overflow in the first step
    kw = dict(adaptive=adaptive, abstol=1e-8, reltol=1e-8)
    sa = [0.0, 0.5, 1.0]
    g, rc, na, nr, _ = gpu("lorenz", alg, u0, p, (0.0, 1.0), 1e-2, saveat=sa, **kw)
    o, orc, ona, onr = oracle.solve("lorenz", alg, u0, p, (0.0, 1.0), 1e-2, dtype="f64", saveat=sa, **kw)
    np.testing.assert_array_equal(rc, orc)
    assert rc[7] == 3 and rc[100] != 0
    assert (np.delete(rc, [7, 100]) == 0).all()
    np.testing.assert_array_equal(na[[7, 100]], ona[[7, 100]])
    ok = rc == 0
    assert traj_relerr(g[..., ok], o[..., ok]).max() <= (1e-12 if not adaptive else 1e-8)
    # failed trajectories: the state saved at t0 is u0, later save points unreached → NaN
    assert np.isnan(g[1:, :, 7]).all() and np.array_equal(g[0, 1:, 7], u0[1:, 7])


@pytest.mark.parametrize("alg", ["tsit5", "vern7", "vern9", "rosenbrock23", "rodas4", "rodas5"])
def test_max_steps(alg):
    u0, p = make_inputs("lorenz", "random10", 40, seed=2, dtype="f64")
    g, rc, na, nr, _ = gpu("lorenz", alg, u0, p, (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-10, reltol=1e-10,
                           max_steps=7)
    o, orc, ona, onr = oracle.solve("lorenz", alg, u0, p, (0.0, 1.0), 1e-3, dtype="f64", adaptive=True,
                                    abstol=1e-10, reltol=1e-10, max_steps=7)
    np.testing.assert_array_equal(rc, orc)
    assert (rc == 1).all() and ((na + nr) == 7).all()
    np.testing.assert_array_equal(na, ona)
    assert traj_relerr(g, o).max() <= 1e-12


@pytest.mark.parametrize("alg", ["tsit5", "rosenbrock23"])
def test_max_steps_above_int32(alg):
    """Attempts are counted as n_accept + n_reject (int32); a cap above INT32_MAX is
    clamped on the host and behaves as "no cap reached" — same results as the oracle
    with the 64-bit cap (step counters)."""
    u0, p = make_inputs("lorenz", "random10", 64, seed=3, dtype="f64")
    kw = dict(adaptive=True, abstol=1e-8, reltol=1e-8, max_steps=1 << 40)
    g, rc, na, nr, _ = gpu("lorenz", alg, u0, p, (0.0, 1.0), 1e-3, **kw)
    o, orc, ona, onr = oracle.solve("lorenz", alg, u0, p, (0.0, 1.0), 1e-3, dtype="f64", **kw)
    assert (rc == 0).all() and (orc == 0).all()
    np.testing.assert_array_equal(na, ona)
    np.testing.assert_array_equal(nr, onr)
    assert traj_relerr(g, o).max() <= 1e-8
