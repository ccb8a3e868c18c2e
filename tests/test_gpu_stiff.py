"""GPU ↔ oracle parity for the stiff test suite on Rosenbrock23 with
the in-kernel forward-mode AD Jacobian (DESIGN R15). The paper runs 8192
trajectories; the oracle side here solves a window of them."""
import numpy as np
import pytest

import oracle
from synth.inputs import make_inputs
from tests.helpers import check_adaptive, check_fixed, gpu, traj_relerr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("model,tf,N", [("orego", 30.0, 300), ("hires", 321.8122, 500), ("pollu", 60.0, 300)])
def test_stiff_suite_parity(model, tf, N):
    u0, p = make_inputs(model, "random10", N, seed=0x57, dtype="f64")
    sa = np.linspace(0.0, tf, 7)
    g, rc, na, nr, _ = gpu(model, "rosenbrock23", u0, p, (0.0, tf), 1e-6, adaptive=True, abstol=1e-8, reltol=1e-8,
                           saveat=sa)
    o, orc, ona, onr = oracle.solve(model, "rosenbrock23", u0, p, (0.0, tf), 1e-6, dtype="f64", adaptive=True,
                                    abstol=1e-8, reltol=1e-8, saveat=sa)
    np.testing.assert_array_equal(rc, orc)
    assert (rc == 0).mean() > 0.99
    check_adaptive(g, o, (na, nr), (ona, onr), tol=1e-8)
    if model == "hires":
        assert np.abs(g[:, 6] + g[:, 7] - u0[7][None, :]).max() < 1e-15


def test_stiff_suite_literature_reference_on_gpu():
    """GPU HIRES / POLLU (test-set y9(0) = 0.01) / OREGO against the IVP test-set references."""
    import json
    from pathlib import Path
    ref = json.loads((Path(__file__).parent / "golden" / "stiff_references.json").read_text())
    for model, tol, bound in [("hires", 1e-10, 2e-6), ("pollu", 1e-10, 1e-6), ("orego", 1e-8, 1e-4)]:
        u0, p = make_inputs(model, "const", 32, dtype="f64")
        if model == "pollu":
            u0[8, :] = ref["pollu"]["y9_0"]
        g, rc, *_ = gpu(model, "rosenbrock23", u0, p, (0.0, ref[model]["tf"]), 1e-6, adaptive=True, abstol=tol,
                        reltol=tol)
        assert (rc == 0).all()
        r = np.array(ref[model]["y"])
        big = np.abs(r) > 1e-10
        rel = np.abs(g[0][:, 0] - r)[big] / np.abs(r[big])
        assert rel.max() < bound, (model, rel.max())


def test_pollu_fp32_and_tsit5_unsupported():
    import paper_2304_06835_b200 as ens
    import torch
    u0, p = make_inputs("pollu", "const", 8, dtype="f64")
    U, P = torch.from_numpy(u0).cuda(), torch.from_numpy(p).cuda()
    with pytest.raises(ens.EnsError) as e:
        ens.solve("pollu", "tsit5", U, P, (0.0, 1.0), 1e-3)
    assert e.value.status == 8
    with pytest.raises(ens.EnsError) as e:
        ens.solve("pollu", "rosenbrock23", U.float(), P.float(), (0.0, 1.0), 1e-3, adaptive=True, abstol=1e-6)
    assert e.value.status == 8
