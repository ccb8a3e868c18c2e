"""Pins for the oracle's Rodas5P (GPURodas5P, Table 4's reference;
NEXT-2; DESIGN R23): the Rosenbrock B-series order conditions of every rooted
tree up to order 5 (main) / 4 (embedded) — the published coefficients satisfy
them to 2e-14 and violate order 6, so a mistyped digit fails — the stiffly
accurate structure, L-stability and the stability function of one step,
measured convergence orders, the Robertson / stiff-suite literature references
 and the dense-output save rule (R24;
tests/test_oracle_dense_output.py)."""
import json
import math
from pathlib import Path

import numpy as np

import oracle
from tests.order_conditions import rosenbrock_residuals

GOLD = Path(__file__).parent / "golden"


def _tab():
    g, A, C = oracle.rodas5p_tableau()
    m = np.concatenate([A[7, :7], [1.0]])       # u_new = Y8 + k8 (stiffly accurate)
    me = np.concatenate([A[7, :7], [0.0]])      # embedded Y8
    return g, A, C, m, me


def test_rodas5p_order_conditions():
    g, A, C, m, me = _tab()
    r = rosenbrock_residuals(A, C, g, m, 6)
    assert max(r[k] for k in range(1, 6)) < 5e-14, r
    assert r[6] > 1e-4
    r = rosenbrock_residuals(A, C, g, me, 5)
    assert max(r[k] for k in range(1, 5)) < 5e-14, r
    assert r[5] > 1e-4
    # stiffly accurate structure: Y7 = Y6 + k6, Y8 = Y7 + k7
    np.testing.assert_array_equal(A[6, :5], A[5, :5])
    np.testing.assert_array_equal(A[7, :6], A[6, :6])
    assert A[6, 5] == 1.0 and A[7, 6] == 1.0 and g == 0.21193756319429014


def _R(z):
    g, A, C, m, me = _tab()
    G = np.linalg.inv(np.diag(np.full(8, 1 / g)) - C)
    bh = A @ G + G
    return 1 + z * (m @ G) @ np.linalg.solve(np.eye(8) - z * bh, np.ones(8))


def test_rodas5p_stability_function_and_L_stability():
    for z in [-0.01, -0.5, -3.0, -1e3, -1e6]:
        out, rc, *_ = oracle.solve("expdecay", "rodas5p", [[1.0]], [[-z]], (0, 1), 1.0)
        assert rc[0] == 0
        R = _R(z)
        assert abs(out[0, 0, 0] - R) <= 1e-12 * max(1.0, abs(R)) + 1e-15, (z, out[0, 0, 0], R)
    assert abs(_R(-1e12)) < 1e-8
    for z in [-0.2, -0.1]:
        assert abs(_R(z) - math.exp(z)) < 0.05 * abs(z) ** 6


def test_rodas5p_convergence_order():
    errs = []
    for k in range(2, 6):
        out, *_ = oracle.solve("harmonic", "rodas5p", [[1.0], [0.0]], [[1.0]], (0, 2), 2.0**-k)
        errs.append(np.abs(out[0, :, 0] - [math.cos(2), -math.sin(2)]).max())
    s = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    # linear problem: Rodas5P's stability function matches e^z closely at order 6 as well
    # (measured slopes 5.8–5.9 before round-off), so the bound is wider than Rodas5's
    assert np.all((s > 4.5) & (s < 6.3)), (s, errs)
    u0, p = [[1.0], [0.0], [0.0]], [[10.0], [28.0], [8 / 3]]
    ref, *_ = oracle.solve("lorenz", "tsit5", u0, p, (0, 0.5), 1e-5)
    errs = []
    for k in range(6, 9):
        out, *_ = oracle.solve("lorenz", "rodas5p", u0, p, (0, 0.5), 2.0**-k)
        errs.append(np.abs(out[0, :, 0] - ref[0, :, 0]).max())
    s = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all((s > 4.4) & (s < 5.9)), (s, errs)


def test_rodas5p_robertson_reference_and_invariant():
    g = json.loads((GOLD / "robertson_reference.json").read_text())
    u0, p = [[1.0], [0.0], [0.0]], [[0.04], [3e7], [1e4]]
    out, rc, na, nr = oracle.solve("robertson", "rodas5p", u0, p, (0, 40), 1e-4, adaptive=True, abstol=1e-10,
                                   reltol=1e-10)
    assert rc[0] == 0
    np.testing.assert_allclose(out[0, :, 0], g["t40"], rtol=1e-6)
    sa = np.linspace(0, 1e5, 100)
    out, rc, na, nr = oracle.solve("robertson", "rodas5p", u0, p, (0, 1e5), 1e-4, adaptive=True, abstol=1e-8,
                                   reltol=1e-8, saveat=sa)
    assert rc[0] == 0
    assert np.abs(out[:, :, 0].sum(1) - 1).max() <= 1e-12
    np.testing.assert_allclose(out[-1, :, 0], g["t1e5"], rtol=2e-3)


def test_rodas5p_stiff_suite_references():
    from synth.inputs import make_inputs
    g = json.loads((GOLD / "stiff_references.json").read_text())
    for model, tol, bound in [("hires", 1e-10, 2e-6), ("pollu", 1e-10, 1e-6), ("orego", 1e-9, 1e-4)]:
        u0, p = make_inputs(model, "const", 1)
        if model == "pollu":
            u0[8, 0] = g["pollu"]["y9_0"]
        kw = dict(adaptive=True, abstol=tol, reltol=tol, p_broadcast=True)
        out, rc, na, nr = oracle.solve(model, "rodas5p", u0, p, (0, g[model]["tf"]), 1e-6, **kw)
        assert rc[0] == 0
        ref = np.array(g[model]["y"])
        big = np.abs(ref) > 1e-10
        rel = np.abs(out[0, :, 0] - ref)[big] / np.abs(ref[big])
        assert rel.max() < bound, (model, rel.max())
        _, _, na4, _ = oracle.solve(model, "rodas4", u0, p, (0, g[model]["tf"]), 1e-6, **kw)
        assert na[0] < na4[0], (model, na[0], na4[0])
        _, _, na5, _ = oracle.solve(model, "rodas5", u0, p, (0, g[model]["tf"]), 1e-6, **kw)
        assert na[0] < 2 * na5[0], (model, na[0], na5[0])   # same order as Rodas5 (HIRES: 563 vs 415)


def test_rodas5p_saveat_and_controller():
    sa = np.array([0.0, 0.37, 1.0, 2.2, 3.0])
    out, rc, *_ = oracle.solve("harmonic", "rodas5p", [[1.0], [0.0]], [[1.0]], (0, 3.0), 0.1, adaptive=True,
                               abstol=1e-11, reltol=1e-11, saveat=sa)
    assert rc[0] == 0
    exact = np.stack([np.cos(sa), -np.sin(sa)], 1)
    assert np.abs(out[:, :, 0] - exact).max() < 1e-9
    c = oracle.controller("rodas5p")
    assert c["beta1"] == 7 / 50 and c["beta2"] == 2 / 25
