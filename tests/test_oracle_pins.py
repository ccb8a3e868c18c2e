"""Pins for the CPU oracle (-m "not gpu").

Each test checks the oracle against something other than itself: the order
conditions of the published tableau, closed forms of the stability polynomial,
measured convergence orders, literature reference values, known-answer vectors,
exact discrete moments, brute-force linear algebra and finite differences.
Citations: P:n = PAPER.md line, S:n = SPEC.md line, SURVEY = SURVEY.md section.
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest

import oracle

GOLD = Path(__file__).parent / "golden"


def gold(name):
    return json.loads((GOLD / name).read_text())


# ------------------------------------------------------------------ tableau --
def _order_conditions(b, A, c):
    """All 17 rooted-tree conditions of order <= 5 (Butcher), as residuals."""
    e = np.ones_like(c)
    Ac, Ac2, Ac3 = A @ c, A @ c**2, A @ c**3
    AAc, AAc2, AAAc = A @ Ac, A @ Ac2, A @ (A @ Ac)
    return {
        "1": b @ e - 1, "2": b @ c - 1 / 2,
        "3a": b @ c**2 - 1 / 3, "3b": b @ Ac - 1 / 6,
        "4a": b @ c**3 - 1 / 4, "4b": b @ (c * Ac) - 1 / 8, "4c": b @ Ac2 - 1 / 12, "4d": b @ AAc - 1 / 24,
        "5a": b @ c**4 - 1 / 5, "5b": b @ (c**2 * Ac) - 1 / 10, "5c": b @ (c * Ac2) - 1 / 15,
        "5d": b @ (c * AAc) - 1 / 30, "5e": b @ (Ac * Ac) - 1 / 20, "5f": b @ Ac3 - 1 / 20,
        "5g": b @ (A @ (c * Ac)) - 1 / 40, "5h": b @ AAc2 - 1 / 60, "5i": b @ AAAc - 1 / 120,
    }


def test_tsit5_tableau_order_conditions():
    """Tsit5 is a 7-stage FSAL pair of order 5(4)."""
    c, A, bt, r = oracle.tsit5_tableau()
    b = A[6].copy()                       # FSAL: b = last row of A, b7 = 0
    assert A[6, 6] == 0 and c[6] == 1.0
    assert np.all(np.triu(A) == 0)        # explicit
    np.testing.assert_allclose(A.sum(1), c, atol=1e-15)     # row sums c_i = sum_j a_ij
    res = _order_conditions(b, A, c)
    assert len(res) == 17
    for name, v in res.items():
        assert abs(v) <= 1e-15 * 8, (name, v)
    # embedded weights b_hat = b - btilde: order exactly 4 ("one order less")
    assert abs(bt.sum()) < 1e-16
    bh = b - bt
    res_h = _order_conditions(bh, A, c)
    for name in ["1", "2", "3a", "3b", "4a", "4b", "4c", "4d"]:
        assert abs(res_h[name]) <= 1e-14, (name, res_h[name])
    assert abs(res_h["5a"]) > 1e-4        # fails an order-5 condition (5.8e-4)


def test_tsit5_embedded_scale_is_the_published_constant():
    """The eight order-≤4 conditions on Tsit5's seven stages have a one-dimensional
    null space, so they fix b̂ = b − b̃ only up to one scale along it (as for any
    embedded pair; Verner's scales are fixed by structural zeros, R21). Tsit5's
    scale is Tsitouras' published choice, b̂7 = −1/66 (b̃7 = 1/66 exactly in fp64):
    the pin here is that literature constant and that b̃ lies on the null direction
    (the estimate's scale is pinned by the published value only)."""
    c, A, bt, r = oracle.tsit5_tableau()
    Ac = A @ c
    M = np.array([np.ones(7), c, c**2, Ac, c**3, c * Ac, A @ c**2, A @ Ac])
    sv = np.linalg.svd(M, compute_uv=False)
    assert (sv > 1e-10).sum() == 6                     # rank 6: a one-dimensional null space
    assert np.abs(M @ bt).max() < 1e-15                # b̃ on that null direction
    assert bt[6] == 1.0 / 66.0


def test_tsit5_interpolant_conditions():
    """P:318 'free 4th-order interpolation': b_i(1) = b_i and the continuous
    order-4 conditions sum b_i(θ) Φ_i = θ^ρ/γ hold for all θ."""
    c, A, bt, r = oracle.tsit5_tableau()
    b = A[6]

    def bth(th):
        out = np.zeros(7)
        out[0] = th * (r[0, 0] + th * (r[0, 1] + th * (r[0, 2] + th * r[0, 3])))
        for i in range(1, 7):
            out[i] = th**2 * (r[i, 1] + th * (r[i, 2] + th * r[i, 3]))
        return out

    np.testing.assert_allclose(bth(1.0), b, atol=1e-14)
    Ac = A @ c
    for th in [0.1, 0.37, 0.5, 0.83, 1.0]:
        w = bth(th)
        conds = [w.sum() - th, w @ c - th**2 / 2, w @ c**2 - th**3 / 3, w @ Ac - th**3 / 6,
                 w @ c**3 - th**4 / 4, w @ (c * Ac) - th**4 / 8, w @ (A @ c**2) - th**4 / 12,
                 w @ (A @ Ac) - th**4 / 24]
        assert max(abs(x) for x in conds) < 1e-13, (th, conds)


# ------------------------------------------------------ Tsit5 closed forms --
def _R_tsit5(z, g6):
    return sum(z**k / math.factorial(k) for k in range(6)) + g6 * z**6


def test_tsit5_expdecay_closed_form():
    """Fixed-step Tsit5 on u'=-λu is u_N = R(-λh)^N u0 (R = stability polynomial)."""
    g = gold("closed_forms.json")
    g6 = g["tsit5_gamma6"]["value"]
    out, rc, na, _ = oracle.solve("expdecay", "tsit5", [[1.0]], [[1.0]], (0, 1), 0.1)
    v = out[0, 0, 0]
    assert rc[0] == 0 and na[0] == 10
    assert abs(v - g["expdecay_tsit5_h0.1_N10"]["value"]) <= 1e-14 * v
    assert abs(v - _R_tsit5(-0.1, g6) ** 10) <= 1e-14 * v
    # γ6 is not the Taylor 1/720: the oracle sees the tableau's own 6th coefficient
    assert abs(_R_tsit5(-0.1, 1 / 720) ** 10 - v) > 1e-13
    # several λ, h (vectorised over trajectories) in fp64 and fp32
    lam = np.array([0.5, 1.0, 3.0, 7.5])
    out, rc, na, _ = oracle.solve("expdecay", "tsit5", np.ones((1, 4)), lam[None, :], (0, 2), 0.05, dtype="f64")
    np.testing.assert_allclose(out[0, 0], _R_tsit5(-lam * 0.05, g6) ** 40, rtol=1e-13)
    # fp32 (R1): the products h·a_ij are rounded to fp32, which perturbs the
    # stability polynomial itself (4.8e-6 after 40 steps at λ = 7.5). The exact
    # expectation is R̃(z)^40 with R̃ built from the fp32-rounded h·a_ij (stage
    # recursion evaluated in fp64); what remains is arithmetic rounding, bounded
    # by one fp32 unit roundoff (2^-24) per step: 40·2^-24 = 2.4e-6.
    c, A, bt, r = oracle.tsit5_tableau()
    out, *_ = oracle.solve("expdecay", "tsit5", np.ones((1, 4)), lam[None, :], (0, 2), 0.05, dtype="f32")
    h32 = np.float32(0.05)
    ha = (h32 * A.astype(np.float32)).astype(np.float64)     # h·a_ij rounded to fp32 (R1)
    for i, l in enumerate(lam):
        l32 = float(np.float32(l))
        u = 1.0
        for _ in range(40):
            K = [-l32 * u]
            for s in range(1, 7):
                y = u + sum(ha[s, j] * K[j] for j in range(s))
                K.append(-l32 * y)
            u = y
        assert abs(float(out[0, 0, i]) - u) <= 40 * 2.0**-24 * abs(u), (l, float(out[0, 0, i]), u)
        # and the rounded-coefficient polynomial is what separates fp32 from R(z)^40
        exact = _R_tsit5(-l * 0.05, g6) ** 40
        assert abs(float(out[0, 0, i]) - exact) <= abs(u - exact) + 40 * 2.0**-24 * abs(u)


def test_tsit5_harmonic_closed_form():
    """x''=-x: u_N = R(hA)^N u0 with A = [[0,1],[-ω²,0]] (matrix polynomial)."""
    g = gold("closed_forms.json")
    g6 = g["tsit5_gamma6"]["value"]
    out, rc, na, _ = oracle.solve("harmonic", "tsit5", [[1.0], [0.0]], [[1.0]], (0, 1), 0.1)
    hx = g["harmonic_tsit5_h0.1_N10"]
    assert abs(out[0, 0, 0] - hx["x"]) <= 1e-14 and abs(out[0, 1, 0] - hx["v"]) <= 1e-14
    w2 = 2.25
    M = 0.1 * np.array([[0, 1.0], [-w2, 0]])
    R = sum(np.linalg.matrix_power(M, k) / math.factorial(k) for k in range(6)) + g6 * np.linalg.matrix_power(M, 6)
    expect = np.linalg.matrix_power(R, 30) @ np.array([0.3, -0.7])
    out, *_ = oracle.solve("harmonic", "tsit5", [[0.3], [-0.7]], [[w2]], (0, 3), 0.1)
    np.testing.assert_allclose(out[0, :, 0], expect, rtol=1e-13, atol=1e-15)


def test_tsit5_convergence_order():
    """Order 5 (S:347 slope in [4.5, 5.5]) on the harmonic oscillator."""
    errs = []
    T = 10.0
    for k in range(2, 6):
        dt = 2.0**-k
        out, *_ = oracle.solve("harmonic", "tsit5", [[1.0], [0.0]], [[1.0]], (0, T), dt)
        errs.append(np.abs(out[0, :, 0] - [math.cos(T), -math.sin(T)]).max())
    slopes = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all((slopes > 4.5) & (slopes < 5.5)), slopes


def test_tsit5_adaptive_tolerance():
    """P:116-120 adaptivity: error controlled by tolerance. S:336: u'=-u at 1e-10 → |err| ≤ 1e-8."""
    errs = {}
    for tol in [1e-6, 1e-8, 1e-10]:
        out, rc, na, nr = oracle.solve("expdecay", "tsit5", [[1.0]], [[1.0]], (0, 1), 1e-3, adaptive=True,
                                       abstol=tol, reltol=tol)
        assert rc[0] == 0
        errs[tol] = abs(out[0, 0, 0] - math.exp(-1))
        assert errs[tol] <= 100 * tol
    assert errs[1e-10] <= 1e-8
    assert errs[1e-6] > errs[1e-8] > errs[1e-10]
    # tighter tolerance ⇒ more steps, roughly tol^(-1/5) growth
    _, _, na6, _ = oracle.solve("lorenz", "tsit5", [[1.0], [0.0], [0.0]], [[10.0], [28.0], [8 / 3]], (0, 1), 1e-3,
                                adaptive=True, abstol=1e-6, reltol=1e-6)
    _, _, na10, _ = oracle.solve("lorenz", "tsit5", [[1.0], [0.0], [0.0]], [[10.0], [28.0], [8 / 3]], (0, 1), 1e-3,
                                 adaptive=True, abstol=1e-10, reltol=1e-10)
    ratio = na10[0] / na6[0]
    assert 10 ** (4 / 5) / 2 < ratio < 10 ** (4 / 5) * 2, ratio


def test_tsit5_adaptive_lorenz_converges():
    """Adaptive Lorenz (BASELINE C1 shape) at decreasing tolerances converges to a
    fine fixed-step solution (order-5 Tsit5, dt=1e-4 → error ≪ 1e-9)."""
    u0 = [[1.0], [0.0], [0.0]]
    p = [[10.0], [28.0], [8 / 3]]
    ref, *_ = oracle.solve("lorenz", "tsit5", u0, p, (0, 1), 1e-4)
    for tol, bound in [(1e-6, 1e-3), (1e-8, 1e-5), (1e-10, 1e-7)]:
        out, rc, *_ = oracle.solve("lorenz", "tsit5", u0, p, (0, 1), 1e-3, adaptive=True, abstol=tol, reltol=tol)
        assert rc[0] == 0
        rel = np.abs(out - ref).max() / np.abs(ref).max()
        assert rel < bound, (tol, rel)


def test_tsit5_interpolation_accuracy_and_grid_points():
    """saveat through the free interpolant: error O(h^5) between grid points;
    saves on grid points equal the step values bit for bit."""
    errs = []
    for dt in [0.1, 0.05]:
        tau = np.array([0.0, 0.033, 0.51, 0.777, 1.0])
        out, rc, na, _ = oracle.solve("expdecay", "tsit5", [[1.0]], [[1.0]], (0, 1), dt, saveat=tau)
        errs.append(np.abs(out[:, 0, 0] - np.exp(-tau)).max())
        assert out[0, 0, 0] == 1.0
        final, *_ = oracle.solve("expdecay", "tsit5", [[1.0]], [[1.0]], (0, 1), dt)
        assert out[-1, 0, 0] == final[0, 0, 0]
    assert errs[0] < 1e-6
    assert errs[0] / errs[1] > 2**4
    # grid-aligned saves (fixed step dt=0.25: τ=0.5 is step 2's end)
    out, *_ = oracle.solve("expdecay", "tsit5", [[1.0]], [[1.0]], (0, 0.5), 0.25, saveat=[0.5])
    fin, *_ = oracle.solve("expdecay", "tsit5", [[1.0]], [[1.0]], (0, 0.5), 0.25)
    assert out[0, 0, 0] == fin[0, 0, 0]


def test_fixed_grid_rule():
    """t∈[0,1], dt=1e-3 → exactly 1000 steps (DESIGN R3)."""
    g = gold("closed_forms.json")["lorenz_fixed_steps"]
    ns, hl = oracle.fixed_grid(0.0, 1.0, g["dt"])
    assert ns == g["nsteps"] and abs(hl - 1e-3) < 1e-15
    ns, hl = oracle.fixed_grid(0.0, 1.0, 0.3)
    assert ns == 4 and abs(hl - 0.1) < 1e-15
    _, rc, na, _ = oracle.solve("lorenz", "tsit5", [[1.0], [0.0], [0.0]], [[10.0], [21.0], [8 / 3]], (0, 1), 1e-3,
                                dtype="f32")
    assert na[0] == 1000 and rc[0] == 0


# ------------------------------------------------------------------- models --
def test_model_worked_values():
    g = gold("spec_worked_values.json")
    for key, model in [("lorenz_f_100", "lorenz"), ("lorenz_f_111", "lorenz"), ("robertson_f_100", "robertson")]:
        e = g[key]
        np.testing.assert_allclose(oracle.rhs(model, e["u"], e["p"]), e["f"], rtol=1e-15, atol=1e-15)
    e = g["lorenz_J_100"]
    np.testing.assert_allclose(oracle.jac("lorenz", e["u"], e["p"]), e["J"], rtol=1e-15)


@pytest.mark.parametrize("model,m", [("lorenz", 3), ("robertson", 3), ("expdecay", 1), ("harmonic", 1)])
def test_jacobian_vs_central_differences(model, m):
    """P:329 requires exact Jacobians; check the analytic J against central FD."""
    rng = np.random.default_rng(3)
    n = oracle.model_dims(model)[0]
    for _ in range(20):
        u = rng.uniform(-2, 2, n) if model != "robertson" else rng.uniform(0, 1, n) * [1, 1e-4, 1]
        p = rng.uniform(0.5, 2.0, m) * ([10, 28, 8 / 3] if model == "lorenz" else
                                         [0.04, 3e7, 1e4] if model == "robertson" else [1.0])
        J = oracle.jac(model, u, p)
        Jfd = np.zeros_like(J)
        for j in range(n):
            eps = 1e-6 * max(1.0, abs(u[j]))
            up, um = u.copy(), u.copy()
            up[j] += eps; um[j] -= eps
            Jfd[:, j] = (oracle.rhs(model, up, p) - oracle.rhs(model, um, p)) / (2 * eps)
        np.testing.assert_allclose(J, Jfd, rtol=1e-5, atol=1e-4 * max(1, np.abs(J).max()) * 1e-3)


def test_sde_diffusion_definitions():
    """P:686 GBM diffusion V·X; DESIGN R9 stochastic Lorenz b = s (add) / s·u (mul)."""
    u = np.array([0.3, -1.2, 2.0])
    np.testing.assert_array_equal(oracle.diffusion("gbm", u, [1.5, 0.01]), 0.01 * u)
    np.testing.assert_array_equal(oracle.diffusion("lorenz_sde_add", u, [10, 28, 8 / 3, 0.1]), [0.1] * 3)
    np.testing.assert_array_equal(oracle.diffusion("lorenz_sde_mul", u, [10, 28, 8 / 3, 0.1]), 0.1 * u)
    np.testing.assert_array_equal(oracle.rhs("gbm", u, [1.5, 0.01]), 1.5 * u)


# --------------------------------------------------------------- controller --
L_FLOOR = math.log2(1e-4)


def test_error_proportion_and_pi_controller():
    """Eq. q RMS reading: S:248 example q = 0.5 (q² = 0.25); P:120 accept
    iff q < 1; PI (DESIGN R2) h_new = h·η·q^{−β1}·q_old^{β2}, factor clamped to
    [1/5, 10]: exponents vanish at q = q_old = 1 → h·η; q = ∞ → h/5; q = 0 → 10h."""
    e = gold("spec_worked_values.json")["q_example"]
    assert oracle.error_q2(e["E"], e["u"], e["unew"], e["abstol"], e["reltol"]) == e["q"] ** 2
    assert oracle.error_q2([1e-3], [1.0], [1.0], 1e-3, 0.0) == 1.0
    assert oracle.error_q2([np.inf], [1.0], [1.0], 1e-3, 0.0) == np.inf
    assert oracle.error_q2([np.nan], [1.0], [1.0], 1e-3, 0.0) == np.inf
    for alg in ["tsit5", "rosenbrock23"]:
        C = oracle.controller(alg)
        h, lo = oracle.pi_step(alg, True, 1.0, 1.0, 0.0)
        assert abs(h - 0.9) < 1e-12 and lo == 0.0
        h, _ = oracle.pi_step(alg, False, 1.0, np.inf, 0.0)
        assert abs(h - 0.2) < 1e-12
        h, lo = oracle.pi_step(alg, True, 1.0, 0.0, 0.0)      # growth clamp: ×10, q_old floored at 1e-4
        assert abs(h - 10.0) < 1e-11 and abs(lo - L_FLOOR) < 1e-12
        # generic value: h η q^-β1 q_old^β2
        q, qold = 0.3, 0.02
        h, lo = oracle.pi_step(alg, True, 1.0, q * q, math.log2(qold))
        assert abs(h - 0.9 * q ** -C["beta1"] * qold ** C["beta2"]) < 1e-12
        assert abs(lo - math.log2(q)) < 1e-13
        # reject: h / min(5, q^β1/η)
        h, _ = oracle.pi_step(alg, False, 1.0, 1.7 ** 2, 0.0)
        assert abs(h - 1.0 / min(5.0, 1.7 ** C["beta1"] / 0.9)) < 1e-12
        # monotone: larger q → smaller h (SPEC stepcontrol invariant)
        hs = [oracle.pi_step(alg, True, 1.0, qq * qq, -1.0)[0] for qq in [0.01, 0.1, 0.5, 0.9]]
        assert all(a >= b for a, b in zip(hs, hs[1:]))
        assert oracle.pi_step(alg, False, 1.0, 1.5 ** 2, -1.0)[0] < 1.0
    assert oracle.controller("tsit5")["beta1"] == 7 / 50 and oracle.controller("rosenbrock23")["beta1"] == 7 / 20


@pytest.mark.parametrize("dtype,tol", [("f32", 3e-7), ("f64", 1e-13)])
def test_controller_log2_exp2(dtype, tol):
    """DESIGN R2: the controller's log2 / exp2 are fixed polynomials over exact IEEE
    operations; pinned to the math library over the range the controller sees."""
    rng = np.random.default_rng(1)
    xs = np.concatenate([10.0 ** rng.uniform(-30, 30, 400), [1e-4, 0.5, 1.0, 1.5, 2.0, 0.7071, 1.4142, 1e-12]])
    for x in xs:
        xt = float(np.float32(x)) if dtype == "f32" else x
        assert abs(oracle.log2_spec(xt, dtype) - math.log2(xt)) <= tol * max(1.0, abs(math.log2(xt))), x
    for z in np.concatenate([rng.uniform(-20, 20, 400), [-3.3219, 2.3219, 0.0, 0.5, -0.5]]):
        zt = float(np.float32(z)) if dtype == "f32" else z
        assert abs(oracle.exp2_spec(zt, dtype) - 2.0 ** zt) <= 2 * tol * 2.0 ** zt, z
    assert oracle.log2_spec(1.0, dtype) == 0.0 and oracle.exp2_spec(0.0, dtype) == 1.0
    assert oracle.log2_spec(8.0, dtype) == 3.0 and oracle.exp2_spec(-3.0, dtype) == 0.125


# ------------------------------------------------------------------------ LU --
def test_lu_examples_and_brute_force():
    """P:253-265 LU + substitution: SPEC examples S:136-147, Cramer's rule on random systems."""
    g = gold("spec_worked_values.json")
    for e in g["lu_examples"]:
        np.testing.assert_allclose(oracle.lu_solve(e["A"], e["b"]), e["x"], rtol=1e-15)
    assert oracle.lu_solve(g["lu_singular"]["A"], [1.0, 1.0]) is None
    rng = np.random.default_rng(5)
    for _ in range(200):
        A = rng.normal(size=(3, 3)) + 3 * np.eye(3) * rng.choice([-1, 1])
        b = rng.normal(size=3)
        det = np.linalg.det(A)
        cramer = np.array([np.linalg.det(np.column_stack([b if j == i else A[:, j] for j in range(3)])) / det
                           for i in range(3)])
        np.testing.assert_allclose(oracle.lu_solve(A, b), cramer, rtol=1e-11, atol=1e-12)
    # pivoting needed: zero leading entry
    A = np.array([[0.0, 2.0, 1.0], [1.0, 1.0, 0.0], [3.0, 0.0, 1.0]])
    b = np.array([1.0, 2.0, 3.0])
    np.testing.assert_allclose(A @ oracle.lu_solve(A, b), b, rtol=1e-14)


# -------------------------------------------------------------- Rosenbrock23 --
def _R_ros23(z, d):
    """Closed-form stability function of the ode23s step on u'=λu, z=hλ,
    derived by hand from k1 = W⁻¹F0, k2 = W⁻¹(F1−k1)+k1, u1 = u + h k2 with
    W = 1 − d z and F1 = λ(u + h/2 k1)."""
    w = 1 - d * z
    hk1 = z / w
    return 1 + hk1 + (z + (z / 2 - 1) * hk1) / w


def test_ros23_stability_function_and_L_stability():
    """P:321 'L-stable': R(z) of one step matches the closed form; R(-∞) = 0
    (pins d = 1/(2+√2)); S:326 |R(-1e6)| ≤ 1e-3."""
    d, e32 = oracle.ros23_consts()
    assert abs(d - 1 / (2 + math.sqrt(2))) < 1e-16 and abs(e32 - (6 + math.sqrt(2))) < 1e-15
    for z in [-0.01, -0.1, -1.0, -10.0, -1e3, -1e6]:
        out, rc, *_ = oracle.solve("expdecay", "rosenbrock23", [[1.0]], [[-z]], (0, 1), 1.0)
        assert rc[0] == 0
        R = out[0, 0, 0]
        assert abs(R - _R_ros23(z, d)) <= 1e-14 * max(1.0, abs(R)) + 1e-16, z
    out, *_ = oracle.solve("expdecay", "rosenbrock23", [[1.0]], [[1e6]], (0, 1), 1.0)
    assert abs(out[0, 0, 0]) <= 1e-3
    assert abs(_R_ros23(-1e15, d)) < 1e-12


def test_ros23_convergence_order():
    """Order 2 (slope in [1.7, 3.2])."""
    errs = []
    for k in range(3, 8):
        out, *_ = oracle.solve("harmonic", "rosenbrock23", [[1.0], [0.0]], [[1.0]], (0, 2), 2.0**-k)
        errs.append(np.abs(out[0, :, 0] - [math.cos(2), -math.sin(2)]).max())
    slopes = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all((slopes > 1.7) & (slopes < 3.2)), slopes


def test_ros23_robertson_reference_and_invariant():
    """P:668-679 Robertson on [0,1e5], h0=1e-4: literature values at t=40 and
    1e5; exact-J Rosenbrock preserves the linear invariant Σy = 1."""
    g = gold("robertson_reference.json")
    u0 = [[1.0], [0.0], [0.0]]
    p = [[0.04], [3e7], [1e4]]
    out, rc, na, nr = oracle.solve("robertson", "rosenbrock23", u0, p, (0, 40), 1e-4, adaptive=True,
                                   abstol=1e-10, reltol=1e-10)
    assert rc[0] == 0
    np.testing.assert_allclose(out[0, :, 0], g["t40"], rtol=2e-6)
    sa = np.linspace(0, 1e5, 100)
    out, rc, na, nr = oracle.solve("robertson", "rosenbrock23", u0, p, (0, 1e5), 1e-4, adaptive=True,
                                   abstol=1e-8, reltol=1e-8, saveat=sa)
    assert rc[0] == 0 and na[0] < 10000
    assert np.abs(out[:, :, 0].sum(1) - 1).max() <= 1e-12
    np.testing.assert_allclose(out[-1, :, 0], g["t1e5"], rtol=2e-3)
    assert np.all(np.isfinite(out))


def test_ros23_interpolant_endpoints():
    """ode23s dense output reproduces u_n at θ=0 and u_{n+1} at θ=1 and is
    second-order accurate between grid points."""
    tau = np.array([0.25, 0.5, 0.6, 1.0])
    out, *_ = oracle.solve("expdecay", "rosenbrock23", [[1.0]], [[1.0]], (0, 1), 0.5, saveat=tau)
    fin, *_ = oracle.solve("expdecay", "rosenbrock23", [[1.0]], [[1.0]], (0, 0.5), 0.5)
    assert out[1, 0, 0] == fin[0, 0, 0]
    errs = []
    for dt in [0.1, 0.05]:
        out, *_ = oracle.solve("expdecay", "rosenbrock23", [[1.0]], [[1.0]], (0, 1), dt, saveat=[0.333, 0.777])
        errs.append(np.abs(out[:, 0, 0] - np.exp(-np.array([0.333, 0.777]))).max())
    assert errs[0] / errs[1] > 3.0


# ------------------------------------------------------------- Philox / RNG --
def test_philox_known_answers():
    for v in gold("philox_kat.json")["vectors"]:
        out = oracle.philox([int(x, 16) for x in v["ctr"]], [int(x, 16) for x in v["key"]])
        assert [int(x) for x in out] == [int(x, 16) for x in v["out"]]


def test_uniforms_exact_open_interval():
    """DESIGN R8: fp32 U=((w>>9)+0.5)2^-23, fp64 U=((wa·2^20 + wb>>12)+0.5)2^-52, exact, in (0,1)."""
    u = oracle.uniforms([0, 0xFFFFFFFF, 512, 0x80000000], "f32")
    assert u[0] == np.float32(0.5 * 2**-23) and u[1] == np.float32((2**23 - 0.5) * 2**-23)
    assert u[2] == np.float32(1.5 * 2**-23) and u[3] == np.float32(0.5 + 0.5 * 2**-23)
    assert np.all((u > 0) & (u < 1))
    d = oracle.uniforms([0, 0, 0xFFFFFFFF, 0xFFFFFFFF], "f64")
    assert d[0] == 0.5 * 2**-52 and d[1] == (2**52 - 0.5) * 2**-52 and d[1] < 1.0


@pytest.mark.parametrize("dtype,tol", [("f32", 2.5e-7), ("f64", 1.5e-15)])   # reference sin(π·t) rounds π·t
def test_box_muller_sincospi(dtype, tol):
    """DESIGN R8: (sin πt, cos πt) for t ∈ (0, 2) by exact quadrant reduction and
    Taylor polynomials on [−¼, ¼]; pinned to the math library, and exact at the
    quadrant points."""
    rng = np.random.default_rng(7)
    ts = np.concatenate([rng.uniform(0, 2, 3000), np.arange(1, 16) / 8])
    for t in ts:
        tt = float(np.float32(t)) if dtype == "f32" else t
        s, c = oracle.sincospi_spec(tt, dtype)
        assert abs(s - math.sin(math.pi * tt)) <= tol and abs(c - math.cos(math.pi * tt)) <= tol, t
    for t, (se, ce) in [(0.5, (1, 0)), (1.0, (0, -1)), (1.5, (-1, 0))]:
        s, c = oracle.sincospi_spec(t, dtype)
        assert abs(s - se) == 0 and abs(c - ce) == 0


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_normals_statistics(dtype):
    """Box–Muller normals (DESIGN R8): mean/variance within 4σ; KS p > 0.01."""
    from scipy import stats
    z = oracle.normals(seed=0xC4, gidx=12345, step0=0, count=200000, dtype=dtype).astype(np.float64).ravel()
    n = z.size
    assert abs(z.mean()) < 4 / math.sqrt(n)
    assert abs(z.var() - 1) < 4 * math.sqrt(2 / n)
    assert stats.kstest(z, "norm").pvalue > 0.01
    # different trajectories / steps give different streams
    a = oracle.normals(1, 0, 0, 4, dtype)
    b = oracle.normals(1, 1, 0, 4, dtype)
    assert not np.array_equal(a, b)
    np.testing.assert_array_equal(oracle.normals(1, 0, 2, 2, dtype), a[2:])


# ----------------------------------------------------------- Euler–Maruyama --
def test_em_zero_noise_is_euler():
    """b ≡ 0 ⇒ EM is explicit Euler: GBM with V=0 gives X0(1+rh)^N (S:395 one-step 0.115)."""
    e = gold("spec_worked_values.json")["em_gbm_one_step"]
    out, rc, na, _ = oracle.solve("gbm", "em", np.full((3, 1), e["X0"]), [e["r"], 0.0], (0, e["h"]), e["h"],
                                  p_broadcast=True)
    np.testing.assert_allclose(out[0, :, 0], e["X1"], rtol=1e-15)
    out, rc, na, _ = oracle.solve("gbm", "em", np.full((3, 2), 0.1), [1.5, 0.0], (0, 1), 1e-3, p_broadcast=True)
    assert na[0] == 1000
    np.testing.assert_allclose(out[0], 0.1 * (1 + 1.5e-3) ** 1000, rtol=1e-12)
    # stochastic Lorenz with s = 0: additive and multiplicative forms coincide bitwise
    a, *_ = oracle.solve("lorenz_sde_add", "em", np.array([[1.0], [0.0], [0.0]]), [10, 28, 8 / 3, 0.0], (0, 1),
                         1e-3, p_broadcast=True, seed=9)
    b, *_ = oracle.solve("lorenz_sde_mul", "em", np.array([[1.0], [0.0], [0.0]]), [10, 28, 8 / 3, 0.0], (0, 1),
                         1e-3, p_broadcast=True, seed=9)
    np.testing.assert_array_equal(a, b)
    # and both equal an explicit-Euler loop on the Lorenz RHS (separate rounding: 1e-12)
    u = np.array([1.0, 0.0, 0.0])
    for _ in range(1000):
        f = np.array([10 * (u[1] - u[0]), u[0] * (28 - u[2]) - u[1], u[0] * u[1] - 8 / 3 * u[2]])
        u = u + 1e-3 * f
    np.testing.assert_allclose(a[0, :, 0], u, rtol=1e-11)


def test_em_gbm_exact_discrete_moments():
    """P:684-688 GBM (X0=0.1, r=1.5, V=0.01), EM h=1e-3, 1000 steps. The EM
    recursion X_{i+1} = X_i(1 + r h + V ΔW) has exact moments
    E = X0(1+rh)^N, E[X²] = X0²((1+rh)² + V²h)^N (independent increments).
    Sample mean within 4 SE of E_h and distinguishable from X0·e^{rT}."""
    X0, r, V, h, N = 0.1, 1.5, 0.01, 1e-3, 1000
    E_h = X0 * (1 + r * h) ** N
    E2_h = X0**2 * ((1 + r * h) ** 2 + V**2 * h) ** N
    var_h = E2_h - E_h**2
    E_c = X0 * math.exp(r)
    paths = 8000
    out, rc, *_ = oracle.solve("gbm", "em", np.full((3, paths), X0), [r, V], (0, 1), h, p_broadcast=True, seed=0xC4)
    x = out[0].ravel()                         # 3 independent components × paths
    se = math.sqrt(var_h / x.size)
    assert abs(x.mean() - E_h) < 4 * se, (x.mean(), E_h, se)
    assert abs(x.mean() - E_c) > 8 * se
    se_var = var_h * math.sqrt(2 / (x.size - 1))
    assert abs(x.var(ddof=1) - var_h) < 4 * se_var


def test_em_saveat_on_grid():
    """DESIGN R11: EM saves the state after the step that ends on τ; τ=t0 saves u0."""
    sa = [0.0, 0.5, 1.0]
    out, *_ = oracle.solve("gbm", "em", np.full((3, 4), 0.1), [1.5, 0.01], (0, 1), 1e-2, p_broadcast=True,
                           seed=3, saveat=sa)
    fin, *_ = oracle.solve("gbm", "em", np.full((3, 4), 0.1), [1.5, 0.01], (0, 1), 1e-2, p_broadcast=True, seed=3)
    half, *_ = oracle.solve("gbm", "em", np.full((3, 4), 0.1), [1.5, 0.01], (0, 0.5), 1e-2, p_broadcast=True,
                            seed=3)
    np.testing.assert_array_equal(out[0], 0.1)
    np.testing.assert_array_equal(out[2], fin[0])
    # the (0, 0.5) run's last step is h_last = 0.5 − 49·0.01 (fp64), one rounding away from 0.01
    np.testing.assert_allclose(out[1], half[0], rtol=1e-14)


# -------------------------------------------------------------------- stats --
def test_stats_exact_small_cases():
    """P:157 ensemble mean/variance: unbiased sample variance (DESIGN R12)."""
    x = np.array([1.0, 2.0, 3.0, 4.0]).reshape(1, 1, 4)
    mean, var, c = oracle.stats(x)
    assert mean[0, 0] == 2.5 and abs(var[0, 0] - 5 / 3) < 1e-16 and c == 4
    # shift invariance with a large offset (two-pass in long double)
    y = x + 1e8
    mean, var, _ = oracle.stats(y)
    assert mean[0, 0] == 1e8 + 2.5 and abs(var[0, 0] - 5 / 3) < 1e-9
    mean, var, c = oracle.stats(x, mask=np.array([1, 0, 1, 0]))
    assert mean[0, 0] == 2.0 and var[0, 0] == 2.0 and c == 2
    # non-finite values (failed trajectories, unreached save points) are excluded
    z = np.array([1.0, np.nan, 3.0, np.inf]).reshape(1, 1, 4)
    mean, var, c = oracle.stats(z)
    assert mean[0, 0] == 2.0 and var[0, 0] == 2.0 and c == 2


# --------------------------------------------------------- failure handling --
def test_retcodes():
    """S:63 retcodes: MaxIters, Diverged (non-finite f(u0)); peers unaffected."""
    u0 = np.array([[1.0, np.nan], [0.0, 0.0], [0.0, 0.0]])
    p = np.array([[10.0, 10.0], [28.0, 28.0], [8 / 3, 8 / 3]])
    out, rc, na, nr = oracle.solve("lorenz", "tsit5", u0, p, (0, 1), 1e-3, adaptive=True, abstol=1e-8, reltol=1e-8)
    assert rc[0] == 0 and rc[1] == 3
    out, rc, na, nr = oracle.solve("lorenz", "tsit5", u0[:, :1], p[:, :1], (0, 1), 1e-3, adaptive=True,
                                   abstol=1e-8, reltol=1e-8, max_steps=10)
    assert rc[0] == 1 and na[0] + nr[0] == 10


# ------------------------------------------------------------ CRN (NEXT-3) --
CRN_P = [2.0, 3.0, 5.0, 0.1, 2.0, 0.05]      # (S, D, τ, ν0, n, η)


def test_crn_drift_worked_values():
    """P:692-705 drift by direct substitution: Hill term (Sσ)^n / ((Sσ)^n + (D A3)^n + 1)."""
    S, D, tau, nu0, n, eta = CRN_P
    y = np.array([0.5, 0.2, 0.3, 1.0 / 3.0])       # Sσ = 1, D·A3 = 1 → H = 1/3
    f = oracle.rhs("crn", y, CRN_P)
    np.testing.assert_allclose(f, [nu0 + 1 / 3 - 0.5, (0.5 - 0.2) / tau, (0.2 - 0.3) / tau, (0.3 - 1 / 3) / tau],
                               rtol=1e-12)
    f0 = oracle.rhs("crn", np.zeros(4), CRN_P)      # σ = 0 → H = 0 (R14 clamps)
    np.testing.assert_allclose(f0, [nu0, 0, 0, 0], atol=1e-50)
    y2 = np.array([1.5, 0.0, 0.0, 0.0])              # Sσ = 3, A3 = 0 → H = 9/10
    assert abs(oracle.rhs("crn", y2, CRN_P)[0] - (nu0 + 0.9 - 1.5)) < 1e-12
    # non-integer Hill exponent
    p = list(CRN_P); p[4] = 2.5
    y3 = np.array([0.8, 0.1, 0.1, 0.4])
    a, b = (2.0 * 0.8) ** 2.5, (3.0 * 0.4) ** 2.5
    assert abs(oracle.rhs("crn", y3, p)[0] - (0.1 + a / (a + b + 1) - 0.8)) < 1e-12


def test_crn_deterministic_steady_state():
    """η = 0: EM is explicit Euler on the drift; it relaxes to the fixed point
    A1 = A2 = A3 = σ*, σ* = ν0 + (Sσ*)^n / ((Sσ*)^n + (Dσ*)^n + 1), found here by bisection."""
    S, D, tau, nu0, n, eta = CRN_P
    g = lambda s: nu0 + (S * s) ** n / ((S * s) ** n + (D * s) ** n + 1) - s
    lo, hi = 1e-9, 2.0
    assert g(lo) > 0 > g(hi)
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        lo, hi = (mid, hi) if g(mid) > 0 else (lo, mid)
    p = list(CRN_P); p[5] = 0.0; p[2] = 0.5      # τ = 0.5: stable fixed point (slow τ oscillates)
    out, rc, na, _ = oracle.solve("crn", "em", np.full((4, 1), nu0), np.array(p)[:, None], (0, 300), 0.1)
    assert rc[0] == 0 and na[0] == 3000
    np.testing.assert_allclose(out[0, :, 0], [lo] * 4, rtol=1e-9)
    # and the same trajectory by fixed-step Tsit5 at t = 20 agrees to O(dt) (Euler is order 1)
    eu, *_ = oracle.solve("crn", "em", np.full((4, 1), nu0), np.array(p)[:, None], (0, 20), 1e-3)
    ts, *_ = oracle.solve("crn", "tsit5", np.full((4, 1), nu0), np.array(p)[:, None], (0, 20), 1e-2)
    assert np.abs(eu - ts).max() < 5e-3 * np.abs(ts).max()


def test_crn_one_step_noise_variance():
    """One EM step from a fixed state over many independent paths: the increment
    variance is h·η²·(ν0 + H + σ) for [σ] and h·η²·(A_{k−1} + A_k)/τ for [A_k]
    (the two Wiener terms of each equation)."""
    S, D, tau, nu0, n, eta = CRN_P
    y = np.array([0.5, 0.2, 0.3, 1.0 / 3.0])
    N, h = 20000, 0.1
    out, *_ = oracle.solve("crn", "em", np.tile(y[:, None], (1, N)), np.tile(np.array(CRN_P)[:, None], (1, N)),
                           (0, h), h, seed=11)
    d = out[0] - y[:, None]
    H = 1 / 3
    mean = h * oracle.rhs("crn", y, CRN_P)
    var = h * eta**2 * np.array([nu0 + H + y[0], (y[0] + y[1]) / tau, (y[1] + y[2]) / tau, (y[2] + y[3]) / tau])
    se_m = np.sqrt(var / N)
    assert np.all(np.abs(d.mean(1) - mean) < 5 * se_m)
    assert np.all(np.abs(d.var(1, ddof=1) / var - 1) < 5 * np.sqrt(2 / N))
    # nw = 8 normals per step: four independent Box–Muller pairs
    z = oracle.normals(3, 7, 0, 20000, "f64", nw=8)
    assert np.abs(np.corrcoef(z.T) - np.eye(8)).max() < 0.04


# ------------------------------------------------- stiff suite (NEXT-4) --
def test_stiff_suite_literature_references():
    """P:733-844 OREGO / HIRES / POLLU with Rosenbrock23 and the forward-mode AD
    Jacobian (R15) against the IVP test-set reference solutions."""
    from synth.inputs import make_inputs
    g = gold("stiff_references.json")
    for model, tol, bound in [("hires", 1e-10, 2e-6), ("pollu", 1e-10, 1e-6), ("orego", 1e-8, 1e-4)]:
        u0, p = make_inputs(model, "const", 1)
        if model == "pollu":
            u0[8, 0] = g["pollu"]["y9_0"]
        out, rc, na, nr = oracle.solve(model, "rosenbrock23", u0, p, (0, g[model]["tf"]), 1e-6, adaptive=True,
                                       abstol=tol, reltol=tol, p_broadcast=True)
        assert rc[0] == 0
        ref = np.array(g[model]["y"])
        big = np.abs(ref) > 1e-10
        rel = np.abs(out[0, :, 0] - ref)[big] / np.abs(ref[big])
        assert rel.max() < bound, (model, rel.max())


def test_hires_linear_invariant():
    """HIRES: d(y7 + y8)/dt = 0 exactly; an exact-Jacobian Rosenbrock
    method preserves the linear invariant y7 + y8 = 0.0057 to rounding."""
    from synth.inputs import make_inputs
    u0, p = make_inputs("hires", "random10", 3, seed=5)
    sa = np.linspace(0, 321.8122, 50)
    out, rc, *_ = oracle.solve("hires", "rosenbrock23", u0, p, (0, 321.8122), 1e-6, adaptive=True, abstol=1e-8,
                               reltol=1e-8, saveat=sa)
    assert (rc == 0).all()
    assert np.abs(out[:, 6, :] + out[:, 7, :] - 0.0057).max() < 1e-15


@pytest.mark.parametrize("model", ["orego", "hires", "pollu"])
def test_ad_jacobian_vs_central_differences(model):
    """Forward-mode AD Jacobian (R15) equals central finite differences."""
    from synth.inputs import make_inputs
    rng = np.random.default_rng(2)
    u0, p = make_inputs(model, "random10", 4, seed=9)
    n = u0.shape[0]
    for i in range(4):
        u = np.abs(u0[:, i]) + rng.uniform(0.01, 1.0, n) * (np.abs(u0[:, i]).max() + 0.1)
        J = oracle.jac(model, u, p[:, i])
        Jfd = np.zeros_like(J)
        for j in range(n):
            eps = 1e-6 * max(1.0, abs(u[j]))
            up, um = u.copy(), u.copy()
            up[j] += eps; um[j] -= eps
            Jfd[:, j] = (oracle.rhs(model, up, p[:, i]) - oracle.rhs(model, um, p[:, i])) / (2 * eps)
        np.testing.assert_allclose(J, Jfd, rtol=1e-5, atol=1e-6 * max(1.0, np.abs(J).max()))
