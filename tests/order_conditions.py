"""Order conditions from rooted trees (test infrastructure; no method arithmetic).

Explicit Runge–Kutta (Butcher): Σ b_i Φ_i(t) = 1/γ(t) with
Φ_i(t) = Π_children Σ_j a_ij Φ_j(child).

Rosenbrock (standard form, exact Jacobian; Hairer & Wanner IV.7):
k_i = h f(y0 + Σ α_ij k_j) + h J Σ_j Γ_ij k_j. In the B-series normalisation
y1 = y0 + Σ_t h^|t| a(t) F(t)/σ(t), exact solution a(t) = 1/γ(t), the stage
coefficients follow the recursion
  k_i(t) = Π_children (Σ_j α_ij k_j(child)) + [t = [u]] Σ_j Γ_ij k_j(u)
(the J-term feeds only trees whose root has a single child), and the method
has order p iff Σ_i b_i k_i(t) = 1/γ(t) for every tree with |t| ≤ p.
The W-form (a, c, m, γ) maps to it by Γ⁻¹ = diag(1/γ) − C, α = A Γ, b = m Γ.
"""
from functools import lru_cache

import numpy as np


@lru_cache(None)
def trees(n):
    """Rooted trees with n nodes, as sorted tuples of child trees."""
    if n == 1:
        return ((),)
    out = set()

    def gen(rem, maxkey, acc):
        if rem == 0:
            out.add(tuple(sorted(acc)))
            return
        for k in range(1, rem + 1):
            for t in trees(k):
                if maxkey is not None and (k, t) > maxkey:
                    continue
                gen(rem - k, (k, t), acc + [t])
    gen(n - 1, None, [])
    return tuple(sorted(out))


def size(t):
    return 1 + sum(size(c) for c in t)


def gamma(t):
    g = size(t)
    for c in t:
        g *= gamma(c)
    return g


def rk_max_residual(b, A, order):
    """max over trees of order `order` of |Σ b_i Φ_i(t) − 1/γ(t)| (explicit RK)."""
    def phi(t):
        v = np.ones(A.shape[0])
        for ch in t:
            v = v * (A @ phi(ch))
        return v
    return max(abs(b @ phi(t) - 1.0 / gamma(t)) for t in trees(order))


def rosenbrock_residuals(Aw, Cw, g, m, max_order):
    """{order: max residual} of a W-form Rosenbrock method (weights m on the
    W-form stages) against the exact-Jacobian B-series conditions."""
    s = Aw.shape[0]
    G = np.linalg.inv(np.diag(np.full(s, 1.0 / g)) - Cw)
    return rosenbrock_residuals_std(Aw @ G, G, m @ G, max_order)


def rosenbrock_residuals_std(alpha, G, b, max_order):
    """Same for the standard form (α, Γ incl. its diagonal, b); Γ = 0 is explicit RK."""
    s = alpha.shape[0]
    memo = {}

    def k(t):
        if t not in memo:
            v = np.ones(s)
            for ch in t:
                v = v * (alpha @ k(ch))
            if len(t) == 1:
                v = v + G @ k(t[0])
            memo[t] = v
        return memo[t]
    return {n: max(abs(b @ k(t) - 1.0 / gamma(t)) for t in trees(n)) for n in range(1, max_order + 1)}
