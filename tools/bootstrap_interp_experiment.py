#!/usr/bin/env python
"""Experiment behind DESIGN R24 (not product code): a Hermite–Birkhoff interpolant
bootstrapped from f-evaluations alone as a stand-in for Verner's lazy interpolants.

Data of one step: y0, y1 (exact here), h·f(y0), h·f(y1); level ℓ adds h·f(P_{ℓ−1}(θ_ℓ))
and raises the polynomial degree by one. Printed: the max error over θ ∈ [0.05, 0.95]
for h = 0.4, 0.2, 0.1 on the harmonic oscillator and the ratio per halving. Every
level stays at ratio ≈ 32 (h^5): the first bootstrap point carries the O(h^5) error of
the cubic Hermite it was evaluated on into every later level, so the construction
cannot reach order 7 / 9 without re-evaluating all points (several sweeps)."""
from fractions import Fraction as Fr

import numpy as np


def hb_matrix(thetas):
    d = 3 + len(thetas)
    rows = [[Fr(1)] + [Fr(0)] * (d - 1), [Fr(1)] * d, [Fr(k) for k in range(1, d + 1)]]
    for t in thetas:
        rows.append([Fr(k) * Fr(t) ** (k - 1) for k in range(1, d + 1)])
    return np.array([[float(x) for x in r] for r in rows])


def bootstrap(thetas, y0, y1, F0, F1, f, h):
    D, used = [h * F0, y1 - y0, h * F1], []

    def P(th, used, D):
        c = np.linalg.solve(hb_matrix(used), np.array(D))
        return y0 + sum(c[k - 1] * th ** k for k in range(1, len(used) + 4))

    for t in thetas:
        D = D + [h * f(P(t, used, D))]
        used = used + [t]
    return lambda th: P(th, used, D)


def main():
    harm = lambda y: np.array([y[1], -y[0]])
    exact = lambda y0, t: np.array([np.cos(t) * y0[0] + np.sin(t) * y0[1], -np.sin(t) * y0[0] + np.cos(t) * y0[1]])
    y0 = np.array([1.0, 0.5])
    for nodes in [(1 / 3, 2 / 3, 1 / 6, 5 / 6), (0.2, 0.8, 0.4, 0.6)]:
        for lev in range(1, 5):
            errs = []
            for h in [0.4, 0.2, 0.1]:
                y1 = exact(y0, h)
                P = bootstrap(nodes[:lev], y0, y1, harm(y0), harm(y1), harm, h)
                errs.append(max(np.abs(P(x) - exact(y0, x * h)).max() for x in np.linspace(0.05, 0.95, 19)))
            print(nodes, "level", lev, ["%.2e" % e for e in errs], ["%.1f" % (errs[i] / errs[i + 1]) for i in range(2)])


if __name__ == "__main__":
    main()
