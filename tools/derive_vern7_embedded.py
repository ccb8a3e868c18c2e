#!/usr/bin/env python
"""Derive the Vern7 embedded-error weights b̃ = b − b̂ (DESIGN R21).

The main 7th-order weights b, the nodes c and the matrix A are Verner's
published "most efficient" 7(6) pair (P:319-320 names GPUVern7; the paper
prints no coefficients). The order-6 embedded weights b̂ are fixed here from
the order conditions: b̂ − b must satisfy every homogeneous condition of order
≤ 6 (37 rooted trees), which on these 10 stages leaves exactly one direction δ;
its scale is set by b̂1 = 0.044063029903460226. Prints b̃ to 17 significant
digits (the literals in oracle/oracle.cpp and csrc/vern7.cuh) and the residuals.
Uses mpmath at 50 digits; no oracle / library code.
"""
import mpmath as mp

mp.mp.dps = 50
D = mp.mpf
C = [D(0), D("0.005"), D("0.10888888888888888"), D("0.16333333333333333"), D("0.4555"),
     D("0.6095094489978381"), D("0.884"), D("0.925"), D(1), D(1)]
A = [[D(0)] * 10 for _ in range(10)]
rows = {
    1: {0: "0.005"},
    2: {0: "-1.07679012345679", 1: "1.185679012345679"},
    3: {0: "0.04083333333333333", 2: "0.1225"},
    4: {0: "0.6389139236255726", 2: "-2.455672638223657", 3: "2.272258714598084"},
    5: {0: "-2.6615773750187572", 2: "10.804513886456137", 3: "-8.3539146573962", 4: "0.820487594956657"},
    6: {0: "6.067741434696772", 2: "-24.711273635911088", 3: "20.427517930788895", 4: "-1.9061579788166472",
        5: "1.006172249242068"},
    7: {0: "12.054670076253203", 2: "-49.75478495046899", 3: "41.142888638604674", 4: "-4.461760149974004",
        5: "2.042334822239175", 6: "-0.09834843665406107"},
    8: {0: "10.138146522881808", 2: "-42.6411360317175", 3: "35.76384003992257", 4: "-4.3480228403929075",
        5: "2.0098622683770357", 6: "0.3487490460338272", 7: "-0.27143900510483127"},
    9: {0: "-45.030072034298676", 2: "187.3272437654589", 3: "-154.02882369350186", 4: "18.56465306347536",
        5: "-7.141809679295079", 6: "1.3088085781613787"},
}
for i, r in rows.items():
    for j, v in r.items():
        A[i][j] = D(v)
B = [D("0.04715561848627222"), D(0), D(0), D("0.25750564298434153"), D("0.2621665397741262"),
     D("0.15216092656738558"), D("0.4939969170032485"), D("-0.29430311714032503"), D("0.08131747232495111"), D(0)]
BHAT1 = D("0.044063029903460226")


def trees(n, memo={}):
    """Rooted trees with n nodes as sorted tuples of children."""
    if n in memo:
        return memo[n]
    if n == 1:
        memo[1] = [()]
        return memo[1]
    out = set()

    def gen(rem, maxkey, acc):
        if rem == 0:
            out.add(tuple(sorted(acc)))
            return
        for k in range(1, rem + 1):
            for t in trees(k):
                key = (k, t)
                if maxkey is not None and key > maxkey:
                    continue
                gen(rem - k, key, acc + [t])
    gen(n - 1, None, [])
    memo[n] = sorted(out)
    return memo[n]


def size(t):
    return 1 + sum(size(c) for c in t)


def gamma(t):
    g = size(t)
    for c in t:
        g *= gamma(c)
    return g


def phi(t):
    v = [D(1)] * 10
    for ch in t:
        w = phi(ch)
        aw = [mp.fsum(A[i][j] * w[j] for j in range(10)) for i in range(10)]
        v = [v[i] * aw[i] for i in range(10)]
    return v


def main():
    conds = [(n, t) for n in range(1, 7) for t in trees(n)]
    M = mp.matrix([phi(t) for _, t in conds])
    # δ with δ8 = −1 (index 7) and δ2 = δ3 = 0 (stages 2, 3 carry no weight in b or b̂): solve the
    # homogeneous system in the other 7 unknowns (least squares; consistent to the literals' rounding)
    cols = [j for j in range(10) if j not in (1, 2, 7)]
    Ms = mp.matrix([[M[r, j] for j in cols] for r in range(M.rows)])
    rhs = mp.matrix([M[r, 7] for r in range(M.rows)])     # Σ_j M_rj δ_j − M_r7 = 0
    x = mp.lu_solve(Ms.T * Ms, Ms.T * rhs)
    delta = [D(0)] * 10
    for k, j in enumerate(cols):
        delta[j] = x[k]
    delta[7] = D(-1)
    res = max(abs(mp.fsum(M[r, j] * delta[j] for j in range(10))) for r in range(M.rows))
    s = (BHAT1 - B[0]) / delta[0]
    bhat = [B[j] + s * delta[j] for j in range(10)]
    btilde = [B[j] - bhat[j] for j in range(10)]
    print(f"# homogeneous residual of delta: {mp.nstr(res, 5)}")
    for k in range(1, 9):
        rb = max(abs(mp.fsum(B[j] * phi(t)[j] for j in range(10)) - D(1) / gamma(t)) for t in trees(k))
        rh = max(abs(mp.fsum(bhat[j] * phi(t)[j] for j in range(10)) - D(1) / gamma(t)) for t in trees(k))
        print(f"# order {k}: max residual b {mp.nstr(rb, 3)}  bhat {mp.nstr(rh, 3)}")
    print("btilde = {" + ", ".join(mp.nstr(v, 17, strip_zeros=False) for v in btilde) + "}")


if __name__ == "__main__":
    main()
