#!/usr/bin/env python
"""Derive the Verner embedded-error weights b̃ = b − b̂ (DESIGN R21).

The main weights b, the nodes c and the matrix A are Verner's published "most
efficient" 7(6) and 9(8) pairs (P:319-320 names GPUVern7 / GPUVern9; the
paper prints no coefficients). The embedded weights b̂ (order p−1) are fixed
here from the order conditions: b̂ − b must satisfy every homogeneous
condition of order ≤ p−1 (37 / 200 rooted trees), which on these stages leaves
exactly one direction δ; its scale is fixed by the structural zeros of
Verner's embedded weights — b̂8 = b̂9 = 0 for the 7(6) pair, b̂14 = b̂15 = 0 for
the 9(8) pair (1-based): the scale is solved from the first zero and the second
must then vanish too, an independent check of the direction δ. Prints b̃ to 17
significant digits (the literals in oracle/oracle.cpp and csrc/verner.cuh),
the implied b̂1 and the residuals. Uses mpmath at 50 digits; no oracle / library code.
Usage: python tools/derive_verner_embedded.py [7|9]
"""
import mpmath as mp

mp.mp.dps = 50
D = mp.mpf
C7 = [D(0), D("0.005"), D("0.10888888888888888"), D("0.16333333333333333"), D("0.4555"),
     D("0.6095094489978381"), D("0.884"), D("0.925"), D(1), D(1)]
ROWS7 = {
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
B7 = {0: "0.04715561848627222", 3: "0.25750564298434153", 4: "0.2621665397741262", 5: "0.15216092656738558",
      6: "0.4939969170032485", 7: "-0.29430311714032503", 8: "0.08131747232495111"}

# Vern9: 16 stages (0-based rows / columns), zero columns 1..6 beyond row 7
C9 = [D(0), D("0.03462"), D("0.09702435063878045"), D("0.14553652595817068"), D("0.561"),
      D("0.22900791159048503"), D("0.544992088409515"), D("0.645"), D("0.48375"), D("0.06757"), D("0.25"),
      D("0.6590650618730999"), D("0.8206"), D("0.9012"), D(1), D(1)]
ROWS9 = {
    1: {0: "0.03462"},
    2: {0: "-0.0389335438857287", 1: "0.13595789452451916"},
    3: {0: "0.03638413148954267", 2: "0.10915239446862801"},
    4: {0: "2.0257639143939694", 2: "-7.638023836496292", 3: "6.173259922102322"},
    5: {0: "0.05112275589406061", 3: "0.17708237945550218", 4: "0.0008027762409222536"},
    6: {0: "0.13160063579752163", 3: "-0.2957276252669636", 4: "0.08781378035642955", 5: "0.6213052975225274"},
    7: {0: "0.07166666666666667", 5: "0.33055335789153195", 6: "0.2427799754418014"},
    8: {0: "0.071806640625", 5: "0.3294380283228177", 6: "0.1165190029271823", 7: "-0.034013671875"},
    9: {0: "0.04836757646340646", 5: "0.03928989925676164", 6: "0.10547409458903446", 7: "-0.021438652846483126",
        8: "-0.10412291746271944"},
    10: {0: "-0.026645614872014785", 5: "0.03333333333333333", 6: "-0.1631072244872467", 7: "0.03396081684127761",
         8: "0.1572319413814626", 9: "0.21522674780318796"},
    11: {0: "0.03689009248708622", 5: "-0.1465181576725543", 6: "0.2242577768172024", 7: "0.02294405717066073",
         8: "-0.0035850052905728597", 9: "0.08669223316444385", 10: "0.43838406519683376"},
    12: {0: "-0.4866012215113341", 5: "-6.304602650282853", 6: "-0.2812456182894729", 7: "-2.679019236219849",
         8: "0.5188156639241577", 9: "1.3653531876033418", 10: "5.8850910885039465", 11: "2.8028087862720628"},
    13: {0: "0.4185367457753472", 5: "6.724547581906459", 6: "-0.42544428016461133", 7: "3.3432791530012653",
         8: "0.6170816631175374", 9: "-0.9299661239399329", 10: "-6.099948804751011", 11: "-3.002206187889399",
         12: "0.2553202529443446"},
    14: {0: "-0.7793740861228848", 5: "-13.937342538107776", 6: "1.2520488533793563", 7: "-14.691500408016868",
         8: "-0.494705058533141", 9: "2.2429749091462368", 10: "13.367893803828643", 11: "14.396650486650687",
         12: "-0.79758133317768", 13: "0.4409353709534278"},
    15: {0: "2.0580513374668867", 5: "22.357937727968032", 6: "0.9094981099755646", 7: "35.89110098240264",
         8: "-3.442515027624454", 9: "-4.865481358036369", 10: "-18.909803813543427", 11: "-34.26354448030452",
         12: "1.2647565216956427"},
}
B9 = {0: "0.014611976858423152", 7: "-0.3915211862331339", 8: "0.23109325002895065", 9: "0.12747667699928525",
      10: "0.2246434176204158", 11: "0.5684352689748513", 12: "0.058258715572158275", 13: "0.13643174034822156",
      14: "0.030570139830827976"}

METHODS = {
    7: dict(C=C7, ROWS=ROWS7, B=B7, BHAT_ZERO=(7, 8), zero=(1, 2), norm=7),
    9: dict(C=C9, ROWS=ROWS9, B=B9, BHAT_ZERO=(13, 14), zero=(1, 2, 3, 4, 5, 6), norm=11),
}
A, B, S = None, None, 0


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


def phi(t, memo={}):
    key = (S, t)
    if key not in memo:
        v = [D(1)] * S
        for ch in t:
            w = phi(ch)
            aw = [mp.fsum(A[i][j] * w[j] for j in range(S)) for i in range(S)]
            v = [v[i] * aw[i] for i in range(S)]
        memo[key] = v
    return memo[key]


def main(p: int):
    global A, B, S
    m = METHODS[p]
    S = len(m["C"])
    A = [[D(0)] * S for _ in range(S)]
    for i, r in m["ROWS"].items():
        for j, v in r.items():
            A[i][j] = D(v)
    B = [D(m["B"].get(j, "0")) for j in range(S)]
    conds = [(n, t) for n in range(1, p) for t in trees(n)]
    M = mp.matrix([phi(t) for _, t in conds])
    # δ with δ_norm = −1 and δ = 0 on the stages without weight in b or b̂: least squares in the
    # remaining unknowns (consistent to the literals' rounding)
    cols = [j for j in range(S) if j not in m["zero"] and j != m["norm"]]
    Ms = mp.matrix([[M[r, j] for j in cols] for r in range(M.rows)])
    rhs = mp.matrix([M[r, m["norm"]] for r in range(M.rows)])     # Σ_j M_rj δ_j − M_r,norm = 0
    x = mp.lu_solve(Ms.T * Ms, Ms.T * rhs)
    delta = [D(0)] * S
    for k, j in enumerate(cols):
        delta[j] = x[k]
    delta[m["norm"]] = D(-1)
    res = max(abs(mp.fsum(M[r, j] * delta[j] for j in range(S))) for r in range(M.rows))
    z0, z1 = m["BHAT_ZERO"]
    s = -B[z0] / delta[z0]                       # b̂_z0 = b_z0 + s·δ_z0 = 0
    bhat = [B[j] + s * delta[j] for j in range(S)]
    print(f"# structural zeros: b_hat[{z0 + 1}] = {mp.nstr(bhat[z0], 3)}, b_hat[{z1 + 1}] = {mp.nstr(bhat[z1], 3)}"
          f" (independent check); implied b_hat1 = {mp.nstr(bhat[0], 17)}")
    btilde = [B[j] - bhat[j] for j in range(S)]
    print(f"# Vern{p}: homogeneous residual of delta: {mp.nstr(res, 5)}")
    rowsum = max(abs(mp.fsum(A[i]) - m["C"][i]) for i in range(S))
    print(f"# row-sum residual {mp.nstr(rowsum, 3)}")
    for k in range(1, p + 2):
        rb = max(abs(mp.fsum(B[j] * phi(t)[j] for j in range(S)) - D(1) / gamma(t)) for t in trees(k))
        rh = max(abs(mp.fsum(bhat[j] * phi(t)[j] for j in range(S)) - D(1) / gamma(t)) for t in trees(k))
        print(f"# order {k}: max residual b {mp.nstr(rb, 3)}  bhat {mp.nstr(rh, 3)}")
    print("btilde = {" + ", ".join(mp.nstr(v, 17, strip_zeros=False) for v in btilde) + "}")


if __name__ == "__main__":
    import sys
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
