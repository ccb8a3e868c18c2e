"""Pins for the oracle's SDE noise stream (DESIGN R8): one normal stream per
trajectory, consumed nw normals per step with nothing dropped, each Philox
call's words feeding Box–Muller pairs in the stated order."""
import math

import numpy as np
import pytest

import oracle

SEED, G = 0x5EED5EED1234, (1 << 35) + 77


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_steps_concatenate_one_stream(dtype):
    """Step s with nw increments reads Z_{nw·s} … Z_{nw·s+nw−1}: the nw = 3 and
    nw = 8 views are re-slicings of the nw = 1 stream, from any start step."""
    z1 = oracle.normals(SEED, G, 0, 96, dtype, nw=1).ravel()
    np.testing.assert_array_equal(oracle.normals(SEED, G, 0, 32, dtype, nw=3).ravel(), z1[:96])
    np.testing.assert_array_equal(oracle.normals(SEED, G, 0, 12, dtype, nw=8).ravel(), z1[:96])
    np.testing.assert_array_equal(oracle.normals(SEED, G, 5, 7, dtype, nw=3).ravel(), z1[15:36])


@pytest.mark.parametrize("dtype,per", [("f32", 4), ("f64", 2)])
def test_call_to_pairs_mapping(dtype, per):
    """Call c (counter (c lo, g lo, g hi, c hi)) gives Z_{per·c…}: each pair's
    R² = Z_cos² + Z_sin² equals −2 ln U of the pair's first uniform, and the
    angle is 2π times its second uniform."""
    z = oracle.normals(SEED, G, 0, 8 * per, dtype, nw=1).ravel().astype(np.float64)
    key = [SEED & 0xFFFFFFFF, SEED >> 32]
    tol = 2e-6 if dtype == "f32" else 1e-13
    for c in [0, 1, 5]:
        w = oracle.philox([c, G & 0xFFFFFFFF, G >> 32, 0], key)
        U = oracle.uniforms(w, dtype).astype(np.float64)
        pairs = [(U[0], U[1]), (U[2], U[3])] if dtype == "f32" else [(U[0], U[1])]
        for q, (ua, ub) in enumerate(pairs):
            zc, zs = z[per * c + 2 * q], z[per * c + 2 * q + 1]
            assert abs(zc * zc + zs * zs - (-2.0 * math.log(ua))) <= tol * max(1.0, -2.0 * math.log(ua))
            ang = math.atan2(zs, zc) % (2 * math.pi)
            assert abs(ang - 2 * math.pi * ub) <= 1e2 * tol or abs(abs(ang - 2 * math.pi * ub) - 2 * math.pi) <= 1e2 * tol
