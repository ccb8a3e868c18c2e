"""Weak convergence on the GPU (-m gpu; SPEC acceptance 6):
GBM dX = rX dt + VX dW (r = 1.5, V = 0.01, X0 = 0.1, T = 1), 2^21
paths per step size, fused ensemble means. The error of the mean against the
exact E[X_T] = X0·e^{rT} falls with slope ≈ 1 for Euler–Maruyama and ≈ 2 for
SIEA, and the finest EM mean is within its bias + 3 standard errors."""
import math

import numpy as np
import pytest

from tests.helpers import gpu

pytestmark = pytest.mark.gpu

X0, R, V, T = 0.1, 1.5, 0.01, 1.0
EXACT = X0 * math.exp(R * T)
N = 1 << 21


def _mean(alg, h):
    u0 = np.full((3, N), X0)
    _, rc, _, _, st = gpu("gbm", alg, u0, np.array([R, V]), (0.0, T), h, seed=7, stats=True, store_states=False)
    assert (rc == 0).all()
    return st[0, :, 1].mean(), st[0, :, 2].mean() / (N - 1)      # the 3 components are independent copies


@pytest.mark.parametrize("alg,hs,lo,hi", [("em", [2.0**-4, 2.0**-5, 2.0**-6, 2.0**-7], 0.8, 1.2),
                                         ("siea", [2.0**-2, 2.0**-3, 2.0**-4], 1.7, 2.3)])
def test_weak_order_slope(alg, hs, lo, hi):
    errs = [abs(_mean(alg, h)[0] - EXACT) for h in hs]
    slopes = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all((slopes > lo) & (slopes < hi)), (alg, errs, slopes)


def test_em_mean_within_bias_and_standard_error():
    h = 2.0**-7
    m, var = _mean("em", h)
    bias = X0 * ((1 + R * h) ** round(T / h)) - EXACT          # the scheme's exact discrete mean − E[X_T]
    se = math.sqrt(var / (3 * N))
    assert abs(m - EXACT - bias) < 3 * se, (m, EXACT, bias, se)
