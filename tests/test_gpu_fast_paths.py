"""Two shortcuts of the packed fp32 Box–Muller replace IEEE operations
by the hardware's fast-path sequences without their range checks: the log2
polynomial's quotient s = (m − 1)/(m + 1) (R2 / R8, §4) and the radius √x.
Exhaustive checks against IEEE division / sqrt over every fp32 input the method
can produce (-m gpu)."""
import pytest

import paper_2304_06835_b200 as ens

pytestmark = pytest.mark.gpu


def test_fast_paths_equal_ieee_everywhere():
    quot, sqrt = ens.check_fast_paths()
    assert quot == 0, f"log2 quotient differs from IEEE division for {quot} fp32 m"
    assert sqrt == 0, f"Box-Muller sqrt differs from IEEE sqrt for {sqrt} fp32 x"
