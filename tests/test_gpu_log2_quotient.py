"""The fp32 log2 polynomial's quotient s = (m − 1)/(m + 1) (DESIGN R2 / R8, §4:
an IEEE division) is computed on the GPU by reciprocal + refinement without the
division's range check. Exhaustive check over every fp32 m the
polynomial can see, scalar and packed forms (-m gpu)."""
import pytest

import paper_2304_06835_b200 as ens

pytestmark = pytest.mark.gpu


def test_log2_quotient_equals_ieee_division_everywhere():
    assert ens.check_log2_quotient() == 0
