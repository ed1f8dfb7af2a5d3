"""phub_hier_beneficial -- the paper's benefit model for hierarchical reduction
 -- against hand-computed cases (-m "not gpu"; the entry
point is host-only).  tests/golden/hier_model_cases.txt holds the cases with
their arithmetic; each checks lhs, rhs and the decision, so a wrong B_bn, a
dropped or swapped C, or a non-strict comparison fails at least one."""
from fractions import Fraction

import pytest

from conftest import read_golden


def _cases():
    return read_golden("hier_model_cases.txt")


@pytest.mark.parametrize("row", _cases(), ids=lambda r: r[0])
def test_benefit_model_golden(row):
    from paper_1805_07891_b200 import capi
    name, N, r, bp, bw, bc, mode, _bbn, lhs, rhs, ben = row
    m = capi.PHUB_CROSS_RACK_SHARDED if mode == "sharded" else capi.PHUB_CROSS_RACK_RING
    got_ben, got_l, got_r = capi.phub_hier_beneficial(int(N), int(r), float(bp), float(bw),
                                                      float(bc), m)
    assert got_ben == bool(int(ben)), name
    assert got_l == pytest.approx(float(Fraction(lhs)), rel=1e-12), name
    assert got_r == pytest.approx(float(Fraction(rhs)), rel=1e-12), name


@pytest.mark.parametrize("args", [
    (0, 2, 1.0, 1.0, 1.0, 0), (4, 1, 1.0, 1.0, 1.0, 0), (4, 2, 0.0, 1.0, 1.0, 0),
    (4, 2, 1.0, float("inf"), 1.0, 0), (4, 2, 1.0, 1.0, -3.0, 0), (4, 2, 1.0, 1.0, 1.0, 7)])
def test_benefit_model_validation(args):
    from paper_1805_07891_b200 import PhubError, capi
    with pytest.raises(PhubError) as e:
        capi.phub_hier_beneficial(*args)
    assert capi.STATUS_NAMES[e.value.status] == "PHUB_ERR_INVALID_ARGUMENT"
