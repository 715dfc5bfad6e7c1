"""the oracle's new_mult family against the reference's own
outputs (tests/golden/make_golden_polyeval.py) -- plain, value_mult + const,
negative/positive addend lifts, classic mult, and the first doubling and
T_3 = 2 T_2 T_1 - T_1 of the Chebyshev basis."""

import numpy as np
import pytest

from boot_fixture import Boot
from oracle import ckks_np
from polyeval_fixture import PolyEval

B, E = Boot(), PolyEval()
P = B.params
RELIN = (E.z["relin/b"], E.z["relin/a"])


def _const(c: float, delta: float, lim: int):
    v = round(c * delta)
    return [v % q for q in P.chain[:lim]]


def _lift(d_prod: float, d_add: float, sign: int) -> int:
    return sign * round(d_prod / d_add)


@pytest.mark.parametrize("case", ["nm_plain", "nm_vm_const", "nm_addend_neg", "nm_addend_pos"])
def test_new_mult_cases(case):
    c1, c2, ad = E.pair("u_c1"), E.pair("u_c2"), E.pair("u_ad")
    d1, d2, dad = E.delta("u_c1"), E.delta("u_c2"), E.delta("u_ad")
    if case == "nm_plain":
        got = ckks_np.new_mult(P, c1, c2, RELIN)
    elif case == "nm_vm_const":
        got = ckks_np.new_mult(P, c1, c2, RELIN, value_mult=2, const_residues=_const(-1.0, d1 * d2, 8))
    elif case == "nm_addend_neg":
        got = ckks_np.new_mult(P, c1, c2, RELIN, value_mult=2,
                               addend=(ad[0], ad[1], _lift(d1 * d2, dad, -1)))
    else:
        got = ckks_np.new_mult(P, c1, c1, RELIN, addend=(ad[0], ad[1], _lift(d1 * d1, dad, 1)))
    want = E.pair(case)
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_classic_mult():
    c1 = tuple(x[:8] for x in E.pair("u_c1"))
    got = ckks_np.mult(P, c1, E.pair("u_c2"), RELIN)
    want = E.pair("mult")
    assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_chebyshev_basis_first_steps():
    t1, d1 = E.pair("T1"), E.delta("T1")
    lim = t1[0].shape[0]
    t2 = ckks_np.new_mult(P, t1, t1, RELIN, value_mult=2, const_residues=_const(-1.0, d1 * d1, lim))
    assert np.array_equal(t2[0], E.pair("T2")[0]) and np.array_equal(t2[1], E.pair("T2")[1])
    d2 = E.delta("T2")
    t3 = ckks_np.new_mult(P, t2, t1, RELIN, value_mult=2,
                          addend=(t1[0], t1[1], _lift(d2 * d1, d1, -1)))
    assert np.array_equal(t3[0], E.pair("T3")[0]) and np.array_equal(t3[1], E.pair("T3")[1])
