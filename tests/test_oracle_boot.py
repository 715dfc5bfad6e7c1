"""Bootstrapping linear transforms: the oracle's
raise_modulus / pt_matvec / conjugate against a real reference BootstrapPlan
run by the reference itself (tests/golden/make_golden_boot.py)."""

import numpy as np
import pytest

from boot_fixture import Boot
from oracle import ckks_np

B = Boot()
P = B.params
DIGITS = len(P.digit_spans(P.limbs))


def _keys():
    return {r: (B.key_b(r), ckks_np.expand_key_a(B.key_seed(r), P.full_moduli, DIGITS, P.n_ring))
            for r in B.meta["rotations"]}


KEYS = _keys()


def test_raise_modulus():
    a, b = ckks_np.raise_modulus(P, B.z["cts_in/a"], B.z["cts_in/b"], P.limbs)
    assert np.array_equal(a, B.z["raised/a"]) and np.array_equal(b, B.z["raised/b"])


@pytest.mark.parametrize("kind", ["cts", "stc"])
def test_matvec_stages(kind):
    a, b = (B.z["raised/a"], B.z["raised/b"]) if kind == "cts" else (B.z["stc_in/a"], B.z["stc_in/b"])
    for si, st in enumerate(B.meta[kind]):
        assert a.shape[0] == st["entry_limbs"]
        a, b = ckks_np.pt_matvec(P, a, b, KEYS, B.stage_diags(kind, si))
        assert np.array_equal(a, B.z[f"{kind}{si}/out/a"]), si
        assert np.array_equal(b, B.z[f"{kind}{si}/out/b"]), si


def test_conjugate_between_stages():
    kb = B.z["key_b/conj"]
    ka = ckks_np.expand_key_a(b"conj" + B.seed_root, P.full_moduli, DIGITS, P.n_ring)
    last = len(B.meta["cts"]) - 1
    a, b = ckks_np.conjugate(P, B.z[f"cts{last}/out/a"], B.z[f"cts{last}/out/b"], kb, ka)
    assert np.array_equal(a, B.z["conj/a"]) and np.array_equal(b, B.z["conj/b"])
