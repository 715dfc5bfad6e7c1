"""Bootstrapping linear transforms on the GPU: a real
reference BootstrapPlan (host-encoded diagonals) and reference keygen keys
(compressed rotation keys, expanded on the device) through raise_modulus,
every CoeffToSlot / SlotToCoeff pt_matvec stage and the conjugation,
bit-exact against the reference's own outputs (tests/golden/boot.npz)."""

import numpy as np
import pytest

from boot_fixture import Boot
from paper_2112_06396_b200 import ckks
from paper_2112_06396_b200.device import to_host
from paper_2112_06396_b200.rnspoly import RnsPoly

pytestmark = pytest.mark.gpu

B = Boot()
P = B.params


def _keys():
    full = P.full_moduli
    rot = {r: ckks.SwitchingKey(full, B.key_b(r), seed=B.key_seed(r)) for r in B.meta["rotations"]}
    conj = ckks.SwitchingKey(full, B.z["key_b/conj"], seed=b"conj" + B.seed_root)
    return ckks.KeySet(P, None, None, rot=rot, conj=conj)


def _ct(a, b, delta=None):
    mods = P.chain[:a.shape[0]]
    return ckks.Ciphertext(RnsPoly(mods, a, "eval"), RnsPoly(mods, b, "eval"),
                           P.delta if delta is None else delta)


def _stages(kind):
    out = []
    for si, st in enumerate(B.meta[kind]):
        raised = P.raised_moduli(st["entry_limbs"])
        d = {o: RnsPoly(raised, m, "eval") for o, m in B.stage_diags(kind, si).items()}
        out.append(ckks.MatvecStage(d, st["diag_delta"], st["entry_limbs"]))
    return out


def _eq(ct, a, b):
    return np.array_equal(to_host(ct.a.data), a) and np.array_equal(to_host(ct.b.data), b)


def test_coeff_to_slot_and_slot_to_coeff_match_reference():
    keys = _keys()
    x = ckks.coeff_to_slot_entry(P, _ct(B.z["cts_in/a"], B.z["cts_in/b"]), 1)
    assert _eq(x, B.z["raised/a"], B.z["raised/b"])
    for si, st in enumerate(_stages("cts")):
        x = ckks.matvec_stages(P, keys, x, [st])
        assert _eq(x, B.z[f"cts{si}/out/a"], B.z[f"cts{si}/out/b"]), si
        assert x.delta == B.meta["cts"][si]["delta"]
    cj = ckks.conjugate(P, keys, x)
    assert _eq(cj, B.z["conj/a"], B.z["conj/b"])
    y = ckks.matvec_stages(P, keys, _ct(B.z["stc_in/a"], B.z["stc_in/b"]), _stages("stc"))
    last = len(B.meta["stc"]) - 1
    assert _eq(y, B.z[f"stc{last}/out/a"], B.z[f"stc{last}/out/b"])
