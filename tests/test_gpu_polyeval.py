"""SURVEY 8(f) row 3 on the GPU: new_mult's fused variants, the plaintext-
constant ops, the reference's Chebyshev / double-angle sine evaluation and a
full bootstrap(), all bit-exact against the reference's own outputs
(tests/golden/make_golden_polyeval.py; plan and keys as tests/golden/boot.npz,
rotation/conjugation keys expanded from their seeds on the device)."""

import numpy as np
import pytest

from boot_fixture import Boot
from paper_2112_06396_b200 import bootstrap as boot
from paper_2112_06396_b200 import ckks
from paper_2112_06396_b200.device import to_host
from paper_2112_06396_b200.rnspoly import RnsPoly
from polyeval_fixture import PolyEval

pytestmark = pytest.mark.gpu

B, E = Boot(), PolyEval()
P = B.params


def _keys():
    full = P.full_moduli
    rot = {r: ckks.SwitchingKey(full, B.key_b(r), seed=B.key_seed(r)) for r in B.meta["rotations"]}
    conj = ckks.SwitchingKey(full, B.z["key_b/conj"], seed=b"conj" + B.seed_root)
    relin = ckks.SwitchingKey(full, E.z["relin/b"], a=E.z["relin/a"])
    return ckks.KeySet(P, None, relin, rot=rot, conj=conj)


@pytest.fixture(scope="module")
def keys():
    return _keys()


def _ct(name):
    a, b = E.pair(name)
    mods = P.chain[:a.shape[0]]
    return ckks.Ciphertext(RnsPoly(mods, a, "eval"), RnsPoly(mods, b, "eval"), E.delta(name))


def _eq(ct, name):
    a, b = E.pair(name)
    ok = np.array_equal(to_host(ct.a.data), a) and np.array_equal(to_host(ct.b.data), b)
    return ok and ct.delta == E.delta(name)


def _stages(kind):
    out = []
    for si, st in enumerate(B.meta[kind]):
        raised = P.raised_moduli(st["entry_limbs"])
        d = {o: RnsPoly(raised, m, "eval") for o, m in B.stage_diags(kind, si).items()}
        out.append(ckks.MatvecStage(d, st["diag_delta"], st["entry_limbs"]))
    return out


def _plan():
    m = E.meta
    return boot.BootstrapPlan(P, m["doublings"], m["degree"], E.z["cheb"], m["const_shift"],
                              _stages("cts"), _stages("stc"), m["input_limbs"], m["output_limbs"])


def test_new_mult_variants(keys):
    c1, c2, ad = _ct("u_c1"), _ct("u_c2"), _ct("u_ad")
    assert _eq(ckks.new_mult(P, keys, c1, c2), "nm_plain")
    assert _eq(ckks.new_mult(P, keys, c1, c2, value_mult=2, const=-1.0), "nm_vm_const")
    assert _eq(ckks.new_mult(P, keys, c1, c2, value_mult=2, addend=ad, addend_sign=-1),
               "nm_addend_neg")
    assert _eq(ckks.new_mult(P, keys, c1, c1, addend=ad, addend_sign=1), "nm_addend_pos")
    assert _eq(ckks.mult(P, keys, ckks.drop_limbs(c1, 8), c2), "mult")


def test_constant_ops():
    c1, c2, ad = _ct("u_c1"), _ct("u_c2"), _ct("u_ad")
    assert _eq(ckks.const_add(P, c1, 0.3125), "const_add")
    assert _eq(ckks.mult_monomial(P, c1, 5), "mult_monomial")
    assert _eq(ckks.const_mult_int(c1, -3), "const_mult_int")
    assert _eq(ckks.pt_combo(P, [(c1, 0.75), (c2, -1.5), (ad, 2.0 ** -7)], 0.125), "pt_combo")


def test_chebyshev_basis_and_sine_eval(keys):
    plan = _plan()
    lo = _ct("lo")
    ct_w = ckks.const_add(P, lo, plan.const_shift)
    assert _eq(ct_w, "ct_w")
    ev = boot.ChebEvaluator(P, keys, ct_w, plan.degree)
    assert sorted(ev.t) == sorted(int(k[1:-2]) for k in E.z.files if k.startswith("T") and k.endswith("/a"))
    for k, t in ev.t.items():
        assert _eq(t, f"T{k}"), k
    out = ev.run(plan.cheb)
    assert _eq(out, "cheb_out")
    for i in range(plan.doublings):
        out = ev._double(out)
        assert _eq(out, f"dbl{i}"), i
    assert _eq(boot.sine_eval(P, keys, plan, _ct("hi")), "sine_hi")


def test_full_bootstrap(keys):
    out = boot.bootstrap(P, keys, _plan(), _ct("boot_in"))
    assert out.limbs == E.meta["output_limbs"]
    assert _eq(out, "boot_out")
