"""Sine-evaluation (PolyEval) and full-bootstrap fixtures from the REFERENCE
(new_mult-based Chebyshev / double-angle evaluation).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_polyeval.py

Same reference BootstrapPlan and keygen as make_golden_boot.py (N=64, L=18,
radices (4, 8), degree 63, 5 doublings), plus the reference's relinearisation
key (expanded, ckks.py:304-305).  Records, all computed by the reference:
  * the Chebyshev basis T_k of _ChebEvaluator.__init__ (bootstrap.py:173-186)
    on ct_w = const_add(lo, const_shift) (bootstrap.py:292),
  * the BSGS Chebyshev output (bootstrap.py:197-210) and every double-angle
    step (bootstrap.py:295-296), i.e. _sine_eval(lo),
  * _sine_eval(hi) and the full bootstrap() output (bootstrap.py:300-333),
  * small unit cases of new_mult's fused variants, pt_combo, const_add,
    mult_monomial and const_mult_int (ckks.py:510-652).
Written to tests/golden/polyeval.npz + polyeval.json.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from ckkslab import bootstrap, ckks, rnspoly  # noqa: E402  (the reference)

LOGN, LIMBS, DNUM, SEED = 6, 18, 3, 3
RADICES, DEGREE, DOUBLINGS = (4, 8), 63, 5


def _ct(mods, rng, delta):
    n = 1 << LOGN
    a = np.stack([rng.integers(0, q, n, dtype=np.uint64) for q in mods])
    b = np.stack([rng.integers(0, q, n, dtype=np.uint64) for q in mods])
    return ckks.Ciphertext(rnspoly.RnsPoly(tuple(mods), a, "eval"),
                           rnspoly.RnsPoly(tuple(mods), b, "eval"), delta)


def _put(arrs, name, ct):
    arrs[name + "/a"], arrs[name + "/b"] = ct.a.data, ct.b.data


def main():
    p = ckks.make_params(logn=LOGN, limbs=LIMBS, dnum=DNUM, seed=SEED)
    plan = bootstrap.make_bootstrap_plan(p, radices=RADICES, degree=DEGREE,
                                         doublings=DOUBLINGS, input_limbs=1)
    keys = ckks.keygen(p, rotations=plan.rotations, need_conj=True)
    assert not keys.relin.compressed
    arrs = {"relin/b": keys.relin.b, "relin/a": keys.relin.a, "cheb": plan.cheb}
    meta = {"const_shift": plan.const_shift, "doublings": plan.doublings,
            "degree": plan.degree, "input_limbs": plan.input_limbs,
            "output_limbs": plan.output_limbs, "deltas": {}}

    # --- the sine evaluation on the real post-CoeffToSlot halves
    rng = np.random.default_rng(2024)
    ct = _ct(p.chain[:1], rng, p.delta)          # = make_golden_boot's cts_in
    _put(arrs, "boot_in", ct)
    meta["deltas"]["boot_in"] = ct.delta
    x = ckks.raise_modulus(p, ckks.drop_limbs(ct, plan.input_limbs), p.limbs)
    for st in plan.cts:
        x = ckks.pt_matvec(p, keys, x, st.diags, st.diag_delta)
    cj = ckks.conjugate(p, keys, x)
    lo = ckks.add(x, cj)
    hi = ckks.negate(ckks.mult_monomial(p, ckks.sub(x, cj), p.n_ring // 2))
    _put(arrs, "lo", lo)
    _put(arrs, "hi", hi)
    meta["deltas"]["lo"] = lo.delta
    meta["deltas"]["hi"] = hi.delta

    ct_w = ckks.const_add(p, lo, plan.const_shift)
    _put(arrs, "ct_w", ct_w)
    meta["deltas"]["ct_w"] = ct_w.delta
    ev = bootstrap._ChebEvaluator(p, keys, ct_w, plan.degree)
    for k, t in ev.t.items():
        _put(arrs, f"T{k}", t)
        meta["deltas"][f"T{k}"] = t.delta
    out = ev.run(plan.cheb)
    _put(arrs, "cheb_out", out)
    meta["deltas"]["cheb_out"] = out.delta
    for i in range(plan.doublings):
        out = ev._double(out)
        _put(arrs, f"dbl{i}", out)
        meta["deltas"][f"dbl{i}"] = out.delta
    sine_hi = bootstrap._sine_eval(p, keys, plan, hi)
    _put(arrs, "sine_hi", sine_hi)
    meta["deltas"]["sine_hi"] = sine_hi.delta

    full = bootstrap.bootstrap(p, keys, plan, ct)
    _put(arrs, "boot_out", full)
    meta["deltas"]["boot_out"] = full.delta

    # --- unit cases of the fused multiply and the plaintext-constant ops
    rng = np.random.default_rng(77)
    c1 = _ct(p.chain[:9], rng, p.delta)
    c2 = _ct(p.chain[:8], rng, p.delta * 1.0000001)
    ad = _ct(p.chain[:10], rng, p.delta * 0.999)
    for name, c in (("u_c1", c1), ("u_c2", c2), ("u_ad", ad)):
        _put(arrs, name, c)
        meta["deltas"][name] = c.delta
    cases = {
        "nm_plain": ckks.new_mult(p, keys, c1, c2),
        "nm_vm_const": ckks.new_mult(p, keys, c1, c2, value_mult=2, const=-1.0),
        "nm_addend_neg": ckks.new_mult(p, keys, c1, c2, value_mult=2, addend=ad,
                                       addend_sign=-1),
        "nm_addend_pos": ckks.new_mult(p, keys, c1, c1, addend=ad, addend_sign=1),
        "mult": ckks.mult(p, keys, ckks.drop_limbs(c1, 8), c2),
        "const_add": ckks.const_add(p, c1, 0.3125),
        "mult_monomial": ckks.mult_monomial(p, c1, 5),
        "const_mult_int": ckks.const_mult_int(c1, -3),
        "pt_combo": ckks.pt_combo(p, [(c1, 0.75), (c2, -1.5), (ad, 2.0 ** -7)], 0.125),
    }
    for name, c in cases.items():
        _put(arrs, name, c)
        meta["deltas"][name] = c.delta
    np.savez_compressed(os.path.join(HERE, "polyeval.npz"), **arrs)
    json.dump(meta, open(os.path.join(HERE, "polyeval.json"), "w"), indent=1)
    print("T keys", sorted(ev.t), "out limbs", full.limbs,
          "bytes", os.path.getsize(os.path.join(HERE, "polyeval.npz")))


if __name__ == "__main__":
    main()
