"""Bootstrapping linear-transform fixtures from the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden_boot.py

Builds a real reference BootstrapPlan (bootstrap.make_bootstrap_plan, host-
encoded diagonals on the raised basis) and real reference keys (keygen:
compressed rotation keys = b-rows + SHAKE256 seed), then runs the reference's
CoeffToSlot entry (drop_limbs + raise_modulus, bootstrap.py:316-318) and every
CoeffToSlot / SlotToCoeff pt_matvec stage (bootstrap.py:320-332) on seeded
ciphertexts.  Everything the GPU test needs is written to
tests/golden/boot.npz (+ boot.json): params, inputs, keys, stage diagonals and
the reference output after every step.
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

from paper_2112_06396_b200.digest import digest  # noqa: E402

LOGN, LIMBS, DNUM, SEED = 6, 18, 3, 3
RADICES, DEGREE, DOUBLINGS = (4, 8), 63, 5


def _ct(mods, rng, delta):
    n = 1 << LOGN
    a = np.stack([rng.integers(0, q, n, dtype=np.uint64) for q in mods])
    b = np.stack([rng.integers(0, q, n, dtype=np.uint64) for q in mods])
    return ckks.Ciphertext(rnspoly.RnsPoly(tuple(mods), a, "eval"),
                           rnspoly.RnsPoly(tuple(mods), b, "eval"), delta)


def main():
    p = ckks.make_params(logn=LOGN, limbs=LIMBS, dnum=DNUM, seed=SEED)
    plan = bootstrap.make_bootstrap_plan(p, radices=RADICES, degree=DEGREE,
                                         doublings=DOUBLINGS, input_limbs=1)
    keys = ckks.keygen(p, rotations=plan.rotations, need_conj=True)
    rng = np.random.default_rng(2024)
    arrs, meta = {}, {"logn": LOGN, "chain": [int(q) for q in p.chain],
                      "special": [int(q) for q in p.special], "dnum": DNUM,
                      "delta": p.delta, "seed": SEED, "rotations": list(plan.rotations),
                      "cts": [], "stc": []}
    seed_root = p.seed.to_bytes(8, "little")
    for r in plan.rotations:
        k = keys.rot[r]
        assert k.compressed and k.seed == b"rot%d" % (r % (2 * p.n_ring)) + seed_root
        arrs[f"key_b/{r}"] = k.b
    # CoeffToSlot entry + stages
    ct = _ct(p.chain[:1], rng, p.delta)
    arrs["cts_in/a"], arrs["cts_in/b"] = ct.a.data, ct.b.data
    x = ckks.raise_modulus(p, ckks.drop_limbs(ct, plan.input_limbs), p.limbs)
    arrs["raised/a"], arrs["raised/b"] = x.a.data, x.b.data
    for si, st in enumerate(plan.cts):
        assert x.limbs == st.entry_limbs
        offs = sorted(st.diags)
        for o in offs:
            arrs[f"cts{si}/diag/{o}"] = st.diags[o].data
        x = ckks.pt_matvec(p, keys, x, st.diags, st.diag_delta)
        arrs[f"cts{si}/out/a"], arrs[f"cts{si}/out/b"] = x.a.data, x.b.data
        meta["cts"].append({"entry_limbs": st.entry_limbs, "diag_delta": st.diag_delta,
                            "offsets": offs, "digest": digest(x.a.data, x.b.data),
                            "delta": x.delta})
    # SlotToCoeff stages on a seeded ciphertext at the STC entry level
    y = _ct(p.chain[:plan.stc[0].entry_limbs], rng, p.delta)
    arrs["stc_in/a"], arrs["stc_in/b"] = y.a.data, y.b.data
    for si, st in enumerate(plan.stc):
        offs = sorted(st.diags)
        for o in offs:
            arrs[f"stc{si}/diag/{o}"] = st.diags[o].data
        y = ckks.pt_matvec(p, keys, y, st.diags, st.diag_delta)
        arrs[f"stc{si}/out/a"], arrs[f"stc{si}/out/b"] = y.a.data, y.b.data
        meta["stc"].append({"entry_limbs": st.entry_limbs, "diag_delta": st.diag_delta,
                            "offsets": offs, "digest": digest(y.a.data, y.b.data),
                            "delta": y.delta})
    # the conjugation between the stages (bootstrap.py:322)
    cj = ckks.conjugate(p, keys, x)
    arrs["conj/a"], arrs["conj/b"] = cj.a.data, cj.b.data
    arrs["key_b/conj"] = keys.conj.b
    np.savez_compressed(os.path.join(HERE, "boot.npz"), **arrs)
    json.dump(meta, open(os.path.join(HERE, "boot.json"), "w"), indent=1)
    print("rotations", len(plan.rotations), "cts", [len(s.diags) for s in plan.cts],
          "stc", [len(s.diags) for s in plan.stc],
          "bytes", os.path.getsize(os.path.join(HERE, "boot.npz")))


if __name__ == "__main__":
    main()
